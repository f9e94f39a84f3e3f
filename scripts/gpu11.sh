cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 300 python scripts/trace_fwd.py C3 2>&1 | tail -45
