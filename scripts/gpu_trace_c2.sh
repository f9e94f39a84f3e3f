cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 300 python scripts/trace_fwd_cta.py C3 0 2>&1 | tail -17
