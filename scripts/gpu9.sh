cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -k fp32 2>&1 | tail -15
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
