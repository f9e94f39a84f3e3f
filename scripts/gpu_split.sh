cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
