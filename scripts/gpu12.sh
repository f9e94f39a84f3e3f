cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
timeout -s KILL 300 python scripts/time_kernels.py C3 2 --det 2>&1 | tail -1
timeout -s KILL 300 python scripts/time_kernels.py C5:8192:128 2 2>&1
timeout -s KILL 300 python scripts/time_kernels.py C5:8192:64 2 2>&1 | head -4
