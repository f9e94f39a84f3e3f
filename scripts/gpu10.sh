cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -6
timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -2
timeout -s KILL 300 python scripts/time_kernels.py C5:8192:128 2 2>&1 | tail -14
