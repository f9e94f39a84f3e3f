# Quick check: GPU parity tests + kernel timings on C3 and C5 8K/32K d=128 subsets
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
timeout -s KILL 300 python scripts/time_kernels.py C5:8192:128 3 2>&1 | grep "^causal \|sliding\|^document"
timeout -s KILL 300 python scripts/time_kernels.py C5:32768:64 3 2>&1 | grep "^causal \|sliding\|^document"
