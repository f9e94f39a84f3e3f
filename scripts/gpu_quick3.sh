# Quick check: GPU tests, kernel timings (C3, C5 8K/32K d=128 and 32K d=64), C2 bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
for c in C5:8192:128 C5:32768:128 C5:32768:64; do echo "== $c"; timeout -s KILL 300 python scripts/time_kernels.py $c 3 2>&1 | grep -v Warn; done
timeout -s KILL 600 python bench.py --config C2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], d['fwd_tflops_kernel'], d['bwd_tflops_kernel'], d['kernels_ms_per_step'])"
