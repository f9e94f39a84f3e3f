# Quick check: GPU tests + C2/C3 bench lines (kernel split)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 600 python bench.py --config C2 --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], d['fwd_tflops_kernel'], d['bwd_tflops_kernel'], d['kernels_ms_per_step'], d['clocks'])"
timeout -s KILL 600 python bench.py --no-e2e --cpu-budget 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['fwd_tflops_kernel'], d['bwd_tflops_kernel'], d['kernels_ms_per_step'], d['clocks'])"
