cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_c3.txt
timeout -s KILL 300 python bench.py --config C2 --steps 10 --warmup 3 --no-e2e --cpu-budget 2 2>&1 | tail -2 | tee gpurun_out/bench_c2.txt
