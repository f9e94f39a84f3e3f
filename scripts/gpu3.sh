cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --cpu-budget 2 2>&1 | tail -3 | tee gpurun_out/bench_c3.txt
