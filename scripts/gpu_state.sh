# State check: GPU tests, smoke, default bench, C5 per-family sweep (kernel times), C4 bench.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
timeout -s KILL 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
for cfg in C5:8192:128 C5:32768:128 C5:131072:128 C5:8192:64 C5:32768:64 C5:131072:64; do
  echo "== $cfg"; timeout -s KILL 600 python scripts/time_kernels.py $cfg 3 2>&1 | grep -v Warn
done 2>&1 | tee gpurun_out/c5_sweep.txt
timeout -s KILL 900 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --cpu-budget 3 2>&1 | tail -1 | tee gpurun_out/bench_c4.json
