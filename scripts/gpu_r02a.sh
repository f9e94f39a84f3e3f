# Round 2, first GPU pass: tests (incl. the new parity / multi-rank tests), smoke, the default
# bench line (sweep + K1 microbench + oracle pool), compute-sanitizer logs.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_state.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
tail -25 gpurun_out/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke.txt
timeout -s KILL 1200 python bench.py > gpurun_out/bench_C3.log 2>&1; tail -1 gpurun_out/bench_C3.log > gpurun_out/bench_C3.json
tail -c 3000 gpurun_out/bench_C3.json
for tool in memcheck synccheck racecheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py all > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_summary.txt
  tail -5 gpurun_out/sanitize_$tool.log
done
