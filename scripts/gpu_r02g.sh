# Session-3 sanity pass at HEAD: GPU tests, smoke, default bench line.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02g
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu_state.txt 2>&1
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee $O/smoke.txt
timeout -s KILL 900 python bench.py > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks','e2e','k1_microbench']})
" 2>&1 | tee $O/bench_summary.txt
