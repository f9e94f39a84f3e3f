# Final verification at HEAD: GPU suite, smoke (incl. the bounded forward), default bench line.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02v
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -2 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee $O/smoke.txt
timeout -s KILL 900 python bench.py > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks','gpu_launches']}, d['e2e']['value'], d['roofline']['frac'])
"
