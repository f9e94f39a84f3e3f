# R33 bounded single pass: GPU suite, forward A/B against the pre-change build, bench lines.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02k
mkdir -p $O
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k bounded > $O/pytest_bounded.txt 2>&1
tail -3 $O/pytest_bounded.txt
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction,full;C2;C5:8192:64:causal_document;C5:32768:64:causal,full" $PWD/ablibs/head.so libflashmask.so --rounds 5 --fwd-only > $O/ab_spec.jsonl 2>&1
cat $O/ab_spec.jsonl
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout -s KILL 600 python bench.py --sweep none > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks','kernels_ms_per_step']}, d['e2e']['value'])
"
