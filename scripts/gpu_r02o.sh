# R33 fixed-reference single pass (BND kernels + two-pass fixup): tests, forward A/B, bench.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02o
mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k bounded > $O/pytest_bounded.txt 2>&1
tail -15 $O/pytest_bounded.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,full,random_eviction,qk_sparse;C2;C5:8192:64:causal_document;C5:32768:64:full" $PWD/ablibs/head.so $PWD/ablibs/bnd.so --rounds 5 --fwd-only > $O/ab_bnd.jsonl 2>&1
cat $O/ab_bnd.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowwise.py tests/test_gpu_lpt.py tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider > $O/pytest_more.txt 2>&1
tail -3 $O/pytest_more.txt
timeout -s KILL 600 python bench.py --sweep none > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks','kernels_ms_per_step']}, d['e2e']['value'])
"
