# R33 BND from N = 16K (per-head key bound): full GPU suite, A/B against the pre-R33 build, bench.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02p
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 > $O/pytest_gpu.txt 2>&1
tail -12 $O/pytest_gpu.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C2;C5:32768:64:causal;C5:131072:128:causal_document" $PWD/ablibs/head.so $PWD/ablibs/bnd2.so --rounds 5 --fwd-only > $O/ab_bnd2.jsonl 2>&1
cat $O/ab_bnd2.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
timeout -s KILL 600 python bench.py --sweep none > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks','kernels_ms_per_step','gpu_launches']}, d['e2e']['value'])
"
