# BND row sum from the bf16-rounded P: precision on the peaked row-wise case + forward A/B.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02y
mkdir -p $O
timeout -s KILL 300 python scripts/rwcheck_tmp.py 2>&1 | tail -8
timeout -s KILL 600 python -m pytest tests/test_gpu_rowwise.py tests/test_gpu_parity.py tests/test_gpu_fwd_pair.py -m gpu -q -p no:cacheprovider -k "bounded" 2>&1 | tail -2
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C5:32768:64:causal;C5:131072:128:causal_document" $PWD/ablibs/pre_rs.so $PWD/ablibs/rs.so --rounds 5 --fwd-only > $O/ab_rs.jsonl 2>&1
cat $O/ab_rs.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
