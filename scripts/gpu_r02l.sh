# R33 v2 (kmax prefetched one entry ahead, lazy q norm, PARTIAL tiles eligible): tests + forward A/B.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02l
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowwise.py -m gpu -x -q -p no:cacheprovider > $O/pytest_parity.txt 2>&1
tail -3 $O/pytest_parity.txt
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction,qk_sparse;C2;C5:8192:64:causal_document;C5:32768:64:causal,full" $PWD/ablibs/head.so libflashmask.so --rounds 5 --fwd-only > $O/ab_spec.jsonl 2>&1
cat $O/ab_spec.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=list(d.keys()); a=d[ks[2]]; b=d[ks[3]]
  print(d['cfg'], d['mask'], a['fwd_tf'], b['fwd_tf'], b['fwd_ratio'])"
