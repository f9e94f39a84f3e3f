# Backward: 32-bit range_bits (no 64-bit interval arithmetic in the compute loop) — tests + A/B.
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "parity or arbitrary or gqa or deterministic" 2>&1 | tail -2
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:random_eviction,causal_document;C5:32768:64:causal,document,random_eviction;C2" $PWD/ablibs/rb_old.so $PWD/ablibs/rb_new.so --rounds 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if not l.startswith('{'): continue
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k].get('bwd_tf')}\" for k in ks))"
