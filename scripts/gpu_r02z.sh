# Bounded pass headroom 96 / sum threshold 2^-90 (was 64 / 2^-60): GPU suite + forward A/B.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction" $PWD/ablibs/h64.so $PWD/ablibs/h96.so --rounds 4 --fwd-only 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if not l.startswith('{'): continue
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
