cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal,full" $PWD/ablibs/h96.so $PWD/ablibs/h64.so --rounds 6 --fwd-only 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if not l.startswith('{'): continue
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
