# K2b (FM_FLAG_FWD_PAIR) vs K2a, both with the bounded pass: every Figure-1 family at 32K and 128K, d=128.
cd $GRAFT_REPO_ROOT
timeout -s KILL 2400 python scripts/ab_libs.py "C5:32768:128;C5:131072:128" libflashmask.so libflashmask.so@8 --rounds 3 --fwd-only 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if not l.startswith('{'): continue
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  a,b=d[ks[0]]['fwd_tf'],d[ks[1]]['fwd_tf']
  print(f\"{d['cfg']:14s} {d['mask']:22s} K2a {a:7.1f}  K2b {b:7.1f}  {b/a:5.3f}\")"
