# R33 v3 (UNMASKED tiles, kmax one entry ahead, conflict-free lazy q norm) vs head, forward only.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02n
mkdir -p $O
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,full,random_eviction;C2;C5:8192:64:causal_document;C5:32768:64:full" $PWD/ablibs/head.so $PWD/ablibs/v3.so $PWD/ablibs/v3.so@32 --rounds 5 --fwd-only > $O/ab_v3.jsonl 2>&1
cat $O/ab_v3.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
