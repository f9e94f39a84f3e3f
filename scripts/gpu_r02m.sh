# R33 variant isolation (forward only).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02m
mkdir -p $O
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,full;C2" $PWD/ablibs/head.so $PWD/ablibs/v2.so $PWD/ablibs/v2.so@32 $PWD/ablibs/v2np.so $PWD/ablibs/v2um.so $PWD/ablibs/v2npum.so --rounds 4 --fwd-only > $O/ab_iso.jsonl 2>&1
cat $O/ab_iso.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
