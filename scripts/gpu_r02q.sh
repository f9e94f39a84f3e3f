# Bounded-forward exp split (FMA-pipe polynomial pairs per 8: 1/2/3/4) A/B, and e2e chunking (8 vs 16 heads).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02q
mkdir -p $O
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C5:32768:64:causal,full;C5:131072:128:causal_document" $PWD/ablibs/bnd3.so $PWD/ablibs/bp1.so $PWD/ablibs/bp2.so $PWD/ablibs/bp4.so --rounds 5 --fwd-only > $O/ab_poly.jsonl 2>&1
cat $O/ab_poly.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
for hg in 8 16 8 16; do
  FM_E2E_HEADS=$hg timeout -s KILL 600 python bench.py --sweep none --cpu-budget 0.5 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('heads $hg', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
