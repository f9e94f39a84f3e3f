# K4: dS^T copied to shared memory by the dQ warpgroup (DS_BY_DQ) — tests + A/B against the previous scheme.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02u
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lpt.py -m gpu -x -q -p no:cacheprovider > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction,sliding_window;C2;C5:131072:128:causal_document" $PWD/ablibs/dsold.so $PWD/ablibs/dsnew.so --rounds 5 > $O/ab_ds.jsonl 2>&1
cat $O/ab_ds.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k].get('bwd_tf')}\" for k in ks))"
