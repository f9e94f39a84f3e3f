# K2b (CTA-pair forward) with the bounded single pass: tests + A/B against K2a's bounded pass.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02t
mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_fwd_pair.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "bounded or pair" > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,full,document,random_eviction,sliding_window;C5:131072:128:causal_document;C4" libflashmask.so libflashmask.so@8 --rounds 5 --fwd-only > $O/ab_pair.jsonl 2>&1
cat $O/ab_pair.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
