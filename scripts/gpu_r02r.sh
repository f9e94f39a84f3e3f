# Persistent fixup launch (one wave, flagged units only): tests + A/B vs the previous build; BND forced at 8K.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02r
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_lpt.py -m gpu -x -q -p no:cacheprovider > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:sliding_window,share_question,causal;C2;C5:8192:64:causal_document,sliding_window;C5:8192:128:full" $PWD/ablibs/bnd3.so $PWD/ablibs/pfix.so $PWD/ablibs/pfix.so@64 --rounds 5 --fwd-only > $O/ab_pfix.jsonl 2>&1
cat $O/ab_pfix.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); ks=[k for k in d if k not in ('cfg','mask')]
  print(d['cfg'], d['mask'], ' '.join(f\"{k.split('/')[-1]}={d[k]['fwd_tf']}\" for k in ks))"
