cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/abbwd
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:64:causal,document;C5:8192:64:causal_document,sliding_window;C5:131072:64:causal_document" libflashmask_head.so libflashmask.so --rounds 4 > $O/ab.jsonl 2>&1
cat $O/ab.jsonl
