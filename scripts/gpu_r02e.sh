cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02e
mkdir -p $O
timeout -s KILL 1500 python scripts/ab_libs.py "C3;C5:32768:128:random_eviction,causal_document,causal;C5:8192:128:causal_document,sliding_window;C2" libflashmask.so libflashmask.so@4 libflashmask_norefine.so --rounds 6 --fwd-only > $O/ab_refine_fwd.jsonl 2>&1
cat $O/ab_refine_fwd.jsonl
