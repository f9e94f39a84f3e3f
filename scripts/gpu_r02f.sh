cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02f
mkdir -p $O
FLASHMASK_LIB=$PWD/paper_2410_01359_b200/libflashmask_dqs.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fwd_bwd_parity or random_config or gqa or deterministic or bf16 or empty or int32" > $O/pytest_dqs.txt 2>&1
tail -3 $O/pytest_dqs.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C5:8192:128:causal_document;C2" libflashmask.so libflashmask_dqs.so --rounds 5 > $O/ab_dqs.jsonl 2>&1
cat $O/ab_dqs.jsonl
timeout -s KILL 900 python scripts/ab_libs.py "C5:32768:128:document,global_sliding_window,prefix_lm_document,prefix_lm_causal;C5:8192:128:document,global_sliding_window" libflashmask.so libflashmask_norefine.so --rounds 5 --fwd-only > $O/ab_refine_noncausal.jsonl 2>&1
cat $O/ab_refine_noncausal.jsonl
