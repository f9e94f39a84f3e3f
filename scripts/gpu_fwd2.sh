# K2b (CTA-pair forward) bring-up: parity tests, then an in-process A/B against K2a.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/fwd2
mkdir -p $O
timeout -s KILL 300 python -m pytest tests/test_gpu_fwd_pair.py -m gpu -x -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "pytest exit $?"; tail -30 $O/pytest.txt
timeout -s KILL 600 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction,causal_document;C5:8192:128:causal_document,sliding_window;C2" libflashmask.so libflashmask.so@8 --rounds 4 --fwd-only > $O/ab.jsonl 2>&1
echo "ab exit $?"; cat $O/ab.jsonl | tail -20
