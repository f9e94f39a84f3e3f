# Round 2: GPU tests after the N<128 kernel-map fix; in-session A/B of the f3 forward; bwd trace.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02d
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
CFGS="C3 C5:32768:128:qk_sparse,random_eviction,causal_document,causal C5:8192:128:qk_sparse,causal_document,sliding_window" \
  timeout -s KILL 1200 bash scripts/gpu_ab.sh libflashmask.so libflashmask_norefine.so > $O/ab_fwd_refine.txt 2>&1
cat $O/ab_fwd_refine.txt
timeout -s KILL 300 python scripts/k1_bench.py 20 > $O/k1_bench.jsonl 2>&1; cat $O/k1_bench.jsonl
timeout -s KILL 600 python scripts/trace_bwd.py C3 > $O/trace_bwd_C3.txt 2>&1; head -60 $O/trace_bwd_C3.txt
timeout -s KILL 600 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py all > $O/sanitize_synccheck.log 2>&1
echo "synccheck exit $?" | tee -a $O/sanitize_summary.txt
