cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/san
mkdir -p $O
timeout -s KILL 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_run.py cases > $O/sanitize_racecheck.log 2>&1
echo "racecheck exit $?"; grep -E "SUMMARY|Race reported|and .* access" $O/sanitize_racecheck.log | sed 's/(CUtensorMap[^)]*)//g' | cut -c1-200 | head
timeout -s KILL 600 python -m pytest tests/test_gpu_fwd_pair.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout -s KILL 600 python scripts/ab_libs.py "C3;C5:32768:128:causal" libflashmask.so libflashmask.so@8 --rounds 3 --fwd-only 2>&1 | tail -2
