cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/lpt
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout -s KILL 600 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_lpt.py -m gpu -q -x -p no:cacheprovider -k "document-4096" > $O/sync.txt 2>&1; echo "synccheck exit $?"; grep "ERROR SUMMARY" $O/sync.txt
timeout -s KILL 1200 python scripts/ab_libs.py "C2" libflashmask_head.so libflashmask.so --rounds 6 > $O/ab.jsonl 2>&1
cat $O/ab.jsonl
