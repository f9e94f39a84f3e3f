cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/k1
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowwise.py tests/test_gpu_fwd_pair.py -m gpu -q -p no:cacheprovider -x > $O/pytest.txt 2>&1
echo "exit $?"; tail -4 $O/pytest.txt
timeout -s KILL 300 python scripts/k1_bench.py 20 > $O/k1_bench.jsonl 2>&1; cat $O/k1_bench.jsonl
