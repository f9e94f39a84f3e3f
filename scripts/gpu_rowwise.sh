cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/rowwise
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_rowwise.py -m gpu -x -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?"; tail -40 $O/pytest.txt
