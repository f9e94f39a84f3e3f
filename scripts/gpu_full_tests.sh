cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/full
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?"; tail -5 $O/pytest.txt
