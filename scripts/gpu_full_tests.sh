cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/full
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.txt 2>&1
echo "exit $?"; tail -3 $O/pytest.txt
timeout -s KILL 900 python bench.py --sweep none > $O/bench.log 2>&1; tail -1 $O/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks']})"
