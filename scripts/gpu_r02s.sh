# Full GPU suite after the persistent-fixup refactor (+ multi-unit fixup, GQA / bf16 bounded tests).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02s
mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "bounded" > $O/pytest_bounded.txt 2>&1
tail -3 $O/pytest_bounded.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
