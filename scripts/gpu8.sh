cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in C5:8192:128 C5:8192:64 C5:32768:128; do
  echo "== $cfg"; timeout -s KILL 900 python scripts/time_kernels.py $cfg 2 2>&1 | tail -13
done
echo "== C4"; timeout -s KILL 900 python scripts/time_kernels.py C4 2 2>&1 | tail -2
