# C5 kernel sweep (12 Figure-1 families + full, N in {8K, 32K, 128K}, d in {64, 128}) with SM
# clocks / throttle reasons sampled during the run.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/sweep
mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 500 > $O/clocks.csv 2>&1 &
SMI=$!
for cfg in C5:8192:128 C5:32768:128 C5:131072:128 C5:8192:64 C5:32768:64 C5:131072:64; do
  echo "== $cfg"; timeout -s KILL 600 python scripts/time_kernels.py $cfg 3 2>&1 | grep -v Warn
done > $O/c5_sweep.txt 2>&1
kill $SMI
tail -3 $O/c5_sweep.txt
