# Experiment: where the dQ reduction costs (stage only / bulk only) and deeper staging
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for L in libflashmask.so libflashmask_c32.so libflashmask_c64.so libflashmask_c32s2q2.so; do
  echo "== $L"
  FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
  FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C5:8192:128 3 2>&1 | grep "^causal \|sliding"
done
for L in libflashmask_c32.so; do
  FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fwd_bwd_parity or gqa" 2>&1 | tail -2
done
