cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for L in libflashmask_poly0.so libflashmask_poly1.so libflashmask_poly2.so libflashmask.so; do
  echo "== $L"; FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
  FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C5:8192:128 2 2>&1 | head -1
done
