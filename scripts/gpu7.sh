cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for L in libflashmask_poly2.so libflashmask.so libflashmask_poly4.so libflashmask_poly5.so; do
  echo "== $L"; FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
done
