# A/B kernel timings in one run: FLASHMASK_LIB variants given as arguments
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
CFGS=${CFGS:-"C3 C5:8192:128"}
for rep in 1 2; do
for L in "$@"; do
  for c in $CFGS; do
    echo "== $L $c"
    FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py $c 3 2>&1 | grep -v Warn | grep "${FILTER:-.}"
  done
done
done
