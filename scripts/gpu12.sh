cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for L in libflashmask.so libflashmask_dkts.so libflashmask.so; do
echo $L; FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
done
timeout -s KILL 300 python scripts/time_kernels.py C3 2 --det 2>&1 | tail -1
timeout -s KILL 300 python scripts/trace_bwd.py 2>&1 | grep -B2 -A6 "s_full pass"
