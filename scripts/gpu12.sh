cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for L in libflashmask.so libflashmask_spinP.so libflashmask_spinS.so libflashmask_nospin.so libflashmask.so; do
echo $L; FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 300 python scripts/time_kernels.py C3 3 2>&1 | tail -1
done
timeout -s KILL 300 python scripts/trace_fwd.py C3 2>&1 | tail -6
