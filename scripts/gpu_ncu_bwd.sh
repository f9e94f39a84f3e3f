cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd2 python scripts/profile_run.py C3 2 > gpurun_out/ncu_bwd2.log 2>&1
tail -2 gpurun_out/ncu_bwd2.log
