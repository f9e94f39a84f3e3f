cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd2 python scripts/profile_run.py C3 2 > gpurun_out/ncu_fwd2.log 2>&1
tail -1 gpurun_out/ncu_fwd2.log
