cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_run.py C3 2 > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd python scripts/profile_run.py C3 2 > gpurun_out/ncu_bwd.log 2>&1
tail -3 gpurun_out/ncu_bwd.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd python scripts/profile_run.py C3 2 > gpurun_out/ncu_fwd.log 2>&1
tail -3 gpurun_out/ncu_fwd.log
ls -la gpurun_out
