# ncu captures of the d=64 forward and backward kernels (C5 N=32K, full mask, 2nd launch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd64 python scripts/profile_run.py C5:32768:64 2 > gpurun_out/ncu_bwd64.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd64 python scripts/profile_run.py C5:32768:64 2 > gpurun_out/ncu_fwd64.log 2>&1
ls -la gpurun_out
