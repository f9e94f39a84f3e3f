# Full measurement pass: tests, smoke, bench lines (C3 default, C2, C4), C5 per-family kernel sweep,
# ncu launch list of the bench command, ncu --set full captures of K4 / K2 (C3) and K4 at d=64.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke.txt
timeout -s KILL 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_C3.json
timeout -s KILL 600 python bench.py --config C2 --no-e2e --cpu-budget 3 2>&1 | tail -1 | tee gpurun_out/bench_C2.json
timeout -s KILL 900 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --cpu-budget 3 2>&1 | tail -1 | tee gpurun_out/bench_C4.json
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | tee gpurun_out/bench_C3_reference.json
for cfg in C5:8192:128 C5:32768:128 C5:131072:128 C5:8192:64 C5:32768:64 C5:131072:64; do
  echo "== $cfg"; timeout -s KILL 600 python scripts/time_kernels.py $cfg 3 2>&1 | grep -v Warn
done 2>&1 | tee gpurun_out/c5_sweep.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5 > gpurun_out/ncu_launch.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd python scripts/profile_run.py C3 2 > gpurun_out/ncu_bwd.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd python scripts/profile_run.py C3 2 > gpurun_out/ncu_fwd.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd64 python scripts/profile_run.py C5:32768:64 2 > gpurun_out/ncu_bwd64.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k1_ -c 4 -o gpurun_out/prof_k1 python scripts/profile_run.py C3 1 > gpurun_out/ncu_k1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"k3_|k5_" -c 2 -o gpurun_out/prof_k35 python scripts/profile_run.py C3 1 > gpurun_out/ncu_k35.log 2>&1
ls gpurun_out
