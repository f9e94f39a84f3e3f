# Full measurement pass: tests, bench (C3 default + C2), launch list, ncu captures of K2/K4.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout -s KILL 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout -s KILL 600 python bench.py --config C2 --no-e2e --cpu-budget 3 2>&1 | tail -1 | tee gpurun_out/bench_c2.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5 > gpurun_out/ncu_launch.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd python scripts/profile_run.py C3 2 > gpurun_out/ncu_bwd.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd python scripts/profile_run.py C3 2 > gpurun_out/ncu_fwd.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k1_ -c 4 -o gpurun_out/prof_k1 python scripts/profile_run.py C3 1 > gpurun_out/ncu_k1.log 2>&1
ls gpurun_out
