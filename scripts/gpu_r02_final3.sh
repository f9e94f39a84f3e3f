# Round 2 final evidence pass (session 3, after the persistent fixup and the K2b bounded pass): GPU tests, smoke, bench lines (C3 default with sweep, C2, C4,
# of the bench command and --set full captures of K4 / K2 (C3), K4 d=64, K1, K3/K5.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02final3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu_state.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee $O/smoke.txt
timeout -s KILL 1200 python bench.py > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
timeout -s KILL 600 python bench.py --config C2 --no-e2e --cpu-budget 3 --sweep none > $O/bench_C2.log 2>&1; tail -1 $O/bench_C2.log > $O/bench_C2.json
timeout -s KILL 900 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --cpu-budget 3 --sweep none > $O/bench_C4.log 2>&1; tail -1 $O/bench_C4.log > $O/bench_C4.json
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_C3_reference.log 2>&1; tail -1 $O/bench_C3_reference.log > $O/bench_C3_reference.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d.get(k) for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks','roofline']})
for r in d.get('sweep') or []: print(r['config'],r['mask'],r['total_tflops'],r['pct_peak'],r['fwd_tflops'],r['bwd_tflops'])
" 2>&1 | tee $O/bench_summary.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5 --sweep none > $O/ncu_launch.log 2>&1
M=sm__inst_executed_pipe_tensor_subpipe_hmma.sum
timeout -s KILL 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o $O/prof_bwd python scripts/profile_run.py C3 2 > $O/ncu_bwd.log 2>&1
timeout -s KILL 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:fm_fwd_kernel -s 2 -c 1 -o $O/prof_fwd python scripts/profile_run.py C3 2 > $O/ncu_fwd.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o $O/prof_bwd64 python scripts/profile_run.py C5:32768:64 2 > $O/ncu_bwd64.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k1_ -c 4 -o $O/prof_k1 python scripts/profile_run.py C3 1 > $O/ncu_k1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"k3_|k5_" -c 2 -o $O/prof_k35 python scripts/profile_run.py C3 1 > $O/ncu_k35.log 2>&1
timeout -s KILL 300 python scripts/k1_bench.py 20 > $O/k1_bench.jsonl 2>&1
ls $O
timeout -s KILL 1500 bash scripts/gpu_sweep.sh > $O/sweep.log 2>&1; cp gpurun_out/sweep/c5_sweep.txt gpurun_out/sweep/clocks.csv $O/ 2>/dev/null
ls $O
