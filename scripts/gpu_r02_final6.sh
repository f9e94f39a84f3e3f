# Round 2 final bench lines at HEAD (K1e timing id, d=64 mask bits): GPU suite, smoke, bench lines, launch list.
# sweep stay from the fourth pass (same kernels on the column-wise bench path).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02final6
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 > $O/pytest_gpu.txt 2>&1
tail -2 $O/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee $O/smoke.txt
timeout -s KILL 1200 python bench.py > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
timeout -s KILL 600 python bench.py --config C2 --no-e2e --cpu-budget 3 --sweep none > $O/bench_C2.log 2>&1; tail -1 $O/bench_C2.log > $O/bench_C2.json
timeout -s KILL 900 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --cpu-budget 3 --sweep none > $O/bench_C4.log 2>&1; tail -1 $O/bench_C4.log > $O/bench_C4.json
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_C3_reference.log 2>&1; tail -1 $O/bench_C3_reference.log > $O/bench_C3_reference.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5 --sweep none > $O/ncu_launch.log 2>&1
python -c "
import json
for f in ['bench_C3','bench_C2','bench_C4']:
    d=json.load(open('$O/'+f+'.json')); print(f, d['value'], d['fwd_tflops_kernel'], d['bwd_tflops_kernel'], d['pct_of_peak'], d.get('clocks'), (d.get('e2e') or {}).get('value'), d['roofline']['frac'])
"
