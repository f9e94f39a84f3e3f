# Round 2: full GPU tests, f3 A/B, bench line, synccheck after the barrier fixes.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02c
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout -s KILL 600 python scripts/ab_refine.py > $O/ab_refine.jsonl 2>&1; cat $O/ab_refine.jsonl
timeout -s KILL 300 python scripts/k1_bench.py 20 > $O/k1_bench.jsonl 2>&1; cat $O/k1_bench.jsonl
timeout -s KILL 1200 python bench.py > $O/bench_C3.log 2>&1; tail -1 $O/bench_C3.log > $O/bench_C3.json
python -c "
import json; d=json.load(open('$O/bench_C3.json'))
print({k:d[k] for k in ['value','fwd_tflops_kernel','bwd_tflops_kernel','clocks']})
for r in d['sweep'] or []: print(r['config'],r['mask'],r['total_tflops'],r['pct_peak'],r['fwd_tflops'],r['bwd_tflops'],r['clocks'])
print(d['k1_microbench'])"
for v in "" f32out; do
timeout -s KILL 600 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py all $v > $O/sanitize_synccheck$v.log 2>&1
echo "synccheck $v exit $?" | tee -a $O/sanitize_summary.txt
done
