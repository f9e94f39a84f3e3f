# K1b whole-range uniform block: parity + microbenchmark A/B; forward poly-pair A/B; C2 launch list.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02h
mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowwise.py -m gpu -x -q -p no:cacheprovider -k "classify or refine" > $O/pytest_k1.txt 2>&1
tail -2 $O/pytest_k1.txt
for r in 1 2 3; do
  FLASHMASK_LIB=$PWD/ablibs/head.so timeout -s KILL 120 python scripts/k1_bench.py 20 2>&1 | head -1 | sed 's/^/head /' >> $O/k1_ab.txt
  timeout -s KILL 120 python scripts/k1_bench.py 20 2>&1 | head -1 | sed 's/^/new  /' >> $O/k1_ab.txt
done
cat $O/k1_ab.txt | python -c "
import sys,json
for l in sys.stdin:
  tag,js=l.split(' ',1); d=json.loads(js.strip()); print(tag, d['K1a_expand']['us'], d['K1b_classify']['us'], d['K1b_classify']['frac_of_hbm'])"
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C2;C5:8192:64:causal_document" $PWD/ablibs/head.so libflashmask.so $PWD/ablibs/poly2.so $PWD/ablibs/poly1.so --rounds 5 --fwd-only > $O/ab_poly.jsonl 2>&1
cat $O/ab_poly.jsonl
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5 --sweep none > $O/ncu_c2.log 2>&1
echo ncu rc=$?
