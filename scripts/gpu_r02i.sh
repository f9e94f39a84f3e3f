# K1c row chunks + K1d warp-per-unit: parity, C2 step A/B; forward pass-2 alternation A/B.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02i
mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lpt.py -m gpu -x -q -p no:cacheprovider -k "refine or lpt or order or back_to_back or split" > $O/pytest_k1cd.txt 2>&1
tail -2 $O/pytest_k1cd.txt
for r in 1 2 3; do
  FLASHMASK_LIB=$PWD/ablibs/head.so timeout -s KILL 300 python bench.py --config C2 --no-e2e --cpu-budget 0.5 --sweep none --steps 20 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('head', d['ms_per_step'], d['value'], d['kernels_ms_per_step'])" >> $O/c2_ab.txt
  timeout -s KILL 300 python bench.py --config C2 --no-e2e --cpu-budget 0.5 --sweep none --steps 20 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('new ', d['ms_per_step'], d['value'], d['kernels_ms_per_step'])" >> $O/c2_ab.txt
done
cat $O/c2_ab.txt
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C2;C5:8192:64:causal_document" libflashmask.so $PWD/ablibs/alt.so --rounds 5 --fwd-only > $O/ab_alt.jsonl 2>&1
cat $O/ab_alt.jsonl
