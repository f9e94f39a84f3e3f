# A/B of whole bench lines (step time incl. launch gaps): FLASHMASK_LIB variants as arguments
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for rep in 1 2; do
for L in "$@"; do
  for c in ${CFGS:-C2 C3}; do
    FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L timeout -s KILL 600 python bench.py --config $c --no-e2e --cpu-budget 0.5 ${BENCH_ARGS:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', '$c', d['value'], d['ms_per_step'], d['fwd_tflops_kernel'], d['bwd_tflops_kernel'], {k: round(v, 3) for k, v in d['kernels_ms_per_step'].items()})"
  done
done
done
