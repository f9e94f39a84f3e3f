# e2e leg: 1 vs 2 compute streams (chunks alternating), interleaved runs.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for ns in 1 2 1 2; do
  FM_E2E_STREAMS=$ns timeout -s KILL 600 python bench.py --sweep none --cpu-budget 0.5 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('streams $ns', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks']['sm_mhz'])"
done
