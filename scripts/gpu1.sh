cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PYTHONUNBUFFERED=1
timeout -s KILL 200 python -m pytest tests/test_gpu_parity.py -x -q -k "classify" 2>&1 | tail -8
for c in "causal 256 128 1 1 fwd" "full 384 128 1 1 fwd" "causal_document 1000 128 1 2 fwd" "causal_document 128 64 1 1 fwd" "causal 256 128 1 1 bwd" "causal_document 1000 128 1 2 bwd" "causal_document 128 64 1 1 bwd"; do
  echo "== $c"; timeout -s KILL 60 python scripts/dev_check.py $c 2>&1 | tail -6
done
