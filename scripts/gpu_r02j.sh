# K4 issuer wait mode A/B (suspend hint / try_wait / test_wait spin).
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/r02j
mkdir -p $O
timeout -s KILL 1200 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C2;C5:32768:64:causal" libflashmask.so $PWD/ablibs/bw1.so $PWD/ablibs/bw2.so --rounds 5 > $O/ab_bwait.jsonl 2>&1
cat $O/ab_bwait.jsonl
