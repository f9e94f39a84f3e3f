cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/fwd2c
mkdir -p $O
timeout -s KILL 300 python scripts/trace_fwd2.py C3 0 > $O/trace_c3.txt 2>&1; sed -n 20,30p $O/trace_c3.txt; tail -2 $O/trace_c3.txt
timeout -s KILL 600 python scripts/ab_libs.py "C3;C5:32768:128:causal,random_eviction;C2" libflashmask.so libflashmask_t0p1.so@8 libflashmask_t0n.so@8 libflashmask_h4t2.so@8 libflashmask_q2t3.so@8 --rounds 4 --fwd-only > $O/ab.jsonl 2>&1
cat $O/ab.jsonl
