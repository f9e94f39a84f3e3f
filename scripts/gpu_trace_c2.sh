cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/tracec2
mkdir -p $O
timeout -s KILL 300 python scripts/trace_fwd_cta.py C3 0 > $O/trace_fwd_c3_0.txt 2>&1; head -34 $O/trace_fwd_c3_0.txt
