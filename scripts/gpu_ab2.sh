cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal;C2;C5:8192:64:causal_document" libflashmask_head.so libflashmask_psleep.so libflashmask_pmsleep.so --rounds 5 --fwd-only 2>&1 | tail -8
