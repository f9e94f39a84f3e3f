cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python scripts/ab_libs.py "C3;C5:32768:128:causal;C2" libflashmask.so libflashmask_nored.so --rounds 4 2>&1 | tail -5
