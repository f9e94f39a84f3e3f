cd $GRAFT_REPO_ROOT
for r in 1 2; do for L in libflashmask_old.so libflashmask.so; do echo "== $L"; FLASHMASK_LIB=$PWD/paper_2410_01359_b200/$L python scripts/time_bwd_only.py C3 3 2>&1 | grep only; done; done
FILTER="call\|^full\|^causal \|sliding_window\|^document\|share" bash scripts/gpu_ab.sh libflashmask_old.so libflashmask.so
