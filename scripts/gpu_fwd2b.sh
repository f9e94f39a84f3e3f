# K2b: exp2 MUFU/poly split A/B and one ncu --set full capture of K2b on C3.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
O=gpurun_out/fwd2b
mkdir -p $O
timeout -s KILL 600 python scripts/ab_libs.py "C3;C5:32768:128:causal;C2" libflashmask.so libflashmask.so@8 libflashmask_p0.so@8 libflashmask_p1.so@8 --rounds 4 --fwd-only > $O/ab.jsonl 2>&1
echo "ab exit $?"; cat $O/ab.jsonl | tail -8
FM_PROFILE_FLAGS=8 timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:fm_fwd2_kernel -s 2 -c 1 -o $O/prof_fwd2 python scripts/profile_run.py C3 2 > $O/ncu_fwd2.log 2>&1
echo "ncu exit $?"; tail -3 $O/ncu_fwd2.log
