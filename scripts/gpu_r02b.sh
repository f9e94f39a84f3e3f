# Round 2, profiling pass: K1 parity (new K1b + a2 counts), K1 microbench, sanitizer re-check,
# ncu launch list of the bench command, full captures of K2 / K4 (C3) and K1b, MMA counts.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "classify or multirank or fwd_bwd_parity or deterministic" > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout -s KILL 300 python scripts/k1_bench.py 20 > $O/k1_bench.jsonl 2>&1; cat $O/k1_bench.jsonl
for tool in synccheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 1000000 --error-exitcode 9 python scripts/sanitize_run.py all f32out > $O/sanitize_${tool}_f32out.log 2>&1
  echo "$tool f32out exit $?" | tee -a $O/sanitize_summary.txt
  grep "ERROR SUMMARY" $O/sanitize_${tool}_f32out.log
  grep "Device Frame" $O/sanitize_${tool}_f32out.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -5
done
timeout -s KILL 600 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py all > $O/sanitize_synccheck.log 2>&1
echo "synccheck bf16 exit $?" | tee -a $O/sanitize_summary.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5 --sweep none > $O/ncu_launch.log 2>&1
timeout -s KILL 900 ncu --set full --metrics sm__inst_executed_pipe_tensor_subpipe_hmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum --clock-control none --import-source on -k regex:fm_bwd_kernel -s 1 -c 1 -o $O/prof_bwd python scripts/profile_run.py C3 2 > $O/ncu_bwd.log 2>&1
timeout -s KILL 900 ncu --set full --metrics sm__inst_executed_pipe_tensor_subpipe_hmma.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum --clock-control none --import-source on -k regex:fm_fwd_kernel -s 1 -c 1 -o $O/prof_fwd python scripts/profile_run.py C3 2 > $O/ncu_fwd.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k1_classify -c 2 -o $O/prof_k1 python scripts/k1_bench.py 1 > $O/ncu_k1.log 2>&1
ls $O
