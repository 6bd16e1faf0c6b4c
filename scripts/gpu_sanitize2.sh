for tool in memcheck synccheck; do
  for case in smoke kvr3 decode; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $case > gpurun_out/sanitizer_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
    tail -2 gpurun_out/sanitizer_${tool}_${case}.log | tee -a gpurun_out/sanitizer_summary.txt
  done
done
KVP_ATTN_TB=0 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_case.py smoke > gpurun_out/sanitizer_synccheck_smoke_tc.log 2>&1; tail -2 gpurun_out/sanitizer_synccheck_smoke_tc.log | tee -a gpurun_out/sanitizer_summary.txt
