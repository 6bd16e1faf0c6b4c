# compute-sanitizer on small cases (profiles/r02/sanitizer_*.log)
for tool in memcheck synccheck racecheck; do
  for case in smoke kvr3 decode; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $case > gpurun_out/sanitizer_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
    tail -3 gpurun_out/sanitizer_${tool}_${case}.log | tee -a gpurun_out/sanitizer_summary.txt
  done
done
