# session 3: sanitizer runs on the kernels changed after the round-2 sanitizer pass
for tool in memcheck synccheck racecheck; do
  for case in f32 ranks smoke; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $case > gpurun_out/sanitizer3_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitizer3_summary.txt
    tail -2 gpurun_out/sanitizer3_${tool}_${case}.log | tee -a gpurun_out/sanitizer3_summary.txt
  done
done
timeout 900 python -m pytest -q -s tests/test_gpu_parity_large.py 2>&1 | grep -E 'max_rel_dev|passed|failed' | tee gpurun_out/parity_large_devs.txt
