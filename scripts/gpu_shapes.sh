set -x
for wl in llama7b-16k falcon7b-8k tiny; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$wl.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 8 -c 1 -o gpurun_out/prof_attn_tc -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 42 -c 1 -o gpurun_out/prof_gemm_o -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gemm_o.log 2>&1
