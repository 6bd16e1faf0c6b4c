set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_auto.log 2>&1
for wl in llama7b-4k llama7b-16k falcon7b-8k; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$wl.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 8 -c 1 -o gpurun_out/prof_attn_v3 -f python bench.py --workload llama7b-4k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn_v3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/prof_gemm_o_v2 -f python scripts/gemm_sweep.py > gpurun_out/ncu_gemm_o_v2.log 2>&1
