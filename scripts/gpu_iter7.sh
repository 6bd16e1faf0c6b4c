set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
for g in 1 0; do
  KVP_GRAPH=$g timeout 600 python bench.py --workload llama7b-4k --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_4k_graph$g.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/prof_gemm_o_v3 -f python scripts/gemm_sweep.py llama_o > gpurun_out/ncu_gemm_o_v3.log 2>&1
