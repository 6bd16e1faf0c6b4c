set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_tail.log 2>&1
KVP_GEMM_TAIL=0 timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_notail.log 2>&1
for wl in llama7b-4k llama7b-16k; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_$wl.log
done
