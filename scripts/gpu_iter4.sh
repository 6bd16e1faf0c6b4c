set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_auto.log 2>&1
KVP_GEMM_BN=256 timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_256.log 2>&1
KVP_GEMM_BN=128 timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_128.log 2>&1
for wl in llama7b-4k llama7b-16k falcon7b-8k; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$wl.log
done
