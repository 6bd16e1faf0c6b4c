set -x
./scripts/microbench/exp2_bench > gpurun_out/exp2_bench.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or strategies" 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
for wl in llama7b-4k llama7b-16k falcon7b-8k; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_$wl.log
done
