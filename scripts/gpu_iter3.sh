set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
for poly in 0 32 48 64; do
  for wl in llama7b-4k llama7b-16k falcon7b-8k; do
    KVP_ATTN_POLY=$poly timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_${wl}_poly$poly.log
  done
done
