set -x
for poly in 0 32; do for wl in llama7b-4k llama7b-16k; do
  KVP_ATTN_POLY=$poly timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_${wl}_p$poly.log
done; done
