set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or strategies or golden or llama" 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
for wl in llama7b-4k llama7b-16k falcon7b-8k; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_$wl.log
done
KVP_ATTN_POLY=32 timeout 600 python bench.py --workload llama7b-16k --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_16k_poly32.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 8 -c 1 -o gpurun_out/prof_attn_v4 -f python bench.py --workload llama7b-4k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn_v4.log 2>&1
