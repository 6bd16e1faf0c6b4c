# final validation after the fp32-mode kernels and the attn_tb rounding fix
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | grep '^{' > gpurun_out/bench_llama7b4k.json
timeout 900 python bench.py --workload llama7b-16k --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/bench_llama7b16k.json
timeout 900 python bench.py --workload falcon7b-8k --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/bench_falcon7b8k.json
