set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 300 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep_auto.log 2>&1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.log
timeout 600 python bench.py --workload llama7b-16k --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_llama7b-16k.log
timeout 600 python bench.py --workload falcon7b-8k --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_falcon7b-8k.log
timeout 900 python scripts/balancer_study.py --C 16384 > gpurun_out/balancer_llama7b_16k.json 2> gpurun_out/balancer.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_reference.log
