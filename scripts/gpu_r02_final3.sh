# final round-2 measurement pass (session 3): smoke, GPU tests, bench lines, launch list, ncu captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | grep '^{' > gpurun_out/bench_llama7b4k.json
timeout 900 python bench.py --workload llama7b-16k --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/bench_llama7b16k.json
timeout 900 python bench.py --workload falcon7b-8k --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/bench_falcon7b8k.json
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fp32 --no-decode --no-table"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_llama7b4k.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 40 -c 4 -o gpurun_out/r02s3_gemm_4k -f python bench.py $ARGS > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 8 -c 1 -o gpurun_out/r02s3_attn_4k -f python bench.py $ARGS > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 8 -c 1 -o gpurun_out/r02s3_attn_falcon8k -f python bench.py --workload falcon7b-8k $ARGS > gpurun_out/ncu_attn_f.log 2>&1
