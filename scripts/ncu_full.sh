# One `ncu --set full` capture per hot kernel class (single launch each, 1 GPU).
set -x
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 40 -c 1 -o gpurun_out/prof_gemm -f python bench.py $ARGS > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 8 -c 1 -o gpurun_out/prof_attn -f python bench.py $ARGS > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:norm_cast -s 8 -c 1 -o gpurun_out/prof_norm -f python bench.py $ARGS > gpurun_out/ncu_norm.log 2>&1
ls -la gpurun_out
