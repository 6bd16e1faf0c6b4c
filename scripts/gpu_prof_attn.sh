set -x
for poly in 0 32; do
KVP_ATTN_POLY=$poly timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 8 -c 1 -o gpurun_out/prof_attn_p$poly -f python bench.py --workload llama7b-16k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_attn_p$poly.log 2>&1
done
