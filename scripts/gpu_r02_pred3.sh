# session 3: refresh the multi-GPU predictions and GEMM sweep with the final kernels; new attention test
mkdir -p gpurun_out/pred
timeout 600 python -m pytest -q tests/test_gpu_attn_variants.py -k rank_chunk 2>&1 | tail -3 | tee gpurun_out/pred/test_rank_chunk.txt
timeout 900 python scripts/balancer_study.py --C 16384 > gpurun_out/pred/balancer_llama7b_16k.json 2> gpurun_out/pred/bal16.err
timeout 600 python scripts/balancer_study.py --C 4096 > gpurun_out/pred/balancer_llama7b_4k.json 2> gpurun_out/pred/bal4.err
timeout 1500 python scripts/context_sweep.py > gpurun_out/pred/context_sweep.jsonl 2> gpurun_out/pred/cs.err
timeout 1200 python scripts/context_sweep.py falcon7b-8k 1024 2048 4096 8192 16384 > gpurun_out/pred/context_sweep_falcon.jsonl 2> gpurun_out/pred/csf.err
timeout 600 python scripts/gemm_sweep.py > gpurun_out/pred/gemm_sweep.jsonl 2> gpurun_out/pred/gemm.err
ls -la gpurun_out/pred; tail -2 gpurun_out/pred/*.err
