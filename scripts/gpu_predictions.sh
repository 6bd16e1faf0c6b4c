#!/bin/bash
# Multi-GPU predictions from per-rank costs measured on this B200 (one GPU): balancer study,
# context sweeps (Llama / Falcon), KVR-P tables, noise study.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/pred
timeout 900 python scripts/balancer_study.py --C 16384 > gpurun_out/pred/balancer_llama7b_16k.json 2> gpurun_out/pred/bal16.err
timeout 600 python scripts/balancer_study.py --C 4096 > gpurun_out/pred/balancer_llama7b_4k.json 2> gpurun_out/pred/bal4.err
timeout 1200 python scripts/context_sweep.py > gpurun_out/pred/context_sweep.jsonl 2> gpurun_out/pred/cs.err
timeout 900 python scripts/context_sweep.py falcon7b-8k 2048 8192 16384 > gpurun_out/pred/context_sweep_falcon.jsonl 2> gpurun_out/pred/csf.err
timeout 900 python scripts/kvrp_table.py > gpurun_out/pred/kvrp_b200.jsonl 2> gpurun_out/pred/kvrp.err
cp -r profiles/r01/kvrp_tables gpurun_out/pred/ 2>/dev/null
timeout 900 python scripts/noise_b200.py > gpurun_out/pred/noise_b200.jsonl 2> gpurun_out/pred/noise.err
ls -la gpurun_out/pred; tail -2 gpurun_out/pred/*.err
