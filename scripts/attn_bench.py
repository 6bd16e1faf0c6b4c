"""bf16 tcgen05 attention in isolation (kvp_bench_attn): Llama-7B / Falcon-7B shapes.
Variants are selected by env (KVP_ATTN_WPQ, KVP_ATTN_POLY, KVP_ATTN_MMA_WAIT), read once per process."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SHAPES = {  # name: (q_rows, offset, heads, kv_heads, head_dim)
    "llama_4k": (4096, 0, 32, 32, 128), "llama_16k": (16384, 0, 32, 32, 128),
    "llama_4k_p8_last": (512, 3584, 32, 32, 128), "llama_16k_p8_last": (2048, 14336, 32, 32, 128), "falcon_8k": (8192, 0, 71, 1, 64),
    "falcon_8k_p8_last": (1024, 7168, 71, 1, 64), "falcon_8k_p4_last": (2048, 6144, 71, 1, 64),
    # rank chunks between one and two waves of 256-row CTAs (the attn_tb / attn_tc crossover)
    "llama_4k_p4_last": (1024, 3072, 32, 32, 128), "llama_rank_1280": (1280, 4096, 32, 32, 128),
    "llama_rank_1536": (1536, 6144, 32, 32, 128), "llama_rank_1792": (1792, 7168, 32, 32, 128),
    "falcon_rank_512": (512, 7680, 71, 1, 64), "falcon_rank_640": (640, 7552, 71, 1, 64),
}
W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
tag = ",".join(f"{k[9:]}={v}" for k, v in sorted(os.environ.items()) if k.startswith("KVP_ATTN_"))
only = set(sys.argv[1:])
for name, (q, off, h, kvh, hd) in SHAPES.items():
    if only and name not in only:
        continue
    ms, tf = W.bench_attn(q, off, h, kvh, hd, 20)
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    print(json.dumps({"variant": tag, "shape": name, "ms": round(ms, 4), "tflops": round(tf, 1), "sm_mhz_after": clk}),
          flush=True)
