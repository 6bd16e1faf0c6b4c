"""tcgen05 GEMM shapes of the Llama-7B / Falcon-7B layer executor in isolation (kvp_bench_gemm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
shapes = {  # name: (M, N, K, epi)
    "llama_qkv": (4096, 12288, 4096, 0), "llama_o": (4096, 4096, 4096, 1), "llama_ffn1": (4096, 8192, 4096, 2),
    "llama_ffn2": (4096, 4096, 8192, 1), "llama_o_store": (4096, 4096, 4096, 3), "llama_ffn2_store": (4096, 4096, 8192, 3),
    "p8_qkv": (512, 12288, 4096, 0), "p8_o": (512, 4096, 4096, 1), "p8_ffn1": (512, 8192, 4096, 2),
    "p8_ffn2": (512, 4096, 8192, 1), "falcon_qkv": (8192, 4672, 4544, 0), "falcon_o": (8192, 4544, 4544, 1),
    "sq8192": (8192, 8192, 8192, 3),
    "l16_qkv": (16384, 12288, 4096, 0), "l16_o": (16384, 4096, 4096, 1), "l16_ffn1": (16384, 8192, 4096, 2),
    "l16_ffn2": (16384, 4096, 8192, 1),
    "p4_qkv": (1024, 12288, 4096, 0), "p4_o": (1024, 4096, 4096, 1), "p4_ffn1": (1024, 8192, 4096, 2),
    "p4_ffn2": (1024, 4096, 8192, 1), "p2_qkv": (2048, 12288, 4096, 0), "p2_o": (2048, 4096, 4096, 1),
    "p2_ffn1": (2048, 8192, 4096, 2), "p2_ffn2": (2048, 4096, 8192, 1),
}
only = set(sys.argv[1:])
out = {}
for name, (M, N, K, epi) in shapes.items():
    if only and name not in only:
        continue
    ms, tf, bn = W.bench_gemm(M, N, K, epi, 20)
    out[name] = {"M": M, "N": N, "K": K, "epi": epi, "ms": ms, "tflops": tf, "bn": bn}
    print(json.dumps({name: out[name]}), flush=True)
