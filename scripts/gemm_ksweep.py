import json, os, sys
sys.path.insert(0, os.getcwd())
from paper_2405_05329_b200 import kvprefill as kv
W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
for (M, N, epi) in ((512, 4096, 1), (512, 4096, 3), (512, 12288, 0), (2048, 4096, 1), (2048, 4096, 3), (4096, 4096, 3)):
    for K in (512, 1024, 2048, 4096, 8192, 16384):
        ms, tf, bn = W.bench_gemm(M, N, K, epi, 20)
        print(json.dumps({"M": M, "N": N, "K": K, "epi": epi, "us": round(ms * 1e3, 2), "tflops": round(tf), "bn": bn}), flush=True)
