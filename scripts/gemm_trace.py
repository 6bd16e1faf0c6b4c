"""Per-CTA timeline of the tcgen05 GEMM (KVP_GEMM_TRACE): for one isolated launch of each shape,
the median over CTAs of entry -> prologue done -> PDL wait -> first stage landed -> last MMA
issued -> epilogue done, against the ideal MMA time of the CTA's tiles.
usage: python scripts/gemm_trace.py [shape ...]   (shapes as in scripts/gemm_sweep.py)
The stamps are compiled out of the default build: rebuild with
KVP_NVCC_FLAGS=-DKVP_GEMM_TRACE_ON=1 first (profiles/r02/gemm_trace_cost.txt)."""
import json
import os
import sys

import numpy as np

os.environ["KVP_GEMM_TRACE"] = "/tmp/gemm_trace.bin"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SH = {"p8_qkv": (512, 12288, 4096, 0), "p8_o": (512, 4096, 4096, 1), "p8_ffn1": (512, 8192, 4096, 2),
      "p8_ffn2": (512, 4096, 8192, 1), "p4_o": (1024, 4096, 4096, 1), "p4_qkv": (1024, 12288, 4096, 0),
      "llama_o": (4096, 4096, 4096, 1), "llama_qkv": (4096, 12288, 4096, 0), "p8_o_store": (512, 4096, 4096, 3)}
W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
for name in sys.argv[1:] or ["p8_o", "p8_qkv", "llama_o"]:
    M, N, K, epi = SH[name]
    ms, tf, bn = W.bench_gemm(M, N, K, epi, 5)
    t = np.fromfile("/tmp/gemm_trace.bin", dtype=np.uint64).reshape(-1, 8).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    ev = (t[:, :6] - t0) / 1e3  # us
    lead = t[:, 3] > 0  # stamps 3 and 4 come from the MMA issuer: pair leaders only
    med = np.median(ev, axis=0)
    med[3:5] = np.median(ev[lead][:, 3:5], axis=0)
    print(json.dumps({"shape": name, "ms": round(ms, 4), "tflops": round(tf, 1), "bn": bn, "ctas": len(t),
                      "tiles_per_cta": sorted(set(int(x) for x in t[:, 7])),
                      "entry_spread_us": round(float(ev[:, 0].max()), 2),
                      "median_us": {"entry": round(med[0], 2), "prologue": round(med[1], 2), "pdl": round(med[2], 2),
                                    "first_stage": round(med[3], 2), "mma_done": round(med[4], 2),
                                    "epi_done": round(med[5], 2)},
                      "max_epi_done_us": round(float(ev[:, 5].max()), 2),
                      "launch_overhead_us": round(ms * 1e3 - float(ev[:, 5].max()), 2),
                      "mainloop_us_median": round(float(np.median(ev[lead][:, 4] - ev[lead][:, 3])), 2)}), flush=True)
