"""Pipeline timeline of one triple-buffered attention CTA (attn_tb.cu, KVP_ATTN_TRACE=<cta>): SM clocks
of the S / PV issues, the softmax phases of both column halves of lane quarter 0 and
the TMA issues per key tile.  usage: python scripts/attn_tb_trace.py [shape] [cta]"""
import os
import sys

import numpy as np

shape = sys.argv[1] if len(sys.argv) > 1 else "llama_16k"
os.environ["KVP_ATTN_TRACE"] = sys.argv[2] if len(sys.argv) > 2 else "0"
os.environ["KVP_ATTN_TRACE_OUT"] = "/tmp/attn_trace.bin"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SH = {"llama_4k": (4096, 0, 32, 32, 128), "llama_16k": (16384, 0, 32, 32, 128)}
W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
ms, tf = W.bench_attn(*SH[shape], 1)
print(f"{shape}: {ms:.3f} ms {tf:.0f} TF/s (traced run)")
t = np.fromfile("/tmp/attn_trace.bin", dtype=np.uint32).reshape(16, 512).astype(np.int64)
n = int((t[1] != 0).sum())
base = t[8, 0]
rel = (t - base) % (1 << 32)
names = ["S_iss", "PV_iss", "sm0:S", "sm1:S", "sm0:xch", "sm1:xch", "sm0:P", "sm1:P", "tmaK", "tmaV"]
print("j   " + " ".join(f"{x:>8}" for x in names))
for j in list(range(min(n, 10))) + list(range(max(10, n - 3), n)):
    print(f"{j:<4}" + " ".join(f"{rel[e, j]:8d}" for e in range(10)))
if n > 8:
    mid = range(4, n - 3)
    d = lambda e1, e0, o=0: np.median([(rel[e1, j + o] - rel[e0, j]) for j in mid])
    per = np.median(np.diff(rel[1, 4:n - 2]))
    print(f"median per key tile: PV issue period {per:.0f} clk (tensor work 1024)")
    print(f" S issue(j)->sm0 S seen(j) {d(2, 0):.0f}, S seen->xchg {d(4, 2):.0f}, xchg->P {d(6, 4):.0f}, "
          f"P(j)->PV issue(j) {d(1, 6):.0f}, sm0 P(j)->S seen(j+1) {d(2, 6, 1):.0f}")
    if (t[10] != 0).sum() > 8:
        print(f" issue of 8 S MMAs {d(10, 0):.0f} clk, of 8 PV MMAs {d(11, 1):.0f} clk")
