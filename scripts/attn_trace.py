"""Pipeline timeline of one attention CTA (KVP_ATTN_TRACE): SM clocks of the MMA issues,
softmax phases and TMA loads per key tile.  usage: python scripts/attn_trace.py [shape] [cta]"""
import os
import sys

import numpy as np

shape = sys.argv[1] if len(sys.argv) > 1 else "llama_16k"
os.environ["KVP_ATTN_TRACE"] = sys.argv[2] if len(sys.argv) > 2 else "0"
os.environ["KVP_ATTN_TRACE_OUT"] = "/tmp/attn_trace.bin"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SH = {"llama_4k": (4096, 0, 32, 32, 128), "llama_16k": (16384, 0, 32, 32, 128), "falcon_8k": (8192, 0, 71, 1, 64)}
W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
ms, tf = W.bench_attn(*SH[shape], 1)
print(f"{shape}: {ms:.3f} ms {tf:.0f} TF/s (traced run)")
t = np.fromfile("/tmp/attn_trace.bin", dtype=np.uint32).reshape(16, 512).astype(np.int64)
n = int((t[0] != 0).sum())
base = t[12, 0]
rel = (t - base) % (1 << 32)
names = ["S_a", "S_b", "PV_a", "PV_b", "sm_a:S", "sm_b:S", "sm_a:ld", "sm_b:ld", "sm_a:max", "sm_b:max",
         "sm_a:P", "sm_b:P", "tmaK", "tmaV"]
print("j   " + " ".join(f"{x:>8}" for x in names))
for j in list(range(min(n, 12))) + list(range(max(12, n - 4), n)):
    print(f"{j:<4}" + " ".join(f"{rel[e, j]:8d}" for e in range(14)))
if n > 8:
    mid = range(4, n - 2)
    d = lambda e1, e0: np.median([(rel[e1, j] - rel[e0, j]) for j in mid])
    per = np.median(np.diff(rel[0, 4:n - 2]))
    print(f"median per key tile: period {per:.0f} clk (tensor work {'2048' if shape != 'falcon_8k' else '1024'})")
    for x, X in ((0, "a"), (1, "b")):
        print(f" tile {X}: S issue->S seen {d(4 + x, 0 + x):.0f}, S seen->ld done {d(6 + x, 4 + x):.0f}, "
              f"ld->max {d(8 + x, 6 + x):.0f}, max->P arrive {d(10 + x, 8 + x):.0f}, P arrive->PV issue {d(2 + x, 10 + x):.0f}")
