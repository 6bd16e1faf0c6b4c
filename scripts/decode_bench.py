"""Decode step on the prefilled KV cache: Llama-7B / Falcon-7B shape, prompt of
C tokens prefilled into a KVCache, then single-row decode steps.  Reports device ms per step
and the achieved HBM bandwidth against the measured peak: algorithmic bytes per step = all
projection weights (bf16) + the K/V cache rows read by attention."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SHAPES = {"llama7b": (4096, 32, 32, 32), "falcon7b": (4544, 71, 1, 32)}
name = sys.argv[1] if len(sys.argv) > 1 else "llama7b"
C_ = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
d, h, kvh, L = SHAPES[name]
cfg = kv.ModelConfig(d, h, kvh, L, 1, "bf16", True)
W = kv.init_weights(cfg)
rng = np.random.default_rng(18)
ctx = rng.uniform(-1, 1, (C_ + steps + 4, d)).astype(np.float32)
cache = kv.KVCache(W, C_ + steps + 4)
_, _, prefill_ms = cache.prefill(ctx[:C_])
for i in range(3):  # warm-up steps, then truncate back
    cache.decode(ctx[C_ + i:C_ + i + 1])
cache.reset(C_)
times = []
for i in range(steps):
    _, ms = cache.decode(ctx[C_ + i:C_ + i + 1])
    times.append(ms)
hd = d // h
q, kvd, f = h * hd, kvh * hd, 2 * d
weight_bytes = 2 * L * (d * (q + 2 * kvd) + q * d + 2 * d * f)
kv_bytes = 2 * L * 2 * kvd * (C_ + steps / 2)  # K and V rows read per step (mean position)
ms = statistics.median(times)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.2
gbs = (weight_bytes + kv_bytes) / (ms * 1e-3) / 1e9
print(json.dumps({"workload": f"{name}-decode-after-{C_}", "prefill_ms": prefill_ms, "decode_ms_per_step": ms,
                  "decode_ms_min": min(times), "bytes_per_step": weight_bytes + kv_bytes, "achieved_gbs": gbs,
                  "hbm_peak_gbs": peak, "frac": gbs / peak, "steps": steps}))
