"""Per-CTA timeline of the tcgen05 attention kernel (KVP_ATTN_CTA_TRACE): start/end
(globaltimer ns), SM and key steps of every CTA.  Fits duration = fixed + per_step * steps,
and reports the gaps between consecutive CTAs on one SM and the idle tail.
usage: python scripts/attn_cta_trace.py [shape ...]"""
import json
import os
import sys

import numpy as np

os.environ["KVP_ATTN_CTA_TRACE"] = "/tmp/attn_cta.bin"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SH = {"llama_4k": (4096, 0, 32, 32, 128), "llama_16k": (16384, 0, 32, 32, 128), "falcon_8k": (8192, 0, 71, 1, 64),
      "llama_4k_p8_last": (512, 3584, 32, 32, 128)}
W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
for name in sys.argv[1:] or ["llama_4k", "llama_16k", "falcon_8k"]:
    ms, tf = W.bench_attn(*SH[name], 3)
    t = np.fromfile("/tmp/attn_cta.bin", dtype=np.uint64).reshape(-1, 4).astype(np.int64)
    t0 = t[:, 0].min()
    st, en, sm, steps = t[:, 0] - t0, t[:, 1] - t0, t[:, 2], t[:, 3]
    dur = en - st
    A = np.vstack([np.ones_like(steps), steps]).T.astype(float)
    (fixed, per), *_ = np.linalg.lstsq(A, dur.astype(float), rcond=None)
    span = en.max()
    gaps = []
    busy = 0
    for s in np.unique(sm):
        idx = np.where(sm == s)[0]
        idx = idx[np.argsort(st[idx])]
        gaps += list(st[idx[1:]] - en[idx[:-1]])
        busy += dur[idx].sum()
    print(json.dumps({"shape": name, "ms": round(ms, 4), "tflops": round(tf, 1), "ctas": len(t),
                      "span_us": round(span / 1e3, 1), "fixed_us": round(fixed / 1e3, 2),
                      "per_step_ns": round(per, 1), "first_start_spread_us": round(np.sort(st)[147] / 1e3, 2),
                      "gap_median_us": round(float(np.median(gaps)) / 1e3, 2) if gaps else None,
                      "sm_busy_frac": round(busy / (span * len(np.unique(sm))), 3),
                      "tail_us": round((span - np.percentile(en, 50)) / 1e3, 1),
                      "last_start_us": round(st.max() / 1e3, 1)}), flush=True)
