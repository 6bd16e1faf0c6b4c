"""In-process engine, p ranks sharing one B200: TTFT of KVR (even) and TSP with the fused KV
handoff (QKV epilogue stores into the receiving ranks' caches; default) against the
copy-engine handoff (KVP_HANDOFF=copy: cumulative [0, b_{i+1}) copy after the projection).
Run once per setting; one JSON line per (strategy, p).  Llama-7B shape, C from argv (4096)."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
W = kv.init_weights(kv.ModelConfig(4096, 32, 32, 32, 1, "bf16", True), [0])
ctx = torch.from_numpy(np.random.default_rng(18).uniform(-1, 1, (C, 4096)).astype(np.float32)).cuda()
ft = torch.empty((1, 4096), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mode = os.environ.get("KVP_HANDOFF", "fused")
for strat in (kv.Strategy.KVR, kv.Strategy.TSP):
    for p in (2, 4, 8):
        part = kv.even_partition(C, p)
        t = []
        for i in range(8):
            flush.zero_()
            torch.cuda.synchronize()
            kv.run_device(strat, ctx.data_ptr(), C, part, W, ft.data_ptr())
            if i >= 3:
                t.append(W.last_ttft_ms())
        print(json.dumps({"handoff": mode, "strategy": strat.name, "p": p, "C": C,
                          "ttft_ms_median": statistics.median(t), "ttft_ms": [round(x, 3) for x in t]}), flush=True)
