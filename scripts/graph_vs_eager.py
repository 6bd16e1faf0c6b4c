"""TTFT of the single-rank prefill: CUDA-graph replay (default) vs eager launches with
per-kernel events (profiling on), interleaved, Llama-7B 4k."""
import os
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
part = kv.even_partition(C, 1)


def step():
    flush.zero_()
    torch.cuda.synchronize()
    kv.run_device(kv.Strategy.KVR, ctx.data_ptr(), C, part, W, ft.data_ptr())
    return W.last_ttft_ms()


for _ in range(3):
    step()
res = {False: [], True: []}
for i in range(12):
    prof = bool(i % 2)
    W.set_profiling(prof)
    res[prof].append(step())
W.set_profiling(False)
print({("eager+events" if k else "graph"): [round(x, 2) for x in v] for k, v in res.items()})
