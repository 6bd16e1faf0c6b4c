"""One KVR run, p ranks on one GPU (Llama-7B shape, C from argv): the ncu target for the fused
handoff's cost inside the QKV GEMM (rank i < p-1 stores its K/V rows twice: own cache + rank
i+1's)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
W = kv.init_weights(kv.ModelConfig(4096, 32, 32, 4, 1, "bf16", True), [0])
ctx = torch.from_numpy(np.random.default_rng(18).uniform(-1, 1, (C, 4096)).astype(np.float32)).cuda()
ft = torch.empty((1, 4096), dtype=torch.float32, device="cuda")
for _ in range(2):
    kv.run_device(kv.Strategy.KVR, ctx.data_ptr(), C, kv.even_partition(C, p), W, ft.data_ptr())
torch.cuda.synchronize()
print("ttft_ms", W.last_ttft_ms())
