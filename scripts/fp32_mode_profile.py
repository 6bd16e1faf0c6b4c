"""fp32 parity mode (ordered SIMT GEMM + SIMT attention) on the Llama-7B shape: TTFT and the
per-kernel split of one profiled prefill.  usage: python scripts/fp32_mode_profile.py [C] [layers]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
W = kv.init_weights(kv.ModelConfig(4096, 32, 32, L, 1, "f32", True), [0])
ctx = torch.from_numpy(kv.random_context(C, 4096, 18)).cuda()
ft = torch.empty((1, 4096), dtype=torch.float32, device="cuda:0")
part = kv.even_partition(C, 1)
kv.run_device(kv.Strategy.KVR, ctx.data_ptr(), C, part, W, ft.data_ptr())
ts = []
for _ in range(2):
    kv.run_device(kv.Strategy.KVR, ctx.data_ptr(), C, part, W, ft.data_ptr())
    ts.append(W.last_ttft_ms())
W.set_profiling(True)
kv.run_device(kv.Strategy.KVR, ctx.data_ptr(), C, part, W, ft.data_ptr())
st = W.kernel_stats()
W.set_profiling(False)
print(json.dumps({"C": C, "layers": L, "ttft_ms": min(ts), "first_token": int(torch.argmax(ft[0]).item()),
                  "kernels": {k: round(v["total_ms"], 3) for k, v in st.items()}}))
