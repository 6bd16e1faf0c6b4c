"""Context-length sweep (BASELINE configs[4]): Llama-7B shape, C = 1k..32k.

* p = 1: MEASURED single-GPU TTFT (device time, the CUDA-graph prefill, L2 flushed before each
  step) and its fraction of the compute roofline (SURVEY 8d algorithmic FLOPs / measured burst
  bf16 peak).
* p = 2/4/8: the reference's simulator (simulate_ttft, bit-exact) on a CostModel calibrated from
  MEASURED per-rank layer times of this B200 at the same C -- KVR-S (searched split), KVR even
  split and the TSP all-gather -- plus the KV handoff bytes per layer and their NVLink time.
This box has one GPU, so the p > 1 rows are predictions from measured costs, labelled as such.
One JSON line per C."""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

args = sys.argv[1:]
shape = "llama7b-4k"
if args and not args[0].isdigit():  # optional shape: llama7b-4k (default) or falcon7b-8k
    shape = args.pop(0)
Cs = [int(x) for x in args] or [1024, 2048, 4096, 8192, 16384, 32768]
w = dict(bench.WORKLOADS[shape])
d, h, kvh, L = w["d_model"], w["n_heads"], w["n_kv_heads"], w["n_layers"]
kv_dim = kvh * (d // h)
peaks = bench.load_peaks()
W = kv.init_weights(kv.ModelConfig(d, h, kvh, L, 1, "bf16", True))
W1 = kv.init_weights(kv.ModelConfig(d, h, kvh, 1, 1, "bf16", True))  # one layer: calibration
model = kv.ModelConfig(d, h, kvh, L, 1, "bf16", True)
net = kv.NetworkModel(bandwidth=770e9 / (2 * kv_dim * 2), latency=10e-6)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for C in Cs:
    ctx = torch.from_numpy(np.random.default_rng(18).uniform(-1, 1, (C, d)).astype(np.float32)).cuda()
    ft = torch.empty((1, d), dtype=torch.float32, device="cuda")
    part = kv.even_partition(C, 1)
    times = []
    for i in range(8):
        flush.zero_()
        torch.cuda.synchronize()
        kv.run_device(kv.Strategy.KVR, ctx.data_ptr(), C, part, W, ft.data_ptr())
        if i >= 3:
            times.append(W.last_ttft_ms())
    ms = statistics.median(times)
    F = bench.algorithmic_flops(w, C)
    line = {"shape": shape.split("-")[0], "C": C, "p1_ttft_ms": ms, "p1_roofline_ms": F / (peaks["bf16"] * 1e12) * 1e3,
            "p1_roofline_frac": F / (peaks["bf16"] * 1e12) / (ms * 1e-3), "algorithmic_tflop": F / 1e12,
            "predicted": {}}
    for p in (2, 4, 8):
        cost = kv.calibrate_cost_model(W1, C, p)
        even = kv.even_partition(C, p)
        found = kv.search_partition(C, p, model, cost, net)
        kvr_e = kv.simulate_ttft(kv.Strategy.KVR, even, model, cost, net)
        tsp = kv.simulate_ttft(kv.Strategy.TSP, even, model, cost, net)
        b = found.partition.boundaries
        busiest = 2 * b[p - 1] * kv_dim * 2  # bytes on link p-2 -> p-1 per layer
        line["predicted"][str(p)] = {
            "kvr_s_ms": found.ttft * 1e3, "kvr_even_ms": kvr_e * 1e3, "tsp_ms": tsp * 1e3,
            "kvr_s_vs_tsp": tsp / found.ttft, "kvr_s_vs_even": kvr_e / found.ttft,
            "kvr_s_partition": b, "speedup_vs_p1_measured": ms / (found.ttft * 1e3),
            "busiest_link_bytes_per_layer": busiest, "busiest_link_ms_at_900gbs": busiest / 900e9 * 1e3}
    print(json.dumps(line), flush=True)
