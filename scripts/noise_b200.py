"""Noise robustness on B200 costs: the reference's noise study
(NoiseSidecar: per layer one adjacent link runs at bandwidth / slowdown; bit-exact
noise_study) on a CostModel calibrated from MEASURED per-rank layer times of this B200 --
KVR-S vs the TSP all-gather, Llama-7B at 16k, p = 4 and 8, slowdowns 2/4/8 on NVLink-class
bandwidth.  Real traffic-generating sidecar GPUs need a multi-GPU node (not this round).
One JSON line per (p, slowdown)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

d, h, kvh, L, C = 4096, 32, 32, 32, 16384
W1 = kv.init_weights(kv.ModelConfig(d, h, kvh, 1, 1, "bf16", True))
model = kv.ModelConfig(d, h, kvh, L, 1, "bf16", True)
kv_dim = kvh * (d // h)
net = kv.NetworkModel(bandwidth=770e9 / (2 * kv_dim * 2), latency=10e-6)
for p in (4, 8):
    cost = kv.calibrate_cost_model(W1, C, p)
    kvr_s = kv.search_partition(C, p, model, cost, net).partition
    even = kv.even_partition(C, p)
    for slow in (2.0, 4.0, 8.0):
        k = kv.noise_study(kv.Strategy.KVR, kvr_s, model, cost, net, slow, 50, 7)
        t = kv.noise_study(kv.Strategy.TSP, even, model, cost, net, slow, 50, 7)
        print(json.dumps({"p": p, "C": C, "slowdown": slow,
                          "kvr_s": {"quiet_ms": k.quiet_ttft * 1e3, "mean_degradation": k.mean_degradation,
                                    "max_degradation": k.max_degradation},
                          "tsp": {"quiet_ms": t.quiet_ttft * 1e3, "mean_degradation": t.mean_degradation,
                                  "max_degradation": t.max_degradation}}), flush=True)
