"""Context-level load balancer on B200 cost data (north star part 3).

1. Calibrate the reference's CostModel from MEASURED per-rank layer times of the B200 layer
   executor (kvp_engine_profile_layer -> kvp_fit_cost_model).
2. NetworkModel from the NVLink peer bandwidth (pairs/s = bytes/s / (2 * kv_dim * 2 B)).
3. KVR-S = hierarchical_grid_search scored by simulate_ttft(KVR) (bit-exact reference search)
   vs the even split (KVR-E) and the TSP all-gather, at p = 2/4/8.
Prints one JSON document (predicted TTFTs are the reference simulator on measured costs)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

SHAPES = {"llama7b": (4096, 32, 32), "falcon7b": (4544, 71, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama7b", choices=sorted(SHAPES))
    ap.add_argument("--C", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--nvlink-gbs", type=float, default=770.0)  # measured peer copy, B200_PROFILING.md
    ap.add_argument("--latency-us", type=float, default=10.0)
    args = ap.parse_args()
    d, h, kvh = SHAPES[args.shape]
    cfg = kv.ModelConfig(d, h, kvh, 1, 1, "bf16", True)  # one layer: layers cost the same
    W = kv.init_weights(cfg)
    kv_dim = kvh * (d // h)
    net = kv.NetworkModel(bandwidth=args.nvlink_gbs * 1e9 / (2 * kv_dim * 2), latency=args.latency_us * 1e-6)
    model = kv.ModelConfig(d, h, kvh, args.layers, 1, "bf16", True)
    out = {"shape": args.shape, "C": args.C, "layers": args.layers, "network": net.__dict__, "p": {}}
    for p in (2, 4, 8):
        t0 = time.perf_counter()
        pts = kv.profile_grid(W, args.C, p)
        cost = kv.calibrate_cost_model(W, args.C, p, points=pts)
        ccost = kv.fit_causal_cost_model(pts)
        calib_s = time.perf_counter() - t0
        even = kv.even_partition(args.C, p)
        t0 = time.perf_counter()
        found = kv.search_partition(args.C, p, model, cost, net)
        search_s = time.perf_counter() - t0
        cfound = kv.search_partition_causal(args.C, p, model, ccost, net)
        kvr_e = kv.simulate_ttft(kv.Strategy.KVR, even, model, cost, net)
        tsp = kv.simulate_ttft(kv.Strategy.TSP, even, model, cost, net)
        star = kv.ttft_star(args.C, p, cost.alpha * args.layers)
        c_kvr_e = kv.simulate_ttft_causal(kv.Strategy.KVR, even, model, ccost, net)
        c_tsp = kv.simulate_ttft_causal(kv.Strategy.TSP, even, model, ccost, net)
        # measured single-rank layer times at the searched partitions (validation)
        per_rank = {}
        for name, part in (("kvr_s", found.partition), ("kvr_s_causal", cfound.partition)):
            bb = part.boundaries
            rows = []
            for i in range(p):
                pm, rm = W.profile_layer(bb[i + 1] - bb[i], bb[i], 3)
                rows.append({"rows": bb[i + 1] - bb[i], "prefix": bb[i], "proj_ms": pm, "rest_ms": rm,
                             "layer_ms": pm + rm})
            per_rank[name] = rows
        out["p"][str(p)] = {
            "samples": [{"rows": c, "prefix": b_, "proj_ms": pr * 1e3, "rest_ms": re * 1e3} for c, b_, pr, re in pts],
            "reference_model": {
                "cost_model": cost.__dict__, "kvr_s_partition": found.partition.boundaries,
                "kvr_s_sizes": found.partition.sizes(), "search_evaluations": found.evaluations,
                "search_levels": found.levels, "search_s": search_s,
                "sim_ttft_ms": {"kvr_s": found.ttft * 1e3, "kvr_even": kvr_e * 1e3, "tsp_even": tsp * 1e3,
                                "ttft_star": star * 1e3},
                "kvr_s_speedup_vs_tsp": tsp / found.ttft, "kvr_s_vs_even": kvr_e / found.ttft},
            "causal_model": {
                "note": "attention priced on causal-visible pairs (tile-skipping kernels, KVR and TSP alike)",
                "cost_model": ccost.__dict__, "kvr_s_partition": cfound.partition.boundaries,
                "kvr_s_sizes": cfound.partition.sizes(),
                "sim_ttft_ms": {"kvr_s": cfound.ttft * 1e3, "kvr_even": c_kvr_e * 1e3, "tsp_even": c_tsp * 1e3},
                "kvr_s_speedup_vs_tsp": c_tsp / cfound.ttft, "kvr_s_vs_even": c_kvr_e / cfound.ttft},
            "calibration_s": calib_s,
            "measured_layer_at_partitions": per_rank,
            "max_rank_layer_ms": {k: max(r["layer_ms"] for r in v) for k, v in per_rank.items()},
        }
        print(json.dumps({"p": p, "ref": out["p"][str(p)]["reference_model"]["sim_ttft_ms"],
                          "causal": out["p"][str(p)]["causal_model"]["sim_ttft_ms"]}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
