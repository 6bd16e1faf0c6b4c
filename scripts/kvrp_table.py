"""KVR-P on B200 costs ("build the table from calibrated B200 cost models").

For p = 2/4/8 and training context lengths C = 2k..32k: calibrate the reference CostModel from
MEASURED per-rank layer times of this B200 at (C, p), run the KVR-S search (bit-exact
hierarchical_grid_search), and store the searched ratios in a PartitionLookupTable (the
reference's JSON schema).  Then, at held-out lengths between the training points, compare the
table's interpolated partition (KVR-P) with a fresh KVR-S search, both scored by the reference
simulator on that length's calibrated costs -- the paper reports KVR-P within 1.1-1.3 % of
KVR-S.  Writes profiles/r01/kvrp_tables/llama7b_p{p}.json and prints one
JSON summary line per p."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_05329_b200 import kvprefill as kv  # noqa: E402

d, h, kvh, L = 4096, 32, 32, 32
W1 = kv.init_weights(kv.ModelConfig(d, h, kvh, 1, 1, "bf16", True))  # one layer: layers cost the same
model = kv.ModelConfig(d, h, kvh, L, 1, "bf16", True)
kv_dim = kvh * (d // h)
net = kv.NetworkModel(bandwidth=770e9 / (2 * kv_dim * 2), latency=10e-6)
train = [2048, 4096, 8192, 16384, 32768]
held = [3072, 6144, 12288, 24576]
out_dir = os.path.join(ROOT, "profiles", "r01", "kvrp_tables")
os.makedirs(out_dir, exist_ok=True)
for p in (2, 4, 8):
    table = kv.PartitionLookupTable(process_count=p)
    for C in train:
        cost = kv.calibrate_cost_model(W1, C, p)
        found = kv.search_partition(C, p, model, cost, net)
        table.insert(C, [s / C for s in found.partition.sizes()])
    table.save(os.path.join(out_dir, f"llama7b_p{p}.json"))
    rows = []
    for C in held:
        cost = kv.calibrate_cost_model(W1, C, p)
        fresh = kv.search_partition(C, p, model, cost, net)
        tpart = kv.partition_from_table(table, C)
        t_tab = kv.simulate_ttft(kv.Strategy.KVR, tpart, model, cost, net)
        t_even = kv.simulate_ttft(kv.Strategy.KVR, kv.even_partition(C, p), model, cost, net)
        rows.append({"C": C, "kvr_s_ms": fresh.ttft * 1e3, "kvr_p_ms": t_tab * 1e3, "kvr_even_ms": t_even * 1e3,
                     "kvr_p_gap_pct": (t_tab / fresh.ttft - 1) * 100, "kvr_p_partition": tpart.boundaries,
                     "kvr_s_partition": fresh.partition.boundaries})
    print(json.dumps({"p": p, "table": f"profiles/r01/kvrp_tables/llama7b_p{p}.json", "train_C": train,
                      "held_out": rows, "max_gap_pct": max(r["kvr_p_gap_pct"] for r in rows)}), flush=True)
