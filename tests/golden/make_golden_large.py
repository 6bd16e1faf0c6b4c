"""Generates tests/golden/golden_large.json: the reference's f32 first token at the benchmarked
shapes (Llama-7B / Falcon-7B widths, all 32 layers, 1k-16k tokens), computed by the
multi-threaded restatement oracle/kvp_oracle_fast.c, which is bit-identical to the reference:
  * against oracle/_ref (the unmodified reference compiled from /root/reference) at reduced
    layer/token counts of the same widths: tests/test_oracle_fast.py;
  * against the reference itself at the full llama7b-4k shape (tests/golden/ref_llama7b-4k.json,
    written by make_golden_ref_large.py; checked below when present).
Inputs are the reference's own: init_weights(ModelConfig{..., seed=1, rms_norm=true}) and
random_context(C, d, 18) (commands.hpp:284 uses config.seed+17).  KVR on any partition is
bitwise the serial forward in the reference (test_engine.cpp:50-99), so one serial pass pins
every partition.  Run in the build container (8 host cores: ~10 minutes in total):
    python tests/golden/make_golden_large.py [name ...]
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

LLAMA = dict(d_model=4096, n_heads=32, n_kv_heads=32, seed=1, rms_norm=True)
FALCON = dict(d_model=4544, n_heads=71, n_kv_heads=1, seed=1, rms_norm=True)
CASES = {
    # the bench workloads (bench.py --workload)
    "llama7b-4k": (dict(LLAMA, n_layers=32), 4096),
    "falcon7b-8k": (dict(FALCON, n_layers=32), 8192),
    "llama7b-16k": (dict(LLAMA, n_layers=32), 16384),
    # quicker cases at the same widths for the parity grid (partitions, fp32 mode)
    "llama7b-1k": (dict(LLAMA, n_layers=32), 1024),
    "falcon7b-1k": (dict(FALCON, n_layers=32), 1024),
    "llama7b-gqa-2k-l4": (dict(LLAMA, n_kv_heads=8, n_layers=4), 2048),
}
PATH = os.path.join(HERE, "golden_large.json")


def run_case(name):
    kw, C_ = CASES[name]
    m = O.Model(precision="f32", **kw)
    ctx = O.random_context(C_, m.d_model, 18, np.float32)
    t0 = time.time()
    hid, last = O.forward_fast_f32(m, ctx)
    secs = time.time() - t0
    order = np.argsort(-last.astype(np.float64), kind="stable")
    return {"name": name, "model": dict(kw, precision="f32"), "C": C_, "context_seed": 18,
            "source": "oracle/kvp_oracle_fast.c (bit-identical restatement of run<float>)",
            "argmax": int(order[0]), "top2_margin": float(last[order[0]] - last[order[1]]),
            "top5": [int(i) for i in order[:5]],
            "hidden_fnv1a64": O.fnv1a64(hid), "last_row_fnv1a64": O.fnv1a64(last.reshape(1, -1)),
            "first_token_hidden": [float(x) for x in last], "seconds": round(secs, 1)}


def main(names):
    out = json.load(open(PATH)) if os.path.exists(PATH) else {"cases": {}}
    for name in names:
        r = run_case(name)
        refp = os.path.join(HERE, f"ref_{name}.json")
        if os.path.exists(refp):  # the reference itself at this shape
            ref = json.load(open(refp))
            r["pinned_by_reference"] = {
                "file": os.path.basename(refp),
                "hidden_equal": ref["hidden_fnv1a64"] == r["hidden_fnv1a64"],
                "first_token_equal": ref["first_token_hidden"] == r["first_token_hidden"]}
        out["cases"][name] = r
        print(name, "argmax", r["argmax"], "margin", r["top2_margin"], f"{r['seconds']} s", flush=True)
        with open(PATH, "w") as f:
            json.dump(out, f, indent=0)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
