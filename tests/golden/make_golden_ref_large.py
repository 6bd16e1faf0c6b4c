"""Runs the UNMODIFIED reference (oracle/_ref/libkvref.so) at a benchmarked shape and writes
tests/golden/ref_<name>.json.  Slow (about an hour on 8 host cores for llama7b-4k: the
reference's dense attention and i-k-j matmul); it pins the fast restatement
(oracle/kvp_oracle_fast.c, tests/golden/make_golden_large.py) at the full shape.  Run in the
build container:
    nice python tests/golden/make_golden_ref_large.py llama7b-4k
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

CASES = {
    # name: (model kwargs, C, partition kind, p)
    "llama7b-4k": (dict(d_model=4096, n_heads=32, n_kv_heads=32, n_layers=32, seed=1, rms_norm=True), 4096, 8),
    "falcon7b-2k-l4": (dict(d_model=4544, n_heads=71, n_kv_heads=1, n_layers=4, seed=1, rms_norm=True), 2048, 8),
}


def main(name: str):
    kw, C_, p = CASES[name]
    ref = O.Reference()
    m = O.Model(precision="f32", **kw)
    t0 = time.time()
    rw = ref.weights(m)
    ctx = ref.random_context(C_, m.d_model, 18, np.float32)
    b = ref.even_partition(C_, p)
    t1 = time.time()
    hid, ft, met = rw.run(O.KVR, ctx, b)
    t2 = time.time()
    row = ft[0]
    order = np.argsort(-row.astype(np.float64))
    out = {"name": name, "source": "oracle/_ref/libkvref.so (unmodified reference run<float>(KVR))",
           "model": dict(kw, precision="f32"), "C": C_, "context_seed": 18, "strategy": "kvr",
           "boundaries": b, "argmax": int(np.argmax(row)),
           "top2_margin": float(row[order[0]] - row[order[1]]),
           "hidden_fnv1a64": O.fnv1a64(hid), "last_row_fnv1a64": O.fnv1a64(ft),
           "first_token_hidden": [float(x) for x in row], "metrics": met,
           "seconds": {"init": round(t1 - t0, 1), "run": round(t2 - t1, 1)}}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"ref_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, out["seconds"], "argmax", out["argmax"])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "llama7b-4k")
