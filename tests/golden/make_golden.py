"""Generates tests/golden/golden.json from the UNMODIFIED reference (oracle/_ref/libkvref.so,
compiled by oracle/Makefile from /root/reference/proj/include).  Run in the build container:
    python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle_pinned.py) and the GPU parity
tests on the GPU box, where /root/reference does not exist."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def main():
    ref = O.Reference()
    out = {"source": "oracle/_ref/libkvref.so built from /root/reference/proj/include (kvprefill)",
           "runs": [], "partitions": [], "searches": [], "metrics": []}
    cases = [("tiny-default", dict(d_model=32, n_heads=4, n_kv_heads=4, n_layers=2, seed=1, rms_norm=False)),
             ("tiny-rms", dict(d_model=32, n_heads=4, n_kv_heads=4, n_layers=2, seed=1, rms_norm=True)),
             ("tiny-mqa", dict(d_model=32, n_heads=4, n_kv_heads=1, n_layers=2, seed=1, rms_norm=False)),
             ("tiny-gqa", dict(d_model=32, n_heads=4, n_kv_heads=2, n_layers=2, seed=1, rms_norm=False))]
    for name, kw in cases:
        for prec in ("f64", "f32"):
            m = O.Model(precision=prec, **kw)
            dt = np.float64 if prec == "f64" else np.float32
            rw = ref.weights(m)
            ctx = ref.random_context(1024, m.d_model, 18, dt)
            hid, ft, met = rw.run(O.KVR, ctx, ref.even_partition(1024, 2))
            out["runs"].append({
                "name": f"{name}-{prec}", "model": dict(kw, precision=prec), "C": 1024, "context_seed": 18,
                "strategy": "kvr", "boundaries": ref.even_partition(1024, 2),
                "argmax": int(np.argmax(ft[0])), "hidden_fnv1a64": O.fnv1a64(hid),
                "first_token_hidden_head": [float(x) for x in ft[0, :4]],
                "first_token_hidden": [float(x) for x in ft[0]], "metrics": met})
    for C_, p in ((9, 3), (10, 4), (7, 3), (5, 1), (16384, 8), (4096, 3)):
        out["partitions"].append({"kind": "even", "C": C_, "p": p, "boundaries": ref.even_partition(C_, p)})
    for C_, r in ((10240, [0.35, 0.255, 0.21, 0.185]), (3, [0.9, 0.05, 0.05]), (16384, [0.3, 0.25, 0.2, 0.15, 0.1]),
                  (12345, [0.5, 0.3, 0.2])):
        out["partitions"].append({"kind": "ratios", "C": C_, "ratios": r, "boundaries": ref.partition_from_ratios(C_, r)})
    for C_, p, L in ((16384, 2, 32), (16384, 4, 32), (4096, 3, 2), (1024, 4, 2), (96, 4, 2)):
        b, t, ev, lv = ref.search_sim("grid", C_, p, L)
        out["searches"].append({"C": C_, "p": p, "n_layers": L, "boundaries": b, "ttft": t, "evaluations": ev,
                                "levels": lv})
    m = O.Model(8, 2, 2, 2, 3, "f64")
    rw = ref.weights(m)
    ctx = ref.random_context(9, 8, 21, np.float64)
    for strat, b in ((O.KVR, [0, 4, 7, 9]), (O.TSP, [0, 3, 6, 9])):
        _, _, met = rw.run(strat, ctx, b)
        out["metrics"].append({"strategy": "kvr" if strat == O.KVR else "tsp", "boundaries": b, "n_layers": 2,
                               "metrics": met})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
