"""Multi-process (N>1) host logic on CPU: paper_2405_05329_b200.distributed.run_rank with a
gloo group of world_size 2 and 3, one process per rank, the oracle as the stand-in layer
executor.  Checks, against the reference's own properties and goldens:
  * KVR and TSP over real process boundaries reproduce the serial forward pass BITWISE (f64);
  * ExecutionMetrics equal the reference's (golden fixture 16/21/18, 11 pairs, 0 barriers;
    TSP 27 each, 18 pairs, L barriers) on every rank;
  * every fault kind (drop / duplicate / corrupt-tag, final-layer drop, TSP corruption)
    surfaces as ProtocolError on EVERY rank, without deadlock (fixed one-message-per-link
    protocol), and the group stays usable afterwards.
"""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, scenarios, outq):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import oracle as O
    from dist_helpers import OracleExecutor
    from paper_2405_05329_b200 import kvprefill as kv
    from paper_2405_05329_b200.distributed import Transport, run_rank

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    tr = Transport()
    results = []
    for sc in scenarios:
        m = O.Model(**sc["model"])
        dt = np.float64 if m.precision == "f64" else np.float32
        w = O.init_weights(m, dt)
        ctx = O.random_context(sc["C"], m.d_model, sc["seed"], dt)
        b = sc["boundaries"]
        fault = None
        if sc.get("fault"):
            k, fr, fl = sc["fault"]
            fault = kv.FaultInjection(kv.FaultInjection.Kind(k), fr, fl)
        strat = kv.Strategy.KVR if sc["strategy"] == "kvr" else kv.Strategy.TSP
        try:
            r = run_rank(strat, ctx[b[rank]:b[rank + 1]], kv.ContextPartition(sc["C"], b), OracleExecutor(m, w), tr,
                         rank, world, m.n_layers, fault)
            results.append({"ok": True, "hidden": r.hidden_rows.tolist(), "first": r.first_token_hidden.tolist(),
                            "metrics": r.metrics.__dict__})
        except kv.Error as e:
            results.append({"ok": False, "err": type(e).__name__, "msg": str(e)})
    dist.destroy_process_group()
    outq.put((rank, results))


def _run(world, scenarios):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenarios, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res = q.get(timeout=300)
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _serial(sc):
    import oracle as O
    m = O.Model(**sc["model"])
    dt = np.float64 if m.precision == "f64" else np.float32
    return O.forward_serial(m, O.init_weights(m, dt), O.random_context(sc["C"], m.d_model, sc["seed"], dt))


SMALL = dict(d_model=16, n_heads=4, n_kv_heads=2, n_layers=2, seed=3, precision="f64", rms_norm=False)
FIX = dict(d_model=8, n_heads=2, n_kv_heads=2, n_layers=2, seed=3, precision="f64", rms_norm=False)


def test_world3_kvr_tsp_bitwise_metrics_and_faults():
    g = {f["strategy"]: f for f in GOLDEN["metrics"]}
    scenarios = [
        dict(model=FIX, C=9, seed=21, strategy="kvr", boundaries=[0, 4, 7, 9]),
        dict(model=FIX, C=9, seed=21, strategy="tsp", boundaries=[0, 3, 6, 9]),
        dict(model=SMALL, C=40, seed=100, strategy="kvr", boundaries=[0, 19, 32, 40]),
        dict(model=dict(SMALL, rms_norm=True), C=33, seed=7, strategy="tsp", boundaries=[0, 11, 22, 33]),
        dict(model=SMALL, C=12, seed=6, strategy="kvr", boundaries=[0, 4, 8, 12], fault=(1, 0, 0)),  # corrupt
        dict(model=SMALL, C=12, seed=6, strategy="kvr", boundaries=[0, 4, 8, 12], fault=(2, 0, 0)),  # drop
        dict(model=SMALL, C=12, seed=6, strategy="kvr", boundaries=[0, 4, 8, 12], fault=(3, 0, 0)),  # duplicate
        dict(model=SMALL, C=12, seed=6, strategy="kvr", boundaries=[0, 4, 8, 12], fault=(2, 0, 1)),  # final drop
        dict(model=SMALL, C=12, seed=6, strategy="tsp", boundaries=[0, 4, 8, 12], fault=(1, 1, 0)),  # tsp corrupt
        dict(model=SMALL, C=12, seed=6, strategy="kvr", boundaries=[0, 4, 8, 12]),  # group still usable
    ]
    out = _run(3, scenarios)
    for i, sc in enumerate(scenarios):
        per_rank = [out[r][i] for r in range(3)]
        if sc.get("fault"):
            assert all(not x["ok"] and x["err"] == "ProtocolError" for x in per_rank), (i, per_rank)
            continue
        assert all(x["ok"] for x in per_rank), per_rank
        hidden = np.concatenate([np.asarray(x["hidden"]) for x in per_rank])
        ref = _serial(sc)
        assert np.array_equal(hidden, ref), i  # the reference's bitwise Serial == KVR == TSP
        assert np.array_equal(np.asarray(per_rank[0]["first"]), ref[-1:])
        metrics = per_rank[0]["metrics"]
        assert all(x["metrics"] == metrics for x in per_rank)
        if i < 2:
            exp = g[sc["strategy"]]["metrics"]
            for k in ("dot_products", "kv_pairs_sent", "kv_pairs_received", "wait_events", "barrier_count"):
                assert metrics[k] == exp[k], (sc["strategy"], k)


def test_world2_even_and_skewed_f32():
    scenarios = [
        dict(model=dict(SMALL, precision="f32"), C=64, seed=9, strategy="kvr", boundaries=[0, 40, 64]),
        dict(model=dict(SMALL, precision="f32"), C=64, seed=9, strategy="tsp", boundaries=[0, 32, 64]),
    ]
    out = _run(2, scenarios)
    for i, sc in enumerate(scenarios):
        hidden = np.concatenate([np.asarray(out[r][i]["hidden"], np.float32) for r in range(2)])
        assert np.array_equal(hidden, _serial(sc))
        m = out[0][i]["metrics"]
        from paper_2405_05329_b200 import kvprefill as kv
        part = kv.ContextPartition(sc["C"], sc["boundaries"])
        strat = kv.Strategy.KVR if sc["strategy"] == "kvr" else kv.Strategy.TSP
        assert m["dot_products"] == [x * 2 for x in kv.dot_product_counts(strat, part)]
        assert sum(m["kv_pairs_sent"]) == 2 * kv.traffic_pairs(strat, part)


def test_peer_watchdog_releases_own_flags_after_timeout():
    """Host side of the peer-transport watchdog (distributed._drain_or_release) without a GPU:
    streams that never drain are given up on after the timeout; the rank then writes the run's
    largest flag value into every one of its OWN flag slots from a side stream (releasing its
    stuck GPU-side waits), lets its streams drain and reports False; streams that drain in time
    report True and signal nothing."""
    import paper_2405_05329_b200.distributed as D

    class Stream:
        def __init__(self, done_after=None):
            self.polls, self.done_after, self.synced = 0, done_after, False
            self.cuda_stream = 1234

        def query(self):
            self.polls += 1
            return self.done_after is not None and self.polls > self.done_after

        def synchronize(self):
            self.synced = True

    class Executor:
        def __init__(self, s):
            self._stream = s

    class Session:
        def __init__(self, c):
            self.comm = c

        def my_flag(self, slot):
            return 0x1000 + 4 * slot

    sent = []
    side = Stream()
    stuck_comp, stuck_comm = Stream(), Stream()
    ok = D._drain_or_release(Executor(stuck_comp), Session(stuck_comm), 77, 0.05,
                             side_stream=lambda: side, signal=lambda st, flag, v: sent.append((st, flag, v)))
    assert ok is False
    assert sent == [(1234, 0x1000 + 4 * s, 77) for s in range(D._FLAG_SLOTS)]
    assert side.synced and stuck_comp.synced and stuck_comm.synced
    sent.clear()
    assert D._drain_or_release(Executor(Stream(3)), Session(Stream(1)), 77, 5.0,
                               side_stream=lambda: side, signal=lambda *a: sent.append(a)) is True
    assert sent == []
