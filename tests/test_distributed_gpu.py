"""Multi-process KV-Runahead on the GPU: two processes (ranks) sharing cuda:0 -- the only
device this run has -- each driving its own B200 layer executor through the kvp_rank_* C-ABI,
with the KV handoff moved by the distributed driver over gloo (host-staged; on a multi-GPU
node the same code moves it with NCCL over NVLink).  The assembled result must equal the
in-process engine bitwise (Serial == KVR across process boundaries)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, strategy, runs, peer, outq):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2405_05329_b200 import kvprefill as kv
    from paper_2405_05329_b200.distributed import GpuExecutor, Transport, run_rank

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "bf16", True), [0])
    ex = GpuExecutor(W, 0)
    tr = Transport(peer=peer)
    strat = kv.Strategy.KVR if strategy == "kvr" else kv.Strategy.TSP
    out = []
    for boundaries in runs:  # consecutive runs on one executor (buffer / mapping reuse)
        C_ = boundaries[-1]
        ctx = O.random_context(C_, 1024, 11, np.float32)
        res = run_rank(strat, ctx[boundaries[rank]:boundaries[rank + 1]], kv.ContextPartition(C_, boundaries),
                       ex, tr, rank, world, 2)
        out.append((res.hidden_rows, res.metrics.__dict__))
    outq.put((rank, out))
    dist.destroy_process_group()


def _run_procs(world, strategy, runs, peer):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, strategy, runs, peer, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


def _check(got, world, strategy, runs):
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2405_05329_b200 import kvprefill as kv
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "bf16", True), [0])
    strat = kv.Strategy.KVR if strategy == "kvr" else kv.Strategy.TSP
    for i, boundaries in enumerate(runs):
        hidden = np.concatenate([got[r][i][0] for r in range(world)])
        C_ = boundaries[-1]
        ref = kv.run(kv.Strategy.Serial, O.random_context(C_, 1024, 11, np.float32), kv.even_partition(C_, 1), W)
        assert np.array_equal(hidden, ref.hidden_out), (strategy, boundaries)
        part = kv.ContextPartition(C_, boundaries)
        m = got[0][i][1]
        assert m["dot_products"] == [x * 2 for x in kv.dot_product_counts(strat, part)]
        assert sum(m["kv_pairs_sent"]) == 2 * kv.traffic_pairs(strat, part)
        assert sum(m["kv_pairs_received"]) == 2 * kv.traffic_pairs(strat, part)


@pytest.mark.parametrize("strategy,boundaries", [("kvr", [0, 300, 517]), ("tsp", [0, 259, 517])])
def test_two_processes_match_in_process_engine(strategy, boundaries):
    from paper_2405_05329_b200 import kvprefill as kv
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")
    got = _run_procs(2, strategy, [boundaries], False)
    _check(got, 2, strategy, [boundaries])


@pytest.mark.parametrize("strategy,world,runs", [
    ("kvr", 2, [[0, 300, 517], [0, 300, 517], [0, 100, 517]]),
    ("kvr", 3, [[0, 200, 390, 517], [0, 200, 390, 517]]),
    ("tsp", 3, [[0, 173, 345, 517], [0, 100, 345, 517]]),
])
def test_peer_memory_handoff_processes(strategy, world, runs):
    """The fused handoff over peer memory (Transport(peer=True)): CUDA IPC mappings of the
    other processes' caches, the QKV epilogue storing the K/V rows into them, stream-ordered
    flags instead of messages, KVR prefix forwarded by the copy engine.  Several runs on one
    executor (epoch-numbered flags, mappings re-opened when the partition changes); results
    bitwise equal to the serial run, accounting equal to the reference's."""
    from paper_2405_05329_b200 import kvprefill as kv
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")
    got = _run_procs(world, strategy, runs, True)
    _check(got, world, strategy, runs)


def test_bench_multi_rank_path_on_one_gpu():
    """bench.py's N>1 path (one process per rank under torchrun: KVR even / KVR-S search / TSP
    all-gather) end to end on the single GPU of this box, with the test hooks that share cuda:0
    and use gloo; on a multi-GPU node the same code runs over NCCL."""
    import json
    import subprocess
    env = dict(os.environ, KVP_BENCH_SHARE_GPU="1", KVP_BENCH_BACKEND="gloo")
    for i, extra in enumerate(([], ["--partition", "search"], ["--strategy", "tsp"], ["--transport", "msg"],
                               ["--strategy", "tsp", "--transport", "msg"])):
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                            "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                            os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "tiny", "--steps", "2",
                            "--warmup", "3", *extra], capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-3000:]
        lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, r.stdout[-2000:]
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
        assert d["config"]["partition"][0] == 0 and d["config"]["partition"][-1] == 1024
        if i == 0:  # the north-star comparison rides every N>1 line
            t = d["strategies"]
            assert {"kvr_even", "kvr_s", "tsp"} <= set(t) and t["kvr_s_over_tsp"] > 0
            assert t["kvr_s"]["partition"][-1] == 1024 and len(d["kernels_per_rank"]) == 2
            assert d["e2e"]["value"] > 0


def test_bench_noise_sidecar_on_one_gpu():
    """bench.py's physical noise study: the reference's seeded per-layer link
    draw drives real background copies into the next rank's memory during the KVR-S and TSP
    runs; the line carries per-trial degradations beside the simulator's noise_study."""
    import json
    import subprocess
    env = dict(os.environ, KVP_BENCH_SHARE_GPU="1", KVP_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "3",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                        os.path.join(ROOT, "bench.py"), "--gpus", "3", "--workload", "tiny", "--steps", "2",
                        "--warmup", "3", "--no-e2e", "--noise-factor", "2", "--noise-trials", "2"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    ns = d["noise_sidecar"]
    assert "error" not in ns and "skipped" not in ns, ns
    for k in ("kvr_s", "tsp"):
        assert len(ns[k]["noisy_ms"]) == 2 and all(x > 0 for x in ns[k]["noisy_ms"])
        assert ns[k]["injected_bytes_total"] > 0
        assert len(ns["simulated"][k]["per_trial"]) == 2


def test_bench_single_process_ranks_table():
    """python bench.py --gpus 1 --ranks 4: the in-process engine with 4 ranks on one GPU; the
    line carries KVR even / KVR-S / TSP TTFTs on the same kernels and the busiest link's
    handoff copy, and the prompt's first token matches the reference's golden argmax."""
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--ranks", "4", "--workload",
                        "tiny", "--steps", "2", "--warmup", "3", "--partition", "search", "--no-cpu-baseline",
                        "--no-decode"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    t = d["strategies"]
    assert {"kvr_even", "kvr_s", "tsp"} <= set(t), t
    assert d["config"]["ranks"] == 4 and len(d["config"]["partition"]) == 5
    assert d["kv_handoff"]["bytes_per_layer"] > 0
    assert d["first_token_matches_reference"] is True


def _decode_worker(rank, world, port, outq):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2405_05329_b200 import kvprefill as kv
    from paper_2405_05329_b200.distributed import GpuExecutor, Transport, decode_on_last_rank, run_rank

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "f32", True), [0])
    b = [0, 200, 331]
    ctx = O.random_context(335, 1024, 13, np.float32)
    ex = GpuExecutor(W, 0, decode_capacity=8)
    run_rank(kv.Strategy.KVR, ctx[b[rank]:b[rank + 1]], kv.ContextPartition(331, b), ex, Transport(), rank, world, 2)
    out = decode_on_last_rank(ex, ctx[331:335], 331, rank, world)
    outq.put((rank, out))
    dist.destroy_process_group()


def test_decode_on_last_rank_after_kvr():
    """The last KVR rank decodes on the prompt's cache (f32 mode: bitwise equal to the serial
    forward over the longer context), result broadcast to every rank."""
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2405_05329_b200 import kvprefill as kv
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_decode_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "f32", True), [0])
    full = kv.run(kv.Strategy.Serial, O.random_context(335, 1024, 13, np.float32), kv.even_partition(335, 1), W)
    assert np.array_equal(got[0], got[1])
    assert np.array_equal(got[1], full.hidden_out[331:335])


def _silent_worker(rank, world, port, strategy, outq):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2405_05329_b200 import kvprefill as kv
    from paper_2405_05329_b200.distributed import GpuExecutor, Transport, run_rank

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "bf16", True), [0])
    ex = GpuExecutor(W, 0)
    tr = Transport(peer=True)
    strat = kv.Strategy.KVR if strategy == "kvr" else kv.Strategy.TSP
    b = [0, 300, 517] if world == 2 else [0, 200, 390, 517]
    ctx = O.random_context(517, 1024, 11, np.float32)
    part = kv.ContextPartition(517, b)
    os.environ["KVP_PEER_SILENT_RANK"] = "0"
    os.environ["KVP_PEER_TIMEOUT_S"] = "3"
    err = None
    try:
        run_rank(strat, ctx[b[rank]:b[rank + 1]], part, ex, tr, rank, world, 2)
    except kv.ProtocolError as e:
        err = str(e)
    # the streams drained and the mappings were dropped: the next run on the same executors works
    os.environ["KVP_PEER_SILENT_RANK"] = "-1"
    res = run_rank(strat, ctx[b[rank]:b[rank + 1]], part, ex, tr, rank, world, 2)
    outq.put((rank, (err, res.hidden_rows)))
    dist.destroy_process_group()


@pytest.mark.parametrize("strategy,world", [("kvr", 2), ("kvr", 3), ("tsp", 2)])
def test_peer_handoff_dead_peer_raises_protocol_error(strategy, world):
    """Hang safety of the peer-memory transport: rank 0 never signals (KVP_PEER_SILENT_RANK),
    so its receivers' GPU-side flag waits would block forever; the watchdog releases them after
    KVP_PEER_TIMEOUT_S and EVERY rank raises ProtocolError (the reference's abort_all wakes all
    blocked receivers, channel.hpp:120-136).  The same executors then run cleanly, bitwise
    equal to the serial run."""
    from paper_2405_05329_b200 import kvprefill as kv
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_silent_worker, args=(r, world, port, strategy, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        assert got[r][0] is not None and "timed out" in got[r][0], got[r][0]
    import oracle as O
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "bf16", True), [0])
    ref = kv.run(kv.Strategy.Serial, O.random_context(517, 1024, 11, np.float32), kv.even_partition(517, 1), W)
    assert np.array_equal(np.concatenate([got[r][1] for r in range(world)]), ref.hidden_out)
