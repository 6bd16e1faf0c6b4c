"""Debug driver for the peer-transport watchdog: 2 processes on cuda:0, rank 0 silent."""
import os
import socket
import sys
import time

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def log(rank, *a):
    with open(f"{ROOT}/gpurun_out/dead_rank{rank}.log", "a") as f:
        print(f"{time.time():.3f}", *a, file=f, flush=True)


def worker(rank, world, port):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_2405_05329_b200 import kvprefill as kv
    from paper_2405_05329_b200 import distributed as D
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    log(rank, "init")
    W = kv.init_weights(kv.ModelConfig(1024, 8, 2, 2, 5, "bf16", True), [0])
    ex = D.GpuExecutor(W, 0)
    tr = D.Transport(peer=True)
    b = [0, 300, 517]
    ctx = O.random_context(517, 1024, 11, np.float32)
    part = kv.ContextPartition(517, b)
    for name in ("qkv", "finish"):
        fn = getattr(ex, name)

        def wrap(*a, _fn=fn, _name=name):
            log(rank, _name, a)
            r = _fn(*a)
            log(rank, _name, "ok")
            return r
        setattr(ex, name, wrap)
    orig = D._drain_or_release

    def traced(executor, ps, top, t):
        log(rank, "drain start top", top)
        r = orig(executor, ps, top, t)
        log(rank, "drain done", r)
        return r
    D._drain_or_release = traced
    os.environ["KVP_PEER_SILENT_RANK"] = "0"
    os.environ["KVP_PEER_TIMEOUT_S"] = "3"
    try:
        D.run_rank(kv.Strategy.KVR, ctx[b[rank]:b[rank + 1]], part, ex, tr, rank, world, 2)
        log(rank, "run 1 returned")
    except kv.ProtocolError as e:
        log(rank, "run 1 ProtocolError", e)
    os.environ["KVP_PEER_SILENT_RANK"] = "-1"
    res = D.run_rank(kv.Strategy.KVR, ctx[b[rank]:b[rank + 1]], part, ex, tr, rank, world, 2)
    log(rank, "run 2 ok", res.hidden_rows.shape)
    dist.destroy_process_group()


if __name__ == "__main__":
    for r in range(2):
        try:
            os.remove(f"{ROOT}/gpurun_out/dead_rank{r}.log")
        except OSError:
            pass
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, port)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        print("exit", p.exitcode)
        if p.exitcode is None:
            p.kill()
