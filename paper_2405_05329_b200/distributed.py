"""Multi-process KV-Runahead: one process per GPU, one rank per process.

The reference runs its ranks as threads exchanging typed messages through Channels
(engine.hpp:223-296, channel.hpp).  Here each rank is a process (torchrun) that drives its
own B200 layer executor through the per-rank C-ABI (kvp_rank_*), and the KV-cache handoff
is point-to-point over a torch.distributed group -- NCCL over NVLink between GPUs, or gloo
for CPU tests -- ordered on the executor's CUDA stream so layer l's transfer overlaps the
sender's layer l+1 compute.

Wire protocol (per link, per layer EXACTLY one message, so a collective transport can never
deadlock): header int64[8] = {MAGIC, kind, layer, source, start, end, 0, 0} followed by the K
and V rows.  The reference's fault injections (send_with_faults, engine.hpp:143-164) become
edits of a per-link outbox: CorruptLayerTag bumps the header's layer, DropMessage leaves the
slot to a CLOSED tombstone, DuplicateMessage re-queues the message so every later slot is
shifted.  Receivers validate headers exactly like recv_checked (engine.hpp:166-179) after the
run; the first error (lowest layer, then rank) is agreed over the group and raised on every
rank, like Fabric::abort_all + rethrow_if_failed (channel.hpp:120-136).

Hang safety of the peer-memory transport: its flag waits are enqueued on the GPU
(cuStreamWaitValue32), so a peer that dies or never signals would block the stream for good.
Before reading its result each rank polls its streams against a deadline
(KVP_PEER_TIMEOUT_S, default 120 s); on expiry it writes the awaited values into its OWN flag
words from a side stream (the stuck waits release, the stream drains) and reports a
ProtocolError that the post-run agreement raises on every rank, after which every rank drops
its peer session -- the analogue of Channel::close waking blocked receivers
(channel.hpp:15-18, 120-136).
"""
from __future__ import annotations

import collections
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import kvprefill as kv

HDR_LEN = 8
MAGIC = 0x4B56524E
KIND_HANDOFF, KIND_GATHER, KIND_CLOSED = 0, 1, 2
_ERR_CODES = {kv.ProtocolError: 6, kv.CacheError: 3}
_ERR_BY_CODE = {6: kv.ProtocolError, 3: kv.CacheError}


# ------------------------------------------------------------------ transport
class Transport:
    """Blocking point-to-point tensor moves over a torch.distributed group.  With NCCL the
    tensors stay on the GPU and the ops are ordered on the caller's current CUDA stream.  With
    gloo, CUDA tensors are staged through host memory (shared-GPU / CPU test runs)."""

    def __init__(self, group=None, peer: Optional[bool] = None):
        """peer: move K/V through peer memory (CUDA IPC mappings of the other ranks' caches,
        NVLink between GPUs) instead of messages -- the QKV epilogue stores the rows straight
        into the receiver's cache and stream-ordered flags say they have landed; the group
        then only carries host metadata.  Default (peer=None): messages, unless the
        environment says KVP_TRANSPORT=peer; bench.py passes peer=True explicitly."""
        import os
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.backend = dist.get_backend(group)
        if peer is None:
            peer = os.environ.get("KVP_TRANSPORT", "") == "peer"
        self.peer = bool(peer) and self._peer_reachable()
        self.peer_requested = bool(peer)

    def _peer_reachable(self) -> bool:
        """The peer transport needs every rank's device to reach every other rank's device
        (same device, or CUDA peer access over NVLink).  Agreed over the group, so all ranks
        take the same transport (collective: every rank constructs its Transport at the same
        point); without CUDA the executors are not device-resident and peer_ok() is False."""
        import torch
        if not torch.cuda.is_available():
            return True
        dist, world = self.dist, self.dist.get_world_size(self.group)
        dev = torch.cuda.current_device()
        devs = [None] * world
        dist.all_gather_object(devs, dev, group=self.group)
        ok = all(d == dev or torch.cuda.can_device_access_peer(dev, d) for d in devs)
        votes = [None] * world
        dist.all_gather_object(votes, ok, group=self.group)
        return all(votes)

    def peer_ok(self, executor) -> bool:
        """The fused peer-memory handoff needs bf16 CUDA executors (tcgen05 QKV epilogue)."""
        dev = getattr(executor, "device", None)
        return (self.peer and dev is not None and getattr(dev, "type", "cpu") == "cuda"
                and executor.cfg.precision == kv.Precision.bf16)

    def _staged(self, t) -> bool:
        return self.backend == "gloo" and t.is_cuda

    def collective_ok(self, executor) -> bool:
        """All-gather collectives run directly on the executor's tensors: NCCL (device) or gloo
        with host tensors; gloo with CUDA tensors keeps the staged point-to-point path."""
        dev = getattr(executor, "device", None)
        on_cuda = dev is not None and getattr(dev, "type", "cpu") == "cuda"
        return self.backend == "nccl" or not on_cuda

    def all_gather_rows(self, buf, start: int, stop: int, C_: int) -> None:
        """buf[start:stop] of every rank into buf[0:C] (equal chunks, rank order).  The layer
        plane may hold more rows (decode capacity): only the prompt's C rows are gathered."""
        self.dist.all_gather_into_tensor(buf[:C_], buf[start:stop].clone(), group=self.group)

    def exchange(self, sends, recvs, wait: bool = True):
        """sends: [(tensor, dst)], recvs: [(tensor, src)] -- one batched group.  wait=False
        (sends only) returns (pending works, the tensors actually on the wire) instead of
        joining them: with NCCL the transfer then runs on the communicator's own stream,
        overlapping the caller's later kernels; the caller keeps the returned tensors alive
        (host-staged copies included: gloo does not) until it joins the works."""
        import torch
        dist = self.dist
        staged_recv = []
        ops = []
        wire = []
        for t, dst in sends:
            if self._staged(t):
                torch.cuda.current_stream().synchronize()
                t = t.cpu()
            t = t.contiguous()
            wire.append(t)
            ops.append(dist.P2POp(dist.isend, t, dst, self.group))
        for t, src in recvs:
            if self._staged(t):
                host = torch.empty(t.shape, dtype=t.dtype)
                staged_recv.append((host, t))
                t = host
            ops.append(dist.P2POp(dist.irecv, t, src, self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        if not wait:
            if recvs:
                raise ValueError("deferred exchange is for sends only")
            return works, wire
        for w in works:
            w.wait()
        for host, dev in staged_recv:
            dev.copy_(host, non_blocking=False)
        return []


# ------------------------------------------------------------------ executors
class GpuExecutor:
    """One rank's B200 layer executor (kvp_rank_* C-ABI); K/V buffers are torch tensors so
    the transport can address them."""

    def __init__(self, weights: kv.WeightSet, device: int = 0, decode_capacity: int = 0):
        """decode_capacity: extra K/V rows kept free after the prompt for decode steps."""
        import torch
        self.torch = torch
        self.w = weights
        self.cfg = weights.config
        self.device = torch.device("cuda", device)
        self.dtype = torch.bfloat16 if self.cfg.precision == kv.Precision.bf16 else torch.float32
        self.decode_capacity = int(decode_capacity)
        self._stream = None
        self.kvbuf = None
        self.peer = None  # _PeerSession of the fused peer-memory handoff

    def begin(self, rows, start: int, held: int):
        torch = self.torch
        import ctypes as C
        L, kvd = self.cfg.n_layers, self.cfg.kv_dim()
        shape = (L, 2, held + self.decode_capacity, kvd)
        if self.kvbuf is None or tuple(self.kvbuf.shape) != shape:
            # kept across runs of the same shape: peers hold IPC mappings of it
            self.kvbuf = torch.zeros(shape, dtype=self.dtype, device=self.device)
        self.held = held
        ptrs = (C.c_void_p * (2 * L))(*[self.kvbuf[l, i].data_ptr() for l in range(L) for i in range(2)])
        self._ptrs = ptrs
        if isinstance(rows, torch.Tensor):
            rows_t = rows.to(self.device, torch.float32).contiguous()
            self._rows = rows_t
            ptr, on_dev = rows_t.data_ptr(), 1
        else:
            rows_np = np.ascontiguousarray(rows, dtype=np.float32)
            self._rows = rows_np
            ptr, on_dev = rows_np.ctypes.data, 0
        self.n_rows = int(self._rows.shape[0])
        kv._check(kv.lib().kvp_rank_begin(self.w.handle, C.c_void_p(ptr), self.n_rows, start, held, on_dev, ptrs),
                  "rank_begin")
        s = C.c_void_p()
        kv._check(kv.lib().kvp_rank_stream(self.w.handle, C.byref(s)), "rank_stream")
        self._stream = torch.cuda.ExternalStream(s.value, device=self.device)

    def stream(self):
        return self.torch.cuda.stream(self._stream)

    def decode(self, rows, position: int):
        """Decode step on this rank's cache (which holds rows [0, position)): appends the rows
        (n <= 8) at [position, position + n) with the decode kernels; returns their final
        hidden rows (host)."""
        import ctypes as C
        r = np.ascontiguousarray(rows, dtype=np.float32)
        n = int(r.shape[0])
        cap = self.held + self.decode_capacity
        if position + n > cap:
            raise kv.CacheError(f"decode needs {position + n} cache rows, the rank holds {cap}")
        lib = kv.lib()
        kv._check(lib.kvp_rank_begin(self.w.handle, C.c_void_p(r.ctypes.data), n, position, cap, 0, self._ptrs),
                  "rank_begin (decode)")
        kv._check(lib.kvp_rank_set_decode(self.w.handle, 1), "rank_set_decode")
        for layer in range(self.cfg.n_layers):
            kv._check(lib.kvp_rank_qkv(self.w.handle, layer), "rank_qkv (decode)")
            kv._check(lib.kvp_rank_finish(self.w.handle, layer, position + n), "rank_finish (decode)")
        out = np.empty((n, self.cfg.d_model), np.float32)
        kv._check(lib.kvp_rank_end(self.w.handle, C.c_void_p(out.ctypes.data), 0, None, None), "rank_end (decode)")
        return out

    def kv(self, layer: int):
        return self.kvbuf[layer, 0], self.kvbuf[layer, 1]

    def qkv(self, layer: int):
        kv._check(kv.lib().kvp_rank_qkv(self.w.handle, layer), "rank_qkv")

    def finish(self, layer: int, k_rows: int):
        kv._check(kv.lib().kvp_rank_finish(self.w.handle, layer, k_rows), "rank_finish")

    def end(self):
        import ctypes as C
        out = np.empty((self.n_rows, self.cfg.d_model), np.float32)
        ms = C.c_float()
        kv._check(kv.lib().kvp_rank_end(self.w.handle, C.c_void_p(out.ctypes.data), 0, None, C.byref(ms)), "rank_end")
        return out, float(ms.value)

    def close(self):
        """Releases the IPC mappings of the peer transport (the caches themselves are torch
        tensors and go with the executor).  Collective: every rank of the group closes (or
        re-creates) its executor together, because the next peer run re-exchanges handles
        with an all-gather that every rank must join."""
        if self.peer is not None:
            self.peer.close()
            self.peer = None

    def raw_stream(self) -> int:
        return self._stream.cuda_stream

    def set_mirrors(self, bufs):
        """bufs: per mirror, 2L device pointers (K_0, V_0, ...) of another rank's cache."""
        import ctypes as C
        flat = [ptr for mirror in bufs for ptr in mirror]
        arr = (C.c_void_p * max(1, len(flat)))(*flat)
        kv._check(kv.lib().kvp_rank_set_mirrors(self.w.handle, len(bufs), arr), "rank_set_mirrors")

    def header(self, values):
        return self.torch.tensor(values, dtype=self.torch.int64, device=self.device)

    def empty_header(self):
        return self.torch.zeros(HDR_LEN, dtype=self.torch.int64, device=self.device)


# ------------------------------------------------------------------ peer-memory handoff
_FLAG_SLOTS = 64  # one int32 per source rank (TSP) / {own rows, forwarded prefix} (KVR)


def _ipc_export(ptr: int):
    import ctypes as C
    h = (C.c_ubyte * 64)()
    off = C.c_int64()
    kv._check(kv.lib().kvp_ipc_export(C.c_void_p(ptr), h, C.byref(off)), "ipc_export")
    return bytes(h), int(off.value)


class _PeerSession:
    """CUDA IPC mappings of the other ranks' KV caches and flag words (opened once per
    partition / strategy, re-used by every run) plus a monotonically growing run epoch: the
    flag value of layer l in run e is e*L + l + 1, so a GEQ wait never needs a reset."""

    def __init__(self, executor):
        torch = executor.torch
        self.ex = executor
        self.flags = torch.zeros(_FLAG_SLOTS, dtype=torch.int32, device=executor.device)
        self.comm = torch.cuda.Stream(device=executor.device)
        self.epoch = 0
        self.key = None
        self.bases = {}     # handle bytes -> mapped base pointer
        self.peers = {}     # rank -> {"kv": [2L ptrs], "flags": ptr}

    def _open(self, handle: bytes) -> int:
        import ctypes as C
        if handle not in self.bases:
            ptr = C.c_void_p()
            kv._check(kv.lib().kvp_ipc_open(handle, 0, C.byref(ptr)), "ipc_open")
            self.bases[handle] = int(ptr.value)
        return self.bases[handle]

    def close(self):
        import ctypes as C
        for base in self.bases.values():
            kv.lib().kvp_ipc_close(C.c_void_p(base), 0)
        self.bases.clear()
        self.peers.clear()

    def setup(self, key, rank: int, world: int, group):
        """Exchange handles when the partition / strategy (hence every rank's buffers)
        changed -- the same decision on every rank, so the collective is always matched."""
        import torch.distributed as dist
        if key == self.key:
            return
        ex = self.ex
        torch = ex.torch
        torch.cuda.current_stream(ex.device).synchronize()
        mine = {"kv": _ipc_export(ex.kvbuf.data_ptr()), "rows": int(ex.kvbuf.shape[2]),
                "flags": _ipc_export(self.flags.data_ptr()), "epoch": self.epoch}
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        # every rank continues from the same epoch: a rank whose session is younger (its
        # executor was re-created) must not wait on flag values another rank's earlier runs
        # already wrote (GEQ waits would pass early)
        self.epoch = max(info["epoch"] for info in everyone)
        self.close()
        L, kvd = ex.cfg.n_layers, ex.cfg.kv_dim()
        es = ex.kvbuf.element_size()
        for j, info in enumerate(everyone):
            if j == rank:
                continue
            base = self._open(info["kv"][0]) + info["kv"][1]
            plane = info["rows"] * kvd * es
            self.peers[j] = {"kv": [base + (2 * l + i) * plane for l in range(L) for i in range(2)],
                             "flags": self._open(info["flags"][0]) + info["flags"][1]}
        self.key = key

    def flag(self, j: int, slot: int) -> int:
        return self.peers[j]["flags"] + 4 * slot

    def my_flag(self, slot: int) -> int:
        return self.flags.data_ptr() + 4 * slot


def _signal(stream: int, flag: int, value: int):
    import ctypes as C
    kv._check(kv.lib().kvp_stream_signal(C.c_void_p(stream), C.c_void_p(flag), value), "stream_signal")


def _wait(stream: int, flag: int, value: int):
    import ctypes as C
    kv._check(kv.lib().kvp_stream_wait(C.c_void_p(stream), C.c_void_p(flag), value), "stream_wait")


def _peer_timeout_s() -> float:
    return float(os.environ.get("KVP_PEER_TIMEOUT_S", "120"))


def _silent_rank() -> int:
    """Hang-safety test hook: KVP_PEER_SILENT_RANK=r makes rank r skip every flag signal of
    the peer transport (a peer that never delivers), so its receivers must time out."""
    return int(os.environ.get("KVP_PEER_SILENT_RANK", "-1"))


def _drain_or_release(executor, ps, top_value: int, timeout_s: float, side_stream=None,
                      signal=None) -> bool:
    """Waits until the rank's compute and comm streams are idle.  True if they drained in
    time; otherwise releases the rank's own stuck flag waits (writes top_value, the largest
    flag value of this run, into every flag slot from a side stream), lets the streams drain
    and returns False (the caller agrees the error and every rank drops its peer session).
    side_stream / signal: injectable for tests (default: a fresh CUDA stream, _signal)."""
    streams = (executor._stream, ps.comm)
    t0 = time.monotonic()
    deadline = t0 + timeout_s
    while not all(s.query() for s in streams):
        now = time.monotonic()
        if now > deadline:
            side = side_stream() if side_stream else executor.torch.cuda.Stream(device=executor.device)
            for slot in range(_FLAG_SLOTS):
                (signal or _signal)(side.cuda_stream, ps.my_flag(slot), top_value)
            side.synchronize()
            for s in streams:
                s.synchronize()
            return False
        if now - t0 > 0.02:  # busy-poll the first 20 ms (the normal case), then back off
            time.sleep(0.001)
    return True


def _warm_kernels(executor, rows, start: int, held: int, k_rows: int, n_layers: int):
    """Runs this chunk shape once through the local layer executor (no peer, no flags, result
    discarded) the first time it is seen.  CUDA loads kernels lazily at their first launch and
    the load waits for the device to drain; in a peer run the first launches after a flag wait
    (attention, FFN) would otherwise wait on a stream that is itself blocked on a peer -- a
    dead peer would then hang the host before the watchdog can act."""
    key = (id(executor.w), len(rows), start, held, k_rows)
    seen = executor.__dict__.setdefault("_warm", set())
    if key in seen:
        return
    executor.begin(rows, start, held)
    executor.set_mirrors([])
    for layer in range(n_layers):
        executor.qkv(layer)
        executor.finish(layer, k_rows)
    executor.end()
    seen.add(key)


def _copy(stream: int, dst: int, src: int, nbytes: int):
    import ctypes as C
    kv._check(kv.lib().kvp_stream_copy(C.c_void_p(stream), C.c_void_p(dst), C.c_void_p(src), nbytes), "stream_copy")


# ------------------------------------------------------------------ the rank driver
@dataclass
class RankResult:
    hidden_rows: np.ndarray           # this rank's final hidden rows [c_i x d]
    first_token_hidden: np.ndarray    # row C-1 (broadcast from the last rank), [1 x d]
    metrics: kv.ExecutionMetrics      # global, identical on every rank
    device_ms: float                  # this rank's device time
    ttft_ms: float                    # max over ranks


@dataclass
class _Link:
    outbox: collections.deque = field(default_factory=collections.deque)


def _header(kind, layer, source, start, end):
    return [MAGIC, kind, layer, source, start, end, 0, 0]


def _apply_fault(fault: Optional[kv.FaultInjection], rank: int, msg: list, link: _Link, counter: list):
    """send_with_faults (engine.hpp:143-164) as an outbox edit; returns nothing."""
    pairs = msg[5] - msg[4]
    K = kv.FaultInjection.Kind
    if fault is not None and fault.kind != K.None_ and fault.rank == rank and fault.layer == msg[2]:
        if fault.kind == K.DropMessage:
            return
        if fault.kind == K.CorruptLayerTag:
            msg = list(msg)
            msg[2] += 1
        if fault.kind == K.DuplicateMessage:
            link.outbox.append(list(msg))
            counter[0] += pairs
    link.outbox.append(list(msg))
    counter[0] += pairs


def _check_header(h, kind, layer, start_expected, end_expected):
    """recv_checked (engine.hpp:166-179) + the KVR prefix check (engine.hpp:272-275)."""
    h = [int(x) for x in h]
    if h[0] != MAGIC or h[1] == KIND_CLOSED:
        return kv.ProtocolError, "channel closed before message arrived"
    if h[1] != kind:
        return kv.ProtocolError, "unexpected message kind"
    if h[2] != layer:
        return kv.ProtocolError, (f"expected message for layer {layer}, got layer {h[2]} "
                                  "(duplicate, dropped, or corrupt handoff)")
    if not (0 <= h[4] < h[5]):
        return kv.CacheError, "segment positions must satisfy 0 <= start < end"
    if (h[4], h[5]) != (start_expected, end_expected):
        return kv.CacheError, (f"handoff covers [{h[4]}, {h[5]}), expected [{start_expected}, {end_expected})")
    return None


def run_rank(strategy: kv.Strategy, rows, partition: kv.ContextPartition, executor, transport: Transport,
             rank: int, world: int, n_layers: int, fault: Optional[kv.FaultInjection] = None,
             group=None) -> RankResult:
    """One rank of run(strategy, context, partition, weights, fault) (engine.hpp:186-318)."""
    import torch.distributed as dist

    partition.validate()
    b = partition.boundaries
    p = partition.process_count()
    if p != world:
        raise kv.InputError(f"partition has {p} ranks but the group has {world}")
    if strategy == kv.Strategy.Serial and p != 1:
        raise kv.InputError("serial strategy requires p == 1")
    C_ = partition.context_length
    start, stop = b[rank], b[rank + 1]
    c = stop - start
    held = stop if strategy == kv.Strategy.KVR else C_
    no_fault = fault is None or fault.kind == kv.FaultInjection.Kind.None_
    # fused peer-memory handoff (no fault injected: faults are message edits, so they keep
    # the message path): the QKV epilogue stores this rank's K/V rows into the receivers'
    # caches; KVR forwards the upstream prefix with one copy-engine copy per tensor as soon
    # as it has landed; stream-ordered flags replace the messages
    use_peer = (no_fault and p > 1 and strategy in (kv.Strategy.KVR, kv.Strategy.TSP) and transport.peer_ok(executor)
            and (strategy == kv.Strategy.KVR or p - 1 <= 8))
    if use_peer:
        _warm_kernels(executor, rows, start, held, stop if strategy == kv.Strategy.KVR else C_, n_layers)
    executor.begin(rows, start, held)

    dots = sent = recvd = waits = 0
    barriers = 0
    inbound = []  # (header tensor, kind, layer, expected start, expected end)
    out_links = collections.defaultdict(_Link)
    sent_ctr = [0]
    in_flight = []  # KVR handoff sends still on the wire (joined before the rank's result)
    sizes = [b[i + 1] - b[i] for i in range(p)]
    gather_collective = (strategy == kv.Strategy.TSP and no_fault and p > 1 and len(set(sizes)) == 1
                         and transport.collective_ok(executor))
    if use_peer:
        if executor.peer is None:
            executor.peer = _PeerSession(executor)
        ps = executor.peer
        ps.setup((tuple(b), int(strategy), world), rank, world, group)
        ps.epoch += 1
        L = n_layers
        es = executor.kvbuf.element_size()
        row_bytes = executor.cfg.kv_dim() * es
        comp, comm = executor.raw_stream(), ps.comm.cuda_stream
        targets = ([rank + 1] if rank + 1 < p else []) if strategy == kv.Strategy.KVR else \
            [j for j in range(p) if j != rank]
        executor.set_mirrors([ps.peers[j]["kv"] for j in targets])
        signal = _signal if _silent_rank() != rank else (lambda *_: None)
    for layer in range(n_layers):
        executor.qkv(layer)
        K, V = executor.kv(layer)
        if use_peer:
            v = ps.epoch * L + layer + 1
            if strategy == kv.Strategy.KVR:
                OWN, PREFIX = 0, 1
                if rank + 1 < p:
                    signal(comp, ps.flag(rank + 1, OWN), v)  # rows [start, stop) are at rank+1
                    sent_ctr[0] += stop
                if rank > 0:
                    waits += 1
                    recvd += start
                    for st in ((comp, comm) if rank + 1 < p else (comp,)):
                        _wait(st, ps.my_flag(OWN), v)
                        if rank > 1:
                            _wait(st, ps.my_flag(PREFIX), v)
                    if rank + 1 < p:  # forward [0, start) on the copy engine
                        dst = ps.peers[rank + 1]["kv"]
                        _copy(comm, dst[2 * layer], K.data_ptr(), start * row_bytes)
                        _copy(comm, dst[2 * layer + 1], V.data_ptr(), start * row_bytes)
                        signal(comm, ps.flag(rank + 1, PREFIX), v)
                k_rows = stop
            else:
                for j in targets:
                    signal(comp, ps.flag(j, rank), v)
                for j in targets:
                    _wait(comp, ps.my_flag(j), v)
                    sent_ctr[0] += stop - start
                    waits += 1
                    recvd += b[j + 1] - b[j]
                waits += 1
                barriers += 1
                k_rows = C_
            dots += c * k_rows
            executor.finish(layer, k_rows)
            continue
        with executor.stream():
            if strategy == kv.Strategy.KVR:
                sends, recvs = [], []
                if rank > 0:
                    hin = executor.empty_header()
                    recvs += [(hin, rank - 1), (K[:start], rank - 1), (V[:start], rank - 1)]
                    inbound.append((hin, KIND_HANDOFF, layer, 0, start))
                    waits += 1
                    recvd += start
                if rank + 1 < p:
                    link = out_links[rank + 1]
                    _apply_fault(fault, rank, _header(KIND_HANDOFF, layer, rank, 0, stop), link, sent_ctr)
                    msg = link.outbox.popleft() if link.outbox else _header(KIND_CLOSED, layer, rank, 0, stop)
                    sends += [(executor.header(msg), rank + 1), (K[:stop], rank + 1), (V[:stop], rank + 1)]
                # the receive must land before the cumulative cache is forwarded (and before
                # this layer's attention); the send is NOT joined here: layer l's K/V buffers
                # are never written again, so its transfer to rank i+1 overlaps this rank's
                # attention/FFN of layer l and the layers after it
                transport.exchange([], recvs)
                in_flight.append(transport.exchange(sends, [], wait=False))  # (works, tensors kept alive)
                k_rows = stop
            elif strategy == kv.Strategy.TSP and gather_collective:
                # no fault can be injected and the chunks are equal: the all-gather is ONE
                # collective per tensor (NCCL all-gather over NVLink/NVSwitch), in place in the
                # [C x kv] layer buffer; the accounting is the reference's
                transport.all_gather_rows(K, start, stop, C_)
                transport.all_gather_rows(V, start, stop, C_)
                for peer in range(p):
                    if peer != rank:
                        sent_ctr[0] += stop - start
                        waits += 1
                        recvd += b[peer + 1] - b[peer]
                waits += 1
                barriers += 1
                k_rows = C_
            elif strategy == kv.Strategy.TSP:
                sends, recvs = [], []
                for peer in range(p):
                    if peer == rank:
                        continue
                    link = out_links[peer]
                    _apply_fault(fault, rank, _header(KIND_GATHER, layer, rank, start, stop), link, sent_ctr)
                    msg = link.outbox.popleft() if link.outbox else _header(KIND_CLOSED, layer, rank, start, stop)
                    sends += [(executor.header(msg), peer), (K[start:stop], peer), (V[start:stop], peer)]
                    hin = executor.empty_header()
                    lo, hi = b[peer], b[peer + 1]
                    recvs += [(hin, peer), (K[lo:hi], peer), (V[lo:hi], peer)]
                    inbound.append((hin, KIND_GATHER, layer, lo, hi))
                    waits += 1
                    recvd += hi - lo
                transport.exchange(sends, recvs)  # the all-gather is the per-layer barrier
                waits += 1
                barriers += 1
                k_rows = C_
            else:
                k_rows = C_
        dots += c * k_rows
        executor.finish(layer, k_rows)
    with executor.stream():
        for works, _ in in_flight:
            for w in works:
                w.wait()
        if use_peer:  # the prefix forwards are part of this rank's run
            executor._stream.wait_stream(ps.comm)
    err = None
    if use_peer and not _drain_or_release(executor, ps, (ps.epoch + 1) * n_layers, _peer_timeout_s()):
        err = (-1, rank, _ERR_CODES[kv.ProtocolError],
               f"peer handoff timed out after {_peer_timeout_s():g} s (a peer never signalled its K/V rows)")
    hidden, ms = executor.end()
    sent = sent_ctr[0]

    # deferred recv_checked: first error by (layer, rank), agreed over the group
    for hin, kind, layer, lo, hi in inbound:
        res = _check_header(hin.cpu().tolist() if hasattr(hin, "cpu") else hin, kind, layer, lo, hi)
        if res is not None and err is None:
            err = (layer, rank, _ERR_CODES[res[0]], res[1])
            break
    everyone = [None] * world
    dist.all_gather_object(everyone, {"err": err, "metrics": (dots, sent, recvd, waits), "ms": ms,
                                      "last": hidden[-1:].tolist() if rank == world - 1 else None},
                           group=group)
    errs = [e["err"] for e in everyone if e["err"] is not None]
    if errs and use_peer:
        # collective teardown: every rank re-exchanges handles and restarts its flag epochs
        # together on the next run
        executor.close()
    if errs:
        first = min(errs, key=lambda t: (t[0], t[1]))
        raise _ERR_BY_CODE[first[2]](f"rank {first[1]}: {first[3]}")
    m = kv.ExecutionMetrics(n_layers=n_layers, barrier_count=barriers,
                            dot_products=[e["metrics"][0] for e in everyone],
                            kv_pairs_sent=[e["metrics"][1] for e in everyone],
                            kv_pairs_received=[e["metrics"][2] for e in everyone],
                            wait_events=[e["metrics"][3] for e in everyone])
    ttft = max(e["ms"] for e in everyone)
    first_token = np.asarray(everyone[-1]["last"], dtype=hidden.dtype)
    return RankResult(hidden, first_token, m, ms, ttft)


def decode_on_last_rank(executor, rows, position: int, rank: int, world: int, group=None):
    """After run_rank(KVR): the last rank holds the whole prompt's KV cache, so it
    runs the decode step (rows at positions [position, position + n)); the result is broadcast
    to every rank.  (Extension: the reference stops at the first token.)"""
    import torch.distributed as dist
    out = [executor.decode(rows, position) if rank == world - 1 else None]
    dist.broadcast_object_list(out, src=world - 1, group=group)
    return out[0]
