"""ctypes front end to the parity oracle.  TEST INFRASTRUCTURE ONLY.

Two libraries sit behind this module:

* ``_build/libkvoracle.so`` -- the plain-C restatement of the reference algorithm
  (``kvp_oracle.c``; every function cites the reference file:line it follows).
* ``_ref/libkvref.so`` -- the UNMODIFIED reference headers (``/root/reference/proj/
  include/kvprefill``) compiled by ``oracle/Makefile`` behind ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may
import this package.  The product (``paper_2405_05329_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "_build", "libkvoracle.so")
_REF = os.path.join(HERE, "_ref", "libkvref.so")

# status codes == errors.hpp exception types (same numbering as include/kvp_b200.h)
ERRORS = {
    1: "ConfigError", 2: "DimensionError", 3: "CacheError", 4: "InputError",
    5: "PartitionError", 6: "ProtocolError", 7: "AssemblyError", 8: "LookupError",
    9: "SearchError", 10: "BudgetError", 11: "CalibrationError", 12: "IoError",
}
SERIAL, TSP, KVR = 0, 1, 2
FAULT_NONE, FAULT_CORRUPT, FAULT_DROP, FAULT_DUP = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        self.code = code
        self.kind = ERRORS.get(code, f"code{code}")
        super().__init__(f"{self.kind} ({where})")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Config(C.Structure):
    _fields_ = [("d_model", C.c_int64), ("n_heads", C.c_int64), ("n_kv_heads", C.c_int64),
                ("n_layers", C.c_int64), ("seed", C.c_uint64), ("precision", C.c_int32),
                ("rms_norm", C.c_int32)]


class _Cost(C.Structure):
    _fields_ = [("alpha", C.c_double), ("proj_coeff", C.c_double),
                ("softmax_coeff", C.c_double), ("fixed_overhead", C.c_double)]


class _Net(C.Structure):
    _fields_ = [("bandwidth", C.c_double), ("latency", C.c_double)]


class _SearchCfg(C.Structure):
    _fields_ = [("grid_width", C.c_int64), ("initial_stride", C.c_int64), ("min_stride", C.c_int64)]


class _SearchRes(C.Structure):
    _fields_ = [("ttft", C.c_double), ("evaluations", C.c_int64), ("levels", C.c_int64)]


class _SimCtx(C.Structure):
    _fields_ = [("n_layers", C.c_int64), ("cost", _Cost), ("net", _Net), ("strategy", C.c_int)]


EVALUATOR = C.CFUNCTYPE(C.c_double, C.POINTER(C.c_int64), C.c_int64, C.c_void_p)


@dataclass
class Model:
    """ModelConfig (config.hpp:22-47)."""
    d_model: int = 32
    n_heads: int = 4
    n_kv_heads: int = 4
    n_layers: int = 2
    seed: int = 1
    precision: str = "f64"
    rms_norm: bool = False

    @property
    def head_dim(self): return self.d_model // self.n_heads
    @property
    def q_dim(self): return self.n_heads * self.head_dim
    @property
    def kv_dim(self): return self.n_kv_heads * self.head_dim
    @property
    def ffn_dim(self): return 2 * self.d_model

    def c(self) -> _Config:
        return _Config(self.d_model, self.n_heads, self.n_kv_heads, self.n_layers, self.seed,
                       1 if self.precision == "f64" else 0, 1 if self.rms_norm else 0)


@dataclass
class CostModel:
    """CostModel defaults (simnet.hpp:27-31)."""
    alpha: float = 1e-6
    proj_coeff: float = 4e-6
    softmax_coeff: float = 1e-7
    fixed_overhead: float = 1e-5

    def c(self): return _Cost(self.alpha, self.proj_coeff, self.softmax_coeff, self.fixed_overhead)


@dataclass
class NetworkModel:
    """NetworkModel defaults (simnet.hpp:48-50); pairs per second."""
    bandwidth: float = 1e7
    latency: float = 1e-6

    @staticmethod
    def zero_comm():
        return NetworkModel(float("inf"), 0.0)

    def c(self): return _Net(self.bandwidth, self.latency)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


class _Lib:
    _inst = None

    def __init__(self):
        if not os.path.exists(_LIB):
            build()
        self.lib = C.CDLL(_LIB)

    @classmethod
    def get(cls):
        if cls._inst is None:
            cls._inst = _Lib()
        return cls._inst.lib


def _check(code, where=""):
    if code != 0:
        raise OracleError(code, where)


# ------------------------------------------------------------------ restatement (port)
def mix_seed(base: int, a: int, b: int = 0) -> int:
    f = _Lib.get().kvo_mix_seed
    f.restype = C.c_uint64
    f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    return int(f(base, a, b))


def random_context(rows: int, d_model: int, seed: int, dtype=np.float32) -> np.ndarray:
    """random_context<T> (weights.hpp:86-89)."""
    out = np.empty((rows, d_model), dtype=dtype)
    fn = _Lib.get().kvo_random_context_f64 if dtype == np.float64 else _Lib.get().kvo_random_context_f32
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_uint64]
    fn(_ptr(out), rows, d_model, seed)
    return out


def init_weights(m: Model, dtype=np.float32) -> list[tuple[np.ndarray, ...]]:
    """init_weights<T> (weights.hpp:54-83): per layer (wq, wk, wv, wo, w1, w2), [in x out]."""
    d, q, kv = m.d_model, m.q_dim, m.kv_dim
    fn = _Lib.get().kvo_layer_weights_f64 if dtype == np.float64 else _Lib.get().kvo_layer_weights_f32
    fn.argtypes = [C.POINTER(_Config), C.c_int64] + [C.c_void_p] * 6
    cfg = m.c()
    layers = []
    for layer in range(m.n_layers):
        mats = (np.empty((d, q), dtype), np.empty((d, kv), dtype), np.empty((d, kv), dtype),
                np.empty((q, d), dtype), np.empty((d, 2 * d), dtype), np.empty((2 * d, d), dtype))
        _check(fn(C.byref(cfg), layer, *[_ptr(x) for x in mats]), "init_weights")
        layers.append(mats)
    return layers


def _wptrs(weights, dtype):
    flat = [np.ascontiguousarray(x, dtype=dtype) for lw in weights for x in lw]
    arr = (C.c_void_p * len(flat))(*[x.ctypes.data for x in flat])
    return flat, arr


def forward_serial(m: Model, weights, context: np.ndarray, want_kv: bool = False):
    """forward_serial (model.hpp:197-211) -> hidden [C x d] (and per-layer K,V)."""
    dtype = context.dtype.type
    sfx = "f64" if dtype == np.float64 else "f32"
    fn = getattr(_Lib.get(), f"kvo_forward_serial_{sfx}")
    fn.argtypes = [C.POINTER(_Config), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    keep, wp = _wptrs(weights, dtype)
    ctx = np.ascontiguousarray(context)
    Cn = ctx.shape[0]
    out = np.empty((Cn, m.d_model), dtype)
    kv = np.empty((m.n_layers, 2, Cn, m.kv_dim), dtype) if want_kv else None
    cfg = m.c()
    _check(fn(C.byref(cfg), wp, _ptr(ctx), Cn, _ptr(out), _ptr(kv) if want_kv else None), "forward")
    return (out, kv) if want_kv else out


_FAST = os.path.join(HERE, "_build", "libkvoracle_fast.so")


def forward_fast_f32(m: Model, context: np.ndarray, want_hidden: bool = True):
    """forward_serial (model.hpp:197-211) in f32 at benchmark sizes: the multi-threaded
    restatement in kvp_oracle_fast.c (same arithmetic as the reference, bit for bit) ->
    (hidden [C x d] or None, last row [d])."""
    if not os.path.exists(_FAST):
        build()
    lib = C.CDLL(_FAST)
    fn = lib.kvof_forward_f32
    fn.argtypes = [C.POINTER(_Config), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    ctx = np.ascontiguousarray(context, dtype=np.float32)
    Cn = ctx.shape[0]
    hid = np.empty((Cn, m.d_model), np.float32) if want_hidden else None
    last = np.empty(m.d_model, np.float32)
    cfg = m.c()
    _check(fn(C.byref(cfg), _ptr(ctx), Cn, _ptr(hid) if want_hidden else None, _ptr(last)), "forward_fast")
    return hid, last


def naive_forward(m: Model, weights, context: np.ndarray) -> np.ndarray:
    """naive_causal_forward (oracle.hpp:34-111), f64."""
    fn = _Lib.get().kvo_naive_forward_f64
    fn.argtypes = [C.POINTER(_Config), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    keep, wp = _wptrs(weights, np.float64)
    ctx = np.ascontiguousarray(context, dtype=np.float64)
    out = np.empty((ctx.shape[0], m.d_model), np.float64)
    cfg = m.c()
    _check(fn(C.byref(cfg), wp, _ptr(ctx), ctx.shape[0], _ptr(out)), "naive")
    return out


def causal_attention(m: Model, Q, K, V, offset: int) -> np.ndarray:
    """causal_attention (model.hpp:112-158)."""
    dtype = Q.dtype.type
    sfx = "f64" if dtype == np.float64 else "f32"
    fn = getattr(_Lib.get(), f"kvo_causal_attention_{sfx}")
    fn.argtypes = [C.POINTER(_Config), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                   C.c_int64, C.c_void_p]
    Q, K, V = (np.ascontiguousarray(x, dtype=dtype) for x in (Q, K, V))
    A = np.empty((Q.shape[0], m.q_dim), dtype)
    cfg = m.c()
    _check(fn(C.byref(cfg), _ptr(Q), Q.shape[0], _ptr(K), _ptr(V), K.shape[0], offset, _ptr(A)),
           "causal_attention")
    return A


def layer_qkv(m: Model, weights, layer: int, hidden: np.ndarray):
    dtype = hidden.dtype.type
    sfx = "f64" if dtype == np.float64 else "f32"
    fn = getattr(_Lib.get(), f"kvo_layer_qkv_{sfx}")
    fn.argtypes = [C.POINTER(_Config), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64] + [C.c_void_p] * 3
    keep, wp = _wptrs(weights, dtype)
    h = np.ascontiguousarray(hidden)
    r = h.shape[0]
    Q = np.empty((r, m.q_dim), dtype)
    K = np.empty((r, m.kv_dim), dtype)
    V = np.empty((r, m.kv_dim), dtype)
    cfg = m.c()
    _check(fn(C.byref(cfg), wp, layer, _ptr(h), r, _ptr(Q), _ptr(K), _ptr(V)), "layer_qkv")
    return Q, K, V


def even_partition(C_: int, p: int) -> list[int]:
    """even_partition (partition.hpp:59-69) -> boundaries."""
    out = np.empty(p + 1 if p >= 1 else 1, np.int64)
    fn = _Lib.get().kvo_even_partition
    fn.argtypes = [C.c_int64, C.c_int64, C.c_void_p]
    _check(fn(C_, p, _ptr(out)), "even_partition")
    return out.tolist()


def partition_from_ratios(C_: int, ratios) -> list[int]:
    """partition_from_ratios (partition.hpp:76-120) -> boundaries."""
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    out = np.empty(len(r) + 1, np.int64)
    fn = _Lib.get().kvo_partition_from_ratios
    fn.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
    _check(fn(C_, _ptr(r), len(r), _ptr(out)), "partition_from_ratios")
    return out.tolist()


def dot_product_counts(strategy: int, boundaries) -> list[int]:
    b, bp = _i64(boundaries)
    p = len(b) - 1
    out = np.empty(p, np.int64)
    fn = _Lib.get().kvo_dot_product_counts
    fn.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
    _check(fn(strategy, int(b[-1]), _ptr(b), p, _ptr(out)), "dot_product_counts")
    return out.tolist()


def traffic_pairs(strategy: int, boundaries) -> int:
    b, _ = _i64(boundaries)
    out = C.c_int64()
    fn = _Lib.get().kvo_traffic_pairs
    fn.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    _check(fn(strategy, int(b[-1]), _ptr(b), len(b) - 1, C.byref(out)), "traffic_pairs")
    return out.value


def simulate_ttft(strategy: int, boundaries, n_layers: int, cost=None, net=None) -> float:
    cost = cost or CostModel()
    net = net or NetworkModel()
    b, _ = _i64(boundaries)
    out = C.c_double()
    fn = _Lib.get().kvo_simulate_ttft
    fn.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(_Cost),
                   C.POINTER(_Net), C.POINTER(C.c_double)]
    cc, nc = cost.c(), net.c()
    _check(fn(strategy, int(b[-1]), _ptr(b), len(b) - 1, n_layers, C.byref(cc), C.byref(nc),
              C.byref(out)), "simulate_ttft")
    return out.value


def ttft_star(C_: int, p: int, alpha: float) -> float:
    out = C.c_double()
    fn = _Lib.get().kvo_ttft_star
    fn.argtypes = [C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_double)]
    _check(fn(C_, p, alpha, C.byref(out)), "ttft_star")
    return out.value


def table_build_cost(T: float, N: int, C_: int, grid_width: int = 5) -> float:
    fn = _Lib.get().kvo_table_build_cost
    fn.restype = C.c_double
    fn.argtypes = [C.c_double, C.c_int64, C.c_int64, C.c_int64]
    v = fn(T, N, C_, grid_width)
    if v < 0:
        raise OracleError(4, "table_build_cost")
    return v


def calibrate_alpha(points) -> float:
    Cs = np.ascontiguousarray([p[0] for p in points], dtype=np.int64)
    ts = np.ascontiguousarray([p[1] for p in points], dtype=np.float64)
    out = C.c_double()
    fn = _Lib.get().kvo_calibrate_alpha
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
    _check(fn(_ptr(Cs), _ptr(ts), len(Cs), C.byref(out)), "calibrate_alpha")
    return out.value


def _search(kind: str, C_: int, p: int, evaluator, grid_width=5, initial_stride=0, min_stride=1,
            budget=1_000_000, sim: _SimCtx | None = None):
    lib = _Lib.get()
    cfg = _SearchCfg(grid_width, initial_stride, min_stride)
    res = _SearchRes()
    out = np.empty(p + 1, np.int64)
    if sim is not None:
        cb = C.cast(lib.kvo_sim_evaluator, EVALUATOR)
        ctx = C.cast(C.pointer(sim), C.c_void_p)
    elif evaluator is None:
        cb, ctx = EVALUATOR(), None
    else:
        cb = EVALUATOR(lambda bp, n, _c: float(evaluator([bp[i] for i in range(n + 1)])))
        ctx = None
    if kind == "grid":
        fn = lib.kvo_hierarchical_grid_search
        fn.argtypes = [C.c_int64, C.c_int64, C.POINTER(_SearchCfg), EVALUATOR, C.c_void_p,
                       C.c_void_p, C.POINTER(_SearchRes)]
        st = fn(C_, p, C.byref(cfg), cb, ctx, _ptr(out), C.byref(res))
    elif kind == "two":
        fn = lib.kvo_binary_search_two
        fn.argtypes = [C.c_int64, C.POINTER(_SearchCfg), EVALUATOR, C.c_void_p, C.c_void_p,
                       C.POINTER(_SearchRes)]
        st = fn(C_, C.byref(cfg), cb, ctx, _ptr(out), C.byref(res))
    else:
        fn = lib.kvo_exhaustive_partition_search
        fn.argtypes = [C.c_int64, C.c_int64, EVALUATOR, C.c_void_p, C.c_int64, C.c_void_p,
                       C.POINTER(_SearchRes)]
        st = fn(C_, p, cb, ctx, budget, _ptr(out), C.byref(res))
    _check(st, kind)
    return out.tolist(), res.ttft, res.evaluations, res.levels


def hierarchical_grid_search(C_, p, evaluator=None, **kw):
    return _search("grid", C_, p, evaluator, **kw)


def binary_search_two(C_, evaluator=None, **kw):
    return _search("two", C_, 2, evaluator, **kw)


def exhaustive_partition_search(C_, p, evaluator=None, **kw):
    return _search("exh", C_, p, evaluator, **kw)


def sim_ctx(n_layers: int, cost=None, net=None, strategy=KVR) -> _SimCtx:
    cost = cost or CostModel()
    net = net or NetworkModel()
    return _SimCtx(n_layers, cost.c(), net.c(), strategy)


def practical_bound(C_: int, p: int, n_layers: int, cost=None):
    cost = cost or CostModel()
    out = np.empty(p + 1, np.int64)
    t = C.c_double()
    fn = _Lib.get().kvo_practical_bound
    fn.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Cost), C.c_void_p, C.POINTER(C.c_double)]
    cc = cost.c()
    _check(fn(C_, p, n_layers, C.byref(cc), _ptr(out), C.byref(t)), "practical_bound")
    return out.tolist(), t.value


def max_rel_dev(a, b) -> float:
    """max_rel_dev (matrix.hpp:101-115): max |a-b| / max(1, |b|)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise OracleError(2, "max_rel_dev")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def fnv1a64(arr: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    for byte in np.ascontiguousarray(arr).tobytes():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


# ------------------------------------------------------------------ the reference itself
class Reference:
    """The unmodified reference compiled by oracle/Makefile (oracle/_ref/libkvref.so)."""

    def __init__(self):
        if not os.path.exists(_REF):
            build()
        if not os.path.exists(_REF):
            raise FileNotFoundError(_REF)
        self.lib = C.CDLL(_REF)
        self.lib.kvref_weights_create.restype = C.c_void_p
        self.lib.kvref_weights_create.argtypes = [C.POINTER(_Config)]
        self.lib.kvref_weights_destroy.argtypes = [C.c_void_p]

    @staticmethod
    def available() -> bool:
        return os.path.exists(_REF)

    def weights(self, m: Model):
        cfg = m.c()
        h = self.lib.kvref_weights_create(C.byref(cfg))
        if not h:
            raise OracleError(1, "kvref_weights_create")
        return _RefWeights(self, h, m)

    def random_context(self, rows, d, seed, dtype=np.float32):
        out = np.empty((rows, d), dtype)
        fn = self.lib.kvref_random_context
        fn.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]
        _check(fn(1 if dtype == np.float64 else 0, rows, d, seed, _ptr(out)), "ref random_context")
        return out

    def even_partition(self, C_, p):
        out = np.empty(max(p + 1, 1), np.int64)
        fn = self.lib.kvref_even_partition
        fn.argtypes = [C.c_int64, C.c_int64, C.c_void_p]
        _check(fn(C_, p, _ptr(out)), "ref even_partition")
        return out.tolist()

    def partition_from_ratios(self, C_, ratios):
        r = np.ascontiguousarray(ratios, np.float64)
        out = np.empty(len(r) + 1, np.int64)
        fn = self.lib.kvref_partition_from_ratios
        fn.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
        _check(fn(C_, _ptr(r), len(r), _ptr(out)), "ref partition_from_ratios")
        return out.tolist()

    def simulate_ttft(self, strategy, boundaries, n_layers, cost=None, net=None):
        cost = cost or CostModel()
        net = net or NetworkModel()
        b, _ = _i64(boundaries)
        out = C.c_double()
        fn = self.lib.kvref_simulate_ttft
        fn.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(_Cost),
                       C.POINTER(_Net), C.POINTER(C.c_double)]
        cc, nc = cost.c(), net.c()
        _check(fn(strategy, int(b[-1]), _ptr(b), len(b) - 1, n_layers, C.byref(cc), C.byref(nc),
                  C.byref(out)), "ref simulate")
        return out.value

    def search_sim(self, which, C_, p, n_layers, cost=None, net=None, grid_width=5,
                   initial_stride=0, min_stride=1):
        cost = cost or CostModel()
        net = net or NetworkModel()
        out = np.empty(p + 1, np.int64)
        t, ev, lv = C.c_double(), C.c_int64(), C.c_int64()
        fn = self.lib.kvref_search_sim
        fn.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                       C.POINTER(_Cost), C.POINTER(_Net), C.c_void_p, C.POINTER(C.c_double),
                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        cc, nc = cost.c(), net.c()
        _check(fn({"grid": 0, "two": 1, "exh": 2}[which], C_, p, grid_width, initial_stride,
                  min_stride, n_layers, C.byref(cc), C.byref(nc), _ptr(out), C.byref(t),
                  C.byref(ev), C.byref(lv)), "ref search")
        return out.tolist(), t.value, ev.value, lv.value

    def practical_bound(self, C_, p, n_layers, cost=None):
        cost = cost or CostModel()
        out = np.empty(p + 1, np.int64)
        t = C.c_double()
        fn = self.lib.kvref_practical_bound
        fn.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Cost), C.c_void_p,
                       C.POINTER(C.c_double)]
        cc = cost.c()
        _check(fn(C_, p, n_layers, C.byref(cc), _ptr(out), C.byref(t)), "ref practical_bound")
        return out.tolist(), t.value

    def noise_study(self, strategy, boundaries, n_layers, factor, trials, seed, cost=None, net=None):
        cost = cost or CostModel()
        net = net or NetworkModel()
        b, _ = _i64(boundaries)
        q, mean, mx = C.c_double(), C.c_double(), C.c_double()
        per = np.zeros(max(trials, 1), np.float64)
        fn = self.lib.kvref_noise_study
        fn.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(_Cost), C.POINTER(_Net),
                       C.c_double, C.c_int64, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                       C.POINTER(C.c_double), C.c_void_p]
        cc, nc = cost.c(), net.c()
        _check(fn(strategy, int(b[-1]), _ptr(b), len(b) - 1, n_layers, C.byref(cc), C.byref(nc), factor, trials,
                  seed, C.byref(q), C.byref(mean), C.byref(mx), _ptr(per)), "ref noise_study")
        return q.value, mean.value, mx.value, per[:trials].tolist()

    def cli(self, sub: str, config_path: str = "", C_: int = -1, out: str = "", table: str = "") -> int:
        """The reference CLI's subcommand through its own commands.hpp (exit code)."""
        fn = self.lib.kvref_cli
        fn.restype = C.c_int
        fn.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_char_p, C.c_char_p]
        return fn(sub.encode(), config_path.encode(), C_, out.encode(), table.encode())

    def table(self, entries: dict, p: int, C_: int):
        keys = list(entries)
        Cs = np.ascontiguousarray(keys, np.int64)
        R = np.ascontiguousarray([entries[k] for k in keys], np.float64)
        rout = np.zeros(p, np.float64)
        bout = np.zeros(p + 1, np.int64)
        fn = self.lib.kvref_table
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        _check(fn(_ptr(Cs), _ptr(R), len(keys), p, C_, _ptr(rout), _ptr(bout)), "ref table")
        return rout.tolist(), bout.tolist()

    def causal_attention(self, m: Model, Q, K, V, offset):
        dtype = np.float64 if m.precision == "f64" else np.float32
        Q, K, V = (np.ascontiguousarray(x, dtype) for x in (Q, K, V))
        A = np.empty((Q.shape[0], m.q_dim), dtype)
        fn = self.lib.kvref_causal_attention
        fn.argtypes = [C.POINTER(_Config), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                       C.c_int64, C.c_int64, C.c_void_p]
        cfg = m.c()
        _check(fn(C.byref(cfg), _ptr(Q), Q.shape[0], _ptr(K), _ptr(V), K.shape[0], offset, _ptr(A)),
               "ref causal_attention")
        return A


class _RefWeights:
    def __init__(self, ref: Reference, handle, m: Model):
        self.ref, self.h, self.m = ref, handle, m
        self.dtype = np.float64 if m.precision == "f64" else np.float32

    def __del__(self):
        try:
            self.ref.lib.kvref_weights_destroy(self.h)
        except Exception:
            pass

    def layers(self):
        m, dt = self.m, self.dtype
        d, q, kv = m.d_model, m.q_dim, m.kv_dim
        fn = self.ref.lib.kvref_weights_layer
        fn.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 6
        out = []
        for layer in range(m.n_layers):
            mats = (np.empty((d, q), dt), np.empty((d, kv), dt), np.empty((d, kv), dt),
                    np.empty((q, d), dt), np.empty((d, 2 * d), dt), np.empty((2 * d, d), dt))
            _check(fn(self.h, layer, *[_ptr(x) for x in mats]), "ref layer")
            out.append(mats)
        return out

    def run(self, strategy, context, boundaries, fault=(FAULT_NONE, 0, 0)):
        """run<T> (engine.hpp:186-318) -> (hidden_out, first_token_hidden, metrics dict)."""
        ctx = np.ascontiguousarray(context, self.dtype)
        b, _ = _i64(boundaries)
        p = len(b) - 1
        Cn = ctx.shape[0]
        hid = np.empty((Cn, self.m.d_model), self.dtype)
        ft = np.empty((1, self.m.d_model), self.dtype)
        met = np.zeros(1 + 4 * p, np.int64)
        fn = self.ref.lib.kvref_run
        fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                       C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        _check(fn(self.h, strategy, _ptr(ctx), Cn, _ptr(b), p, fault[0], fault[1], fault[2],
                  _ptr(hid), _ptr(ft), _ptr(met)), "ref run")
        metrics = {"barrier_count": int(met[0]), "dot_products": met[1:1 + p].tolist(),
                   "kv_pairs_sent": met[1 + p:1 + 2 * p].tolist(),
                   "kv_pairs_received": met[1 + 2 * p:1 + 3 * p].tolist(),
                   "wait_events": met[1 + 3 * p:1 + 4 * p].tolist()}
        return hid, ft, metrics
