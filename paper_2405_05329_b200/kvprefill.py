"""Python mirror of the reference ``kvprefill`` API over the B200 C-ABI (``libkvp_b200.so``).

Same names, argument meaning and error behaviour as the C++ reference headers
(``/root/reference/proj/include/kvprefill``): ``ModelConfig`` (config.hpp:22-47),
``ContextPartition`` / ``even_partition`` / ``partition_from_ratios`` (partition.hpp),
``SearchConfig`` / ``hierarchical_grid_search`` / ``binary_search_two`` (search.hpp),
``run`` / ``ExecutionResult`` / ``ExecutionMetrics`` / ``FaultInjection`` (engine.hpp),
``layer_qkv`` / ``causal_attention`` / ``layer_finish`` / ``forward_serial`` (model.hpp),
``simulate_ttft`` / ``ttft_star`` / ``practical_bound`` / ``calibrate_alpha`` (simnet.hpp).
Each reference exception type is a Python exception class here (errors.hpp:8-46).

There is no CPU fallback: every compute call goes to the sm_100a kernels in the shared
library; loading fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KVP_LIB_PATH: A/B tuning only (an alternative build of the same library)
LIB_PATH = os.environ.get("KVP_LIB_PATH") or os.path.join(_HERE, "_lib", "libkvp_b200.so")
MAX_RANKS = 64


# ------------------------------------------------------------------ errors (errors.hpp)
class Error(RuntimeError):
    code = -1


class ConfigError(Error): code = 1
class DimensionError(Error): code = 2
class CacheError(Error): code = 3
class InputError(Error): code = 4
class PartitionError(Error): code = 5
class ProtocolError(Error): code = 6
class AssemblyError(Error): code = 7
class LookupError_(Error): code = 8
class SearchError(Error): code = 9
class BudgetError(Error): code = 10
class CalibrationError(Error): code = 11
class IoError(Error): code = 12
class CudaError(Error): code = 100
class NcclError(Error): code = 101


_BY_CODE = {c.code: c for c in (ConfigError, DimensionError, CacheError, InputError, PartitionError,
                                ProtocolError, AssemblyError, LookupError_, SearchError, BudgetError,
                                CalibrationError, IoError, CudaError, NcclError)}


# ------------------------------------------------------------------ C structs
class _ModelCfg(C.Structure):
    _fields_ = [("d_model", C.c_int64), ("n_heads", C.c_int64), ("n_kv_heads", C.c_int64),
                ("n_layers", C.c_int64), ("seed", C.c_uint64), ("precision", C.c_int32),
                ("rms_norm", C.c_int32)]


class _Fault(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rank", C.c_int64), ("layer", C.c_int64)]


class _Metrics(C.Structure):
    _fields_ = [("n_layers", C.c_int64), ("barrier_count", C.c_int64), ("p", C.c_int64),
                ("dot_products", C.c_int64 * MAX_RANKS), ("kv_pairs_sent", C.c_int64 * MAX_RANKS),
                ("kv_pairs_received", C.c_int64 * MAX_RANKS), ("wait_events", C.c_int64 * MAX_RANKS)]


class _KStats(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


class _Cost(C.Structure):
    _fields_ = [("alpha", C.c_double), ("proj_coeff", C.c_double), ("softmax_coeff", C.c_double),
                ("fixed_overhead", C.c_double)]


class _Net(C.Structure):
    _fields_ = [("bandwidth", C.c_double), ("latency", C.c_double)]


class _SearchCfg(C.Structure):
    _fields_ = [("grid_width", C.c_int64), ("initial_stride", C.c_int64), ("min_stride", C.c_int64)]


class _SearchRes(C.Structure):
    _fields_ = [("ttft", C.c_double), ("evaluations", C.c_int64), ("levels", C.c_int64)]


_EVAL = C.CFUNCTYPE(C.c_double, C.POINTER(C.c_int64), C.c_int64, C.c_void_p)

_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_SIGS = {
    "kvp_abi_version": (C.c_int32, []),
    "kvp_last_error": (C.c_char_p, []),
    "kvp_device_count": (C.c_int32, []),
    "kvp_engine_create": (C.c_int, [C.POINTER(_ModelCfg), C.POINTER(C.c_int32), C.c_int32, C.POINTER(_P)]),
    "kvp_engine_load_layer": (C.c_int, [_P, C.c_int64] + [_P] * 6),
    "kvp_engine_destroy": (C.c_int, [_P]),
    "kvp_engine_run": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _I64P, C.c_int64, C.POINTER(_Fault), _P, _P,
                                 C.POINTER(_Metrics)]),
    "kvp_engine_run_device": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _I64P, C.c_int64, C.POINTER(_Fault), _P,
                                        _P, C.POINTER(_Metrics)]),
    "kvp_engine_layer_times": (C.c_int, [_P, C.c_int64, _P, _P, _P]),
    "kvp_engine_last_ttft_ms": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "kvp_engine_last_launch_count": (C.c_int, [_P, _I64P]),
    "kvp_engine_set_profiling": (C.c_int, [_P, C.c_int32]),
    "kvp_engine_kernel_stats": (C.c_int, [_P, C.POINTER(_KStats), C.c_int32, C.POINTER(C.c_int32)]),
    "kvp_engine_profile_layer": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_float),
                                           C.POINTER(C.c_float)]),
    "kvp_bench_attn": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 C.POINTER(C.c_float)]),
    "kvp_bench_gemm": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_float),
                                 C.POINTER(C.c_int32)]),
    "kvp_rank_begin": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]),
    "kvp_rank_stream": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "kvp_rank_kv": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "kvp_rank_qkv": (C.c_int, [_P, C.c_int64]),
    "kvp_rank_finish": (C.c_int, [_P, C.c_int64, C.c_int64]),
    "kvp_rank_end": (C.c_int, [_P, _P, C.c_int32, _P, C.POINTER(C.c_float)]),
    "kvp_rank_set_decode": (C.c_int, [_P, C.c_int32]),
    "kvp_rank_set_mirrors": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_void_p)]),
    "kvp_ipc_export": (C.c_int, [_P, _P, C.POINTER(C.c_int64)]),
    "kvp_ipc_open": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_void_p)]),
    "kvp_ipc_close": (C.c_int, [_P, C.c_int64]),
    "kvp_stream_signal": (C.c_int, [_P, _P, C.c_uint32]),
    "kvp_stream_wait": (C.c_int, [_P, _P, C.c_uint32]),
    "kvp_stream_copy": (C.c_int, [_P, _P, _P, C.c_int64]),
    "kvp_kv_cache_create": (C.c_int, [_P, C.c_int64, C.POINTER(_P)]),
    "kvp_kv_cache_destroy": (C.c_int, [_P]),
    "kvp_kv_cache_length": (C.c_int, [_P, _I64P]),
    "kvp_kv_cache_reset": (C.c_int, [_P, C.c_int64]),
    "kvp_prefill_cached": (C.c_int, [_P, _P, _P, C.c_int64, _P, _P, C.POINTER(C.c_float)]),
    "kvp_decode": (C.c_int, [_P, _P, _P, C.c_int64, _P, C.POINTER(C.c_float)]),
    "kvp_forward_serial": (C.c_int, [_P, _P, C.c_int64, _P, _P]),
    "kvp_engine_set_rope": (C.c_int, [_P, C.c_double]),
    "kvp_random_context": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, _P]),
    "kvp_random_context_device": (C.c_int, [_P, C.c_int64, C.c_uint64, _P]),
    "kvp_layer_qkv": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _P, _P, _P]),
    "kvp_causal_attention": (C.c_int, [_P, _P, C.c_int64, _P, _P, C.c_int64, C.c_int64, _P]),
    "kvp_layer_finish": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _P, _P, _P, C.c_int64, C.c_int64, _P]),
    "kvp_validate_partition": (C.c_int, [C.c_int64, _I64P, C.c_int64]),
    "kvp_even_partition": (C.c_int, [C.c_int64, C.c_int64, _I64P]),
    "kvp_partition_from_ratios": (C.c_int, [C.c_int64, _P, C.c_int64, _I64P]),
    "kvp_dot_product_counts": (C.c_int, [C.c_int32, C.c_int64, _I64P, C.c_int64, _I64P]),
    "kvp_traffic_pairs": (C.c_int, [C.c_int32, C.c_int64, _I64P, C.c_int64, _I64P]),
    "kvp_simulate_ttft": (C.c_int, [C.c_int32, C.c_int64, _I64P, C.c_int64, C.c_int64, C.POINTER(_Cost),
                                    C.POINTER(_Net), C.POINTER(C.c_double)]),
    "kvp_ttft_star": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_double)]),
    "kvp_calibrate_alpha": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_double)]),
    "kvp_hierarchical_grid_search": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(_SearchCfg), _EVAL, _P, _I64P,
                                               C.POINTER(_SearchRes)]),
    "kvp_binary_search_two": (C.c_int, [C.c_int64, C.POINTER(_SearchCfg), _EVAL, _P, _I64P,
                                        C.POINTER(_SearchRes)]),
    "kvp_search_partition": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Cost), C.POINTER(_Net),
                                       C.POINTER(_SearchCfg), _I64P, C.POINTER(_SearchRes)]),
    "kvp_practical_bound": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Cost), _I64P,
                                      C.POINTER(C.c_double)]),
    "kvp_simulate_ttft_causal": (C.c_int, [C.c_int32, C.c_int64, _I64P, C.c_int64, C.c_int64, C.POINTER(_Cost),
                                           C.POINTER(_Net), C.POINTER(C.c_double)]),
    "kvp_search_partition_causal": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Cost), C.POINTER(_Net),
                                              C.POINTER(_SearchCfg), _I64P, C.POINTER(_SearchRes)]),
    "kvp_simulate_ttft_noisy": (C.c_int, [C.c_int32, C.c_int64, _I64P, C.c_int64, C.c_int64, C.POINTER(_Cost),
                                          C.POINTER(_Net), C.c_uint64, C.c_double, C.POINTER(C.c_double)]),
    "kvp_noise_degraded_link": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_int64)]),
    "kvp_noise_trial_seed": (C.c_int, [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]),
    "kvp_noise_study": (C.c_int, [C.c_int32, C.c_int64, _I64P, C.c_int64, C.c_int64, C.POINTER(_Cost),
                                  C.POINTER(_Net), C.c_double, C.c_int64, C.c_uint64, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "kvp_interpolate_partition": (C.c_int, [_I64P, _P, C.c_int64, C.c_int64, C.c_int64, _P]),
    "kvp_partition_from_table": (C.c_int, [_I64P, _P, C.c_int64, C.c_int64, C.c_int64, _I64P]),
    "kvp_fit_cost_model": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.POINTER(_Cost)]),
}
EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Loads libkvp_b200.so (no fallback: a missing library is an ImportError)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(code: int, where: str = "") -> None:
    if code != 0:
        msg = lib().kvp_last_error().decode(errors="replace")
        raise _BY_CODE.get(code, Error)(f"{where}: {msg}" if where else msg)


def device_count() -> int:
    return int(lib().kvp_device_count())


def _i64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def _vp(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


# ------------------------------------------------------------------ config.hpp
class Precision(enum.IntEnum):
    f32 = 0
    f64 = 1
    bf16 = 2  # additive: bf16 operands, f32 accumulation (tcgen05)


@dataclass
class ModelConfig:
    d_model: int = 32
    n_heads: int = 4
    n_kv_heads: int = 4
    n_layers: int = 2
    seed: int = 1
    precision: Precision | str = Precision.f64
    rms_norm: bool = False

    def __post_init__(self):
        if isinstance(self.precision, str):
            self.precision = Precision[self.precision]

    def head_dim(self): return self.d_model // self.n_heads
    def q_dim(self): return self.n_heads * self.head_dim()
    def kv_dim(self): return self.n_kv_heads * self.head_dim()
    def ffn_dim(self): return 2 * self.d_model

    def validate(self) -> None:
        if self.d_model <= 0 or self.n_heads <= 0 or self.n_kv_heads <= 0 or self.n_layers <= 0:
            raise ConfigError("model dimensions must be positive")
        if self.d_model % self.n_heads:
            raise ConfigError(f"d_model ({self.d_model}) must be divisible by n_heads ({self.n_heads})")
        if self.n_heads % self.n_kv_heads:
            raise ConfigError(f"n_heads ({self.n_heads}) must be divisible by n_kv_heads ({self.n_kv_heads})")

    def _c(self) -> _ModelCfg:
        return _ModelCfg(self.d_model, self.n_heads, self.n_kv_heads, self.n_layers, self.seed,
                         int(self.precision), 1 if self.rms_norm else 0)


# ------------------------------------------------------------------ partition.hpp
@dataclass
class ContextPartition:
    context_length: int = 0
    boundaries: list = field(default_factory=list)

    def process_count(self) -> int:
        return len(self.boundaries) - 1

    def sizes(self) -> list:
        b = self.boundaries
        return [b[i + 1] - b[i] for i in range(len(b) - 1)]

    def validate(self) -> None:
        b = _i64(self.boundaries)
        if len(b) < 2:
            raise PartitionError("boundaries must run from 0 to the context length")
        _check(lib().kvp_validate_partition(self.context_length, _ip(b), len(b) - 1), "validate")

    @staticmethod
    def from_sizes(sizes: Sequence[int]) -> "ContextPartition":
        b = [0]
        for c in sizes:
            b.append(b[-1] + int(c))
        part = ContextPartition(b[-1], b)
        part.validate()
        return part


def even_partition(C_: int, p: int) -> ContextPartition:
    out = np.zeros(max(p, 1) + 1, np.int64)
    _check(lib().kvp_even_partition(C_, p, _ip(out)), "even_partition")
    return ContextPartition(C_, out.tolist())


def partition_from_ratios(C_: int, ratios: Sequence[float]) -> ContextPartition:
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    out = np.zeros(len(r) + 1, np.int64)
    _check(lib().kvp_partition_from_ratios(C_, _vp(r), len(r), _ip(out)), "partition_from_ratios")
    return ContextPartition(C_, out.tolist())


# ------------------------------------------------------------------ engine.hpp
class Strategy(enum.IntEnum):
    Serial = 0
    TSP = 1
    KVR = 2


@dataclass
class FaultInjection:
    class Kind(enum.IntEnum):
        None_ = 0
        CorruptLayerTag = 1
        DropMessage = 2
        DuplicateMessage = 3

    kind: "FaultInjection.Kind" = Kind.None_
    rank: int = 0
    layer: int = 0


@dataclass
class ExecutionMetrics:
    n_layers: int = 1
    barrier_count: int = 0
    dot_products: list = field(default_factory=list)
    kv_pairs_sent: list = field(default_factory=list)
    kv_pairs_received: list = field(default_factory=list)
    wait_events: list = field(default_factory=list)

    def per_layer_dot_products(self, rank): return self.dot_products[rank] // self.n_layers
    def per_layer_pairs_received(self, rank): return self.kv_pairs_received[rank] // self.n_layers
    def total_pairs_sent(self): return sum(self.kv_pairs_sent)
    def per_layer_pairs_sent(self): return self.total_pairs_sent() // self.n_layers
    def total_rows_sent(self): return 2 * self.total_pairs_sent()
    def per_layer_rows_sent(self): return 2 * self.per_layer_pairs_sent()

    @staticmethod
    def _from_c(m: _Metrics) -> "ExecutionMetrics":
        p = m.p
        return ExecutionMetrics(m.n_layers, m.barrier_count, list(m.dot_products[:p]), list(m.kv_pairs_sent[:p]),
                                list(m.kv_pairs_received[:p]), list(m.wait_events[:p]))


@dataclass
class ExecutionResult:
    hidden_out: np.ndarray
    first_token_hidden: np.ndarray
    metrics: ExecutionMetrics

    @property
    def first_token(self) -> int:
        """argmax over first_token_hidden: the reference exposes hidden state, not logits
        (SPEC.md:111), so the 'first token' is the argmax of the d_model-wide readout."""
        return int(np.argmax(self.first_token_hidden))


def dot_product_counts(strategy: Strategy, partition: ContextPartition) -> list:
    b = _i64(partition.boundaries)
    out = np.zeros(len(b) - 1, np.int64)
    _check(lib().kvp_dot_product_counts(int(strategy), partition.context_length, _ip(b), len(b) - 1, _ip(out)),
           "dot_product_counts")
    return out.tolist()


def traffic_pairs(strategy: Strategy, partition: ContextPartition) -> int:
    b = _i64(partition.boundaries)
    out = C.c_int64()
    _check(lib().kvp_traffic_pairs(int(strategy), partition.context_length, _ip(b), len(b) - 1, C.byref(out)),
           "traffic_pairs")
    return out.value


class WeightSet:
    """init_weights<T> (weights.hpp:54-83) materialised ON the GPU(s): the handle owns the
    device weights and the prefill engine (one host thread + streams per rank)."""

    def __init__(self, config: ModelConfig, devices: Sequence[int] = (0,)):
        config.validate()
        self.config = config
        dev = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        cfg = config._c()
        _check(lib().kvp_engine_create(C.byref(cfg), dev, len(devices), C.byref(h)), "init_weights")
        self._h = h

    @property
    def handle(self):
        return self._h

    def load_layer(self, layer: int, wq, wk, wv, wo, w1, w2) -> None:
        mats = [_f32(x) for x in (wq, wk, wv, wo, w1, w2)]
        _check(lib().kvp_engine_load_layer(self._h, layer, *[_vp(m) for m in mats]), "load_layer")

    def set_rope(self, theta: float) -> None:
        """Opt-in rotary position embedding (an extension: the reference model has none).
        theta > 0 rotates pairs (2i, 2i+1) of every Q and K head at absolute position t by
        t * theta^(-2i/head_dim) inside the QKV projection (bf16 engines, head_dim % 32 == 0);
        theta <= 0 turns it off."""
        _check(lib().kvp_engine_set_rope(self._h, float(theta)), "set_rope")

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().kvp_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layer_times(self, rank: int):
        """(proj_ms, rest_ms, wait_ms) per layer of the last run on `rank` (CUDA events)."""
        L = self.config.n_layers
        a, b, c = (np.zeros(L, np.float32) for _ in range(3))
        _check(lib().kvp_engine_layer_times(self._h, rank, _vp(a), _vp(b), _vp(c)), "layer_times")
        return a, b, c

    def last_ttft_ms(self) -> float:
        v = C.c_float()
        _check(lib().kvp_engine_last_ttft_ms(self._h, C.byref(v)), "last_ttft_ms")
        return float(v.value)

    def set_profiling(self, on: bool) -> None:
        _check(lib().kvp_engine_set_profiling(self._h, 1 if on else 0), "set_profiling")

    def kernel_stats(self) -> dict:
        """{class: {launches, total_ms, flops, bytes}} of the last (profiled) run."""
        arr = (_KStats * 16)()
        n = C.c_int32()
        _check(lib().kvp_engine_kernel_stats(self._h, arr, 16, C.byref(n)), "kernel_stats")
        return {arr[i].name.decode(): {"launches": arr[i].launches, "total_ms": arr[i].total_ms,
                                       "flops": arr[i].flops, "bytes": arr[i].bytes} for i in range(n.value)}

    def profile_layer(self, rows: int, offset: int, reps: int = 5):
        """(proj_ms, rest_ms): one rank's layer executor timed in isolation (CUDA events)."""
        a, b = C.c_float(), C.c_float()
        _check(lib().kvp_engine_profile_layer(self._h, rows, offset, reps, C.byref(a), C.byref(b)), "profile_layer")
        return float(a.value), float(b.value)

    def bench_gemm(self, M: int, N: int, K: int, epi: int = 3, reps: int = 10):
        """(median ms, TFLOP/s, tile width) of one tcgen05 GEMM shape in isolation."""
        ms, bn = C.c_float(), C.c_int32()
        _check(lib().kvp_bench_gemm(self._h, M, N, K, epi, reps, C.byref(ms), C.byref(bn)), "bench_gemm")
        return float(ms.value), 2.0 * M * N * K / (ms.value * 1e-3) / 1e12, int(bn.value)

    def bench_attn(self, q_rows: int, offset: int, n_heads: int, n_kv_heads: int, head_dim: int, reps: int = 10):
        """Median device ms of the bf16 attention kernel alone and its causal-visible TFLOP/s."""
        ms = C.c_float()
        _check(lib().kvp_bench_attn(self._h, q_rows, offset, n_heads, n_kv_heads, head_dim, reps, C.byref(ms)),
               "bench_attn")
        pairs = q_rows * offset + q_rows * (q_rows + 1) / 2
        return ms.value, 4.0 * head_dim * n_heads * pairs / (ms.value * 1e-3) / 1e12

    def last_launch_count(self) -> int:
        v = C.c_int64()
        _check(lib().kvp_engine_last_launch_count(self._h, C.byref(v)), "last_launch_count")
        return int(v.value)


def init_weights(config: ModelConfig, devices: Sequence[int] = (0,)) -> WeightSet:
    return WeightSet(config, devices)


def _fault(f: Optional[FaultInjection]):
    if f is None:
        return None
    return C.byref(_Fault(int(f.kind), f.rank, f.layer))


def run(strategy: Strategy, context, partition: ContextPartition, weights: WeightSet,
        fault: Optional[FaultInjection] = None, want_hidden: bool = True) -> ExecutionResult:
    """run<T> (engine.hpp:186-318)."""
    ctx = _f32(context)
    d = weights.config.d_model
    if ctx.ndim != 2 or ctx.shape[1] != d:
        raise DimensionError("context must be C x d_model")
    b = _i64(partition.boundaries)
    if len(b) < 2:
        raise PartitionError("boundaries must run from 0 to the context length")
    if partition.context_length != ctx.shape[0]:
        raise InputError(f"partition covers {partition.context_length} tokens but the context has "
                         f"{ctx.shape[0]} rows")
    Cn = ctx.shape[0]
    hid = np.empty((Cn, d), np.float32) if want_hidden else None
    ft = np.empty((1, d), np.float32)
    m = _Metrics()
    _check(lib().kvp_engine_run(weights.handle, int(strategy), _vp(ctx), Cn, _ip(b), len(b) - 1, _fault(fault),
                                _vp(hid), _vp(ft), C.byref(m)), "run")
    return ExecutionResult(hid, ft, ExecutionMetrics._from_c(m))


def run_device(strategy: Strategy, context_ptr: int, C_: int, partition: ContextPartition, weights: WeightSet,
               first_token_ptr: int, hidden_ptr: int = 0) -> ExecutionMetrics:
    """run() with inputs/outputs already resident in HBM (device pointers on devices[0])."""
    b = _i64(partition.boundaries)
    m = _Metrics()
    _check(lib().kvp_engine_run_device(weights.handle, int(strategy), C.c_void_p(context_ptr), C_, _ip(b),
                                       len(b) - 1, None, C.c_void_p(hidden_ptr or None),
                                       C.c_void_p(first_token_ptr or None), C.byref(m)), "run_device")
    return ExecutionMetrics._from_c(m)


# ------------------------------------------------------------------ KV cache + decode (8f #4)
class KVCache:
    """Device K/V cache of `capacity` rows per layer for the prompt + decode steps (new: the
    reference stops at the first token, engine.hpp:88).  prefill() runs the single-rank prompt
    phase into it; decode() appends up to 8 rows at the next positions, attending to the whole
    cache -- the rows a longer serial forward would produce (causal prefix property)."""

    def __init__(self, weights: WeightSet, capacity: int):
        self.w = weights
        h = C.c_void_p()
        _check(lib().kvp_kv_cache_create(weights.handle, int(capacity), C.byref(h)), "kv_cache_create")
        self._h = h
        self.capacity = int(capacity)

    @property
    def length(self) -> int:
        v = C.c_int64()
        _check(lib().kvp_kv_cache_length(self._h, C.byref(v)), "kv_cache_length")
        return int(v.value)

    def reset(self, length: int = 0) -> None:
        _check(lib().kvp_kv_cache_reset(self._h, int(length)), "kv_cache_reset")

    def prefill(self, context, want_hidden: bool = False):
        """Prompt phase into the cache (length := C); returns (first_token_hidden [1 x d],
        hidden_out [C x d] or None, device ms)."""
        ctx = _f32(context)
        d = self.w.config.d_model
        if ctx.ndim != 2 or ctx.shape[1] != d:
            raise DimensionError("context must be C x d_model")
        ft = np.empty((1, d), np.float32)
        hid = np.empty(ctx.shape, np.float32) if want_hidden else None
        ms = C.c_float()
        _check(lib().kvp_prefill_cached(self.w.handle, self._h, _vp(ctx), ctx.shape[0], _vp(hid), _vp(ft),
                                        C.byref(ms)), "prefill_cached")
        return ft, hid, float(ms.value)

    def decode(self, rows):
        """Appends rows (n x d, n <= 8) at positions [length, length + n); returns (their final
        hidden rows, device ms)."""
        r = _f32(rows)
        d = self.w.config.d_model
        if r.ndim != 2 or r.shape[1] != d:
            raise DimensionError("decode rows must be n x d_model")
        out = np.empty(r.shape, np.float32)
        ms = C.c_float()
        _check(lib().kvp_decode(self.w.handle, self._h, _vp(r), r.shape[0], _vp(out), C.byref(ms)), "decode")
        return out, float(ms.value)

    def close(self) -> None:
        if self._h:
            lib().kvp_kv_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ model.hpp
@dataclass
class CausalMask:
    offset: int = 0
    rows: int = 0


@dataclass
class LayerQKV:
    Q: np.ndarray
    K: np.ndarray
    V: np.ndarray


def layer_qkv(hidden, weights: WeightSet, layer: int) -> LayerQKV:
    cfg = weights.config
    h = _f32(hidden)
    if h.ndim != 2 or h.shape[1] != cfg.d_model:
        raise DimensionError(f"qkv_project: hidden width {h.shape[-1]} != d_model {cfg.d_model}")
    r = h.shape[0]
    Q = np.empty((r, cfg.q_dim()), np.float32)
    K = np.empty((r, cfg.kv_dim()), np.float32)
    V = np.empty((r, cfg.kv_dim()), np.float32)
    _check(lib().kvp_layer_qkv(weights.handle, layer, _vp(h), r, _vp(Q), _vp(K), _vp(V)), "layer_qkv")
    return LayerQKV(Q, K, V)


def causal_attention(Q, K, V, mask: CausalMask, weights: WeightSet) -> np.ndarray:
    cfg = weights.config
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    if K.shape != V.shape:
        raise DimensionError("causal_attention: K/V shape mismatch")
    if Q.shape[0] != mask.rows:
        raise DimensionError("causal_attention: Q rows != mask rows")
    if K.shape[0] < mask.offset + Q.shape[0]:
        raise CacheError(f"causal_attention: cache holds {K.shape[0]} rows, need at least "
                         f"{mask.offset + Q.shape[0]}")
    A = np.empty((Q.shape[0], cfg.q_dim()), np.float32)
    _check(lib().kvp_causal_attention(weights.handle, _vp(Q), Q.shape[0], _vp(K), _vp(V), K.shape[0],
                                      mask.offset, _vp(A)), "causal_attention")
    return A


def layer_finish(hidden, Q, K_full, V_full, offset: int, weights: WeightSet, layer: int) -> np.ndarray:
    cfg = weights.config
    h, Q, K, V = _f32(hidden), _f32(Q), _f32(K_full), _f32(V_full)
    if K.shape != V.shape:
        raise DimensionError("causal_attention: K/V shape mismatch")
    if K.shape[0] < offset + h.shape[0]:
        raise CacheError("causal_attention: cache too short for the mask")
    out = np.empty((h.shape[0], cfg.d_model), np.float32)
    _check(lib().kvp_layer_finish(weights.handle, layer, _vp(h), h.shape[0], _vp(Q), _vp(K), _vp(V), K.shape[0],
                                  offset, _vp(out)), "layer_finish")
    return out


@dataclass
class KVCacheSegment:
    """KVCacheSegment (kv_cache.hpp:14-31): K and V rows of one layer for token positions
    [start_pos, end_pos)."""
    layer: int
    start_pos: int
    end_pos: int
    K: np.ndarray
    V: np.ndarray

    def token_rows(self) -> int:
        return self.end_pos - self.start_pos

    def validate(self) -> None:
        if self.start_pos < 0 or self.start_pos >= self.end_pos:
            raise CacheError("segment positions must satisfy 0 <= start < end")
        if self.K.shape[0] != self.token_rows() or self.K.shape != self.V.shape:
            raise CacheError("segment K/V rows must match the covered token range")


def validate_cache_coverage(segments: Sequence[KVCacheSegment], expected_tokens: int) -> None:
    """validate_cache_coverage (kv_cache.hpp:41-55)."""
    nxt = 0
    for seg in segments:
        seg.validate()
        if seg.start_pos != nxt:
            raise CacheError(f"cache gap: expected segment at position {nxt}, got {seg.start_pos}")
        nxt = seg.end_pos
    if nxt != expected_tokens:
        raise CacheError(f"cache covers {nxt} tokens, expected {expected_tokens}")


def forward_serial(context, weights: WeightSet):
    """forward_serial (model.hpp:197-211) -> (final hidden states [C x d], one KVCacheSegment
    per layer covering [0, C), copied back from the device cache)."""
    ctx = _f32(context)
    if ctx.ndim != 2 or ctx.shape[0] < 1:
        raise InputError("forward_serial: empty context")
    cfg = weights.config
    if ctx.shape[1] != cfg.d_model:
        raise DimensionError(f"qkv_project: hidden width {ctx.shape[1]} != d_model {cfg.d_model}")
    Cn = ctx.shape[0]
    hid = np.empty((Cn, cfg.d_model), np.float32)
    kvb = np.empty((cfg.n_layers, 2, Cn, cfg.kv_dim()), np.float32)
    _check(lib().kvp_forward_serial(weights.handle, _vp(ctx), Cn, _vp(hid), _vp(kvb)), "forward_serial")
    return hid, [KVCacheSegment(l, 0, Cn, kvb[l, 0], kvb[l, 1]) for l in range(cfg.n_layers)]


def random_context(rows: int, d_model: int, seed: int) -> np.ndarray:
    """random_context<float> (weights.hpp:86-89): rows x d_model uniform [-1, 1) from the
    SplitMix64 stream mix_seed(seed, 0xc7, 17) -- the reference's prompt, bit for bit."""
    out = np.empty((int(rows), int(d_model)), np.float32)
    _check(lib().kvp_random_context(int(rows), int(d_model), int(seed), _vp(out)), "random_context")
    return out


def random_context_device(weights: WeightSet, rows: int, seed: int, out_ptr: int) -> None:
    """random_context generated on the engine's first device into a [rows x d_model] f32
    device buffer (same values as random_context)."""
    _check(lib().kvp_random_context_device(weights.handle, int(rows), int(seed), C.c_void_p(out_ptr)),
           "random_context_device")


# ------------------------------------------------------------------ search.hpp / simnet.hpp
@dataclass
class CostModel:
    alpha: float = 1e-6
    proj_coeff: float = 4e-6
    softmax_coeff: float = 1e-7
    fixed_overhead: float = 1e-5

    def _c(self): return _Cost(self.alpha, self.proj_coeff, self.softmax_coeff, self.fixed_overhead)


@dataclass
class NetworkModel:
    bandwidth: float = 1e7
    latency: float = 1e-6

    @staticmethod
    def zero_comm() -> "NetworkModel":
        return NetworkModel(float("inf"), 0.0)

    def _c(self): return _Net(self.bandwidth, self.latency)


@dataclass
class SearchConfig:
    grid_width: int = 5
    initial_stride: int = 0
    min_stride: int = 1
    evaluator: Optional[Callable[[ContextPartition], float]] = None

    def _c(self): return _SearchCfg(self.grid_width, self.initial_stride, self.min_stride)

    def resolve_initial_stride(self, C_: int, p: int) -> int:
        if self.initial_stride > 0:
            return self.initial_stride
        target = C_ / (4.0 * p)
        s = 1
        while s < target:
            s *= 2
        return max(s, self.min_stride)


@dataclass
class SearchResult:
    partition: ContextPartition
    ttft: float
    evaluations: int
    levels: int


def _wrap_eval(C_: int, fn):
    if fn is None:
        return _EVAL()
    return _EVAL(lambda bp, p, _u: float(fn(ContextPartition(C_, [bp[i] for i in range(p + 1)]))))


def hierarchical_grid_search(C_: int, p: int, config: SearchConfig) -> SearchResult:
    out = np.zeros(p + 1 if p >= 1 else 2, np.int64)
    res = _SearchRes()
    cfg = config._c()
    ev = _wrap_eval(C_, config.evaluator)
    _check(lib().kvp_hierarchical_grid_search(C_, p, C.byref(cfg), ev, None, _ip(out), C.byref(res)),
           "hierarchical_grid_search")
    return SearchResult(ContextPartition(C_, out.tolist()), res.ttft, res.evaluations, res.levels)


def binary_search_two(C_: int, config: SearchConfig) -> SearchResult:
    out = np.zeros(3, np.int64)
    res = _SearchRes()
    cfg = config._c()
    ev = _wrap_eval(C_, config.evaluator)
    _check(lib().kvp_binary_search_two(C_, C.byref(cfg), ev, None, _ip(out), C.byref(res)), "binary_search_two")
    return SearchResult(ContextPartition(C_, out.tolist()), res.ttft, res.evaluations, res.levels)


def simulate_ttft(strategy: Strategy, partition: ContextPartition, model: ModelConfig, cost: CostModel,
                  net: NetworkModel) -> float:
    b = _i64(partition.boundaries)
    out = C.c_double()
    cc, nc = cost._c(), net._c()
    _check(lib().kvp_simulate_ttft(int(strategy), partition.context_length, _ip(b), len(b) - 1, model.n_layers,
                                   C.byref(cc), C.byref(nc), C.byref(out)), "simulate_ttft")
    return out.value


def search_partition(C_: int, p: int, model: ModelConfig, cost: CostModel, net: NetworkModel,
                     config: Optional[SearchConfig] = None) -> SearchResult:
    """KVR-S: hierarchical grid search scored by simulate_ttft(KVR) (commands.hpp:252-278)."""
    config = config or SearchConfig()
    out = np.zeros(p + 1, np.int64)
    res = _SearchRes()
    cc, nc, sc = cost._c(), net._c(), config._c()
    _check(lib().kvp_search_partition(C_, p, model.n_layers, C.byref(cc), C.byref(nc), C.byref(sc), _ip(out),
                                      C.byref(res)), "search_partition")
    return SearchResult(ContextPartition(C_, out.tolist()), res.ttft, res.evaluations, res.levels)


def simulate_ttft_causal(strategy: Strategy, partition: ContextPartition, model: ModelConfig, cost: CostModel,
                         net: NetworkModel) -> float:
    """Extension: simulate_ttft with attention priced on causal-visible pairs (B200 kernels)."""
    b = _i64(partition.boundaries)
    out = C.c_double()
    cc, nc = cost._c(), net._c()
    _check(lib().kvp_simulate_ttft_causal(int(strategy), partition.context_length, _ip(b), len(b) - 1,
                                          model.n_layers, C.byref(cc), C.byref(nc), C.byref(out)),
           "simulate_ttft_causal")
    return out.value


def search_partition_causal(C_: int, p: int, model: ModelConfig, cost: CostModel, net: NetworkModel,
                            config: Optional[SearchConfig] = None) -> SearchResult:
    config = config or SearchConfig()
    out = np.zeros(p + 1, np.int64)
    res = _SearchRes()
    cc, nc, sc = cost._c(), net._c(), config._c()
    _check(lib().kvp_search_partition_causal(C_, p, model.n_layers, C.byref(cc), C.byref(nc), C.byref(sc),
                                             _ip(out), C.byref(res)), "search_partition_causal")
    return SearchResult(ContextPartition(C_, out.tolist()), res.ttft, res.evaluations, res.levels)


def ttft_star(C_: int, p: int, alpha: float) -> float:
    out = C.c_double()
    _check(lib().kvp_ttft_star(C_, p, alpha, C.byref(out)), "ttft_star")
    return out.value


def practical_bound(C_: int, p: int, model: ModelConfig, cost: CostModel):
    out = np.zeros(p + 1, np.int64)
    t = C.c_double()
    cc = cost._c()
    _check(lib().kvp_practical_bound(C_, p, model.n_layers, C.byref(cc), _ip(out), C.byref(t)), "practical_bound")
    return ContextPartition(C_, out.tolist()), t.value


def calibrate_alpha(measurements) -> float:
    Cs = np.ascontiguousarray([m[0] for m in measurements], dtype=np.int64)
    ts = np.ascontiguousarray([m[1] for m in measurements], dtype=np.float64)
    out = C.c_double()
    _check(lib().kvp_calibrate_alpha(_vp(Cs), _vp(ts), len(Cs), C.byref(out)), "calibrate_alpha")
    return out.value


def fit_cost_model(local_rows, held_rows, proj_s, rest_s) -> CostModel:
    """Calibrates the balancer's CostModel from measured per-layer device times."""
    a = _i64(local_rows)
    b = _i64(held_rows)
    c = np.ascontiguousarray(proj_s, dtype=np.float64)
    d = np.ascontiguousarray(rest_s, dtype=np.float64)
    out = _Cost()
    _check(lib().kvp_fit_cost_model(_vp(a), _vp(b), _vp(c), _vp(d), len(a), C.byref(out)), "fit_cost_model")
    return CostModel(out.alpha, out.proj_coeff, out.softmax_coeff, out.fixed_overhead)


def profile_grid(weights: WeightSet, C_: int, p: int, reps: int = 3):
    """Measured per-rank layer times on a grid of (local rows c, prefix b) points spanning the
    partitions a search at (C, p) visits: list of (c, b, proj_s, rest_s)."""
    pts = []
    for frac in (0.5, 1.0, 1.5):
        c = max(1, int(round(frac * C_ / p)))
        for b in sorted({0, C_ // 4, C_ // 2, (3 * C_) // 4}):
            if b + c > C_:
                continue
            pm, rm = weights.profile_layer(c, b, reps)
            pts.append((c, b, pm * 1e-3, rm * 1e-3))
    return pts


def fit_causal_cost_model(points) -> CostModel:
    """Extension: CostModel whose alpha prices causal-visible pairs c*(b + (c+1)/2) -- the work
    of the tile-skipping B200 attention -- for simulate_ttft_causal / search_partition_causal."""
    c = np.array([x[0] for x in points], np.float64)
    b = np.array([x[1] for x in points], np.float64)
    proj = np.array([x[2] for x in points], np.float64)
    rest = np.array([x[3] for x in points], np.float64)
    a = float(np.dot(proj, c) / np.dot(c, c))
    X = np.stack([c * (b + 0.5 * (c + 1)), c, np.ones_like(c)], 1)
    w, *_ = np.linalg.lstsq(X, rest, rcond=None)
    w = np.maximum(w, 0.0)
    return CostModel(alpha=float(max(w[0], 1e-300)), proj_coeff=a, softmax_coeff=float(w[1]),
                     fixed_overhead=float(w[2]))


def calibrate_cost_model(weights: WeightSet, C_: int, p: int, reps: int = 3, points=None) -> CostModel:
    """Fits the balancer's CostModel to MEASURED B200 layer times: one rank's layer executor is
    timed in isolation on a grid of (local rows, prefix) points that spans the partitions
    the search will visit at (C, p), then kvp_fit_cost_model solves proj ~ a*c and
    rest ~ alpha*c*held + s*c + f.  Times are per layer; simulate_ttft multiplies by L."""
    pts = points if points is not None else profile_grid(weights, C_, p, reps)
    return fit_cost_model([x[0] for x in pts], [x[0] + x[1] for x in pts], [x[2] for x in pts],
                          [x[3] for x in pts])


@dataclass
class NoiseSidecar:
    """simnet.hpp:65-78: per layer one adjacent link (drawn from (seed, layer)) runs at
    bandwidth / slowdown_factor."""
    seed: int = 1
    slowdown_factor: float = 1.0

    def degraded_link(self, layer: int, link_count: int) -> int:
        """simnet.hpp:71-75: the adjacent link (i -> i+1) slowed in `layer` (-1 without links)."""
        out = C.c_int64()
        _check(lib().kvp_noise_degraded_link(C.c_uint64(self.seed), layer, link_count, C.byref(out)),
               "noise_degraded_link")
        return int(out.value)

    @staticmethod
    def for_trial(study_seed: int, trial: int, slowdown_factor: float) -> "NoiseSidecar":
        """noise_study's sidecar of trial t: seed mix_seed(seed, 0x7472, t) (simnet.hpp:342-344)."""
        out = C.c_uint64()
        _check(lib().kvp_noise_trial_seed(C.c_uint64(study_seed), trial, C.byref(out)), "noise_trial_seed")
        return NoiseSidecar(int(out.value), slowdown_factor)


def simulate_ttft_noisy(strategy: Strategy, partition: ContextPartition, model: ModelConfig, cost: CostModel,
                        net: NetworkModel, noise: NoiseSidecar) -> float:
    b = _i64(partition.boundaries)
    out = C.c_double()
    cc, nc = cost._c(), net._c()
    _check(lib().kvp_simulate_ttft_noisy(int(strategy), partition.context_length, _ip(b), len(b) - 1,
                                         model.n_layers, C.byref(cc), C.byref(nc), noise.seed, noise.slowdown_factor,
                                         C.byref(out)), "simulate_ttft_noisy")
    return out.value


@dataclass
class NoiseStudy:
    quiet_ttft: float
    mean_degradation: float
    max_degradation: float
    per_trial: list


def noise_study(strategy: Strategy, partition: ContextPartition, model: ModelConfig, cost: CostModel,
                net: NetworkModel, slowdown_factor: float, trials: int, seed: int) -> NoiseStudy:
    """noise_study (simnet.hpp:332-353)."""
    b = _i64(partition.boundaries)
    q, mean, mx = C.c_double(), C.c_double(), C.c_double()
    per = np.zeros(max(trials, 1), np.float64)
    cc, nc = cost._c(), net._c()
    _check(lib().kvp_noise_study(int(strategy), partition.context_length, _ip(b), len(b) - 1, model.n_layers,
                                 C.byref(cc), C.byref(nc), slowdown_factor, trials, seed, C.byref(q), C.byref(mean),
                                 C.byref(mx), _vp(per)), "noise_study")
    return NoiseStudy(q.value, mean.value, mx.value, per[:trials].tolist())


@dataclass
class PartitionLookupTable:
    """KVR-P table (lookup_table.hpp:22-39): context length -> ratios, JSON schema
    {"p": int, "entries": [{"context_length": int, "ratios": [float]}]} (lookup_table.hpp:72-97)."""
    process_count: int = 0
    entries: dict = field(default_factory=dict)

    def insert(self, context_length: int, ratios) -> None:
        if self.process_count < 1:
            raise LookupError_("table process count not set")
        if len(ratios) != self.process_count:
            raise LookupError_("ratio vector arity must equal the table process count")
        if any(r < 0 for r in ratios):
            raise LookupError_("table ratios must be non-negative")
        if abs(sum(ratios) - 1.0) > 1e-9:
            raise LookupError_("table ratios must sum to 1")
        if context_length < 1:
            raise LookupError_("context length must be positive")
        self.entries[int(context_length)] = [float(r) for r in ratios]

    def _arrays(self):
        keys = sorted(self.entries)
        Cs = np.asarray(keys, np.int64)
        R = np.ascontiguousarray([self.entries[k] for k in keys], dtype=np.float64).reshape(len(keys), -1) \
            if keys else np.zeros((0, max(self.process_count, 1)))
        return Cs, R

    def to_json(self) -> dict:
        return {"p": self.process_count,
                "entries": [{"context_length": k, "ratios": self.entries[k]} for k in sorted(self.entries)]}

    @staticmethod
    def from_json(doc: dict) -> "PartitionLookupTable":
        try:
            t = PartitionLookupTable(int(doc["p"]))
            for e in doc["entries"]:
                t.insert(int(e["context_length"]), list(e["ratios"]))
        except (KeyError, TypeError, ValueError) as ex:
            raise LookupError_(f"malformed lookup table: {ex}")
        return t

    def save(self, path: str) -> None:
        import json
        try:
            with open(path, "w") as f:
                json.dump(self.to_json(), f, indent=2, sort_keys=True)  # nlohmann::json key order
                f.write("\n")
        except OSError as ex:
            raise IoError(f"cannot open table file for writing: {path}: {ex}")

    @staticmethod
    def load(path: str) -> "PartitionLookupTable":
        import json
        try:
            with open(path) as f:
                doc = json.load(f)
        except OSError as ex:
            raise IoError(f"cannot open table file: {path}: {ex}")
        except ValueError as ex:
            raise LookupError_(f"malformed lookup table JSON in {path}: {ex}")
        return PartitionLookupTable.from_json(doc)


def interpolate_partition(table: PartitionLookupTable, C_: int) -> list:
    Cs, R = table._arrays()
    p = max(table.process_count, 0)
    out = np.zeros(max(p, 1), np.float64)
    _check(lib().kvp_interpolate_partition(_ip(Cs), _vp(R), len(Cs), p, C_, _vp(out)), "interpolate_partition")
    return out[:p].tolist()


def partition_from_table(table: PartitionLookupTable, C_: int) -> ContextPartition:
    Cs, R = table._arrays()
    p = max(table.process_count, 0)
    out = np.zeros(max(p, 1) + 1, np.int64)
    _check(lib().kvp_partition_from_table(_ip(Cs), _vp(R), len(Cs), p, C_, _ip(out)), "partition_from_table")
    return ContextPartition(C_, out[:p + 1].tolist())


def max_rel_dev(a, b) -> float:
    """max_rel_dev (matrix.hpp:101-115): max |a - b| / max(1, |b|)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise DimensionError("deviation requires equal shapes")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))
