"""Test-only pieces for the multi-process driver: a CPU layer executor built on the ORACLE
(the checker), so the host-side protocol of paper_2405_05329_b200.distributed runs under
gloo on CPU with world_size 2-4 and can be compared bit-for-bit with the reference's
serial forward pass."""
import numpy as np
import torch

import oracle as O
from paper_2405_05329_b200.distributed import HDR_LEN


class OracleExecutor:
    def __init__(self, model: O.Model, weights):
        self.m = model
        self.w = weights
        self.dtype = np.float64 if model.precision == "f64" else np.float32
        self.tdt = torch.float64 if model.precision == "f64" else torch.float32

    def begin(self, rows, start, held):
        self.h = np.ascontiguousarray(rows, dtype=self.dtype)
        self.start = start
        self.kvbuf = torch.zeros((self.m.n_layers, 2, held, self.m.kv_dim), dtype=self.tdt)

    def stream(self):
        import contextlib
        return contextlib.nullcontext()

    def kv(self, layer):
        return self.kvbuf[layer, 0], self.kvbuf[layer, 1]

    def qkv(self, layer):
        Q, K, V = O.layer_qkv(self.m, self.w, layer, self.h)
        self.Q = Q
        c = self.h.shape[0]
        self.kvbuf[layer, 0, self.start:self.start + c] = torch.from_numpy(K)
        self.kvbuf[layer, 1, self.start:self.start + c] = torch.from_numpy(V)

    def finish(self, layer, k_rows):
        import ctypes as C
        K = self.kvbuf[layer, 0, :k_rows].numpy().copy()
        V = self.kvbuf[layer, 1, :k_rows].numpy().copy()
        sfx = "f64" if self.dtype == np.float64 else "f32"
        fn = getattr(O._Lib.get(), f"kvo_layer_finish_{sfx}")
        fn.argtypes = [C.POINTER(O._Config), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                       C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        keep, wp = O._wptrs(self.w, self.dtype)
        out = np.empty_like(self.h)
        cfg = self.m.c()
        assert fn(C.byref(cfg), wp, layer, O._ptr(self.h), self.h.shape[0], O._ptr(self.Q), O._ptr(K),
                  O._ptr(V), k_rows, self.start, O._ptr(out)) == 0
        self.h = out

    def end(self):
        return self.h, 0.0

    def header(self, values):
        return torch.tensor(values, dtype=torch.int64)

    def empty_header(self):
        return torch.zeros(HDR_LEN, dtype=torch.int64)
