"""Decode on the prefilled KV cache (no reference counterpart, so parity rests on
the reference model's causal prefix property): prefilling C rows into a KVCache and decoding
rows C, C+1, ... must give the hidden rows a serial forward over the longer context gives
(forward_serial, model.hpp:197-211).
  * f32 mode: the decode step runs the same ordered SIMT kernels as a KVR rank with offset C,
    so it equals the GPU serial run bit for bit and the oracle within the f32 bound;
  * bf16 mode: the decode step runs the HBM-bound GEMV and split-key attention (different
    accumulation order from the tcgen05 path): within 2e-2 of the GPU serial run and within the
    bf16 bound of the oracle, argmax equal."""
import numpy as np
import pytest

import oracle as O
from paper_2405_05329_b200 import kvprefill as kv

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-1


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")


def _serial(W, ctx):
    return kv.run(kv.Strategy.Serial, ctx, kv.even_partition(ctx.shape[0], 1), W).hidden_out


@pytest.mark.parametrize("d,h,kvh,L,rms", [(32, 4, 4, 2, False), (64, 4, 2, 2, True)])
def test_decode_f32_bitwise_equals_serial(d, h, kvh, L, rms):
    W = kv.init_weights(kv.ModelConfig(d, h, kvh, L, 1, "f32", rms))
    C_, steps = 100, [1, 3, 1]
    ctx = O.random_context(C_ + sum(steps), d, 18, np.float32)
    cache = kv.KVCache(W, C_ + sum(steps))
    ft, _, _ = cache.prefill(ctx[:C_])
    full = _serial(W, ctx)
    assert np.array_equal(ft, full[C_ - 1:C_])
    pos = C_
    for n in steps:
        out, ms = cache.decode(ctx[pos:pos + n])
        assert np.array_equal(out, full[pos:pos + n]), (pos, n)
        pos += n
        assert cache.length == pos and ms > 0
    m = O.Model(d, h, kvh, L, 1, "f32", rms)
    ref = O.forward_serial(m, O.init_weights(m, np.float32), ctx)
    assert kv.max_rel_dev(full[C_:], ref[C_:]) <= 1e-4
    cache.close()
    W.close()


@pytest.mark.parametrize("d,h,kvh", [(1024, 8, 8), (1024, 8, 2), (512, 8, 1)])
def test_decode_bf16_matches_serial(d, h, kvh):
    L = 2
    W = kv.init_weights(kv.ModelConfig(d, h, kvh, L, 3, "bf16", True))
    C_, steps = 300, [1, 4, 1, 8]
    ctx = O.random_context(C_ + sum(steps), d, 7, np.float32)
    cache = kv.KVCache(W, C_ + sum(steps))
    cache.prefill(ctx[:C_])
    full = _serial(W, ctx)
    m = O.Model(d, h, kvh, L, 3, "f32", True)
    ref = O.forward_serial(m, O.init_weights(m, np.float32), ctx)
    pos = C_
    for n in steps:
        out, _ = cache.decode(ctx[pos:pos + n])
        assert kv.max_rel_dev(out, full[pos:pos + n]) <= 2e-2, (pos, n)
        assert kv.max_rel_dev(out, ref[pos:pos + n]) <= BF16_TOL, (pos, n)
        top2 = np.sort(ref[pos + n - 1])[-2:]
        if top2[1] - top2[0] > BF16_TOL * max(1.0, abs(top2[1])):
            assert int(np.argmax(out[-1])) == int(np.argmax(ref[pos + n - 1]))
        pos += n
    # re-decoding from a truncated cache reproduces the same rows (deterministic kernels)
    cache.reset(C_)
    first, _ = cache.decode(ctx[C_:C_ + 1])
    cache.reset(C_)
    again, _ = cache.decode(ctx[C_:C_ + 1])
    assert np.array_equal(again, first)
    cache.close()
    W.close()


def test_decode_errors():
    W = kv.init_weights(kv.ModelConfig(256, 2, 2, 1, 1, "bf16", False))
    cache = kv.KVCache(W, 20)
    ctx = O.random_context(20, 256, 1, np.float32)
    with pytest.raises(kv.CacheError):
        cache.decode(ctx[:1])  # nothing prefilled
    cache.prefill(ctx[:16])
    with pytest.raises(kv.InputError):
        cache.decode(ctx[:9])  # more than 8 rows per step
    cache.decode(ctx[16:20])
    with pytest.raises(kv.CacheError):
        cache.decode(ctx[:1])  # capacity exhausted
    with pytest.raises(kv.CacheError):
        cache.reset(21)
    cache.close()
    W.close()
