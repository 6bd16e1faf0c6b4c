"""Opt-in rotary position embedding (north star: "RMSNorm/RoPE ... fused elementwise kernels";
the reference model itself has none -- SURVEY 0 -- so it is off by default and absent from the
f32 parity mode).  Checked against a plain PyTorch fp32 restatement of the reference model
(model.hpp:29-211) with RoPE applied to Q and K, and by the properties the engine must keep
with it on: KVR / TSP on any partition equal the serial run bit for bit (every rank rotates
its rows by their ABSOLUTE positions), decode continues the prompt, and switching it off
restores the reference model exactly."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2405_05329_b200 import kvprefill as kv

pytestmark = pytest.mark.gpu
THETA = 10000.0
TOL = 5e-2  # bf16 operands / fp32 accumulation against the fp32 restatement


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if kv.device_count() == 0:
        pytest.skip("no CUDA device")


def rope_ref(X, pos, hd, theta):
    """Pairs (2i, 2i+1) of each head rotate by pos * theta^(-2i/hd) (fp32)."""
    C_, w = X.shape
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float32) / hd))
    ang = pos[:, None].to(torch.float32) * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)
    x = X.view(C_, w // hd, hd // 2, 2)
    x0, x1 = x[..., 0], x[..., 1]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.stack((x0 * c - x1 * s, x0 * s + x1 * c), dim=-1).reshape(C_, w)


def torch_forward(m, weights, ctx, theta):
    """model.hpp forward_serial in fp32 torch, RoPE on Q and K when theta > 0."""
    hd, group = m.head_dim, m.n_heads // m.n_kv_heads
    h = torch.from_numpy(np.array(ctx, dtype=np.float32))
    C_ = h.shape[0]
    pos = torch.arange(C_)
    mask = torch.triu(torch.ones(C_, C_, dtype=torch.bool), 1)

    def norm(x):
        return x * torch.rsqrt((x * x).mean(dim=1, keepdim=True) + 1e-6) if m.rms_norm else x

    for wq, wk, wv, wo, w1, w2 in weights:
        wq, wk, wv, wo, w1, w2 = (torch.from_numpy(w) for w in (wq, wk, wv, wo, w1, w2))
        x = norm(h)
        Q, K, V = x @ wq, x @ wk, x @ wv
        if theta > 0:
            Q, K = rope_ref(Q, pos, hd, theta), rope_ref(K, pos, hd, theta)
        A = torch.empty_like(Q)
        for hh in range(m.n_heads):
            g = hh // group
            s = (Q[:, hh * hd:(hh + 1) * hd] @ K[:, g * hd:(g + 1) * hd].T) / np.sqrt(hd)
            s = s.masked_fill(mask, float("-inf"))
            A[:, hh * hd:(hh + 1) * hd] = torch.softmax(s, dim=1) @ V[:, g * hd:(g + 1) * hd]
        h1 = h + A @ wo
        h = h1 + torch.relu(norm(h1) @ w1) @ w2
    return h.numpy()


@pytest.mark.parametrize("d,h,kvh", [(512, 4, 2), (256, 4, 1)])  # hd 128 GQA, hd 64 MQA
def test_rope_matches_torch_fp32_and_strategies_stay_bitwise(d, h, kvh):
    m = O.Model(d, h, kvh, 2, 3, "f32", True)
    C_ = 700
    ctx = O.random_context(C_, d, 18, np.float32)
    ref_rope = torch_forward(m, O.init_weights(m, np.float32), ctx, THETA)
    W = kv.init_weights(kv.ModelConfig(d, h, kvh, 2, 3, "bf16", True))
    plain = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(C_, 1), W)
    W.set_rope(THETA)
    serial = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(C_, 1), W)
    dev = kv.max_rel_dev(serial.hidden_out, ref_rope)
    assert dev <= TOL, dev
    # it is really applied: the rotary model differs from the reference (no-RoPE) model
    assert kv.max_rel_dev(plain.hidden_out, ref_rope) > 4 * dev
    # every rank rotates by absolute positions: KVR (skewed) and TSP equal the serial run
    kvr = kv.run(kv.Strategy.KVR, ctx, kv.partition_from_ratios(C_, [0.5, 0.3, 0.2]), W)
    tsp = kv.run(kv.Strategy.TSP, ctx, kv.even_partition(C_, 4), W)
    assert np.array_equal(kvr.hidden_out, serial.hidden_out)
    assert np.array_equal(tsp.hidden_out, serial.hidden_out)
    # off again: the reference model, bit for bit
    W.set_rope(0)
    again = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(C_, 1), W)
    assert np.array_equal(again.hidden_out, plain.hidden_out)
    W.close()


def test_rope_decode_continues_the_prompt():
    m = O.Model(512, 4, 2, 2, 5, "f32", True)
    ctx = O.random_context(300, 512, 9, np.float32)
    W = kv.init_weights(kv.ModelConfig(512, 4, 2, 2, 5, "bf16", True))
    W.set_rope(THETA)
    full = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(300, 1), W)
    cache = kv.KVCache(W, 300)
    cache.prefill(ctx[:296])
    out, _ = cache.decode(ctx[296:])
    assert kv.max_rel_dev(out, full.hidden_out[296:]) <= 2e-2
    ref = torch_forward(m, O.init_weights(m, np.float32), ctx, THETA)
    assert kv.max_rel_dev(out, ref[296:]) <= TOL
    cache.close()
    W.close()


def test_rope_is_not_available_in_the_parity_mode():
    W = kv.init_weights(kv.ModelConfig(256, 4, 4, 1, 1, "f32", True))
    with pytest.raises(kv.ConfigError):
        W.set_rope(THETA)
    W.close()
