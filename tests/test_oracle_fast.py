"""Pins the multi-threaded f32 restatement (oracle/kvp_oracle_fast.c) that generates the
benchmark-shape goldens (tests/golden/golden_large.json) against the unmodified reference
(oracle/_ref) at the same widths with fewer layers/tokens, bit for bit; and the product's
random_context (C-ABI + Python mirror) against the reference's weights.hpp:86-89."""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2405_05329_b200 import kvprefill as kv

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_large.json")
ref_missing = not O.Reference.available()


@pytest.mark.skipif(ref_missing, reason="oracle/_ref not built")
@pytest.mark.parametrize("kw,C_,p", [
    (dict(d_model=32, n_heads=4, n_kv_heads=4, n_layers=2, seed=1, rms_norm=False), 1024, 2),  # configs[0]
    (dict(d_model=32, n_heads=4, n_kv_heads=1, n_layers=2, seed=1, rms_norm=True), 300, 3),
    (dict(d_model=512, n_heads=8, n_kv_heads=2, n_layers=3, seed=5, rms_norm=False), 333, 3),
    (dict(d_model=4096, n_heads=32, n_kv_heads=32, n_layers=1, seed=1, rms_norm=True), 80, 2),  # Llama-7B width
    (dict(d_model=4544, n_heads=71, n_kv_heads=1, n_layers=1, seed=1, rms_norm=True), 40, 2),  # Falcon-7B width
])
def test_fast_oracle_bitwise_vs_reference(kw, C_, p):
    m = O.Model(precision="f32", **kw)
    ref = O.Reference()
    ctx = ref.random_context(C_, m.d_model, 18, np.float32)
    hid, last = O.forward_fast_f32(m, ctx)
    h_ref, ft, _ = ref.weights(m).run(O.KVR, ctx, ref.even_partition(C_, p))
    assert np.array_equal(hid.view(np.uint32), h_ref.view(np.uint32))
    assert np.array_equal(last.view(np.uint32), ft[0].view(np.uint32))


@pytest.mark.skipif(ref_missing, reason="oracle/_ref not built")
@pytest.mark.parametrize("rows,d,seed", [(1024, 32, 18), (7, 4096, 18), (3, 4544, 1 + 17)])
def test_random_context_is_the_references(rows, d, seed):
    want = O.Reference().random_context(rows, d, seed, np.float32)
    got = kv.random_context(rows, d, seed)
    assert got.dtype == np.float32 and np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_golden_large_fixture_shape():
    g = json.load(open(GOLDEN))["cases"]
    for name in ("llama7b-4k", "falcon7b-8k", "llama7b-1k", "falcon7b-1k"):
        c = g[name]
        assert len(c["first_token_hidden"]) == c["model"]["d_model"]
        assert c["argmax"] == int(np.argmax(np.asarray(c["first_token_hidden"], np.float32)))
        if "pinned_by_reference" in c:
            assert c["pinned_by_reference"]["hidden_equal"] and c["pinned_by_reference"]["first_token_equal"]
