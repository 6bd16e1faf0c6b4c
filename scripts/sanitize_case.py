"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
`smoke` = __graft_entry__.smoke(); `kvr3` = the fused-handoff KVR chain with 3 ranks on one
GPU (bf16 tcgen05 path: the QKV epilogue stores into the next rank's cache, the upstream
prefix forwarded on the copy engine) checked bitwise against the serial run; `decode` = a
prefill + decode step on the KV cache (GEMV + split-key decode attention); `f32` = the fp32
parity mode at head_dim 128 and 64 (ordered SIMT GEMM, tiled SIMT attention) over a ragged
split, bitwise against its serial run; `ranks` = rank chunks at Llama width that take
attn_tc and attn_tb (wave-fill selection), bitwise against the serial launch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(case):
    from paper_2405_05329_b200 import kvprefill as kv
    if case == "smoke":
        import __graft_entry__
        __graft_entry__.smoke()
    elif case == "kvr3":
        W = kv.init_weights(kv.ModelConfig(512, 4, 4, 2, 1, "bf16", True))
        ctx = kv.random_context(600, 512, 18)
        s = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(600, 1), W)
        r = kv.run(kv.Strategy.KVR, ctx, kv.partition_from_ratios(600, [0.5, 0.3, 0.2]), W)
        t = kv.run(kv.Strategy.TSP, ctx, kv.even_partition(600, 3), W)
        assert np.array_equal(s.hidden_out, r.hidden_out) and np.array_equal(s.hidden_out, t.hidden_out)
    elif case == "decode":
        W = kv.init_weights(kv.ModelConfig(512, 8, 2, 2, 1, "bf16", True))
        ctx = kv.random_context(260, 512, 18)
        c = kv.KVCache(W, 264)
        c.prefill(ctx[:256])
        c.decode(ctx[256:260])
    elif case == "f32":
        for d, h, kvh in ((256, 2, 2), (256, 4, 1)):  # head_dim 128 MHA, head_dim 64 MQA
            W = kv.init_weights(kv.ModelConfig(d, h, kvh, 2, 1, "f32", True))
            ctx = kv.random_context(301, d, 18)
            s = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(301, 1), W)
            r = kv.run(kv.Strategy.KVR, ctx, kv.partition_from_ratios(301, [0.55, 0.45]), W)
            assert np.array_equal(s.hidden_out, r.hidden_out)
            W.close()
    elif case == "ranks":
        W = kv.init_weights(kv.ModelConfig(4096, 32, 32, 1, 1, "bf16"))
        C_ = 2560
        Q = kv.random_context(C_, 4096, 41) * 4.0
        K = kv.random_context(C_, 4096, 42) * 4.0
        V = kv.random_context(C_, 4096, 43)
        full = kv.causal_attention(Q, K, V, kv.CausalMask(0, C_), W)
        for off in (1280, 2048):  # 1280 rows: attn_tc (160 two-tile CTAs vs 320), 512 rows: attn_tb
            part = kv.causal_attention(Q[off:], K, V, kv.CausalMask(off, C_ - off), W)
            assert np.array_equal(part, full[off:]), off
    print("case", case, "ok")


if __name__ == "__main__":
    main(sys.argv[1])
