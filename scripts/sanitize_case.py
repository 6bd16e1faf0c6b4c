"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
`smoke` = __graft_entry__.smoke(); `kvr3` = the fused-handoff KVR chain with 3 ranks on one
GPU (bf16 tcgen05 path: the QKV epilogue stores into the next rank's cache, the upstream
prefix forwarded on the copy engine) checked bitwise against the serial run; `decode` = a
prefill + decode step on the KV cache (GEMV + split-key decode attention)."""
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
    print("case", case, "ok")


if __name__ == "__main__":
    main(sys.argv[1])
