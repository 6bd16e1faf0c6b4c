import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_2405_05329_b200 import kvprefill as kv
W = kv.init_weights(kv.ModelConfig(4096, 32, 32, 2, 1, "bf16", True))
C_ = 2048
ctx = O.random_context(C_, 4096, 18, np.float32)
s1 = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(C_, 1), W).hidden_out
s2 = kv.run(kv.Strategy.Serial, ctx, kv.even_partition(C_, 1), W).hidden_out
print("serial determinism", np.array_equal(s1, s2), np.abs(s1 - s2).max())
for name, part in (("kvr", kv.partition_from_ratios(C_, [0.4, 0.3, 0.2, 0.1])), ("even4", kv.even_partition(C_, 4)),
                   ("even2", kv.even_partition(C_, 2))):
    r = kv.run(kv.Strategy.KVR, ctx, part, W).hidden_out
    bad = np.where(np.any(r != s1, axis=1))[0]
    print(name, part.boundaries, "rows differing:", len(bad), bad[:10], bad[-10:] if len(bad) else "", np.abs(r - s1).max())
# attention with big-magnitude inputs
W1 = kv.init_weights(kv.ModelConfig(1024, 8, 8, 1, 1, "bf16", False))
for scale in (1.0, 4.0, 16.0):
    Q = O.random_context(C_, 1024, 31, np.float32) * scale
    K = O.random_context(C_, 1024, 32, np.float32) * scale
    V = O.random_context(C_, 1024, 33, np.float32)
    full = kv.causal_attention(Q, K, V, kv.CausalMask(0, C_), W1)
    for lo, hi in ((819, 1433), (1433, 1843), (5, 300)):
        part = kv.causal_attention(Q[lo:hi], K[:hi], V[:hi], kv.CausalMask(lo, hi - lo), W1)
        bad = np.where(np.any(part != full[lo:hi], axis=1))[0]
        print("attn scale", scale, lo, hi, "rows differing", len(bad), bad[:8] + lo if len(bad) else "")
