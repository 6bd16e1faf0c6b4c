"""Quick numerics sanity of the B200 path against the oracle (dev helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2405_05329_b200 as kv

def cmp(name, a, b):
    print(f"{name}: max_rel_dev={kv.max_rel_dev(a, b):.3e}", flush=True)

print("devices", kv.device_count(), flush=True)
# 1) fp32 tiny config T vs reference
for prec in ("f32", "bf16"):
  for rms in (False, True):
    m = O.Model(32, 4, 4, 2, 1, "f32", rms)
    w = O.init_weights(m, np.float32)
    ctx = O.random_context(1024, 32, 18, np.float32)
    ref = O.forward_serial(m, w, ctx)
    cfg = kv.ModelConfig(32, 4, 4, 2, 1, prec, rms)
    W = kv.init_weights(cfg)
    for strat, part in ((kv.Strategy.Serial, kv.even_partition(1024, 1)), (kv.Strategy.KVR, kv.even_partition(1024, 2)), (kv.Strategy.TSP, kv.even_partition(1024, 3))):
        r = W and kv.run(strat, ctx, part, W)
        cmp(f"T {prec} rms={rms} {strat.name}", r.hidden_out, ref)
        print("   argmax", r.first_token, int(np.argmax(ref[-1])), r.metrics)
# 2) GEMM/attention path at tcgen05 shapes: one layer d=1024 h=8 (hd=128)
for prec in ("f32", "bf16"):
    m = O.Model(1024, 8, 8, 1, 3, "f32", True)
    w = O.init_weights(m, np.float32)
    ctx = O.random_context(300, 1024, 5, np.float32)
    t=time.time(); ref = O.forward_serial(m, w, ctx); print("oracle s", time.time()-t)
    W = kv.init_weights(kv.ModelConfig(1024, 8, 8, 1, 3, prec, True))
    q = kv.layer_qkv(ctx, W, 0)
    Q, K, V = O.layer_qkv(m, w, 0, ctx)
    cmp(f"qkv {prec} Q", q.Q, Q); cmp(f"qkv {prec} K", q.K, K); cmp(f"qkv {prec} V", q.V, V)
    A = kv.causal_attention(Q, K, V, kv.CausalMask(0, 300), W)
    cmp(f"attn {prec}", A, O.causal_attention(m, Q, K, V, 0))
    A2 = kv.causal_attention(Q[100:], K, V, kv.CausalMask(100, 200), W)
    cmp(f"attn offset {prec}", A2, O.causal_attention(m, Q[100:], K, V, 100))
    for strat, part in ((kv.Strategy.Serial, kv.even_partition(300, 1)), (kv.Strategy.KVR, kv.partition_from_ratios(300, [.5,.3,.2])), (kv.Strategy.TSP, kv.even_partition(300, 4))):
        r = kv.run(strat, ctx, part, W)
        cmp(f"run {prec} {strat.name}", r.hidden_out, ref)
print("OK")
