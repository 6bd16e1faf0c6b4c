"""CPU tests of the product library's host half: the C-ABI loads and exports every symbol
declared in include/kvp_b200.h, and the partition plan / load balancer / simulator behind it
(plan.cpp) match the oracle BIT-EXACTLY (partitions, TTFTs, evaluation and level counts).
No compute call is made here: these run without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2405_05329_b200 import kvprefill as kv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "kvp_b200.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"^\s*(?:kvp_status|int32_t|const char\*)\s+(kvp_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 25
    lib = C.CDLL(kv.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(kv.EXPORTED)
    assert kv.lib().kvp_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    if kv.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(kv.CudaError):
        kv.init_weights(kv.ModelConfig(32, 4, 4, 2, 1, "f32"))


def test_config_errors_match_reference():  # config.hpp:36-46
    for bad in (dict(d_model=30, n_heads=4), dict(n_heads=4, n_kv_heads=3), dict(n_layers=0)):
        with pytest.raises(kv.ConfigError):
            kv.ModelConfig(**bad).validate()
    with pytest.raises(kv.ConfigError):  # f64 has no GPU path
        kv.init_weights(kv.ModelConfig(32, 4, 4, 2, 1, "f64"))


def test_partitions_match_oracle():
    rng = np.random.default_rng(7)
    for _ in range(300):
        p = int(rng.integers(1, 9))
        C_ = p + int(rng.integers(0, 20000))
        assert kv.even_partition(C_, p).boundaries == O.even_partition(C_, p)
        r = rng.random(p) + 0.02
        r = (r / r.sum()).tolist()
        assert kv.partition_from_ratios(C_, r).boundaries == O.partition_from_ratios(C_, r)
    assert kv.partition_from_ratios(10240, [0.35, 0.255, 0.21, 0.185]).sizes() == [3584, 2611, 2150, 1895]
    assert kv.partition_from_ratios(3, [0.9, 0.05, 0.05]).sizes() == [1, 1, 1]
    for C_, r in ((10, [0.5, 0.4]), (10, [1.5, -0.5]), (2, [0.4, 0.3, 0.3])):
        with pytest.raises(kv.PartitionError):
            kv.partition_from_ratios(C_, r)
    with pytest.raises(kv.PartitionError):
        kv.even_partition(3, 4)
    with pytest.raises(kv.PartitionError):
        kv.ContextPartition(5, [0, 3, 3, 5]).validate()


def test_accounting_matches_oracle():
    part = kv.ContextPartition.from_sizes([4, 3, 2])
    assert kv.dot_product_counts(kv.Strategy.KVR, part) == [16, 21, 18]
    assert kv.traffic_pairs(kv.Strategy.KVR, part) == 11
    assert kv.traffic_pairs(kv.Strategy.TSP, kv.even_partition(9, 3)) == 18
    with pytest.raises(kv.InputError):
        kv.dot_product_counts(kv.Strategy.Serial, kv.even_partition(8, 2))
    assert kv.dot_product_counts(kv.Strategy.Serial, kv.even_partition(8, 1)) == [64]
    rng = np.random.default_rng(3)
    for _ in range(100):
        p = int(rng.integers(1, 9))
        b = kv.even_partition(p + int(rng.integers(0, 500)), p)
        for s in (kv.Strategy.KVR, kv.Strategy.TSP):
            assert kv.dot_product_counts(s, b) == O.dot_product_counts(int(s), b.boundaries)
            assert kv.traffic_pairs(s, b) == O.traffic_pairs(int(s), b.boundaries)


def test_simulator_bit_exact():
    rng = np.random.default_rng(11)
    for _ in range(200):
        p = int(rng.integers(1, 9))
        C_ = p + int(rng.integers(0, 30000))
        r = rng.random(p) + 0.05
        b = O.partition_from_ratios(C_, (r / r.sum()).tolist())
        L = int(rng.integers(1, 40))
        cost = O.CostModel(float(rng.random()) * 1e-6 + 1e-9, float(rng.random()) * 1e-5, 1e-7, 1e-5)
        net = O.NetworkModel(float(rng.random()) * 1e8 + 1.0, float(rng.random()) * 1e-5)
        for s in ((O.KVR, O.TSP) if p > 1 else (O.KVR, O.SERIAL)):
            a = kv.simulate_ttft(kv.Strategy(s), kv.ContextPartition(C_, b), kv.ModelConfig(n_layers=L),
                                 kv.CostModel(**cost.__dict__), kv.NetworkModel(**net.__dict__))
            assert a == O.simulate_ttft(s, b, L, cost, net)
    with pytest.raises(kv.ConfigError):
        kv.simulate_ttft(kv.Strategy.KVR, kv.even_partition(64, 2), kv.ModelConfig(), kv.CostModel(alpha=0),
                         kv.NetworkModel())
    with pytest.raises(kv.InputError):
        kv.simulate_ttft(kv.Strategy.Serial, kv.even_partition(64, 2), kv.ModelConfig(), kv.CostModel(),
                         kv.NetworkModel())


@pytest.mark.parametrize("C_,p,L", [(16384, 2, 32), (16384, 4, 32), (4096, 3, 2), (1024, 4, 2), (96, 4, 2),
                                    (8192, 5, 32)])
def test_balancer_search_bit_exact(C_, p, L):
    got = kv.search_partition(C_, p, kv.ModelConfig(n_layers=L), kv.CostModel(), kv.NetworkModel())
    exp = O.hierarchical_grid_search(C_, p, sim=O.sim_ctx(L))
    assert (got.partition.boundaries, got.ttft, got.evaluations, got.levels) == tuple(exp)


def test_search_with_callback_evaluator_matches_oracle():
    def chain_cost(part):
        worst, held = 0.0, 0
        for c in part.sizes():
            held += c
            worst = max(worst, float(c) * float(held))
        return worst

    def chain_cost_b(b):
        return chain_cost(kv.ContextPartition(b[-1], list(b)))

    for C_, p in ((96, 4), (130, 3), (300, 2)):
        g = kv.hierarchical_grid_search(C_, p, kv.SearchConfig(evaluator=chain_cost))
        o = O.hierarchical_grid_search(C_, p, chain_cost_b)
        assert (g.partition.boundaries, g.ttft, g.evaluations, g.levels) == tuple(o)
    for C_ in (16, 48, 96, 130):
        g = kv.binary_search_two(C_, kv.SearchConfig(evaluator=chain_cost))
        o = O.binary_search_two(C_, chain_cost_b)
        assert (g.partition.boundaries, g.ttft, g.evaluations, g.levels) == tuple(o)
    cfg = kv.SearchConfig(evaluator=chain_cost, min_stride=2)
    assert cfg.resolve_initial_stride(96, 4) == 8
    assert kv.hierarchical_grid_search(96, 4, cfg).levels == 3
    with pytest.raises(kv.SearchError):
        kv.hierarchical_grid_search(32, 2, kv.SearchConfig())
    with pytest.raises(kv.SearchError):
        kv.hierarchical_grid_search(32, 2, kv.SearchConfig(grid_width=2, evaluator=chain_cost))


def test_bounds_and_calibration():
    for C_ in (512, 4096, 16384):
        assert kv.ttft_star(C_, 1, 3e-7) == O.ttft_star(C_, 1, 3e-7) == 3e-7 * C_ * C_
        assert kv.ttft_star(C_, 2, 3e-7) == 0.375 * 3e-7 * C_ * C_
    with pytest.raises(kv.InputError):
        kv.ttft_star(64, 0, 1e-6)
    for p in (1, 2, 4):
        part, t = kv.practical_bound(4096, p, kv.ModelConfig(n_layers=2), kv.CostModel())
        ob, ot = O.practical_bound(4096, p, 2)
        assert part.boundaries == ob and t == ot
    a = 2.5e-6
    assert abs(kv.calibrate_alpha([(c, a * c * c) for c in (256, 512, 1024, 2048)]) / a - 1) < 1e-12
    with pytest.raises(kv.CalibrationError):
        kv.calibrate_alpha([])


def test_fit_cost_model_recovers_generator():
    true = kv.CostModel(alpha=3e-9, proj_coeff=2e-6, softmax_coeff=5e-7, fixed_overhead=4e-5)
    rows, held, proj, rest = [], [], [], []
    for c, h in ((512, 512), (512, 2048), (1024, 4096), (2048, 2048), (256, 8192), (4096, 16384)):
        rows.append(c)
        held.append(h)
        proj.append(true.proj_coeff * c)
        rest.append(true.alpha * c * h + true.softmax_coeff * c + true.fixed_overhead)
    fit = kv.fit_cost_model(rows, held, proj, rest)
    for k in ("alpha", "proj_coeff", "softmax_coeff", "fixed_overhead"):
        assert abs(getattr(fit, k) / getattr(true, k) - 1) < 1e-6, k
    with pytest.raises(kv.CalibrationError):
        kv.fit_cost_model([], [], [], [])


# ---------------------------------------------------------------- SURVEY 8f next rows
def test_noise_study_semantics():  # test_simnet.cpp:128-184
    part = kv.even_partition(1024, 4)
    m = kv.ModelConfig(n_layers=2)
    quiet = kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 1.0, 8, 42)
    assert quiet.mean_degradation == 0.0 and quiet.max_degradation == 0.0 and all(d == 0.0 for d in quiet.per_trial)
    a = kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 16.0, 12, 9)
    b = kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 16.0, 12, 9)
    assert a.per_trial == b.per_trial
    harsh = kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 256.0, 12, 9)
    assert harsh.mean_degradation >= a.mean_degradation and harsh.max_degradation >= a.max_degradation
    tsp = kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 256.0, 12, 7)
    kvr = kv.noise_study(kv.Strategy.KVR, part, m, kv.CostModel(), kv.NetworkModel(), 256.0, 12, 7)
    assert tsp.mean_degradation > kvr.mean_degradation
    with pytest.raises(kv.InputError):
        kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 16.0, 0, 9)
    with pytest.raises(kv.ConfigError):
        kv.noise_study(kv.Strategy.TSP, part, m, kv.CostModel(), kv.NetworkModel(), 0.5, 4, 9)


def test_acceptance_criterion7_noise():  # acceptance.cpp:290-313
    even = kv.even_partition(2048, 4)
    m = kv.ModelConfig(n_layers=2)
    factor = 4.0
    while factor <= 1048576.0:
        tsp = kv.noise_study(kv.Strategy.TSP, even, m, kv.CostModel(), kv.NetworkModel(), factor, 20, 2026)
        if tsp.mean_degradation >= 0.08:
            kvr = kv.noise_study(kv.Strategy.KVR, even, m, kv.CostModel(), kv.NetworkModel(), factor, 20, 2026)
            assert kvr.mean_degradation < tsp.mean_degradation
            return
        factor *= 2.0
    raise AssertionError("gather never reached 8% mean degradation")


def test_lookup_table_interpolation_and_io(tmp_path):  # test_table_io.cpp:38-112
    t = kv.PartitionLookupTable(2)
    t.insert(1000, [0.6, 0.4])
    t.insert(3000, [0.7, 0.3])
    assert kv.interpolate_partition(t, 1000) == [0.6, 0.4]
    mid = kv.interpolate_partition(t, 2000)
    assert abs(mid[0] - 0.65) < 1e-12 and abs(sum(mid) - 1) < 1e-15
    assert kv.interpolate_partition(t, 10) == [0.6, 0.4]      # clamp below
    assert kv.interpolate_partition(t, 9000) == [0.7, 0.3]    # clamp above
    assert kv.partition_from_table(t, 2000).sizes() == [1300, 700]
    with pytest.raises(kv.LookupError_):
        kv.interpolate_partition(kv.PartitionLookupTable(2), 10)
    with pytest.raises(kv.LookupError_):
        t.insert(5, [0.5, 0.4])
    path = str(tmp_path / "table.json")
    t.save(path)
    again = kv.PartitionLookupTable.load(path)
    assert again.entries == t.entries and again.process_count == 2
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(kv.LookupError_):
        kv.PartitionLookupTable.load(str(tmp_path / "bad.json"))
    with pytest.raises(kv.IoError):
        kv.PartitionLookupTable.load(str(tmp_path / "missing.json"))


def test_acceptance_criterion6_table_vs_fresh_search():  # acceptance.cpp:251-286
    m = kv.ModelConfig(n_layers=2)
    t = kv.PartitionLookupTable(4)
    for C_ in (512, 2560, 4608, 6656):
        found = kv.search_partition(C_, 4, m, kv.CostModel(), kv.NetworkModel())
        t.insert(C_, [c / C_ for c in found.partition.sizes()])
    for C_ in (1536, 3584, 5632):
        pred = kv.simulate_ttft(kv.Strategy.KVR, kv.partition_from_table(t, C_), m, kv.CostModel(), kv.NetworkModel())
        fresh = kv.search_partition(C_, 4, m, kv.CostModel(), kv.NetworkModel())
        assert (pred - fresh.ttft) / fresh.ttft <= 0.05


@pytest.mark.skipif(not O.Reference.available(), reason="oracle/_ref not built")
def test_noise_and_table_bit_exact_vs_reference():
    ref = O.Reference()
    rng = np.random.default_rng(17)
    for _ in range(30):
        p = int(rng.integers(2, 7))
        C_ = p * 8 + int(rng.integers(0, 5000))
        b = kv.even_partition(C_, p)
        for s in (kv.Strategy.KVR, kv.Strategy.TSP):
            factor = float(2.0 ** rng.integers(0, 12))
            got = kv.noise_study(s, b, kv.ModelConfig(n_layers=3), kv.CostModel(), kv.NetworkModel(), factor, 7, 11)
            exp = ref.noise_study(int(s), b.boundaries, 3, factor, 7, 11)
            assert (got.quiet_ttft, got.mean_degradation, got.max_degradation, got.per_trial) == exp
        entries = {}
        for _k in range(int(rng.integers(1, 5))):
            r = rng.random(p) + 0.01
            entries[int(rng.integers(1, 20000))] = (r / r.sum()).tolist()
        t = kv.PartitionLookupTable(p)
        for k, v in entries.items():
            t.insert(k, v)
        q = int(rng.integers(p, 25000))
        r_ref, b_ref = ref.table(entries, p, q)
        assert kv.interpolate_partition(t, q) == r_ref
        assert kv.partition_from_table(t, q).boundaries == b_ref


def test_causal_cost_model_extension():
    """Extension (not in the reference): attention priced on causal-visible pairs."""
    m = kv.ModelConfig(64, 4, 4, 2, 1, "f32", True)
    cost = kv.CostModel(alpha=1e-6, proj_coeff=0.0, softmax_coeff=0.0, fixed_overhead=0.0)
    net = kv.NetworkModel(bandwidth=1e30, latency=0.0)
    one = kv.even_partition(1000, 1)
    dense = kv.simulate_ttft(kv.Strategy.KVR, one, m, cost, net)
    causal = kv.simulate_ttft_causal(kv.Strategy.KVR, one, m, cost, net)
    assert abs(dense - 2 * 1e-6 * 1000 * 1000) < 1e-12
    assert abs(causal - 2 * 1e-6 * 1000 * 500.5) < 1e-12
    even = kv.even_partition(8192, 4)
    for s in (kv.Strategy.KVR, kv.Strategy.TSP):
        assert kv.simulate_ttft_causal(s, even, m, cost, net) < kv.simulate_ttft(s, even, m, cost, net)
    found = kv.search_partition_causal(8192, 4, m, cost, net)
    sizes = found.partition.sizes()
    assert sum(sizes) == 8192
    assert all(sizes[i] >= sizes[i + 1] for i in range(3))
    assert found.ttft <= kv.simulate_ttft_causal(kv.Strategy.KVR, even, m, cost, net)


def test_noise_sidecar_link_draw():  # simnet.hpp:65-78, 342-344; rng.hpp:10-37
    """The physical sidecar (bench.py --noise-factor) slows exactly the links the reference's
    NoiseSidecar draws: restated here from rng.hpp's SplitMix64 / mix_seed."""
    M = (1 << 64) - 1

    def nxt(state):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return state, z ^ (z >> 31)

    def mix_seed(base, a, b=0):
        _, s = nxt(base)
        s ^= (a * 0xD1342543DE82EF95) & M
        _, h = nxt(s)
        return h ^ ((b * 0xAF251AF3B0F025B5) & M)

    for study_seed in (1, 7, 2**63 + 5):
        for t in range(4):
            sc = kv.NoiseSidecar.for_trial(study_seed, t, 2.0)
            assert sc.seed == mix_seed(study_seed, 0x7472, t) and sc.slowdown_factor == 2.0
            for links in (1, 3, 7):
                for layer in range(6):
                    _, r = nxt(mix_seed(sc.seed, 0x6E6F, layer))
                    assert sc.degraded_link(layer, links) == r % links
    assert kv.NoiseSidecar(3, 2.0).degraded_link(0, 0) == -1
