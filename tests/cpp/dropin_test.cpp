// Drop-in check: reference-style client code (the shapes of test_engine.cpp / acceptance.cpp)
// compiled against the drop-in with the reference's own include line (include/kvprefill/ forwards
// to include/kvprefill_b200/kvprefill.hpp) and linked to libkvp_b200.so.
// Exit 0 = all checks passed; prints one line per check.
#include <cstdio>
#include <string>

#include "kvprefill/kvprefill.hpp"

using namespace kvprefill;

static int failures = 0;
static void expect(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::string(argv[1]) == "--gpu";
    // host-only parts of the API (no device needed)
    expect(even_partition(10, 4).sizes() == std::vector<int64_t>({3, 3, 2, 2}), "even_partition(10,4)");
    expect(partition_from_ratios(10240, {0.35, 0.255, 0.21, 0.185}).sizes() ==
               std::vector<int64_t>({3584, 2611, 2150, 1895}),
           "partition_from_ratios golden");
    bool threw = false;
    try {
        even_partition(3, 4);
    } catch (const PartitionError&) {
        threw = true;
    }
    expect(threw, "PartitionError type preserved across the C-ABI");
    expect(traffic_pairs(Strategy::KVR, ContextPartition::from_sizes({4, 3, 2})) == 11, "traffic_pairs KVR fixture");
    ModelConfig sim;
    sim.n_layers = 32;
    const auto found = search_partition(16384, 4, sim, CostModel{}, NetworkModel{});
    expect(found.partition.boundaries == std::vector<int64_t>({0, 6564, 10621, 13754, 16384}), "KVR-S search p=4 16k");
    // kv_cache.hpp: segment validation and coverage (host types)
    KVCacheSegment<float> s0{0, 0, 4, Matrix<float>(4, 8), Matrix<float>(4, 8)};
    KVCacheSegment<float> s1{0, 4, 9, Matrix<float>(5, 8), Matrix<float>(5, 8)};
    bool covered = true;
    try {
        validate_cache_coverage<float>({s0, s1}, 9);
    } catch (const Error&) {
        covered = false;
    }
    bool gap = false;
    try {
        validate_cache_coverage<float>({s1}, 9);
    } catch (const CacheError&) {
        gap = true;
    }
    expect(covered && gap, "validate_cache_coverage: gap-free accepted, gap -> CacheError");
    // weights.hpp random_context: the reference's SplitMix64 prompt, host side
    std::vector<float> via_abi(1024 * 32);
    detail::check(kvp_random_context(1024, 32, 18, via_abi.data()), "random_context");
    expect(random_context<float>(1024, 32, 18).values == via_abi, "random_context header == C-ABI");
    if (!gpu) return failures ? 1 : 0;

    // device parts: the reference's accounting fixture and bitwise strategy equivalence
    ModelConfig mc;
    mc.d_model = 8;
    mc.n_heads = 2;
    mc.n_kv_heads = 2;
    mc.n_layers = 2;
    mc.seed = 3;
    mc.precision = Precision::f32;
    const auto w = init_weights<float>(mc);
    const auto ctx = random_context<float>(9, mc.d_model, 21);
    const auto kvr = run(Strategy::KVR, ctx, ContextPartition::from_sizes({4, 3, 2}), w);
    expect(kvr.metrics.per_layer_dot_products(0) == 16 && kvr.metrics.per_layer_dot_products(1) == 21 &&
               kvr.metrics.per_layer_dot_products(2) == 18,
           "KVR dots 16/21/18");
    expect(kvr.metrics.per_layer_pairs_sent() == 11 && kvr.metrics.per_layer_rows_sent() == 22 &&
               kvr.metrics.barrier_count == 0,
           "KVR 11 pairs / 22 rows / 0 barriers");
    const auto tsp = run(Strategy::TSP, ctx, even_partition(9, 3), w);
    expect(tsp.metrics.per_layer_pairs_sent() == 18 && tsp.metrics.barrier_count == mc.n_layers,
           "TSP 18 pairs / L barriers");
    const auto serial = run(Strategy::Serial, ctx, even_partition(9, 1), w);
    expect(serial.hidden_out == kvr.hidden_out && serial.hidden_out == tsp.hidden_out, "Serial == KVR == TSP bitwise");
    // forward_serial (model.hpp:197-211): hidden states + one [0, C) segment per layer
    const auto fs = forward_serial(ctx, w);
    expect(fs.first == serial.hidden_out && fs.second.size() == 2, "forward_serial hidden == run(Serial)");
    bool segs_ok = true;
    for (const auto& seg : fs.second) {
        try {
            validate_cache_coverage<float>({seg}, 9);
        } catch (const Error&) {
            segs_ok = false;
        }
    }
    const auto qkv0 = layer_qkv(ctx, w, 0);
    expect(segs_ok && fs.second[0].K == qkv0.K && fs.second[0].V == qkv0.V,
           "forward_serial segments cover [0, C); layer 0 K/V == layer_qkv (f32, bitwise)");
    bool narrow = false;
    try {
        run(Strategy::Serial, Matrix<float>(9, 4), even_partition(9, 1), w);
    } catch (const DimensionError&) {
        narrow = true;
    }
    expect(narrow, "context width != d_model -> DimensionError");
    bool proto = false;
    try {
        FaultInjection f;
        f.kind = FaultInjection::Kind::DropMessage;
        run(Strategy::KVR, ctx, even_partition(9, 3), w, f);
    } catch (const ProtocolError&) {
        proto = true;
    }
    expect(proto, "dropped handoff -> ProtocolError");
    mc.precision = Precision::bf16;
    mc.d_model = 1024;
    mc.n_heads = 8;
    mc.n_kv_heads = 8;
    mc.rms_norm = true;
    const auto wb = init_weights<float>(mc);
    const auto big = random_context<float>(512, mc.d_model, 18);
    const auto a = run(Strategy::KVR, big, partition_from_ratios(512, {0.4, 0.3, 0.2, 0.1}), wb);
    const auto b = run(Strategy::Serial, big, even_partition(512, 1), wb);
    expect(a.hidden_out == b.hidden_out, "bf16 tcgen05 path: KVR(p=4) == Serial bitwise");
    // decode on the prefilled cache (f32 parity mode): rows 9.. equal a longer serial run
    const auto ctx12 = random_context<float>(12, 8, 21);
    Matrix<float> head(9, 8), tail(3, 8);
    std::copy(ctx12.values.begin(), ctx12.values.begin() + 72, head.values.begin());
    std::copy(ctx12.values.begin() + 72, ctx12.values.end(), tail.values.begin());
    KVCache<float> cache(w, 12);
    cache.prefill(head);
    const auto dec = cache.decode(tail);
    const auto longer = run(Strategy::Serial, ctx12, even_partition(12, 1), w);
    expect(std::equal(dec.values.begin(), dec.values.end(), longer.hidden_out.values.begin() + 72) &&
               cache.length() == 12,
           "KVCache decode == serial forward over the longer context (f32, bitwise)");
    return failures ? 1 : 0;
}
