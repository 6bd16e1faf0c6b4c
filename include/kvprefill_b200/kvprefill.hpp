// kvprefill_b200/kvprefill.hpp -- C++ drop-in for the reference's kvprefill hot path.
//
// A program written against the reference (/root/reference/proj/include/kvprefill/
// kvprefill.hpp) switches to the B200 path by including this header instead and linking
// libkvp_b200.so.  Same namespace (kvprefill), same type and function names, same argument
// meaning and the same exception classes (errors.hpp:8-46); every computation goes through
// the C-ABI in kvp_b200.h to the sm_100a kernels.  Differences, all additive:
//   * Precision gains bf16 (bf16 operands, f32 accumulation); f64 raises ConfigError (no GPU
//     path) -- keep the reference itself for f64 oracles;
//   * WeightSet<T> owns the device-resident weights + engine; init_weights<T>(cfg, devices)
//     takes an optional device list (rank r runs on devices[r % n]);
//   * KVR-S balancing from measured times: fit_cost_model + search_partition.
// The KVR-P lookup table and the noise study are here too (lookup_table.hpp, simnet.hpp);
// their JSON file I/O is in table_io.hpp (needs nlohmann/json); the commands.hpp CLI is the
// separate tool tools/kvprefill_b200_main.cpp.
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <type_traits>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../kvp_b200.h"

namespace kvprefill {

// ---------------------------------------------------------------- errors.hpp
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error { using Error::Error; };
struct DimensionError : Error { using Error::Error; };
struct CacheError : Error { using Error::Error; };
struct InputError : Error { using Error::Error; };
struct PartitionError : Error { using Error::Error; };
struct ProtocolError : Error { using Error::Error; };
struct AssemblyError : Error { using Error::Error; };
struct LookupError : Error { using Error::Error; };
struct SearchError : Error { using Error::Error; };
struct BudgetError : Error { using Error::Error; };
struct CalibrationError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / NCCL failure (no reference twin)

namespace detail {
[[noreturn]] inline void raise(kvp_status s, const char* where) {
    const std::string msg = std::string(where) + ": " + kvp_last_error();
    switch (s) {
        case KVP_ERR_CONFIG: throw ConfigError(msg);
        case KVP_ERR_DIMENSION: throw DimensionError(msg);
        case KVP_ERR_CACHE: throw CacheError(msg);
        case KVP_ERR_INPUT: throw InputError(msg);
        case KVP_ERR_PARTITION: throw PartitionError(msg);
        case KVP_ERR_PROTOCOL: throw ProtocolError(msg);
        case KVP_ERR_ASSEMBLY: throw AssemblyError(msg);
        case KVP_ERR_LOOKUP: throw LookupError(msg);
        case KVP_ERR_SEARCH: throw SearchError(msg);
        case KVP_ERR_BUDGET: throw BudgetError(msg);
        case KVP_ERR_CALIBRATION: throw CalibrationError(msg);
        case KVP_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}
inline void check(kvp_status s, const char* where) {
    if (s != KVP_OK) raise(s, where);
}
}  // namespace detail

// ---------------------------------------------------------------- rng.hpp (host seeding)
class SplitMix64 {
  public:
    explicit SplitMix64(uint64_t seed) : s_(seed) {}
    uint64_t next() {
        uint64_t z = (s_ += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double next_symmetric() { return 2.0 * next_unit() - 1.0; }

  private:
    uint64_t s_;
};

inline uint64_t mix_seed(uint64_t base, uint64_t a, uint64_t b = 0) {
    SplitMix64 g(base);
    SplitMix64 h(g.next() ^ (a * 0xd1342543de82ef95ULL));
    return h.next() ^ (b * 0xaf251af3b0f025b5ULL);
}

// ---------------------------------------------------------------- matrix.hpp (host values)
template <typename T>
struct Matrix {
    int64_t rows = 0, cols = 0;
    std::vector<T> values;
    Matrix() = default;
    Matrix(int64_t r, int64_t c) : rows(r), cols(c), values(static_cast<size_t>(r * c), T(0)) {
        if (r < 0 || c < 0) throw DimensionError("matrix dimensions must be non-negative");
    }
    T& at(int64_t r, int64_t c) { return values[static_cast<size_t>(r * cols + c)]; }
    const T& at(int64_t r, int64_t c) const { return values[static_cast<size_t>(r * cols + c)]; }
    std::span<const T> row(int64_t r) const { return {values.data() + r * cols, static_cast<size_t>(cols)}; }
    bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }
    Matrix slice_rows(int64_t b, int64_t e) const {
        if (b < 0 || e > rows || b > e) throw DimensionError("row slice out of range");
        Matrix out(e - b, cols);
        std::memcpy(out.values.data(), values.data() + b * cols, static_cast<size_t>((e - b) * cols) * sizeof(T));
        return out;
    }
    bool operator==(const Matrix& o) const { return rows == o.rows && cols == o.cols && values == o.values; }
};
using MatrixF = Matrix<float>;

template <typename A, typename B>
double max_rel_dev(const Matrix<A>& a, const Matrix<B>& b) {
    if (!(a.rows == b.rows && a.cols == b.cols)) throw DimensionError("deviation requires equal shapes");
    double worst = 0.0;
    for (size_t i = 0; i < a.values.size(); ++i) {
        const double r = static_cast<double>(b.values[i]);
        worst = std::max(worst, std::abs(static_cast<double>(a.values[i]) - r) / std::max(1.0, std::abs(r)));
    }
    return worst;
}

// ---------------------------------------------------------------- config.hpp
enum class Precision { f32 = KVP_F32, f64 = KVP_F64, bf16 = KVP_BF16 };

struct ModelConfig {
    int64_t d_model = 32, n_heads = 4, n_kv_heads = 4, n_layers = 2;
    uint64_t seed = 1;
    Precision precision = Precision::f64;
    bool rms_norm = false;
    int64_t head_dim() const { return d_model / n_heads; }
    int64_t q_dim() const { return n_heads * head_dim(); }
    int64_t kv_dim() const { return n_kv_heads * head_dim(); }
    int64_t ffn_dim() const { return 2 * d_model; }
    void validate() const {
        if (d_model <= 0 || n_heads <= 0 || n_kv_heads <= 0 || n_layers <= 0)
            throw ConfigError("model dimensions must be positive");
        if (d_model % n_heads != 0) throw ConfigError("d_model must be divisible by n_heads");
        if (n_heads % n_kv_heads != 0) throw ConfigError("n_heads must be divisible by n_kv_heads");
    }
    kvp_model_config c() const {
        return kvp_model_config{d_model, n_heads, n_kv_heads, n_layers, seed, static_cast<int32_t>(precision),
                                rms_norm ? 1 : 0};
    }
};

// ---------------------------------------------------------------- partition.hpp
struct ContextPartition {
    int64_t context_length = 0;
    std::vector<int64_t> boundaries;
    int64_t process_count() const { return static_cast<int64_t>(boundaries.size()) - 1; }
    std::vector<int64_t> sizes() const {
        std::vector<int64_t> s;
        for (size_t i = 0; i + 1 < boundaries.size(); ++i) s.push_back(boundaries[i + 1] - boundaries[i]);
        return s;
    }
    void validate() const {
        if (boundaries.size() < 2) throw PartitionError("boundaries must run from 0 to the context length");
        detail::check(kvp_validate_partition(context_length, boundaries.data(), process_count()), "validate");
    }
    static ContextPartition from_sizes(const std::vector<int64_t>& sizes) {
        ContextPartition p;
        p.boundaries.push_back(0);
        for (int64_t c : sizes) p.boundaries.push_back(p.boundaries.back() + c);
        p.context_length = p.boundaries.back();
        p.validate();
        return p;
    }
    bool operator==(const ContextPartition& o) const {
        return context_length == o.context_length && boundaries == o.boundaries;
    }
};

inline ContextPartition even_partition(int64_t C, int64_t p) {
    ContextPartition out;
    out.context_length = C;
    out.boundaries.assign(static_cast<size_t>(std::max<int64_t>(p, 1) + 1), 0);
    detail::check(kvp_even_partition(C, p, out.boundaries.data()), "even_partition");
    return out;
}

inline ContextPartition partition_from_ratios(int64_t C, const std::vector<double>& ratios) {
    ContextPartition out;
    out.context_length = C;
    out.boundaries.assign(ratios.size() + 1, 0);
    detail::check(kvp_partition_from_ratios(C, ratios.data(), static_cast<int64_t>(ratios.size()),
                                            out.boundaries.data()),
                  "partition_from_ratios");
    return out;
}

// ---------------------------------------------------------------- search.hpp
using TtftEvaluator = std::function<double(const ContextPartition&)>;

struct SearchConfig {
    int64_t grid_width = 5, initial_stride = 0, min_stride = 1;
    TtftEvaluator evaluator;
};

struct SearchResult {
    ContextPartition partition;
    double ttft = 0.0;
    int64_t evaluations = 0, levels = 0;
};

namespace detail {
struct EvalCtx {
    int64_t C;
    const TtftEvaluator* fn;
};
inline double trampoline(const int64_t* b, int64_t p, void* u) {
    auto* c = static_cast<EvalCtx*>(u);
    ContextPartition part;
    part.context_length = c->C;
    part.boundaries.assign(b, b + p + 1);
    return (*c->fn)(part);
}
}  // namespace detail

inline SearchResult hierarchical_grid_search(int64_t C, int64_t p, const SearchConfig& cfg) {
    SearchResult r;
    r.partition.context_length = C;
    r.partition.boundaries.assign(static_cast<size_t>(std::max<int64_t>(p, 1) + 1), 0);
    kvp_search_config sc{cfg.grid_width, cfg.initial_stride, cfg.min_stride};
    detail::EvalCtx ctx{C, &cfg.evaluator};
    kvp_search_result res{};
    detail::check(kvp_hierarchical_grid_search(C, p, &sc, cfg.evaluator ? detail::trampoline : nullptr, &ctx,
                                               r.partition.boundaries.data(), &res),
                  "hierarchical_grid_search");
    r.ttft = res.ttft;
    r.evaluations = res.evaluations;
    r.levels = res.levels;
    return r;
}

inline SearchResult binary_search_two(int64_t C, const SearchConfig& cfg) {
    SearchResult r;
    r.partition.context_length = C;
    r.partition.boundaries.assign(3, 0);
    kvp_search_config sc{cfg.grid_width, cfg.initial_stride, cfg.min_stride};
    detail::EvalCtx ctx{C, &cfg.evaluator};
    kvp_search_result res{};
    detail::check(kvp_binary_search_two(C, &sc, cfg.evaluator ? detail::trampoline : nullptr, &ctx,
                                        r.partition.boundaries.data(), &res),
                  "binary_search_two");
    r.ttft = res.ttft;
    r.evaluations = res.evaluations;
    r.levels = res.levels;
    return r;
}

// ---------------------------------------------------------------- weights.hpp
template <typename T>
class WeightSet {
  public:
    ModelConfig config;
    WeightSet() = default;
    WeightSet(const ModelConfig& c, const std::vector<int32_t>& devices) : config(c) {
        c.validate();
        const kvp_model_config kc = c.c();
        kvp_engine* e = nullptr;
        detail::check(kvp_engine_create(&kc, devices.data(), static_cast<int32_t>(devices.size()), &e), "init_weights");
        engine_.reset(e, [](kvp_engine* x) { kvp_engine_destroy(x); });
    }
    kvp_engine* engine() const { return engine_.get(); }
    // Opt-in rotary position embedding (extension, bf16 only; kvp_engine_set_rope).
    void set_rope(double theta) const { detail::check(kvp_engine_set_rope(engine_.get(), theta), "set_rope"); }

  private:
    std::shared_ptr<kvp_engine> engine_;
};

// init_weights<T> (weights.hpp:54-83): generated on the device(s), bit-identical values.
// T is the host element type of contexts/outputs (float); the device precision is
// config.precision (f32 parity mode or bf16).
template <typename T = float>
WeightSet<T> init_weights(const ModelConfig& config, const std::vector<int32_t>& devices = {0}) {
    static_assert(std::is_same_v<T, float>, "the B200 path exchanges float host matrices");
    return WeightSet<T>(config, devices);
}

// random_context<T> (weights.hpp:86-89), host side.
template <typename T = float>
Matrix<T> random_context(int64_t rows, int64_t d_model, uint64_t seed) {
    Matrix<T> m(rows, d_model);
    SplitMix64 g(mix_seed(seed, 0xc7u, 17));
    for (auto& v : m.values) v = static_cast<T>(g.next_symmetric() * 1.0);
    return m;
}

// ---------------------------------------------------------------- kv_cache.hpp / model.hpp
// KVCacheSegment (kv_cache.hpp:14-31): K and V rows of one layer for token positions
// [start_pos, end_pos); host copies of the device cache rows.
template <typename T>
struct KVCacheSegment {
    int64_t layer = 0;
    int64_t start_pos = 0;  // inclusive
    int64_t end_pos = 0;    // exclusive
    Matrix<T> K;
    Matrix<T> V;

    int64_t token_rows() const { return end_pos - start_pos; }

    void validate() const {
        if (start_pos < 0 || start_pos >= end_pos) throw CacheError("segment positions must satisfy 0 <= start < end");
        if (K.rows != token_rows() || !K.same_shape(V))
            throw CacheError("segment K/V rows must match the covered token range");
    }
};

struct CausalMask {
    int64_t offset = 0, rows = 0;
};

// validate_cache_coverage (kv_cache.hpp:41-55): segments of one layer, gap-free from 0,
// jointly covering [0, expected_tokens).
template <typename T>
void validate_cache_coverage(const std::vector<KVCacheSegment<T>>& segments, int64_t expected_tokens) {
    int64_t next = 0;
    for (const auto& seg : segments) {
        seg.validate();
        if (seg.start_pos != next)
            throw CacheError("cache gap: expected segment at position " + std::to_string(next) + ", got " +
                             std::to_string(seg.start_pos));
        next = seg.end_pos;
    }
    if (next != expected_tokens)
        throw CacheError("cache covers " + std::to_string(next) + " tokens, expected " +
                         std::to_string(expected_tokens));
}

template <typename T>
struct LayerQKV {
    Matrix<T> Q, K, V;
};

template <typename T>
LayerQKV<T> layer_qkv(const Matrix<T>& hidden, const WeightSet<T>& w, int64_t layer) {
    const ModelConfig& c = w.config;
    if (hidden.cols != c.d_model) throw DimensionError("qkv_project: hidden width != d_model");
    LayerQKV<T> out{Matrix<T>(hidden.rows, c.q_dim()), Matrix<T>(hidden.rows, c.kv_dim()),
                    Matrix<T>(hidden.rows, c.kv_dim())};
    detail::check(kvp_layer_qkv(w.engine(), layer, hidden.values.data(), hidden.rows, out.Q.values.data(),
                                out.K.values.data(), out.V.values.data()),
                  "layer_qkv");
    return out;
}

template <typename T>
Matrix<T> causal_attention(const Matrix<T>& Q, const Matrix<T>& K, const Matrix<T>& V, const CausalMask& mask,
                           const WeightSet<T>& w) {
    if (K.rows != V.rows || !K.same_shape(V)) throw DimensionError("causal_attention: K/V shape mismatch");
    if (Q.rows != mask.rows) throw DimensionError("causal_attention: Q rows != mask rows");
    if (K.rows < mask.offset + Q.rows)
        throw CacheError("causal_attention: cache holds " + std::to_string(K.rows) + " rows, need at least " +
                         std::to_string(mask.offset + Q.rows));
    // the reference indexes Q/K/V by head offsets (model.hpp:139-154); the C-ABI reads exactly
    // q_dim / kv_dim columns per row, so narrower matrices are rejected here
    if (Q.cols != w.config.q_dim() || K.cols != w.config.kv_dim())
        throw DimensionError("causal_attention: Q/K/V widths " + std::to_string(Q.cols) + "/" + std::to_string(K.cols) +
                             " != q_dim/kv_dim " + std::to_string(w.config.q_dim()) + "/" +
                             std::to_string(w.config.kv_dim()));
    Matrix<T> A(Q.rows, w.config.q_dim());
    detail::check(kvp_causal_attention(w.engine(), Q.values.data(), Q.rows, K.values.data(), V.values.data(), K.rows,
                                       mask.offset, A.values.data()),
                  "causal_attention");
    return A;
}

template <typename T>
Matrix<T> layer_finish(const Matrix<T>& hidden, const Matrix<T>& Q, const Matrix<T>& K_full, const Matrix<T>& V_full,
                       int64_t offset, const WeightSet<T>& w, int64_t layer) {
    const ModelConfig& c = w.config;
    if (!K_full.same_shape(V_full)) throw DimensionError("causal_attention: K/V shape mismatch");
    if (Q.rows != hidden.rows) throw DimensionError("causal_attention: Q rows != mask rows");
    if (K_full.rows < offset + Q.rows)
        throw CacheError("causal_attention: cache holds " + std::to_string(K_full.rows) + " rows, need at least " +
                         std::to_string(offset + Q.rows));
    if (hidden.cols != c.d_model) throw DimensionError("add shape mismatch");
    if (Q.cols != c.q_dim() || K_full.cols != c.kv_dim())
        throw DimensionError("causal_attention: Q/K/V widths " + std::to_string(Q.cols) + "/" +
                             std::to_string(K_full.cols) + " != q_dim/kv_dim " + std::to_string(c.q_dim()) + "/" +
                             std::to_string(c.kv_dim()));
    Matrix<T> out(hidden.rows, w.config.d_model);
    detail::check(kvp_layer_finish(w.engine(), layer, hidden.values.data(), hidden.rows, Q.values.data(),
                                   K_full.values.data(), V_full.values.data(), K_full.rows, offset, out.values.data()),
                  "layer_finish");
    return out;
}

// ---------------------------------------------------------------- engine.hpp
enum class Strategy { Serial = KVP_SERIAL, TSP = KVP_TSP, KVR = KVP_KVR };

struct FaultInjection {
    enum class Kind { None = 0, CorruptLayerTag, DropMessage, DuplicateMessage };
    Kind kind = Kind::None;
    int64_t rank = 0, layer = 0;
};

struct ExecutionMetrics {
    int64_t n_layers = 1, barrier_count = 0;
    std::vector<int64_t> dot_products, kv_pairs_sent, kv_pairs_received, wait_events;
    int64_t per_layer_dot_products(int64_t r) const { return dot_products[static_cast<size_t>(r)] / n_layers; }
    int64_t per_layer_pairs_received(int64_t r) const { return kv_pairs_received[static_cast<size_t>(r)] / n_layers; }
    int64_t total_pairs_sent() const {
        int64_t t = 0;
        for (int64_t v : kv_pairs_sent) t += v;
        return t;
    }
    int64_t per_layer_pairs_sent() const { return total_pairs_sent() / n_layers; }
    int64_t total_rows_sent() const { return 2 * total_pairs_sent(); }
    int64_t per_layer_rows_sent() const { return 2 * per_layer_pairs_sent(); }
};

template <typename T>
struct ExecutionResult {
    Matrix<T> hidden_out;
    Matrix<T> first_token_hidden;
    ExecutionMetrics metrics;
};

inline std::vector<int64_t> dot_product_counts(Strategy s, const ContextPartition& part) {
    std::vector<int64_t> out(static_cast<size_t>(std::max<int64_t>(part.process_count(), 1)));
    detail::check(kvp_dot_product_counts(static_cast<int32_t>(s), part.context_length, part.boundaries.data(),
                                         part.process_count(), out.data()),
                  "dot_product_counts");
    return out;
}

inline int64_t traffic_pairs(Strategy s, const ContextPartition& part) {
    int64_t out = 0;
    detail::check(kvp_traffic_pairs(static_cast<int32_t>(s), part.context_length, part.boundaries.data(),
                                    part.process_count(), &out),
                  "traffic_pairs");
    return out;
}

// run<T> (engine.hpp:186-318): p ranks, one host thread + CUDA streams each.
template <typename T>
ExecutionResult<T> run(Strategy strategy, const Matrix<T>& context, const ContextPartition& partition,
                       const WeightSet<T>& weights, const FaultInjection& fault = {}) {
    partition.validate();
    if (partition.context_length != context.rows)
        throw InputError("partition covers " + std::to_string(partition.context_length) +
                         " tokens but the context has " + std::to_string(context.rows) + " rows");
    const int64_t d = weights.config.d_model, C = context.rows, p = partition.process_count();
    if (context.cols != d)  // qkv_project (model.hpp:68-70)
        throw DimensionError("qkv_project: hidden width " + std::to_string(context.cols) + " != d_model " +
                             std::to_string(d));
    ExecutionResult<T> r;
    r.hidden_out = Matrix<T>(C, d);
    r.first_token_hidden = Matrix<T>(1, d);
    kvp_fault f{static_cast<int32_t>(fault.kind), fault.rank, fault.layer};
    kvp_metrics m{};
    detail::check(kvp_engine_run(weights.engine(), static_cast<int32_t>(strategy), context.values.data(), C,
                                 partition.boundaries.data(), p, &f, r.hidden_out.values.data(),
                                 r.first_token_hidden.values.data(), &m),
                  "run");
    r.metrics.n_layers = m.n_layers;
    r.metrics.barrier_count = m.barrier_count;
    r.metrics.dot_products.assign(m.dot_products, m.dot_products + p);
    r.metrics.kv_pairs_sent.assign(m.kv_pairs_sent, m.kv_pairs_sent + p);
    r.metrics.kv_pairs_received.assign(m.kv_pairs_received, m.kv_pairs_received + p);
    r.metrics.wait_events.assign(m.wait_events, m.wait_events + p);
    return r;
}

// forward_serial (model.hpp:197-211): final hidden states (row C-1 is the first-token readout)
// and one cache segment per layer covering [0, C), copied back from the device cache.
template <typename T>
std::pair<Matrix<T>, std::vector<KVCacheSegment<T>>> forward_serial(const Matrix<T>& context,
                                                                    const WeightSet<T>& weights) {
    if (context.rows < 1) throw InputError("forward_serial: empty context");
    const ModelConfig& c = weights.config;
    if (context.cols != c.d_model)
        throw DimensionError("qkv_project: hidden width " + std::to_string(context.cols) + " != d_model " +
                             std::to_string(c.d_model));
    const int64_t C = context.rows, kv = c.kv_dim();
    Matrix<T> h(C, c.d_model);
    std::vector<float> kvbuf(static_cast<size_t>(c.n_layers * 2 * C * kv));
    detail::check(kvp_forward_serial(weights.engine(), context.values.data(), C, h.values.data(), kvbuf.data()),
                  "forward_serial");
    std::vector<KVCacheSegment<T>> cache;
    cache.reserve(static_cast<size_t>(c.n_layers));
    for (int64_t l = 0; l < c.n_layers; ++l) {
        KVCacheSegment<T> seg{l, 0, C, Matrix<T>(C, kv), Matrix<T>(C, kv)};
        const float* k = kvbuf.data() + (2 * l) * C * kv;
        std::copy(k, k + C * kv, seg.K.values.begin());
        std::copy(k + C * kv, k + 2 * C * kv, seg.V.values.begin());
        cache.push_back(std::move(seg));
    }
    return {std::move(h), std::move(cache)};
}

// Hidden states only (no K/V copy back to the host).
template <typename T>
Matrix<T> forward_serial_hidden(const Matrix<T>& context, const WeightSet<T>& weights) {
    if (context.rows < 1) throw InputError("forward_serial: empty context");
    return run(Strategy::Serial, context, even_partition(context.rows, 1), weights).hidden_out;
}

// ---------------------------------------------------------------- simnet.hpp (balancer)
struct CostModel {
    double alpha = 1e-6, proj_coeff = 4e-6, softmax_coeff = 1e-7, fixed_overhead = 1e-5;
    kvp_cost_model c() const { return {alpha, proj_coeff, softmax_coeff, fixed_overhead}; }
    void validate() const {  // simnet.hpp:32-36
        if (!(alpha > 0)) throw ConfigError("cost.alpha must be positive");
        if (proj_coeff < 0 || softmax_coeff < 0 || fixed_overhead < 0)
            throw ConfigError("cost coefficients must be non-negative");
    }
};

struct NetworkModel {
    double bandwidth = 1e7, latency = 1e-6;
    static NetworkModel zero_comm() { return {std::numeric_limits<double>::infinity(), 0.0}; }
    kvp_network_model c() const { return {bandwidth, latency}; }
    void validate() const {  // simnet.hpp:51-54
        if (!(bandwidth > 0)) throw ConfigError("network.bandwidth must be positive");
        if (latency < 0) throw ConfigError("network.latency must be non-negative");
    }
};

inline double simulate_ttft_value(Strategy s, const ContextPartition& part, const ModelConfig& model,
                                  const CostModel& cost, const NetworkModel& net) {
    double out = 0;
    const kvp_cost_model cc = cost.c();
    const kvp_network_model nc = net.c();
    detail::check(kvp_simulate_ttft(static_cast<int32_t>(s), part.context_length, part.boundaries.data(),
                                    part.process_count(), model.n_layers, &cc, &nc, &out),
                  "simulate_ttft");
    return out;
}

inline double ttft_star(int64_t C, int64_t p, double alpha) {
    double out = 0;
    detail::check(kvp_ttft_star(C, p, alpha, &out), "ttft_star");
    return out;
}

// KVR-S: the context-level load balancer (grid search scored by the chain simulator).
inline SearchResult search_partition(int64_t C, int64_t p, const ModelConfig& model, const CostModel& cost,
                                     const NetworkModel& net, const SearchConfig& cfg = {}) {
    SearchResult r;
    r.partition.context_length = C;
    r.partition.boundaries.assign(static_cast<size_t>(p + 1), 0);
    const kvp_cost_model cc = cost.c();
    const kvp_network_model nc = net.c();
    kvp_search_config sc{cfg.grid_width, cfg.initial_stride, cfg.min_stride};
    kvp_search_result res{};
    detail::check(kvp_search_partition(C, p, model.n_layers, &cc, &nc, &sc, r.partition.boundaries.data(), &res),
                  "search_partition");
    r.ttft = res.ttft;
    r.evaluations = res.evaluations;
    r.levels = res.levels;
    return r;
}

// practical_bound / ttft_practical_lower (simnet.hpp:297-321).
struct PracticalBound {
    ContextPartition partition;
    double ttft = 0.0;
};

inline PracticalBound practical_bound(int64_t C, int64_t p, const ModelConfig& model, const CostModel& cost) {
    PracticalBound b;
    b.partition.context_length = C;
    b.partition.boundaries.assign(static_cast<size_t>(std::max<int64_t>(p, 1) + 1), 0);
    const kvp_cost_model cc = cost.c();
    detail::check(kvp_practical_bound(C, p, model.n_layers, &cc, b.partition.boundaries.data(), &b.ttft),
                  "practical_bound");
    return b;
}

inline double ttft_practical_lower(int64_t C, int64_t p, const ModelConfig& model, const CostModel& cost) {
    return practical_bound(C, p, model, cost).ttft;
}

// noise_study (simnet.hpp:323-353): seeded trials with one slowed link per layer.
struct NoiseStudy {
    double quiet_ttft = 0, mean_degradation = 0, max_degradation = 0;
    std::vector<double> per_trial;
};

inline NoiseStudy noise_study(Strategy s, const ContextPartition& part, const ModelConfig& model,
                              const CostModel& cost, const NetworkModel& net, double slowdown_factor,
                              int64_t trials, uint64_t seed) {
    NoiseStudy r;
    r.per_trial.assign(static_cast<size_t>(std::max<int64_t>(trials, 1)), 0.0);
    const kvp_cost_model cc = cost.c();
    const kvp_network_model nc = net.c();
    detail::check(kvp_noise_study(static_cast<int32_t>(s), part.context_length, part.boundaries.data(),
                                  part.process_count(), model.n_layers, &cc, &nc, slowdown_factor, trials, seed,
                                  &r.quiet_ttft, &r.mean_degradation, &r.max_degradation, r.per_trial.data()),
                  "noise_study");
    r.per_trial.resize(static_cast<size_t>(std::max<int64_t>(trials, 0)));
    return r;
}

// KVR-P lookup table (lookup_table.hpp:22-70): context length -> per-rank ratios for one p.
struct PartitionLookupTable {
    int64_t process_count = 0;
    std::map<int64_t, std::vector<double>> entries;

    void insert(int64_t context_length, std::vector<double> ratios) {
        if (process_count < 1) throw LookupError("table process count not set");
        if (static_cast<int64_t>(ratios.size()) != process_count)
            throw LookupError("ratio vector arity must equal the table process count");
        double sum = 0;
        for (double r : ratios) {
            if (r < 0) throw LookupError("table ratios must be non-negative");
            sum += r;
        }
        if (std::abs(sum - 1.0) > 1e-9) throw LookupError("table ratios must sum to 1");
        if (context_length < 1) throw LookupError("context length must be positive");
        entries[context_length] = std::move(ratios);
    }
};

namespace detail {
struct FlatTable {
    std::vector<int64_t> keys;
    std::vector<double> ratios;
    explicit FlatTable(const PartitionLookupTable& t) {
        for (const auto& [c, r] : t.entries) {
            keys.push_back(c);
            ratios.insert(ratios.end(), r.begin(), r.end());
        }
    }
};
}  // namespace detail

// ---------------------------------------------------------------- decode (extension)
// The reference stops at the first token (engine.hpp:88).  KVCache keeps the prompt's K/V on
// the device so decode steps can append rows at the next positions.
template <typename T = float>
class KVCache {
  public:
    KVCache(const WeightSet<T>& w, int64_t capacity) : w_(w) {
        kvp_kv_cache* c = nullptr;
        detail::check(kvp_kv_cache_create(w.engine(), capacity, &c), "kv_cache_create");
        cache_.reset(c, [](kvp_kv_cache* x) { kvp_kv_cache_destroy(x); });
    }
    int64_t length() const {
        int64_t n = 0;
        detail::check(kvp_kv_cache_length(cache_.get(), &n), "kv_cache_length");
        return n;
    }
    void reset(int64_t length) { detail::check(kvp_kv_cache_reset(cache_.get(), length), "kv_cache_reset"); }
    // prompt phase into the cache; returns first_token_hidden [1 x d]
    Matrix<T> prefill(const Matrix<T>& context) {
        if (context.cols != w_.config.d_model) throw DimensionError("prefill: context width != d_model");
        Matrix<T> ft(1, w_.config.d_model);
        detail::check(kvp_prefill_cached(w_.engine(), cache_.get(), context.values.data(), context.rows, nullptr,
                                         ft.values.data(), nullptr),
                      "prefill_cached");
        return ft;
    }
    // appends rows (n <= 8) at positions [length, length + n); returns their final hidden rows
    Matrix<T> decode(const Matrix<T>& rows) {
        if (rows.cols != w_.config.d_model) throw DimensionError("decode: row width != d_model");
        Matrix<T> out(rows.rows, rows.cols);
        detail::check(kvp_decode(w_.engine(), cache_.get(), rows.values.data(), rows.rows, out.values.data(), nullptr),
                      "decode");
        return out;
    }

  private:
    WeightSet<T> w_;
    std::shared_ptr<kvp_kv_cache> cache_;
};

inline std::vector<double> interpolate_partition(const PartitionLookupTable& table, int64_t C) {
    const detail::FlatTable f(table);
    std::vector<double> out(static_cast<size_t>(std::max<int64_t>(table.process_count, 1)));
    detail::check(kvp_interpolate_partition(f.keys.data(), f.ratios.data(), static_cast<int64_t>(f.keys.size()),
                                            table.process_count, C, out.data()),
                  "interpolate_partition");
    out.resize(static_cast<size_t>(std::max<int64_t>(table.process_count, 0)));
    return out;
}

inline ContextPartition partition_from_table(const PartitionLookupTable& table, int64_t C) {
    const detail::FlatTable f(table);
    ContextPartition out;
    out.context_length = C;
    out.boundaries.assign(static_cast<size_t>(std::max<int64_t>(table.process_count, 1) + 1), 0);
    detail::check(kvp_partition_from_table(f.keys.data(), f.ratios.data(), static_cast<int64_t>(f.keys.size()),
                                           table.process_count, C, out.boundaries.data()),
                  "partition_from_table");
    return out;
}

}  // namespace kvprefill
