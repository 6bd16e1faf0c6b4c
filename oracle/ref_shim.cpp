// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile straight from the reference
// sources where they lie (-I /root/reference/proj/include), output only into
// oracle/_ref/libkvref.so (git-ignored, shipped to the GPU box by gpurun).  It is used
// to pin the C restatement (kvp_oracle.c), to generate tests/golden/ and as the
// "reference" CPU baseline leg of bench.py.  No reference source is copied into the repo.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <iostream>
#include <memory>
#include <string>

#include "kvprefill/kvprefill.hpp"

using namespace kvprefill;

namespace {

int code_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const ConfigError&) { return 1; } catch (const DimensionError&) { return 2; }
    catch (const CacheError&) { return 3; } catch (const InputError&) { return 4; }
    catch (const PartitionError&) { return 5; } catch (const ProtocolError&) { return 6; }
    catch (const AssemblyError&) { return 7; } catch (const LookupError&) { return 8; }
    catch (const SearchError&) { return 9; } catch (const BudgetError&) { return 10; }
    catch (const CalibrationError&) { return 11; } catch (const IoError&) { return 12; }
    catch (...) { return 99; }
}

#define GUARD(body)                                   \
    try {                                             \
        body;                                         \
    } catch (...) {                                   \
        return code_of(std::current_exception());     \
    }                                                 \
    return 0;

struct RefConfig {
    int64_t d_model, n_heads, n_kv_heads, n_layers;
    uint64_t seed;
    int32_t precision;
    int32_t rms_norm;
};

ModelConfig to_model(const RefConfig* c) {
    ModelConfig m;
    m.d_model = c->d_model;
    m.n_heads = c->n_heads;
    m.n_kv_heads = c->n_kv_heads;
    m.n_layers = c->n_layers;
    m.seed = c->seed;
    m.precision = c->precision == 1 ? Precision::f64 : Precision::f32;
    m.rms_norm = c->rms_norm != 0;
    return m;
}

ContextPartition to_part(int64_t C, const int64_t* b, int64_t p) {
    ContextPartition part;
    part.context_length = C;
    part.boundaries.assign(b, b + p + 1);
    return part;
}

template <typename T>
Matrix<T> to_matrix(const T* v, int64_t rows, int64_t cols) {
    Matrix<T> m(rows, cols);
    std::memcpy(m.values.data(), v, static_cast<size_t>(rows * cols) * sizeof(T));
    return m;
}

struct Handle {
    int32_t precision;
    WeightSet<float> wf;
    WeightSet<double> wd;
};

template <typename T>
int run_t(const WeightSet<T>& w, int strategy, const T* ctx, int64_t C, const int64_t* b, int64_t p,
          int fault_kind, int64_t fault_rank, int64_t fault_layer, T* hidden_out, T* first_token,
          int64_t* metrics) {
    GUARD({
        FaultInjection f;
        f.kind = static_cast<FaultInjection::Kind>(fault_kind);
        f.rank = fault_rank;
        f.layer = fault_layer;
        const auto r = run(static_cast<Strategy>(strategy), to_matrix(ctx, C, w.config.d_model),
                           to_part(C, b, p), w, f);
        if (hidden_out)
            std::memcpy(hidden_out, r.hidden_out.values.data(), r.hidden_out.values.size() * sizeof(T));
        if (first_token)
            std::memcpy(first_token, r.first_token_hidden.values.data(),
                        r.first_token_hidden.values.size() * sizeof(T));
        if (metrics) {  // [barrier, dots[p], sent[p], recv[p], waits[p]]
            metrics[0] = r.metrics.barrier_count;
            for (int64_t i = 0; i < p; ++i) {
                metrics[1 + i] = r.metrics.dot_products[i];
                metrics[1 + p + i] = r.metrics.kv_pairs_sent[i];
                metrics[1 + 2 * p + i] = r.metrics.kv_pairs_received[i];
                metrics[1 + 3 * p + i] = r.metrics.wait_events[i];
            }
        }
    })
}

}  // namespace

extern "C" {

void* kvref_weights_create(const RefConfig* c) {
    try {
        auto h = std::make_unique<Handle>();
        h->precision = c->precision;
        if (c->precision == 1)
            h->wd = init_weights<double>(to_model(c));
        else
            h->wf = init_weights<float>(to_model(c));
        return h.release();
    } catch (...) {
        return nullptr;
    }
}

void kvref_weights_destroy(void* h) { delete static_cast<Handle*>(h); }

// Copies one layer's six matrices out (row-major, reference [in x out] layout).
int kvref_weights_layer(void* hv, int64_t layer, void* wq, void* wk, void* wv, void* wo, void* w1,
                        void* w2) {
    auto* h = static_cast<Handle*>(hv);
    GUARD({
        auto copy = [](auto& m, void* dst) {
            std::memcpy(dst, m.values.data(), m.values.size() * sizeof(m.values[0]));
        };
        if (h->precision == 1) {
            const auto& l = h->wd.layer(layer);
            copy(l.wq, wq); copy(l.wk, wk); copy(l.wv, wv); copy(l.wo, wo); copy(l.w1, w1); copy(l.w2, w2);
        } else {
            const auto& l = h->wf.layer(layer);
            copy(l.wq, wq); copy(l.wk, wk); copy(l.wv, wv); copy(l.wo, wo); copy(l.w1, w1); copy(l.w2, w2);
        }
    })
}

int kvref_random_context(int32_t precision, int64_t rows, int64_t d, uint64_t seed, void* out) {
    GUARD({
        if (precision == 1) {
            auto m = random_context<double>(rows, d, seed);
            std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
        } else {
            auto m = random_context<float>(rows, d, seed);
            std::memcpy(out, m.values.data(), m.values.size() * sizeof(float));
        }
    })
}

// run<T>(strategy, context, partition, weights, fault) -- engine.hpp:186-318.
int kvref_run(void* hv, int strategy, const void* ctx, int64_t C, const int64_t* b, int64_t p,
              int fault_kind, int64_t fault_rank, int64_t fault_layer, void* hidden_out,
              void* first_token, int64_t* metrics) {
    auto* h = static_cast<Handle*>(hv);
    if (h->precision == 1)
        return run_t<double>(h->wd, strategy, static_cast<const double*>(ctx), C, b, p, fault_kind,
                             fault_rank, fault_layer, static_cast<double*>(hidden_out),
                             static_cast<double*>(first_token), metrics);
    return run_t<float>(h->wf, strategy, static_cast<const float*>(ctx), C, b, p, fault_kind,
                        fault_rank, fault_layer, static_cast<float*>(hidden_out),
                        static_cast<float*>(first_token), metrics);
}

// naive_causal_forward (oracle.hpp:34-111), f64 only.
int kvref_naive_forward(void* hv, const double* ctx, int64_t C, double* out) {
    auto* h = static_cast<Handle*>(hv);
    GUARD({
        auto m = naive_causal_forward(to_matrix(ctx, C, h->wd.config.d_model), h->wd);
        std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
    })
}

// causal_attention (model.hpp:112-158), for per-op parity.
int kvref_causal_attention(const RefConfig* c, const void* Q, int64_t q_rows, const void* K,
                           const void* V, int64_t k_rows, int64_t offset, void* A) {
    GUARD({
        const ModelConfig m = to_model(c);
        if (c->precision == 1) {
            auto a = causal_attention(to_matrix(static_cast<const double*>(Q), q_rows, m.q_dim()),
                                      to_matrix(static_cast<const double*>(K), k_rows, m.kv_dim()),
                                      to_matrix(static_cast<const double*>(V), k_rows, m.kv_dim()),
                                      CausalMask{offset, q_rows}, m);
            std::memcpy(A, a.values.data(), a.values.size() * sizeof(double));
        } else {
            auto a = causal_attention(to_matrix(static_cast<const float*>(Q), q_rows, m.q_dim()),
                                      to_matrix(static_cast<const float*>(K), k_rows, m.kv_dim()),
                                      to_matrix(static_cast<const float*>(V), k_rows, m.kv_dim()),
                                      CausalMask{offset, q_rows}, m);
            std::memcpy(A, a.values.data(), a.values.size() * sizeof(float));
        }
    })
}

int kvref_even_partition(int64_t C, int64_t p, int64_t* out) {
    GUARD({
        auto part = even_partition(C, p);
        std::memcpy(out, part.boundaries.data(), part.boundaries.size() * sizeof(int64_t));
    })
}

int kvref_partition_from_ratios(int64_t C, const double* ratios, int64_t p, int64_t* out) {
    GUARD({
        auto part = partition_from_ratios(C, std::vector<double>(ratios, ratios + p));
        std::memcpy(out, part.boundaries.data(), part.boundaries.size() * sizeof(int64_t));
    })
}

struct RefCost { double alpha, proj_coeff, softmax_coeff, fixed_overhead; };
struct RefNet { double bandwidth, latency; };

static CostModel to_cost(const RefCost* c) {
    CostModel m;
    m.alpha = c->alpha;
    m.proj_coeff = c->proj_coeff;
    m.softmax_coeff = c->softmax_coeff;
    m.fixed_overhead = c->fixed_overhead;
    return m;
}

static NetworkModel to_net(const RefNet* n) {
    NetworkModel m;
    m.bandwidth = n->bandwidth;
    m.latency = n->latency;
    return m;
}

int kvref_simulate_ttft(int strategy, int64_t C, const int64_t* b, int64_t p, int64_t n_layers,
                        const RefCost* cost, const RefNet* net, double* out) {
    GUARD({
        ModelConfig m;
        m.n_layers = n_layers;
        *out = simulate_ttft(static_cast<Strategy>(strategy), to_part(C, b, p), m, to_cost(cost),
                             to_net(net))
                   .ttft;
    })
}

// hierarchical_grid_search / binary_search_two with the simulate_ttft(KVR) evaluator
// (commands.hpp:558-562).  which: 0 grid, 1 bisection, 2 exhaustive.
int kvref_search_sim(int which, int64_t C, int64_t p, int64_t grid_width, int64_t initial_stride,
                     int64_t min_stride, int64_t n_layers, const RefCost* cost, const RefNet* net,
                     int64_t* out, double* ttft, int64_t* evals, int64_t* levels) {
    GUARD({
        ModelConfig m;
        m.n_layers = n_layers;
        const CostModel cm = to_cost(cost);
        const NetworkModel nm = to_net(net);
        SearchConfig s;
        s.grid_width = grid_width;
        s.initial_stride = initial_stride;
        s.min_stride = min_stride;
        s.evaluator = [&](const ContextPartition& part) {
            return simulate_ttft(Strategy::KVR, part, m, cm, nm).ttft;
        };
        SearchResult r = which == 0   ? hierarchical_grid_search(C, p, s)
                         : which == 1 ? binary_search_two(C, s)
                                      : exhaustive_partition_search(C, p, s.evaluator);
        std::memcpy(out, r.partition.boundaries.data(), r.partition.boundaries.size() * sizeof(int64_t));
        *ttft = r.ttft;
        *evals = r.evaluations;
        *levels = r.levels;
    })
}

int kvref_practical_bound(int64_t C, int64_t p, int64_t n_layers, const RefCost* cost, int64_t* out,
                          double* ttft) {
    GUARD({
        ModelConfig m;
        m.n_layers = n_layers;
        auto pb = practical_bound(C, p, m, to_cost(cost));
        std::memcpy(out, pb.partition.boundaries.data(), pb.partition.boundaries.size() * sizeof(int64_t));
        *ttft = pb.ttft;
    })
}

// noise_study (simnet.hpp:332-353)
int kvref_noise_study(int strategy, int64_t C, const int64_t* b, int64_t p, int64_t n_layers, const RefCost* cost,
                      const RefNet* net, double factor, int64_t trials, uint64_t seed, double* quiet, double* mean,
                      double* mx, double* per_trial) {
    GUARD({
        ModelConfig m;
        m.n_layers = n_layers;
        const auto st = noise_study(static_cast<Strategy>(strategy), to_part(C, b, p), m, to_cost(cost), to_net(net),
                                    factor, trials, seed);
        *quiet = st.quiet_ttft;
        *mean = st.mean_degradation;
        *mx = st.max_degradation;
        for (size_t i = 0; i < st.per_trial.size(); ++i) per_trial[i] = st.per_trial[i];
    })
}

// interpolate_partition / partition_from_table (lookup_table.hpp:44-70)
int kvref_table(const int64_t* Cs, const double* ratios, int64_t n, int64_t p, int64_t C, double* ratios_out,
                int64_t* boundaries_out) {
    GUARD({
        PartitionLookupTable t;
        t.process_count = p;
        for (int64_t i = 0; i < n; ++i) t.insert(Cs[i], std::vector<double>(ratios + i * p, ratios + (i + 1) * p));
        const auto r = interpolate_partition(t, C);
        std::memcpy(ratios_out, r.data(), r.size() * sizeof(double));
        const auto part = partition_from_table(t, C);
        std::memcpy(boundaries_out, part.boundaries.data(), part.boundaries.size() * sizeof(int64_t));
    })
}

int kvref_ttft_star(int64_t C, int64_t p, double alpha, double* out) { GUARD({ *out = ttft_star(C, p, alpha); }) }

double kvref_table_build_cost(double T, int64_t N, int64_t C) { return table_build_cost(T, N, C); }


// The reference CLI's subcommands (commands.hpp cmd_*), config from a JSON file, with the
// --out / --table overrides of tools/kvprefill_main.cpp; returns the CLI exit code
// (ConfigError -> 2, other Error -> 1).
int kvref_cli(const char* sub, const char* config_path, int64_t predict_c, const char* out_path,
              const char* table_path) {
    try {
        ExperimentConfig cfg;
        if (config_path && *config_path) cfg = load_experiment_config(config_path);
        if (out_path && *out_path) cfg.out_path = out_path;
        if (table_path && *table_path) cfg.table_path = table_path;
        const std::string s(sub);
        int rc = 2;
        if (s == "verify") rc = cmd_verify(cfg);
        else if (s == "sweep") rc = cmd_sweep(cfg);
        else if (s == "search") rc = cmd_search(cfg);
        else if (s == "predict") rc = cmd_predict(cfg, predict_c);
        else if (s == "noise") rc = cmd_noise(cfg);
        std::cout.flush();
        std::cerr.flush();
        return rc;
    } catch (const ConfigError&) {
        return 2;
    } catch (const Error&) {
        return 1;
    }
}
}  // extern "C"
