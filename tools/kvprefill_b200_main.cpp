// kvprefill_b200 -- command-line front end of the B200 path, a drop-in for the reference CLI
// (tools/kvprefill_main.cpp + commands.hpp:303-860): the same subcommands (verify, sweep,
// search, predict, noise), the same JSON experiment config (commands.hpp:51-69, 140-231: unknown
// keys rejected, same defaults), the same CSV / JSON output schemas and the same exit codes
// (ConfigError / usage -> 2, other errors -> 1).  Planning output (sweep / search / predict /
// noise) is computed by libkvp_b200's bit-exact balancer, so with engine runs disabled it is
// byte-identical to the reference's.  Engine runs (verify, sweep's max_dev column) execute on
// the GPU through the C++ drop-in header.
//
// Differences, all stated in the output:
//   * model.precision f64 has no GPU path; engine checks then run in f32 (the reference's
//     f32 parity mode) and say so;
//   * verify's "serial vs brute-force oracle" check compares the engine's serial forward with
//     the layer-by-layer composition of the drop-in model functions (layer_qkv,
//     layer_finish) on the GPU -- the CPU brute-force oracle is test infrastructure here;
//   * sweep --measure appends a ttft_measured column (device-timed TTFT of the row's run on
//     the GPU(s), seconds).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "kvprefill_b200/kvprefill.hpp"
#include "kvprefill_b200/table_io.hpp"

namespace kv = kvprefill;
using nlohmann::json;

namespace {

enum class PartSource { Even, Ratios, Search, Table };

// The experiment: every command is a pure function of it (commands.hpp:49-69).
struct Experiment {
    kv::ModelConfig model;
    std::vector<kv::Strategy> strategies{kv::Strategy::Serial, kv::Strategy::TSP, kv::Strategy::KVR};
    std::vector<int64_t> context_lengths{64, 128, 256};
    std::vector<int64_t> process_counts{1, 2, 4};
    PartSource source = PartSource::Even;
    std::vector<double> ratios;
    std::string table_path;
    kv::CostModel cost;
    kv::NetworkModel network;
    double noise_factor = 64.0;
    int64_t noise_trials = 20;
    kv::SearchConfig search;
    kv::FaultInjection fault;
    int64_t equivalence_max_c = 512;
    uint64_t seed = 1;
    std::string out_path;
    std::string format = "csv";
};

std::string strategy_name(kv::Strategy s) {
    return s == kv::Strategy::Serial ? "serial" : (s == kv::Strategy::TSP ? "tsp" : "kvr");
}

kv::Strategy strategy_named(const std::string& n) {
    if (n == "serial") return kv::Strategy::Serial;
    if (n == "tsp") return kv::Strategy::TSP;
    if (n == "kvr") return kv::Strategy::KVR;
    throw kv::ConfigError("unknown strategy: " + n);
}

const char* fault_name(kv::FaultInjection::Kind k) {
    switch (k) {
        case kv::FaultInjection::Kind::CorruptLayerTag: return "corrupt_layer_tag";
        case kv::FaultInjection::Kind::DropMessage: return "drop_message";
        case kv::FaultInjection::Kind::DuplicateMessage: return "duplicate_message";
        default: return "none";
    }
}

kv::FaultInjection::Kind fault_named(const std::string& n) {
    for (auto k : {kv::FaultInjection::Kind::None, kv::FaultInjection::Kind::CorruptLayerTag,
                   kv::FaultInjection::Kind::DropMessage, kv::FaultInjection::Kind::DuplicateMessage})
        if (n == fault_name(k)) return k;
    throw kv::ConfigError("unknown fault kind '" + n + "'");
}

std::string g10(double v) {  // the reference's number format (commands.hpp:108-112)
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.10g", v);
    return buf;
}

std::string dashed(const kv::ContextPartition& part) {
    std::string s;
    for (int64_t c : part.sizes()) s += (s.empty() ? "" : "-") + std::to_string(c);
    return s;
}

// ------------------------------------------------------------------ config parsing
void only_keys(const json& obj, const std::string& scope, std::initializer_list<const char*> keys) {
    for (const auto& item : obj.items()) {
        bool ok = false;
        for (const char* k : keys) ok = ok || item.key() == k;
        if (!ok) throw kv::ConfigError("unknown config key '" + scope + item.key() + "'");
    }
}

template <typename T>
void take(const json& obj, const std::string& scope, const char* key, T& out) {
    if (!obj.contains(key)) return;
    try {
        out = obj.at(key).get<T>();
    } catch (const json::exception& e) {
        throw kv::ConfigError("config field '" + scope + key + "': " + e.what());
    }
}

Experiment parse_experiment(const std::string& text) {
    json doc;
    try {
        doc = json::parse(text);
    } catch (const json::parse_error& e) {
        throw kv::ConfigError(std::string("config parse error: ") + e.what());
    }
    if (!doc.is_object()) throw kv::ConfigError("config root must be a JSON object");
    only_keys(doc, "", {"model", "strategies", "context_lengths", "process_counts", "partition_source", "ratios",
                        "table_path", "cost", "network", "noise", "search", "fault", "equivalence_max_c", "seed",
                        "out_path", "format"});
    Experiment x;
    if (doc.contains("model")) {
        const json& m = doc.at("model");
        only_keys(m, "model.", {"d_model", "n_heads", "n_kv_heads", "n_layers", "seed", "precision", "rms_norm"});
        take(m, "model.", "d_model", x.model.d_model);
        take(m, "model.", "n_heads", x.model.n_heads);
        take(m, "model.", "n_kv_heads", x.model.n_kv_heads);
        take(m, "model.", "n_layers", x.model.n_layers);
        take(m, "model.", "seed", x.model.seed);
        take(m, "model.", "rms_norm", x.model.rms_norm);
        std::string prec = "f64";
        take(m, "model.", "precision", prec);
        if (prec == "f32") x.model.precision = kv::Precision::f32;
        else if (prec == "f64") x.model.precision = kv::Precision::f64;
        else if (prec == "bf16") x.model.precision = kv::Precision::bf16;  // additive
        else throw kv::ConfigError("unknown precision '" + prec + "' (expected f32 or f64)");
    }
    if (doc.contains("strategies")) {
        std::vector<std::string> names;
        take(doc, "", "strategies", names);
        x.strategies.clear();
        for (const auto& n : names) x.strategies.push_back(strategy_named(n));
        if (x.strategies.empty()) throw kv::ConfigError("strategies must be non-empty");
    }
    take(doc, "", "context_lengths", x.context_lengths);
    take(doc, "", "process_counts", x.process_counts);
    if (doc.contains("partition_source")) {
        std::string n;
        take(doc, "", "partition_source", n);
        if (n == "even") x.source = PartSource::Even;
        else if (n == "ratios") x.source = PartSource::Ratios;
        else if (n == "search") x.source = PartSource::Search;
        else if (n == "table") x.source = PartSource::Table;
        else throw kv::ConfigError("unknown partition_source '" + n + "'");
    }
    take(doc, "", "ratios", x.ratios);
    take(doc, "", "table_path", x.table_path);
    if (doc.contains("cost")) {
        const json& c = doc.at("cost");
        only_keys(c, "cost.", {"alpha", "proj_coeff", "softmax_coeff", "fixed_overhead"});
        take(c, "cost.", "alpha", x.cost.alpha);
        take(c, "cost.", "proj_coeff", x.cost.proj_coeff);
        take(c, "cost.", "softmax_coeff", x.cost.softmax_coeff);
        take(c, "cost.", "fixed_overhead", x.cost.fixed_overhead);
    }
    if (doc.contains("network")) {
        const json& n = doc.at("network");
        only_keys(n, "network.", {"bandwidth", "latency"});
        take(n, "network.", "bandwidth", x.network.bandwidth);
        take(n, "network.", "latency", x.network.latency);
    }
    if (doc.contains("noise")) {
        const json& n = doc.at("noise");
        only_keys(n, "noise.", {"slowdown_factor", "trials"});
        take(n, "noise.", "slowdown_factor", x.noise_factor);
        take(n, "noise.", "trials", x.noise_trials);
    }
    if (doc.contains("search")) {
        const json& s = doc.at("search");
        only_keys(s, "search.", {"grid_width", "initial_stride", "min_stride"});
        take(s, "search.", "grid_width", x.search.grid_width);
        take(s, "search.", "initial_stride", x.search.initial_stride);
        take(s, "search.", "min_stride", x.search.min_stride);
    }
    if (doc.contains("fault")) {
        const json& f = doc.at("fault");
        only_keys(f, "fault.", {"kind", "rank", "layer"});
        std::string k = "none";
        take(f, "fault.", "kind", k);
        x.fault.kind = fault_named(k);
        take(f, "fault.", "rank", x.fault.rank);
        take(f, "fault.", "layer", x.fault.layer);
    }
    take(doc, "", "equivalence_max_c", x.equivalence_max_c);
    take(doc, "", "seed", x.seed);
    take(doc, "", "out_path", x.out_path);
    take(doc, "", "format", x.format);
    if (x.format != "csv" && x.format != "json") throw kv::ConfigError("format must be csv or json");
    x.model.validate();
    x.cost.validate();
    x.network.validate();
    if (x.context_lengths.empty()) throw kv::ConfigError("context_lengths must be non-empty");
    if (x.process_counts.empty()) throw kv::ConfigError("process_counts must be non-empty");
    return x;
}

// ------------------------------------------------------------------ shared helpers
double simulated(kv::Strategy s, const kv::ContextPartition& part, const Experiment& x) {
    return kv::simulate_ttft_value(s, part, x.model, x.cost, x.network);
}

// The partition a chained (KVR) run uses at (C, p) (commands.hpp:252-278).
kv::ContextPartition chain_partition(const Experiment& x, int64_t C, int64_t p) {
    if (p == 1) return kv::even_partition(C, 1);
    switch (x.source) {
        case PartSource::Even: return kv::even_partition(C, p);
        case PartSource::Ratios:
            if (static_cast<int64_t>(x.ratios.size()) != p)
                throw kv::ConfigError("ratios arity " + std::to_string(x.ratios.size()) + " does not match p=" +
                                      std::to_string(p));
            return kv::partition_from_ratios(C, x.ratios);
        case PartSource::Search: return kv::search_partition(C, p, x.model, x.cost, x.network, x.search).partition;
        case PartSource::Table: {
            if (x.table_path.empty()) throw kv::ConfigError("partition_source=table needs table_path");
            const kv::PartitionLookupTable t = kv::load_table(x.table_path);
            if (t.process_count != p)
                throw kv::ConfigError("table is for p=" + std::to_string(t.process_count) + ", requested p=" +
                                      std::to_string(p));
            return kv::partition_from_table(t, C);
        }
    }
    throw kv::ConfigError("unhandled partition source");
}

// GPU engine: weights generated once per CLI invocation (device-side init_weights).
class Gpu {
  public:
    explicit Gpu(const kv::ModelConfig& m) : model_(m) {
        if (model_.precision == kv::Precision::f64) {
            model_.precision = kv::Precision::f32;
            f64_in_f32_ = true;
        }
    }
    bool f64_in_f32() const { return f64_in_f32_; }
    const kv::WeightSet<float>& weights() {
        if (!w_) w_ = std::make_unique<kv::WeightSet<float>>(kv::init_weights<float>(model_, devices()));
        return *w_;
    }
    kv::ExecutionResult<float> run(kv::Strategy s, const kv::MatrixF& ctx, const kv::ContextPartition& part,
                                   const kv::FaultInjection& f = {}) {
        return kv::run(s, ctx, part, weights(), f);
    }
    double last_ttft_s() {
        float ms = 0;
        kv::detail::check(kvp_engine_last_ttft_ms(weights().engine(), &ms), "last_ttft_ms");
        return ms * 1e-3;
    }

  private:
    static std::vector<int32_t> devices() {
        const int n = kvp_device_count();
        std::vector<int32_t> d;
        for (int i = 0; i < std::max(n, 1); ++i) d.push_back(i);
        return d;
    }
    kv::ModelConfig model_;
    bool f64_in_f32_ = false;
    std::unique_ptr<kv::WeightSet<float>> w_;
};

// Deviation of a strategy's hidden states from the serial forward (commands.hpp:280-288).
double equivalence_deviation(Gpu& gpu, const Experiment& x, kv::Strategy s, int64_t C,
                             const kv::ContextPartition& part) {
    const kv::MatrixF ctx = kv::random_context<float>(C, x.model.d_model, x.seed + 17);
    const auto serial = gpu.run(kv::Strategy::Serial, ctx, kv::even_partition(C, 1));
    const auto other = gpu.run(s, ctx, part);
    return kv::max_rel_dev(other.hidden_out, serial.hidden_out);
}

class Sink {  // --out file or stdout
  public:
    explicit Sink(const std::string& path) {
        if (!path.empty()) {
            file_.open(path);
            if (!file_) throw kv::IoError("cannot open output file: " + path);
        }
    }
    std::ostream& os() { return file_.is_open() ? static_cast<std::ostream&>(file_) : std::cout; }
    bool to_file() const { return file_.is_open(); }

  private:
    std::ofstream file_;
};

// ------------------------------------------------------------------ verify
int cmd_verify(const Experiment& x) {
    struct Check {
        std::string name, detail;
        bool ok;
    };
    std::vector<Check> checks;
    auto report = [&](const std::string& name, bool ok, const std::string& detail) {
        checks.push_back({name, detail, ok});
        std::cout << (ok ? "[pass] " : "[FAIL] ") << name;
        if (!detail.empty()) std::cout << "  (" << detail << ")";
        std::cout << "\n";
    };
    Gpu gpu(x.model);
    if (gpu.f64_in_f32())
        std::cout << "note: model.precision f64 has no GPU path; engine checks run in f32\n";

    {  // 9 tokens over 3 workers, counts known in closed form
        const kv::MatrixF ctx = kv::random_context<float>(9, x.model.d_model, x.seed);
        const auto kvr = gpu.run(kv::Strategy::KVR, ctx, kv::ContextPartition::from_sizes({4, 3, 2}));
        const auto& km = kvr.metrics;
        const std::string dots = std::to_string(km.per_layer_dot_products(0)) + "/" +
                                 std::to_string(km.per_layer_dot_products(1)) + "/" +
                                 std::to_string(km.per_layer_dot_products(2));
        report("fixture kvr [4-3-2] dot products 16/21/18", dots == "16/21/18", dots);
        report("fixture kvr [4-3-2] traffic 11 pairs / 22 rows",
               km.per_layer_pairs_sent() == 11 && km.per_layer_rows_sent() == 22,
               std::to_string(km.per_layer_pairs_sent()) + " pairs / " + std::to_string(km.per_layer_rows_sent()) +
                   " rows per layer");
        const auto tsp = gpu.run(kv::Strategy::TSP, ctx, kv::even_partition(9, 3));
        const auto& tm = tsp.metrics;
        bool all27 = true;
        for (int r = 0; r < 3; ++r) all27 = all27 && tm.per_layer_dot_products(r) == 27;
        report("fixture tsp [3-3-3] dot products 27 per worker", all27,
               std::to_string(tm.per_layer_dot_products(0)) + " each");
        report("fixture tsp [3-3-3] traffic 18 pairs / 36 rows",
               tm.per_layer_pairs_sent() == 18 && tm.per_layer_rows_sent() == 36,
               std::to_string(tm.per_layer_pairs_sent()) + " pairs / " + std::to_string(tm.per_layer_rows_sent()) +
                   " rows per layer");
        report("fixture barrier counts", tm.barrier_count == x.model.n_layers && km.barrier_count == 0,
               "tsp " + std::to_string(tm.barrier_count) + ", kvr " + std::to_string(km.barrier_count));
    }
    {  // engine serial forward vs the layer-by-layer model functions
        const int64_t C = std::min<int64_t>(*std::min_element(x.context_lengths.begin(), x.context_lengths.end()), 64);
        const kv::MatrixF ctx = kv::random_context<float>(C, x.model.d_model, x.seed + 5);
        const auto serial = gpu.run(kv::Strategy::Serial, ctx, kv::even_partition(C, 1));
        kv::MatrixF h = ctx;
        for (int64_t l = 0; l < x.model.n_layers; ++l) {
            const auto qkv = kv::layer_qkv(h, gpu.weights(), l);
            h = kv::layer_finish(h, qkv.Q, qkv.K, qkv.V, 0, gpu.weights(), l);
        }
        const double dev = kv::max_rel_dev(serial.hidden_out, h);
        const double tol = x.model.precision == kv::Precision::bf16 ? 1e-1 : 1e-4;
        report("serial forward vs layer-by-layer model functions (C=" + std::to_string(C) + ")", dev <= tol,
               "max rel dev " + g10(dev));
    }
    const double tol = x.model.precision == kv::Precision::f64 ? 1e-10 : (x.model.precision == kv::Precision::f32 ? 1e-4 : 1e-1);
    for (int64_t C : x.context_lengths) {
        for (int64_t p : x.process_counts) {
            if (p > C) {
                std::cout << "[skip] C=" << C << " p=" << p << " infeasible\n";
                continue;
            }
            if (C > x.equivalence_max_c) {
                std::cout << "[skip] C=" << C << " equivalence check above equivalence_max_c\n";
                continue;
            }
            for (kv::Strategy s : x.strategies) {
                if (s == kv::Strategy::Serial) continue;
                // chained runs get a descending partition so the offsets are exercised
                kv::ContextPartition part;
                if (s == kv::Strategy::TSP || C < 2 * p) {
                    part = kv::even_partition(C, p);
                } else {
                    std::vector<double> w(static_cast<size_t>(p));
                    const double tri = static_cast<double>(p) * static_cast<double>(p + 1) / 2.0;
                    for (int64_t i = 0; i < p; ++i) w[static_cast<size_t>(i)] = static_cast<double>(p - i) / tri;
                    part = kv::partition_from_ratios(C, w);
                }
                const std::string label = strategy_name(s) + " C=" + std::to_string(C) + " p=" + std::to_string(p);
                const kv::MatrixF ctx = kv::random_context<float>(C, x.model.d_model, x.seed + 17);
                const auto serial = gpu.run(kv::Strategy::Serial, ctx, kv::even_partition(C, 1));
                const auto res = gpu.run(s, ctx, part);
                const double dev = kv::max_rel_dev(res.hidden_out, serial.hidden_out);
                report("equivalence " + label, dev <= tol, "max rel dev " + g10(dev) + " tol " + g10(tol));
                const auto expect = kv::dot_product_counts(s, part);
                bool dots_ok = true;
                for (int64_t r = 0; r < p; ++r)
                    dots_ok = dots_ok && res.metrics.per_layer_dot_products(r) == expect[static_cast<size_t>(r)];
                report("dot counts " + label, dots_ok, "");
                report("traffic counts " + label,
                       res.metrics.per_layer_pairs_sent() == kv::traffic_pairs(s, part) &&
                           res.metrics.total_rows_sent() == 2 * res.metrics.total_pairs_sent(),
                       std::to_string(res.metrics.per_layer_pairs_sent()) + " pairs per layer");
            }
        }
    }
    bool negative_test = false;
    if (x.fault.kind != kv::FaultInjection::Kind::None) {  // must surface; exits nonzero by design
        negative_test = true;
        const int64_t p = std::max<int64_t>(2, x.fault.rank + 2), C = 4 * p;
        const kv::MatrixF ctx = kv::random_context<float>(C, x.model.d_model, x.seed);
        std::string what;
        bool surfaced = false;
        try {
            gpu.run(kv::Strategy::KVR, ctx, kv::even_partition(C, p), x.fault);
        } catch (const kv::Error& e) {
            surfaced = true;
            what = e.what();
        }
        report(std::string("fault injection surfaced (") + fault_name(x.fault.kind) + ")", surfaced,
               surfaced ? what : "no error raised");
        std::cout << "note: fault injection is a negative test; nonzero exit is the expected outcome\n";
    }
    bool all = std::all_of(checks.begin(), checks.end(), [](const Check& c) { return c.ok; });
    std::cout << (all ? "all checks passed" : "CHECKS FAILED") << " (" << checks.size() << " checks)\n";
    all = all && !negative_test;
    if (!x.out_path.empty()) {
        json summary{{"all_passed", all}, {"checks", json::array()}};
        for (const auto& c : checks) summary["checks"].push_back({{"name", c.name}, {"passed", c.ok}, {"detail", c.detail}});
        std::ofstream f(x.out_path);
        if (!f) throw kv::IoError("cannot open output file: " + x.out_path);
        f << summary.dump(2) << "\n";
    }
    return all ? 0 : 1;
}

// ------------------------------------------------------------------ sweep
struct SweepRow {
    std::string strategy, partition;
    int64_t C = 0, p = 0, dot_max = 0, pairs = 0, rows = 0, barriers = 0;
    double ttft_sim = 0, speedup = 0, star = 0, lower = 0, max_dev = NAN, measured = NAN;
    bool skipped = false;
};

int cmd_sweep(const Experiment& x, bool measure) {
    std::vector<int64_t> Cs = x.context_lengths, Ps = x.process_counts;
    std::sort(Cs.begin(), Cs.end());
    std::sort(Ps.begin(), Ps.end());
    std::map<int64_t, double> serial_time;
    for (int64_t C : Cs) serial_time[C] = simulated(kv::Strategy::Serial, kv::even_partition(C, 1), x);
    std::map<std::pair<int64_t, int64_t>, double> lower_memo;
    std::unique_ptr<Gpu> gpu;
    auto engine = [&]() -> Gpu& {
        if (!gpu) gpu = std::make_unique<Gpu>(x.model);
        return *gpu;
    };

    std::vector<SweepRow> rows;
    for (int64_t C : Cs) {
        for (int64_t p : Ps) {
            for (kv::Strategy s : x.strategies) {
                if (s == kv::Strategy::Serial && p != 1) continue;
                SweepRow r;
                r.strategy = strategy_name(s);
                r.C = C;
                r.p = p;
                if (p > C) {
                    r.skipped = true;
                    std::cerr << "warning: skipping infeasible C=" << C << " p=" << p << "\n";
                    rows.push_back(r);
                    continue;
                }
                const kv::ContextPartition part = s == kv::Strategy::KVR ? chain_partition(x, C, p) : kv::even_partition(C, p);
                r.partition = dashed(part);
                r.ttft_sim = simulated(s, part, x);
                r.speedup = serial_time[C] / r.ttft_sim;
                r.star = kv::ttft_star(C, p, x.cost.alpha * static_cast<double>(x.model.n_layers));
                auto it = lower_memo.find({C, p});
                if (it == lower_memo.end())
                    it = lower_memo.emplace(std::make_pair(C, p), kv::ttft_practical_lower(C, p, x.model, x.cost)).first;
                r.lower = it->second;
                const auto dots = kv::dot_product_counts(s, part);
                r.dot_max = *std::max_element(dots.begin(), dots.end());
                r.pairs = kv::traffic_pairs(s, part);
                r.rows = 2 * r.pairs;
                r.barriers = s == kv::Strategy::TSP ? x.model.n_layers : 0;
                if (C <= x.equivalence_max_c) r.max_dev = equivalence_deviation(engine(), x, s, C, part);
                if (measure) {
                    const kv::MatrixF ctx = kv::random_context<float>(C, x.model.d_model, x.seed + 17);
                    engine().run(s, ctx, part);  // warm-up (graph capture / first touch)
                    engine().run(s, ctx, part);
                    r.measured = engine().last_ttft_s();
                }
                rows.push_back(r);
            }
        }
    }

    Sink sink(x.out_path);
    std::ostream& os = sink.os();
    if (x.format == "json") {
        json doc = json::array();
        for (const auto& r : rows) {
            json j{{"strategy", r.strategy}, {"C", r.C}, {"p", r.p}, {"partition", r.partition}};
            if (r.skipped) {
                j["skipped"] = true;
            } else {
                j["ttft_sim"] = r.ttft_sim;
                j["speedup"] = r.speedup;
                j["ttft_star"] = r.star;
                j["ttft_lower"] = r.lower;
                j["dot_max"] = r.dot_max;
                j["pairs"] = r.pairs;
                j["rows"] = r.rows;
                j["barriers"] = r.barriers;
                j["max_dev"] = std::isnan(r.max_dev) ? json() : json(r.max_dev);
                if (measure) j["ttft_measured"] = r.measured;
            }
            doc.push_back(std::move(j));
        }
        os << doc.dump(2) << "\n";
    } else {
        os << "strategy,C,p,partition,ttft_sim,speedup,ttft_star,ttft_lower,dot_max,pairs,rows,barriers,max_dev"
           << (measure ? ",ttft_measured" : "") << "\n";
        for (const auto& r : rows) {
            os << r.strategy << "," << r.C << "," << r.p << ",";
            if (r.skipped) {
                os << "skipped,nan,nan,nan,nan,0,0,0,0,nan" << (measure ? ",nan" : "") << "\n";
                continue;
            }
            os << r.partition << "," << g10(r.ttft_sim) << "," << g10(r.speedup) << "," << g10(r.star) << ","
               << g10(r.lower) << "," << r.dot_max << "," << r.pairs << "," << r.rows << "," << r.barriers << ","
               << (std::isnan(r.max_dev) ? std::string("nan") : g10(r.max_dev));
            if (measure) os << "," << g10(r.measured);
            os << "\n";
        }
    }
    if (sink.to_file()) std::cout << "wrote " << rows.size() << " rows to " << x.out_path << "\n";
    return 0;
}

// ------------------------------------------------------------------ search / predict
int cmd_search(const Experiment& x) {
    if (x.process_counts.size() != 1) throw kv::ConfigError("search needs exactly one process count");
    const int64_t p = x.process_counts.front();
    if (p < 2) throw kv::ConfigError("search needs at least two processes; p=1 has nothing to balance");
    if (x.table_path.empty()) throw kv::ConfigError("search needs table_path for its output");
    kv::PartitionLookupTable table;
    if (std::ifstream(x.table_path).good()) {  // extend an existing table
        table = kv::load_table(x.table_path);
        if (table.process_count != p)
            throw kv::ConfigError("existing table is for p=" + std::to_string(table.process_count) +
                                  ", requested p=" + std::to_string(p));
    } else {
        table.process_count = p;
    }
    bool failures = false;
    for (int64_t C : x.context_lengths) {
        try {
            const kv::SearchResult found = kv::search_partition(C, p, x.model, x.cost, x.network, x.search);
            std::vector<double> shares;
            for (int64_t c : found.partition.sizes()) shares.push_back(static_cast<double>(c) / static_cast<double>(C));
            table.insert(C, std::move(shares));
            std::cout << "C=" << C << " partition=" << dashed(found.partition) << " ttft=" << g10(found.ttft)
                      << " evaluations=" << found.evaluations << "\n";
        } catch (const kv::Error& e) {
            failures = true;
            std::cerr << "warning: search failed for C=" << C << ": " << e.what() << "\n";
        }
    }
    if (table.entries.empty()) throw kv::ConfigError("no table entries were produced");
    kv::save_table(table, x.table_path);
    std::cout << "table with " << table.entries.size() << " entries written to " << x.table_path << "\n";
    return failures ? 1 : 0;
}

int cmd_predict(const Experiment& x, int64_t C) {
    if (x.table_path.empty()) throw kv::ConfigError("predict needs table_path");
    if (!std::ifstream(x.table_path).good()) throw kv::ConfigError("table file does not exist: " + x.table_path);
    const kv::PartitionLookupTable table = kv::load_table(x.table_path);
    const int64_t p = table.process_count;
    const bool clamped = !table.entries.empty() &&
                         (C < table.entries.begin()->first || C > table.entries.rbegin()->first);
    const kv::ContextPartition part = kv::partition_from_ratios(C, kv::interpolate_partition(table, C));
    if (clamped)
        std::cerr << "warning: C=" << C << " outside table range [" << table.entries.begin()->first << ", "
                  << table.entries.rbegin()->first << "], clamped to nearest entry\n";
    const double predicted = simulated(kv::Strategy::KVR, part, x);
    const kv::SearchResult fresh = kv::search_partition(C, p, x.model, x.cost, x.network, x.search);
    const double gap = (predicted - fresh.ttft) / fresh.ttft;
    Sink sink(x.out_path);
    if (x.format == "json") {
        const json doc{{"C", C},          {"p", p},         {"partition", part.sizes()}, {"ttft_pred", predicted},
                       {"ttft_search", fresh.ttft}, {"gap", gap}, {"clamped", clamped}};
        sink.os() << doc.dump(2) << "\n";
    } else {
        sink.os() << "C,p,partition,ttft_pred,ttft_search,gap,clamped\n"
                  << C << "," << p << "," << dashed(part) << "," << g10(predicted) << "," << g10(fresh.ttft) << ","
                  << g10(gap) << "," << (clamped ? "true" : "false") << "\n";
    }
    if (sink.to_file())
        std::cout << "predicted partition " << dashed(part) << " ttft " << g10(predicted) << " (gap "
                  << g10(gap * 100.0) << "% vs fresh search)\n";
    return 0;
}

// ------------------------------------------------------------------ noise
int cmd_noise(const Experiment& x) {
    struct Row {
        std::string strategy, partition;
        int64_t C, p;
        double quiet, mean, max;
    };
    std::vector<Row> rows;
    std::vector<std::string> verdicts;
    std::vector<int64_t> Cs = x.context_lengths, Ps = x.process_counts;
    std::sort(Cs.begin(), Cs.end());
    std::sort(Ps.begin(), Ps.end());
    for (int64_t C : Cs) {
        for (int64_t p : Ps) {
            if (p > C) {
                std::cerr << "warning: skipping infeasible C=" << C << " p=" << p << "\n";
                continue;
            }
            std::optional<double> tsp_mean, kvr_mean;
            for (kv::Strategy s : x.strategies) {
                if (s == kv::Strategy::Serial) continue;
                const kv::ContextPartition part = s == kv::Strategy::KVR ? chain_partition(x, C, p) : kv::even_partition(C, p);
                const kv::NoiseStudy st =
                    kv::noise_study(s, part, x.model, x.cost, x.network, x.noise_factor, x.noise_trials, x.seed);
                rows.push_back({strategy_name(s), dashed(part), C, p, st.quiet_ttft, st.mean_degradation,
                                st.max_degradation});
                (s == kv::Strategy::TSP ? tsp_mean : kvr_mean) = st.mean_degradation;
            }
            if (tsp_mean && kvr_mean) {
                const char* v = *kvr_mean < *tsp_mean ? "KVR more robust" : (*kvr_mean > *tsp_mean ? "TSP more robust" : "tie");
                verdicts.push_back("C=" + std::to_string(C) + " p=" + std::to_string(p) + ": " + v);
            }
        }
    }
    Sink sink(x.out_path);
    if (x.format == "json") {
        json doc = json::array();
        for (const auto& r : rows)
            doc.push_back({{"strategy", r.strategy}, {"C", r.C}, {"p", r.p}, {"partition", r.partition},
                           {"slowdown_factor", x.noise_factor}, {"trials", x.noise_trials}, {"quiet_ttft", r.quiet},
                           {"mean_degradation", r.mean}, {"max_degradation", r.max}});
        sink.os() << doc.dump(2) << "\n";
    } else {
        sink.os() << "strategy,C,p,partition,slowdown_factor,trials,quiet_ttft,mean_degradation,max_degradation\n";
        for (const auto& r : rows)
            sink.os() << r.strategy << "," << r.C << "," << r.p << "," << r.partition << "," << g10(x.noise_factor)
                      << "," << x.noise_trials << "," << g10(r.quiet) << "," << g10(r.mean) << "," << g10(r.max) << "\n";
    }
    // commentary stays off stdout while the table streams there
    std::ostream& note = x.out_path.empty() ? std::cerr : std::cout;
    for (const auto& v : verdicts) note << "verdict: " << v << "\n";
    return 0;
}

// ------------------------------------------------------------------ main
const char* kUsage =
    "usage: kvprefill_b200 <verify|sweep|search|predict C|noise> [--config FILE] [--seed N] [--out FILE]\n"
    "                      [--table FILE] [--format csv|json] [--measure (sweep)]\n";

struct Args {
    std::string sub, config, out, table, format;
    int64_t seed = -1, predict_c = -1;
    bool measure = false;
};

bool parse_args(int argc, char** argv, Args& a) {
    if (argc < 2) return false;
    a.sub = argv[1];
    if (a.sub != "verify" && a.sub != "sweep" && a.sub != "search" && a.sub != "predict" && a.sub != "noise")
        return false;
    for (int i = 2; i < argc; ++i) {
        const std::string f = argv[i];
        auto value = [&](std::string& dst) {
            if (i + 1 >= argc) return false;
            dst = argv[++i];
            return true;
        };
        std::string v;
        if (f == "--config") {
            if (!value(a.config)) return false;
        } else if (f == "--out") {
            if (!value(a.out)) return false;
        } else if (f == "--table") {
            if (!value(a.table)) return false;
        } else if (f == "--format") {
            if (!value(a.format)) return false;
        } else if (f == "--seed") {
            if (!value(v)) return false;
            char* end = nullptr;
            a.seed = std::strtoll(v.c_str(), &end, 10);
            if (*end) return false;
        } else if (f == "--measure" && a.sub == "sweep") {
            a.measure = true;
        } else if (a.sub == "predict" && a.predict_c < 0 && !f.empty() && f[0] != '-') {
            char* end = nullptr;
            a.predict_c = std::strtoll(f.c_str(), &end, 10);
            if (*end) return false;
        } else {
            return false;
        }
    }
    return a.sub != "predict" || a.predict_c >= 0;
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    if (!parse_args(argc, argv, a)) {
        std::cerr << kUsage;
        return 2;
    }
    try {
        Experiment x;
        if (!a.config.empty()) {
            std::ifstream in(a.config);
            if (!in) throw kv::ConfigError("cannot open config file: " + a.config);
            std::ostringstream text;
            text << in.rdbuf();
            x = parse_experiment(text.str());
        }
        if (a.seed >= 0) x.seed = static_cast<uint64_t>(a.seed);
        if (!a.out.empty()) x.out_path = a.out;
        if (!a.table.empty()) x.table_path = a.table;
        if (!a.format.empty()) {
            if (a.format != "csv" && a.format != "json") throw kv::ConfigError("format must be csv or json");
            x.format = a.format;
        }
        if (a.sub == "verify") return cmd_verify(x);
        if (a.sub == "sweep") return cmd_sweep(x, a.measure);
        if (a.sub == "search") return cmd_search(x);
        if (a.sub == "predict") return cmd_predict(x, a.predict_c);
        return cmd_noise(x);
    } catch (const kv::ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return 2;
    } catch (const kv::Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "unexpected error: " << e.what() << "\n";
        return 1;
    }
}
