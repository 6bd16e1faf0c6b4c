// plan.cpp -- partition plan + context-level load balancer (host C++), C-ABI exported.
//
// Reference: partition.hpp (ContextPartition, even_partition, partition_from_ratios,
// SearchOffsets), search.hpp (SearchConfig, BestTracker, binary_search_two,
// hierarchical_grid_search), simnet.hpp (CostModel, NetworkModel, simulate_ttft, ttft_star,
// practical_bound, calibrate_alpha), engine.hpp:95-121 (dot_product_counts, traffic_pairs).
// Bit-exact parity is a requirement: the arithmetic below keeps the
// reference's operand order, the 80-bit long double share computation and the tie-breaks,
// so the same inputs give the same partitions, TTFTs, evaluation and level counts.  New
// here: kvp_fit_cost_model, which calibrates the balancer from measured B200 layer times.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "../../include/kvp_b200.h"
#include "status.hpp"

namespace kvp {

using Bounds = std::vector<int64_t>;

static void check_partition(int64_t C, const int64_t* b, int64_t p) {
    if (p < 1 || b == nullptr || b[0] != 0 || b[p] != C)
        throw Error(KVP_ERR_PARTITION, "boundaries must run from 0 to the context length");
    for (int64_t i = 0; i < p; ++i)
        if (b[i] >= b[i + 1]) throw Error(KVP_ERR_PARTITION, "partition sizes must be at least 1");
}

static Bounds bounds_from_sizes(const std::vector<int64_t>& sizes) {
    Bounds b(sizes.size() + 1, 0);
    std::partial_sum(sizes.begin(), sizes.end(), b.begin() + 1);
    check_partition(b.back(), b.data(), static_cast<int64_t>(sizes.size()));
    return b;
}

Bounds even_split(int64_t C, int64_t p) {
    if (p < 1) throw Error(KVP_ERR_PARTITION, "process count must be at least 1");
    if (C < p) throw Error(KVP_ERR_PARTITION, "cannot split " + std::to_string(C) + " tokens over " +
                                                  std::to_string(p) + " workers");
    std::vector<int64_t> sizes(static_cast<size_t>(p));
    for (int64_t i = 0; i < p; ++i) sizes[static_cast<size_t>(i)] = C / p + (i < C % p ? 1 : 0);
    return bounds_from_sizes(sizes);
}

Bounds ratio_split(int64_t C, const double* ratios, int64_t p) {
    if (p < 1) throw Error(KVP_ERR_PARTITION, "ratio vector must be non-empty");
    if (C < p) throw Error(KVP_ERR_PARTITION, "context shorter than the ratio vector");
    long double total = 0;
    for (int64_t i = 0; i < p; ++i) {
        if (!(ratios[i] > 0)) throw Error(KVP_ERR_PARTITION, "ratios must be positive");
        total += static_cast<long double>(ratios[i]);
    }
    if (std::fabs(static_cast<double>(total) - 1.0) > 1e-6) throw Error(KVP_ERR_PARTITION, "ratios must sum to 1");
    std::vector<int64_t> sizes(static_cast<size_t>(p));
    std::vector<long double> rem(static_cast<size_t>(p));
    int64_t used = 0;
    for (int64_t i = 0; i < p; ++i) {
        const long double exact = static_cast<long double>(C) * static_cast<long double>(ratios[i]) / total;
        const int64_t fl = static_cast<int64_t>(std::floor(exact));
        sizes[static_cast<size_t>(i)] = fl;
        rem[static_cast<size_t>(i)] = exact - static_cast<long double>(fl);
        used += fl;
    }
    std::vector<int64_t> rank(static_cast<size_t>(p));
    std::iota(rank.begin(), rank.end(), 0);
    std::stable_sort(rank.begin(), rank.end(),
                     [&](int64_t x, int64_t y) { return rem[static_cast<size_t>(x)] > rem[static_cast<size_t>(y)]; });
    for (int64_t k = 0, left = C - used; k < left; ++k) sizes[static_cast<size_t>(rank[static_cast<size_t>(k % p)])]++;
    for (auto& s : sizes) {
        while (s < 1) {
            auto big = std::max_element(sizes.begin(), sizes.end());
            if (*big <= 1) throw Error(KVP_ERR_PARTITION, "cannot enforce minimum slice size");
            --*big;
            ++s;
        }
    }
    return bounds_from_sizes(sizes);
}

// ---------------------------------------------------------------- simulator
static void check_cost(const kvp_cost_model& c) {
    if (!(c.alpha > 0)) throw Error(KVP_ERR_CONFIG, "cost.alpha must be positive");
    if (c.proj_coeff < 0 || c.softmax_coeff < 0 || c.fixed_overhead < 0)
        throw Error(KVP_ERR_CONFIG, "cost coefficients must be non-negative");
}

static void check_net(const kvp_network_model& n) {
    if (!(n.bandwidth > 0)) throw Error(KVP_ERR_CONFIG, "network.bandwidth must be positive");
    if (n.latency < 0) throw Error(KVP_ERR_CONFIG, "network.latency must be non-negative");
}

static double wire_seconds(double pairs, double bw, double lat) { return pairs <= 0 ? 0.0 : lat + pairs / bw; }

// NoiseSidecar (simnet.hpp:65-78): per layer one adjacent link, drawn from (seed, layer) only,
// runs at bandwidth / factor.
struct Noise {
    bool on = false;
    uint64_t seed = 1;
    double factor = 1.0;
    bool causal = false;  // extension: price attention on causal-visible pairs (B200 kernels)
};

static uint64_t sm_next(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static uint64_t mix(uint64_t base, uint64_t a, uint64_t b) {
    uint64_t g = base;
    uint64_t h = sm_next(g) ^ (a * 0xd1342543de82ef95ULL);
    return sm_next(h) ^ (b * 0xaf251af3b0f025b5ULL);
}

static double link_bw(const kvp_network_model& net, const Noise& nz, int64_t layer, int64_t link, int64_t links) {
    if (nz.on && nz.factor > 1.0 && links >= 1) {
        uint64_t st = mix(nz.seed, 0x6e6fu, static_cast<uint64_t>(layer));
        if (static_cast<int64_t>(sm_next(st) % static_cast<uint64_t>(links)) == link) return net.bandwidth / nz.factor;
    }
    return net.bandwidth;
}

double simulate(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t L, const kvp_cost_model& cost,
                const kvp_network_model& net, const Noise& nz = Noise{}) {
    check_partition(C, b, p);
    check_cost(cost);
    check_net(net);
    if (strategy == KVP_SERIAL && p != 1) throw Error(KVP_ERR_INPUT, "serial strategy requires p == 1");
    std::vector<double> t(static_cast<size_t>(p), 0.0);
    std::vector<double> proj(static_cast<size_t>(p), 0.0);
    for (int64_t layer = 0; layer < L; ++layer) {
        if (strategy == KVP_TSP) {
            for (int64_t i = 0; i < p; ++i)
                proj[static_cast<size_t>(i)] = t[static_cast<size_t>(i)] + cost.proj_coeff * static_cast<double>(b[i + 1] - b[i]);
            const double gather = *std::max_element(proj.begin(), proj.end());
            const double rounds = std::ceil(std::log2(static_cast<double>(std::max<int64_t>(p, 1))));
            double worst = 0.0;
            for (int64_t k = 0; k + 1 < p; ++k) {
                const double share = static_cast<double>(std::max(b[k + 1], C - b[k + 1]));
                worst = std::max(worst, net.latency + share / link_bw(net, nz, layer, k, p - 1));
            }
            const double released = gather + rounds * worst;
            for (int64_t i = 0; i < p; ++i) {
                const int64_t c = b[i + 1] - b[i];
                const double pairs = nz.causal ? static_cast<double>(b[i]) + 0.5 * static_cast<double>(c + 1)
                                               : static_cast<double>(C);
                const double attn = cost.alpha * static_cast<double>(c) * pairs;
                t[static_cast<size_t>(i)] = released + attn + cost.softmax_coeff * static_cast<double>(c) + cost.fixed_overhead;
            }
        } else {
            double up_start = 0.0, up_wire = 0.0;
            for (int64_t i = 0; i < p; ++i) {
                const int64_t c = b[i + 1] - b[i], held = b[i + 1];
                const double pe = t[static_cast<size_t>(i)] + cost.proj_coeff * static_cast<double>(c);
                const double ready = i > 0 ? std::max(pe, up_start + up_wire) : pe;
                double sent = -std::numeric_limits<double>::infinity();
                if (i + 1 < p) {
                    const double w = wire_seconds(static_cast<double>(held), link_bw(net, nz, layer, i, p - 1), net.latency);
                    sent = ready + w;
                    up_start = ready;
                    up_wire = w;
                }
                const double pairs = nz.causal ? static_cast<double>(b[i]) + 0.5 * static_cast<double>(c + 1)
                                               : static_cast<double>(held);
                const double attn_end = ready + cost.alpha * static_cast<double>(c) * pairs;
                double end = attn_end + cost.softmax_coeff * static_cast<double>(c) + cost.fixed_overhead;
                if (i + 1 < p) end = std::max(end, sent);
                t[static_cast<size_t>(i)] = end;
            }
        }
    }
    return *std::max_element(t.begin(), t.end());
}

// ---------------------------------------------------------------- search
struct Incumbent {
    const Bounds* even = nullptr;
    bool set = false;
    Bounds part;
    double ttft = std::numeric_limits<double>::infinity();

    static int64_t dist(const Bounds& a, const Bounds& e) {
        int64_t d = 0;
        for (size_t i = 0; i < a.size(); ++i) d += std::llabs(a[i] - e[i]);
        return d;
    }
    void offer(const Bounds& cand, double v) {
        if (!set) {
            set = true;
            part = cand;
            ttft = v;
            return;
        }
        if (v > ttft) return;
        if (v < ttft) {
            part = cand;
            ttft = v;
            return;
        }
        const int64_t dn = dist(cand, *even), dc = dist(part, *even);
        if (dn < dc || (dn == dc && cand < part)) part = cand;
    }
};

static void check_search(const kvp_search_config& s, kvp_evaluator ev) {
    if (s.grid_width < 3) throw Error(KVP_ERR_SEARCH, "grid_width must be at least 3");
    if (s.min_stride < 1) throw Error(KVP_ERR_SEARCH, "min_stride must be at least 1");
    if (s.initial_stride != 0 && s.initial_stride < s.min_stride)
        throw Error(KVP_ERR_SEARCH, "initial_stride must be at least min_stride");
    if (!ev) throw Error(KVP_ERR_SEARCH, "search requires an evaluator");
}

static int64_t first_stride(const kvp_search_config& s, int64_t C, int64_t p) {
    if (s.initial_stride > 0) return s.initial_stride;
    const double target = static_cast<double>(C) / (4.0 * static_cast<double>(p));
    int64_t st = 1;
    while (static_cast<double>(st) < target) st *= 2;
    return std::max(st, s.min_stride);
}

Bounds grid_search(int64_t C, int64_t p, const kvp_search_config& s, kvp_evaluator ev, void* user,
                   kvp_search_result* res) {
    check_search(s, ev);
    if (p < 2) throw Error(KVP_ERR_SEARCH, "hierarchical_grid_search requires p >= 2");
    const Bounds even = even_split(C, p);
    res->evaluations = 0;
    res->levels = 0;
    Incumbent best;
    best.even = &even;
    best.offer(even, ev(even.data(), p, user));
    res->evaluations++;
    const int64_t axes = p - 1, half = s.grid_width / 2;
    int64_t stride = first_stride(s, C, p);
    std::vector<int64_t> odo(static_cast<size_t>(axes));
    Bounds cand(static_cast<size_t>(p + 1));
    for (;;) {
        res->levels++;
        const Bounds center = best.part;
        Incumbent level;
        level.even = &even;
        std::fill(odo.begin(), odo.end(), 0);
        bool any = false;
        for (;;) {
            cand = center;
            for (int64_t a = 0; a < axes; ++a) cand[static_cast<size_t>(a + 1)] += (odo[static_cast<size_t>(a)] - half) * stride;
            bool feasible = true;
            for (int64_t i = 0; i < p && feasible; ++i) feasible = cand[static_cast<size_t>(i)] < cand[static_cast<size_t>(i + 1)];
            if (feasible) {
                level.offer(cand, ev(cand.data(), p, user));
                res->evaluations++;
                any = true;
            }
            int64_t a = axes - 1;
            while (a >= 0 && ++odo[static_cast<size_t>(a)] == s.grid_width) odo[static_cast<size_t>(a--)] = 0;
            if (a < 0) break;
        }
        if (!any) throw Error(KVP_ERR_SEARCH, "all grid points infeasible");
        best.offer(level.part, level.ttft);
        if (stride == s.min_stride) break;
        stride = std::max(s.min_stride, stride / 2);
    }
    res->ttft = best.ttft;
    return best.part;
}

Bounds bisect_two(int64_t C, const kvp_search_config& s, kvp_evaluator ev, void* user, kvp_search_result* res) {
    check_search(s, ev);
    if (C < 2) throw Error(KVP_ERR_SEARCH, "binary_search_two requires C >= 2");
    const Bounds even = even_split(C, 2);
    const int64_t mid = even[1], step = s.min_stride;
    const int64_t lo_u = -((mid - 1) / step), hi_u = (C - 1 - mid) / step;
    res->evaluations = 0;
    std::unordered_map<int64_t, double> memo;
    auto at = [&](int64_t u) {
        auto it = memo.find(u);
        if (it != memo.end()) return it->second;
        const Bounds part{0, mid + u * step, C};
        const double v = ev(part.data(), 2, user);
        res->evaluations++;
        memo.emplace(u, v);
        return v;
    };
    int64_t lo = lo_u, hi = hi_u;
    while (hi - lo > 8) {
        const int64_t m1 = lo + (hi - lo) / 3, m2 = hi - (hi - lo) / 3;
        if (at(m1) < at(m2))
            hi = m2;
        else
            lo = m1;
    }
    int64_t pick = 0;
    double best = std::numeric_limits<double>::infinity();
    for (int64_t u = lo; u <= hi; ++u) {
        const double v = at(u);
        const bool nearer = std::llabs(u) < std::llabs(pick) || (std::llabs(u) == std::llabs(pick) && u > pick);
        if (v < best || (v == best && nearer)) {
            best = v;
            pick = u;
        }
    }
    if (lo_u <= 0 && 0 <= hi_u && at(0) <= best) {
        best = at(0);
        pick = 0;
    }
    res->ttft = best;
    res->levels = 1;
    return Bounds{0, mid + pick * step, C};
}

struct SimUser {
    int64_t L;
    kvp_cost_model cost;
    kvp_network_model net;
    bool causal = false;
};

static double sim_eval(const int64_t* b, int64_t p, void* u) {
    const SimUser* s = static_cast<const SimUser*>(u);
    Noise nz;
    nz.causal = s->causal;
    return simulate(KVP_KVR, b[p], b, p, s->L, s->cost, s->net, nz);
}

// Least squares with non-negativity by active-set elimination over <= 3 unknowns.
static void nnls_small(const std::vector<std::vector<double>>& X, const std::vector<double>& y, std::vector<double>& w) {
    const size_t k = X.empty() ? 0 : X[0].size();
    std::vector<bool> active(k, true);
    for (int iter = 0; iter < 8; ++iter) {
        std::vector<size_t> idx;
        for (size_t j = 0; j < k; ++j)
            if (active[j]) idx.push_back(j);
        const size_t m = idx.size();
        std::vector<double> A(m * m, 0.0), rhs(m, 0.0);
        for (size_t r = 0; r < X.size(); ++r)
            for (size_t a = 0; a < m; ++a) {
                rhs[a] += X[r][idx[a]] * y[r];
                for (size_t bcol = 0; bcol < m; ++bcol) A[a * m + bcol] += X[r][idx[a]] * X[r][idx[bcol]];
            }
        // Gaussian elimination with partial pivoting
        std::vector<double> sol(m, 0.0);
        for (size_t c = 0; c < m; ++c) {
            size_t piv = c;
            for (size_t r = c + 1; r < m; ++r)
                if (std::fabs(A[r * m + c]) > std::fabs(A[piv * m + c])) piv = r;
            if (std::fabs(A[piv * m + c]) < 1e-300) continue;
            if (piv != c) {
                for (size_t q = 0; q < m; ++q) std::swap(A[c * m + q], A[piv * m + q]);
                std::swap(rhs[c], rhs[piv]);
            }
            for (size_t r = c + 1; r < m; ++r) {
                const double f = A[r * m + c] / A[c * m + c];
                for (size_t q = c; q < m; ++q) A[r * m + q] -= f * A[c * m + q];
                rhs[r] -= f * rhs[c];
            }
        }
        for (size_t c = m; c-- > 0;) {
            if (std::fabs(A[c * m + c]) < 1e-300) continue;
            double acc = rhs[c];
            for (size_t q = c + 1; q < m; ++q) acc -= A[c * m + q] * sol[q];
            sol[c] = acc / A[c * m + c];
        }
        w.assign(k, 0.0);
        bool neg = false;
        for (size_t a = 0; a < m; ++a) {
            if (sol[a] < 0) {
                active[idx[a]] = false;
                neg = true;
            } else {
                w[idx[a]] = sol[a];
            }
        }
        if (!neg) return;
    }
}

}  // namespace kvp

using namespace kvp;

extern "C" {

kvp_status kvp_validate_partition(int64_t C, const int64_t* b, int64_t p) {
    return guard([&] { check_partition(C, b, p); });
}

kvp_status kvp_even_partition(int64_t C, int64_t p, int64_t* out) {
    return guard([&] {
        const Bounds b = even_split(C, p);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_partition_from_ratios(int64_t C, const double* ratios, int64_t p, int64_t* out) {
    return guard([&] {
        const Bounds b = ratio_split(C, ratios, p);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_dot_product_counts(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t* out) {
    return guard([&] {
        check_partition(C, b, p);
        if (strategy == KVP_SERIAL && p != 1) throw Error(KVP_ERR_INPUT, "serial strategy requires a single-worker partition");
        for (int64_t i = 0; i < p; ++i) out[i] = (b[i + 1] - b[i]) * (strategy == KVP_KVR ? b[i + 1] : C);
    });
}

kvp_status kvp_traffic_pairs(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t* out) {
    return guard([&] {
        check_partition(C, b, p);
        int64_t total = 0;
        if (strategy == KVP_TSP) total = (p - 1) * C;
        if (strategy == KVP_KVR)
            for (int64_t i = 0; i + 1 < p; ++i) total += b[i + 1];
        *out = total;
    });
}

kvp_status kvp_simulate_ttft(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t L,
                             const kvp_cost_model* cost, const kvp_network_model* net, double* out) {
    return guard([&] { *out = simulate(strategy, C, b, p, L, *cost, *net); });
}

kvp_status kvp_ttft_star(int64_t C, int64_t p, double alpha, double* out) {
    return guard([&] {
        if (p < 1) throw Error(KVP_ERR_INPUT, "ttft_star requires p >= 1");
        const double pd = static_cast<double>(p), Cd = static_cast<double>(C);
        *out = alpha * Cd * Cd / 2.0 * (1.0 / pd + 1.0 / (pd * pd));
    });
}

kvp_status kvp_calibrate_alpha(const int64_t* Cs, const double* ts, int64_t n, double* out) {
    return guard([&] {
        if (n < 1) throw Error(KVP_ERR_CALIBRATION, "no measurements to fit");
        double num = 0, den = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (Cs[i] <= 0) throw Error(KVP_ERR_CALIBRATION, "context lengths must be positive");
            const double c2 = static_cast<double>(Cs[i]) * static_cast<double>(Cs[i]);
            num += ts[i] * c2;
            den += c2 * c2;
        }
        *out = num / den;
    });
}

kvp_status kvp_hierarchical_grid_search(int64_t C, int64_t p, const kvp_search_config* cfg, kvp_evaluator ev,
                                        void* user, int64_t* out, kvp_search_result* res) {
    return guard([&] {
        const Bounds b = grid_search(C, p, *cfg, ev, user, res);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_binary_search_two(int64_t C, const kvp_search_config* cfg, kvp_evaluator ev, void* user,
                                 int64_t* out, kvp_search_result* res) {
    return guard([&] {
        const Bounds b = bisect_two(C, *cfg, ev, user, res);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_search_partition(int64_t C, int64_t p, int64_t L, const kvp_cost_model* cost,
                                const kvp_network_model* net, const kvp_search_config* cfg, int64_t* out,
                                kvp_search_result* res) {
    return guard([&] {
        if (p == 1) {  // every source degenerates to [C] (commands.hpp:255)
            const Bounds b = even_split(C, 1);
            std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
            res->ttft = simulate(KVP_SERIAL, C, b.data(), 1, L, *cost, *net);
            res->evaluations = 1;
            res->levels = 0;
            return;
        }
        SimUser u{L, *cost, *net};
        const Bounds b = grid_search(C, p, *cfg, sim_eval, &u, res);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_practical_bound(int64_t C, int64_t p, int64_t L, const kvp_cost_model* cost, int64_t* out,
                               double* ttft) {
    return guard([&] {
        if (p < 1) throw Error(KVP_ERR_INPUT, "practical bound requires p >= 1");
        const kvp_network_model quiet{std::numeric_limits<double>::infinity(), 0.0};
        if (p == 1) {
            const Bounds b = even_split(C, 1);
            std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
            *ttft = simulate(KVP_SERIAL, C, b.data(), 1, L, *cost, quiet);
            return;
        }
        SimUser u{L, *cost, quiet};
        kvp_search_config cfg{5, 0, 1};
        kvp_search_result r{};
        const Bounds b = grid_search(C, p, cfg, sim_eval, &u, &r);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
        *ttft = r.ttft;
    });
}

kvp_status kvp_simulate_ttft_causal(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t L,
                                    const kvp_cost_model* cost, const kvp_network_model* net, double* out) {
    return guard([&] {
        Noise nz;
        nz.causal = true;
        *out = simulate(strategy, C, b, p, L, *cost, *net, nz);
    });
}

kvp_status kvp_search_partition_causal(int64_t C, int64_t p, int64_t L, const kvp_cost_model* cost,
                                       const kvp_network_model* net, const kvp_search_config* cfg, int64_t* out,
                                       kvp_search_result* res) {
    return guard([&] {
        Noise nz;
        nz.causal = true;
        if (p == 1) {
            const Bounds b = even_split(C, 1);
            std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
            res->ttft = simulate(KVP_SERIAL, C, b.data(), 1, L, *cost, *net, nz);
            res->evaluations = 1;
            res->levels = 0;
            return;
        }
        SimUser u{L, *cost, *net, true};
        const Bounds b = grid_search(C, p, *cfg, sim_eval, &u, res);
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_simulate_ttft_noisy(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t L,
                                   const kvp_cost_model* cost, const kvp_network_model* net, uint64_t noise_seed,
                                   double factor, double* out) {
    return guard([&] {
        Noise nz;
        nz.on = true;
        nz.seed = noise_seed;
        nz.factor = factor;
        *out = simulate(strategy, C, b, p, L, *cost, *net, nz);
    });
}

kvp_status kvp_noise_study(int32_t strategy, int64_t C, const int64_t* b, int64_t p, int64_t L,
                           const kvp_cost_model* cost, const kvp_network_model* net, double factor, int64_t trials,
                           uint64_t seed, double* quiet, double* mean, double* mx, double* per_trial) {
    return guard([&] {
        if (trials < 1) throw Error(KVP_ERR_INPUT, "noise_study requires trials >= 1");
        if (!(factor >= 1.0)) throw Error(KVP_ERR_CONFIG, "slowdown_factor must be >= 1");
        const double q = simulate(strategy, C, b, p, L, *cost, *net);
        double sum = 0.0, worst = 0.0;
        for (int64_t t = 0; t < trials; ++t) {
            Noise nz;
            nz.on = true;
            nz.seed = mix(seed, 0x7472u, static_cast<uint64_t>(t));
            nz.factor = factor;
            const double d = (simulate(strategy, C, b, p, L, *cost, *net, nz) - q) / q;
            if (per_trial) per_trial[t] = d;
            sum += d;
            worst = std::max(worst, d);
        }
        *quiet = q;
        *mean = sum / static_cast<double>(trials);
        *mx = worst;
    });
}

kvp_status kvp_noise_degraded_link(uint64_t sidecar_seed, int64_t layer, int64_t link_count, int64_t* link_out) {
    return guard([&] {
        if (!link_out) throw Error(KVP_ERR_INPUT, "null argument");
        if (link_count < 1) {
            *link_out = -1;
            return;
        }
        uint64_t st = mix(sidecar_seed, 0x6e6fu, static_cast<uint64_t>(layer));
        *link_out = static_cast<int64_t>(sm_next(st) % static_cast<uint64_t>(link_count));
    });
}

kvp_status kvp_noise_trial_seed(uint64_t study_seed, int64_t trial, uint64_t* sidecar_seed_out) {
    return guard([&] {
        if (!sidecar_seed_out) throw Error(KVP_ERR_INPUT, "null argument");
        *sidecar_seed_out = mix(study_seed, 0x7472u, static_cast<uint64_t>(trial));
    });
}

// PartitionLookupTable::insert validation (lookup_table.hpp:26-38) + interpolate_partition.
static std::vector<double> interpolate(const int64_t* Cs, const double* ratios, int64_t n, int64_t p, int64_t C) {
    if (p < 1) throw Error(KVP_ERR_LOOKUP, "table process count not set");
    std::map<int64_t, std::vector<double>> entries;
    for (int64_t i = 0; i < n; ++i) {
        std::vector<double> r(ratios + i * p, ratios + (i + 1) * p);
        double sum = 0;
        for (double x : r) {
            if (x < 0) throw Error(KVP_ERR_LOOKUP, "table ratios must be non-negative");
            sum += x;
        }
        if (std::abs(sum - 1.0) > 1e-9) throw Error(KVP_ERR_LOOKUP, "table ratios must sum to 1");
        if (Cs[i] < 1) throw Error(KVP_ERR_LOOKUP, "context length must be positive");
        entries[Cs[i]] = std::move(r);
    }
    if (entries.empty()) throw Error(KVP_ERR_LOOKUP, "lookup table is empty");
    const auto hit = entries.find(C);
    if (hit != entries.end()) return hit->second;
    const auto hi = entries.upper_bound(C);
    if (hi == entries.begin()) return hi->second;          // below range: clamp
    if (hi == entries.end()) return std::prev(hi)->second;  // above range: clamp
    const auto lo = std::prev(hi);
    const double t = static_cast<double>(C - lo->first) / static_cast<double>(hi->first - lo->first);
    std::vector<double> out(lo->second.size());
    double sum = 0;
    for (size_t i = 0; i < out.size(); ++i) {
        out[i] = (1.0 - t) * lo->second[i] + t * hi->second[i];
        sum += out[i];
    }
    for (double& r : out) r /= sum;
    return out;
}

kvp_status kvp_interpolate_partition(const int64_t* Cs, const double* ratios, int64_t n, int64_t p, int64_t C,
                                     double* out) {
    return guard([&] {
        const auto r = interpolate(Cs, ratios, n, p, C);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

kvp_status kvp_partition_from_table(const int64_t* Cs, const double* ratios, int64_t n, int64_t p, int64_t C,
                                    int64_t* out) {
    return guard([&] {
        const auto r = interpolate(Cs, ratios, n, p, C);
        const Bounds b = ratio_split(C, r.data(), static_cast<int64_t>(r.size()));
        std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

kvp_status kvp_fit_cost_model(const int64_t* local_rows, const int64_t* held_rows, const double* proj_s,
                              const double* rest_s, int64_t n, kvp_cost_model* out) {
    return guard([&] {
        if (n < 1) throw Error(KVP_ERR_CALIBRATION, "no measurements to fit");
        // proj_s ~ a * c  (through the origin)
        double num = 0, den = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (local_rows[i] <= 0 || held_rows[i] < local_rows[i])
                throw Error(KVP_ERR_CALIBRATION, "samples need 0 < local_rows <= held_rows");
            num += proj_s[i] * static_cast<double>(local_rows[i]);
            den += static_cast<double>(local_rows[i]) * static_cast<double>(local_rows[i]);
        }
        // rest_s ~ alpha * c * held + s * c + f
        std::vector<std::vector<double>> X;
        std::vector<double> y;
        for (int64_t i = 0; i < n; ++i) {
            const double c = static_cast<double>(local_rows[i]), h = static_cast<double>(held_rows[i]);
            X.push_back({c * h, c, 1.0});
            y.push_back(rest_s[i]);
        }
        std::vector<double> w;
        nnls_small(X, y, w);
        out->proj_coeff = num / den;
        out->alpha = w[0] > 0 ? w[0] : 1e-300;
        out->softmax_coeff = w[1];
        out->fixed_overhead = w[2];
    });
}

}  // extern "C"

// random_context<float> (weights.hpp:86-89) on the host: stream mix_seed(seed, 0xc7, 17),
// value = float((2u - 1) * 1.0) in double, row-major fill (weights.hpp:41-47).
kvp_status kvp_random_context(int64_t rows, int64_t d_model, uint64_t seed, float* out) {
    return kvp::guard([&] {
        if (rows < 0 || d_model < 0) throw kvp::Error(KVP_ERR_DIMENSION, "matrix dimensions must be non-negative");
        if (!out && rows * d_model > 0) throw kvp::Error(KVP_ERR_INPUT, "null output");
        auto next = [](uint64_t& st) {
            uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            return z ^ (z >> 31);
        };
        uint64_t g = seed;  // mix_seed (rng.hpp:28-37)
        uint64_t h = next(g) ^ (0xc7ULL * 0xd1342543de82ef95ULL);
        uint64_t st = next(h) ^ (17ULL * 0xaf251af3b0f025b5ULL);
        for (int64_t i = 0; i < rows * d_model; ++i) {
            const double u = static_cast<double>(next(st) >> 11) * 0x1.0p-53;
            out[i] = static_cast<float>((2.0 * u - 1.0) * 1.0);
        }
    });
}
