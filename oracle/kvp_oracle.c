/*
 * kvp_oracle.c -- CPU restatement of the kvprefill reference (see kvp_oracle.h).
 * TEST INFRASTRUCTURE ONLY: the checker for the B200 product, never part of it.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -march, matching the
 * reference's Release build so f32/f64 rounding sequences are identical).
 */
#include "kvp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp:10-37 */
uint64_t kvo_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t kvo_mix_seed(uint64_t base, uint64_t a, uint64_t b) {
    uint64_t g = base;
    uint64_t s = kvo_splitmix_next(&g) ^ (a * 0xd1342543de82ef95ULL);
    uint64_t h = s;
    return kvo_splitmix_next(&h) ^ (b * 0xaf251af3b0f025b5ULL);
}

/* --------------------------------------------------------------- config.hpp:36-46 */
int kvo_validate_config(const kvo_config* c) {
    if (c->d_model <= 0 || c->n_heads <= 0 || c->n_kv_heads <= 0 || c->n_layers <= 0)
        return KVO_CONFIG;
    if (c->d_model % c->n_heads != 0) return KVO_CONFIG;
    if (c->n_heads % c->n_kv_heads != 0) return KVO_CONFIG;
    return KVO_OK;
}

/* ------------------------------------------------------- model core, both precisions */
#define REAL float
#define SFX f32
#define EXPF expf
#define SQRTF sqrtf
#define PENALTY (-1e9f)
#include "kvp_oracle_model.inc"
#undef REAL
#undef SFX
#undef EXPF
#undef SQRTF
#undef PENALTY

#define REAL double
#define SFX f64
#define EXPF exp
#define SQRTF sqrt
#define PENALTY (-1e18)
#include "kvp_oracle_model.inc"
#undef REAL
#undef SFX
#undef EXPF
#undef SQRTF
#undef PENALTY

void kvo_seeded_matrix_f32(float* out, int64_t rows, int64_t cols, double scale, uint64_t stream) {
    seeded_f32(out, rows, cols, scale, stream);
}

/* oracle.hpp:34-111 naive_causal_forward: f64, masked terms excluded, no max
 * subtraction, reverse-order accumulation. */
static void slow_mm(const double* a, int64_t rows, int64_t inner, const double* b, int64_t cols,
                    double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
            double acc = 0;
            for (int64_t k = inner - 1; k >= 0; --k) acc += a[i * inner + k] * b[k * cols + j];
            out[i * cols + j] = acc;
        }
}

static void slow_norm(const kvo_config* c, const double* x, int64_t rows, int64_t cols, double* out) {
    if (!c->rms_norm) {
        memcpy(out, x, (size_t)(rows * cols) * sizeof(double));
        return;
    }
    for (int64_t i = 0; i < rows; ++i) {
        double ms = 0;
        for (int64_t j = cols - 1; j >= 0; --j) ms += x[i * cols + j] * x[i * cols + j];
        const double inv = 1.0 / sqrt(ms / (double)cols + 1e-6);
        for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = x[i * cols + j] * inv;
    }
}

int kvo_naive_forward_f64(const kvo_config* c, const double* const* w, const double* context,
                          int64_t C, double* hidden_out) {
    int st = kvo_validate_config(c);
    if (st) return st;
    if (C < 1) return KVO_INPUT;
    const int64_t d = c->d_model, hd = d / c->n_heads, q = c->n_heads * hd, kv = c->n_kv_heads * hd;
    const int64_t group = c->n_heads / c->n_kv_heads;
    double* h = (double*)malloc((size_t)(C * d) * sizeof(double));
    double* x = (double*)malloc((size_t)(C * d) * sizeof(double));
    double* Q = (double*)malloc((size_t)(C * q) * sizeof(double));
    double* K = (double*)malloc((size_t)(C * kv) * sizeof(double));
    double* V = (double*)malloc((size_t)(C * kv) * sizeof(double));
    double* A = (double*)malloc((size_t)(C * q) * sizeof(double));
    double* t = (double*)malloc((size_t)(C * 2 * d) * sizeof(double));
    double* t2 = (double*)malloc((size_t)(C * d) * sizeof(double));
    double* h1 = (double*)malloc((size_t)(C * d) * sizeof(double));
    double* wr = (double*)malloc((size_t)(C + 1) * sizeof(double));
    memcpy(h, context, (size_t)(C * d) * sizeof(double));
    const double scale = 1.0 / sqrt((double)hd);
    for (int64_t l = 0; l < c->n_layers; ++l) {
        const double* const* lw = w + 6 * l;
        slow_norm(c, h, C, d, x);
        slow_mm(x, C, d, lw[0], q, Q);
        slow_mm(x, C, d, lw[1], kv, K);
        slow_mm(x, C, d, lw[2], kv, V);
        for (int64_t head = 0; head < c->n_heads; ++head) {
            const int64_t qo = head * hd, ko = (head / group) * hd;
            for (int64_t i = 0; i < C; ++i) {
                double total = 0;
                for (int64_t j = i; j >= 0; --j) {
                    double s = 0;
                    for (int64_t dd = hd - 1; dd >= 0; --dd) s += Q[i * q + qo + dd] * K[j * kv + ko + dd];
                    wr[j] = exp(s * scale);
                    total += wr[j];
                }
                for (int64_t dd = 0; dd < hd; ++dd) {
                    double acc = 0;
                    for (int64_t j = i; j >= 0; --j) acc += (wr[j] / total) * V[j * kv + ko + dd];
                    A[i * q + qo + dd] = acc;
                }
            }
        }
        slow_mm(A, C, q, lw[3], d, t2);
        for (int64_t i = 0; i < C * d; ++i) h1[i] = h[i] + t2[i];
        slow_norm(c, h1, C, d, x);
        slow_mm(x, C, d, lw[4], 2 * d, t);
        for (int64_t i = 0; i < C * 2 * d; ++i) t[i] = t[i] > 0 ? t[i] : 0;
        slow_mm(t, C, 2 * d, lw[5], d, t2);
        for (int64_t i = 0; i < C * d; ++i) h[i] = h1[i] + t2[i];
    }
    memcpy(hidden_out, h, (size_t)(C * d) * sizeof(double));
    free(h); free(x); free(Q); free(K); free(V); free(A); free(t); free(t2); free(h1); free(wr);
    return KVO_OK;
}

/* -------------------------------------------------------------- partition.hpp */
/* ContextPartition::validate (partition.hpp:31-37) */
int kvo_validate_partition(int64_t C, const int64_t* b, int64_t p) {
    if (p < 1 || b[0] != 0 || b[p] != C) return KVO_PARTITION;
    for (int64_t i = 0; i < p; ++i)
        if (b[i] >= b[i + 1]) return KVO_PARTITION;
    return KVO_OK;
}

static int from_sizes(const int64_t* sizes, int64_t p, int64_t* b) {
    int64_t pos = 0;
    b[0] = 0;
    for (int64_t i = 0; i < p; ++i) {
        pos += sizes[i];
        b[i + 1] = pos;
    }
    return kvo_validate_partition(pos, b, p);
}

/* even_partition (partition.hpp:59-69): remainder to the earliest workers. */
int kvo_even_partition(int64_t C, int64_t p, int64_t* b) {
    if (p < 1) return KVO_PARTITION;
    if (C < p) return KVO_PARTITION;
    int64_t* sizes = (int64_t*)malloc((size_t)p * sizeof(int64_t));
    for (int64_t i = 0; i < p; ++i) sizes[i] = C / p + (i < C % p ? 1 : 0);
    int st = from_sizes(sizes, p, b);
    free(sizes);
    return st;
}

/* partition_from_ratios (partition.hpp:76-120): long-double shares, floor, leftover to
 * the largest fractional parts (stable, lower index first), then min-1 fix-up from the
 * currently largest slice (first on ties). */
int kvo_partition_from_ratios(int64_t C, const double* ratios, int64_t p, int64_t* b) {
    if (p < 1) return KVO_PARTITION;
    if (C < p) return KVO_PARTITION;
    long double sum = 0;
    for (int64_t i = 0; i < p; ++i) {
        if (!(ratios[i] > 0)) return KVO_PARTITION;
        sum += (long double)ratios[i];
    }
    if (fabs((double)sum - 1.0) > 1e-6) return KVO_PARTITION;
    int64_t* sizes = (int64_t*)malloc((size_t)p * sizeof(int64_t));
    long double* fracs = (long double*)malloc((size_t)p * sizeof(long double));
    int64_t* order = (int64_t*)malloc((size_t)p * sizeof(int64_t));
    int64_t assigned = 0;
    for (int64_t i = 0; i < p; ++i) {
        const long double share = (long double)C * (long double)ratios[i] / sum;
        const int64_t whole = (int64_t)floorl(share);
        sizes[i] = whole;
        fracs[i] = share - (long double)whole;
        assigned += whole;
    }
    const int64_t leftover = C - assigned;
    /* stable insertion sort by fraction, descending */
    for (int64_t i = 0; i < p; ++i) {
        int64_t v = order[i] = i, j = i;
        while (j > 0 && fracs[v] > fracs[order[j - 1]]) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = v;
    }
    for (int64_t k = 0; k < leftover; ++k) sizes[order[k % p]] += 1;
    int st = KVO_OK;
    for (int64_t i = 0; i < p && st == KVO_OK; ++i) {
        while (sizes[i] < 1) {
            int64_t largest = 0;
            for (int64_t j = 1; j < p; ++j)
                if (sizes[j] > sizes[largest]) largest = j;
            if (sizes[largest] <= 1) {
                st = KVO_PARTITION;
                break;
            }
            sizes[largest] -= 1;
            sizes[i] += 1;
        }
    }
    if (st == KVO_OK) st = from_sizes(sizes, p, b);
    free(sizes);
    free(fracs);
    free(order);
    return st;
}

/* table_build_cost (partition.hpp:143-148), printed-form exponent placement. */
double kvo_table_build_cost(double T, int64_t N, int64_t C, int64_t grid_width) {
    if (N < 2 || C < 2) return -1.0;
    const double combos = pow((double)(N - 1), (double)grid_width);
    const double levels = log2((double)C) / log2((double)(grid_width - 1));
    return T * combos * levels;
}

/* ------------------------------------------------------ engine.hpp:95-121 */
int kvo_dot_product_counts(int strategy, int64_t C, const int64_t* b, int64_t p, int64_t* out) {
    int st = kvo_validate_partition(C, b, p);
    if (st) return st;
    if (strategy == KVO_SERIAL && p != 1) return KVO_INPUT;
    for (int64_t i = 0; i < p; ++i) {
        const int64_t held = (strategy == KVO_TSP || strategy == KVO_SERIAL) ? C : b[i + 1];
        out[i] = (b[i + 1] - b[i]) * held;
    }
    return KVO_OK;
}

int kvo_traffic_pairs(int strategy, int64_t C, const int64_t* b, int64_t p, int64_t* out) {
    int st = kvo_validate_partition(C, b, p);
    if (st) return st;
    if (strategy == KVO_SERIAL) {
        *out = 0;
        return KVO_OK;
    }
    if (strategy == KVO_TSP) {
        *out = (p - 1) * C;
        return KVO_OK;
    }
    int64_t total = 0;
    for (int64_t i = 0; i + 1 < p; ++i) total += b[i + 1];
    *out = total;
    return KVO_OK;
}

/* ------------------------------------------------------------ simnet.hpp */
static int validate_cost(const kvo_cost* c) {
    if (!(c->alpha > 0)) return KVO_CONFIG;
    if (c->proj_coeff < 0 || c->softmax_coeff < 0 || c->fixed_overhead < 0) return KVO_CONFIG;
    return KVO_OK;
}

static int validate_net(const kvo_net* n) {
    if (!(n->bandwidth > 0)) return KVO_CONFIG;
    if (n->latency < 0) return KVO_CONFIG;
    return KVO_OK;
}

static double transfer_seconds(double pairs, double bandwidth, double latency) {
    if (pairs <= 0) return 0.0;
    return latency + pairs / bandwidth;
}

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* simulate_ttft (simnet.hpp:164-278), quiet network (no NoiseSidecar). */
int kvo_simulate_ttft(int strategy, int64_t C, const int64_t* b, int64_t p, int64_t L,
                      const kvo_cost* cost, const kvo_net* net, double* ttft_out) {
    int st = kvo_validate_partition(C, b, p);
    if (st) return st;
    if ((st = validate_cost(cost))) return st;
    if ((st = validate_net(net))) return st;
    if (strategy == KVO_SERIAL && p != 1) return KVO_INPUT;
    double* done = (double*)calloc((size_t)p, sizeof(double));
    double* proj_end = (double*)calloc((size_t)p, sizeof(double));
    const int64_t links = p - 1;
    for (int64_t layer = 0; layer < L; ++layer) {
        if (strategy == KVO_TSP) {
            for (int64_t i = 0; i < p; ++i)
                proj_end[i] = done[i] + cost->proj_coeff * (double)(b[i + 1] - b[i]);
            double gather_start = proj_end[0];
            for (int64_t i = 1; i < p; ++i)
                if (proj_end[i] > gather_start) gather_start = proj_end[i];
            double slowest_link = 0.0;
            const double rounds = ceil(log2((double)(p > 1 ? p : 1)));
            for (int64_t link = 0; link < links; ++link) {
                const int64_t left = b[link + 1];
                const double share = (double)(left > C - left ? left : C - left);
                slowest_link = dmax(slowest_link, net->latency + share / net->bandwidth);
            }
            const double barrier_end = gather_start + rounds * slowest_link;
            for (int64_t i = 0; i < p; ++i) {
                const int64_t c_i = b[i + 1] - b[i];
                const double attn = cost->alpha * (double)c_i * (double)C;
                done[i] = barrier_end + attn + cost->softmax_coeff * (double)c_i + cost->fixed_overhead;
            }
        } else {
            double upstream_send_start = 0.0, upstream_transfer = 0.0;
            for (int64_t i = 0; i < p; ++i) {
                const int64_t c_i = b[i + 1] - b[i];
                const int64_t held = b[i + 1];
                const double pe = done[i] + cost->proj_coeff * (double)c_i;
                double cache_ready = pe;
                if (i > 0) {
                    const double recv_ready = upstream_send_start + upstream_transfer;
                    cache_ready = dmax(pe, recv_ready);
                }
                int has_send = 0;
                double send_end = 0;
                if (i + 1 < p) {
                    has_send = 1;
                    const double send_start = cache_ready;
                    const double tt = transfer_seconds((double)held, net->bandwidth, net->latency);
                    send_end = send_start + tt;
                    upstream_send_start = send_start;
                    upstream_transfer = tt;
                }
                const double attn_end = cache_ready + cost->alpha * (double)c_i * (double)held;
                double layer_end = attn_end + cost->softmax_coeff * (double)c_i + cost->fixed_overhead;
                if (has_send) layer_end = dmax(layer_end, send_end);
                done[i] = layer_end;
            }
        }
    }
    double t = done[0];
    for (int64_t i = 1; i < p; ++i)
        if (done[i] > t) t = done[i];
    *ttft_out = t;
    free(done);
    free(proj_end);
    return KVO_OK;
}

/* ttft_star (simnet.hpp:282-287) */
int kvo_ttft_star(int64_t C, int64_t p, double alpha, double* out) {
    if (p < 1) return KVO_INPUT;
    const double pd = (double)p, Cd = (double)C;
    *out = alpha * Cd * Cd / 2.0 * (1.0 / pd + 1.0 / (pd * pd));
    return KVO_OK;
}

/* calibrate_alpha (simnet.hpp:356-366) */
int kvo_calibrate_alpha(const int64_t* Cs, const double* ts, int64_t n, double* alpha_out) {
    if (n < 1) return KVO_CALIBRATION;
    double num = 0, den = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (Cs[i] <= 0) return KVO_CALIBRATION;
        const double c2 = (double)Cs[i] * (double)Cs[i];
        num += ts[i] * c2;
        den += c2 * c2;
    }
    *alpha_out = num / den;
    return KVO_OK;
}

/* ------------------------------------------------------------ search.hpp */
int64_t kvo_resolve_initial_stride(const kvo_search_config* cfg, int64_t C, int64_t p) {
    if (cfg->initial_stride > 0) return cfg->initial_stride;
    const double target = (double)C / (4.0 * (double)p);
    int64_t stride = 1;
    while ((double)stride < target) stride *= 2;
    return stride > cfg->min_stride ? stride : cfg->min_stride;
}

static int validate_search(const kvo_search_config* cfg, kvo_evaluator ev) {
    if (cfg->grid_width < 3) return KVO_SEARCH;
    if (cfg->min_stride < 1) return KVO_SEARCH;
    if (cfg->initial_stride != 0 && cfg->initial_stride < cfg->min_stride) return KVO_SEARCH;
    if (!ev) return KVO_SEARCH;
    return KVO_OK;
}

/* BestTracker (search.hpp:61-84) */
typedef struct {
    const int64_t* even;
    int64_t n; /* p + 1 */
    int has;
    int64_t* part;
    double ttft;
} tracker;

static int64_t even_distance(const int64_t* a, const int64_t* even, int64_t n) {
    int64_t d = 0;
    for (int64_t i = 0; i < n; ++i) d += llabs(a[i] - even[i]);
    return d;
}

static int lex_less(const int64_t* a, const int64_t* b, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        if (a[i] < b[i]) return 1;
        if (a[i] > b[i]) return 0;
    }
    return 0;
}

static void offer(tracker* t, const int64_t* cand, double value) {
    if (!t->has) {
        t->has = 1;
        memcpy(t->part, cand, (size_t)t->n * sizeof(int64_t));
        t->ttft = value;
        return;
    }
    if (value > t->ttft) return;
    if (value < t->ttft) {
        memcpy(t->part, cand, (size_t)t->n * sizeof(int64_t));
        t->ttft = value;
        return;
    }
    const int64_t dn = even_distance(cand, t->even, t->n), dold = even_distance(t->part, t->even, t->n);
    if (dn < dold || (dn == dold && lex_less(cand, t->part, t->n)))
        memcpy(t->part, cand, (size_t)t->n * sizeof(int64_t));
}

/* hierarchical_grid_search (search.hpp:156-207) */
int kvo_hierarchical_grid_search(int64_t C, int64_t p, const kvo_search_config* cfg, kvo_evaluator ev,
                                 void* ctx, int64_t* out, kvo_search_result* res) {
    int st = validate_search(cfg, ev);
    if (st) return st;
    if (p < 2) return KVO_SEARCH;
    const int64_t n = p + 1;
    int64_t* even = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    if ((st = kvo_even_partition(C, p, even))) {
        free(even);
        return st;
    }
    int64_t* inc_part = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* lvl_part = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* center = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* cand = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* digit = (int64_t*)calloc((size_t)p, sizeof(int64_t));
    tracker inc = {even, n, 0, inc_part, INFINITY};
    res->evaluations = 0;
    res->levels = 0;
    offer(&inc, even, ev(even, p, ctx));
    res->evaluations += 1;
    const int64_t axes = p - 1, half = cfg->grid_width / 2;
    int64_t stride = kvo_resolve_initial_stride(cfg, C, p);
    for (;;) {
        res->levels += 1;
        memcpy(center, inc.part, (size_t)n * sizeof(int64_t));
        tracker lvl = {even, n, 0, lvl_part, INFINITY};
        memset(digit, 0, (size_t)p * sizeof(int64_t));
        int found = 0;
        for (;;) {
            memcpy(cand, center, (size_t)n * sizeof(int64_t));
            for (int64_t a = 0; a < axes; ++a) cand[a + 1] += (digit[a] - half) * stride;
            int ok = 1;
            for (int64_t i = 0; i + 1 < n; ++i)
                if (cand[i] >= cand[i + 1]) ok = 0;
            if (ok) {
                offer(&lvl, cand, ev(cand, p, ctx));
                res->evaluations += 1;
                found = 1;
            }
            int64_t a = axes - 1;
            while (a >= 0 && ++digit[a] == cfg->grid_width) {
                digit[a] = 0;
                --a;
            }
            if (a < 0) break;
        }
        if (!found) {
            st = KVO_SEARCH;
            break;
        }
        offer(&inc, lvl.part, lvl.ttft);
        if (stride == cfg->min_stride) break;
        stride = stride / 2 > cfg->min_stride ? stride / 2 : cfg->min_stride;
    }
    if (st == KVO_OK) {
        memcpy(out, inc.part, (size_t)n * sizeof(int64_t));
        res->ttft = inc.ttft;
    }
    free(even); free(inc_part); free(lvl_part); free(center); free(cand); free(digit);
    return st;
}

/* binary_search_two (search.hpp:92-150) */
typedef struct {
    int64_t* keys;
    double* vals;
    int64_t n, cap;
} ucache;

int kvo_binary_search_two(int64_t C, const kvo_search_config* cfg, kvo_evaluator ev, void* ctx,
                          int64_t* out, kvo_search_result* res) {
    int st = validate_search(cfg, ev);
    if (st) return st;
    if (C < 2) return KVO_SEARCH;
    int64_t even[3];
    if ((st = kvo_even_partition(C, 2, even))) return st;
    const int64_t mid = even[1], step = cfg->min_stride;
    const int64_t lo_units = -((mid - 1) / step), hi_units = (C - 1 - mid) / step;
    ucache cache = {0, 0, 0, 0};
    res->evaluations = 0;
#define EVAL_UNITS(u, outv)                                                        \
    do {                                                                           \
        int64_t _u = (u), _k;                                                      \
        for (_k = 0; _k < cache.n; ++_k)                                           \
            if (cache.keys[_k] == _u) break;                                       \
        if (_k < cache.n) {                                                        \
            outv = cache.vals[_k];                                                 \
        } else {                                                                   \
            int64_t _part[3] = {0, mid + _u * step, C};                            \
            double _v = ev(_part, 2, ctx);                                         \
            res->evaluations += 1;                                                 \
            if (cache.n == cache.cap) {                                            \
                cache.cap = cache.cap ? 2 * cache.cap : 64;                        \
                cache.keys = (int64_t*)realloc(cache.keys, (size_t)cache.cap * 8); \
                cache.vals = (double*)realloc(cache.vals, (size_t)cache.cap * 8);  \
            }                                                                      \
            cache.keys[cache.n] = _u;                                              \
            cache.vals[cache.n++] = _v;                                            \
            outv = _v;                                                             \
        }                                                                          \
    } while (0)
    int64_t lo = lo_units, hi = hi_units;
    while (hi - lo > 8) {
        const int64_t m1 = lo + (hi - lo) / 3, m2 = hi - (hi - lo) / 3;
        double v1, v2;
        EVAL_UNITS(m1, v1);
        EVAL_UNITS(m2, v2);
        if (v1 < v2)
            hi = m2;
        else
            lo = m1;
    }
    int64_t best_units = 0;
    double best = INFINITY;
    for (int64_t u = lo; u <= hi; ++u) {
        double v;
        EVAL_UNITS(u, v);
        const int closer = llabs(u) < llabs(best_units) || (llabs(u) == llabs(best_units) && u > best_units);
        if (v < best || (v == best && closer)) {
            best = v;
            best_units = u;
        }
    }
    if (lo_units <= 0 && 0 <= hi_units) {
        double v0;
        EVAL_UNITS(0, v0);
        if (v0 <= best) {
            best = v0;
            best_units = 0;
        }
    }
#undef EVAL_UNITS
    out[0] = 0;
    out[1] = mid + best_units * step;
    out[2] = C;
    res->ttft = best;
    res->levels = 1;
    free(cache.keys);
    free(cache.vals);
    return KVO_OK;
}

/* exhaustive_partition_search (oracle.hpp:117-158) */
int kvo_exhaustive_partition_search(int64_t C, int64_t p, kvo_evaluator ev, void* ctx, int64_t budget,
                                    int64_t* out, kvo_search_result* res) {
    if (!ev) return KVO_SEARCH;
    if (p < 1 || C < p) return KVO_PARTITION;
    double combos = 1;
    for (int64_t k = 1; k < p; ++k) combos = combos * (double)(C - k) / (double)k;
    if (combos > (double)budget) return KVO_BUDGET;
    const int64_t n = p + 1;
    int64_t* even = (int64_t*)malloc((size_t)n * 8);
    kvo_even_partition(C, p, even);
    int64_t* best_part = (int64_t*)malloc((size_t)n * 8);
    int64_t* part = (int64_t*)malloc((size_t)n * 8);
    tracker best = {even, n, 0, best_part, INFINITY};
    res->evaluations = 0;
    int64_t* bounds = part + 1; /* b_1..b_{p-1} */
    part[0] = 0;
    part[p] = C;
    for (int64_t k = 0; k + 1 < p; ++k) bounds[k] = k + 1;
    for (;;) {
        offer(&best, part, ev(part, p, ctx));
        res->evaluations += 1;
        int64_t k = p - 2;
        while (k >= 0 && bounds[k] == C - (p - 1 - k)) --k;
        if (k < 0) break;
        bounds[k] += 1;
        for (int64_t j = k + 1; j + 1 < p; ++j) bounds[j] = bounds[j - 1] + 1;
    }
    memcpy(out, best.part, (size_t)n * 8);
    res->ttft = best.ttft;
    res->levels = 1;
    free(even); free(best_part); free(part);
    return KVO_OK;
}

double kvo_sim_evaluator(const int64_t* b, int64_t p, void* vctx) {
    const kvo_sim_ctx* s = (const kvo_sim_ctx*)vctx;
    double t = NAN;
    kvo_simulate_ttft(s->strategy, b[p], b, p, s->n_layers, &s->cost, &s->net, &t);
    return t;
}

/* practical_bound (simnet.hpp:297-316): searched partition, zero communication. */
int kvo_practical_bound(int64_t C, int64_t p, int64_t n_layers, const kvo_cost* cost, int64_t* out,
                        double* ttft_out) {
    if (p < 1) return KVO_INPUT;
    kvo_sim_ctx s;
    s.n_layers = n_layers;
    s.cost = *cost;
    s.net.bandwidth = INFINITY;
    s.net.latency = 0.0;
    if (p == 1) {
        int st = kvo_even_partition(C, 1, out);
        if (st) return st;
        return kvo_simulate_ttft(KVO_SERIAL, C, out, 1, n_layers, cost, &s.net, ttft_out);
    }
    s.strategy = KVO_KVR;
    kvo_search_config cfg = {5, 0, 1};
    kvo_search_result r;
    int st = kvo_hierarchical_grid_search(C, p, &cfg, kvo_sim_evaluator, &s, out, &r);
    if (st == KVO_OK) *ttft_out = r.ttft;
    return st;
}
