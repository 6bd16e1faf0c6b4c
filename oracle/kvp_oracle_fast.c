/*
 * kvp_oracle_fast.c -- the f32 reference forward pass at benchmark shapes (Llama-7B, Falcon-7B
 * at 4k-16k tokens), multi-threaded and blocked but operation-for-operation the reference's
 * arithmetic.  TEST INFRASTRUCTURE ONLY (see kvp_oracle.h): it generates the large golden
 * fixtures (tests/golden/make_golden_large.py) that the GPU parity tests read; the product
 * never links it.
 *
 * Why it is bit-identical to the reference's run<float> (checked against oracle/_ref in
 * tests/test_oracle_fast.py, and against the reference itself at llama7b-4k in
 * tests/golden/ref_llama7b-4k.json):
 *  - matmul (matrix.hpp:76-91) computes out[i,j] = (((0 + a[i,0]b[0,j]) + a[i,1]b[1,j]) + ...),
 *    every product rounded to float before the add (the reference's Release build has no FMA
 *    contraction; this file is built with -ffp-contract=off).  Register tiling over (i, j)
 *    and splitting rows/columns over threads keep exactly that sequence per element.
 *  - causal_attention (model.hpp:112-158) scores every key row; a masked score is
 *    s - 1e9 (float), whose exp(s - max) underflows to exactly 0, so skipping masked keys
 *    adds exact zeros to the row sum and to the PV accumulators: same bits.  Scores keep the
 *    sequential-over-d order (vectorised over keys against a transposed K), PV keeps the
 *    sequential-over-keys order (vectorised over d), exps use the same libm expf.
 *  - rms_norm_rows (model.hpp:29-40), relu and add are elementwise in the reference order.
 *  - init_weights (weights.hpp:41-83): SplitMix64 is a counter generator, so element n of a
 *    stream is mix(state0 + (n+1)*gamma); generated in parallel, same doubles, same casts.
 * The reference's KVR result is bitwise equal to its serial forward (test_engine.cpp:50-99),
 * so one serial pass gives the golden for every partition.
 */
#include <cpuid.h>
#include <immintrin.h>
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "kvp_oracle.h"

#define GAMMA 0x9e3779b97f4a7c15ULL

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* weights.hpp:41-47 seeded_matrix, element-parallel */
static void seeded_par(float* out, int64_t n, double scale, uint64_t stream) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t z = mix64(stream + (uint64_t)(i + 1) * GAMMA);
        const double u = (double)(z >> 11) * 0x1.0p-53;
        out[i] = (float)((2.0 * u - 1.0) * scale);
    }
}

/* matrix.hpp:76-91, out = a[rows x inner] . b[inner x cols] (out zero-initialised, i-k-j
 * accumulation per element, no FMA).  Tiles of 4 rows x 64 columns held in zmm registers. */
static void mm_tile_scalar(const float* a, int64_t inner, const float* b, int64_t cols, float* out, int64_t i0,
                           int64_t i1, int64_t j0, int64_t j1) {
    for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) {
            float acc = 0.f;
            for (int64_t k = 0; k < inner; ++k) acc += a[i * inner + k] * b[k * cols + j];
            out[i * cols + j] = acc;
        }
}

__attribute__((target("avx512f"))) static void mm_avx512(const float* a, int64_t rows, int64_t inner,
                                                          const float* b, int64_t cols, float* out) {
    const int64_t RB = 64, NB = 64;
    const int64_t nrb = (rows + RB - 1) / RB, ncb = cols / NB;
    /* B packed as [column block][k][64]: the tile loop reads 256 contiguous bytes per k
     * (a row-major B has a power-of-two-ish stride that thrashes the cache sets) */
    float* bp = (float*)aligned_alloc(64, (size_t)(ncb * inner * NB) * sizeof(float) + 64);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t cb = 0; cb < ncb; ++cb)
        for (int64_t k = 0; k < inner; ++k)
            memcpy(bp + (cb * inner + k) * NB, b + k * cols + cb * NB, NB * sizeof(float));
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int64_t cb = 0; cb < ncb; ++cb)
        for (int64_t rb = 0; rb < nrb; ++rb) {
            const int64_t j0 = cb * NB;
            const float* bs = bp + cb * inner * NB;
            const int64_t r0 = rb * RB, r1 = r0 + RB < rows ? r0 + RB : rows;
            int64_t i = r0;
            for (; i + 4 <= r1; i += 4) {
                __m512 c[4][4];
                for (int r = 0; r < 4; ++r)
                    for (int q = 0; q < 4; ++q) c[r][q] = _mm512_setzero_ps();
                const float* a0 = a + i * inner;
                for (int64_t k = 0; k < inner; ++k) {
                    const float* bk = bs + k * NB;
                    const __m512 b0 = _mm512_load_ps(bk), b1 = _mm512_load_ps(bk + 16),
                                 b2 = _mm512_load_ps(bk + 32), b3 = _mm512_load_ps(bk + 48);
                    for (int r = 0; r < 4; ++r) {
                        const __m512 av = _mm512_set1_ps(a0[r * inner + k]);
                        c[r][0] = _mm512_add_ps(c[r][0], _mm512_mul_ps(av, b0));
                        c[r][1] = _mm512_add_ps(c[r][1], _mm512_mul_ps(av, b1));
                        c[r][2] = _mm512_add_ps(c[r][2], _mm512_mul_ps(av, b2));
                        c[r][3] = _mm512_add_ps(c[r][3], _mm512_mul_ps(av, b3));
                    }
                }
                for (int r = 0; r < 4; ++r)
                    for (int q = 0; q < 4; ++q) _mm512_storeu_ps(out + (i + r) * cols + j0 + 16 * q, c[r][q]);
            }
            for (; i < r1; ++i) {
                __m512 c0 = _mm512_setzero_ps(), c1 = c0, c2 = c0, c3 = c0;
                for (int64_t k = 0; k < inner; ++k) {
                    const float* bk = bs + k * NB;
                    const __m512 av = _mm512_set1_ps(a[i * inner + k]);
                    c0 = _mm512_add_ps(c0, _mm512_mul_ps(av, _mm512_load_ps(bk)));
                    c1 = _mm512_add_ps(c1, _mm512_mul_ps(av, _mm512_load_ps(bk + 16)));
                    c2 = _mm512_add_ps(c2, _mm512_mul_ps(av, _mm512_load_ps(bk + 32)));
                    c3 = _mm512_add_ps(c3, _mm512_mul_ps(av, _mm512_load_ps(bk + 48)));
                }
                _mm512_storeu_ps(out + i * cols + j0, c0);
                _mm512_storeu_ps(out + i * cols + j0 + 16, c1);
                _mm512_storeu_ps(out + i * cols + j0 + 32, c2);
                _mm512_storeu_ps(out + i * cols + j0 + 48, c3);
            }
        }
    free(bp);
    if (ncb * NB < cols) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < rows; ++i) mm_tile_scalar(a, inner, b, cols, out, i, i + 1, ncb * NB, cols);
    }
}

static int has_avx512f(void) {
    unsigned a = 0, b = 0, c = 0, d = 0;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return 0;
    return (b >> 16) & 1u;
}

static void mm(const float* a, int64_t rows, int64_t inner, const float* b, int64_t cols, float* out) {
    if (has_avx512f()) {
        mm_avx512(a, rows, inner, b, cols, out);
        return;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) mm_tile_scalar(a, inner, b, cols, out, i, i + 1, 0, cols);
}

/* model.hpp:29-45 maybe_norm (rms_norm_rows: no gain, eps 1e-6, float arithmetic) */
static void maybe_norm(const kvo_config* c, const float* x, int64_t rows, int64_t cols, float* out) {
    if (!c->rms_norm) {
        memcpy(out, x, (size_t)(rows * cols) * sizeof(float));
        return;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        float mean_sq = 0;
        for (int64_t j = 0; j < cols; ++j) mean_sq += x[i * cols + j] * x[i * cols + j];
        mean_sq /= (float)cols;
        const float inv = 1.0f / sqrtf(mean_sq + 1e-6f);
        for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = x[i * cols + j] * inv;
    }
}

/* model.hpp:112-158 causal_attention with offset 0 over k_rows == q_rows (serial). */
__attribute__((target("avx512f"))) static void attention(const kvo_config* c, const float* Q, const float* K,
                                                          const float* V, int64_t C, float* A) {
    const int64_t hd = c->d_model / c->n_heads, group = c->n_heads / c->n_kv_heads;
    const int64_t q = c->n_heads * hd, kv = c->n_kv_heads * hd;
    const float scale = 1.0f / sqrtf((float)hd);
    const int64_t Cp = ((C + 15) & ~(int64_t)15) + 16; /* +64 B: no power-of-two row stride */
    /* K^T per kv head: [kvh][hd][Cp] */
    float* Kt = (float*)aligned_alloc(64, (size_t)(c->n_kv_heads * hd * Cp) * sizeof(float));
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t g = 0; g < c->n_kv_heads; ++g)
        for (int64_t d = 0; d < hd; ++d) {
            float* row = Kt + (g * hd + d) * Cp;
            for (int64_t j = 0; j < C; ++j) row[j] = K[j * kv + g * hd + d];
            for (int64_t j = C; j < Cp; ++j) row[j] = 0.f;
        }
    const int nt = omp_get_max_threads();
    float* scratch = (float*)aligned_alloc(64, (size_t)(nt * (Cp + hd + 16)) * sizeof(float));
#pragma omp parallel
    {
        float* s = scratch + (size_t)omp_get_thread_num() * (size_t)(Cp + hd + 16);
        float* acc = s + Cp;
#pragma omp for collapse(2) schedule(dynamic, 8)
        for (int64_t h = 0; h < c->n_heads; ++h)
            for (int64_t ii = 0; ii < C; ++ii) {
                const int64_t i = C - 1 - ii; /* long rows first */
                const int64_t g = h / group;
                const float* qi = Q + i * q + h * hd;
                const float* kt = Kt + g * hd * Cp;
                const int64_t vis = i + 1; /* keys 0..i */
                /* scores: s_j = ((0 + q0 k0) + q1 k1) + ...  then * scale */
                for (int64_t j = 0; j < vis; j += 16) {
                    __m512 sv = _mm512_setzero_ps();
                    for (int64_t d = 0; d < hd; ++d)
                        sv = _mm512_add_ps(sv, _mm512_mul_ps(_mm512_set1_ps(qi[d]), _mm512_loadu_ps(kt + d * Cp + j)));
                    _mm512_storeu_ps(s + j, _mm512_mul_ps(sv, _mm512_set1_ps(scale)));
                }
                float row_max = -1e9f;
                for (int64_t j = 0; j < vis; ++j)
                    if (s[j] > row_max) row_max = s[j];
                float sum = 0;
                for (int64_t j = 0; j < vis; ++j) {
                    s[j] = expf(s[j] - row_max);
                    sum += s[j];
                }
                for (int64_t d = 0; d < hd; d += 16) {
                    const __mmask16 mk = hd - d >= 16 ? (__mmask16)0xFFFF : (__mmask16)((1u << (hd - d)) - 1u);
                    __m512 av = _mm512_setzero_ps();
                    const float* vcol = V + g * hd + d;
                    for (int64_t j = 0; j < vis; ++j)
                        av = _mm512_add_ps(av, _mm512_mul_ps(_mm512_set1_ps(s[j]), _mm512_maskz_loadu_ps(mk, vcol + j * kv)));
                    _mm512_mask_storeu_ps(acc + d, mk, av);
                }
                float* ai = A + i * q + h * hd;
                for (int64_t d = 0; d < hd; ++d) ai[d] = acc[d] / sum;
            }
    }
    free(scratch);
    free(Kt);
}

/* weights.hpp:54-83 for one layer, reference layouts [in x out] */
static void layer_weights(const kvo_config* c, int64_t layer, float* wq, float* wk, float* wv, float* wo, float* w1,
                          float* w2) {
    const int64_t d = c->d_model, hd = d / c->n_heads, q = c->n_heads * hd, kv = c->n_kv_heads * hd;
    const double scale = 1.0 / sqrt((double)d);
    const uint64_t L = (uint64_t)layer;
    seeded_par(wq, d * q, scale, kvo_mix_seed(c->seed, L, 1));
    seeded_par(wk, d * kv, scale, kvo_mix_seed(c->seed, L, 2));
    seeded_par(wv, d * kv, scale, kvo_mix_seed(c->seed, L, 3));
    seeded_par(wo, q * d, scale, kvo_mix_seed(c->seed, L, 4));
    seeded_par(w1, d * 2 * d, scale, kvo_mix_seed(c->seed, L, 5));
    seeded_par(w2, 2 * d * d, scale, kvo_mix_seed(c->seed, L, 6));
}

/*
 * forward_serial (model.hpp:197-211) in f32 at any size.  context [C x d]; hidden_out
 * [C x d] (may be NULL), last_row [d] (the first-token readout, engine.hpp:88).  Needs an
 * AVX-512 host (KVO_CONFIG otherwise).  Returns a KVO status.
 */
int kvof_forward_f32(const kvo_config* c, const float* context, int64_t C, float* hidden_out, float* last_row) {
    int st = kvo_validate_config(c);
    if (st) return st;
    if (C < 1) return KVO_INPUT;
    const int64_t d = c->d_model, hd = d / c->n_heads, q = c->n_heads * hd, kv = c->n_kv_heads * hd, f = 2 * d;
    if (!has_avx512f()) return KVO_CONFIG;
    float *wq = malloc(sizeof(float) * d * q), *wk = malloc(sizeof(float) * d * kv), *wv = malloc(sizeof(float) * d * kv),
          *wo = malloc(sizeof(float) * q * d), *w1 = malloc(sizeof(float) * d * f), *w2 = malloc(sizeof(float) * f * d);
    float *h = malloc(sizeof(float) * C * d), *x = malloc(sizeof(float) * C * d), *Q = malloc(sizeof(float) * C * q),
          *K = malloc(sizeof(float) * C * kv), *V = malloc(sizeof(float) * C * kv), *A = malloc(sizeof(float) * C * q),
          *t = malloc(sizeof(float) * C * f), *h1 = malloc(sizeof(float) * C * d);
    memcpy(h, context, sizeof(float) * C * d);
    for (int64_t l = 0; l < c->n_layers; ++l) {
        layer_weights(c, l, wq, wk, wv, wo, w1, w2);
        /* layer_qkv (model.hpp:189-192) */
        maybe_norm(c, h, C, d, x);
        mm(x, C, d, wq, q, Q);
        mm(x, C, d, wk, kv, K);
        mm(x, C, d, wv, kv, V);
        /* layer_finish (model.hpp:164-175) */
        attention(c, Q, K, V, C, A);
        mm(A, C, q, wo, d, t);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < C * d; ++i) h1[i] = h[i] + t[i];
        maybe_norm(c, h1, C, d, x);
        mm(x, C, d, w1, f, t);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < C * f; ++i)
            if (t[i] < 0.f) t[i] = 0.f;
        mm(t, C, f, w2, d, A);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < C * d; ++i) h[i] = h1[i] + A[i];
    }
    if (hidden_out) memcpy(hidden_out, h, sizeof(float) * C * d);
    if (last_row) memcpy(last_row, h + (C - 1) * d, sizeof(float) * d);
    free(wq); free(wk); free(wv); free(wo); free(w1); free(w2);
    free(h); free(x); free(Q); free(K); free(V); free(A); free(t); free(h1);
    return KVO_OK;
}
