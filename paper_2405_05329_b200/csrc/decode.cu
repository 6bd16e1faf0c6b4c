// decode.cu -- the decode step on the prefilled KV cache: a few new query rows
// (M <= 8) after `position` cached tokens.  Everything here is HBM-bound: the projections stream
// the weights once (8.6 GB for Llama-7B) and the attention streams the KV cache once, so the
// kernels are built for bytes in flight, not for tensor cores.
//
//   gemv_bf16     Y[M x N] = X[M x K] . B[N x K]^T  (B = the K-major weight the tcgen05 GEMM
//                 uses), f32 accumulation, the SAME epilogues as gemm_bf16_tc (QKV split into the
//                 cache rows, residual + bf16 copy, ReLU, consumer-side RMSNorm row scale).  One
//                 warp owns 4 output columns over the whole K (16-byte loads of four weight rows
//                 in flight per lane, X through the read-only path), so the result is
//                 deterministic.  Producer-side RMSNorm partials come from a separate tiny kernel
//                 (M x N floats).
//   attn_decode   split-key flash decoding: CTA = (kv head, key segment); each warp takes one
//                 (query head of the group, query row) at a time, lanes split head_dim, online
//                 softmax over the segment's visible keys; partial (m, l, o) per segment are
//                 merged by a second kernel in segment order (deterministic).
// Reference semantics: layer_qkv / layer_finish / causal_attention (model.hpp:112-192) for rows
// at absolute positions [position, position + M).
#include <cmath>
#include <stdexcept>

#include "kernels.cuh"
#include "ptx.cuh"

namespace kvp {

namespace {

constexpr int GV_WARPS = 4;  // warps per CTA
constexpr int GV_COLS = 4;   // output columns per warp
constexpr int GV_MAXM = 8;

__device__ __forceinline__ void bf16x8_to_f32(const uint4 v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}

struct GvArgs {
    const bf16* X;
    int64_t ldx;
    const bf16* B;
    int M, N, K;
    GemmEpilogue ep;
    float inv_norm_cols;
};

template <int MM, int KIND>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_bf16_kernel(GvArgs g) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = (blockIdx.x * GV_WARPS + warp) * GV_COLS;
    if (n0 >= g.N) return;
    float acc[MM][GV_COLS];
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c) acc[r][c] = 0.f;
    const bf16* wrow[GV_COLS];
#pragma unroll
    for (int c = 0; c < GV_COLS; ++c) wrow[c] = g.B + static_cast<int64_t>(min(n0 + c, g.N - 1)) * g.K;
    // K is a multiple of 8 (host-checked): each lane takes 8 consecutive k per step
    for (int k = lane * 8; k < g.K; k += 32 * 8 * 2) {
        uint4 wv[2][GV_COLS];
        bool has2 = k + 256 < g.K;
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c) {
            wv[0][c] = __ldcs(reinterpret_cast<const uint4*>(wrow[c] + k));  // streamed once
            if (has2) wv[1][c] = __ldcs(reinterpret_cast<const uint4*>(wrow[c] + k + 256));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (u == 1 && !has2) break;
            const int kk = k + u * 256;
#pragma unroll
            for (int r = 0; r < MM; ++r) {
                float xf[8];
                const int rr = r < g.M ? r : g.M - 1;  // padded rows recompute the last one
                bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(g.X + rr * g.ldx + kk)), xf);
#pragma unroll
                for (int c = 0; c < GV_COLS; ++c) {
                    float wf[8];
                    bf16x8_to_f32(wv[u][c], wf);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[r][c] = fmaf(xf[i], wf[i], acc[r][c]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], o);
    if (lane != 0) return;
    const GemmEpilogue& ep = g.ep;
#pragma unroll
    for (int r = 0; r < MM; ++r) {
        if (r >= g.M) break;
        float scale = 1.f;
        if constexpr (KIND != EPI_RESID) {
            if (ep.ssq_in != nullptr) {
                float ss = 0.f;
                for (int q = 0; q < ep.ssq_parts; ++q) ss += ep.ssq_in[r * ep.ssq_parts + q];
                scale = 1.0f / sqrtf(ss * g.inv_norm_cols + 1e-6f);
            }
        }
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c) {
            const int64_t n = n0 + c;
            if (n >= g.N) break;
            float v = acc[r][c];
            if constexpr (KIND == EPI_RESID) {
                v += ep.resid[r * ep.ldr + n];
                ep.outf[r * ep.ldf + n] = v;
                if (ep.outb) ep.outb[r * ep.ldb + n] = __float2bfloat16_rn(v);
            } else {
                v *= scale;
                if constexpr (KIND == EPI_RELU) v = v < 0.f ? 0.f : v;
                bf16* dst;
                if constexpr (KIND == EPI_QKV) {
                    const int64_t e0 = ep.n0, e1 = ep.n0 + ep.n1;
                    dst = n < e0 ? ep.out0 + r * ep.ld0 + n
                                 : (n < e1 ? ep.out1 + r * ep.ld1 + (n - e0) : ep.out2 + r * ep.ld2 + (n - e1));
                } else {
                    dst = ep.out0 + r * ep.ld0 + n;
                }
                *dst = __float2bfloat16_rn(v);
            }
        }
    }
}

// per-row partial sums of squares over 64-column groups of the f32 rows (producer side of the
// fused RMSNorm): one warp per (row, group)
__global__ void ssq_parts_kernel(const float* y, int64_t ldy, int M, int N, float* out, int parts) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= M * parts) return;
    const int r = warp / parts, p = warp % parts;
    float s = 0.f;
    for (int c = p * 64 + lane; c < min(N, p * 64 + 64); c += 32) s = fmaf(y[r * ldy + c], y[r * ldy + c], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r * parts + p] = s;
}

template <int MM, int KIND>
void gemv_launch(const GvArgs& g, cudaStream_t s) {
    const int cols_per_cta = GV_WARPS * GV_COLS;
    const unsigned grid = static_cast<unsigned>((g.N + cols_per_cta - 1) / cols_per_cta);
    note_launch();
    gemv_bf16_kernel<MM, KIND><<<grid, GV_WARPS * 32, 0, s>>>(g);
}

template <int MM>
void gemv_kind(const GvArgs& g, int kind, cudaStream_t s) {
    switch (kind) {
        case EPI_QKV: gemv_launch<MM, EPI_QKV>(g, s); break;
        case EPI_RESID: gemv_launch<MM, EPI_RESID>(g, s); break;
        case EPI_RELU: gemv_launch<MM, EPI_RELU>(g, s); break;
        default: gemv_launch<MM, EPI_STORE>(g, s); break;
    }
}

// ------------------------------------------------------------------ decode attention
constexpr int AD_WARPS = 4;

template <int HD>
__global__ void __launch_bounds__(AD_WARPS * 32)
    attn_decode_kernel(const bf16* Q, const bf16* K, const bf16* V, AttnShape sh, int seg, int n_seg, float sl2,
                       float* part) {
    constexpr int PL = HD / 32;  // head_dim elements per lane
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x / n_seg, sidx = blockIdx.x % n_seg;
    const int group = sh.n_heads / sh.n_kv_heads;
    const int64_t k_lo = static_cast<int64_t>(sidx) * seg;
    const int64_t k_hi = k_lo + seg < sh.k_rows ? k_lo + seg : sh.k_rows;
    const int items = group * static_cast<int>(sh.q_rows);
    for (int it = warp; it < items; it += AD_WARPS) {
        const int hq = g * group + it % group;  // query head
        const int i = it / group;               // query row
        const int64_t vis = sh.offset + i + 1;  // causal: keys <= offset + i
        const int64_t last = k_hi < vis ? k_hi : vis;
        float q[PL];
        {
            const bf16* qp = Q + i * sh.ldq + static_cast<int64_t>(hq) * HD + lane * PL;
#pragma unroll
            for (int e = 0; e < PL; ++e) q[e] = __bfloat162float(qp[e]) * sl2;  // log2-domain scores
        }
        float m = -INFINITY, l = 0.f, o[PL];
#pragma unroll
        for (int e = 0; e < PL; ++e) o[e] = 0.f;
        const bf16* kb = K + static_cast<int64_t>(g) * HD + lane * PL;
        const bf16* vb = V + static_cast<int64_t>(g) * HD + lane * PL;
        for (int64_t j = k_lo; j < last; j += 4) {
            float sc[4], vv[4][PL];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t jj = j + u < last ? j + u : last - 1;
                const bf16* kr = kb + jj * sh.ldkv;
                const bf16* vr = vb + jj * sh.ldkv;
                float d = 0.f;
#pragma unroll
                for (int e = 0; e < PL; ++e) {
                    d = fmaf(q[e], __bfloat162float(kr[e]), d);
                    vv[u][e] = __bfloat162float(vr[e]);
                }
                sc[u] = d;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], off);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (j + u >= last) break;
                const float mn = fmaxf(m, sc[u]);
                const float alpha = exp2f(m - mn), p = exp2f(sc[u] - mn);
                l = l * alpha + p;
#pragma unroll
                for (int e = 0; e < PL; ++e) o[e] = fmaf(p, vv[u][e], o[e] * alpha);
                m = mn;
            }
        }
        // partial record: [m, l, o[HD]] per (query row, query head, segment)
        float* rec = part + ((static_cast<int64_t>(i) * sh.n_heads + hq) * n_seg + sidx) * (HD + 2);
        if (lane == 0) {
            rec[0] = m;
            rec[1] = l;
        }
#pragma unroll
        for (int e = 0; e < PL; ++e) rec[2 + lane * PL + e] = o[e];
    }
}

// merge the segments of each (row, head) in segment order: one warp per (row, head)
template <int HD>
__global__ void attn_decode_combine(const float* part, int n_seg, int rows, int heads, int64_t ldo, bf16* O) {
    constexpr int PL = HD / 32;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows * heads) return;
    const int i = w / heads, hq = w % heads;
    const float* base = part + static_cast<int64_t>(w) * n_seg * (HD + 2);
    float mx = -INFINITY;
    for (int s = 0; s < n_seg; ++s) mx = fmaxf(mx, base[s * (HD + 2)]);
    float l = 0.f, o[PL];
#pragma unroll
    for (int e = 0; e < PL; ++e) o[e] = 0.f;
    for (int s = 0; s < n_seg; ++s) {
        const float* rec = base + s * (HD + 2);
        if (rec[0] == -INFINITY) continue;  // segment with no visible key
        const float a = exp2f(rec[0] - mx);
        l = fmaf(rec[1], a, l);
#pragma unroll
        for (int e = 0; e < PL; ++e) o[e] = fmaf(rec[2 + lane * PL + e], a, o[e]);
    }
    const float inv = 1.0f / l;
    bf16* orow = O + i * ldo + static_cast<int64_t>(hq) * HD + lane * PL;
#pragma unroll
    for (int e = 0; e < PL; ++e) orow[e] = __float2bfloat16_rn(o[e] * inv);
}

template <int HD>
void attn_decode_launch(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, float* part,
                        int seg, int n_seg, cudaStream_t s) {
    const float sl2 = (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f;
    note_launch();
    attn_decode_kernel<HD><<<static_cast<unsigned>(sh.n_kv_heads * n_seg), AD_WARPS * 32, 0, s>>>(Q, K, V, sh, seg,
                                                                                                   n_seg, sl2, part);
    const int warps = static_cast<int>(sh.q_rows) * sh.n_heads;
    note_launch();
    attn_decode_combine<HD><<<static_cast<unsigned>((warps + 3) / 4), 128, 0, s>>>(part, n_seg, static_cast<int>(sh.q_rows),
                                                                                   sh.n_heads, sh.ldo, O);
}

}  // namespace

void gemv_bf16(const bf16* X, int64_t M, int64_t K, const bf16* B, int64_t N, const GemmEpilogue& ep,
               cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    if (M > GV_MAXM) throw std::runtime_error("gemv_bf16: at most 8 rows");
    if (K % 8 != 0 || (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
        throw std::runtime_error("gemv_bf16: K must be a multiple of 8 and operands 16-byte aligned");
    GvArgs g{X, K, B, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), ep,
             ep.norm_cols ? 1.0f / static_cast<float>(ep.norm_cols) : 0.f};
    switch (M) {
        case 1: gemv_kind<1>(g, ep.kind, s); break;
        case 2: gemv_kind<2>(g, ep.kind, s); break;
        case 3: case 4: gemv_kind<4>(g, ep.kind, s); break;  // rows >= M are never stored
        default: gemv_kind<8>(g, ep.kind, s); break;
    }
    if (ep.kind == EPI_RESID && ep.ssq_out != nullptr) {
        const int warps = static_cast<int>(M) * ep.ssq_parts;
        note_launch();
        ssq_parts_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(ep.outf, ep.ldf, static_cast<int>(M),
                                                                               static_cast<int>(N), ep.ssq_out,
                                                                               ep.ssq_parts);
    }
}

int64_t attn_decode_scratch_floats(const AttnShape& sh) {
    const int seg = attn_decode_segment(sh);
    const int64_t n_seg = (sh.k_rows + seg - 1) / seg;
    return sh.q_rows * sh.n_heads * n_seg * (sh.head_dim + 2);
}

int attn_decode_segment(const AttnShape& sh) {
    // enough (kv head, segment) CTAs to keep every SM streaming: ~4 per SM, >= 64 keys each
    const int64_t want = 4 * 148;
    int64_t seg = (sh.k_rows * sh.n_kv_heads + want - 1) / want;
    seg = ((seg + 63) / 64) * 64;
    return static_cast<int>(seg < 64 ? 64 : seg);
}

void attn_decode_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, float* scratch,
                      cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    const int seg = attn_decode_segment(sh);
    const int n_seg = static_cast<int>((sh.k_rows + seg - 1) / seg);
    switch (sh.head_dim) {
        case 64: attn_decode_launch<64>(Q, K, V, O, sh, scratch, seg, n_seg, s); break;
        case 128: attn_decode_launch<128>(Q, K, V, O, sh, scratch, seg, n_seg, s); break;
        default: throw std::runtime_error("attn_decode_bf16: head_dim must be 64 or 128");
    }
}

}  // namespace kvp
