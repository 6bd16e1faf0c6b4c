// decode.cu -- the decode step on the prefilled KV cache: a few new query rows
// (M <= 8) after `position` cached tokens.  Everything here is HBM-bound: the projections stream
// the weights once (8.6 GB for Llama-7B) and the attention streams the KV cache once, so the
// kernels are built for bytes in flight, not for tensor cores.
//
//   gemv_bf16     Y[M x N] = X[M x K] . B[N x K]^T  (B = the K-major weight the tcgen05 GEMM
//                 uses), f32 accumulation, the SAME epilogues as gemm_bf16_tc (QKV split into the
//                 cache rows, residual + bf16 copy, ReLU, consumer-side RMSNorm row scale).  A
//                 warp owns 4 output columns over K (or a 1/2, 1/4 slice of K for narrow N, added
//                 in warp order), 16-byte streaming loads of four weight rows in flight per lane,
//                 X through the read-only path: deterministic.  In a decode session the
//                 consumer GEMV computes the RMSNorm row scale from the f32 rows itself
//                 (norm_src); ssq_parts_kernel serves the partial-sum form otherwise.
//   attn_decode   split-key flash decoding: one warp per (kv head, key segment, item chunk),
//                 looping over its (query head of the group, query row) items; 8 lanes read a
//                 key row as 16-byte pieces (4 keys per warp step, 4 steps in flight), each
//                 8-lane group keeps its own online softmax (rescaled only when its max grows),
//                 merged by shuffles; the partial (m, l, o) of the segments are merged by a
//                 second kernel in segment order (deterministic).
// Reference semantics: layer_qkv / layer_finish / causal_attention (model.hpp:112-192) for rows
// at absolute positions [position, position + M).
#include <cmath>
#include <cstdlib>
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

// Launch with programmatic dependent launch (each decode kernel calls griddep_wait() before
// touching its inputs): the many short kernels of a decode step overlap their launch/prologue
// with the previous kernel's tail.
template <typename Kern, typename... Args>
void pdl_launch(Kern kern, unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    note_launch();
    cudaLaunchKernelEx(&cfg, kern, args...);
}

struct GvArgs {
    const bf16* X;
    int64_t ldx;
    const bf16* B;
    int M, N, K;
    GemmEpilogue ep;
    float inv_norm_cols;
};

template <int MM, int KIND, int KS, int U>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_bf16_kernel(GvArgs g) {
    // KS warps of the CTA split K for the same 4 columns (more bytes in flight for narrow N);
    // their partials are added in warp order (deterministic)
    __shared__ float red[GV_WARPS][MM][GV_COLS];
    __shared__ float row_ss[GV_WARPS][MM];
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if constexpr (KIND != EPI_RESID) {
        if (g.ep.norm_src != nullptr) {  // fused RMSNorm straight from the f32 rows (CTA-wide)
#pragma unroll
            for (int r = 0; r < MM; ++r) {
                const int rr = r < g.M ? r : g.M - 1;
                const float* src = g.ep.norm_src + rr * g.ep.ld_norm;
                float ss = 0.f;
                for (int c = threadIdx.x * 4; c < g.ep.norm_cols; c += GV_WARPS * 32 * 4) {
                    const float4 v = *reinterpret_cast<const float4*>(src + c);
                    ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                if (lane == 0) row_ss[warp][r] = ss;
            }
        }
    }
    __syncthreads();
    const int kg = warp % KS, cg = warp / KS;
    const int n0 = (blockIdx.x * (GV_WARPS / KS) + cg) * GV_COLS;
    const int kchunk = ((g.K + KS - 1) / KS + 7) / 8 * 8;
    const int k_begin = kg * kchunk, k_end = min(g.K, k_begin + kchunk);
    float acc[MM][GV_COLS];
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c) acc[r][c] = 0.f;
    if (n0 < g.N) {
        const bf16* wrow[GV_COLS];
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c) wrow[c] = g.B + static_cast<int64_t>(min(n0 + c, g.N - 1)) * g.K;
        // K is a multiple of 8 (host-checked): each lane takes 8 consecutive k per step
        for (int k = k_begin + lane * 8; k < k_end; k += 32 * 8 * U) {
            // U 16-byte pieces of each of the 4 weight rows in flight per lane
            uint4 wv[U][GV_COLS];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int c = 0; c < GV_COLS; ++c)
                    if (k + u * 256 < k_end) wv[u][c] = __ldcs(reinterpret_cast<const uint4*>(wrow[c] + k + u * 256));
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k + u * 256 >= k_end) break;
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
    }
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
        for (int c = 0; c < GV_COLS; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], o);
    if constexpr (KS > 1) {
        if (lane == 0)
#pragma unroll
            for (int r = 0; r < MM; ++r)
#pragma unroll
                for (int c = 0; c < GV_COLS; ++c) red[warp][r][c] = acc[r][c];
        __syncthreads();
        if (kg != 0) return;
#pragma unroll
        for (int r = 0; r < MM; ++r)
#pragma unroll
            for (int c = 0; c < GV_COLS; ++c) {
                float v = red[warp][r][c];
#pragma unroll
                for (int q = 1; q < KS; ++q) v += red[warp + q][r][c];
                acc[r][c] = v;
            }
    }
    if (lane != 0 || n0 >= g.N) return;
    const GemmEpilogue& ep = g.ep;
#pragma unroll
    for (int r = 0; r < MM; ++r) {
        if (r >= g.M) break;
        float scale = 1.f;
        if constexpr (KIND != EPI_RESID) {
            if (ep.norm_src != nullptr) {
                float ss = 0.f;
#pragma unroll
                for (int q = 0; q < GV_WARPS; ++q) ss += row_ss[q][r];
                scale = 1.0f / sqrtf(ss * g.inv_norm_cols + 1e-6f);
            } else if (ep.ssq_in != nullptr) {
                float ss = 0.f;
                for (int q = 0; q < ep.ssq_parts; ++q) ss += ep.ssq_in[r * ep.ssq_parts + q];
                scale = 1.0f / sqrtf(ss * g.inv_norm_cols + 1e-6f);
            }
        }
        if constexpr (KIND == EPI_QKV) {
            // opt-in rotary embedding of the Q and K columns (GemmEpilogue::rope_*): GV_COLS is
            // even and n0 a multiple of it, so the column group holds whole (2i, 2i+1) pairs
            if (ep.rope_hd > 0 && n0 < ep.n0 + ep.n1) {
                const int64_t rc0 = n0 < ep.n0 ? n0 : n0 - ep.n0;
                const float fpos = static_cast<float>(ep.rope_pos0 + r);
#pragma unroll
                for (int c = 0; c < GV_COLS; c += 2) {
                    float sn, cs;
                    sincosf(fpos * __ldg(ep.rope_inv_freq + ((rc0 + c) % ep.rope_hd) / 2), &sn, &cs);
                    // the rotation is linear, so it commutes with the RMSNorm row scale
                    const float x0 = acc[r][c], x1 = acc[r][c + 1];
                    acc[r][c] = x0 * cs - x1 * sn;
                    acc[r][c + 1] = x0 * sn + x1 * cs;
                }
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
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();
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
    // split K over 1, 2 or 4 warps so that >= ~24 weight-streaming warps land on every SM
    const int64_t col_warps = (g.N + GV_COLS - 1) / GV_COLS;
    const int ks = col_warps >= 24 * 148 ? 1 : (col_warps >= 12 * 148 ? 2 : 4);
    const int cols_per_cta = (GV_WARPS / ks) * GV_COLS;
    const unsigned grid = static_cast<unsigned>((g.N + cols_per_cta - 1) / cols_per_cta);
    static const int unroll = [] {
        const char* e = getenv("KVP_GEMV_UNROLL");
        return e ? atoi(e) : 2;
    }();
    if (unroll == 4) {
        if (ks == 1)
            pdl_launch(gemv_bf16_kernel<MM, KIND, 1, 4>, grid, GV_WARPS * 32, s, g);
        else if (ks == 2)
            pdl_launch(gemv_bf16_kernel<MM, KIND, 2, 4>, grid, GV_WARPS * 32, s, g);
        else
            pdl_launch(gemv_bf16_kernel<MM, KIND, 4, 4>, grid, GV_WARPS * 32, s, g);
    } else {
        if (ks == 1)
            pdl_launch(gemv_bf16_kernel<MM, KIND, 1, 2>, grid, GV_WARPS * 32, s, g);
        else if (ks == 2)
            pdl_launch(gemv_bf16_kernel<MM, KIND, 2, 2>, grid, GV_WARPS * 32, s, g);
        else
            pdl_launch(gemv_bf16_kernel<MM, KIND, 4, 2>, grid, GV_WARPS * 32, s, g);
    }
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
// target warps per SM for the split-key grid (KVP_DECODE_WPSM tunes it)
int decode_warps_per_sm() {
    static const int w = [] {
        const char* e = getenv("KVP_DECODE_WPSM");
        return e ? atoi(e) : 32;
    }();
    return w > 0 ? w : 32;
}

constexpr int AD_WARPS = 4;  // warps per CTA; every warp owns one key segment
constexpr int AD_LPK = 8;    // lanes per key: a key row is read as 8 x 16-byte (hd 128) pieces
constexpr int AD_KPS = 32 / AD_LPK;  // keys per warp step
constexpr int AD_U = 4;              // warp steps in flight

__device__ __forceinline__ void load_bf16x(const bf16* p, float* f, int n) {
    // n = 8 or 16 consecutive bf16 (16-byte aligned) -> f32 (the query row)
    for (int v = 0; v < n / 8; ++v) {
        float t[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(p + 8 * v), t);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[8 * v + e] = t[e];
    }
}

template <int HD, int HPW>
__global__ void __launch_bounds__(AD_WARPS * 32)
    attn_decode_kernel(const bf16* Q, const bf16* K, const bf16* V, AttnShape sh, int seg, int n_seg, int n_ich,
                       float sl2, float* part) {
    // HPW query heads of one GQA/MQA group per warp item: every K/V piece a lane loads and
    // converts serves HPW dot products and HPW P.V updates
    constexpr int EPL = HD / AD_LPK;  // head_dim elements per lane (16 or 8)
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ksub = lane / AD_LPK, sl = lane % AD_LPK;
    // global warp index -> (kv head, key segment, item chunk)
    const int wid = blockIdx.x * AD_WARPS + warp;
    const int ich = wid % n_ich, wseg = wid / n_ich;
    const int g = wseg / n_seg, sidx = wseg % n_seg;
    if (g >= sh.n_kv_heads) return;
    const int group = sh.n_heads / sh.n_kv_heads;
    const int hchunks = (group + HPW - 1) / HPW;
    const int64_t k_lo = static_cast<int64_t>(sidx) * seg;
    const int64_t k_hi = k_lo + seg < sh.k_rows ? k_lo + seg : sh.k_rows;
    const bf16* kb = K + static_cast<int64_t>(g) * HD + sl * EPL;
    const bf16* vb = V + static_cast<int64_t>(g) * HD + sl * EPL;
    const int items = hchunks * static_cast<int>(sh.q_rows);
    for (int it = ich; it < items; it += n_ich) {
        const int hc = it % hchunks;  // chunk of HPW query heads of the group
        const int i = it / hchunks;   // query row
        const int64_t vis = sh.offset + i + 1;  // causal: keys <= offset + i
        const int64_t last = k_hi < vis ? k_hi : vis;
        float q[HPW][EPL], m[HPW], l[HPW], o[HPW][EPL];
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
            const int hg = min(hc * HPW + hh, group - 1);  // padded heads recompute the last one
            load_bf16x(Q + i * sh.ldq + static_cast<int64_t>(g * group + hg) * HD + sl * EPL, q[hh], EPL);
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                q[hh][e] *= sl2;  // log2-domain scores
                o[hh][e] = 0.f;
            }
            m[hh] = -INFINITY;  // every group of AD_LPK lanes keeps its own online-softmax state
            l[hh] = 0.f;
        }
        // AD_U key steps (4 keys each) of raw 16-byte K/V pieces in flight per lane, converted
        // on use; the online softmax rescales o only when the group's running max grows
        for (int64_t j0 = k_lo; j0 < last; j0 += AD_U * AD_KPS) {
            uint4 kr[AD_U][EPL / 8], vr[AD_U][EPL / 8];
            bool ok[AD_U];
#pragma unroll
            for (int u = 0; u < AD_U; ++u) {
                const int64_t j = j0 + u * AD_KPS + ksub;
                ok[u] = j < last;
                const int64_t jj = ok[u] ? j : last - 1;
#pragma unroll
                for (int v = 0; v < EPL / 8; ++v) {
                    kr[u][v] = *reinterpret_cast<const uint4*>(kb + jj * sh.ldkv + 8 * v);
                    vr[u][v] = *reinterpret_cast<const uint4*>(vb + jj * sh.ldkv + 8 * v);
                }
            }
#pragma unroll
            for (int u = 0; u < AD_U; ++u) {
                float sc[HPW];
#pragma unroll
                for (int hh = 0; hh < HPW; ++hh) sc[hh] = 0.f;
#pragma unroll
                for (int v = 0; v < EPL / 8; ++v) {
                    float t[8];
                    bf16x8_to_f32(kr[u][v], t);
#pragma unroll
                    for (int hh = 0; hh < HPW; ++hh)
#pragma unroll
                        for (int e = 0; e < 8; ++e) sc[hh] = fmaf(q[hh][8 * v + e], t[e], sc[hh]);
                }
#pragma unroll
                for (int hh = 0; hh < HPW; ++hh)
#pragma unroll
                    for (int off = 1; off < AD_LPK; off <<= 1) sc[hh] += __shfl_xor_sync(0xffffffffu, sc[hh], off);
                if (ok[u]) {
                    float p[HPW];
#pragma unroll
                    for (int hh = 0; hh < HPW; ++hh) {
                        if (sc[hh] > m[hh]) {  // new running max: rescale (exp2(-inf) = 0 first)
                            const float alpha = exp2f(m[hh] - sc[hh]);
                            l[hh] *= alpha;
#pragma unroll
                            for (int e = 0; e < EPL; ++e) o[hh][e] *= alpha;
                            m[hh] = sc[hh];
                        }
                        p[hh] = exp2f(sc[hh] - m[hh]);
                        l[hh] += p[hh];
                    }
#pragma unroll
                    for (int v = 0; v < EPL / 8; ++v) {
                        float t[8];
                        bf16x8_to_f32(vr[u][v], t);
#pragma unroll
                        for (int hh = 0; hh < HPW; ++hh)
#pragma unroll
                            for (int e = 0; e < 8; ++e) o[hh][8 * v + e] = fmaf(p[hh], t[e], o[hh][8 * v + e]);
                    }
                }
            }
        }
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
            if (hc * HPW + hh >= group) break;
            const int hq = g * group + hc * HPW + hh;
            // merge the AD_KPS lane groups (lanes sl, sl+8, sl+16, sl+24 hold the same hd slice)
            float mx = m[hh];
#pragma unroll
            for (int off = AD_LPK; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            const float a = (m[hh] == -INFINITY) ? 0.f : exp2f(m[hh] - mx);
            float lh = l[hh] * a;
            float oh[EPL];
#pragma unroll
            for (int e = 0; e < EPL; ++e) oh[e] = o[hh][e] * a;
#pragma unroll
            for (int off = AD_LPK; off < 32; off <<= 1) {
                lh += __shfl_xor_sync(0xffffffffu, lh, off);
#pragma unroll
                for (int e = 0; e < EPL; ++e) oh[e] += __shfl_xor_sync(0xffffffffu, oh[e], off);
            }
            // partial record: [m, l, o[HD]] per (query row, query head, segment)
            float* rec = part + ((static_cast<int64_t>(i) * sh.n_heads + hq) * n_seg + sidx) * (HD + 2);
            if (lane == 0) {
                rec[0] = mx;
                rec[1] = lh;
            }
            if (ksub == 0) {
#pragma unroll
                for (int e = 0; e < EPL; ++e) rec[2 + sl * EPL + e] = oh[e];
            }
        }
    }
}

// merge the segments of each (row, head) in segment order: one CTA of HD threads per
// (row, head); the per-segment weights exp2(m_s - max) go through smem, then thread t sums
// element t over the segments (independent, coalesced loads)
constexpr int CB_G = 4;  // segment groups per output dimension in attn_decode_combine

template <int HD>
__global__ void __launch_bounds__(HD * CB_G) attn_decode_combine(const float* part, int n_seg, int rows, int heads,
                                                                 int64_t ldo, bf16* O) {
    // Merges the segment partials (m, l, o[HD]) of one (row, head) in a FIXED order
    // (deterministic): max and weights in parallel over segments, l by a fixed shuffle tree;
    // thread (g, d) accumulates o[d] over segments s = g (mod CB_G) -- all of its loads
    // independent and in flight at once -- and the CB_G group sums are added in order.
    extern __shared__ float wts[];  // [n_seg] segment weights
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();
    constexpr int NT = HD * CB_G, NW = NT / 32;
    const int w = blockIdx.x, t = threadIdx.x;
    if (w >= rows * heads) return;
    const int i = w / heads, hq = w % heads;
    const float* base = part + static_cast<int64_t>(w) * n_seg * (HD + 2);
    __shared__ float red[NW], lred[NW];
    __shared__ float po[CB_G - 1][HD];
    float mx = -INFINITY;
    for (int s = t; s < n_seg; s += NT) mx = fmaxf(mx, base[s * (HD + 2)]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((t & 31) == 0) red[t >> 5] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int q = 1; q < NW; ++q) mx = fmaxf(mx, red[q]);
    float lp = 0.f;
    for (int s = t; s < n_seg; s += NT) {
        const float ms = base[s * (HD + 2)];
        const float wt = ms == -INFINITY ? 0.f : exp2f(ms - mx);  // a segment with no visible key weighs 0
        wts[s] = wt;
        lp = fmaf(base[s * (HD + 2) + 1], wt, lp);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, off);
    if ((t & 31) == 0) lred[t >> 5] = lp;
    __syncthreads();
    const int d = t % HD, g = t / HD;
    const float* col = base + 2 + d;
    float o = 0.f;
#pragma unroll 16
    for (int s = g; s < n_seg; s += CB_G) o = fmaf(col[s * (HD + 2)], wts[s], o);
    if (g > 0) po[g - 1][d] = o;
    __syncthreads();
    if (g == 0) {
        float l = lred[0];
#pragma unroll
        for (int q = 1; q < NW; ++q) l += lred[q];
#pragma unroll
        for (int q = 0; q < CB_G - 1; ++q) o += po[q][d];
        O[i * ldo + static_cast<int64_t>(hq) * HD + d] = __float2bfloat16_rn(o / l);
    }
}

template <int HD>
void attn_decode_launch(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, float* part,
                        int seg, int n_seg, cudaStream_t s) {
    const float sl2 = (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f;
    // item chunks: enough warps for ~32 per SM when the (kv head, segment) grid is short
    const int group = sh.n_heads / sh.n_kv_heads;
    const int hpw = group >= 4 ? (HD == 64 ? 4 : 2) : 1;
    const int items = ((group + hpw - 1) / hpw) * static_cast<int>(sh.q_rows);
    const int base = sh.n_kv_heads * n_seg;
    int n_ich = (decode_warps_per_sm() * 148 + base - 1) / base;
    n_ich = n_ich < 1 ? 1 : (n_ich > items ? items : n_ich);
    const int warps = base * n_ich;
    const unsigned blocks = static_cast<unsigned>((warps + AD_WARPS - 1) / AD_WARPS);
    if (hpw == 4)
        pdl_launch(attn_decode_kernel<HD, 4>, blocks, AD_WARPS * 32, s, Q, K, V, sh, seg, n_seg, n_ich, sl2, part);
    else if (hpw == 2)
        pdl_launch(attn_decode_kernel<HD, 2>, blocks, AD_WARPS * 32, s, Q, K, V, sh, seg, n_seg, n_ich, sl2, part);
    else
        pdl_launch(attn_decode_kernel<HD, 1>, blocks, AD_WARPS * 32, s, Q, K, V, sh, seg, n_seg, n_ich, sl2, part);
    const int cw = static_cast<int>(sh.q_rows) * sh.n_heads;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(cw));
    cfg.blockDim = dim3(HD * CB_G);
    cfg.dynamicSmemBytes = static_cast<size_t>(n_seg) * 4;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    note_launch();
    cudaLaunchKernelEx(&cfg, attn_decode_combine<HD>, static_cast<const float*>(part), n_seg,
                       static_cast<int>(sh.q_rows), sh.n_heads, sh.ldo, O);
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
        pdl_launch(ssq_parts_kernel, static_cast<unsigned>((warps + 7) / 8), 256, s, static_cast<const float*>(ep.outf),
                   ep.ldf, static_cast<int>(M), static_cast<int>(N), ep.ssq_out, ep.ssq_parts);
    }
}

int64_t attn_decode_scratch_floats(const AttnShape& sh) {
    const int seg = attn_decode_segment(sh);
    const int64_t n_seg = (sh.k_rows + seg - 1) / seg;
    return sh.q_rows * sh.n_heads * n_seg * (sh.head_dim + 2);
}

int attn_decode_segment(const AttnShape& sh) {
    // keys per warp: enough (kv head, segment) warps to keep every SM streaming (~32 warps per
    // SM), at least 64 keys each
    const int64_t want = static_cast<int64_t>(decode_warps_per_sm()) * 148;
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
