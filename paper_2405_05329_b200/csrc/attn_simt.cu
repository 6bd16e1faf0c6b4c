// attn_simt.cu -- generic prefix-causal attention (any head_dim <= 256), f32 math.
// Used by the fp32 parity mode and by bf16 shapes whose head_dim is below the tensor-core
// tile (e.g. the reference's tiny d=32/h=4 workload, hd=8).
//
// Semantics of causal_attention (model.hpp:112-158): query i (absolute offset+i) sees keys
// [0, offset+i]; masked keys get exactly zero weight (the reference's -1e9 / -1e18 penalty
// underflows exp() to 0), so they are skipped instead of scored.  One warp per (query row,
// head): lanes stride over keys for the scores, then over head_dim for P.V.
#include "kernels.cuh"

namespace kvp {

namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
    if constexpr (sizeof(T) == 4)
        return *reinterpret_cast<const float*>(p);
    else
        return __bfloat162float(*reinterpret_cast<const bf16*>(p));
}

template <typename T>
__device__ __forceinline__ void st(T* p, float v) {
    if constexpr (sizeof(T) == 4)
        *reinterpret_cast<float*>(p) = v;
    else
        *reinterpret_cast<bf16*>(p) = __float2bfloat16_rn(v);
}

constexpr int WARPS = 4;

template <typename T>
__global__ void __launch_bounds__(WARPS * 32) attn_simt_kernel(const T* __restrict__ Q, const T* __restrict__ K,
                                                               const T* __restrict__ V, T* __restrict__ O,
                                                               AttnShape sh) {
    __shared__ float sq[WARPS][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * (int64_t)WARPS + w;
    const int h = blockIdx.y;
    if (i >= sh.q_rows) return;
    const int hd = sh.head_dim;
    const int g = h / (sh.n_heads / sh.n_kv_heads);
    const T* q = Q + i * sh.ldq + (int64_t)h * hd;
    for (int d = lane; d < hd; d += 32) sq[w][d] = ld(q + d);
    __syncwarp();
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    const int64_t n_vis = sh.offset + i + 1;
    const T* kb = K + (int64_t)g * hd;
    const T* vb = V + (int64_t)g * hd;

    auto score = [&](int64_t j) {
        const T* kr = kb + j * sh.ldkv;
        float s = 0.f;
        for (int d = 0; d < hd; ++d) s += sq[w][d] * ld(kr + d);
        return s * scale;
    };

    float m = -INFINITY;
    for (int64_t j = lane; j < n_vis; j += 32) m = fmaxf(m, score(j));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));

    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = 0.f;
    float l = 0.f;
    for (int64_t j0 = 0; j0 < n_vis; j0 += 32) {
        const int64_t j = j0 + lane;
        const float p = j < n_vis ? expf(score(j) - m) : 0.f;
        l += p;
        const int cnt = (n_vis - j0) < 32 ? static_cast<int>(n_vis - j0) : 32;
        for (int t = 0; t < cnt; ++t) {
            const float pt = __shfl_sync(0xffffffffu, p, t);
            const T* vr = vb + (j0 + t) * sh.ldkv;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int d = lane + 32 * u;
                if (d < hd) acc[u] += pt * ld(vr + d);
            }
        }
    }
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    T* orow = O + i * sh.ldo + (int64_t)h * hd;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int d = lane + 32 * u;
        if (d < hd) st(orow + d, acc[u] / l);
    }
}

// fp32 parity mode at head_dim 64 / 128 (the Llama / Falcon shapes): a tiled flash-style SIMT
// kernel.  CTA = 64 query rows of one head, 256 threads; per 64-key tile: K (transposed) and V
// staged in smem, S = Q K^T with 4 x 4 scores per thread, online softmax (row max / sum over
// the 16 lanes that share a row group, accurate expf), P through smem, O += P V with 4 rows x
// HD/16 columns per thread -- every thread owns the same 4 rows in S and O, so the re-base of O
// stays in registers.  Fully masked key tiles are never visited; keys beyond the causal limit
// get exactly zero weight, as in the reference (model.hpp:112-158).
template <int HD>
struct TiledCfg {
    static constexpr int BQ = 64, BK = 64, THREADS = 256, OC = HD / 16;  // O columns per thread
    static constexpr int SMEM = (HD * BQ + HD * BK + BK * HD + BK * BQ) * 4;
};

template <int HD>
__global__ void __launch_bounds__(256) attn_f32_tiled_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                                            const float* __restrict__ V, float* __restrict__ O,
                                                            AttnShape sh) {
    using C = TiledCfg<HD>;
    constexpr int BQ = C::BQ, BK = C::BK, OC = C::OC;
    extern __shared__ __align__(16) float smem_f[];
    float* sQ = smem_f;            // [HD][BQ]  (transposed)
    float* sK = sQ + HD * BQ;      // [HD][BK]  (transposed)
    float* sV = sK + HD * BK;      // [BK][HD]
    float* sP = sV + BK * HD;      // [BK][BQ]
    const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
    const int h = blockIdx.x;
    const int nqb = static_cast<int>((sh.q_rows + BQ - 1) / BQ);
    const int64_t q0 = static_cast<int64_t>(nqb - 1 - static_cast<int>(blockIdx.y)) * BQ;  // heavy blocks first
    const int g = h / (sh.n_heads / sh.n_kv_heads);
    const float* qb = Q + static_cast<int64_t>(h) * HD;
    const float* kb = K + static_cast<int64_t>(g) * HD;
    const float* vb = V + static_cast<int64_t>(g) * HD;
    // Q block -> sQ[d][r]: rows fastest across lanes, so the transposed stores hit 32 banks
    for (int e = tid; e < BQ * HD / 4; e += 256) {
        const int r = e % BQ, d = (e / BQ) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q0 + r < sh.q_rows) v = *reinterpret_cast<const float4*>(qb + (q0 + r) * sh.ldq + d);
        sQ[(d + 0) * BQ + r] = v.x;
        sQ[(d + 1) * BQ + r] = v.y;
        sQ[(d + 2) * BQ + r] = v.z;
        sQ[(d + 3) * BQ + r] = v.w;
    }
    const float scale = 1.0f / sqrtf(static_cast<float>(HD));
    int64_t last = sh.offset + q0 + BQ - 1;  // last visible key of the block
    if (last > sh.k_rows - 1) last = sh.k_rows - 1;
    const int n_tiles = static_cast<int>(last / BK) + 1;
    float m[4], l[4], acc[4][OC];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.f;
#pragma unroll
        for (int c = 0; c < OC; ++c) acc[i][c] = 0.f;
    }
    for (int t = 0; t < n_tiles; ++t) {
        const int64_t k0 = static_cast<int64_t>(t) * BK;
        __syncthreads();  // the previous tile's PV is done with sV / sP (and sQ is written)
        for (int e = tid; e < BK * HD / 4; e += 256) {  // K transposed: keys fastest across lanes
            const int r = e % BK, d = (e / BK) * 4;
            float4 kv4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k0 + r < sh.k_rows) kv4 = *reinterpret_cast<const float4*>(kb + (k0 + r) * sh.ldkv + d);
            sK[(d + 0) * BK + r] = kv4.x;
            sK[(d + 1) * BK + r] = kv4.y;
            sK[(d + 2) * BK + r] = kv4.z;
            sK[(d + 3) * BK + r] = kv4.w;
        }
        for (int e = tid; e < BK * HD / 4; e += 256) {  // V as is: dims fastest (coalesced)
            const int r = e / (HD / 4), d = (e % (HD / 4)) * 4;
            float4 vv4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k0 + r < sh.k_rows) vv4 = *reinterpret_cast<const float4*>(vb + (k0 + r) * sh.ldkv + d);
            *reinterpret_cast<float4*>(sV + r * HD + d) = vv4;
        }
        __syncthreads();
        float sc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) sc[i][j] = 0.f;
#pragma unroll 8
        for (int d = 0; d < HD; ++d) {
            const float4 a = *reinterpret_cast<const float4*>(sQ + d * BQ + tr * 4);
            const float4 b = *reinterpret_cast<const float4*>(sK + d * BK + tc * 4);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) sc[i][j] = fmaf(av[i], bv[j], sc[i][j]);
        }
        float alpha[4], ps[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t qabs = sh.offset + q0 + tr * 4 + i;
            float mx = -INFINITY;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t key = k0 + tc * 4 + j;
                sc[i][j] = (key <= qabs && key < sh.k_rows) ? sc[i][j] * scale : -INFINITY;
                mx = fmaxf(mx, sc[i][j]);
            }
#pragma unroll
            for (int o = 8; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float m_new = fmaxf(m[i], mx);  // finite: key 0 is visible to every row
            alpha[i] = expf(m[i] - m_new);
            m[i] = m_new;
            ps[i] = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sc[i][j] = sc[i][j] == -INFINITY ? 0.f : expf(sc[i][j] - m_new);
                ps[i] += sc[i][j];
            }
        }
        // P -> sP[key][row group]: one float4 (4 rows) per key, row group XOR-swizzled by the
        // key's group of 4 so the 8 lanes of each store phase hit 8 different bank groups
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int key = tc * 4 + j;
            *reinterpret_cast<float4*>(sP + (key * (BQ / 4) + (tr ^ tc)) * 4) =
                make_float4(sc[0][j], sc[1][j], sc[2][j], sc[3][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int o = 8; o; o >>= 1) ps[i] += __shfl_xor_sync(0xffffffffu, ps[i], o);
            l[i] = l[i] * alpha[i] + ps[i];
#pragma unroll
            for (int c = 0; c < OC; ++c) acc[i][c] *= alpha[i];
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < BK; ++k) {
            const float4 p4 = *reinterpret_cast<const float4*>(sP + (k * (BQ / 4) + (tr ^ (k >> 2))) * 4);
            const float pv[4] = {p4.x, p4.y, p4.z, p4.w};
            float vv[OC];
#pragma unroll
            for (int c = 0; c < OC; c += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(sV + k * HD + (c / 4) * 64 + tc * 4);
                vv[c] = v4.x;
                vv[c + 1] = v4.y;
                vv[c + 2] = v4.z;
                vv[c + 3] = v4.w;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int c = 0; c < OC; ++c) acc[i][c] = fmaf(pv[i], vv[c], acc[i][c]);
        }
    }
    // thread (tr, tc) holds rows tr*4+i, columns (c/4)*64 + tc*4 + c%4
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = q0 + tr * 4 + i;
        if (r >= sh.q_rows) continue;
        const float inv = 1.0f / l[i];
        float* orow = O + r * sh.ldo + static_cast<int64_t>(h) * HD;
#pragma unroll
        for (int c = 0; c < OC; c += 4)
            *reinterpret_cast<float4*>(orow + (c / 4) * 64 + tc * 4) =
                make_float4(acc[i][c] * inv, acc[i][c + 1] * inv, acc[i][c + 2] * inv, acc[i][c + 3] * inv);
    }
}

template <int HD>
void launch_tiled(const float* Q, const float* K, const float* V, float* O, const AttnShape& sh, cudaStream_t s) {
    using C = TiledCfg<HD>;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        cudaFuncSetAttribute(attn_f32_tiled_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        configured = dev;
    }
    dim3 grid(static_cast<unsigned>(sh.n_heads), static_cast<unsigned>((sh.q_rows + C::BQ - 1) / C::BQ));
    note_launch();
    attn_f32_tiled_kernel<HD><<<grid, C::THREADS, C::SMEM, s>>>(Q, K, V, O, sh);
}

template <typename T>
void launch(const T* Q, const T* K, const T* V, T* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    dim3 grid(static_cast<unsigned>((sh.q_rows + WARPS - 1) / WARPS), static_cast<unsigned>(sh.n_heads));
    note_launch();
    attn_simt_kernel<T><<<grid, WARPS * 32, 0, s>>>(Q, K, V, O, sh);
}

}  // namespace

void attn_simt_f32(const float* Q, const float* K, const float* V, float* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    // the tiled kernel reads rows as float4: 16-byte aligned rows and bases
    const bool aligned = sh.ldq % 4 == 0 && sh.ldkv % 4 == 0 && sh.ldo % 4 == 0 &&
                         ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(K) |
                           reinterpret_cast<uintptr_t>(V) | reinterpret_cast<uintptr_t>(O)) & 15) == 0;
    if (aligned && sh.head_dim == 128) return launch_tiled<128>(Q, K, V, O, sh, s);
    if (aligned && sh.head_dim == 64) return launch_tiled<64>(Q, K, V, O, sh, s);
    launch<float>(Q, K, V, O, sh, s);
}

void attn_simt_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    launch<bf16>(Q, K, V, O, sh, s);
}

}  // namespace kvp
