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

template <typename T>
void launch(const T* Q, const T* K, const T* V, T* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    dim3 grid(static_cast<unsigned>((sh.q_rows + WARPS - 1) / WARPS), static_cast<unsigned>(sh.n_heads));
    note_launch();
    attn_simt_kernel<T><<<grid, WARPS * 32, 0, s>>>(Q, K, V, O, sh);
}

}  // namespace

void attn_simt_f32(const float* Q, const float* K, const float* V, float* O, const AttnShape& sh, cudaStream_t s) {
    launch<float>(Q, K, V, O, sh, s);
}

void attn_simt_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    launch<bf16>(Q, K, V, O, sh, s);
}

}  // namespace kvp
