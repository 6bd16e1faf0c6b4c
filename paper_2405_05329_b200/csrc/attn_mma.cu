// attn_mma.cu -- bf16 prefix-causal flash attention for head_dim 64 / 128 (first
// tensor-core version; warp-level mma.sync m16n8k16 with f32 accumulation).
//
// Reference: causal_attention (model.hpp:112-158) scores every cached key and masks with an
// additive -1e9 penalty.  Here a (64-query x 64-key) tile is only visited when at least
// one of its keys is visible to one of its queries (keys [0, offset + last query]); the
// tile that straddles the diagonal is masked element-wise against ABSOLUTE positions, so
// the arbitrary prefix offset b_i of a KV-Runahead rank costs nothing extra.
//
// Key tiles are aligned to absolute key 0 and every row's online softmax is row-local, so a
// row's output is bitwise independent of which rank / query tile computes it: Serial, TSP
// and KVR produce identical bits (the reference's own bit-exactness property,
// test_engine.cpp:50-88).  Fully masked trailing tiles leave (m, l, O) unchanged exactly.
#include <cstdlib>

#include "kernels.cuh"

namespace kvp {

namespace {

constexpr int BLOCK_M = 64;  // 4 warps x 16 query rows
constexpr int BLOCK_N = 64;  // keys per tile
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Row-major [rows x HD] bf16 tile in smem, 16-byte chunks XOR-swizzled by (row & 7).
template <int HD>
__device__ __forceinline__ uint32_t tile_off(int row, int chunk) {
    return static_cast<uint32_t>((row * (HD / 8) + (chunk ^ (row & 7))) * 16);
}

template <int HD>
__device__ __forceinline__ void load_tile(uint32_t s_base, const bf16* g, int64_t ld, int64_t row0, int64_t rows) {
    constexpr int CH = HD / 8;
    for (int e = threadIdx.x; e < BLOCK_N * CH; e += THREADS) {
        const int r = e / CH, c = e % CH;
        const int64_t gr = row0 + r;
        const bool ok = gr < rows;
        const bf16* src = g + (ok ? gr : 0) * ld + c * 8;
        cp_async16(s_base + tile_off<HD>(r, c), src, ok);
    }
}

template <int HD>
__global__ void __launch_bounds__(THREADS) attn_mma_kernel(const bf16* __restrict__ Q, const bf16* __restrict__ K,
                                                           const bf16* __restrict__ V, bf16* __restrict__ O,
                                                           AttnShape sh) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int TILE = BLOCK_N * HD * 2;
    const uint32_t sQ = smem_addr(smem);
    const uint32_t sK = sQ + TILE;      // 2 buffers
    const uint32_t sV = sK + 2 * TILE;  // 2 buffers

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_qt = static_cast<int>((sh.q_rows + BLOCK_M - 1) / BLOCK_M);
    const int qt = num_qt - 1 - static_cast<int>(blockIdx.y);  // heaviest tiles (all heads) first
    const int h = blockIdx.x;
    const int g = h / (sh.n_heads / sh.n_kv_heads);
    const int64_t q0 = static_cast<int64_t>(qt) * BLOCK_M;
    const int64_t last_q = (q0 + BLOCK_M - 1 < sh.q_rows - 1) ? q0 + BLOCK_M - 1 : sh.q_rows - 1;
    const int64_t max_key = sh.offset + last_q;  // highest visible key of this tile
    const int n_kt = static_cast<int>(max_key / BLOCK_N) + 1;

    const bf16* Qh = Q + static_cast<int64_t>(h) * HD;
    const bf16* Kh = K + static_cast<int64_t>(g) * HD;
    const bf16* Vh = V + static_cast<int64_t>(g) * HD;

    load_tile<HD>(sQ, Qh + q0 * sh.ldq, sh.ldq, 0, sh.q_rows - q0);
    load_tile<HD>(sK, Kh, sh.ldkv, 0, sh.k_rows);
    load_tile<HD>(sV, Vh, sh.ldkv, 0, sh.k_rows);
    cp_commit();

    // softmax in log2 domain: p = 2^(s*scale*log2e - m*scale*log2e)
    const float sl2 = (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f;
    const int64_t row_a = sh.offset + q0 + warp * 16 + (lane >> 2);  // absolute query positions
    const int64_t row_b = row_a + 8;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    uint32_t qf[HD / 16][4];

    for (int kt = 0; kt < n_kt; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < n_kt) {
            load_tile<HD>(sK + (buf ^ 1) * TILE, Kh, sh.ldkv, static_cast<int64_t>(kt + 1) * BLOCK_N, sh.k_rows);
            load_tile<HD>(sV + (buf ^ 1) * TILE, Vh, sh.ldkv, static_cast<int64_t>(kt + 1) * BLOCK_N, sh.k_rows);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kt == 0) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const int r = warp * 16 + (lane & 15);
                const int c = kk * 2 + (lane >> 4);
                ldsm_x4(sQ + tile_off<HD>(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
            }
        }
        // S = Q K^T for 16 rows x 64 keys per warp
        float s[BLOCK_N / 8][4];
#pragma unroll
        for (int i = 0; i < BLOCK_N / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
        const uint32_t kb = sK + buf * TILE;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
            for (int nt = 0; nt < BLOCK_N / 8; nt += 2) {
                const int r = nt * 8 + (lane & 7) + ((lane >> 4) << 3);
                const int c = kk * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kb + tile_off<HD>(r, c), b0, b1, b2, b3);
                mma16816(s[nt], qf[kk], b0, b1);
                mma16816(s[nt + 1], qf[kk], b2, b3);
            }
        }
        // mask against absolute positions (only the tile crossing the diagonal needs it)
        const int64_t key0 = static_cast<int64_t>(kt) * BLOCK_N;
        if (key0 + BLOCK_N - 1 > sh.offset + q0 + warp * 16) {
#pragma unroll
            for (int nt = 0; nt < BLOCK_N / 8; ++nt) {
                const int64_t j = key0 + nt * 8 + 2 * (lane & 3);
                if (j > row_a) s[nt][0] = -INFINITY;
                if (j + 1 > row_a) s[nt][1] = -INFINITY;
                if (j > row_b) s[nt][2] = -INFINITY;
                if (j + 1 > row_b) s[nt][3] = -INFINITY;
            }
        }
        float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < BLOCK_N / 8; ++nt) {
            mx_a = fmaxf(mx_a, fmaxf(s[nt][0], s[nt][1]));
            mx_b = fmaxf(mx_b, fmaxf(s[nt][2], s[nt][3]));
        }
        mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
        mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
        mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
        mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
        const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
        const float base_a = (mn_a == -INFINITY) ? 0.f : mn_a * sl2;
        const float base_b = (mn_b == -INFINITY) ? 0.f : mn_b * sl2;
        const float al_a = exp2f(m_a * sl2 - base_a), al_b = exp2f(m_b * sl2 - base_b);
        m_a = mn_a;
        m_b = mn_b;
        l_a *= al_a;
        l_b *= al_b;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= al_a;
            o[i][1] *= al_a;
            o[i][2] *= al_b;
            o[i][3] *= al_b;
        }
        uint32_t pf[BLOCK_N / 16][4];
#pragma unroll
        for (int nt = 0; nt < BLOCK_N / 8; ++nt) {
            const float p0 = exp2f(fmaf(s[nt][0], sl2, -base_a));
            const float p1 = exp2f(fmaf(s[nt][1], sl2, -base_a));
            const float p2 = exp2f(fmaf(s[nt][2], sl2, -base_b));
            const float p3 = exp2f(fmaf(s[nt][3], sl2, -base_b));
            l_a += p0 + p1;
            l_b += p2 + p3;
            pf[nt >> 1][(nt & 1) * 2 + 0] = pack2(p0, p1);
            pf[nt >> 1][(nt & 1) * 2 + 1] = pack2(p2, p3);
        }
        // O += P V
        const uint32_t vb = sV + buf * TILE;
#pragma unroll
        for (int kc = 0; kc < BLOCK_N / 16; ++kc) {
#pragma unroll
            for (int dt = 0; dt < HD / 8; dt += 2) {
                const int r = kc * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = dt + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vb + tile_off<HD>(r, c), b0, b1, b2, b3);
                mma16816(o[dt], pf[kc], b0, b1);
                mma16816(o[dt + 1], pf[kc], b2, b3);
            }
        }
        __syncthreads();
    }
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    const float inv_a = 1.f / l_a, inv_b = 1.f / l_b;
    const int64_t ra = q0 + warp * 16 + (lane >> 2), rb = ra + 8;
    bf16* Oh = O + static_cast<int64_t>(h) * HD;
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt) {
        const int col = dt * 8 + 2 * (lane & 3);
        if (ra < sh.q_rows)
            *reinterpret_cast<uint32_t*>(Oh + ra * sh.ldo + col) = pack2(o[dt][0] * inv_a, o[dt][1] * inv_a);
        if (rb < sh.q_rows)
            *reinterpret_cast<uint32_t*>(Oh + rb * sh.ldo + col) = pack2(o[dt][2] * inv_b, o[dt][3] * inv_b);
    }
}

template <int HD>
void launch(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    constexpr int smem = 5 * BLOCK_N * HD * 2;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        cudaFuncSetAttribute(attn_mma_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        configured = dev;
    }
    dim3 grid(static_cast<unsigned>(sh.n_heads), static_cast<unsigned>((sh.q_rows + BLOCK_M - 1) / BLOCK_M));
    note_launch();
    attn_mma_kernel<HD><<<grid, THREADS, smem, s>>>(Q, K, V, O, sh);
}

}  // namespace

bool attn_bf16_supported(int head_dim) { return head_dim == 64 || head_dim == 128; }

void attn_bf16_mma(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    if (sh.head_dim == 128)
        launch<128>(Q, K, V, O, sh, s);
    else if (sh.head_dim == 64)
        launch<64>(Q, K, V, O, sh, s);
    else
        attn_simt_bf16(Q, K, V, O, sh, s);
}

// tcgen05 kernel by default; KVP_ATTN=mma selects the warp-level mma.sync kernel (A/B runs).
void attn_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    static const bool use_mma = [] {
        const char* e = getenv("KVP_ATTN");
        return e && e[0] == 'm';
    }();
    if (!use_mma && attn_tc_supported(sh.head_dim))
        attn_bf16_tc(Q, K, V, O, sh, s);
    else
        attn_bf16_mma(Q, K, V, O, sh, s);
}

}  // namespace kvp
