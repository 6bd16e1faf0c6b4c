// gemm_simt.cu -- fp32 parity-mode GEMM (Precision::f32, config.hpp:10).
//
// The reference matmul (matrix.hpp:76-91) accumulates out[i][j] += a[i][k] * b[k][j] in
// ascending k with a rounded multiply and a rounded add.  This kernel keeps exactly that
// per-element order (__fmul_rn / __fadd_rn, no FMA contraction), so every projection of the
// fp32 mode is bit-identical to the reference; only the attention exp differs in ulps.
#include "kernels.cuh"

namespace kvp {

namespace {
// 128 x 128 output tile per 256-thread CTA, 8 x 8 outputs per thread (two 4-row x two 4-column
// groups 64 apart, so the operand reads are conflict-free LDS.128), k staged through smem in
// slabs of 16 with the next slab's global loads in flight in registers.  Per k each thread
// issues 4 LDS.128 for 64 multiply + 64 add instructions.
constexpr int TM = 128, TN = 128, TK = 16;

template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t M, int64_t K,
                                                       int64_t lda, const float* __restrict__ B, int64_t N,
                                                       float* __restrict__ Cm, int64_t ldc,
                                                       const float* __restrict__ resid, int64_t ldr) {
    __shared__ __align__(16) float sA[2][TK][TM];  // A slab transposed: [k][row]
    __shared__ __align__(16) float sB[2][TK][TN];  // B slab: [k][col]
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t m0 = blockIdx.y * (int64_t)TM, n0 = blockIdx.x * (int64_t)TN;
    // global -> register staging: A: 128 rows x 16 k = 512 float4 (2 per thread, k-contiguous);
    // B: 16 k x 128 cols = 512 float4 (2 per thread, column-contiguous).  Vector loads only when
    // the row stride keeps them 16-byte aligned; tails are zero-filled.
    const bool a_vec = (lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    const bool b_vec = (N % 4 == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
    float4 ra[2], rb[2];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int e = tid + t * 256;
            const int r = e >> 2, c = (e & 3) * 4;  // A: row r, k offset c
            const int64_t gr = m0 + r, gc = k0 + c;
            if (a_vec && gr < M && gc + 3 < K) {
                ra[t] = __ldg(reinterpret_cast<const float4*>(A + gr * lda + gc));
            } else {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = (gr < M && gc + q < K) ? A[gr * lda + gc + q] : 0.f;
                ra[t] = make_float4(v[0], v[1], v[2], v[3]);
            }
            const int kr = e >> 5, cc = (e & 31) * 4;  // B: k row kr, column cc
            const int64_t bk = k0 + kr, bc = n0 + cc;
            if (b_vec && bk < K && bc + 3 < N) {
                rb[t] = __ldg(reinterpret_cast<const float4*>(B + bk * N + bc));
            } else {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = (bk < K && bc + q < N) ? B[bk * N + bc + q] : 0.f;
                rb[t] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int e = tid + t * 256;
            const int r = e >> 2, c = (e & 3) * 4;
            sA[buf][c + 0][r] = ra[t].x;
            sA[buf][c + 1][r] = ra[t].y;
            sA[buf][c + 2][r] = ra[t].z;
            sA[buf][c + 3][r] = ra[t].w;
            const int kr = e >> 5, cc = (e & 31) * 4;
            *reinterpret_cast<float4*>(&sB[buf][kr][cc]) = rb[t];
        }
    };
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    load(0);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = 0; k0 < K; k0 += TK) {
        const bool more = k0 + TK < K;
        if (more) load(k0 + TK);  // in flight while this slab is consumed
        const int kk = (K - k0) < TK ? static_cast<int>(K - k0) : TK;
        // ascending k, a rounded multiply then a rounded add: matrix.hpp:76-91's order exactly
#pragma unroll 4
        for (int k = 0; k < kk; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&sA[buf][k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&sA[buf][k][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&sB[buf][k][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&sB[buf][k][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
        if (more) {
            stash(buf ^ 1);  // the other buffer: last read one iteration ago, before this sync
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (c >= N) continue;
            float v = acc[i][j];
            if constexpr (EPI == SEPI_RESID) v = __fadd_rn(resid[r * ldr + c], v);
            if constexpr (EPI == SEPI_RELU) v = v < 0.f ? 0.f : v;  // relu, model.hpp:47-52
            Cm[r * ldc + c] = v;
        }
    }
}
}  // namespace

void gemm_f32_simt(const float* A, int64_t M, int64_t K, int64_t lda, const float* B, int64_t N, float* Cm,
                   int64_t ldc, int epi, const float* resid, int64_t ldr, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    dim3 grid(static_cast<unsigned>((N + TN - 1) / TN), static_cast<unsigned>((M + TM - 1) / TM));
    note_launch();
    switch (epi) {
        case SEPI_RESID: gemm_f32_kernel<SEPI_RESID><<<grid, 256, 0, s>>>(A, M, K, lda, B, N, Cm, ldc, resid, ldr); break;
        case SEPI_RELU: gemm_f32_kernel<SEPI_RELU><<<grid, 256, 0, s>>>(A, M, K, lda, B, N, Cm, ldc, resid, ldr); break;
        default: gemm_f32_kernel<SEPI_STORE><<<grid, 256, 0, s>>>(A, M, K, lda, B, N, Cm, ldc, resid, ldr); break;
    }
}

}  // namespace kvp
