// gemm_simt.cu -- fp32 parity-mode GEMM (Precision::f32, config.hpp:10).
//
// The reference matmul (matrix.hpp:76-91) accumulates out[i][j] += a[i][k] * b[k][j] in
// ascending k with a rounded multiply and a rounded add.  This kernel keeps exactly that
// per-element order (__fmul_rn / __fadd_rn, no FMA contraction), so every projection of the
// fp32 mode is bit-identical to the reference; only the attention exp differs in ulps.
// 64 x 64 output tile per 256-thread CTA, 4 x 4 per thread, k staged through smem.
#include "kernels.cuh"

namespace kvp {

namespace {
constexpr int TM = 64, TN = 64, TK = 16;

template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t M, int64_t K,
                                                       int64_t lda, const float* __restrict__ B, int64_t N,
                                                       float* __restrict__ Cm, int64_t ldc,
                                                       const float* __restrict__ resid, int64_t ldr) {
    __shared__ float sA[TK][TM + 4];
    __shared__ float sB[TK][TN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = blockIdx.y * (int64_t)TM, n0 = blockIdx.x * (int64_t)TN;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int64_t k0 = 0; k0 < K; k0 += TK) {
        for (int e = threadIdx.x; e < TM * TK; e += 256) {
            const int r = e / TK, c = e % TK;
            const int64_t gr = m0 + r, gc = k0 + c;
            sA[c][r] = (gr < M && gc < K) ? A[gr * lda + gc] : 0.f;
        }
        for (int e = threadIdx.x; e < TK * TN; e += 256) {
            const int r = e / TN, c = e % TN;
            const int64_t gr = k0 + r, gc = n0 + c;
            sB[r][c] = (gr < K && gc < N) ? B[gr * N + gc] : 0.f;
        }
        __syncthreads();
        const int kk = (K - k0) < TK ? static_cast<int>(K - k0) : TK;
        for (int k = 0; k < kk; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sA[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sB[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = m0 + ty * 4 + i;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = n0 + tx * 4 + j;
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
