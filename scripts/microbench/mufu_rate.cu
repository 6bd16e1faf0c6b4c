// MUFU.EX2 issue rate per SMSP on sm_100a: one CTA per SM, W warps per SMSP, each thread
// runs 64 independent ex2 per iteration (plus the softmax companions: FFMA2 for x, FADD2
// for the row sum, F2FP pack) -- clocks per warp-instruction of MUFU.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pk(float a, float b) { unsigned r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r; }

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = -0.001f * (threadIdx.x + i);
    float acc = 0.f; unsigned px = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float nb = -1e-7f * it;
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
            float a = fmaf(v[i], 0.127f, nb), b = fmaf(v[i + 1], 0.127f, nb);
            float ea = ex2(a), eb = ex2(b);
            if (MODE >= 1) { acc += ea + eb; }
            if (MODE >= 2) { px ^= pk(ea, eb); }
            if (MODE == 0) { v[i] = ea; v[i + 1] = eb; }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (float)(px & 1) + v[threadIdx.x & 63];
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    long long h[148];
    const int iters = 2000;
    for (int mode = 0; mode < 3; ++mode)
        for (int wps = 1; wps <= 4; wps *= 2) {
            const int threads = 128 * wps;
            auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
            kern<<<148, threads>>>(out, 10, cyc);
            kern<<<148, threads>>>(out, iters, cyc);
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
            const double mufu_per_smsp = double(iters) * 64 * wps;  // warp-instructions per SMSP
            printf("mode %d (%s) warps/SMSP %d: %.2f clk per MUFU warp-instr per SMSP (%.1f ex2/clk/SM)\n", mode,
                   mode == 0 ? "ex2 only" : mode == 1 ? "+sum" : "+sum+pack", wps, c / mufu_per_smsp,
                   4 * 32 * mufu_per_smsp / c);
        }
    return 0;
}
