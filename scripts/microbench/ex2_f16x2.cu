// MUFU exp2 throughput on one SM: ex2.approx.ftz.f32 (1 result / lane / instruction) against
// ex2.approx.f16x2 (2 results / lane / instruction).  16 warps per CTA, 1 CTA, 8 independent
// chains per thread; prints results per clock per SM for each form.
#include <cstdio>
#include <cuda_fp16.h>

__global__ void k_f32(float* out, long long* clk, int iters) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    __syncthreads();
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += v[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *clk = t1 - t0;
}

__global__ void k_f16x2(float* out, long long* clk, int iters) {
    unsigned v[8];
    for (int i = 0; i < 8; ++i) {
        __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f * (threadIdx.x + i));
        v[i] = *reinterpret_cast<unsigned*>(&h);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
    __syncthreads();
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) {
        __half2 h = *reinterpret_cast<__half2*>(&v[i]);
        s += __low2float(h) + __high2float(h);
    }
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *clk = t1 - t0;
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 4096 * 4);
    cudaMalloc(&clk, 8);
    const int iters = 4096, threads = 512;
    for (int form = 0; form < 2; ++form) {
        for (int rep = 0; rep < 2; ++rep) {
            if (form == 0) k_f32<<<1, threads>>>(out, clk, iters);
            else k_f16x2<<<1, threads>>>(out, clk, iters);
        }
        long long c = 0;
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double results = double(threads) * iters * 8 * (form ? 2 : 1);
        printf("%s: %.2f results/clk/SM (%.2f instr/clk/SM)\n", form ? "ex2.approx.f16x2" : "ex2.approx.ftz.f32",
               results / c, results / c / (form ? 2 : 1));
    }
    return 0;
}
