// Per-SMSP issue cost of the instructions in the attention softmax loop on sm_100a:
// cycles per warp-instruction per SMSP with 4 warps per SMSP, 8 independent chains per thread
// (throughput, not latency).  Measured with clock64 inside the kernel (no clock assumptions).
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
#define IT 256

template <int OP>
__device__ __forceinline__ void op(float (&x)[CH], float c) {
#pragma unroll
    for (int i = 0; i < CH; i += 2) {
        if (OP == 0) {  // FFMA (3 reg)
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(c), "f"(x[i + 1]));
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i + 1]) : "f"(c), "f"(x[i]));
        } else if (OP == 1) {  // FFMA2
            asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%2}; fma.rn.f32x2 a,a,b,a; mov.b64 {%0,%1},a;}"
                         : "+f"(x[i]), "+f"(x[i + 1]) : "f"(c));
        } else if (OP == 2) {  // FADD2
            asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%2}; add.rn.f32x2 a,a,b; mov.b64 {%0,%1},a;}"
                         : "+f"(x[i]), "+f"(x[i + 1]) : "f"(c));
        } else if (OP == 3) {  // FMNMX
            asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(x[i + 1]));
            asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i + 1]) : "f"(x[i]));
        } else if (OP == 4) {  // FMNMX3
            asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(x[i + 1]), "f"(c));
            asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[i + 1]) : "f"(x[i]), "f"(c));
        } else if (OP == 5) {  // MUFU.EX2
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i + 1]));
        } else if (OP == 6) {  // F2FP pack (cvt.rn.bf16x2.f32), result fed back as float bits
            unsigned r;
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[i + 1]));
            x[i] = __uint_as_float(r);
        } else if (OP == 7) {  // SHL + IADD (exponent insert)
            unsigned u = __float_as_uint(x[i]), v = __float_as_uint(x[i + 1]);
            asm volatile("shl.b32 %0, %0, 23; add.s32 %0, %0, %1;" : "+r"(u) : "r"(v));
            x[i] = __uint_as_float(u);
            asm volatile("shl.b32 %0, %0, 23; add.s32 %0, %0, %1;" : "+r"(v) : "r"(u));
            x[i + 1] = __uint_as_float(v);
        } else if (OP == 8) {  // IMAD exponent insert: u = u * 2^23 + v
            unsigned u = __float_as_uint(x[i]), v = __float_as_uint(x[i + 1]);
            asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(u) : "r"(v));
            x[i] = __uint_as_float(u);
            asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(v) : "r"(u));
            x[i + 1] = __uint_as_float(v);
        } else if (OP == 9) {  // HFMA2 (f16x2)
            unsigned u = __float_as_uint(x[i]), v = __float_as_uint(x[i + 1]);
            asm volatile("fma.rn.f16x2 %0, %0, %1, %0;" : "+r"(u) : "r"(v));
            asm volatile("fma.rn.f16x2 %0, %0, %1, %0;" : "+r"(v) : "r"(u));
            x[i] = __uint_as_float(u); x[i + 1] = __uint_as_float(v);
        } else if (OP == 10) {  // MUFU + FFMA2 interleaved 1:1
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%2}; fma.rn.f32x2 a,a,b,a; mov.b64 {%0,%1},a;}"
                         : "+f"(x[i]), "+f"(x[i + 1]) : "f"(c));
        } else if (OP == 11) {  // MUFU + FMNMX interleaved 1:1
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i + 1]) : "f"(c));
        } else if (OP == 12) {  // FFMA2 + FMNMX interleaved 1:1
            asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%2}; fma.rn.f32x2 a,a,b,a; mov.b64 {%0,%1},a;}"
                         : "+f"(x[i]), "+f"(x[i + 1]) : "f"(c));
            asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(c));
        } else if (OP == 13) {  // ex2.approx.ftz.bf16x2
            unsigned u = __float_as_uint(x[i]);
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u));
            x[i] = __uint_as_float(u);
        } else if (OP == 14) {  // FMUL2
            asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%2}; mul.rn.f32x2 a,a,b; mov.b64 {%0,%1},a;}"
                         : "+f"(x[i]), "+f"(x[i + 1]) : "f"(c));
        } else if (OP == 15) {  // add.rm.f32x2 (round-down magic add of the emulated exp2)
            asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%2}; add.rm.ftz.f32x2 a,a,b; mov.b64 {%0,%1},a;}"
                         : "+f"(x[i]), "+f"(x[i + 1]) : "f"(c));
        }
    }
}
// instructions per op() call per thread
__host__ __device__ constexpr int instrs(int o) {
    return o == 1 || o == 2 || o == 6 || o == 13 || o == 14 || o == 15 ? CH / 2 : (o == 7 ? 2 * CH : CH);
}

template <int OP>
__global__ void bench(float* out, long long* cyc, float c) {
    float x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = c * (threadIdx.x + i) * 1e-3f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < IT; ++it) op<OP>(x, c);
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, float* out, long long* cyc, int warps) {
    bench<OP><<<148, warps * 32>>>(out, cyc, 0.5f);
    bench<OP><<<148, warps * 32>>>(out, cyc, 0.5f);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double per_smsp_instr = double(IT) * instrs(OP) * (warps / 4);
    printf("%-34s warps/SMSP %2d: %6.2f clk per warp-instr per SMSP\n", name, warps / 4, m / per_smsp_instr);
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    cudaMalloc(&cyc, 148 * sizeof(long long));
    for (int w : {4, 16}) {
        run<0>("FFMA", out, cyc, w);
        run<1>("FFMA2 (f32x2)", out, cyc, w);
        run<2>("FADD2 (f32x2)", out, cyc, w);
        run<14>("FMUL2 (f32x2)", out, cyc, w);
        run<15>("FADD2.RM (f32x2)", out, cyc, w);
        run<3>("FMNMX", out, cyc, w);
        run<4>("FMNMX3", out, cyc, w);
        run<5>("MUFU.EX2", out, cyc, w);
        run<13>("ex2.bf16x2", out, cyc, w);
        run<6>("F2FP.BF16 pack", out, cyc, w);
        run<7>("SHL+IADD (per instr)", out, cyc, w);
        run<8>("IMAD", out, cyc, w);
        run<9>("HFMA2", out, cyc, w);
        run<10>("MUFU+FFMA2 1:1 (per instr)", out, cyc, w);
        run<11>("MUFU+FMNMX 1:1 (per instr)", out, cyc, w);
        run<12>("FFMA2+FMNMX 1:1 (per instr)", out, cyc, w);
    }
    return 0;
}
