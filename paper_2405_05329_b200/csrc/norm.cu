// norm.cu -- rms_norm_rows (model.hpp:29-40, gain-free, eps 1e-6) fused with the bf16
// cast that feeds the next tcgen05 GEMM, plus the bit-exact f32 parity variant.
// HBM-bound: 4 B read + 2 B written per element (bf16 path).
#include "kernels.cuh"

namespace kvp {

// One warp per row, 16-byte vector loads (cols % 4 == 0) with a scalar tail path.
__global__ void norm_cast_bf16_kernel(const float* __restrict__ x, bf16* __restrict__ y, int64_t rows,
                                      int64_t cols, int norm) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int lane = threadIdx.x & 31;
    const bool vec = (cols % 4) == 0;
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
        const float* xr = x + r * cols;
        bf16* yr = y + r * cols;
        float inv = 1.0f;
        if (norm) {
            float ss = 0.f;
            if (vec) {
                for (int64_t c = lane * 4; c < cols; c += 128) {
                    const float4 v = *reinterpret_cast<const float4*>(xr + c);
                    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
                }
            } else {
                for (int64_t c = lane; c < cols; c += 32) ss += xr[c] * xr[c];
            }
            for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            inv = 1.0f / sqrtf(ss / static_cast<float>(cols) + 1e-6f);
        }
        if (vec) {
            for (int64_t c = lane * 4; c < cols; c += 128) {
                const float4 v = *reinterpret_cast<const float4*>(xr + c);
                __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv, v.y * inv);
                __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv, v.w * inv);
                uint2 packed;
                packed.x = *reinterpret_cast<uint32_t*>(&a);
                packed.y = *reinterpret_cast<uint32_t*>(&b);
                *reinterpret_cast<uint2*>(yr + c) = packed;
            }
        } else {
            for (int64_t c = lane; c < cols; c += 32) yr[c] = __float2bfloat16_rn(xr[c] * inv);
        }
    }
}

// Reference order: mean_sq += x*x sequentially in column order (no FMA), /= cols,
// inv = 1 / sqrt(mean_sq + 1e-6), y = x * inv.  One thread per row.
__global__ void norm_f32_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* xr = x + r * cols;
    float ms = 0.f;
    for (int64_t c = 0; c < cols; ++c) ms = __fadd_rn(ms, __fmul_rn(xr[c], xr[c]));
    ms = __fdiv_rn(ms, static_cast<float>(cols));
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, 1e-6f)));
    for (int64_t c = 0; c < cols; ++c) y[r * cols + c] = __fmul_rn(xr[c], inv);
}

// One warp per row; each 64-column group is one float2 per lane, reduced in a fixed
// shuffle order (deterministic).
__global__ void prep_bf16_ssq_kernel(const float* __restrict__ x, bf16* __restrict__ y, float* __restrict__ ssq,
                                     int64_t rows, int64_t cols) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int lane = threadIdx.x & 31;
    const int parts = static_cast<int>((cols + 63) / 64);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
        const float* xr = x + r * cols;
        bf16* yr = y + r * cols;
        for (int g = 0; g < parts; ++g) {
            const int64_t c = static_cast<int64_t>(g) * 64 + lane * 2;
            float ss = 0.f;
            if (c < cols) {
                const float2 v = *reinterpret_cast<const float2*>(xr + c);
                ss = v.x * v.x + v.y * v.y;
                __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
                *reinterpret_cast<__nv_bfloat162*>(yr + c) = a;
            }
            for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            if (lane == 0) ssq[r * parts + g] = ss;
        }
    }
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, bf16* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __float2bfloat16_rn(x[i]);
}

__global__ void cast_f32_kernel(const bf16* __restrict__ x, float* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __bfloat162float(x[i]);
}

static int blocks_for(int64_t n, int per_block) {
    int64_t b = (n + per_block - 1) / per_block;
    if (b > 148 * 32) b = 148 * 32;
    return static_cast<int>(b < 1 ? 1 : b);
}

void launch_norm_cast_bf16(const float* x, bf16* y, int64_t rows, int64_t cols, bool norm, cudaStream_t s) {
    if (rows <= 0) return;
    note_launch();
    norm_cast_bf16_kernel<<<blocks_for(rows, 8), 256, 0, s>>>(x, y, rows, cols, norm ? 1 : 0);
}

void launch_norm_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t s) {
    if (rows <= 0) return;
    note_launch();
    norm_f32_kernel<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, s>>>(x, y, rows, cols);
}

void launch_cast_bf16(const float* x, bf16* y, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    note_launch();
    cast_bf16_kernel<<<blocks_for(n, 256), 256, 0, s>>>(x, y, n);
}

void launch_prep_bf16_ssq(const float* x, bf16* y, float* ssq, int64_t rows, int64_t cols, cudaStream_t s) {
    if (rows <= 0) return;
    note_launch();
    prep_bf16_ssq_kernel<<<blocks_for(rows, 8), 256, 0, s>>>(x, y, ssq, rows, cols);
}

void launch_cast_f32(const bf16* x, float* y, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    note_launch();
    cast_f32_kernel<<<blocks_for(n, 256), 256, 0, s>>>(x, y, n);
}

// Timing helper: one thread spins on the global timer for ns nanoseconds, so the host can
// enqueue the timed launches (tensor-map encodes, launch calls) while the stream is busy and
// the events around them see device time only.
__global__ void spin_kernel(uint64_t ns) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
        __nanosleep(1000);
    }
}

void launch_spin(uint64_t ns, cudaStream_t s) { spin_kernel<<<1, 32, 0, s>>>(ns); }

}  // namespace kvp
