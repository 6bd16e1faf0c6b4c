// weights.cu -- init_weights (weights.hpp:41-83) generated ON the device.
//
// SplitMix64 is a counter generator: the k-th draw of a stream seeded s is
// mix(s + (k+1) * 0x9e3779b97f4a7c15), so every element is generated independently and
// the whole 8.6 GB Llama-7B bf16 weight set materialises in HBM in milliseconds instead of
// the reference's ~0.9 s/layer host loop.  The arithmetic is the reference's, in IEEE
// double ((z >> 11) * 2^-53, 2u - 1, * scale) followed by one RN cast to float, so the f32
// values are bit-identical to init_weights<float>; bf16 mode is an RNE cast of those.
#include "kernels.cuh"

namespace kvp {

__device__ __forceinline__ float seeded_value(uint64_t stream_seed, uint64_t k, double scale) {
    uint64_t z = stream_seed + (k + 1ull) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z = z ^ (z >> 31);
    const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    const double sym = __dsub_rn(__dmul_rn(2.0, u), 1.0);
    return __double2float_rn(__dmul_rn(sym, scale));
}

__global__ void seeded_f32_kernel(float* out, int64_t n, double scale, uint64_t seed) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = seeded_value(seed, static_cast<uint64_t>(k), scale);
}

// Output index o = c * rows + r of the transposed matrix <- reference element k = r * cols + c.
__global__ void seeded_bf16_t_kernel(bf16* out_t, int64_t rows, int64_t cols, double scale, uint64_t seed) {
    const int64_t n = rows * cols;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = o / rows, r = o - c * rows;
        out_t[o] = __float2bfloat16_rn(seeded_value(seed, static_cast<uint64_t>(r * cols + c), scale));
    }
}

__global__ void transpose_bf16_kernel(const float* in, int64_t rows, int64_t cols, bf16* out_t) {
    __shared__ float tile[32][33];
    const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out_t[c * rows + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
}

static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return static_cast<int>(b > 148 * 64 ? 148 * 64 : (b < 1 ? 1 : b));
}

void launch_seeded_f32(float* out, int64_t rows, int64_t cols, double scale, uint64_t seed, cudaStream_t s) {
    note_launch();
    seeded_f32_kernel<<<grid_for(rows * cols), 256, 0, s>>>(out, rows * cols, scale, seed);
}

void launch_seeded_bf16_t(bf16* out_t, int64_t rows, int64_t cols, double scale, uint64_t seed,
                          int64_t t_row_off, cudaStream_t s) {
    note_launch();
    seeded_bf16_t_kernel<<<grid_for(rows * cols), 256, 0, s>>>(out_t + t_row_off * rows, rows, cols, scale, seed);
}

void launch_transpose_to_bf16(const float* in, int64_t rows, int64_t cols, bf16* out_t, int64_t t_row_off,
                              cudaStream_t s) {
    note_launch();
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out_t + t_row_off * rows);
}

}  // namespace kvp
