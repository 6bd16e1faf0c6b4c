// kernels.cuh -- host launchers for the sm_100a kernels of the per-rank layer executor.
// Every launcher enqueues on the given stream and never synchronises.  Shapes: rows are
// tokens (token-major, row-major everywhere, like the reference Matrix<T>, matrix.hpp:15).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace kvp {

using bf16 = __nv_bfloat16;

// Counts every kernel launch issued by this library (the bench's gpu_launches claim).
void note_launch();
int64_t launch_count();
// Programmatic dependent launch for the tcgen05 kernels (KVP_PDL=0 disables).
bool pdl_enabled();

// ---------------------------------------------------------------- weights.cu
// Fills a rows x cols matrix from init_weights' SplitMix64 stream (weights.hpp:41-47),
// value = float((2u - 1) * scale).  f32 variant writes the reference [rows x cols] layout;
// bf16 variant writes the TRANSPOSED [cols x rows] K-major layout used as the tcgen05 B
// operand, at row offset `t_row_off` of a packed matrix with leading dimension `ld` (= rows).
void launch_seeded_f32(float* out, int64_t rows, int64_t cols, double scale, uint64_t stream_seed,
                       cudaStream_t s);
void launch_seeded_bf16_t(bf16* out_t, int64_t rows, int64_t cols, double scale, uint64_t stream_seed,
                          int64_t t_row_off, cudaStream_t s);
// Host f32 [rows x cols] (already on device) -> bf16 transposed at row offset.
void launch_transpose_to_bf16(const float* in, int64_t rows, int64_t cols, bf16* out_t, int64_t t_row_off,
                              cudaStream_t s);

// ---------------------------------------------------------------- norm.cu
// y = bf16(x * (mean(x^2) + 1e-6)^-1/2) if norm else bf16(x)  (model.hpp:29-45 + cast).
void launch_norm_cast_bf16(const float* x, bf16* y, int64_t rows, int64_t cols, bool norm, cudaStream_t s);
// f32 rms_norm_rows with the reference's sequential accumulation order (bit-exact).
void launch_norm_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t s);
void launch_cast_bf16(const float* x, bf16* y, int64_t n, cudaStream_t s);
// y = bf16(x) and ssq[r, g] = sum of x^2 over columns [64g, 64g+64) of row r (the layer-0
// input of the fused-norm pipeline; later layers get both from the GEMM epilogues).
void launch_prep_bf16_ssq(const float* x, bf16* y, float* ssq, int64_t rows, int64_t cols, cudaStream_t s);
void launch_cast_f32(const bf16* x, float* y, int64_t n, cudaStream_t s);
// timing helper (not counted as a product launch): keeps the stream busy for ns nanoseconds
void launch_spin(uint64_t ns, cudaStream_t s);

// ---------------------------------------------------------------- gemm_tc.cu
// D = A[M x K] . B[N x K]^T on tcgen05 (bf16 in, f32 accumulate in TMEM), epilogue fused.
enum GemmEpi : int {
    EPI_QKV = 0,    // split bf16 store: cols [0,n0) -> out0, [n0,n0+n1) -> out1, rest -> out2
    EPI_RESID = 1,  // outf[r, c] = resid[r, c] + acc   (f32, residual stream)
    EPI_RELU = 2,   // out0[r, c] = bf16(max(acc, 0))
    EPI_STORE = 3,  // out0[r, c] = bf16(acc)
};
struct GemmEpilogue {
    int kind = EPI_STORE;
    bf16* out0 = nullptr;
    int64_t ld0 = 0, n0 = 0;
    bf16* out1 = nullptr;
    int64_t ld1 = 0, n1 = 0;
    bf16* out2 = nullptr;
    int64_t ld2 = 0;
    float* outf = nullptr;
    int64_t ldf = 0;
    const float* resid = nullptr;
    int64_t ldr = 0;
    // Fused RMSNorm (model.hpp:29-45).  Producer side (EPI_RESID): also write bf16(out) to
    // outb and per-row partial sums of squares over each 64-column group to ssq_out
    // [rows x ceil(N/64)].  Consumer side (EPI_QKV / EPI_RELU / EPI_STORE): scale row r of
    // the accumulator by (sum(ssq_in[r,:]) / norm_cols + 1e-6)^-1/2 before the epilogue op
    // (norm(x).W == diag(1/rms).(x.W); ReLU commutes with the positive scale).
    bf16* outb = nullptr;
    int64_t ldb = 0;
    float* ssq_out = nullptr;
    const float* ssq_in = nullptr;
    int ssq_parts = 0;
    int64_t norm_cols = 0;
    // gemv_bf16 only: the consumer computes the row scale from the f32 rows themselves
    // (norm_src[r, 0:norm_cols], row stride ld_norm) instead of ssq_in partials
    const float* norm_src = nullptr;
    int64_t ld_norm = 0;
    // EPI_QKV (tcgen05 GEMM) only: the K and V columns are ALSO stored into up to
    // KVP_MAX_MIRRORS other buffers with out1/out2's row stride -- other ranks' KV caches
    // (peer memory over NVLink, or IPC-mapped), so the KV handoff rides the projection's
    // epilogue tile by tile instead of a copy after it
    bf16* mirror_k[8] = {};
    bf16* mirror_v[8] = {};
    int n_mirror = 0;
    // EPI_QKV only, opt-in extension (the reference model has no positional encoding): rotary
    // embedding of the Q and K columns before they are stored (and mirrored).  Pairs
    // (2i, 2i+1) of every head (head_dim rope_hd) of row r rotate by angle
    // (rope_pos0 + r) * rope_inv_freq[i] (device table of rope_hd/2 floats).  rope_hd = 0: off.
    int rope_hd = 0;
    int64_t rope_pos0 = 0;
    const float* rope_inv_freq = nullptr;
};
constexpr int KVP_MAX_MIRRORS = 8;
inline int ssq_parts_for(int64_t cols) { return static_cast<int>((cols + 63) / 64); }
// KVP_GEMM_TRACE: write the per-CTA stamps of the last tcgen05 GEMM launch (tuning only)
void gemm_trace_dump();
void gemm_bf16_tc(const bf16* A, int64_t M, int64_t K, const bf16* B, int64_t N, const GemmEpilogue& ep,
                  cudaStream_t s);
// tile width the dispatcher picks for this shape (128 or 256)
int gemm_bf16_tc_bn(int64_t M, int64_t N);

// ---------------------------------------------------------------- gemm_simt.cu
// fp32 parity GEMM: C = A[M x K] . B[K x N] (reference layout), sequential k order with
// separately rounded multiply and add -> bit-identical to matrix.hpp:76-91.
enum SimtEpi : int { SEPI_STORE = 0, SEPI_RESID = 1, SEPI_RELU = 2 };
void gemm_f32_simt(const float* A, int64_t M, int64_t K, int64_t lda, const float* B, int64_t N, float* C,
                   int64_t ldc, int epi, const float* resid, int64_t ldr, cudaStream_t s);

// ---------------------------------------------------------------- attention
// Prefix-causal attention (model.hpp:112-158 semantics): query row i (absolute position
// offset + i) attends keys [0, offset + i].  Q: q_rows x ldq, K/V: k_rows x ldkv (head g
// at columns [g*hd, (g+1)*hd)), O: q_rows x ldo.  Query head h reads kv head h / group.
struct AttnShape {
    int64_t q_rows = 0, k_rows = 0, offset = 0;
    int n_heads = 1, n_kv_heads = 1, head_dim = 1;
    int64_t ldq = 0, ldkv = 0, ldo = 0;
};
// bf16 tensor-core flash attention (head_dim 64 / 128), tile-skipping, online softmax.
bool attn_bf16_supported(int head_dim);
void attn_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s);
// the two implementations behind attn_bf16: tcgen05/TMEM (default) and warp-level mma.sync
bool attn_tc_supported(int head_dim);
void attn_bf16_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s);
// head_dim 128, one query tile per CTA, S triple-buffered in TMEM (attn_tb.cu)
void attn_bf16_tb(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s);
void attn_bf16_mma(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s);
// Generic SIMT attention (any head_dim <= 256): f32 math; T = float or bf16 I/O.
void attn_simt_f32(const float* Q, const float* K, const float* V, float* O, const AttnShape& sh,
                   cudaStream_t s);
void attn_simt_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s);

// ---------------------------------------------------------------- decode.cu
// Decode step (M <= 8 new rows on the prefilled cache): HBM-bound GEMV with gemm_bf16_tc's
// epilogues, and split-key decode attention (scratch: attn_decode_scratch_floats floats).
void gemv_bf16(const bf16* X, int64_t M, int64_t K, const bf16* B, int64_t N, const GemmEpilogue& ep,
               cudaStream_t s);
int attn_decode_segment(const AttnShape& sh);
int64_t attn_decode_scratch_floats(const AttnShape& sh);
void attn_decode_bf16(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, float* scratch,
                      cudaStream_t s);

}  // namespace kvp
