// gemm_tc.cu -- the projection GEMMs of the per-rank layer executor on 5th-gen tensor
// cores (reference sites: qkv_project model.hpp:65-73, A.Wo / f.W1 / mid.W2 model.hpp:172-174,
// all through matrix.hpp:76-91 matmul).
//
// D[M x N] = A[M x K] . B[N x K]^T, bf16 operands, f32 accumulation in TMEM.
//  * persistent: one CTA per SM (grid = min(#tiles, #SMs)), static round-robin tile order,
//    M-fastest rasterisation so the CTAs in flight share the same weight columns in L2;
//  * warp roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = tcgen05.mma
//    issuer (one lane) + TMEM owner, warps 2..5 = epilogue (TMEM -> registers -> global);
//  * 4-stage smem ring of 128 x 64 (A) and BN x 64 (B) bf16 tiles, 128-byte swizzle,
//    full/empty mbarriers; MMA completion frees a stage via tcgen05.commit;
//  * two TMEM accumulators (2 x BN columns) so the epilogue of tile t overlaps the MMAs
//    of tile t+1;
//  * fused epilogues: Q/K/V split store straight into the rank's KV-cache rows (replaces
//    the reference's vcat, engine.hpp:277-278), f32 residual add, ReLU + bf16 cast.
// Operand tails (M, N, K not multiples of the tile) are zero-filled by TMA; the epilogue
// predicates rows and columns.
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "kernels.cuh"
#include "ptx.cuh"

namespace kvp {

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// 2D bf16 tensor [outer x inner] with row stride ld (elements), box [box_outer x 64],
// 128-byte swizzle (the canonical K-major SW128 UMMA layout).
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {ld * 2};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}


namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (2 per TMEM lane quarter)
constexpr int EPI_WARPS = 8;

// NCTA = 1: one CTA per 128 x BN tile.  NCTA = 2: a CTA pair (cluster of 2 on one TPC) per
// 256 x BN tile -- each CTA loads its 128 A rows and HALF of the B columns, the leader issues
// tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' smem, each CTA's TMEM receives its own
// 128 accumulator rows.  Per-SM smem traffic per FLOP drops by a third and the freed smem
// buys 6 pipeline stages instead of 4.
template <int BN, int NCTA>
struct Cfg {
    static constexpr int STAGES = NCTA == 2 ? (BN == 256 ? 6 : 8) : 4;
    static constexpr int B_ROWS = BN / NCTA;  // B rows this CTA loads per stage
    static constexpr uint32_t A_BYTES = BM * BK * 2;
    static constexpr uint32_t B_BYTES = B_ROWS * BK * 2;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t TMEM_COLS = 2 * BN;
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr uint32_t STAGING = EPI_WARPS * 32 * 32 * 4;  // EPI_RESID transpose tiles
    static constexpr uint32_t smem_for(int kind) { return SMEM + (kind == EPI_RESID ? STAGING : 0); }
};

// EPI_QKV with the fused-handoff mirror stores (GemmEpilogue::n_mirror > 0): a separate
// instantiation, so the plain QKV epilogue carries none of the mirror code
constexpr int EPI_QKV_MIRROR = 4;

struct EpiArgs {
    bf16* out0;
    int64_t ld0, n0;
    bf16* out1;
    int64_t ld1, n1;
    bf16* out2;
    int64_t ld2;
    float* outf;
    int64_t ldf;
    const float* resid;
    int64_t ldr;
    bf16* outb;
    int64_t ldb;
    float* ssq_out;
    const float* ssq_in;
    int ssq_parts;
    float inv_norm_cols;
    bf16* mk[8];  // EPI_QKV mirrors of the K / V columns (GemmEpilogue::mirror_k/v)
    bf16* mv[8];
    int n_mirror;
    int rope_hd;  // EPI_ROPE kinds: GemmEpilogue::rope_*
    int64_t rope_pos0;
    const float* rope_inv_freq;
};

// EPI_QKV / EPI_QKV_MIRROR | EPI_ROPE: the same epilogue with the rotary embedding applied to
// the Q and K columns (a separate instantiation: the parity path carries none of it)
constexpr int EPI_ROPE = 8;

// Rotary embedding of one 32-column chunk of the Q or K region (region-relative first column
// rc0, a multiple of 32; head_dim a multiple of 32, so a chunk never straddles a head): pair
// (2i, 2i+1) of the head rotates by pos * inv_freq[i], f32 sincos with full range reduction.
__device__ __forceinline__ void rope_chunk(float (&v)[32], int64_t rc0, int64_t pos, int hd,
                                           const float* __restrict__ inv_freq) {
    const int d0 = static_cast<int>(rc0 % hd);
    const float fpos = static_cast<float>(pos);
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        float sn, cs;
        sincosf(fpos * __ldg(inv_freq + ((d0 + j) >> 1)), &sn, &cs);
        const float x0 = v[j], x1 = v[j + 1];
        v[j] = x0 * cs - x1 * sn;
        v[j + 1] = x0 * sn + x1 * cs;
    }
}

// QKV split / ReLU / plain bf16 store of one 32-column chunk (lane = row).
template <int KIND_>
__device__ __forceinline__ void store_chunk(const EpiArgs& ep, int64_t row, int64_t col0, int64_t N,
                                            const uint32_t (&r)[32], float row_scale) {
    constexpr int KIND = KIND_ & ~EPI_ROPE;
    constexpr bool ROPE = (KIND_ & EPI_ROPE) != 0;
    const bool full = col0 + 32 <= N;
    {
        bf16* o;
        int region = 0;  // EPI_QKV: 1 = K, 2 = V chunk (also stored to the mirrors)
        int64_t region_off = 0;
        int64_t rc0 = col0;  // region-relative first column (RoPE)
        if constexpr (KIND == EPI_QKV || KIND == EPI_QKV_MIRROR) {
            // chunks straddling the Q|K|V column boundaries (q or kv not a multiple of 32)
            // take the per-element path
            const int64_t e0 = ep.n0, e1 = ep.n0 + ep.n1;
            if ((col0 < e0 && col0 + 32 > e0) || (col0 < e1 && col0 + 32 > e1)) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (col0 + j >= N) continue;
                    const int64_t c = col0 + j;
                    bf16* dst = c < e0 ? ep.out0 + row * ep.ld0 + c
                                       : (c < e1 ? ep.out1 + row * ep.ld1 + (c - e0) : ep.out2 + row * ep.ld2 + (c - e1));
                    const bf16 val = __float2bfloat16_rn(__uint_as_float(r[j]) * row_scale);
                    *dst = val;
                    if constexpr (KIND == EPI_QKV_MIRROR)
#pragma unroll
                        for (int m = 0; m < 8; ++m)
                            if (m < ep.n_mirror && c >= e0)
                                *(c < e1 ? ep.mk[m] + row * ep.ld1 + (c - e0) : ep.mv[m] + row * ep.ld2 + (c - e1)) = val;
                }
                return;
            }
            if (col0 < ep.n0) {
                o = ep.out0 + row * ep.ld0 + col0;
            } else if (col0 < ep.n0 + ep.n1) {
                o = ep.out1 + row * ep.ld1 + (col0 - ep.n0);
                region_off = row * ep.ld1 + (col0 - ep.n0);
                region = 1;
                rc0 = col0 - ep.n0;
            } else {
                o = ep.out2 + row * ep.ld2 + (col0 - ep.n0 - ep.n1);
                region_off = row * ep.ld2 + (col0 - ep.n0 - ep.n1);
                region = 2;
            }
        } else {
            o = ep.out0 + row * ep.ld0 + col0;
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            v[j] = __uint_as_float(r[j]) * row_scale;
            if constexpr (KIND == EPI_RELU) v[j] = v[j] < 0.f ? 0.f : v[j];
        }
        if constexpr (ROPE)
            if (region != 2) rope_chunk(v, rc0, ep.rope_pos0 + row, ep.rope_hd, ep.rope_inv_freq);
        if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
                uint4 pk;
                pk.x = ptx::pack_bf16(v[j + 0], v[j + 1]);
                pk.y = ptx::pack_bf16(v[j + 2], v[j + 3]);
                pk.z = ptx::pack_bf16(v[j + 4], v[j + 5]);
                pk.w = ptx::pack_bf16(v[j + 6], v[j + 7]);
                *reinterpret_cast<uint4*>(o + j) = pk;
                if constexpr (KIND == EPI_QKV_MIRROR)
#pragma unroll
                    for (int m = 0; m < 8; ++m)
                        if (region && m < ep.n_mirror)
                            *reinterpret_cast<uint4*>((region == 1 ? ep.mk[m] : ep.mv[m]) + region_off + j) = pk;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (col0 + j < N) {
                    o[j] = __float2bfloat16_rn(v[j]);
                    if constexpr (KIND == EPI_QKV_MIRROR)
#pragma unroll
                        for (int m = 0; m < 8; ++m)
                            if (region && m < ep.n_mirror) (region == 1 ? ep.mk[m] : ep.mv[m])[region_off + j] = o[j];
                }
        }
    }
}

// EPI_RESID epilogue, one 32x32 chunk per warp, coalesced: the accumulator (lane = row, from
// tcgen05.ld 32x32b) is transposed through a 4 KB XOR-swizzled smem tile so that lane l then
// owns rows {l/8 + 4i : i < 8} x columns [4*(l%8), 4*(l%8)+4) -- every global access of the
// warp covers 4 full 128-byte row segments instead of 32 scattered 16-byte pieces.
struct ResidT {
    int64_t row0;  // first row of the warp's 32-row slab
    uint32_t rsub, cg;
};

__device__ __forceinline__ void resid_fetch(const EpiArgs& ep, const ResidT& t, int64_t col0, int M, int N,
                                            float4 (&rv)[8]) {
    const bool full = t.row0 + 32 <= M && col0 + 32 <= N;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = t.row0 + t.rsub + 4 * i;
        const int64_t col = col0 + 4 * t.cg;
        if (full) {
            // read once: evict-first, so the residual stream does not push the operand tiles
            // out of L2
            rv[i] = __ldcs(reinterpret_cast<const float4*>(ep.resid + row * ep.ldr + col));
        } else {
            float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (row < M && col + q < N) e[q] = ep.resid[row * ep.ldr + col + q];
            rv[i] = make_float4(e[0], e[1], e[2], e[3]);
        }
    }
}

__device__ __forceinline__ float sq4(float4 v) {
    return __fmaf_rn(v.w, v.w, __fmaf_rn(v.z, v.z, __fmaf_rn(v.y, v.y, __fmul_rn(v.x, v.x))));
}

// Adds the chunk to the prefetched residual, stores f32 + bf16, accumulates per-row partial
// sums of squares in ss[i] (row rsub + 4i).
__device__ __forceinline__ void resid_store(const EpiArgs& ep, const ResidT& t, int64_t col0, int M, int N,
                                            const uint32_t (&r)[32], const float4 (&rv)[8], float* stg,
                                            float (&ss)[8]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int g = 0; g < 8; ++g)
        *reinterpret_cast<float4*>(stg + lane * 32 + ((g ^ (lane & 7)) << 2)) =
            make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]), __uint_as_float(r[4 * g + 2]),
                        __uint_as_float(r[4 * g + 3]));
    __syncwarp();
    const bool full = t.row0 + 32 <= M && col0 + 32 <= N;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t rr = t.rsub + 4 * i;
        const float4 a = *reinterpret_cast<const float4*>(stg + rr * 32 + ((t.cg ^ (rr & 7)) << 2));
        float4 v;
        v.x = rv[i].x + a.x;
        v.y = rv[i].y + a.y;
        v.z = rv[i].z + a.z;
        v.w = rv[i].w + a.w;
        const int64_t row = t.row0 + rr, col = col0 + 4 * t.cg;
        if (full) {
            // the f32 residual is next read layers/kernels later: streaming store; the bf16
            // copy (the next GEMM's A operand) keeps the default policy
            __stcs(reinterpret_cast<float4*>(ep.outf + row * ep.ldf + col), v);
            if (ep.outb) {
                uint2 pk;
                pk.x = ptx::pack_bf16(v.x, v.y);
                pk.y = ptx::pack_bf16(v.z, v.w);
                *reinterpret_cast<uint2*>(ep.outb + row * ep.ldb + col) = pk;
            }
            ss[i] = __fadd_rn(ss[i], sq4(v));
        } else if (row < M) {
            float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (col + q < N) {
                    ep.outf[row * ep.ldf + col + q] = e[q];
                    if (ep.outb) ep.outb[row * ep.ldb + col + q] = __float2bfloat16_rn(e[q]);
                } else {
                    e[q] = 0.f;
                }
            }
            // same rounding sequence as the full path: a row's partial never depends on
            // whether its 32-row slab is complete (partition-independent results)
            ss[i] = __fadd_rn(ss[i], sq4(make_float4(e[0], e[1], e[2], e[3])));
        }
    }
    __syncwarp();  // the tile is rewritten by the next chunk
}

// Reduce-scatter of ss[0..7] over the 8 lanes sharing rsub (7 shuffles): afterwards lane cg
// holds the total for row rsub + 4*cg; written as the row's partial of 64-column group grp.
__device__ __forceinline__ void resid_ssq_flush(const EpiArgs& ep, const ResidT& t, int M, int64_t grp,
                                                float (&ss)[8]) {
    float a4[4], a2[2], a1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const bool hi = t.cg & 4;
        const float send = hi ? ss[j] : ss[j + 4];
        a4[j] = (hi ? ss[j + 4] : ss[j]) + __shfl_xor_sync(0xffffffffu, send, 4);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const bool hi = t.cg & 2;
        const float send = hi ? a4[j] : a4[j + 2];
        a2[j] = (hi ? a4[j + 2] : a4[j]) + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    {
        const bool hi = t.cg & 1;
        const float send = hi ? a2[0] : a2[1];
        a1 = (hi ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, send, 1);
    }
    const int64_t row = t.row0 + t.rsub + 4 * t.cg;
    if (row < M) ep.ssq_out[row * ep.ssq_parts + grp] = a1;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss[i] = 0.f;
}

// tuning only (build with KVP_NVCC_FLAGS=-DKVP_GEMM_TRACE_ON=1, run with KVP_GEMM_TRACE=<file>):
// per-CTA globaltimer stamps -- 0 entry, 1 prologue done, 2 previous grid complete (PDL), 3 first
// stage landed, 4 last MMA issued, 5 epilogue done; 6 = SM id, 7 = tiles (scripts/gemm_trace.py).
// Compiled out by default: the runtime check inside the converged MMA issue loop cost the
// QKV / FFN1 GEMMs 4-5 % in isolation and 12 % inside the layer step (profiles/r02/gemm_trace_cost.txt).
#ifndef KVP_GEMM_TRACE_ON
#define KVP_GEMM_TRACE_ON 0
#endif
#define GT(ev)                                                                  \
    do {                                                                        \
        if (KVP_GEMM_TRACE_ON && trace) trace[blockIdx.x * 8 + (ev)] = ptx::globaltimer(); \
    } while (0)

template <int BN, int KIND, int NCTA>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmBh, int M, int N, int K, int n_full, int group_m,
                   unsigned long long* trace, EpiArgs ep) {
    using C = Cfg<BN, NCTA>;
    constexpr int STAGES = C::STAGES;
    constexpr int TM = BM * NCTA;  // rows of one (pair) tile
    if (threadIdx.x == 0) GT(0);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment by pointer arithmetic on the __shared__ array, so the compiler keeps
    // the shared state space (LDS/STS instead of generic loads/stores)
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = NCTA == 2 ? ptx::cluster_ctarank() : 0u;
    const int unit = static_cast<int>(blockIdx.x) / NCTA, n_units = static_cast<int>(gridDim.x) / NCTA;
    const int num_m = (M + TM - 1) / TM, num_n = (N + BN - 1) / BN;
    // Tiles [0, n_full) are BN wide; the remaining (last partial wave of) BN tiles run as two
    // BN/2-wide tiles each so the persistent grid's final round is evenly filled.  Only the
    // tile width changes, not the per-element K order: results are identical either way.
    const int num_tiles = n_full + 2 * (num_m * num_n - n_full);
    // Grouped rasterisation: tiles run in groups of `group_m` M-blocks, M-fastest inside a
    // group, so the CTAs in flight share a group_m x ~(148/group_m) block of the output: the
    // group's A rows (group_m*TM*K*2 bytes, sized on the host to stay in L2) are read from
    // HBM once and each weight column block once per group.
    auto coords = [&](int big, int& m_blk, int& n_blk) {
        const int per_group = group_m * num_n;
        const int grp = big / per_group, rem = big - grp * per_group;
        const int g_m = min(group_m, num_m - grp * group_m);
        m_blk = grp * group_m + rem % g_m;
        n_blk = rem / g_m;
    };
    auto decode = [&](int tile, int& m_blk, int& col_base, int& width) {
        int n_blk;
        if (tile < n_full) {
            coords(tile, m_blk, n_blk);
            col_base = n_blk * BN;
            width = BN;
        } else {
            const int k = tile - n_full;
            coords(n_full + (k >> 1), m_blk, n_blk);
            col_base = n_blk * BN + (k & 1) * (BN / 2);
            width = BN / 2;
        }
    };
    const int num_kb = (K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        ptx::tma_prefetch_desc(&tmBh);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], EPI_WARPS * NCTA);  // both CTAs' epilogues free a buffer
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) {
        if constexpr (NCTA == 2)
            ptx::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
        else
            ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (NCTA == 2) ptx::cluster_sync();  // peer barriers initialised before any remote use
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the prologue above overlapped the previous kernel's tail; no global memory is
    // touched before the previous grid has completed
    if (threadIdx.x == 0) GT(1);
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();
    if (threadIdx.x == 0) GT(2);

    if (warp == 0) {
        // TMA producer: the whole warp runs the loop converged; one elect.sync lane arms the
        // stage barrier and issues the loads (ptx::*_w).  (L2 cache policies on these loads
        // -- evict_last A / evict_first B, or either alone -- were measured and did not help,
        // profiles/r02/gemm_l2hint.txt.)
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = unit; tile < num_tiles; tile += n_units) {
            int m_blk, col_base, width;
            decode(tile, m_blk, col_base, width);
            const bool narrow = width != BN;
            const uint32_t bytes = C::A_BYTES + (narrow ? C::B_BYTES / 2 : C::B_BYTES);
            const int a_row = m_blk * TM + static_cast<int>(rank) * BM;
            const int b_row = col_base + static_cast<int>(rank) * (width / NCTA);
            for (int kb = 0; kb < num_kb; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                if constexpr (NCTA == 2) {
                    // both CTAs' bytes land on the leader's stage barrier
                    if (rank == 0) ptx::mbar_arrive_expect_tx_w(&full[stage], 2 * bytes);
                    const uint32_t bar = ptx::cluster_addr(&full[stage], 0);
                    ptx::tma_load_2d_pair_w(sA + stage * C::A_BYTES, &tmA, bar, kb * BK, a_row);
                    ptx::tma_load_2d_pair_w(sB + stage * C::B_BYTES, narrow ? &tmBh : &tmB, bar, kb * BK, b_row);
                } else {
                    ptx::mbar_arrive_expect_tx_w(&full[stage], bytes);
                    ptx::tma_load_2d_w(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, a_row);
                    ptx::tma_load_2d_w(sB + stage * C::B_BYTES, narrow ? &tmBh : &tmB, &full[stage], kb * BK, b_row);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // in a pair only the leader issues the MMAs: the whole warp runs the loop converged and
        // one elect.sync lane issues (ptx::*_w), descriptors advanced by constant offsets
        if (rank == 0) {
            constexpr uint32_t idesc_w = ptx::idesc_bf16(TM, BN), idesc_n = ptx::idesc_bf16(TM, BN / 2);
            const uint64_t adesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sA), 16, 1024);
            const uint64_t bdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sB), 16, 1024);
            int stage = 0;
            uint32_t phase = 0;
            int t = 0;
            for (int tile = unit; tile < num_tiles; tile += n_units, ++t) {
                int m_blk_u, col_base_u, width;
                decode(tile, m_blk_u, col_base_u, width);
                const uint32_t idesc = width == BN ? idesc_w : idesc_n;
                const uint32_t buf = t & 1, aphase = (t >> 1) & 1;
                ptx::mbar_wait(&tempty[buf], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + buf * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    if (KVP_GEMM_TRACE_ON && t == 0 && kb == 0 && lane == 0) GT(3);
                    const uint64_t ad0 = adesc0 + static_cast<uint64_t>((stage * C::A_BYTES) >> 4);
                    const uint64_t bd0 = bdesc0 + static_cast<uint64_t>((stage * C::B_BYTES) >> 4);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = ad0 + static_cast<uint64_t>((k * 32) >> 4);
                        const uint64_t bd = bd0 + static_cast<uint64_t>((k * 32) >> 4);
                        if constexpr (NCTA == 2)
                            ptx::mma_bf16_ss_pair_w(d_tmem, ad, bd, idesc, (kb | k) != 0);
                        else
                            ptx::mma_bf16_ss_w(d_tmem, ad, bd, idesc, (kb | k) != 0);
                    }
                    if constexpr (NCTA == 2)
                        ptx::mma_commit_pair_w(&empty[stage], 0x3);
                    else
                        ptx::mma_commit_w(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (NCTA == 2)
                    ptx::mma_commit_pair_w(&tfull[buf], 0x3);
                else
                    ptx::mma_commit_w(&tfull[buf]);
            }
            if (KVP_GEMM_TRACE_ON && lane == 0) GT(4);
        }
    } else {
        // Epilogue warps 2..9: warp w may touch TMEM lanes [32*(w%4), 32*(w%4)+32); the two
        // warps of a lane quarter split the tile's columns (more loads in flight per row).
        const uint32_t quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        constexpr int MY_MAX = BN / 64;  // 32-column chunks per warp group on a full-width tile
        int t = 0;
        for (int tile = unit; tile < num_tiles; tile += n_units, ++t) {
            int m_blk, col_base, width;
            decode(tile, m_blk, col_base, width);
            const int MY = width / 64;
            const uint32_t buf = t & 1, aphase = (t >> 1) & 1;
            const int64_t row0 = static_cast<int64_t>(m_blk) * TM + rank * BM;  // this CTA's rows
            const int64_t row = row0 + quarter * 32 + lane;
            const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + buf * BN;
            if constexpr (KIND == EPI_RESID) {
                // The residual does not depend on the accumulator: fetch its first two chunks
                // while the tile's MMAs are still running, then keep two chunks in flight
                // (the last tile's epilogue of a small-M GEMM is fully exposed).
                const ResidT rt{row0 + quarter * 32, lane >> 3, lane & 7};
                float* stg = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES + 256) + (warp - 2) * 1024;
                float4 rva[8], rvb[8];
                float ss[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) ss[i] = 0.f;
                const int64_t cbase = static_cast<int64_t>(col_base) + half * MY * 32;
                resid_fetch(ep, rt, cbase, M, N, rva);
                if (MY > 1 && cbase + 32 < N) resid_fetch(ep, rt, cbase + 32, M, N, rvb);
                ptx::mbar_wait(&tfull[buf], aphase);
                ptx::tc_fence_after();
                // chunk cc of this warp's columns from register buffer rv; refill rv with chunk cc + 2
                auto chunk = [&](int cc, float4(&rv)[8]) {
                    const int c = half * MY + cc;
                    const int64_t col0 = static_cast<int64_t>(col_base) + c * 32;
                    uint32_t r[32];
                    ptx::tmem_ld32(taddr + c * 32, r);
                    ptx::tmem_ld_wait();
                    resid_store(ep, rt, col0, M, N, r, rv, stg, ss);
                    if (cc + 2 < MY && col0 + 64 < N) resid_fetch(ep, rt, col0 + 64, M, N, rv);
                    // one partial per 64-column group, independent of BN and of the warp split
                    if (ep.ssq_out != nullptr && (((c + 1) & 1) == 0 || col0 + 32 >= N))
                        resid_ssq_flush(ep, rt, M, col0 >> 6, ss);
                };
#pragma unroll 1
                for (int cc = 0; cc < MY_MAX; cc += 2) {
                    if (cc >= MY || cbase + cc * 32 >= N) break;  // warp-uniform
                    chunk(cc, rva);
                    if (cc + 1 >= MY || cbase + (cc + 1) * 32 >= N) break;
                    chunk(cc + 1, rvb);
                }
            } else {
                ptx::mbar_wait(&tfull[buf], aphase);
                ptx::tc_fence_after();
                float row_scale = 1.f;
                if (ep.ssq_in != nullptr && row < M) {
                    const float* sp = ep.ssq_in + row * ep.ssq_parts;
                    float ss = 0.f;
                    for (int q = 0; q < ep.ssq_parts; ++q) ss += sp[q];
                    row_scale = 1.0f / sqrtf(ss * ep.inv_norm_cols + 1e-6f);
                }
#pragma unroll 1
                for (int cc = 0; cc < MY; ++cc) {
                    const int c = half * MY + cc;
                    const int64_t col0 = static_cast<int64_t>(col_base) + c * 32;
                    if (col0 >= N) break;  // warp-uniform
                    uint32_t r[32];
                    ptx::tmem_ld32(taddr + c * 32, r);
                    ptx::tmem_ld_wait();
                    if (row < M) store_chunk<KIND>(ep, row, col0, N, r, row_scale);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (NCTA == 2)
                    ptx::mbar_arrive_cluster(ptx::cluster_addr(&tempty[buf], 0));
                else
                    ptx::mbar_arrive(&tempty[buf]);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (KVP_GEMM_TRACE_ON && threadIdx.x == 0 && trace) {
        GT(5);
        trace[blockIdx.x * 8 + 6] = ptx::smid();
        trace[blockIdx.x * 8 + 7] = static_cast<unsigned long long>((num_tiles - unit + n_units - 1) / n_units);
    }
    if constexpr (NCTA == 2) ptx::cluster_sync();  // the pair's TMEM and barriers outlive both CTAs' use
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (NCTA == 2)
            ptx::tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
        else
            ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

// KVP_GEMM_TRACE: device buffer for the per-CTA stamps of the most recent launch
static const char* gemm_trace_path() {
    static const char* p = getenv("KVP_GEMM_TRACE");
    return p;
}
static unsigned long long* g_trace = nullptr;
static unsigned long long* gemm_trace_buffer() {
    if (!gemm_trace_path()) return nullptr;
    if (!g_trace && cudaMalloc(&g_trace, 1024 * 8 * sizeof(unsigned long long)) != cudaSuccess) g_trace = nullptr;
    if (g_trace) cudaMemset(g_trace, 0, 1024 * 8 * sizeof(unsigned long long));
    return g_trace;
}

template <int BN, int KIND, int NCTA>
void launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbh, int M, int N, int K,
               const EpiArgs& ep, cudaStream_t s) {
    using Cf = Cfg<BN, NCTA>;
    auto kern = gemm_tc_kernel<BN, KIND, NCTA>;
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_dev != dev) {  // attribute is per device; cheap to re-set
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::smem_for(KIND));
        if (NCTA == 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        configured_dev = dev;
    }
    constexpr int TM = BM * NCTA;
    const int tiles = ((M + TM - 1) / TM) * ((N + BN - 1) / BN);
    const int units = num_sms() / NCTA;  // persistent: one CTA (pair) per SM (pair)
    const int grid_units = tiles < units ? tiles : units;
    // split the last partial round into half-width tiles when they fit in one round
    static const bool split_tail = [] {
        const char* e = getenv("KVP_GEMM_TAIL");
        return !(e && e[0] == '0');
    }();
    const int rem = tiles % grid_units;
    const int n_full =
        (split_tail && BN == 256 && tiles > grid_units && rem > 0 && 2 * rem <= grid_units) ? tiles - rem : tiles;
    // M-blocks per raster group: keep the group's A rows within ~32 MB of L2
    static const int forced_group = [] {
        const char* e = getenv("KVP_GEMM_GROUP");
        return e ? atoi(e) : 0;
    }();
    const int num_m = (M + TM - 1) / TM;
    int group_m = forced_group > 0 ? forced_group : static_cast<int>((32ll << 20) / (static_cast<int64_t>(TM) * K * 2));
    group_m = group_m < 4 ? 4 : group_m;
    group_m = group_m > num_m ? num_m : group_m;
    unsigned long long* trace = gemm_trace_buffer();
    note_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid_units * NCTA));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Cf::smem_for(KIND);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NCTA;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, tbh, M, N, K, n_full, group_m, trace, ep);
}

template <int BN, int NCTA>
void dispatch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbh, int M, int N, int K,
              const GemmEpilogue& g, cudaStream_t s) {
    EpiArgs ep{g.out0, g.ld0, g.n0, g.out1, g.ld1, g.n1, g.out2, g.ld2, g.outf, g.ldf, g.resid, g.ldr,
               g.outb, g.ldb, g.ssq_out, g.ssq_in, g.ssq_parts, g.norm_cols ? 1.0f / static_cast<float>(g.norm_cols) : 0.f,
               {}, {}, g.kind == EPI_QKV ? g.n_mirror : 0, g.rope_hd, g.rope_pos0, g.rope_inv_freq};
    for (int m = 0; m < ep.n_mirror; ++m) {
        ep.mk[m] = g.mirror_k[m];
        ep.mv[m] = g.mirror_v[m];
    }
    switch (g.kind) {
        case EPI_QKV:
            if (ep.rope_hd > 0) {
                if (ep.n_mirror > 0)
                    launch_tc<BN, EPI_QKV_MIRROR | EPI_ROPE, NCTA>(ta, tb, tbh, M, N, K, ep, s);
                else
                    launch_tc<BN, EPI_QKV | EPI_ROPE, NCTA>(ta, tb, tbh, M, N, K, ep, s);
            } else if (ep.n_mirror > 0) {
                launch_tc<BN, EPI_QKV_MIRROR, NCTA>(ta, tb, tbh, M, N, K, ep, s);
            } else {
                launch_tc<BN, EPI_QKV, NCTA>(ta, tb, tbh, M, N, K, ep, s);
            }
            break;
        case EPI_RESID: launch_tc<BN, EPI_RESID, NCTA>(ta, tb, tbh, M, N, K, ep, s); break;
        case EPI_RELU: launch_tc<BN, EPI_RELU, NCTA>(ta, tb, tbh, M, N, K, ep, s); break;
        default: launch_tc<BN, EPI_STORE, NCTA>(ta, tb, tbh, M, N, K, ep, s); break;
    }
}

}  // namespace

// CTA pairs whenever both CTAs of a pair get rows (KVP_GEMM_PAIR=0: single-CTA tiles only).
static bool use_pair(int64_t M) {
    static const bool pair_ok = [] {
        const char* e = getenv("KVP_GEMM_PAIR");
        return !(e && e[0] == '0');
    }();
    return pair_ok && M > BM;
}

int gemm_bf16_tc_bn(int64_t M, int64_t N) {
    // Tile width: BN=256 feeds the tensor core with the least smem traffic per FLOP; BN=128
    // halves the tile so the persistent grid quantises better (e.g. 4096x4096 outputs are 256
    // pair tiles = 3.46 waves of 74 SM pairs at BN=256 but 6.92 waves at BN=128).  Pick the
    // width with the best (wave efficiency x per-tile efficiency); KVP_GEMM_BN=128|256 forces one.
    static const int forced = [] {
        const char* e = getenv("KVP_GEMM_BN");
        return e ? atoi(e) : 0;
    }();
    const bool pair = use_pair(M);
    const int64_t tm = pair ? 2 * BM : BM;
    const int units = num_sms() / (pair ? 2 : 1);
    auto score = [&](int64_t bn, double tile_eff) {
        const int64_t tiles = ((M + tm - 1) / tm) * ((N + bn - 1) / bn);
        double waves = static_cast<double>((tiles + units - 1) / units);
        // launch_tc runs a last partial round of wide tiles as half-width tiles when they fit
        const int64_t rem = tiles % units;
        if (bn == 256 && tiles > units && rem > 0 && 2 * rem <= units) waves -= 0.5;
        const double useful = static_cast<double>(M) * N / (waves * units * tm * bn);
        return useful * tile_eff;
    };
    // per-FLOP efficiency of the narrow tile relative to BN=256 (measured; the narrow pair
    // tile went from 0.65 to ~0.8 with the converged MMA issue, profiles/r02/gemm_bn.txt)
    bool wide = score(256, 1.0) >= score(128, pair ? 0.8 : 0.72);
    if (N < 256) wide = false;
    if (forced == 128) wide = false;
    if (forced == 256 && N >= 256) wide = true;
    return wide ? 256 : 128;
}

void gemm_trace_dump() {
    if (!gemm_trace_path() || !g_trace) return;
    std::vector<unsigned long long> h(1024 * 8);
    if (cudaMemcpy(h.data(), g_trace, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    if (FILE* f = fopen(gemm_trace_path(), "wb")) {
        fwrite(h.data(), sizeof(h[0]), h.size(), f);
        fclose(f);
    }
}

void gemm_bf16_tc(const bf16* A, int64_t M, int64_t K, const bf16* B, int64_t N, const GemmEpilogue& ep,
                  cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    if (K % 8 != 0 || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
        throw std::runtime_error("gemm_bf16_tc: K must be a multiple of 8 and operands 16-byte aligned");
    const int BN = gemm_bf16_tc_bn(M, N);
    const bool wide = BN == 256;
    const bool pair = use_pair(M);
    const uint32_t b_rows = static_cast<uint32_t>(BN / (pair ? 2 : 1));
    CUtensorMap ta, tb, tbh;
    if (!make_tmap_bf16(&ta, A, K, M, K, BK, BM) || !make_tmap_bf16(&tb, B, K, N, K, BK, b_rows) ||
        !make_tmap_bf16(&tbh, B, K, N, K, BK, b_rows / 2)) {
        char msg[160];
        snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled failed (M=%lld N=%lld K=%lld)", (long long)M,
                 (long long)N, (long long)K);
        throw std::runtime_error(msg);
    }
    if (pair)
        wide ? dispatch<256, 2>(ta, tb, tbh, (int)M, (int)N, (int)K, ep, s)
             : dispatch<128, 2>(ta, tb, tbh, (int)M, (int)N, (int)K, ep, s);
    else
        wide ? dispatch<256, 1>(ta, tb, tbh, (int)M, (int)N, (int)K, ep, s)
             : dispatch<128, 1>(ta, tb, tbh, (int)M, (int)N, (int)K, ep, s);
}

}  // namespace kvp
