// attn_tc.cu -- prefix-causal flash attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Reference: causal_attention (model.hpp:112-158).  One CTA owns TWO 128-query tiles (a, b)
// of one head -- absolute positions offset + q0 ... offset + q0 + 255 -- and walks the
// 128-key tiles [0, offset + last query]; each K/V tile is loaded once for both query tiles.
//   warp 0      TMA producer: Q_a, Q_b once, then K and V tiles through separate smem rings
//               (K runs a stage ahead: it is released as soon as both S MMAs have read it);
//   warp 1      MMA issuer (one lane) + TMEM owner, ping-pong between the tiles:
//                 S_x = Q_x K_j^T  (SS: A=Q smem, B=K smem, both K-major SW128) -> TMEM S_x
//                 O_x += P_x V_j   (TS: A=P_x in TMEM, packed bf16 over S_x; B=V smem MN-major)
//               so the tensor core works on one tile while the other tile's softmax runs;
//   warps 2..5  softmax of tile a, warps 6..9 softmax of tile b: one thread per query row
//               (= TMEM lane), mask of the diagonal tile against absolute positions, online
//               softmax in the log2 domain with the scale folded into one FFMA per element,
//               P written back into TMEM as bf16; O is rescaled in TMEM only when a row max
//               grows by more than 2^8 (exact: l and O always share the same stale max).
// TMEM: S_a [0,128) | S_b [128,256) | O_a [256, 256+hd) | O_b [384, 384+hd).
// Key tiles are aligned to absolute key 0, fully masked tiles are skipped per query tile and
// rows are independent, so results are bitwise independent of how the context is split over
// ranks (Serial == TSP == KVR).
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <stdexcept>

#include "kernels.cuh"
#include "ptx.cuh"
#include "softmax.cuh"

namespace kvp {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);
int num_sms();

namespace {
using namespace smx;

constexpr int BQ = 128;  // queries per tile (NT tiles per CTA)
// warp 0 TMA, warp 1 MMA, warps 2 .. 2+4*NT-1 softmax (four per query tile)
template <int NT>
constexpr int threads_for() { return 64 + NT * 128; }
constexpr uint32_t TMEM_COLS = 512;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: p <= 2^8 between rescales
constexpr int DEFAULT_POLY_128 = 0;        // exp2 column pairs (of 16) on the FMA pipe
constexpr int DEFAULT_POLY_64 = 0;

// K and V tiles have separate smem rings: K(j) is released as soon as both S MMAs of key
// tile j are done, so K(j+1..) streams in while the softmax of tile j runs.
// NT query tiles of BQ rows per CTA, BKV-key tiles.  TMEM: S_x (fp32, BKV columns, P packed
// over its first BKV/2) at x*BKV, O_x (HD columns) at NT*BKV + x*HD.
template <int HD, int NT, int BKV>
struct ACfg {
    static_assert(NT * (BKV + HD) <= 512, "TMEM holds NT x (S + O)");
    static_assert(BKV % 32 == 0 && BKV <= 128, "key tile");
    static constexpr int HALVES = HD / 64;  // 64-wide (128 B) TMA boxes
    static constexpr uint32_t O_BASE = NT * BKV;
    static constexpr uint32_t Q_BYTES = BQ * HD * 2;
    static constexpr uint32_t KV_BYTES = BKV * HD * 2;
    static constexpr int KST = HD == 64 ? 4 : 3;  // K stages
    static constexpr int VST = HD == 64 ? 3 : 2;  // V stages
    static constexpr uint32_t XCH = 0;
    static constexpr uint32_t NEED = NT * Q_BYTES + (KST + VST) * KV_BYTES + 256 + XCH;
    // + up to 1 KB of slack for aligning the dynamic smem base to 1024 B (the SW128 atoms)
    static constexpr uint32_t SMEM = NEED + 1024 <= 232448 ? NEED + 1024 : 232448;
    static_assert(NEED + 512 <= 232448, "attention smem over the 227 KB opt-in limit");
};

struct AttnArgs {
    int64_t q_rows, k_rows, offset;
    int n_heads, group;
    int64_t ldo;
    bf16* O;
    float sl2;     // softmax scale * log2(e)
    int mma_wait;  // 1: the MMA issuer waits for PV(j) before S(j+1) reuses its TMEM columns
    uint32_t* trace;  // tuning only (KVP_ATTN_TRACE): SM clock of pipeline events of one CTA
    int trace_blk;
    unsigned long long* cta_trace;  // tuning only (KVP_ATTN_CTA_TRACE): per CTA {start, end, smid, steps}
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// trace[ev * 512 + j] = clock() of event ev for key tile j, CTA (blockIdx.y * gridDim.x + blockIdx.x) == trace_blk
#ifndef KVP_ATTN_TRACE_ON
#define KVP_ATTN_TRACE_ON 0  // tuning builds: KVP_NVCC_FLAGS=-DKVP_ATTN_TRACE_ON=1
#endif
#define ATTN_TRACE(ev, j)                                                                              \
    do {                                                                                               \
        if (KVP_ATTN_TRACE_ON && a.trace && static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x) == a.trace_blk && (j) < 512) \
            a.trace[(ev) * 512 + (j)] = static_cast<uint32_t>(clock());                                \
    } while (0)

template <int HD, int NT, int BKV, int NPOLY>
__global__ void __launch_bounds__(threads_for<NT>(), 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
    using C = ACfg<HD, NT, BKV>;
    constexpr int KST = C::KST, VST = C::VST;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment by pointer arithmetic on the __shared__ array, so the compiler keeps
    // the shared state space (LDS/STS instead of generic loads/stores)
    const uint32_t pad = (1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u;
    if (pad + C::NEED > C::SMEM) __trap();  // dynamic smem base too far from 1 KB alignment
    uint8_t* smem = smem_raw + pad;
    uint8_t* sQ = smem;                    // [NT] query tiles
    uint8_t* sK = sQ + NT * C::Q_BYTES;    // [KST] stages
    uint8_t* sV = sK + KST * C::KV_BYTES;  // [VST] stages
    uint64_t* bar = reinterpret_cast<uint64_t*>(sV + VST * C::KV_BYTES);
    uint64_t* q_full = bar;
    uint64_t* k_full = bar + 1;              // [KST]
    uint64_t* k_empty = k_full + KST;        // [KST]
    uint64_t* v_full = k_empty + KST;        // [VST]
    uint64_t* v_empty = v_full + VST;        // [VST]
    uint64_t* s_full = v_empty + VST;        // [NT] query tiles
    uint64_t* p_full = s_full + NT;          // [NT] query tiles
    uint64_t* o_done = p_full + NT;          // [NT] query tiles
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + NT);

    const unsigned long long t_start = KVP_ATTN_TRACE_ON && a.cta_trace && threadIdx.x == 0 ? globaltimer() : 0;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_groups = static_cast<int>((a.q_rows + NT * BQ - 1) / (NT * BQ));
    // grid = (heads, query groups): the block scheduler walks x fastest, so ALL heads of the
    // heaviest (latest) query group are dispatched first -- a global longest-first order over
    // the causal work imbalance
    const int grp = num_groups - 1 - static_cast<int>(blockIdx.y);
    const int h = blockIdx.x;
    const int g = h / a.group;
    const int64_t q0 = static_cast<int64_t>(grp) * NT * BQ;
    // key tiles needed by each query tile (non-decreasing: the last tile reads every K/V tile)
    int n_kt[NT];
#pragma unroll
    for (int x = 0; x < NT; ++x) {
        const int64_t last = (q0 + (x + 1) * BQ - 1 < a.q_rows - 1) ? q0 + (x + 1) * BQ - 1 : a.q_rows - 1;
        n_kt[x] = static_cast<int>((a.offset + last) / BKV) + 1;
        if (x > 0 && n_kt[x] < n_kt[x - 1]) n_kt[x] = n_kt[x - 1];
    }

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmQ);
        ptx::tma_prefetch_desc(&tmK);
        ptx::tma_prefetch_desc(&tmV);
        ptx::mbar_init(q_full, 1);
        for (int s = 0; s < KST; ++s) {
            ptx::mbar_init(&k_full[s], 1);
            ptx::mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < VST; ++s) {
            ptx::mbar_init(&v_full[s], 1);
            ptx::mbar_init(&v_empty[s], 1);
        }
        for (int s = 0; s < NT; ++s) {
            ptx::mbar_init(&s_full[s], 1);
            ptx::mbar_init(&p_full[s], 4);  // the 4 softmax warps of the tile
            ptx::mbar_init(&o_done[s], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // PDL: prologue overlapped with the previous kernel's tail; wait before touching its outputs
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();

    if (warp == 0) {
        ptx::mbar_arrive_expect_tx_w(q_full, NT * C::Q_BYTES);
        for (int x = 0; x < NT; ++x)
            for (int hv = 0; hv < C::HALVES; ++hv)
                ptx::tma_load_2d_w(sQ + x * C::Q_BYTES + hv * BQ * 128, &tmQ, q_full, h * HD + hv * 64,
                                 static_cast<int32_t>(q0 + x * BQ));
        // K(t), V(t) in need order; K(t) waits for the S MMAs of key tile t - KST, V(t) for
        // its PV MMAs, so K runs a stage further ahead (blocking waits: the producer lane
        // never spins on the issue slots of the softmax warps of its SMSP)
        for (int t = 0; t < n_kt[NT - 1]; ++t) {
            const int sk = t % KST, sv = t % VST;
            ptx::mbar_wait(&k_empty[sk], ((t / KST) & 1) ^ 1);
            ATTN_TRACE(12, t);
            ptx::mbar_arrive_expect_tx_w(&k_full[sk], C::KV_BYTES);
            for (int hv = 0; hv < C::HALVES; ++hv)
                ptx::tma_load_2d_w(sK + sk * C::KV_BYTES + hv * BKV * 128, &tmK, &k_full[sk], g * HD + hv * 64,
                                 t * BKV);
            ptx::mbar_wait(&v_empty[sv], ((t / VST) & 1) ^ 1);
            ATTN_TRACE(13, t);
            ptx::mbar_arrive_expect_tx_w(&v_full[sv], C::KV_BYTES);
            for (int hv = 0; hv < C::HALVES; ++hv)
                ptx::tma_load_2d_w(sV + sv * C::KV_BYTES + hv * BKV * 128, &tmV, &v_full[sv], g * HD + hv * 64,
                                 t * BKV);
        }
    } else if (warp == 1) {
        // the whole warp runs the issue loop converged; one elected lane issues each
        // tcgen05.mma / commit (ptx::*_w).  Descriptors are built once and advanced by
        // constant offsets (the 14-bit address field holds addr >> 4).
        constexpr uint32_t idesc_s = ptx::idesc_bf16(BQ, BKV, 0);
        constexpr uint32_t idesc_o = ptx::idesc_bf16(BQ, HD, 1);  // B = V is MN-major
        const uint64_t qdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 16, 1024);
        const uint64_t kdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sK), 16, 1024);
        const uint64_t vdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sV), BKV * 128, 1024);
        auto issue_s = [&](int x, int t) {
            const int s = t % KST;
            ptx::mbar_wait(&k_full[s], (t / KST) & 1);
            ptx::tc_fence_after();
            if (x < 2 && lane == 0) ATTN_TRACE(0 + x, t);
            const uint64_t qd = qdesc0 + static_cast<uint64_t>((x * C::Q_BYTES) >> 4);
            const uint64_t kd = kdesc0 + static_cast<uint64_t>((s * C::KV_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < HD / 16; ++k) {
                const uint64_t off_q = ((k >> 2) * (BQ * 128) + (k & 3) * 32) >> 4;
                const uint64_t off_k = ((k >> 2) * (BKV * 128) + (k & 3) * 32) >> 4;
                ptx::mma_bf16_ss_w(tmem + x * BKV, qd + off_q, kd + off_k, idesc_s, k != 0);
            }
            ptx::mma_commit_w(&s_full[x]);
            if (x == NT - 1) ptx::mma_commit_w(&k_empty[s]);  // the last tile is the last reader of K(t)
        };
        auto issue_pv = [&](int x, int t) {
            const int s = t % VST;
            ptx::mbar_wait(&p_full[x], t & 1);
            ptx::mbar_wait(&v_full[s], (t / VST) & 1);
            ptx::tc_fence_after();
            if (x < 2 && lane == 0) ATTN_TRACE(2 + x, t);
            const uint64_t vd = vdesc0 + static_cast<uint64_t>((s * C::KV_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < BKV / 16; ++k) {
                // B = V[keys 16k..16k+15][hd]: MN-major SW128, LBO = next 64-wide hd block,
                // SBO = next 8 keys.
                ptx::mma_bf16_ts_w(tmem + C::O_BASE + x * HD, tmem + x * BKV + k * 8,
                                   vd + static_cast<uint64_t>((k * 16 * 128) >> 4), idesc_o, (t | k) != 0);
            }
            ptx::mma_commit_w(&o_done[x]);
            if (x == NT - 1) ptx::mma_commit_w(&v_empty[s]);  // the last tile is the last reader of V(t)
        };
        ptx::mbar_wait(q_full, 0);
        for (int x = 0; x < NT; ++x) issue_s(x, 0);
        for (int j = 0; j < n_kt[NT - 1]; ++j) {
#pragma unroll
            for (int x = 0; x < NT; ++x) {
                if (j >= n_kt[x]) continue;
                issue_pv(x, j);
                if (j + 1 < n_kt[x]) {
                    // S_x(j+1) overwrites the TMEM columns P_x(j) is read from: tcgen05.mma
                    // ops of one thread execute in issue order, so waiting for PV_x(j) is
                    // only needed when the pipeline is not trusted (a.mma_wait)
                    if (a.mma_wait) ptx::mbar_wait(&o_done[x], j & 1);
                    issue_s(x, j + 1);
                }
            }
        }
    } else {
        // 4*NT softmax warps: warps 2+4x .. 5+4x own query tile x; warp w reads TMEM lane
        // quarter w % 4, one thread per query row (all BKV keys of the tile, no exchange).
        const int x = (warp - 2) >> 2;                         // query tile
        const uint32_t quarter = warp & 3;                     // TMEM lane quarter this warp may access
        const int xrow = static_cast<int>(quarter) * 32 + lane;
        const int64_t row = q0 + x * BQ + xrow;
        const int abs_row = static_cast<int>(a.offset + row);  // positions < 2^31 (host-checked)
        const int tile_first_abs = abs_row - xrow;
        const uint32_t lane_base = tmem + ((quarter * 32u) << 16);
        const int nt = n_kt[x];
        const float2 sl2v = make_float2(a.sl2, a.sl2);
        const float2 sl2y = make_float2(a.sl2 * (1.f / 256.f), a.sl2 * (1.f / 256.f));
        float m_run = -INFINITY, l = 0.f;
        // exp2 of the row's BKV scores against base m (log2 units), P -> TMEM as packed bf16
        // over the first BKV/2 S columns; returns the row sum of P
        auto exp_store = [&](const float (&sv)[BKV], float m, bool diag) -> float {
            const float2 nb2 = make_float2(-m, -m);
            // poly columns: y = sat(x / 256 + POLY_BIAS / 256) straight from the score
            const float2 yb2 = make_float2((POLY_BIAS - m) * (1.f / 256.f), (POLY_BIAS - m) * (1.f / 256.f));
            float2 lacc = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < BKV / 32; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = c * 32 + 2 * i;
                    float2 pv;
                    // NPOLY of every 16 column pairs take exp2 on the FMA pipe, the rest on MUFU
                    if (i >= 16 - NPOLY) {
                        pv = ex2_poly_sat(ffma2_sat(make_float2(sv[col], sv[col + 1]), sl2y, yb2));
                        if (diag) {  // the FMA-pipe exp2 clamps -inf: zero masked keys
                            pv.x = sv[col] == -INFINITY ? 0.f : pv.x;
                            pv.y = sv[col + 1] == -INFINITY ? 0.f : pv.y;
                        }
                    } else {
                        const float2 xv = ffma2(make_float2(sv[col], sv[col + 1]), sl2v, nb2);
                        pv.x = ex2_mufu(xv.x);
                        pv.y = ex2_mufu(xv.y);
                    }
                    lacc = fadd2(lacc, pv);
                    pk[i] = ptx::pack_bf16(pv.x, pv.y);
                }
                ptx::tmem_st16(lane_base + x * BKV + c * 16, pk);
            }
            return lacc.x + lacc.y;
        };
        for (int j = 0; j < nt; ++j) {
            ptx::mbar_wait(&s_full[x], j & 1);
            // PV_x(j-1) completed before S_x(j) (issued behind it): observe its phase every step,
            // so no o_done phase completes unwaited (compute-sanitizer synccheck) -- free here
            if (j > 0) ptx::mbar_wait(&o_done[x], (j - 1) & 1);
            ptx::tc_fence_after();
            const bool tr = quarter == 0 && lane == 0 && x < 2;
            if (tr) ATTN_TRACE(4 + x, j);
            float sv[BKV];
            {
                uint32_t r[BKV / 32][32];
#pragma unroll
                for (int c = 0; c < BKV / 32; ++c) ptx::tmem_ld32(lane_base + x * BKV + c * 32, r[c]);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < BKV / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[c][i]);
            }
            if (tr) ATTN_TRACE(6 + x, j);
            const bool diag = j * BKV + BKV - 1 > tile_first_abs;
            if (diag) {
                // keys [j*BKV, j*BKV + nvis) are visible to this row; 32-bit compares against
                // compile-time column indices, applied only on the diagonal tile
                const int v = abs_row - j * BKV + 1;
                const int nvis = v < 0 ? 0 : (v > BKV ? BKV : v);
#pragma unroll
                for (int i = 0; i < BKV; ++i) sv[i] = i < nvis ? sv[i] : -INFINITY;
            }
            // row max: four independent FMNMX3 chains (two new columns per instruction)
            static_assert(BKV % 8 == 0, "row max layout");
            float m4[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
            for (int i = 4; i + 8 <= BKV; i += 8) {
#pragma unroll
                for (int k = 0; k < 4; ++k) m4[k] = fmax3(m4[k], sv[i + k], sv[i + 4 + k]);
            }
            const float mx = fmax3(fmax3(m4[0], m4[1], sv[BKV - 4]), fmax3(m4[2], m4[3], sv[BKV - 3]),
                                   fmaxf(sv[BKV - 2], sv[BKV - 1])) * a.sl2;  // scale > 0
            if (tr) ATTN_TRACE(8 + x, j);
            const bool need = mx > m_run + RESCALE_THRESHOLD;
            if (__any_sync(0xffffffffu, need)) {
                const float m_new = need ? mx : m_run;
                const float alpha = need ? exp2f(m_run - m_new) : 1.0f;
                if (j > 0) {  // PV_x(j-1) complete: waited for at the top of the step
#pragma unroll
                    for (int c = 0; c < HD / 16; ++c) {
                        uint32_t r[16];
                        ptx::tmem_ld16(lane_base + C::O_BASE + x * HD + c * 16, r);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                        ptx::tmem_st16(lane_base + C::O_BASE + x * HD + c * 16, r);
                    }
                    ptx::tmem_st_wait();
                }
                l = __fmul_rn(l, alpha);  // explicit roundings: attn_tb.cu restates them
                m_run = m_new;
            }
            const float lsum = exp_store(sv, m_run, diag);
            l = __fadd_rn(l, lsum);
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (tr) ATTN_TRACE(10 + x, j);
            if (lane == 0) ptx::mbar_arrive(&p_full[x]);
        }
        // epilogue: O / l -> bf16
        const float inv = 1.0f / l;
        ptx::mbar_wait(&o_done[x], (nt - 1) & 1);
        ptx::tc_fence_after();
        bf16* orow = a.O + row * a.ldo + static_cast<int64_t>(h) * HD;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(lane_base + C::O_BASE + x * HD + c * 32, r);
            ptx::tmem_ld_wait();
            if (row < a.q_rows) {
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    uint4 v;
                    v.x = ptx::pack_bf16(__uint_as_float(r[i + 0]) * inv, __uint_as_float(r[i + 1]) * inv);
                    v.y = ptx::pack_bf16(__uint_as_float(r[i + 2]) * inv, __uint_as_float(r[i + 3]) * inv);
                    v.z = ptx::pack_bf16(__uint_as_float(r[i + 4]) * inv, __uint_as_float(r[i + 5]) * inv);
                    v.w = ptx::pack_bf16(__uint_as_float(r[i + 6]) * inv, __uint_as_float(r[i + 7]) * inv);
                    *reinterpret_cast<uint4*>(orow + c * 32 + i) = v;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<TMEM_COLS>(tmem);
    }
    if (KVP_ATTN_TRACE_ON && a.cta_trace && threadIdx.x == 0) {
        unsigned long long* r = a.cta_trace + 4 * (blockIdx.y * gridDim.x + blockIdx.x);
        uint32_t smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        r[0] = t_start;
        r[1] = globaltimer();
        r[2] = smid;
        r[3] = static_cast<unsigned long long>(n_kt[NT - 1]);
    }
}

int mma_wait_flag() {
    static const int w = [] {
        const char* e = getenv("KVP_ATTN_MMA_WAIT");
        return e ? atoi(e) : 0;
    }();
    return w;
}

template <int HD, int NT, int BKV, int NPOLY>
void launch(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    CUtensorMap tq, tk, tv;
    if (!make_tmap_bf16(&tq, Q, static_cast<uint64_t>(sh.n_heads) * HD, sh.q_rows, sh.ldq, 64, BQ) ||
        !make_tmap_bf16(&tk, K, static_cast<uint64_t>(sh.n_kv_heads) * HD, sh.k_rows, sh.ldkv, 64, BKV) ||
        !make_tmap_bf16(&tv, V, static_cast<uint64_t>(sh.n_kv_heads) * HD, sh.k_rows, sh.ldkv, 64, BKV))
        throw std::runtime_error("attn_tc: cuTensorMapEncodeTiled failed");
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        cudaFuncSetAttribute(attn_tc_kernel<HD, NT, BKV, NPOLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ACfg<HD, NT, BKV>::SMEM);
        configured = dev;
    }
    AttnArgs a{sh.q_rows, sh.k_rows, sh.offset, sh.n_heads, sh.n_heads / sh.n_kv_heads, sh.ldo, O,
               (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f, mma_wait_flag(), nullptr, -1, nullptr};
    dim3 grid(static_cast<unsigned>(sh.n_heads), static_cast<unsigned>((sh.q_rows + NT * BQ - 1) / (NT * BQ)));
    // tuning only: KVP_ATTN_CTA_TRACE=<file> records {start ns, end ns, smid, key steps} per CTA
    static const char* cta_env = getenv("KVP_ATTN_CTA_TRACE");
    const size_t n_cta = static_cast<size_t>(grid.x) * grid.y;
    if (cta_env) {
        static unsigned long long* cbuf = nullptr;
        static size_t cap = 0;
        if (cap < n_cta) {
            if (cbuf) cudaFree(cbuf);
            cudaMalloc(&cbuf, n_cta * 4 * sizeof(unsigned long long));
            cap = n_cta;
        }
        a.cta_trace = cbuf;
    }
    // tuning only: KVP_ATTN_TRACE=<cta> records one CTA's pipeline events into KVP_ATTN_TRACE_OUT
    static const char* trace_env = getenv("KVP_ATTN_TRACE");
    if (trace_env) {
        static uint32_t* buf = nullptr;
        if (!buf) cudaMalloc(&buf, 16 * 512 * sizeof(uint32_t));
        cudaMemsetAsync(buf, 0, 16 * 512 * sizeof(uint32_t), s);
        a.trace = buf;
        a.trace_blk = atoi(trace_env);
    }
    note_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads_for<NT>());
    cfg.dynamicSmemBytes = ACfg<HD, NT, BKV>::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, attn_tc_kernel<HD, NT, BKV, NPOLY>, tq, tk, tv, a);
    if (a.cta_trace) {
        std::vector<unsigned long long> host(n_cta * 4);
        cudaMemcpyAsync(host.data(), a.cta_trace, host.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (FILE* f = fopen(cta_env, "wb")) {
            fwrite(host.data(), host.size() * sizeof(unsigned long long), 1, f);
            fclose(f);
        }
    }
    if (a.trace) {
        uint32_t host[16 * 512];
        cudaMemcpyAsync(host, a.trace, sizeof(host), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const char* out = getenv("KVP_ATTN_TRACE_OUT");
        if (FILE* f = fopen(out ? out : "attn_trace.bin", "wb")) {
            fwrite(host, sizeof(host), 1, f);
            fclose(f);
        }
    }
}

template <int HD, int NT, int BKV>
void launch_poly(int np, const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    switch (np) {
        case 0: launch<HD, NT, BKV, 0>(Q, K, V, O, sh, s); break;
        case 2: launch<HD, NT, BKV, 2>(Q, K, V, O, sh, s); break;
        case 4: launch<HD, NT, BKV, 4>(Q, K, V, O, sh, s); break;
        default: throw std::runtime_error("attn_tc: KVP_ATTN_POLY must be 0, 2 or 4");
    }
}

}  // namespace

bool attn_tc_supported(int head_dim) { return head_dim == 64 || head_dim == 128; }

void attn_bf16_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    // KVP_ATTN_POLY = column pairs (of every 16) whose exp2 runs on the FMA pipe
    static const int poly = [] {
        const char* e = getenv("KVP_ATTN_POLY");
        return e ? atoi(e) : -1;
    }();
    if (sh.head_dim != 128 && sh.head_dim != 64) throw std::runtime_error("attn_tc: head_dim must be 64 or 128");
    if (sh.offset + sh.q_rows + 128 >= (int64_t(1) << 31)) throw std::runtime_error("attn_tc: positions must be < 2^31");
    // hd 64: two query tiles x 128-key tiles; KVP_ATTN_HD64_TILES=3 selects three query tiles x
    // 96-key tiles (TMEM 3 x (96 + 64) columns, three softmax warps per SMSP's MUFU) -- measured
    // no faster: the in-order MMA issuer then waits ~1200 clk per tile for its turn
    static const int hd64_tiles = [] {
        const char* e = getenv("KVP_ATTN_HD64_TILES");
        return e ? atoi(e) : 2;
    }();
    const bool h128 = sh.head_dim == 128;
    // The double-buffered one-tile-per-CTA kernel (attn_tb.cu) or this kernel's two-tile CTAs:
    // bitwise identical, so the choice never changes a row.  KVP_ATTN_TB=0 / 1 forces either.
    static const int tb = [] {
        const char* e = getenv("KVP_ATTN_TB");
        return e ? atoi(e) : -1;
    }();
    const int64_t ctas256 = static_cast<int64_t>(sh.n_heads) * ((sh.q_rows + 255) / 256);
    // hd 64 (Falcon) the same way, while this kernel runs its default two 128-key tiles -- the
    // layout attn_tb restates bit for bit
    const bool tb_ok = h128 || hd64_tiles == 2;
    bool pick_tb;
    if (sh.offset >= sh.q_rows) {
        // a later rank's chunk: every CTA walks about the same number of key tiles, so the
        // choice is wave quantisation -- attn_tb's CTAs are half as tall (twice as many); take it
        // when its last wave is fuller, or (hd 128) when this kernel's grid is a single partial
        // wave.  Measured isolated (profiles/r02/attn_select_rank.txt, TF/s tc / tb): Llama rank
        // chunks of 512 / 1024 / 1280 / 1536 / 1792 / 2048 rows 437/715, 773/815, 674/782,
        // 801/955, 917/896, 1099/1027; Falcon 512 / 640 / 1024 rows 582/564, 401/497, 623/597 --
        // the rule picks the faster kernel in all nine.
        const int64_t sms = num_sms();
        auto fill = [&](int64_t c) { return static_cast<double>(c) / (((c + sms - 1) / sms) * sms); };
        const int64_t ctas128 = static_cast<int64_t>(sh.n_heads) * ((sh.q_rows + 127) / 128);
        const double f_tc = fill(ctas256), f_tb = fill(ctas128);
        pick_tb = f_tb > 1.02 * f_tc || (h128 && ctas256 <= sms && f_tb >= f_tc);
    } else {
        // the causal grid of a first chunk / the serial prompt: longest-first two-tile CTAs on
        // big grids (4k p = 1 in the full step: 5.8 vs 5.9 ms; 16k: ~1215 vs ~1085 TF/s)
        pick_tb = ctas256 <= 2 * 148;
    }
    if (tb_ok && (tb == 1 || (tb < 0 && pick_tb))) return attn_bf16_tb(Q, K, V, O, sh, s);
    const int np = poly >= 0 ? poly : (h128 ? DEFAULT_POLY_128 : DEFAULT_POLY_64);
    if (h128)
        launch_poly<128, 2, 128>(np, Q, K, V, O, sh, s);
    else if (hd64_tiles == 2)
        launch_poly<64, 2, 128>(np, Q, K, V, O, sh, s);
    else
        launch_poly<64, 3, 96>(np, Q, K, V, O, sh, s);
}

}  // namespace kvp
