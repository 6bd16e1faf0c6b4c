// attn_tb.cu -- prefix-causal flash attention with the score tile and P double-buffered in
// tensor memory (tcgen05, one 128-query tile per CTA); head_dim 128 or 64.
//
// Reference: causal_attention (model.hpp:112-158).  A CTA owns 128 query rows of one head and
// walks the 128-key tiles [0, offset + last query]:
//   S_j  = Q K_j^T   (SS MMA, M = N = 128)  -> S buffer j % 2 in TMEM
//   O   += P_j V_j   (TS MMA: A = P_j, bf16 packed in P buffer j % 2; B = V_j MN-major)
// The MMA issuer computes S_{j+2} as soon as the softmax has read S_j into registers
// (`s_free`), and PV_j when P_j lands: the scores of the next tiles never wait for the
// softmax.  (In attn_tc.cu P aliases its tile's only S buffer, so each query tile runs the
// chain S -> softmax -> PV -> S, ~3.4k clk for 1k clk of its own MMAs.)
// TMEM (512 columns): S_0 | S_1 (128 f32 columns each) | P_0 | P_1 (64 columns each) | O (HD).
// Warps: 0 TMA producer (Q, K), 10 TMA producer (V), 1 MMA issuer + TMEM owner (all three run
// converged; one elect.sync lane issues), 2..9 softmax in two sets (set j % 2 owns key tile j,
// one thread per query row; warp w reads TMEM lane quarter w % 4).  The running row max and
// the row sum are handed between the sets in tile order, so each SMSP has two softmax warps in
// different phases of consecutive tiles feeding its MUFU, and every row gets exactly
// attn_tc.cu's operations in attn_tc.cu's order -- the two kernels are bitwise identical, and
// which one a rank's grid selects never changes a result.  O is rescaled in TMEM only when a
// row max grows by more than 2^8; key tiles are aligned to absolute key 0 and rows are
// independent, so results do not depend on how the context is split over ranks.
// (Variants measured and not kept -- CTA pairs, three sets, two threads per row, two issuing
// warps, a persistent grid, FMA-pipe exp2: profiles/r02/README.md.)
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "kernels.cuh"
#include "ptx.cuh"
#include "softmax.cuh"

namespace kvp {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

namespace {
using namespace smx;

constexpr int BQ = 128;  // query rows per CTA
constexpr int BK = 128;  // keys per tile
constexpr int NS = 2;    // S buffers (and P buffers)
constexpr int THREADS = 352;  // 11 warps
constexpr uint32_t P_COL = NS * BK;                  // P_0 | P_1 at TMEM columns 256, 320 (bf16 packed)
constexpr uint32_t O_COL = P_COL + NS * BK / 2;      // O at TMEM column 384 (HD columns)
constexpr uint32_t BAR_BYTES = 256;
constexpr uint32_t XCH_BYTES = 5 * BQ * 4;  // running row max handed between the sets + row sums
constexpr float RESCALE_THRESHOLD = 8.0f;
// head_dim 128 (Llama) or 64 (Falcon): Q / K / V tiles are HD / 64 SW128 boxes of 64 dims
template <int HD>
struct TbCfg {
    static constexpr int KST = HD == 128 ? 3 : 4, VST = HD == 128 ? 2 : 3;
    static constexpr uint32_t Q_BYTES = BQ * HD * 2;   // 32 / 16 KB
    static constexpr uint32_t KV_BYTES = BK * HD * 2;  // 32 / 16 KB
    static constexpr uint32_t NEED = Q_BYTES + (KST + VST) * KV_BYTES + BAR_BYTES + XCH_BYTES;
    static constexpr uint32_t SMEM = NEED + 1024;
    static_assert(SMEM <= 232448, "attention smem over the 227 KB opt-in limit");
    static_assert(O_COL + HD <= 512, "TMEM holds S x 2, P x 2 and O");
};

struct PairArgs {
    int64_t q_rows, offset;
    int group;
    int64_t ldo;
    bf16* O;
    float sl2;                      // softmax scale * log2(e)
    unsigned long long* cta_trace;  // tuning only (KVP_ATTN_CTA_TRACE)
    uint32_t* trace;                // tuning only (KVP_ATTN_TRACE): SM clock of pipeline events of one CTA
    int trace_blk;
};

// trace[ev * 512 + j] = clock() of event ev for key tile j in CTA a.trace_blk
#ifndef KVP_ATTN_TRACE_ON
#define KVP_ATTN_TRACE_ON 0  // tuning builds: KVP_NVCC_FLAGS=-DKVP_ATTN_TRACE_ON=1
#endif
#define TB_TRACE(ev, j)                                                                                     \
    do {                                                                                                    \
        if (KVP_ATTN_TRACE_ON && a.trace && static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x) == a.trace_blk && (j) < 512)   \
            a.trace[(ev) * 512 + (j)] = static_cast<uint32_t>(clock());                                     \
    } while (0)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int HD, int NPOLY>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tb_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, PairArgs a) {
    using TC = TbCfg<HD>;
    constexpr int KST = TC::KST, VST = TC::VST;
    constexpr uint32_t Q_BYTES = TC::Q_BYTES, KV_BYTES = TC::KV_BYTES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + Q_BYTES;
    uint8_t* sV = sK + KST * KV_BYTES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sV + VST * KV_BYTES);
    uint64_t* q_full = bar;
    uint64_t* k_full = q_full + 1;  // [KST]
    uint64_t* k_empty = k_full + KST;
    uint64_t* v_full = k_empty + KST;
    uint64_t* v_empty = v_full + VST;
    uint64_t* s_full = v_empty + VST;  // [NS]
    uint64_t* s_free = s_full + NS;    // [NS] S_j read into registers (4 warps of set j & 1)
    uint64_t* p_full = s_free + NS;    // [NS] P_j in TMEM (4 warps of set j & 1)
    uint64_t* o_done = p_full + NS;    // [2] PV_j completion, alternating
    uint64_t* o_final = o_done + 2;
    uint64_t* l_ready = o_final + 1;  // [2 sets][4 lane quarters] row sum after the set's tile
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(l_ready + 8);
    float* xm = reinterpret_cast<float*>(smem + Q_BYTES + (KST + VST) * KV_BYTES + BAR_BYTES);  // [BQ] running max
    float* xl = xm + BQ;                                                                      // [2][BQ] row sum by tile parity

    const unsigned long long t_start = KVP_ATTN_TRACE_ON && a.cta_trace && threadIdx.x == 0 ? gtimer() : 0;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = static_cast<int>(blockIdx.x);
    const int g = h / a.group;
    const int num_tiles = static_cast<int>((a.q_rows + BQ - 1) / BQ);
    // heaviest (latest) query tiles first: the block scheduler walks x (heads) fastest
    const int qt = num_tiles - 1 - static_cast<int>(blockIdx.y);
    const int64_t q0 = static_cast<int64_t>(qt) * BQ;
    const int64_t last = q0 + BQ - 1 < a.q_rows - 1 ? q0 + BQ - 1 : a.q_rows - 1;
    const int n = static_cast<int>((a.offset + last) / BK) + 1;  // key tiles

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
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&s_full[s], 1);
            ptx::mbar_init(&s_free[s], 4);  // the 4 softmax warps of the set that owns buffer s
            ptx::mbar_init(&p_full[s], 4);
        }
        ptx::mbar_init(&o_done[0], 1);
        ptx::mbar_init(&o_done[1], 1);
        ptx::mbar_init(o_final, 1);
        for (int s = 0; s < 8; ++s) ptx::mbar_init(&l_ready[s], 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();

    if (warp == 0) {
        // K producer: Q, then K_t as soon as S_{t-KST} has read its stage.  V has its own
        // producer (warp 10): a V stage waits for PV_{t-VST}, and a single producer would hold
        // the next K behind it (measured: the S issue then trails PV completion + a TMA round trip)
        ptx::mbar_arrive_expect_tx_w(q_full, Q_BYTES);
        for (int hv = 0; hv < HD / 64; ++hv)
            ptx::tma_load_2d_w(sQ + hv * BQ * 128, &tmQ, q_full, h * HD + hv * 64, static_cast<int32_t>(q0));
        for (int t = 0; t < n; ++t) {
            const int sk = t % KST;
            ptx::mbar_wait(&k_empty[sk], ((t / KST) & 1) ^ 1);
            TB_TRACE(8, t);
            ptx::mbar_arrive_expect_tx_w(&k_full[sk], KV_BYTES);
            for (int hv = 0; hv < HD / 64; ++hv)
                ptx::tma_load_2d_w(sK + sk * KV_BYTES + hv * BK * 128, &tmK, &k_full[sk], g * HD + hv * 64, t * BK);
        }
    } else if (warp == 10) {
        for (int t = 0; t < n; ++t) {
            const int sv = t % VST;
            ptx::mbar_wait(&v_empty[sv], ((t / VST) & 1) ^ 1);
            TB_TRACE(9, t);
            ptx::mbar_arrive_expect_tx_w(&v_full[sv], KV_BYTES);
            for (int hv = 0; hv < HD / 64; ++hv)
                ptx::tma_load_2d_w(sV + sv * KV_BYTES + hv * BK * 128, &tmV, &v_full[sv], g * HD + hv * 64, t * BK);
        }
    } else if (warp == 1) {
        // the whole warp runs the issue loop converged; one elected lane issues each
        // tcgen05.mma / commit.  Descriptors are built once and advanced by constant offsets
        // (the 14-bit address field holds addr >> 4: +2 per 32-byte K step, no carry).
        constexpr uint32_t idesc_s = ptx::idesc_bf16(BQ, BK, 0);
        constexpr uint32_t idesc_o = ptx::idesc_bf16(BQ, HD, 1);  // B = V is MN-major
        const uint64_t qdesc = ptx::smem_desc_sw128(ptx::smem_u32(sQ), 16, 1024);
        const uint64_t kdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sK), 16, 1024);
        const uint64_t vdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(sV), BK * 128, 1024);
        auto issue_s = [&](int t) {
            const int s = t % KST;
            ptx::mbar_wait(&k_full[s], (t / KST) & 1);
            ptx::tc_fence_after();
            if (lane == 0) TB_TRACE(0, t);
            const uint64_t kdesc = kdesc0 + static_cast<uint64_t>((s * KV_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < HD / 16; ++k) {
                const uint64_t off_q = ((k >> 2) * (BQ * 128) + (k & 3) * 32) >> 4;
                const uint64_t off_k = ((k >> 2) * (BK * 128) + (k & 3) * 32) >> 4;
                ptx::mma_bf16_ss_w(tmem + (t % NS) * BK, qdesc + off_q, kdesc + off_k, idesc_s, k != 0);
            }
            if (lane == 0) TB_TRACE(10, t);  // all 8 S MMAs accepted by the issue queue
            ptx::mma_commit_w(&s_full[t % NS]);
            ptx::mma_commit_w(&k_empty[s]);
        };
        ptx::mbar_wait(q_full, 0);
        issue_s(0);
        if (n > 1) issue_s(1);
        for (int j = 0; j < n; ++j) {
            const int b = j & 1, sv = j % VST;
            // S_{j+2} reuses S buffer b as soon as the softmax has read S_j into registers
            // (early in its step): the scores never wait for P_j or PV_j
            if (j + 2 < n) {
                ptx::mbar_wait(&s_free[b], (j >> 1) & 1);
                issue_s(j + 2);
            }
            ptx::mbar_wait(&p_full[b], (j >> 1) & 1);
            ptx::mbar_wait(&v_full[sv], (j / VST) & 1);
            ptx::tc_fence_after();
            if (lane == 0) TB_TRACE(1, j);
            const uint64_t vdesc = vdesc0 + static_cast<uint64_t>((sv * KV_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                // keys 16k..16k+15: P_b packed at columns 8k .. 8k + 7; V rows 16k.. (SBO 1024 per 8)
                const uint32_t pa = tmem + P_COL + b * (BK / 2) + k * 8;
                ptx::mma_bf16_ts_w(tmem + O_COL, pa, vdesc + static_cast<uint64_t>((k * 16 * 128) >> 4), idesc_o,
                                   (j | k) != 0);
            }
            if (lane == 0) TB_TRACE(11, j);  // all 8 PV MMAs accepted
            ptx::mma_commit_w(&o_done[j & 1]);
            ptx::mma_commit_w(&v_empty[sv]);
        }
        ptx::mma_commit_w(o_final);
    } else if (warp >= 2 && warp < 10) {
        // two softmax sets: warps 2..5 take the even key tiles, 6..9 the odd ones, one thread per
        // query row (TMEM lane).  The only serial link between consecutive tiles is the running
        // row max, handed to the other set through shared memory + a named barrier as soon as it
        // is known, so one set's exp2 overlaps the other's TMEM loads and row max.
        const int set = static_cast<int>(warp - 2) >> 2;
        const uint32_t quarter = warp & 3;
        const int xrow = static_cast<int>(quarter) * 32 + static_cast<int>(lane);
        const int64_t row = q0 + xrow;
        const int abs_row = static_cast<int>(a.offset + row);  // positions < 2^31 (host-checked)
        const int warp_first_abs = abs_row - static_cast<int>(lane);
        const uint32_t lane_base = tmem + ((quarter * 32u) << 16);
        const uint32_t bar_in = (set == 0 ? 5u : 1u) + quarter, bar_out = (set == 0 ? 1u : 5u) + quarter;
        const float2 sl2v = make_float2(a.sl2, a.sl2);
        const float2 sl2y = make_float2(a.sl2 * (1.f / 256.f), a.sl2 * (1.f / 256.f));
        // The row sum runs through the tiles in order, l_j = l_{j-1} * alpha_j + lsum_j -- the
        // very operations and order of attn_tc.cu, so the two kernels give bitwise equal rows
        // and Serial == KVR stays bitwise whichever kernel a rank's grid selects.  l_{j-1} comes
        // from the other set; each set finalises its tile j one tile later (at j + 2, after the
        // row-max handoff), when the other set has long published l_{j-1}.
        float pend_alpha = 1.f, pend_lsum = 0.f;
        int pend_j = -1;
        auto finalize_l = [&]() {
            float l_prev = 0.f;
            if (pend_j > 0) {
                ptx::mbar_wait(&l_ready[(1 - set) * 4 + quarter], ((pend_j - 1) >> 1) & 1);
                l_prev = xl[((pend_j - 1) & 1) * BQ + xrow];
            }
            // attn_tc.cu's two roundings (l *= alpha, then l += lsum) -- an FFMA here would round
            // once and break the bitwise equality whenever a row max was re-based at a tile j > 0
            xl[(pend_j & 1) * BQ + xrow] = __fadd_rn(__fmul_rn(l_prev, pend_alpha), pend_lsum);
            __threadfence_block();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&l_ready[set * 4 + quarter]);
            pend_j = -1;
        };
        for (int j = set; j < n; j += 2) {
            const int b = set;  // == j & 1
            ptx::mbar_wait(&s_full[b], (j >> 1) & 1);
            ptx::tc_fence_after();
            const bool tr = quarter == 0 && lane == 0;
            if (tr) TB_TRACE(2 + set, j);
            const uint32_t sb = lane_base + b * BK;
            float sv[BK];
            {
                uint32_t r[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld32(sb + c * 32, r[c]);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[c][i]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&s_free[b]);  // S_j is in registers: S_{j+2} may overwrite it
            const bool diag = j * BK + BK - 1 > warp_first_abs;
            if (diag) {
                const int vis = abs_row - j * BK + 1;
                const int nvis = vis < 0 ? 0 : (vis > BK ? BK : vis);
#pragma unroll
                for (int i = 0; i < BK; ++i) sv[i] = i < nvis ? sv[i] : -INFINITY;
            }
            float m4[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
            for (int i = 4; i + 8 <= BK; i += 8) {
#pragma unroll
                for (int k = 0; k < 4; ++k) m4[k] = fmax3(m4[k], sv[i + k], sv[i + 4 + k]);
            }
            const float mx = fmax3(fmax3(m4[0], m4[1], sv[BK - 4]), fmax3(m4[2], m4[3], sv[BK - 3]),
                                   fmaxf(sv[BK - 2], sv[BK - 1])) * a.sl2;  // scale > 0
            // the running max after tile j-1 (from the other set), then publish the one after j
            float m_prev = -INFINITY;
            if (j > 0) {
                ptx::named_sync(bar_in, 64);
                m_prev = xm[xrow];
            }
            const bool need = mx > m_prev + RESCALE_THRESHOLD;
            const float m_new = need ? mx : m_prev;
            xm[xrow] = m_new;
            if (j + 1 < n) ptx::named_arrive(bar_out, 64);
            if (tr) TB_TRACE(4 + set, j);
            if (j > 0 && __any_sync(0xffffffffu, need)) {
                // O must hold exactly PV_0..PV_{j-1} (PV_{j-3} completed before S_j, so the
                // alternating barrier cannot alias)
                const float alpha = need ? exp2f(m_prev - m_new) : 1.0f;
                ptx::mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int c = 0; c < HD / 16; ++c) {
                    uint32_t r[16];
                    const uint32_t oc = lane_base + O_COL + c * 16;
                    ptx::tmem_ld16(oc, r);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                    ptx::tmem_st16(oc, r);
                }
                ptx::tmem_st_wait();
            }
            // the row sum's rescale factor, exactly as attn_tc.cu applies it (1 when the max holds)
            const float alpha_l = need ? exp2f(m_prev - m_new) : 1.0f;
            if (pend_j >= 0) finalize_l();  // this set's previous tile (j - 2)
            // P_b was last read by PV_{j-2}: complete long ago (checked, not assumed)
            if (j >= 2) {
                ptx::mbar_wait(&o_done[b], ((j - 2) >> 1) & 1);
                ptx::tc_fence_after();
            }
            // P = 2^(s * sl2 - m) -> bf16, 128 keys packed into the 64 columns of P_b
            const float2 nb2 = make_float2(-m_new, -m_new);
            const float2 yb2 = make_float2((POLY_BIAS - m_new) * (1.f / 256.f), (POLY_BIAS - m_new) * (1.f / 256.f));
            float2 lacc = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < BK / 32; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = c * 32 + 2 * i;
                    float2 pv;
                    if (i >= 16 - NPOLY) {
                        pv = ex2_poly_sat(ffma2_sat(make_float2(sv[col], sv[col + 1]), sl2y, yb2));
                        if (diag) {
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
                ptx::tmem_st16(lane_base + P_COL + b * (BK / 2) + c * 16, pk);
            }
            const float lsum = lacc.x + lacc.y;
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (tr) TB_TRACE(6 + set, j);
            if (lane == 0) ptx::mbar_arrive(&p_full[b]);
            pend_alpha = alpha_l;  // l_j is finalised at this set's next tile (or after the loop)
            pend_lsum = lsum;
            pend_j = j;
        }
        if (pend_j >= 0) finalize_l();
        // epilogue: l_{n-1} from whichever set ran the last tile; each set stores half the row
        ptx::named_sync(9 + quarter, 64);
        const float inv = 1.0f / xl[((n - 1) & 1) * BQ + xrow];
        ptx::mbar_wait(o_final, 0);
        ptx::tc_fence_after();
        bf16* orow = a.O + row * a.ldo + static_cast<int64_t>(h) * HD + set * (HD / 2);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(lane_base + O_COL + set * (HD / 2) + c * 32, r);
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
        ptx::tmem_dealloc<512>(tmem);
    }
    if (KVP_ATTN_TRACE_ON && a.cta_trace && threadIdx.x == 0) {
        unsigned long long* r = a.cta_trace + 4 * (blockIdx.y * gridDim.x + blockIdx.x);
        uint32_t smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        r[0] = t_start;
        r[1] = gtimer();
        r[2] = smid;
        r[3] = static_cast<unsigned long long>(n);
    }
}

template <int HD, int NPOLY>
void launch(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    constexpr uint32_t SMEM = TbCfg<HD>::SMEM;
    CUtensorMap tq, tk, tv;
    if (!make_tmap_bf16(&tq, Q, static_cast<uint64_t>(sh.n_heads) * HD, sh.q_rows, sh.ldq, 64, BQ) ||
        !make_tmap_bf16(&tk, K, static_cast<uint64_t>(sh.n_kv_heads) * HD, sh.k_rows, sh.ldkv, 64, BK) ||
        !make_tmap_bf16(&tv, V, static_cast<uint64_t>(sh.n_kv_heads) * HD, sh.k_rows, sh.ldkv, 64, BK))
        throw std::runtime_error("attn_tb: cuTensorMapEncodeTiled failed");
    auto kern = attn_tb_kernel<HD, NPOLY>;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        configured = dev;
    }
    PairArgs a{sh.q_rows, sh.offset, sh.n_heads / sh.n_kv_heads, sh.ldo, O,
               (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f, nullptr, nullptr, -1};
    static const char* trace_env = getenv("KVP_ATTN_TRACE");
    static uint32_t* tbuf = nullptr;
    if (trace_env) {
        if (!tbuf) cudaMalloc(&tbuf, 16 * 512 * sizeof(uint32_t));
        cudaMemsetAsync(tbuf, 0, 16 * 512 * sizeof(uint32_t), s);
        a.trace = tbuf;
        a.trace_blk = atoi(trace_env);
    }
    const dim3 grid(static_cast<unsigned>(sh.n_heads), static_cast<unsigned>((sh.q_rows + BQ - 1) / BQ));
    static const char* cta_env = getenv("KVP_ATTN_CTA_TRACE");
    const size_t n_cta = static_cast<size_t>(grid.x) * grid.y;
    static unsigned long long* cbuf = nullptr;
    static size_t cap = 0;
    if (cta_env) {
        if (cap < n_cta) {
            if (cbuf) cudaFree(cbuf);
            cudaMalloc(&cbuf, n_cta * 4 * sizeof(unsigned long long));
            cap = n_cta;
        }
        a.cta_trace = cbuf;
    }
    note_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, a);
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
    if (a.cta_trace) {
        std::vector<unsigned long long> host(n_cta * 4);
        cudaMemcpyAsync(host.data(), a.cta_trace, host.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (FILE* f = fopen(cta_env, "wb")) {
            fwrite(host.data(), host.size() * sizeof(unsigned long long), 1, f);
            fclose(f);
        }
    }
}

}  // namespace

void attn_bf16_tb(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    if (sh.head_dim != 128 && sh.head_dim != 64) throw std::runtime_error("attn_tb: head_dim must be 64 or 128");
    if (sh.offset + sh.q_rows + 2 * BQ >= (int64_t(1) << 31)) throw std::runtime_error("attn_tb: positions must be < 2^31");
    static const int poly = [] {
        const char* e = getenv("KVP_ATTN_POLY");
        return e ? atoi(e) : 0;
    }();
    const bool h128 = sh.head_dim == 128;
    switch (poly) {
        case 0: h128 ? launch<128, 0>(Q, K, V, O, sh, s) : launch<64, 0>(Q, K, V, O, sh, s); break;
        case 2: h128 ? launch<128, 2>(Q, K, V, O, sh, s) : launch<64, 2>(Q, K, V, O, sh, s); break;
        case 4: h128 ? launch<128, 4>(Q, K, V, O, sh, s) : launch<64, 4>(Q, K, V, O, sh, s); break;
        default: throw std::runtime_error("attn_tb: KVP_ATTN_POLY must be 0, 2 or 4");
    }
}

}  // namespace kvp
