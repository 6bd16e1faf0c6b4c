// attn_tc.cu -- prefix-causal flash attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Reference: causal_attention (model.hpp:112-158).  One CTA owns TWO 128-query tiles (a, b)
// of one head -- absolute positions offset + q0 ... offset + q0 + 255 -- and walks the
// 128-key tiles [0, offset + last query]; each K/V tile is loaded once for both query tiles.
//   warp 0      TMA producer: Q_a, Q_b once, then K/V tiles through a 2-stage smem ring;
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
#include <cstdlib>
#include <mutex>
#include <stdexcept>

#include "kernels.cuh"
#include "ptx.cuh"

namespace kvp {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

namespace {

constexpr int BQ = 128;   // queries per tile (two tiles per CTA)
constexpr int BKV = 128;  // keys per tile
constexpr int THREADS = 576;  // warp 0 TMA, warp 1 MMA, warps 2..17 softmax (8 per query tile)
constexpr uint32_t TMEM_COLS = 512;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: p <= 2^8 between rescales

template <int HD>
struct ACfg {
    static constexpr int HALVES = HD / 64;  // 64-wide (128 B) TMA boxes
    static constexpr uint32_t Q_BYTES = BQ * HD * 2;
    static constexpr uint32_t KV_BYTES = BKV * HD * 2;
    static constexpr uint32_t SMEM = 2 * Q_BYTES + 4 * KV_BYTES + 1024 + 256 + 6144;  // + row-max/sum exchange
};

// ---- packed f32x2 arithmetic (sm_100: FFMA2 / FADD2) and exp2 on two pipes ----
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
// MUFU.EX2 (ex2(-inf) = +0 exactly)
__device__ __forceinline__ float ex2_mufu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x on the FMA pipe: x = n + f with n = rint(x) (magic-number add), 2^f by a degree-3
// minimax polynomial on [-1/2, 1/2] (max rel. error 1.0e-4, far below bf16's 3.9e-3), 2^n
// added into the exponent bits.  x is clamped at -125 (masked lanes are zeroed by the
// caller), x <= 8 by the rescale threshold.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -125.f);
    x.y = fmaxf(x.y, -125.f);
    const float2 magic = make_float2(12582912.f, 12582912.f), neg1 = make_float2(-1.f, -1.f);
    const float2 t = fadd2(x, magic);
    const float2 n = fadd2(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = ffma2(n, neg1, x);
    float2 p = ffma2(make_float2(0.055008821f, 0.055008821f), f, make_float2(0.24221078f, 0.24221078f));
    p = ffma2(p, f, make_float2(0.6932829f, 0.6932829f));
    p = ffma2(p, f, make_float2(1.f, 1.f));
    float2 r;
    r.x = __uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23));
    r.y = __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23));
    return r;
}

struct AttnArgs {
    int64_t q_rows, k_rows, offset;
    int n_heads, group;
    int64_t ldo;
    bf16* O;
    float sl2;  // softmax scale * log2(e)
};

template <int HD, int POLY_FROM>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
    using C = ACfg<HD>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment by pointer arithmetic on the __shared__ array, so the compiler keeps
    // the shared state space (LDS/STS instead of generic loads/stores)
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint8_t* sQ = smem;                  // [2] query tiles
    uint8_t* sK = sQ + 2 * C::Q_BYTES;   // [2] stages
    uint8_t* sV = sK + 2 * C::KV_BYTES;  // [2] stages
    uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * C::KV_BYTES);
    uint64_t* q_full = bar;
    uint64_t* k_full = bar + 1;    // [2] stages
    uint64_t* v_full = bar + 3;    // [2] stages
    uint64_t* kv_empty = bar + 5;  // [2] stages
    uint64_t* s_full = bar + 7;    // [2] query tiles
    uint64_t* p_full = bar + 9;    // [2] query tiles
    uint64_t* o_done = bar + 11;   // [2] query tiles
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 13);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_pairs = static_cast<int>((a.q_rows + 2 * BQ - 1) / (2 * BQ));
    // grid = (heads, pairs): the block scheduler walks x fastest, so ALL heads of the heaviest
    // (latest) query pair are dispatched first -- a global longest-first order over the causal
    // work imbalance
    const int pair = num_pairs - 1 - static_cast<int>(blockIdx.y);
    const int h = blockIdx.x;
    const int g = h / a.group;
    const int64_t q0 = static_cast<int64_t>(pair) * 2 * BQ;
    // key tiles needed by each query tile (tile b covers tile a's range plus one)
    const int64_t last_a = (q0 + BQ - 1 < a.q_rows - 1) ? q0 + BQ - 1 : a.q_rows - 1;
    const int64_t last_b = (q0 + 2 * BQ - 1 < a.q_rows - 1) ? q0 + 2 * BQ - 1 : a.q_rows - 1;
    const int n_kt[2] = {static_cast<int>((a.offset + last_a) / BKV) + 1,
                         static_cast<int>((a.offset + (last_b > last_a ? last_b : last_a)) / BKV) + 1};

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmQ);
        ptx::tma_prefetch_desc(&tmK);
        ptx::tma_prefetch_desc(&tmV);
        ptx::mbar_init(q_full, 1);
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&k_full[s], 1);
            ptx::mbar_init(&v_full[s], 1);
            ptx::mbar_init(&kv_empty[s], 1);
            ptx::mbar_init(&s_full[s], 1);
            ptx::mbar_init(&p_full[s], 8);
            ptx::mbar_init(&o_done[s], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(q_full, 2 * C::Q_BYTES);
            for (int x = 0; x < 2; ++x)
                for (int hv = 0; hv < C::HALVES; ++hv)
                    ptx::tma_load_2d(sQ + x * C::Q_BYTES + hv * BQ * 128, &tmQ, q_full, h * HD + hv * 64,
                                     static_cast<int32_t>(q0 + x * BQ));
            for (int t = 0; t < n_kt[1]; ++t) {
                const int s = t & 1;
                ptx::mbar_wait(&kv_empty[s], ((t >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&k_full[s], C::KV_BYTES);
                for (int hv = 0; hv < C::HALVES; ++hv)
                    ptx::tma_load_2d(sK + s * C::KV_BYTES + hv * BKV * 128, &tmK, &k_full[s], g * HD + hv * 64, t * BKV);
                ptx::mbar_arrive_expect_tx(&v_full[s], C::KV_BYTES);
                for (int hv = 0; hv < C::HALVES; ++hv)
                    ptx::tma_load_2d(sV + s * C::KV_BYTES + hv * BKV * 128, &tmV, &v_full[s], g * HD + hv * 64, t * BKV);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc_s = ptx::idesc_bf16(BQ, BKV, 0);
            constexpr uint32_t idesc_o = ptx::idesc_bf16(BQ, HD, 1);  // B = V is MN-major
            auto issue_s = [&](int x, int t) {
                const int s = t & 1;
                ptx::mbar_wait(&k_full[s], (t >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t q_addr = ptx::smem_u32(sQ + x * C::Q_BYTES);
                const uint32_t k_addr = ptx::smem_u32(sK + s * C::KV_BYTES);
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint32_t off = (k >> 2) * (BQ * 128) + (k & 3) * 32;
                    const uint64_t ad = ptx::smem_desc_sw128(q_addr + off, 16, 1024);
                    const uint64_t bd = ptx::smem_desc_sw128(k_addr + (k >> 2) * (BKV * 128) + (k & 3) * 32, 16, 1024);
                    ptx::mma_bf16_ss(tmem + x * 128, ad, bd, idesc_s, k != 0);
                }
                ptx::mma_commit(&s_full[x]);
            };
            auto issue_pv = [&](int x, int t) {
                const int s = t & 1;
                ptx::mbar_wait(&p_full[x], t & 1);
                ptx::mbar_wait(&v_full[s], (t >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t v_addr = ptx::smem_u32(sV + s * C::KV_BYTES);
#pragma unroll
                for (int k = 0; k < BKV / 16; ++k) {
                    // B = V[keys 16k..16k+15][hd]: MN-major SW128, LBO = next 64-wide hd block,
                    // SBO = next 8 keys.
                    const uint64_t bd = ptx::smem_desc_sw128(v_addr + k * 16 * 128, BKV * 128, 1024);
                    ptx::mma_bf16_ts(tmem + 256 + x * 128, tmem + x * 128 + k * 8, bd, idesc_o, (t | k) != 0);
                }
                ptx::mma_commit(&o_done[x]);
            };
            ptx::mbar_wait(q_full, 0);
            issue_s(0, 0);
            issue_s(1, 0);
            for (int j = 0; j < n_kt[1]; ++j) {
                if (j < n_kt[0]) {
                    issue_pv(0, j);
                    if (j + 1 < n_kt[0]) {
                        ptx::mbar_wait(&o_done[0], j & 1);  // S_a held P_a(j)
                        issue_s(0, j + 1);
                    }
                }
                issue_pv(1, j);
                ptx::mma_commit(&kv_empty[j & 1]);  // tile b is the last reader of stage j%2
                if (j + 1 < n_kt[1]) {
                    ptx::mbar_wait(&o_done[1], j & 1);
                    issue_s(1, j + 1);
                }
            }
        }
    } else {
        // 16 softmax warps: 8 per query tile; the two warps of a TMEM lane quarter split the
        // tile's 128 key columns (and the O columns) and exchange row max / row sum through smem.
        const int sw = warp - 2;
        const int x = sw >> 3;                // query tile
        const int sub = (sw >> 2) & 1;        // key half (and O half) of this warp
        const uint32_t quarter = warp & 3;    // TMEM lane quarter this warp may access
        constexpr int KC = BKV / 2, OC = HD / 2;
        const int xrow = static_cast<int>(quarter) * 32 + lane;
        const int64_t row = q0 + x * BQ + xrow;
        const int64_t abs_row = a.offset + row;
        const uint32_t lane_base = tmem + ((quarter * 32u) << 16);
        const uint32_t s_col = x * 128 + sub * KC;        // fp32 S columns of my key half
        const uint32_t p_col = x * 128 + sub * (KC / 2);  // packed bf16 P columns of my key half
        const uint32_t o_col = 256 + x * 128 + sub * OC;
        float* xch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bar) + 256);  // [2 par][2 x][2 sub][128]
        const uint32_t bar_id = 1 + x * 4 + quarter;      // named barrier of the two partner warps
        const int nt = n_kt[x];
        const int64_t tile_first_abs = a.offset + q0 + x * BQ;
        float m_run = -INFINITY, l = 0.f;
        for (int j = 0; j < nt; ++j) {
            ptx::mbar_wait(&s_full[x], j & 1);
            ptx::tc_fence_after();
            float sv[KC];
#pragma unroll
            for (int c = 0; c < KC / 32; ++c) {
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + s_col + c * 32, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[i]);
            }
            const int64_t key0 = static_cast<int64_t>(j) * BKV + sub * KC;  // first key of my half
            const bool diag = static_cast<int64_t>(j) * BKV + BKV - 1 > tile_first_abs;
            if (diag) {
                // keys [key0, key0 + nvis) are visible to this row; 32-bit compares against
                // compile-time column indices, applied only on the diagonal tile
                const int64_t v = abs_row - key0 + 1;
                const int nvis = v < 0 ? 0 : (v > KC ? KC : static_cast<int>(v));
#pragma unroll
                for (int i = 0; i < KC; ++i) sv[i] = i < nvis ? sv[i] : -INFINITY;
            }
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < KC; ++i) mx = fmaxf(mx, sv[i]);
            float* xb = xch + (j & 1) * 512 + x * 256;
            xb[sub * 128 + xrow] = mx;
            asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
            mx = fmaxf(mx, xb[(sub ^ 1) * 128 + xrow]);  // row max over all 128 keys
            mx *= a.sl2;                                   // scale > 0: max commutes with it
            const bool need = mx > m_run + RESCALE_THRESHOLD;
            if (__any_sync(0xffffffffu, need)) {
                const float m_new = need ? mx : m_run;
                const float alpha = need ? exp2f(m_run - m_new) : 1.0f;
                if (j > 0) {
                    ptx::mbar_wait(&o_done[x], (j - 1) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int c = 0; c < OC / 16; ++c) {
                        uint32_t r[16];
                        ptx::tmem_ld16(lane_base + o_col + c * 16, r);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                        ptx::tmem_st16(lane_base + o_col + c * 16, r);
                    }
                    ptx::tmem_st_wait();
                }
                l *= alpha;
                m_run = m_new;
            }
            const float nbv = (m_run == -INFINITY) ? 0.f : -m_run;
            const float2 sl2v = make_float2(a.sl2, a.sl2), nb2 = make_float2(nbv, nbv);
            float2 lacc = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < KC / 32; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = c * 32 + 2 * i;
                    const int gcol = sub * KC + col;  // the exp2 unit depends on the key column only
                    const float2 xv = ffma2(make_float2(sv[col], sv[col + 1]), sl2v, nb2);
                    float2 pv;
                    if (gcol >= POLY_FROM) {
                        pv = ex2_poly2(xv);
                        if (diag) {  // the FMA-pipe exp2 clamps -inf: zero masked keys
                            pv.x = sv[col] == -INFINITY ? 0.f : pv.x;
                            pv.y = sv[col + 1] == -INFINITY ? 0.f : pv.y;
                        }
                    } else {
                        pv.x = ex2_mufu(xv.x);
                        pv.y = ex2_mufu(xv.y);
                    }
                    lacc = fadd2(lacc, pv);
                    pk[i] = ptx::pack_bf16(pv.x, pv.y);
                }
                ptx::tmem_st16(lane_base + p_col + c * 16, pk);  // P over S, packed bf16
            }
            l += lacc.x + lacc.y;
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&p_full[x]);
        }
        // epilogue: O / (l_0 + l_1) -> bf16, each warp its O half
        float* lb = xch + 1024 + x * 256;
        lb[sub * 128 + xrow] = l;
        asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        const float lo = lb[xrow], hi = lb[128 + xrow];
        const float inv = 1.0f / (lo + hi);  // same order on both partners
        ptx::mbar_wait(&o_done[x], (nt - 1) & 1);
        ptx::tc_fence_after();
        bf16* orow = a.O + row * a.ldo + static_cast<int64_t>(h) * HD + sub * OC;
#pragma unroll
        for (int c = 0; c < OC / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(lane_base + o_col + c * 32, r);
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
}

template <int HD, int POLY_FROM>
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
        cudaFuncSetAttribute(attn_tc_kernel<HD, POLY_FROM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ACfg<HD>::SMEM);
        configured = dev;
    }
    AttnArgs a{sh.q_rows, sh.k_rows, sh.offset, sh.n_heads, sh.n_heads / sh.n_kv_heads, sh.ldo, O,
               (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f};
    dim3 grid(static_cast<unsigned>(sh.n_heads), static_cast<unsigned>((sh.q_rows + 2 * BQ - 1) / (2 * BQ)));
    note_launch();
    attn_tc_kernel<HD, POLY_FROM><<<grid, THREADS, ACfg<HD>::SMEM, s>>>(tq, tk, tv, a);
}

}  // namespace

bool attn_tc_supported(int head_dim) { return head_dim == 64 || head_dim == 128; }

void attn_bf16_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    // KVP_ATTN_POLY = number of key columns (of 128) whose exp2 runs on the FMA pipe
    static const int poly = [] {
        const char* e = getenv("KVP_ATTN_POLY");
        return e ? atoi(e) : 0;
    }();
    if (sh.head_dim != 128 && sh.head_dim != 64) throw std::runtime_error("attn_tc: head_dim must be 64 or 128");
    const bool h128 = sh.head_dim == 128;
    switch (poly) {
        case 48: h128 ? launch<128, 80>(Q, K, V, O, sh, s) : launch<64, 80>(Q, K, V, O, sh, s); break;
        case 64: h128 ? launch<128, 64>(Q, K, V, O, sh, s) : launch<64, 64>(Q, K, V, O, sh, s); break;
        case 32: h128 ? launch<128, 96>(Q, K, V, O, sh, s) : launch<64, 96>(Q, K, V, O, sh, s); break;
        default: h128 ? launch<128, 128>(Q, K, V, O, sh, s) : launch<64, 128>(Q, K, V, O, sh, s); break;
    }
}

}  // namespace kvp
