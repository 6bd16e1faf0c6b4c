// attn_tc.cu -- prefix-causal flash attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Reference: causal_attention (model.hpp:112-158).  One CTA owns a 128-query tile of one head
// (absolute positions offset + q0 ...) and walks the 128-key tiles [0, offset + last query]:
//   warp 0      TMA producer: Q once, then K/V tiles through a 2-stage smem ring;
//   warp 1      MMA issuer (one lane) + TMEM owner:
//                 S_j = Q K_j^T   (SS: A=Q smem, B=K smem, both K-major SW128) -> TMEM S[j%2]
//                 O  += P_j V_j   (TS: A=P_j in TMEM, packed bf16 over S[j%2]; B=V smem MN-major)
//   warps 2..5  softmax, one thread per query row (= TMEM lane): read S_j, mask the diagonal
//               tile against absolute positions, online softmax in the log2 domain, write
//               P_j (bf16) back into TMEM; rescale O in TMEM only when a row max grows by
//               more than 2^8 (exact: l and O always share the same stale max), then the
//               normalised epilogue O / l -> bf16.
// TMEM: S0 [0,128) | S1 [128,256) | O [256, 256+hd) of a 512-column allocation.
// Rows are independent and key tiles are aligned to absolute key 0, so results are bitwise
// independent of how the context is split over ranks (Serial == TSP == KVR).
#include <mutex>
#include <stdexcept>

#include "kernels.cuh"
#include "ptx.cuh"

namespace kvp {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

namespace {

constexpr int BQ = 128;  // queries per CTA
constexpr int BKV = 128; // keys per tile
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: p <= 2^8 between rescales

template <int HD>
struct ACfg {
    static constexpr int HALVES = HD / 64;                    // 64-wide (128 B) TMA boxes
    static constexpr uint32_t Q_BYTES = BQ * HD * 2;
    static constexpr uint32_t KV_BYTES = BKV * HD * 2;
    static constexpr uint32_t SMEM = Q_BYTES + 4 * KV_BYTES + 1024 + 256;
    static constexpr uint32_t O_COL = 256;
};

struct AttnArgs {
    int64_t q_rows, k_rows, offset;
    int n_heads, group;
    int64_t ldo;
    bf16* O;
    float sl2;  // softmax scale * log2(e)
};

template <int HD>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
    using C = ACfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::Q_BYTES;       // 2 stages
    uint8_t* sV = sK + 2 * C::KV_BYTES;  // 2 stages
    uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * C::KV_BYTES);
    uint64_t* q_full = bar;
    uint64_t* k_full = bar + 1;   // [2]
    uint64_t* v_full = bar + 3;   // [2]
    uint64_t* kv_empty = bar + 5; // [2]
    uint64_t* s_full = bar + 7;   // [2]
    uint64_t* p_full = bar + 9;   // [2]
    uint64_t* o_done = bar + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 12);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_qt = static_cast<int>((a.q_rows + BQ - 1) / BQ);
    const int qt = num_qt - 1 - static_cast<int>(blockIdx.x);  // heaviest tiles first
    const int h = blockIdx.y;
    const int g = h / a.group;
    const int64_t q0 = static_cast<int64_t>(qt) * BQ;
    const int64_t last_q = (q0 + BQ - 1 < a.q_rows - 1) ? q0 + BQ - 1 : a.q_rows - 1;
    const int n_kt = static_cast<int>((a.offset + last_q) / BKV) + 1;

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
            ptx::mbar_init(&p_full[s], 4);
        }
        ptx::mbar_init(o_done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(q_full, C::Q_BYTES);
            for (int hv = 0; hv < C::HALVES; ++hv)
                ptx::tma_load_2d(sQ + hv * BQ * 128, &tmQ, q_full, h * HD + hv * 64, static_cast<int32_t>(q0));
            for (int t = 0; t < n_kt; ++t) {
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
            const uint32_t q_addr = ptx::smem_u32(sQ);
            auto issue_s = [&](int t) {
                const int s = t & 1;
                ptx::mbar_wait(&k_full[s], (t >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t k_addr = ptx::smem_u32(sK + s * C::KV_BYTES);
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint32_t off = (k >> 2) * (BQ * 128) + (k & 3) * 32;
                    const uint64_t ad = ptx::smem_desc_sw128(q_addr + off, 16, 1024);
                    const uint64_t bd = ptx::smem_desc_sw128(k_addr + (k >> 2) * (BKV * 128) + (k & 3) * 32, 16, 1024);
                    ptx::mma_bf16_ss(tmem + s * 128, ad, bd, idesc_s, k != 0);
                }
                ptx::mma_commit(&s_full[s]);
            };
            ptx::mbar_wait(q_full, 0);
            issue_s(0);
            for (int j = 0; j < n_kt; ++j) {
                const int b = j & 1;
                if (j + 1 < n_kt) {
                    if (j >= 1) ptx::mbar_wait(o_done, (j - 1) & 1);  // S[(j+1)%2] held P_{j-1}
                    issue_s(j + 1);
                }
                ptx::mbar_wait(&p_full[b], (j >> 1) & 1);
                ptx::mbar_wait(&v_full[b], (j >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t v_addr = ptx::smem_u32(sV + b * C::KV_BYTES);
#pragma unroll
                for (int k = 0; k < BKV / 16; ++k) {
                    // B = V[keys 16k..16k+15][hd]: MN-major SW128, LBO = next 64-wide hd block,
                    // SBO = next 8 keys.
                    const uint64_t bd = ptx::smem_desc_sw128(v_addr + k * 16 * 128, BKV * 128, 1024);
                    ptx::mma_bf16_ts(tmem + C::O_COL, tmem + b * 128 + k * 8, bd, idesc_o, (j | k) != 0);
                }
                ptx::mma_commit(o_done);
                ptx::mma_commit(&kv_empty[b]);
            }
        }
    } else {
        const uint32_t quarter = warp & 3;
        const int64_t row = q0 + quarter * 32 + lane;  // local query row
        const int64_t abs_row = a.offset + row;
        const uint32_t lane_base = tmem + ((quarter * 32u) << 16);
        float m_run = -INFINITY, l = 0.f;
        for (int j = 0; j < n_kt; ++j) {
            const int b = j & 1;
            ptx::mbar_wait(&s_full[b], (j >> 1) & 1);
            ptx::tc_fence_after();
            float x[BKV];
#pragma unroll
            for (int c = 0; c < BKV / 32; ++c) {
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + b * 128 + c * 32, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) x[c * 32 + i] = __uint_as_float(r[i]) * a.sl2;
            }
            const int64_t key0 = static_cast<int64_t>(j) * BKV;
            if (key0 + BKV - 1 > a.offset + q0) {  // tile crosses the causal diagonal
#pragma unroll
                for (int i = 0; i < BKV; ++i)
                    if (key0 + i > abs_row) x[i] = -INFINITY;
            }
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < BKV; ++i) mx = fmaxf(mx, x[i]);
            const bool need = mx > m_run + RESCALE_THRESHOLD;
            if (__any_sync(0xffffffffu, need)) {
                const float m_new = need ? mx : m_run;
                const float alpha = need ? exp2f(m_run - m_new) : 1.0f;
                if (j > 0) {
                    ptx::mbar_wait(o_done, (j - 1) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int c = 0; c < HD / 16; ++c) {
                        uint32_t r[16];
                        ptx::tmem_ld16(lane_base + C::O_COL + c * 16, r);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                        ptx::tmem_st16(lane_base + C::O_COL + c * 16, r);
                    }
                    ptx::tmem_st_wait();
                }
                l *= alpha;
                m_run = m_new;
            }
            const float base = (m_run == -INFINITY) ? 0.f : m_run;
#pragma unroll
            for (int c = 0; c < BKV / 32; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float p0 = exp2f(x[c * 32 + 2 * i] - base);
                    const float p1 = exp2f(x[c * 32 + 2 * i + 1] - base);
                    l += p0 + p1;
                    pk[i] = ptx::pack_bf16(p0, p1);
                }
                ptx::tmem_st16(lane_base + b * 128 + c * 16, pk);  // P_j over S_j, packed bf16
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&p_full[b]);
        }
        // epilogue: O / l -> bf16
        ptx::mbar_wait(o_done, (n_kt - 1) & 1);
        ptx::tc_fence_after();
        const float inv = 1.0f / l;
        bf16* orow = a.O + row * a.ldo + static_cast<int64_t>(h) * HD;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(lane_base + C::O_COL + c * 32, r);
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

template <int HD>
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
        cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<HD>::SMEM);
        configured = dev;
    }
    AttnArgs a{sh.q_rows, sh.k_rows, sh.offset, sh.n_heads, sh.n_heads / sh.n_kv_heads, sh.ldo, O,
               (1.0f / sqrtf(static_cast<float>(HD))) * 1.4426950408889634f};
    dim3 grid(static_cast<unsigned>((sh.q_rows + BQ - 1) / BQ), static_cast<unsigned>(sh.n_heads));
    note_launch();
    attn_tc_kernel<HD><<<grid, THREADS, ACfg<HD>::SMEM, s>>>(tq, tk, tv, a);
}

}  // namespace

bool attn_tc_supported(int head_dim) { return head_dim == 64 || head_dim == 128; }

void attn_bf16_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* O, const AttnShape& sh, cudaStream_t s) {
    if (sh.q_rows <= 0) return;
    if (sh.head_dim == 128)
        launch<128>(Q, K, V, O, sh, s);
    else if (sh.head_dim == 64)
        launch<64>(Q, K, V, O, sh, s);
    else
        throw std::runtime_error("attn_tc: head_dim must be 64 or 128");
}

}  // namespace kvp
