// engine.cpp -- the in-process KV-Runahead prompt phase on B200s (C-ABI in kvp_b200.h).
//
// Mirrors run<T> (engine.hpp:186-318): one host thread per rank (engine.hpp:298-309), typed
// ordered mailboxes between ranks with close / abort semantics (channel.hpp:19-144), the same
// message checks (recv_checked, engine.hpp:166-179), fault injection (send_with_faults,
// engine.hpp:143-164) and exact ExecutionMetrics accounting.  What changes is where the data
// lives and moves:
//  * each rank owns a device (devices[r % n]) and two streams: `comp` runs the layer
//    executor kernels, `comm` moves KV-cache rows;
//  * per layer the rank's K/V live in one contiguous token-major buffer [held x kv]; the QKV
//    GEMM epilogue writes the rank's own rows at their absolute position, the upstream prefix
//    [0, b_i) is copied in by rank i-1 (cudaMemcpyAsync / peer copy on the copy engines), so
//    the reference's vcat (engine.hpp:277-278) disappears;
//  * a mailbox message carries {kind, layer, source, [start,end)} plus the CUDA event that
//    completes when the rows have landed; the receiver validates the header on the host
//    exactly like the reference and makes its compute stream wait on the event.
// Nothing here computes on the CPU: every FLOP is a kernel from kernels.cuh.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/kvp_b200.h"
#include "kernels.cuh"
#include "status.hpp"

namespace kvp {

// ------------------------------------------------------------------ globals
static thread_local std::string t_last_error;
void set_last_error(const std::string& msg) { t_last_error = msg; }

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("KVP_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// rng.hpp:10-37 (host side: only the stream seeds are derived here)
static uint64_t splitmix_next(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static uint64_t mix_seed(uint64_t base, uint64_t a, uint64_t b) {
    uint64_t g = base;
    uint64_t h = splitmix_next(g) ^ (a * 0xd1342543de82ef95ULL);
    return splitmix_next(h) ^ (b * 0xaf251af3b0f025b5ULL);
}

// ------------------------------------------------------------------ device memory
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(dev);
            cudaFree(p);
            cudaSetDevice(cur);
        }
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t n, int device) {
        if (n <= bytes && device == dev) return;
        release();
        dev = device;
        KVP_CUDA(cudaMalloc(&p, n ? n : 16));
        bytes = n;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ------------------------------------------------------------------ model shape
struct Shape {
    int64_t d, h, kvh, L, hd, q, kv, f;
    uint64_t seed;
    int prec;  // KVP_F32 / KVP_BF16
    bool rms;
    size_t es() const { return prec == KVP_BF16 ? 2 : 4; }
};

static Shape make_shape(const kvp_model_config& c) {
    if (c.d_model <= 0 || c.n_heads <= 0 || c.n_kv_heads <= 0 || c.n_layers <= 0)
        throw Error(KVP_ERR_CONFIG, "model dimensions must be positive");
    if (c.d_model % c.n_heads != 0) throw Error(KVP_ERR_CONFIG, "d_model must be divisible by n_heads");
    if (c.n_heads % c.n_kv_heads != 0) throw Error(KVP_ERR_CONFIG, "n_heads must be divisible by n_kv_heads");
    if (c.precision == KVP_F64) throw Error(KVP_ERR_CONFIG, "precision f64 has no GPU path (use f32 or bf16)");
    if (c.precision != KVP_F32 && c.precision != KVP_BF16) throw Error(KVP_ERR_CONFIG, "unknown precision");
    Shape s;
    s.d = c.d_model;
    s.h = c.n_heads;
    s.kvh = c.n_kv_heads;
    s.L = c.n_layers;
    s.hd = s.d / s.h;
    s.q = s.h * s.hd;
    s.kv = s.kvh * s.hd;
    s.f = 2 * s.d;  // ffn_dim (config.hpp:34)
    s.seed = c.seed;
    s.prec = c.precision;
    s.rms = c.rms_norm != 0;
    if (s.prec == KVP_BF16 && (s.d % 8 || s.q % 8 || s.kv % 8))
        throw Error(KVP_ERR_CONFIG, "bf16 mode needs d_model, q_dim and kv_dim multiples of 8 (TMA row alignment)");
    return s;
}

// Weights of one device.  bf16: packed K-major B operands (tcgen05 GEMM):
//   wqkv_t [(q+2kv) x d], wo_t [d x q], w1_t [2d x d], w2_t [d x 2d].
// f32: the reference [in x out] matrices (SIMT parity GEMM).
struct LayerW {
    bf16 *wqkv_t = nullptr, *wo_t = nullptr, *w1_t = nullptr, *w2_t = nullptr;
    float *wq = nullptr, *wk = nullptr, *wv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;
};

struct DeviceWeights {
    int device = 0;
    DevBuf blob;
    DevBuf rope;  // opt-in rotary embedding: inv_freq[head_dim / 2] (kvp_engine_set_rope)
    std::vector<LayerW> layers;

    void init(const Shape& s, int dev) {
        device = dev;
        KVP_CUDA(cudaSetDevice(dev));
        const size_t per_layer = static_cast<size_t>(s.d * (s.q + 2 * s.kv) + s.q * s.d + 2 * s.d * s.f);
        blob.ensure(per_layer * s.L * s.es() + 256, dev);
        layers.resize(static_cast<size_t>(s.L));
        uint8_t* p = blob.as<uint8_t>();
        const double scale = 1.0 / std::sqrt(static_cast<double>(s.d));  // weights.hpp:57
        cudaStream_t st = nullptr;
        for (int64_t l = 0; l < s.L; ++l) {
            LayerW& w = layers[static_cast<size_t>(l)];
            const uint64_t L = static_cast<uint64_t>(l);
            if (s.prec == KVP_BF16) {
                w.wqkv_t = reinterpret_cast<bf16*>(p);
                p += s.d * (s.q + 2 * s.kv) * 2;
                w.wo_t = reinterpret_cast<bf16*>(p);
                p += s.q * s.d * 2;
                w.w1_t = reinterpret_cast<bf16*>(p);
                p += s.d * s.f * 2;
                w.w2_t = reinterpret_cast<bf16*>(p);
                p += s.f * s.d * 2;
                launch_seeded_bf16_t(w.wqkv_t, s.d, s.q, scale, mix_seed(s.seed, L, 1), 0, st);
                launch_seeded_bf16_t(w.wqkv_t, s.d, s.kv, scale, mix_seed(s.seed, L, 2), s.q, st);
                launch_seeded_bf16_t(w.wqkv_t, s.d, s.kv, scale, mix_seed(s.seed, L, 3), s.q + s.kv, st);
                launch_seeded_bf16_t(w.wo_t, s.q, s.d, scale, mix_seed(s.seed, L, 4), 0, st);
                launch_seeded_bf16_t(w.w1_t, s.d, s.f, scale, mix_seed(s.seed, L, 5), 0, st);
                launch_seeded_bf16_t(w.w2_t, s.f, s.d, scale, mix_seed(s.seed, L, 6), 0, st);
            } else {
                auto take = [&](int64_t n) {
                    float* r = reinterpret_cast<float*>(p);
                    p += n * 4;
                    return r;
                };
                w.wq = take(s.d * s.q);
                w.wk = take(s.d * s.kv);
                w.wv = take(s.d * s.kv);
                w.wo = take(s.q * s.d);
                w.w1 = take(s.d * s.f);
                w.w2 = take(s.f * s.d);
                launch_seeded_f32(w.wq, s.d, s.q, scale, mix_seed(s.seed, L, 1), st);
                launch_seeded_f32(w.wk, s.d, s.kv, scale, mix_seed(s.seed, L, 2), st);
                launch_seeded_f32(w.wv, s.d, s.kv, scale, mix_seed(s.seed, L, 3), st);
                launch_seeded_f32(w.wo, s.q, s.d, scale, mix_seed(s.seed, L, 4), st);
                launch_seeded_f32(w.w1, s.d, s.f, scale, mix_seed(s.seed, L, 5), st);
                launch_seeded_f32(w.w2, s.f, s.d, scale, mix_seed(s.seed, L, 6), st);
            }
        }
        KVP_CUDA(cudaGetLastError());
        KVP_CUDA(cudaDeviceSynchronize());
    }

    void load(const Shape& s, int64_t l, const float* const* host) {
        KVP_CUDA(cudaSetDevice(device));
        LayerW& w = layers[static_cast<size_t>(l)];
        const int64_t rows[6] = {s.d, s.d, s.d, s.q, s.d, s.f};
        const int64_t cols[6] = {s.q, s.kv, s.kv, s.d, s.f, s.d};
        if (s.prec == KVP_F32) {
            float* dst[6] = {w.wq, w.wk, w.wv, w.wo, w.w1, w.w2};
            for (int i = 0; i < 6; ++i)
                KVP_CUDA(cudaMemcpy(dst[i], host[i], rows[i] * cols[i] * 4, cudaMemcpyHostToDevice));
            return;
        }
        DevBuf tmp;
        bf16* dst[6] = {w.wqkv_t, w.wqkv_t, w.wqkv_t, w.wo_t, w.w1_t, w.w2_t};
        const int64_t off[6] = {0, s.q, s.q + s.kv, 0, 0, 0};
        for (int i = 0; i < 6; ++i) {
            tmp.ensure(rows[i] * cols[i] * 4, device);
            KVP_CUDA(cudaMemcpy(tmp.p, host[i], rows[i] * cols[i] * 4, cudaMemcpyHostToDevice));
            launch_transpose_to_bf16(tmp.as<float>(), rows[i], cols[i], dst[i], off[i], nullptr);
            KVP_CUDA(cudaDeviceSynchronize());
        }
    }
};

// ------------------------------------------------------------------ fabric
// Message kinds: WorkerMessage::Kind (engine.hpp:41).
enum MsgKind { KV_HANDOFF = 0, GATHER_SHARE = 1 };

struct Msg {
    int kind;
    int64_t layer, source, start, end;
    cudaEvent_t ready;
};

class Mailbox {  // Channel<M> semantics (channel.hpp:19-53)
  public:
    void post(const Msg& m) {
        {
            std::lock_guard<std::mutex> g(mu_);
            if (closed_) throw Error(KVP_ERR_PROTOCOL, "send on closed channel");
            q_.push_back(m);
        }
        cv_.notify_one();
    }
    Msg take() {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return closed_ || !q_.empty(); });
        if (q_.empty()) throw Error(KVP_ERR_PROTOCOL, "channel closed before message arrived");
        Msg m = q_.front();
        q_.pop_front();
        return m;
    }
    void close() {
        {
            std::lock_guard<std::mutex> g(mu_);
            closed_ = true;
        }
        cv_.notify_all();
    }

  private:
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Msg> q_;
    bool closed_ = false;
};

class Gate {  // AbortableBarrier semantics (channel.hpp:58-97)
  public:
    explicit Gate(int64_t parties) : parties_(parties) {}
    void arrive_and_wait() {
        std::unique_lock<std::mutex> g(mu_);
        if (aborted_) throw Error(KVP_ERR_PROTOCOL, "barrier aborted");
        if (++arrived_ == parties_) {
            arrived_ = 0;
            ++gen_;
            g.unlock();
            cv_.notify_all();
            return;
        }
        const int64_t mine = gen_;
        cv_.wait(g, [&] { return gen_ != mine || aborted_; });
        if (gen_ == mine) throw Error(KVP_ERR_PROTOCOL, "barrier aborted");
    }
    void abort() {
        {
            std::lock_guard<std::mutex> g(mu_);
            aborted_ = true;
        }
        cv_.notify_all();
    }
    int64_t generations() {
        std::lock_guard<std::mutex> g(mu_);
        return gen_;
    }

  private:
    std::mutex mu_;
    std::condition_variable cv_;
    int64_t parties_, arrived_ = 0, gen_ = 0;
    bool aborted_ = false;
};

class Fabric {  // Fabric<M> (channel.hpp:103-144)
  public:
    explicit Fabric(int64_t p) : p_(p), gate_(p) {
        boxes_.reserve(static_cast<size_t>(p * p));
        for (int64_t i = 0; i < p * p; ++i) boxes_.push_back(std::make_unique<Mailbox>());
    }
    Mailbox& link(int64_t from, int64_t to) { return *boxes_[static_cast<size_t>(from * p_ + to)]; }
    Gate& gate() { return gate_; }
    void close_from(int64_t r) {
        for (int64_t t = 0; t < p_; ++t) link(r, t).close();
    }
    void fail(std::exception_ptr e) {
        {
            std::lock_guard<std::mutex> g(mu_);
            if (!first_) first_ = e;
        }
        for (auto& b : boxes_) b->close();
        gate_.abort();
    }
    void rethrow() {
        std::exception_ptr e;
        {
            std::lock_guard<std::mutex> g(mu_);
            e = first_;
        }
        if (e) std::rethrow_exception(e);
    }

  private:
    int64_t p_;
    std::vector<std::unique_ptr<Mailbox>> boxes_;
    Gate gate_;
    std::mutex mu_;
    std::exception_ptr first_;
};

// ------------------------------------------------------------------ rank state
struct RankCtx {
    int device = -1;
    cudaStream_t comp = nullptr, comm = nullptr;
    DevBuf h, h1, x, q, a, mid, kv, ssq;
    int64_t held = 0;  // rows per layer K (and V) buffer
    std::vector<void*> ext_kv;  // caller-owned per-layer K/V buffers (multi-process mode)
    std::vector<void*> mirror_bufs;  // multi-process fused handoff: [n_mirror][L][K,V] peer buffers
    int n_mirror = 0;
    bool decode = false;        // decode step: HBM-bound GEMV + split-key attention kernels
    int64_t pos0 = 0;           // absolute position of this rank's first row (RoPE)
    const float* rope_inv = nullptr;  // RoPE inv_freq table on this rank's device (nullptr: off)
    int rope_hd = 0;
    DevBuf scratch;             // decode attention partials
    std::vector<cudaEvent_t> ev_send, ev_ready, t_start, t_qkv, t_attn, t_end;
    cudaEvent_t ev_begin = nullptr, ev_done = nullptr;
    // profiling: (class, flops, bytes, start event, end event) per launch
    struct Mark {
        int cls;
        double flops, bytes;
        cudaEvent_t a, b;
    };
    bool profiling = false;
    // CUDA graph of a single-rank prefill (all layers), keyed by shape + buffer identity
    cudaGraphExec_t graph = nullptr;
    uint64_t graph_key = 0;
    int64_t graph_launches = 0;
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    cudaEvent_t pooled() {
        if (pool_used == pool.size()) {
            cudaEvent_t e;
            KVP_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[pool_used++];
    }
    template <typename F>
    void timed(int cls, double flops, double bytes, F&& launch) {
        if (!profiling) {
            launch();
            return;
        }
        Mark m{cls, flops, bytes, pooled(), pooled()};
        KVP_CUDA(cudaEventRecord(m.a, comp));
        launch();
        KVP_CUDA(cudaEventRecord(m.b, comp));
        marks.push_back(m);
    }

    void setup(int dev, int64_t L) {
        if (device == dev && static_cast<int64_t>(t_start.size()) == L) return;
        teardown();
        device = dev;
        KVP_CUDA(cudaSetDevice(dev));
        KVP_CUDA(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
        KVP_CUDA(cudaStreamCreateWithFlags(&comm, cudaStreamNonBlocking));
        auto mk = [&](std::vector<cudaEvent_t>& v, unsigned flags) {
            v.resize(static_cast<size_t>(L));
            for (auto& e : v) KVP_CUDA(cudaEventCreateWithFlags(&e, flags));
        };
        mk(ev_send, cudaEventDisableTiming);
        mk(ev_ready, cudaEventDisableTiming);
        mk(t_start, cudaEventDefault);
        mk(t_qkv, cudaEventDefault);
        mk(t_attn, cudaEventDefault);
        mk(t_end, cudaEventDefault);
        KVP_CUDA(cudaEventCreate(&ev_begin));
        KVP_CUDA(cudaEventCreate(&ev_done));
    }
    void teardown() {
        if (device < 0) return;
        cudaSetDevice(device);
        for (auto* v : {&ev_send, &ev_ready, &t_start, &t_qkv, &t_attn, &t_end}) {
            for (auto e : *v) cudaEventDestroy(e);
            v->clear();
        }
        if (graph) cudaGraphExecDestroy(graph);
        graph = nullptr;
        graph_key = 0;
        for (auto ev : pool) cudaEventDestroy(ev);
        pool.clear();
        pool_used = 0;
        marks.clear();
        if (ev_begin) cudaEventDestroy(ev_begin);
        if (ev_done) cudaEventDestroy(ev_done);
        if (comp) cudaStreamDestroy(comp);
        if (comm) cudaStreamDestroy(comm);
        ev_begin = ev_done = nullptr;
        comp = comm = nullptr;
        device = -1;
    }
    ~RankCtx() {
        h.release(); h1.release(); x.release(); q.release(); a.release(); mid.release(); kv.release();
        ssq.release();
        teardown();
    }
    void alloc(const Shape& s, int64_t rows, int64_t held_rows, bool own_kv = true) {
        const size_t es = s.es();
        if (own_kv) ext_kv.clear();
        h.ensure(rows * s.d * 4, device);
        h1.ensure(rows * s.d * 4, device);
        x.ensure(rows * s.d * es, device);
        q.ensure(rows * s.q * es, device);
        a.ensure(rows * s.q * es, device);
        mid.ensure(rows * s.f * es, device);
        ssq.ensure(rows * ssq_parts_for(s.d) * 4, device);
        if (own_kv) kv.ensure(static_cast<size_t>(s.L) * 2 * held_rows * s.kv * es, device);
        held = held_rows;
    }
    // K or V of layer l: [held x kv], element size es.
    void* kv_ptr(const Shape& s, int64_t l, int which) const {
        if (!ext_kv.empty()) return ext_kv[static_cast<size_t>(2 * l + which)];
        return kv.as<uint8_t>() + ((2 * l + which) * held * s.kv) * s.es();
    }
};

// ------------------------------------------------------------------ layer executor
enum KernelClass { K_NORM = 0, K_GEMM_QKV, K_ATTN, K_GEMM_O, K_GEMM_FFN1, K_GEMM_FFN2, K_NUM };
static const char* kKernelNames[K_NUM] = {"norm", "gemm_qkv", "attention", "gemm_o", "gemm_ffn1", "gemm_ffn2"};

// layer_qkv (model.hpp:189-192): norm -> fused QKV GEMM; K/V rows land at `kdst`/`vdst`.
// Where the QKV epilogue also stores this rank's K/V rows (fused KV handoff): pointers at
// the same rows of other ranks' layer buffers.
struct KvMirrors {
    void* k[KVP_MAX_MIRRORS];
    void* v[KVP_MAX_MIRRORS];
    int n = 0;
};

static void exec_qkv(const Shape& s, const LayerW& w, RankCtx& R, int64_t c, void* kdst, void* vdst,
                     bool prep = true, const KvMirrors* mir = nullptr) {
    if (mir && mir->n > 0 && (s.prec != KVP_BF16 || R.decode))
        throw Error(KVP_ERR_CONFIG, "the fused KV handoff needs the bf16 tcgen05 projection");
    const double gf = 2.0 * c * s.d * (s.q + 2 * s.kv);
    if (s.prec == KVP_BF16) {
        // x = bf16(h) and its per-128-column sums of squares; from layer 1 on the previous
        // layer's FFN2 epilogue already produced both (fused RMSNorm).
        if (prep)
            R.timed(K_NORM, 0, c * s.d * 6.0, [&] {
                launch_prep_bf16_ssq(R.h.as<float>(), R.x.as<bf16>(), R.ssq.as<float>(), c, s.d, R.comp);
            });
        GemmEpilogue ep;
        ep.kind = EPI_QKV;
        ep.out0 = R.q.as<bf16>();
        ep.ld0 = s.q;
        ep.n0 = s.q;
        ep.out1 = static_cast<bf16*>(kdst);
        ep.ld1 = s.kv;
        ep.n1 = s.kv;
        ep.out2 = static_cast<bf16*>(vdst);
        ep.ld2 = s.kv;
        if (s.rms) {
            ep.ssq_in = R.ssq.as<float>();
            ep.ssq_parts = ssq_parts_for(s.d);
            ep.norm_cols = s.d;
            if (R.decode) {  // the decode GEMV computes the row scale from the f32 rows
                ep.ssq_in = nullptr;
                ep.norm_src = R.h.as<float>();
                ep.ld_norm = s.d;
            }
        }
        if (R.rope_inv) {
            ep.rope_hd = static_cast<int>(s.hd);
            ep.rope_pos0 = R.pos0;
            ep.rope_inv_freq = R.rope_inv;
        }
        if (mir) {
            ep.n_mirror = mir->n;
            for (int m = 0; m < mir->n; ++m) {
                ep.mirror_k[m] = static_cast<bf16*>(mir->k[m]);
                ep.mirror_v[m] = static_cast<bf16*>(mir->v[m]);
            }
        }
        R.timed(K_GEMM_QKV, gf, 0, [&] {
            if (R.decode)
                gemv_bf16(R.x.as<bf16>(), c, s.d, w.wqkv_t, s.q + 2 * s.kv, ep, R.comp);
            else
                gemm_bf16_tc(R.x.as<bf16>(), c, s.d, w.wqkv_t, s.q + 2 * s.kv, ep, R.comp);
        });
    } else {
        const float* x = R.h.as<float>();
        if (s.rms) {
            R.timed(K_NORM, 0, c * s.d * 8.0, [&] { launch_norm_f32(R.h.as<float>(), R.x.as<float>(), c, s.d, R.comp); });
            x = R.x.as<float>();
        }
        R.timed(K_GEMM_QKV, gf, 0, [&] {
            gemm_f32_simt(x, c, s.d, s.d, w.wq, s.q, R.q.as<float>(), s.q, SEPI_STORE, nullptr, 0, R.comp);
            gemm_f32_simt(x, c, s.d, s.d, w.wk, s.kv, static_cast<float*>(kdst), s.kv, SEPI_STORE, nullptr, 0, R.comp);
            gemm_f32_simt(x, c, s.d, s.d, w.wv, s.kv, static_cast<float*>(vdst), s.kv, SEPI_STORE, nullptr, 0, R.comp);
        });
    }
}

// layer_finish (model.hpp:164-175): attention over keys [0, k_rows) with offset, O-proj +
// residual, norm, FFN (ReLU) + residual.  Result overwrites R.h.
static void exec_finish(const Shape& s, const LayerW& w, RankCtx& R, int64_t c, const void* K, const void* V,
                        int64_t k_rows, int64_t offset) {
    AttnShape sh;
    sh.q_rows = c;
    sh.k_rows = k_rows;
    sh.offset = offset;
    sh.n_heads = static_cast<int>(s.h);
    sh.n_kv_heads = static_cast<int>(s.kvh);
    sh.head_dim = static_cast<int>(s.hd);
    sh.ldq = s.q;
    sh.ldkv = s.kv;
    sh.ldo = s.q;
    // algorithmic attention work: 4 * head_dim * heads per causal-visible (query, key) pair
    const double pairs = static_cast<double>(c) * static_cast<double>(offset) + 0.5 * c * (c + 1.0);
    const double af = 4.0 * s.hd * s.h * pairs;
    if (s.prec == KVP_BF16) {
        R.timed(K_ATTN, af, 0, [&] {
            if (R.decode && (sh.head_dim == 64 || sh.head_dim == 128)) {
                R.scratch.ensure(static_cast<size_t>(attn_decode_scratch_floats(sh)) * 4, R.device);
                attn_decode_bf16(R.q.as<bf16>(), static_cast<const bf16*>(K), static_cast<const bf16*>(V), R.a.as<bf16>(),
                                 sh, R.scratch.as<float>(), R.comp);
            } else if (attn_bf16_supported(sh.head_dim))
                attn_bf16(R.q.as<bf16>(), static_cast<const bf16*>(K), static_cast<const bf16*>(V), R.a.as<bf16>(), sh,
                          R.comp);
            else
                attn_simt_bf16(R.q.as<bf16>(), static_cast<const bf16*>(K), static_cast<const bf16*>(V), R.a.as<bf16>(),
                               sh, R.comp);
        });
        GemmEpilogue e1;
        e1.kind = EPI_RESID;
        e1.outf = R.h1.as<float>();
        e1.ldf = s.d;
        e1.resid = R.h.as<float>();
        e1.ldr = s.d;
        e1.outb = R.x.as<bf16>();  // bf16(h1): the FFN1 A operand
        e1.ldb = s.d;
        if (s.rms && !R.decode) {
            e1.ssq_out = R.ssq.as<float>();
            e1.ssq_parts = ssq_parts_for(s.d);
        }
        // decode rows (R.decode) take the HBM-bound GEMV with the same epilogues
        auto mm = [&](const bf16* A, int64_t K_, const bf16* B, int64_t N_, const GemmEpilogue& ep) {
            if (R.decode)
                gemv_bf16(A, c, K_, B, N_, ep, R.comp);
            else
                gemm_bf16_tc(A, c, K_, B, N_, ep, R.comp);
        };
        R.timed(K_GEMM_O, 2.0 * c * s.q * s.d, 0, [&] { mm(R.a.as<bf16>(), s.q, w.wo_t, s.d, e1); });
        GemmEpilogue e2;
        e2.kind = EPI_RELU;
        e2.out0 = R.mid.as<bf16>();
        e2.ld0 = s.f;
        if (s.rms) {  // relu(norm(h1).W1) = relu(diag(1/rms).(bf16(h1).W1))
            e2.ssq_in = R.ssq.as<float>();
            e2.ssq_parts = ssq_parts_for(s.d);
            e2.norm_cols = s.d;
            if (R.decode) {
                e2.ssq_in = nullptr;
                e2.norm_src = R.h1.as<float>();
                e2.ld_norm = s.d;
            }
        }
        R.timed(K_GEMM_FFN1, 2.0 * c * s.d * s.f, 0, [&] { mm(R.x.as<bf16>(), s.d, w.w1_t, s.f, e2); });
        GemmEpilogue e3;
        e3.kind = EPI_RESID;
        e3.outf = R.h.as<float>();
        e3.ldf = s.d;
        e3.resid = R.h1.as<float>();
        e3.ldr = s.d;
        e3.outb = R.x.as<bf16>();  // bf16(h): the next layer's QKV A operand
        e3.ldb = s.d;
        if (s.rms && !R.decode) {
            e3.ssq_out = R.ssq.as<float>();
            e3.ssq_parts = ssq_parts_for(s.d);
        }
        R.timed(K_GEMM_FFN2, 2.0 * c * s.f * s.d, 0, [&] { mm(R.mid.as<bf16>(), s.f, w.w2_t, s.d, e3); });
    } else {
        R.timed(K_ATTN, af, 0, [&] {
            attn_simt_f32(R.q.as<float>(), static_cast<const float*>(K), static_cast<const float*>(V), R.a.as<float>(), sh,
                          R.comp);
        });
        R.timed(K_GEMM_O, 2.0 * c * s.q * s.d, 0, [&] {
            gemm_f32_simt(R.a.as<float>(), c, s.q, s.q, w.wo, s.d, R.h1.as<float>(), s.d, SEPI_RESID, R.h.as<float>(), s.d,
                          R.comp);
        });
        const float* f = R.h1.as<float>();
        if (s.rms) {
            R.timed(K_NORM, 0, c * s.d * 8.0, [&] { launch_norm_f32(R.h1.as<float>(), R.x.as<float>(), c, s.d, R.comp); });
            f = R.x.as<float>();
        }
        R.timed(K_GEMM_FFN1, 2.0 * c * s.d * s.f, 0, [&] {
            gemm_f32_simt(f, c, s.d, s.d, w.w1, s.f, R.mid.as<float>(), s.f, SEPI_RELU, nullptr, 0, R.comp);
        });
        R.timed(K_GEMM_FFN2, 2.0 * c * s.f * s.d, 0, [&] {
            gemm_f32_simt(R.mid.as<float>(), c, s.f, s.f, w.w2, s.d, R.h.as<float>(), s.d, SEPI_RESID, R.h1.as<float>(),
                          s.d, R.comp);
        });
    }
}

// ------------------------------------------------------------------ engine
struct RunMetrics {
    std::vector<int64_t> dots, sent, recv, waits;
};

}  // namespace kvp

struct kvp_engine {
    kvp::Shape s;
    std::vector<int> devices;
    std::vector<std::unique_ptr<kvp::DeviceWeights>> weights;  // per device slot
    std::vector<std::unique_ptr<kvp::RankCtx>> ranks;
    std::unique_ptr<kvp::RankCtx> util;
    std::mutex mu;
    int64_t last_p = 0;
    float last_ttft = 0.f;
    int64_t last_launches = 0;
    bool profiling = false;
    // multi-process rank session
    bool in_session = false;
    int64_t sess_rows = 0, sess_start = 0, sess_launch0 = 0;
    bool peer_ok = true;  // every device pair of this engine can address each other's memory
    // opt-in rotary embedding (extension; 0 = off, the reference model): base theta and a
    // generation counter that invalidates captured prefill graphs when it changes
    double rope_theta = 0.0;
    uint64_t rope_gen = 0;
    const float* rope_table(int slot) const {
        return rope_theta > 0 ? weights[static_cast<size_t>(slot)]->rope.as<float>() : nullptr;
    }
};

namespace kvp {

static const LayerW& layer_of(kvp_engine* e, int slot, int64_t l) {
    if (l < 0 || l >= e->s.L) throw Error(KVP_ERR_DIMENSION, "layer index " + std::to_string(l) + " out of range");
    return e->weights[static_cast<size_t>(slot)]->layers[static_cast<size_t>(l)];
}

static void run_engine(kvp_engine* e, int32_t strategy, const float* ctx, int64_t C, const int64_t* b, int64_t p,
                       const kvp_fault* fault_in, float* hid, float* ft, kvp_metrics* met) {
    const Shape& s = e->s;
    if (p < 1 || b == nullptr || b[0] != 0 || b[p] != C)
        throw Error(KVP_ERR_PARTITION, "boundaries must run from 0 to the context length");
    for (int64_t i = 0; i < p; ++i)
        if (b[i] >= b[i + 1]) throw Error(KVP_ERR_PARTITION, "partition sizes must be at least 1");
    if (ctx == nullptr) throw Error(KVP_ERR_INPUT, "null context");
    if (strategy != KVP_SERIAL && strategy != KVP_TSP && strategy != KVP_KVR)
        throw Error(KVP_ERR_CONFIG, "unknown strategy");
    if (strategy == KVP_SERIAL && p != 1) throw Error(KVP_ERR_INPUT, "serial strategy requires p == 1");
    if (p > KVP_MAX_RANKS) throw Error(KVP_ERR_INPUT, "too many ranks");
    const kvp_fault fault = fault_in ? *fault_in : kvp_fault{KVP_FAULT_NONE, 0, 0};

    while (static_cast<int64_t>(e->ranks.size()) < p) e->ranks.push_back(std::make_unique<RankCtx>());
    const int nd = static_cast<int>(e->devices.size());
    for (int64_t r = 0; r < p; ++r) {
        RankCtx& R = *e->ranks[static_cast<size_t>(r)];
        R.setup(e->devices[static_cast<size_t>(r % nd)], s.L);
        const int64_t c = b[r + 1] - b[r];
        const int64_t held = (strategy == KVP_KVR) ? b[r + 1] : C;
        R.alloc(s, c, held);
        R.profiling = e->profiling;
        R.pos0 = b[r];
        R.rope_inv = e->rope_table(static_cast<int>(r % nd));
        R.rope_hd = R.rope_inv ? static_cast<int>(s.hd) : 0;
        // a rank session (kvp_rank_begin / KVCache.decode) may have left rank 0 in decode
        // mode or holding peer mirrors: the prefill engine owns neither
        R.decode = false;
        R.n_mirror = 0;
        R.mirror_bufs.clear();
        R.marks.clear();
        R.pool_used = 0;
    }
    e->in_session = false;

    // Fused KV handoff (bf16): the QKV epilogue stores the rank's K/V rows straight into the
    // receiving ranks' layer buffers (peer memory over NVLink between GPUs), so the transfer
    // overlaps the projection tile by tile.  KVR: own rows -> rank r+1 from the epilogue, the
    // upstream prefix [0, b_r) forwarded by the copy engine as soon as it has landed; TSP:
    // own rows -> every peer (the all-gather inside the GEMM).  KVP_HANDOFF=copy restores the
    // copy-engine path (cumulative [0, b_{r+1}) copy after the projection).
    static const bool handoff_copy = [] {
        const char* h = getenv("KVP_HANDOFF");
        return h && std::strcmp(h, "copy") == 0;
    }();
    const bool fused = !handoff_copy && s.prec == KVP_BF16 && e->peer_ok && p > 1 &&
                       (strategy == KVP_KVR || (strategy == KVP_TSP && p - 1 <= KVP_MAX_MIRRORS));

    RunMetrics m;
    m.dots.assign(static_cast<size_t>(p), 0);
    m.sent.assign(static_cast<size_t>(p), 0);
    m.recv.assign(static_cast<size_t>(p), 0);
    m.waits.assign(static_cast<size_t>(p), 0);
    Fabric fab(p);
    const int64_t launches0 = launch_count();
    const auto wall0 = std::chrono::steady_clock::now();

    // send_with_faults (engine.hpp:143-164)
    auto send = [&](Mailbox& box, Msg msg, int64_t rank, int64_t& counter) {
        const int64_t pairs = msg.end - msg.start;
        if (fault.kind != KVP_FAULT_NONE && fault.rank == rank && fault.layer == msg.layer) {
            if (fault.kind == KVP_FAULT_DROP_MESSAGE) return;
            if (fault.kind == KVP_FAULT_CORRUPT_LAYER_TAG) msg.layer += 1;
            if (fault.kind == KVP_FAULT_DUPLICATE_MESSAGE) {
                box.post(msg);
                counter += pairs;
            }
        }
        box.post(msg);
        counter += pairs;
    };
    // recv_checked (engine.hpp:166-179)
    auto recv = [&](Mailbox& box, int kind, int64_t layer, int64_t& waits) {
        waits += 1;
        Msg msg = box.take();
        if (msg.kind != kind) throw Error(KVP_ERR_PROTOCOL, "unexpected message kind");
        if (msg.layer != layer)
            throw Error(KVP_ERR_PROTOCOL, "expected message for layer " + std::to_string(layer) + ", got layer " +
                                              std::to_string(msg.layer) + " (duplicate, dropped, or corrupt handoff)");
        if (msg.start < 0 || msg.start >= msg.end)
            throw Error(KVP_ERR_CACHE, "segment positions must satisfy 0 <= start < end");
        return msg;
    };

    auto worker = [&](int64_t r) {
        RankCtx& R = *e->ranks[static_cast<size_t>(r)];
        const int slot = static_cast<int>(r % nd);
        KVP_CUDA(cudaSetDevice(R.device));
        const int64_t start = b[r], stop = b[r + 1], c = stop - start;
        const size_t es = s.es();
        const size_t row_kv = static_cast<size_t>(s.kv) * es;
        KVP_CUDA(cudaEventRecord(R.ev_begin, R.comp));
        KVP_CUDA(cudaMemcpyAsync(R.h.p, ctx + start * s.d, c * s.d * 4, cudaMemcpyDefault, R.comp));
        // Single-rank prefill (serial / KVR p=1): no cross-rank protocol inside the layer loop,
        // so the 5L kernels + timing events are captured once into a CUDA graph and replayed
        // (removes per-launch host and GPU front-end gaps).  KVP_GRAPH=0 disables.
        static const bool use_graph = [] {
            const char* g = getenv("KVP_GRAPH");
            return !(g && g[0] == '0');
        }();
        if (p == 1 && strategy != KVP_TSP && use_graph && !R.profiling) {
            const uint64_t key = (static_cast<uint64_t>(c) << 20) ^ (reinterpret_cast<uintptr_t>(R.h.p) >> 4) ^
                                 (reinterpret_cast<uintptr_t>(R.kv.p) << 7) ^ (reinterpret_cast<uintptr_t>(R.x.p) << 13) ^
                                 static_cast<uint64_t>(strategy) ^ (e->rope_gen << 44);
            if (!R.graph || R.graph_key != key) {
                if (R.graph) cudaGraphExecDestroy(R.graph);
                R.graph = nullptr;
                const int64_t l0 = launch_count();
                cudaGraph_t g = nullptr;
                KVP_CUDA(cudaStreamBeginCapture(R.comp, cudaStreamCaptureModeThreadLocal));
                try {
                    for (int64_t l = 0; l < s.L; ++l) {
                        const LayerW& w = e->weights[static_cast<size_t>(slot)]->layers[static_cast<size_t>(l)];
                        uint8_t* K = static_cast<uint8_t*>(R.kv_ptr(s, l, 0));
                        uint8_t* V = static_cast<uint8_t*>(R.kv_ptr(s, l, 1));
                        KVP_CUDA(cudaEventRecord(R.t_start[l], R.comp));
                        exec_qkv(s, w, R, c, K, V, l == 0);
                        KVP_CUDA(cudaEventRecord(R.t_qkv[l], R.comp));
                        KVP_CUDA(cudaEventRecord(R.t_attn[l], R.comp));
                        exec_finish(s, w, R, c, K, V, c, 0);
                        KVP_CUDA(cudaEventRecord(R.t_end[l], R.comp));
                    }
                } catch (...) {
                    // never leave the stream in capture mode: later runs would all fail
                    cudaGraph_t dead = nullptr;
                    cudaStreamEndCapture(R.comp, &dead);
                    if (dead) cudaGraphDestroy(dead);
                    cudaGetLastError();
                    throw;
                }
                KVP_CUDA(cudaStreamEndCapture(R.comp, &g));
                KVP_CUDA(cudaGraphInstantiate(&R.graph, g, 0));
                cudaGraphDestroy(g);
                R.graph_key = key;
                R.graph_launches = launch_count() - l0;
            } else {
                for (int64_t i = 0; i < R.graph_launches; ++i) note_launch();
            }
            KVP_CUDA(cudaGraphLaunch(R.graph, R.comp));
            for (int64_t l = 0; l < s.L; ++l) m.dots[0] += c * c;
            if (ft) KVP_CUDA(cudaMemcpyAsync(ft, R.h.as<float>() + (c - 1) * s.d, s.d * 4, cudaMemcpyDefault, R.comp));
            KVP_CUDA(cudaEventRecord(R.ev_done, R.comp));
            if (hid) KVP_CUDA(cudaMemcpyAsync(hid, R.h.p, c * s.d * 4, cudaMemcpyDefault, R.comp));
            fab.close_from(r);
            return;
        }
        for (int64_t l = 0; l < s.L; ++l) {
            const LayerW& w = e->weights[static_cast<size_t>(slot)]->layers[static_cast<size_t>(l)];
            uint8_t* K = static_cast<uint8_t*>(R.kv_ptr(s, l, 0));
            uint8_t* V = static_cast<uint8_t*>(R.kv_ptr(s, l, 1));
            KVP_CUDA(cudaEventRecord(R.t_start[l], R.comp));
            KvMirrors mir;
            if (fused) {
                for (int64_t peer = 0; peer < p; ++peer) {
                    if (peer == r || (strategy == KVP_KVR && peer != r + 1)) continue;
                    RankCtx& P = *e->ranks[static_cast<size_t>(peer)];
                    mir.k[mir.n] = static_cast<uint8_t*>(P.kv_ptr(s, l, 0)) + start * row_kv;
                    mir.v[mir.n] = static_cast<uint8_t*>(P.kv_ptr(s, l, 1)) + start * row_kv;
                    ++mir.n;
                }
            }
            exec_qkv(s, w, R, c, K + start * row_kv, V + start * row_kv, l == 0, &mir);
            KVP_CUDA(cudaGetLastError());
            KVP_CUDA(cudaEventRecord(R.t_qkv[l], R.comp));
            int64_t k_rows;
            if (strategy == KVP_TSP && fused) {
                // the all-gather rode the QKV epilogue: t_qkv[l] marks this rank's rows in
                // every peer's layer buffer
                for (int64_t peer = 0; peer < p; ++peer) {
                    if (peer == r) continue;
                    send(fab.link(r, peer), Msg{GATHER_SHARE, l, r, start, stop, R.t_qkv[l]}, r,
                         m.sent[static_cast<size_t>(r)]);
                }
                std::vector<std::pair<int64_t, int64_t>> segs{{start, stop}};
                for (int64_t peer = 0; peer < p; ++peer) {
                    if (peer == r) continue;
                    Msg in = recv(fab.link(peer, r), GATHER_SHARE, l, m.waits[static_cast<size_t>(r)]);
                    m.recv[static_cast<size_t>(r)] += in.end - in.start;
                    KVP_CUDA(cudaStreamWaitEvent(R.comp, in.ready, 0));
                    segs.emplace_back(in.start, in.end);
                }
                std::sort(segs.begin(), segs.end());
                int64_t next = 0;  // validate_cache_coverage (kv_cache.hpp:41-55)
                for (auto& sg : segs) {
                    if (sg.first != next)
                        throw Error(KVP_ERR_CACHE, "cache gap: expected segment at position " + std::to_string(next));
                    next = sg.second;
                }
                if (next != C) throw Error(KVP_ERR_CACHE, "cache does not cover the context");
                fab.gate().arrive_and_wait();
                m.waits[static_cast<size_t>(r)] += 1;
                k_rows = C;
            } else if (strategy == KVP_KVR && fused) {
                Msg in{};
                if (r > 0) {
                    in = recv(fab.link(r - 1, r), KV_HANDOFF, l, m.waits[static_cast<size_t>(r)]);
                    if (in.start != 0 || in.end != start)
                        throw Error(KVP_ERR_CACHE, "handoff covers [" + std::to_string(in.start) + ", " +
                                                       std::to_string(in.end) + "), expected prefix [0, " +
                                                       std::to_string(start) + ")");
                    m.recv[static_cast<size_t>(r)] += in.end - in.start;
                    KVP_CUDA(cudaStreamWaitEvent(R.comp, in.ready, 0));
                }
                if (r + 1 < p) {
                    // rows [start, stop) went to rank r+1 from the epilogue; forward the
                    // upstream prefix [0, start) once it has landed here, on the copy engine
                    // (independent of this rank's projection), then announce [0, stop)
                    RankCtx& N = *e->ranks[static_cast<size_t>(r + 1)];
                    if (r > 0) {
                        KVP_CUDA(cudaStreamWaitEvent(R.comm, in.ready, 0));
                        KVP_CUDA(cudaMemcpyAsync(N.kv_ptr(s, l, 0), K, start * row_kv, cudaMemcpyDefault, R.comm));
                        KVP_CUDA(cudaMemcpyAsync(N.kv_ptr(s, l, 1), V, start * row_kv, cudaMemcpyDefault, R.comm));
                    }
                    KVP_CUDA(cudaStreamWaitEvent(R.comm, R.t_qkv[l], 0));
                    KVP_CUDA(cudaEventRecord(R.ev_send[l], R.comm));
                    send(fab.link(r, r + 1), Msg{KV_HANDOFF, l, r, 0, stop, R.ev_send[l]}, r,
                         m.sent[static_cast<size_t>(r)]);
                }
                k_rows = stop;
            } else if (strategy == KVP_TSP) {
                // all-gather: push own rows [start, stop) into every peer's layer buffer
                KVP_CUDA(cudaStreamWaitEvent(R.comm, R.t_qkv[l], 0));
                for (int64_t peer = 0; peer < p; ++peer) {
                    if (peer == r) continue;
                    RankCtx& P = *e->ranks[static_cast<size_t>(peer)];
                    uint8_t* pk = static_cast<uint8_t*>(P.kv_ptr(s, l, 0));
                    uint8_t* pv = static_cast<uint8_t*>(P.kv_ptr(s, l, 1));
                    KVP_CUDA(cudaMemcpyAsync(pk + start * row_kv, K + start * row_kv, c * row_kv, cudaMemcpyDefault, R.comm));
                    KVP_CUDA(cudaMemcpyAsync(pv + start * row_kv, V + start * row_kv, c * row_kv, cudaMemcpyDefault, R.comm));
                }
                KVP_CUDA(cudaEventRecord(R.ev_send[l], R.comm));
                for (int64_t peer = 0; peer < p; ++peer) {
                    if (peer == r) continue;
                    send(fab.link(r, peer), Msg{GATHER_SHARE, l, r, start, stop, R.ev_send[l]}, r,
                         m.sent[static_cast<size_t>(r)]);
                }
                std::vector<std::pair<int64_t, int64_t>> segs{{start, stop}};
                for (int64_t peer = 0; peer < p; ++peer) {
                    if (peer == r) continue;
                    Msg in = recv(fab.link(peer, r), GATHER_SHARE, l, m.waits[static_cast<size_t>(r)]);
                    m.recv[static_cast<size_t>(r)] += in.end - in.start;
                    KVP_CUDA(cudaStreamWaitEvent(R.comp, in.ready, 0));
                    segs.emplace_back(in.start, in.end);
                }
                std::sort(segs.begin(), segs.end());
                int64_t next = 0;  // validate_cache_coverage (kv_cache.hpp:41-55)
                for (auto& sg : segs) {
                    if (sg.first != next)
                        throw Error(KVP_ERR_CACHE, "cache gap: expected segment at position " + std::to_string(next));
                    next = sg.second;
                }
                if (next != C) throw Error(KVP_ERR_CACHE, "cache does not cover the context");
                fab.gate().arrive_and_wait();
                m.waits[static_cast<size_t>(r)] += 1;
                k_rows = C;
            } else if (strategy == KVP_KVR) {
                if (r > 0) {
                    Msg in = recv(fab.link(r - 1, r), KV_HANDOFF, l, m.waits[static_cast<size_t>(r)]);
                    if (in.start != 0 || in.end != start)
                        throw Error(KVP_ERR_CACHE, "handoff covers [" + std::to_string(in.start) + ", " +
                                                       std::to_string(in.end) + "), expected prefix [0, " +
                                                       std::to_string(start) + ")");
                    m.recv[static_cast<size_t>(r)] += in.end - in.start;
                    KVP_CUDA(cudaStreamWaitEvent(R.comp, in.ready, 0));
                }
                if (r + 1 < p) {
                    // forward the cumulative cache [0, stop) to rank r+1 (engine.hpp:283-288)
                    RankCtx& N = *e->ranks[static_cast<size_t>(r + 1)];
                    KVP_CUDA(cudaEventRecord(R.ev_ready[l], R.comp));
                    KVP_CUDA(cudaStreamWaitEvent(R.comm, R.ev_ready[l], 0));
                    KVP_CUDA(cudaMemcpyAsync(N.kv_ptr(s, l, 0), K, stop * row_kv, cudaMemcpyDefault, R.comm));
                    KVP_CUDA(cudaMemcpyAsync(N.kv_ptr(s, l, 1), V, stop * row_kv, cudaMemcpyDefault, R.comm));
                    KVP_CUDA(cudaEventRecord(R.ev_send[l], R.comm));
                    send(fab.link(r, r + 1), Msg{KV_HANDOFF, l, r, 0, stop, R.ev_send[l]}, r,
                         m.sent[static_cast<size_t>(r)]);
                }
                k_rows = stop;
            } else {
                k_rows = C;
            }
            m.dots[static_cast<size_t>(r)] += c * k_rows;
            KVP_CUDA(cudaEventRecord(R.t_attn[l], R.comp));
            exec_finish(s, w, R, c, K, V, k_rows, start);
            KVP_CUDA(cudaGetLastError());
            KVP_CUDA(cudaEventRecord(R.t_end[l], R.comp));
        }
        if (r == p - 1 && ft) KVP_CUDA(cudaMemcpyAsync(ft, R.h.as<float>() + (c - 1) * s.d, s.d * 4, cudaMemcpyDefault, R.comp));
        KVP_CUDA(cudaEventRecord(R.ev_done, R.comp));
        if (hid) KVP_CUDA(cudaMemcpyAsync(hid + start * s.d, R.h.p, c * s.d * 4, cudaMemcpyDefault, R.comp));
        fab.close_from(r);
    };

    std::vector<std::thread> threads;
    threads.reserve(static_cast<size_t>(p));
    for (int64_t r = 0; r < p; ++r) {
        threads.emplace_back([&, r] {
            try {
                worker(r);
            } catch (...) {
                fab.fail(std::current_exception());
            }
        });
    }
    for (auto& t : threads) t.join();
    // drain every stream before reporting (buffers stay valid, errors surface here)
    cudaError_t sync_err = cudaSuccess;
    for (int64_t r = 0; r < p; ++r) {
        RankCtx& R = *e->ranks[static_cast<size_t>(r)];
        cudaSetDevice(R.device);
        cudaError_t a = cudaStreamSynchronize(R.comm), c2 = cudaStreamSynchronize(R.comp);
        if (sync_err == cudaSuccess) sync_err = a != cudaSuccess ? a : c2;
    }
    fab.rethrow();
    if (sync_err != cudaSuccess) throw Error(KVP_ERR_CUDA, std::string("device failure: ") + cudaGetErrorString(sync_err));

    // device TTFT: earliest rank start -> last rank done (same device); wall clock otherwise
    bool one_dev = true;
    for (int64_t r = 1; r < p; ++r) one_dev &= e->ranks[static_cast<size_t>(r)]->device == e->ranks[0]->device;
    if (one_dev) {
        float lo = 0.f, hi = 0.f;
        for (int64_t r = 0; r < p; ++r) {
            float t0 = 0.f, t1 = 0.f;
            cudaEventElapsedTime(&t0, e->ranks[0]->ev_begin, e->ranks[static_cast<size_t>(r)]->ev_begin);
            cudaEventElapsedTime(&t1, e->ranks[0]->ev_begin, e->ranks[static_cast<size_t>(r)]->ev_done);
            lo = std::min(lo, t0);
            hi = std::max(hi, t1);
        }
        e->last_ttft = hi - lo;
    } else {
        e->last_ttft = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    }
    e->last_p = p;
    e->last_launches = launch_count() - launches0;

    if (met) {
        std::memset(met, 0, sizeof(*met));
        met->n_layers = s.L;
        met->p = p;
        met->barrier_count = fab.gate().generations();
        for (int64_t r = 0; r < p; ++r) {
            met->dot_products[r] = m.dots[static_cast<size_t>(r)];
            met->kv_pairs_sent[r] = m.sent[static_cast<size_t>(r)];
            met->kv_pairs_received[r] = m.recv[static_cast<size_t>(r)];
            met->wait_events[r] = m.waits[static_cast<size_t>(r)];
        }
    }
}

// Per-op helpers run on a private rank context on devices[0].
static RankCtx& util_ctx(kvp_engine* e, int64_t rows, int64_t held) {
    if (!e->util) e->util = std::make_unique<RankCtx>();
    e->util->setup(e->devices[0], e->s.L);
    e->util->alloc(e->s, rows, held);
    return *e->util;
}

// host f32 -> device buffer in the engine's element type
static void upload_elems(const Shape& s, void* dst, const float* src, int64_t n, DevBuf& tmp, cudaStream_t st) {
    if (s.prec == KVP_F32) {
        KVP_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyHostToDevice, st));
        return;
    }
    KVP_CUDA(cudaMemcpyAsync(tmp.p, src, n * 4, cudaMemcpyHostToDevice, st));
    launch_cast_bf16(tmp.as<float>(), static_cast<bf16*>(dst), n, st);
}

static void download_elems(const Shape& s, float* dst, const void* src, int64_t n, DevBuf& tmp, cudaStream_t st) {
    if (s.prec == KVP_F32) {
        KVP_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToHost, st));
        return;
    }
    launch_cast_f32(static_cast<const bf16*>(src), tmp.as<float>(), n, st);
    KVP_CUDA(cudaMemcpyAsync(dst, tmp.p, n * 4, cudaMemcpyDeviceToHost, st));
}

}  // namespace kvp

using namespace kvp;

extern "C" {

int32_t kvp_abi_version(void) { return KVP_ABI_VERSION; }
const char* kvp_last_error(void) { return t_last_error.c_str(); }
int32_t kvp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

kvp_status kvp_engine_create(const kvp_model_config* cfg, const int32_t* devices, int32_t n_devices, kvp_engine** out) {
    return guard([&] {
        if (!cfg || !out) throw Error(KVP_ERR_INPUT, "null argument");
        *out = nullptr;
        auto e = std::make_unique<kvp_engine>();
        e->s = make_shape(*cfg);
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw Error(KVP_ERR_CUDA, "no CUDA device: the B200 path has no CPU fallback");
        }
        if (n_devices <= 0 || !devices) {
            e->devices = {0};
        } else {
            for (int i = 0; i < n_devices; ++i) {
                if (devices[i] < 0 || devices[i] >= count) throw Error(KVP_ERR_INPUT, "bad device ordinal");
                e->devices.push_back(devices[i]);
            }
        }
        for (int dev : e->devices) {
            auto w = std::make_unique<DeviceWeights>();
            w->init(e->s, dev);
            e->weights.push_back(std::move(w));
        }
        // peer access between the devices of this engine (KV handoff over NVLink)
        for (int a : e->devices)
            for (int bdev : e->devices)
                if (a != bdev) {
                    int ok = 0;
                    cudaDeviceCanAccessPeer(&ok, a, bdev);
                    e->peer_ok &= ok != 0;
                    if (ok) {
                        cudaSetDevice(a);
                        cudaDeviceEnablePeerAccess(bdev, 0);
                        cudaGetLastError();
                    }
                }
        *out = e.release();
    });
}

kvp_status kvp_engine_load_layer(kvp_engine* e, int64_t layer, const float* wq, const float* wk, const float* wv,
                                 const float* wo, const float* w1, const float* w2) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        if (layer < 0 || layer >= e->s.L) throw Error(KVP_ERR_DIMENSION, "layer index out of range");
        const float* mats[6] = {wq, wk, wv, wo, w1, w2};
        for (auto& w : e->weights) w->load(e->s, layer, mats);
    });
}

// Opt-in rotary position embedding (extension: the reference model has none).
// Pairs (2i, 2i+1) of every Q and K head rotate by position * theta^(-2i/head_dim), applied in
// the QKV projection's epilogue before the rows reach the KV cache (and the handoff mirrors).
kvp_status kvp_engine_set_rope(kvp_engine* e, double theta) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        if (theta > 0) {
            if (s.prec != KVP_BF16)
                throw Error(KVP_ERR_CONFIG, "RoPE is a bf16-mode extension; the f32 parity mode keeps the reference model");
            if (s.hd % 32 != 0) throw Error(KVP_ERR_CONFIG, "RoPE needs head_dim to be a multiple of 32");
            // inv_freq[i] = 1 / theta^(2i / head_dim) in f32 (the usual fp32 table)
            std::vector<float> inv(static_cast<size_t>(s.hd / 2));
            for (int64_t i = 0; i < s.hd / 2; ++i)
                inv[static_cast<size_t>(i)] =
                    1.0f / std::pow(static_cast<float>(theta), static_cast<float>(2 * i) / static_cast<float>(s.hd));
            for (auto& w : e->weights) {
                KVP_CUDA(cudaSetDevice(w->device));
                w->rope.ensure(inv.size() * 4, w->device);
                KVP_CUDA(cudaMemcpy(w->rope.p, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
            }
        }
        e->rope_theta = theta > 0 ? theta : 0.0;
        e->rope_gen += 1;
    });
}

// random_context<float> (weights.hpp:86-89) generated on devices[0]: same stream and values
// as the host kvp_random_context (SplitMix64 is a counter generator).
kvp_status kvp_random_context_device(kvp_engine* e, int64_t rows, uint64_t seed, float* out_dev) {
    return guard([&] {
        if (!e || !out_dev) throw Error(KVP_ERR_INPUT, "null argument");
        if (rows < 0) throw Error(KVP_ERR_DIMENSION, "matrix dimensions must be non-negative");
        std::lock_guard<std::mutex> g(e->mu);
        KVP_CUDA(cudaSetDevice(e->devices[0]));
        if (rows > 0) launch_seeded_f32(out_dev, rows, e->s.d, 1.0, mix_seed(seed, 0xc7u, 17), nullptr);
        KVP_CUDA(cudaGetLastError());
        KVP_CUDA(cudaDeviceSynchronize());
    });
}

kvp_status kvp_engine_destroy(kvp_engine* e) {
    return guard([&] {
        if (!e) return;
        {
            std::lock_guard<std::mutex> g(e->mu);
            for (auto& r : e->ranks)
                if (r->device >= 0) {
                    cudaSetDevice(r->device);
                    cudaDeviceSynchronize();
                }
        }
        delete e;
    });
}

kvp_status kvp_engine_run(kvp_engine* e, int32_t strategy, const float* context, int64_t C, const int64_t* boundaries,
                          int64_t p, const kvp_fault* fault, float* hidden_out, float* first_token, kvp_metrics* metrics) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        run_engine(e, strategy, context, C, boundaries, p, fault, hidden_out, first_token, metrics);
    });
}

// forward_serial (model.hpp:197-211): the p = 1 prompt phase, plus one KVCacheSegment per
// layer covering [0, C) (kv_cache.hpp:14-31): kv_out is [L][2][C][kv] f32 (K then V).
kvp_status kvp_forward_serial(kvp_engine* e, const float* context, int64_t C, float* hidden_out, float* kv_out) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        if (C < 1) throw Error(KVP_ERR_INPUT, "forward_serial: empty context");
        std::lock_guard<std::mutex> g(e->mu);
        const int64_t b[2] = {0, C};
        run_engine(e, KVP_SERIAL, context, C, b, 1, nullptr, hidden_out, nullptr, nullptr);
        if (!kv_out) return;
        const Shape& s = e->s;
        RankCtx& R = *e->ranks[0];
        KVP_CUDA(cudaSetDevice(R.device));
        DevBuf tmp;
        if (s.prec != KVP_F32) tmp.ensure(static_cast<size_t>(C) * s.kv * 4, R.device);
        for (int64_t l = 0; l < s.L; ++l)
            for (int which = 0; which < 2; ++which) {
                download_elems(s, kv_out + (2 * l + which) * C * s.kv, R.kv_ptr(s, l, which), C * s.kv, tmp, R.comp);
                KVP_CUDA(cudaStreamSynchronize(R.comp));
            }
    });
}

kvp_status kvp_engine_run_device(kvp_engine* e, int32_t strategy, const float* context_dev, int64_t C,
                                 const int64_t* boundaries, int64_t p, const kvp_fault* fault, float* hidden_out_dev,
                                 float* first_token_dev, kvp_metrics* metrics) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        run_engine(e, strategy, context_dev, C, boundaries, p, fault, hidden_out_dev, first_token_dev, metrics);
    });
}

kvp_status kvp_engine_layer_times(kvp_engine* e, int64_t rank, float* proj_ms, float* rest_ms, float* wait_ms) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        if (rank < 0 || rank >= e->last_p) throw Error(KVP_ERR_INPUT, "rank out of range for the last run");
        RankCtx& R = *e->ranks[static_cast<size_t>(rank)];
        cudaSetDevice(R.device);
        for (int64_t l = 0; l < e->s.L; ++l) {
            float a = 0, bb = 0, c = 0;
            KVP_CUDA(cudaEventElapsedTime(&a, R.t_start[l], R.t_qkv[l]));
            KVP_CUDA(cudaEventElapsedTime(&bb, R.t_attn[l], R.t_end[l]));
            KVP_CUDA(cudaEventElapsedTime(&c, R.t_qkv[l], R.t_attn[l]));
            if (proj_ms) proj_ms[l] = a;
            if (rest_ms) rest_ms[l] = bb;
            if (wait_ms) wait_ms[l] = c;
        }
    });
}

kvp_status kvp_engine_last_ttft_ms(kvp_engine* e, float* ms) {
    return guard([&] {
        if (!e || !ms) throw Error(KVP_ERR_INPUT, "null argument");
        *ms = e->last_ttft;
    });
}

kvp_status kvp_engine_last_launch_count(kvp_engine* e, int64_t* count) {
    return guard([&] {
        if (!e || !count) throw Error(KVP_ERR_INPUT, "null argument");
        *count = e->last_launches;
    });
}

kvp_status kvp_engine_set_profiling(kvp_engine* e, int32_t on) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        e->profiling = on != 0;
    });
}

kvp_status kvp_engine_kernel_stats(kvp_engine* e, kvp_kernel_stats* out, int32_t max_entries, int32_t* n_out) {
    return guard([&] {
        if (!e || !out || !n_out) throw Error(KVP_ERR_INPUT, "null argument");
        std::lock_guard<std::mutex> g(e->mu);
        kvp_kernel_stats acc[K_NUM];
        std::memset(acc, 0, sizeof acc);
        for (int k = 0; k < K_NUM; ++k) std::snprintf(acc[k].name, sizeof acc[k].name, "%s", kKernelNames[k]);
        for (int64_t r = 0; r < e->last_p; ++r) {
            RankCtx& R = *e->ranks[static_cast<size_t>(r)];
            cudaSetDevice(R.device);
            for (const auto& m : R.marks) {
                float ms = 0.f;
                KVP_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
                acc[m.cls].launches += 1;
                acc[m.cls].total_ms += ms;
                acc[m.cls].flops += m.flops;
                acc[m.cls].bytes += m.bytes;
            }
        }
        const int n = std::min<int>(max_entries, K_NUM);
        for (int k = 0; k < n; ++k) out[k] = acc[k];
        *n_out = n;
    });
}

kvp_status kvp_engine_profile_layer(kvp_engine* e, int64_t rows, int64_t offset, int32_t reps, float* proj_ms,
                                    float* rest_ms) {
    return guard([&] {
        if (!e || !proj_ms || !rest_ms) throw Error(KVP_ERR_INPUT, "null argument");
        if (rows < 1 || offset < 0 || reps < 1) throw Error(KVP_ERR_INPUT, "rows >= 1, offset >= 0, reps >= 1");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        const LayerW& w = layer_of(e, 0, 0);
        const int64_t held = offset + rows;
        RankCtx& R = util_ctx(e, rows, held);
        KVP_CUDA(cudaSetDevice(R.device));
        // synthetic activations: a seeded uniform context and a seeded prefix cache
        launch_seeded_f32(R.h.as<float>(), rows, s.d, 1.0, 0x5eedull, R.comp);
        if (s.prec == KVP_BF16) {
            DevBuf tmp;
            tmp.ensure(held * s.kv * 4, R.device);
            for (int which = 0; which < 2; ++which) {
                launch_seeded_f32(tmp.as<float>(), held, s.kv, 1.0, 0x5eed1ull + which, R.comp);
                launch_cast_bf16(tmp.as<float>(), static_cast<bf16*>(R.kv_ptr(s, 0, which)), held * s.kv, R.comp);
            }
            KVP_CUDA(cudaStreamSynchronize(R.comp));
        } else {
            for (int which = 0; which < 2; ++which)
                launch_seeded_f32(static_cast<float*>(R.kv_ptr(s, 0, which)), held, s.kv, 1.0, 0x5eed1ull + which, R.comp);
        }
        cudaEvent_t ev[3];
        for (auto& x : ev) KVP_CUDA(cudaEventCreate(&x));
        std::vector<float> pa, ra;
        uint8_t* K = static_cast<uint8_t*>(R.kv_ptr(s, 0, 0));
        uint8_t* V = static_cast<uint8_t*>(R.kv_ptr(s, 0, 1));
        const size_t row_kv = static_cast<size_t>(s.kv) * s.es();
        const bool prof = R.profiling;
        R.profiling = false;
        for (int i = 0; i < reps + 1; ++i) {
            launch_spin(300000, R.comp);  // device time only: the host enqueues behind the spin
            KVP_CUDA(cudaEventRecord(ev[0], R.comp));
            exec_qkv(s, w, R, rows, K + offset * row_kv, V + offset * row_kv, true);
            KVP_CUDA(cudaEventRecord(ev[1], R.comp));
            exec_finish(s, w, R, rows, K, V, held, offset);
            KVP_CUDA(cudaEventRecord(ev[2], R.comp));
            KVP_CUDA(cudaEventSynchronize(ev[2]));
            float a = 0, b = 0;
            KVP_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
            KVP_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
            if (i > 0) {  // first run warms up
                pa.push_back(a);
                ra.push_back(b);
            }
        }
        R.profiling = prof;
        for (auto& x : ev) cudaEventDestroy(x);
        std::sort(pa.begin(), pa.end());
        std::sort(ra.begin(), ra.end());
        *proj_ms = pa[pa.size() / 2];
        *rest_ms = ra[ra.size() / 2];
    });
}

kvp_status kvp_bench_gemm(kvp_engine* e, int64_t M, int64_t N, int64_t K, int32_t epi, int32_t reps, float* ms,
                          int32_t* bn_out) {
    return guard([&] {
        if (!e || !ms) throw Error(KVP_ERR_INPUT, "null argument");
        if (M < 1 || N < 16 || K < 8 || reps < 1) throw Error(KVP_ERR_INPUT, "bad GEMM shape");
        std::lock_guard<std::mutex> g(e->mu);
        KVP_CUDA(cudaSetDevice(e->devices[0]));
        // KVP_GEMM_BENCH_CHAIN=c: time `reps` launches back to back (PDL-chained, as inside a
        // layer step) cycling c weight copies, so the weights stream from HBM as in a real
        // layer sequence; default: isolated launches behind a spin kernel, median
        static const int chain = [] {
            const char* v = getenv("KVP_GEMM_BENCH_CHAIN");
            return v ? std::max(1, atoi(v)) : 0;
        }();
        const int copies = chain > 0 ? chain : 1;
        DevBuf a, b, of, ob, rf;
        a.ensure(M * K * 2, e->devices[0]);
        b.ensure(copies * N * K * 2, e->devices[0]);
        of.ensure(M * N * 4, e->devices[0]);
        ob.ensure(M * N * 2, e->devices[0]);
        rf.ensure(M * N * 4, e->devices[0]);
        DevBuf tmp;
        tmp.ensure(std::max(M, N) * K * 4, e->devices[0]);
        cudaStream_t st = nullptr;
        launch_seeded_f32(tmp.as<float>(), M, K, 1.0, 11, st);
        launch_cast_bf16(tmp.as<float>(), a.as<bf16>(), M * K, st);
        launch_seeded_f32(tmp.as<float>(), N, K, 0.02, 12, st);
        launch_cast_bf16(tmp.as<float>(), b.as<bf16>(), N * K, st);
        for (int c = 1; c < copies; ++c)
            KVP_CUDA(cudaMemcpyAsync(b.as<bf16>() + c * N * K, b.as<bf16>(), N * K * 2, cudaMemcpyDeviceToDevice, st));
        launch_seeded_f32(rf.as<float>(), M, N, 1.0, 13, st);
        GemmEpilogue ep;
        ep.kind = epi;
        ep.out0 = ob.as<bf16>();
        ep.ld0 = N;
        ep.n0 = N;
        if (epi == EPI_QKV) {  // split like a fused Wqkv: q = N - 2*(N/6) ... three column blocks
            const int64_t kvw = ((N / 6) / 32) * 32;
            ep.n0 = N - 2 * kvw;
            ep.ld0 = ep.n0;
            ep.out1 = ob.as<bf16>() + M * ep.n0;
            ep.ld1 = kvw;
            ep.n1 = kvw;
            ep.out2 = ep.out1 + M * kvw;
            ep.ld2 = kvw;
        }
        ep.outf = of.as<float>();
        ep.ldf = N;
        ep.resid = rf.as<float>();
        ep.ldr = N;
        if (epi == EPI_RESID) {
            ep.outb = ob.as<bf16>();
            ep.ldb = N;
        }
        cudaEvent_t e0, e1;
        KVP_CUDA(cudaEventCreate(&e0));
        KVP_CUDA(cudaEventCreate(&e1));
        std::vector<float> t;
        if (chain > 0) {
            for (int i = 0; i < copies; ++i)  // warm-up
                gemm_bf16_tc(a.as<bf16>(), M, K, b.as<bf16>() + (i % copies) * N * K, N, ep, st);
            KVP_CUDA(cudaEventRecord(e0, st));
            for (int i = 0; i < reps; ++i)
                gemm_bf16_tc(a.as<bf16>(), M, K, b.as<bf16>() + (i % copies) * N * K, N, ep, st);
            KVP_CUDA(cudaEventRecord(e1, st));
            KVP_CUDA(cudaEventSynchronize(e1));
            float x = 0;
            KVP_CUDA(cudaEventElapsedTime(&x, e0, e1));
            t.push_back(x / reps);
        }
        for (int i = 0; chain == 0 && i < reps + 1; ++i) {
            launch_spin(100000, st);  // device time only: the host enqueues behind the spin
            KVP_CUDA(cudaEventRecord(e0, st));
            gemm_bf16_tc(a.as<bf16>(), M, K, b.as<bf16>(), N, ep, st);
            KVP_CUDA(cudaEventRecord(e1, st));
            KVP_CUDA(cudaEventSynchronize(e1));
            float x = 0;
            KVP_CUDA(cudaEventElapsedTime(&x, e0, e1));
            if (i) t.push_back(x);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        gemm_trace_dump();
        std::sort(t.begin(), t.end());
        *ms = t[t.size() / 2];
        if (bn_out) *bn_out = gemm_bf16_tc_bn(M, N);
    });
}

kvp_status kvp_bench_attn(kvp_engine* e, int64_t q_rows, int64_t offset, int32_t n_heads, int32_t n_kv_heads,
                          int32_t head_dim, int32_t reps, float* ms) {
    return guard([&] {
        if (!e || !ms) throw Error(KVP_ERR_INPUT, "null argument");
        if (q_rows < 1 || offset < 0 || reps < 1 || n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads)
            throw Error(KVP_ERR_INPUT, "bad attention shape");
        if (!attn_tc_supported(head_dim)) throw Error(KVP_ERR_INPUT, "head_dim must be 64 or 128");
        std::lock_guard<std::mutex> g(e->mu);
        KVP_CUDA(cudaSetDevice(e->devices[0]));
        const int64_t k_rows = offset + q_rows, qd = int64_t(n_heads) * head_dim, kvd = int64_t(n_kv_heads) * head_dim;
        DevBuf q, k, v, o, tmp;
        q.ensure(q_rows * qd * 2, e->devices[0]);
        k.ensure(k_rows * kvd * 2, e->devices[0]);
        v.ensure(k_rows * kvd * 2, e->devices[0]);
        o.ensure(q_rows * qd * 2, e->devices[0]);
        tmp.ensure(std::max(q_rows * qd, k_rows * kvd) * 4, e->devices[0]);
        cudaStream_t st = nullptr;
        launch_seeded_f32(tmp.as<float>(), q_rows, qd, 2.0, 21, st);
        launch_cast_bf16(tmp.as<float>(), q.as<bf16>(), q_rows * qd, st);
        launch_seeded_f32(tmp.as<float>(), k_rows, kvd, 2.0, 22, st);
        launch_cast_bf16(tmp.as<float>(), k.as<bf16>(), k_rows * kvd, st);
        launch_seeded_f32(tmp.as<float>(), k_rows, kvd, 1.0, 23, st);
        launch_cast_bf16(tmp.as<float>(), v.as<bf16>(), k_rows * kvd, st);
        AttnShape sh;
        sh.q_rows = q_rows;
        sh.k_rows = k_rows;
        sh.offset = offset;
        sh.n_heads = n_heads;
        sh.n_kv_heads = n_kv_heads;
        sh.head_dim = head_dim;
        sh.ldq = qd;
        sh.ldkv = kvd;
        sh.ldo = qd;
        cudaEvent_t e0, e1;
        KVP_CUDA(cudaEventCreate(&e0));
        KVP_CUDA(cudaEventCreate(&e1));
        std::vector<float> t;
        for (int i = 0; i < reps + 1; ++i) {
            launch_spin(100000, st);  // device time only: the host enqueues behind the spin
            KVP_CUDA(cudaEventRecord(e0, st));
            attn_bf16(q.as<bf16>(), k.as<bf16>(), v.as<bf16>(), o.as<bf16>(), sh, st);
            KVP_CUDA(cudaEventRecord(e1, st));
            KVP_CUDA(cudaEventSynchronize(e1));
            float x = 0;
            KVP_CUDA(cudaEventElapsedTime(&x, e0, e1));
            if (i) t.push_back(x);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        std::sort(t.begin(), t.end());
        *ms = t[t.size() / 2];
    });
}

kvp_status kvp_rank_begin(kvp_engine* e, const float* rows, int64_t n_rows, int64_t start, int64_t held,
                          int32_t rows_on_device, void* const* kv_bufs) {
    return guard([&] {
        if (!e || !rows) throw Error(KVP_ERR_INPUT, "null argument");
        if (n_rows < 1 || start < 0 || held < start + n_rows)
            throw Error(KVP_ERR_CACHE, "rank session needs n_rows >= 1 and held >= start + n_rows");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        if (e->ranks.empty()) e->ranks.push_back(std::make_unique<RankCtx>());
        RankCtx& R = *e->ranks[0];
        R.setup(e->devices[0], s.L);
        R.alloc(s, n_rows, held, kv_bufs == nullptr);
        if (kv_bufs) R.ext_kv.assign(kv_bufs, kv_bufs + 2 * s.L);
        R.profiling = e->profiling;
        R.decode = false;
        R.pos0 = start;
        R.rope_inv = e->rope_table(0);
        R.rope_hd = R.rope_inv ? static_cast<int>(s.hd) : 0;
        R.n_mirror = 0;
        R.mirror_bufs.clear();
        R.marks.clear();
        R.pool_used = 0;
        KVP_CUDA(cudaSetDevice(R.device));
        KVP_CUDA(cudaEventRecord(R.ev_begin, R.comp));
        KVP_CUDA(cudaMemcpyAsync(R.h.p, rows, n_rows * s.d * 4, rows_on_device ? cudaMemcpyDeviceToDevice
                                                                                 : cudaMemcpyHostToDevice, R.comp));
        e->in_session = true;
        e->sess_rows = n_rows;
        e->sess_start = start;
        e->sess_launch0 = launch_count();
        e->last_p = 1;
    });
}

static RankCtx& session_rank(kvp_engine* e) {
    if (!e || !e->in_session) throw Error(KVP_ERR_INPUT, "no rank session (call kvp_rank_begin)");
    RankCtx& R = *e->ranks[0];
    KVP_CUDA(cudaSetDevice(R.device));
    return R;
}

kvp_status kvp_rank_stream(kvp_engine* e, void** stream) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        *stream = session_rank(e).comp;
    });
}

kvp_status kvp_rank_set_decode(kvp_engine* e, int32_t on) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        RankCtx& R = session_rank(e);
        if (on && e->sess_rows > 8) throw Error(KVP_ERR_INPUT, "decode steps take at most 8 new rows");
        R.decode = on != 0 && e->s.prec == KVP_BF16;  // f32 keeps the ordered SIMT kernels
    });
}

kvp_status kvp_rank_set_mirrors(kvp_engine* e, int32_t n_mirrors, void* const* mirror_bufs) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        RankCtx& R = session_rank(e);
        if (n_mirrors < 0 || n_mirrors > KVP_MAX_MIRRORS)
            throw Error(KVP_ERR_INPUT, "at most " + std::to_string(KVP_MAX_MIRRORS) + " mirrors");
        if (n_mirrors > 0 && e->s.prec != KVP_BF16)
            throw Error(KVP_ERR_CONFIG, "the fused KV handoff needs the bf16 tcgen05 projection");
        if (n_mirrors > 0 && !mirror_bufs) throw Error(KVP_ERR_INPUT, "null mirror buffers");
        R.n_mirror = n_mirrors;
        R.mirror_bufs.assign(mirror_bufs, mirror_bufs + static_cast<size_t>(n_mirrors) * 2 * e->s.L);
        for (void* ptr : R.mirror_bufs)
            if (!ptr) throw Error(KVP_ERR_INPUT, "null mirror buffer");
    });
}

}  // extern "C"

namespace kvp {
// driver-API entry points (no -lcuda at link time: fetched through the runtime)
template <typename Fn>
static Fn driver_fn(const char* name) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        throw Error(KVP_ERR_CUDA, std::string("driver entry point unavailable: ") + name);
    return reinterpret_cast<Fn>(ptr);
}
using StreamValueFn = int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
using AddrRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
}  // namespace kvp

extern "C" {

kvp_status kvp_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset) {
    return guard([&] {
        if (!dev_ptr || !handle64 || !offset) throw Error(KVP_ERR_INPUT, "null argument");
        static const auto range = driver_fn<AddrRangeFn>("cuMemGetAddressRange");
        unsigned long long base = 0;
        size_t size = 0;
        if (range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
            throw Error(KVP_ERR_CUDA, "not a device allocation");
        cudaIpcMemHandle_t h;
        KVP_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
        std::memcpy(handle64, &h, sizeof(h));
        *offset = static_cast<int64_t>(reinterpret_cast<unsigned long long>(dev_ptr) - base);
    });
}

kvp_status kvp_ipc_open(const void* handle64, int64_t offset, void** dev_ptr) {
    return guard([&] {
        if (!handle64 || !dev_ptr || offset < 0) throw Error(KVP_ERR_INPUT, "bad argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        void* base = nullptr;
        KVP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        *dev_ptr = static_cast<uint8_t*>(base) + offset;
    });
}

kvp_status kvp_ipc_close(void* dev_ptr, int64_t offset) {
    return guard([&] {
        if (!dev_ptr) throw Error(KVP_ERR_INPUT, "null pointer");
        KVP_CUDA(cudaIpcCloseMemHandle(static_cast<uint8_t*>(dev_ptr) - offset));
    });
}

kvp_status kvp_stream_signal(void* stream, void* flag, uint32_t value) {
    return guard([&] {
        if (!flag) throw Error(KVP_ERR_INPUT, "null flag");
        static const auto write = driver_fn<StreamValueFn>("cuStreamWriteValue32");
        // default flags: the write is preceded by a stream-scoped system-wide memory fence
        if (write(static_cast<cudaStream_t>(stream), reinterpret_cast<unsigned long long>(flag), value, 0) != 0)
            throw Error(KVP_ERR_CUDA, "cuStreamWriteValue32 failed");
    });
}

kvp_status kvp_stream_wait(void* stream, const void* flag, uint32_t value) {
    return guard([&] {
        if (!flag) throw Error(KVP_ERR_INPUT, "null flag");
        static const auto wait = driver_fn<StreamValueFn>("cuStreamWaitValue32");
        // CU_STREAM_WAIT_VALUE_GEQ (0): values only grow (run epoch * layers + layer + 1)
        if (wait(static_cast<cudaStream_t>(stream), reinterpret_cast<unsigned long long>(flag), value, 0) != 0)
            throw Error(KVP_ERR_CUDA, "cuStreamWaitValue32 failed");
    });
}

kvp_status kvp_stream_copy(void* stream, void* dst, const void* src, int64_t bytes) {
    return guard([&] {
        if (bytes < 0 || ((!dst || !src) && bytes > 0)) throw Error(KVP_ERR_INPUT, "bad copy");
        if (bytes > 0)
            KVP_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                                     static_cast<cudaStream_t>(stream)));
    });
}

kvp_status kvp_rank_kv(kvp_engine* e, int64_t layer, void** K, void** V) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        RankCtx& R = session_rank(e);
        if (layer < 0 || layer >= e->s.L) throw Error(KVP_ERR_DIMENSION, "layer index out of range");
        *K = R.kv_ptr(e->s, layer, 0);
        *V = R.kv_ptr(e->s, layer, 1);
    });
}

kvp_status kvp_rank_qkv(kvp_engine* e, int64_t layer) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        RankCtx& R = session_rank(e);
        const Shape& s = e->s;
        const LayerW& w = layer_of(e, 0, layer);
        const size_t row_kv = static_cast<size_t>(s.kv) * s.es();
        uint8_t* K = static_cast<uint8_t*>(R.kv_ptr(s, layer, 0));
        uint8_t* V = static_cast<uint8_t*>(R.kv_ptr(s, layer, 1));
        KVP_CUDA(cudaEventRecord(R.t_start[layer], R.comp));
        KvMirrors mir;
        for (int m = 0; m < R.n_mirror; ++m) {
            const size_t at = (static_cast<size_t>(m) * s.L + static_cast<size_t>(layer)) * 2;
            mir.k[m] = static_cast<uint8_t*>(R.mirror_bufs[at]) + e->sess_start * row_kv;
            mir.v[m] = static_cast<uint8_t*>(R.mirror_bufs[at + 1]) + e->sess_start * row_kv;
        }
        mir.n = R.decode ? 0 : R.n_mirror;
        exec_qkv(s, w, R, e->sess_rows, K + e->sess_start * row_kv, V + e->sess_start * row_kv, layer == 0, &mir);
        KVP_CUDA(cudaGetLastError());
        KVP_CUDA(cudaEventRecord(R.t_qkv[layer], R.comp));
    });
}

kvp_status kvp_rank_finish(kvp_engine* e, int64_t layer, int64_t k_rows) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        RankCtx& R = session_rank(e);
        const Shape& s = e->s;
        const LayerW& w = layer_of(e, 0, layer);
        if (k_rows < e->sess_start + e->sess_rows || k_rows > R.held)
            throw Error(KVP_ERR_CACHE, "finish needs sess_start + rows <= k_rows <= held");
        KVP_CUDA(cudaEventRecord(R.t_attn[layer], R.comp));
        exec_finish(s, w, R, e->sess_rows, R.kv_ptr(s, layer, 0), R.kv_ptr(s, layer, 1), k_rows, e->sess_start);
        KVP_CUDA(cudaGetLastError());
        KVP_CUDA(cudaEventRecord(R.t_end[layer], R.comp));
    });
}

kvp_status kvp_rank_end(kvp_engine* e, float* out_rows, int32_t out_on_device, float* last_row, float* ms) {
    return guard([&] {
        std::lock_guard<std::mutex> g(e->mu);
        RankCtx& R = session_rank(e);
        const Shape& s = e->s;
        // the first-token row's D2H is inside the timed span (it is part of TTFT); the optional
        // full hidden block copy is not
        if (last_row)
            KVP_CUDA(cudaMemcpyAsync(last_row, R.h.as<float>() + (e->sess_rows - 1) * s.d, s.d * 4,
                                     cudaMemcpyDeviceToHost, R.comp));
        KVP_CUDA(cudaEventRecord(R.ev_done, R.comp));
        if (out_rows)
            KVP_CUDA(cudaMemcpyAsync(out_rows, R.h.p, e->sess_rows * s.d * 4,
                                     out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, R.comp));
        KVP_CUDA(cudaStreamSynchronize(R.comp));
        float t = 0.f;
        KVP_CUDA(cudaEventElapsedTime(&t, R.ev_begin, R.ev_done));
        if (ms) *ms = t;
        e->last_ttft = t;
        e->last_launches = launch_count() - e->sess_launch0;  // this rank's kernels of the session
        e->in_session = false;
    });
}

kvp_status kvp_layer_qkv(kvp_engine* e, int64_t layer, const float* hidden, int64_t rows, float* Q, float* K, float* V) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        const LayerW& w = layer_of(e, 0, layer);
        if (rows <= 0) throw Error(KVP_ERR_INPUT, "empty hidden block");
        RankCtx& R = util_ctx(e, rows, rows);
        KVP_CUDA(cudaSetDevice(R.device));
        KVP_CUDA(cudaMemcpyAsync(R.h.p, hidden, rows * s.d * 4, cudaMemcpyHostToDevice, R.comp));
        exec_qkv(s, w, R, rows, R.kv_ptr(s, 0, 0), R.kv_ptr(s, 0, 1));
        DevBuf tmp;
        tmp.ensure(rows * std::max(s.q, s.kv) * 4, R.device);
        download_elems(s, Q, R.q.p, rows * s.q, tmp, R.comp);
        KVP_CUDA(cudaStreamSynchronize(R.comp));
        download_elems(s, K, R.kv_ptr(s, 0, 0), rows * s.kv, tmp, R.comp);
        KVP_CUDA(cudaStreamSynchronize(R.comp));
        download_elems(s, V, R.kv_ptr(s, 0, 1), rows * s.kv, tmp, R.comp);
        KVP_CUDA(cudaStreamSynchronize(R.comp));
    });
}

static void attention_op(kvp_engine* e, const float* Q, int64_t q_rows, const float* K, const float* V, int64_t k_rows,
                         int64_t offset, RankCtx& R) {
    const Shape& s = e->s;
    if (q_rows <= 0) throw Error(KVP_ERR_DIMENSION, "causal_attention: empty query block");
    if (k_rows < offset + q_rows)
        throw Error(KVP_ERR_CACHE, "causal_attention: cache holds " + std::to_string(k_rows) + " rows, need at least " +
                                       std::to_string(offset + q_rows));
    DevBuf tmp;
    tmp.ensure(std::max(q_rows * s.q, k_rows * s.kv) * 4, R.device);
    upload_elems(s, R.q.p, Q, q_rows * s.q, tmp, R.comp);
    KVP_CUDA(cudaStreamSynchronize(R.comp));
    upload_elems(s, R.kv_ptr(s, 0, 0), K, k_rows * s.kv, tmp, R.comp);
    KVP_CUDA(cudaStreamSynchronize(R.comp));
    upload_elems(s, R.kv_ptr(s, 0, 1), V, k_rows * s.kv, tmp, R.comp);
    KVP_CUDA(cudaStreamSynchronize(R.comp));
}

kvp_status kvp_causal_attention(kvp_engine* e, const float* Q, int64_t q_rows, const float* K, const float* V,
                                int64_t k_rows, int64_t offset, float* A) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        if (offset < 0) throw Error(KVP_ERR_CACHE, "negative mask offset");
        RankCtx& R = util_ctx(e, std::max<int64_t>(q_rows, 1), std::max<int64_t>(k_rows, 1));
        KVP_CUDA(cudaSetDevice(R.device));
        attention_op(e, Q, q_rows, K, V, k_rows, offset, R);
        AttnShape sh;
        sh.q_rows = q_rows;
        sh.k_rows = k_rows;
        sh.offset = offset;
        sh.n_heads = static_cast<int>(s.h);
        sh.n_kv_heads = static_cast<int>(s.kvh);
        sh.head_dim = static_cast<int>(s.hd);
        sh.ldq = s.q;
        sh.ldkv = s.kv;
        sh.ldo = s.q;
        if (s.prec == KVP_BF16) {
            if (attn_bf16_supported(sh.head_dim))
                attn_bf16(R.q.as<bf16>(), static_cast<bf16*>(R.kv_ptr(s, 0, 0)), static_cast<bf16*>(R.kv_ptr(s, 0, 1)),
                          R.a.as<bf16>(), sh, R.comp);
            else
                attn_simt_bf16(R.q.as<bf16>(), static_cast<bf16*>(R.kv_ptr(s, 0, 0)),
                               static_cast<bf16*>(R.kv_ptr(s, 0, 1)), R.a.as<bf16>(), sh, R.comp);
        } else {
            attn_simt_f32(R.q.as<float>(), static_cast<float*>(R.kv_ptr(s, 0, 0)), static_cast<float*>(R.kv_ptr(s, 0, 1)),
                          R.a.as<float>(), sh, R.comp);
        }
        KVP_CUDA(cudaGetLastError());
        DevBuf tmp;
        tmp.ensure(q_rows * s.q * 4, R.device);
        download_elems(s, A, R.a.p, q_rows * s.q, tmp, R.comp);
        KVP_CUDA(cudaStreamSynchronize(R.comp));
    });
}

kvp_status kvp_layer_finish(kvp_engine* e, int64_t layer, const float* hidden, int64_t rows, const float* Q,
                            const float* K, const float* V, int64_t k_rows, int64_t offset, float* out) {
    return guard([&] {
        if (!e) throw Error(KVP_ERR_INPUT, "null engine");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        const LayerW& w = layer_of(e, 0, layer);
        if (offset < 0) throw Error(KVP_ERR_CACHE, "negative mask offset");
        RankCtx& R = util_ctx(e, std::max<int64_t>(rows, 1), std::max<int64_t>(k_rows, 1));
        KVP_CUDA(cudaSetDevice(R.device));
        attention_op(e, Q, rows, K, V, k_rows, offset, R);
        KVP_CUDA(cudaMemcpyAsync(R.h.p, hidden, rows * s.d * 4, cudaMemcpyHostToDevice, R.comp));
        exec_finish(s, w, R, rows, R.kv_ptr(s, 0, 0), R.kv_ptr(s, 0, 1), k_rows, offset);
        KVP_CUDA(cudaGetLastError());
        KVP_CUDA(cudaMemcpyAsync(out, R.h.p, rows * s.d * 4, cudaMemcpyDeviceToHost, R.comp));
        KVP_CUDA(cudaStreamSynchronize(R.comp));
    });
}

}  // extern "C"

// ------------------------------------------------------------------ KV cache + decode (8f #4)
struct kvp_kv_cache {
    kvp_engine* e = nullptr;
    kvp::DevBuf buf;
    int64_t capacity = 0, length = 0;
    std::vector<void*> ptrs;  // K_0, V_0, K_1, ...: [capacity x kv] each
};

kvp_status kvp_kv_cache_create(kvp_engine* e, int64_t capacity, kvp_kv_cache** out) {
    return guard([&] {
        if (!e || !out) throw Error(KVP_ERR_INPUT, "null argument");
        if (capacity < 1) throw Error(KVP_ERR_CACHE, "cache capacity must be >= 1");
        std::lock_guard<std::mutex> g(e->mu);
        const Shape& s = e->s;
        KVP_CUDA(cudaSetDevice(e->devices[0]));
        auto c = std::make_unique<kvp_kv_cache>();
        c->e = e;
        c->capacity = capacity;
        const size_t per = static_cast<size_t>(capacity) * s.kv * s.es();
        c->buf.ensure(per * 2 * s.L, e->devices[0]);
        for (int64_t i = 0; i < 2 * s.L; ++i) c->ptrs.push_back(c->buf.as<uint8_t>() + i * per);
        *out = c.release();
    });
}

kvp_status kvp_kv_cache_destroy(kvp_kv_cache* c) {
    return guard([&] { delete c; });
}

kvp_status kvp_kv_cache_length(const kvp_kv_cache* c, int64_t* length) {
    return guard([&] {
        if (!c || !length) throw Error(KVP_ERR_INPUT, "null argument");
        *length = c->length;
    });
}

kvp_status kvp_kv_cache_reset(kvp_kv_cache* c, int64_t length) {
    return guard([&] {
        if (!c) throw Error(KVP_ERR_INPUT, "null argument");
        if (length < 0 || length > c->length) throw Error(KVP_ERR_CACHE, "can only truncate the cache");
        c->length = length;
    });
}

// one rank session over rows [start, start + n) of a cache: the same per-layer schedule as a
// KVR rank whose prefix [0, start) is already in place
static void cached_session(kvp_engine* e, kvp_kv_cache* c, const float* rows, int64_t n, int32_t rows_on_device,
                           bool decode, float* out_rows, float* last_row, float* ms) {
    auto ok = [](kvp_status st) {
        if (st != KVP_OK) throw Error(st, kvp_last_error());
    };
    if (!c || c->e != e) throw Error(KVP_ERR_INPUT, "cache belongs to another engine");
    if (n < 1) throw Error(KVP_ERR_INPUT, "no rows");
    const int64_t start = c->length;
    if (start + n > c->capacity) throw Error(KVP_ERR_CACHE, "cache capacity exceeded");
    ok(kvp_rank_begin(e, rows, n, start, c->capacity, rows_on_device, c->ptrs.data()));
    if (decode) ok(kvp_rank_set_decode(e, 1));
    for (int64_t l = 0; l < e->s.L; ++l) {
        ok(kvp_rank_qkv(e, l));
        ok(kvp_rank_finish(e, l, start + n));
    }
    ok(kvp_rank_end(e, out_rows, 0, last_row, ms));
    c->length = start + n;
}

kvp_status kvp_prefill_cached(kvp_engine* e, kvp_kv_cache* c, const float* context, int64_t C, float* hidden_out,
                              float* first_token_hidden, float* ms) {
    return guard([&] {
        if (!e || !context) throw Error(KVP_ERR_INPUT, "null argument");
        cached_session(e, c, context, C, 0, false, hidden_out, first_token_hidden, ms);
    });
}

kvp_status kvp_decode(kvp_engine* e, kvp_kv_cache* c, const float* rows, int64_t n_rows, float* out_rows,
                      float* ms) {
    return guard([&] {
        if (!e || !rows) throw Error(KVP_ERR_INPUT, "null argument");
        if (c && c->length == 0) throw Error(KVP_ERR_CACHE, "decode needs a prefilled cache");
        if (n_rows > 8) throw Error(KVP_ERR_INPUT, "decode steps take at most 8 new rows");
        cached_session(e, c, rows, n_rows, 0, true, out_rows, nullptr, ms);
    });
}
