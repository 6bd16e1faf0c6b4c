/*
 * kvp_b200.h -- C-ABI of libkvp_b200.so, the B200-native KV-Runahead prompt phase.
 *
 * This is the drop-in boundary for the reference's hot path (kvprefill, a header-only
 * C++20 library with no FFI of its own).  Each entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj/include/kvprefill/).
 * Plain pointers and sizes only: no torch, no C++ types.  Host arrays are row-major
 * float32 unless stated; "_device" variants take device pointers on the engine's
 * first device.  Every call returns a kvp_status; KVP_OK == 0.  The first error of a
 * call is described by kvp_last_error() (thread-local).
 *
 * There is no CPU fallback: without a CUDA device every compute entry point returns
 * KVP_ERR_CUDA.  Precision f64 has no GPU path and returns KVP_ERR_CONFIG.
 */
#ifndef KVP_B200_H
#define KVP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVP_ABI_VERSION 1
#define KVP_MAX_RANKS 64

/* One code per exception type of errors.hpp:8-46, same order. */
typedef enum kvp_status {
    KVP_OK = 0,
    KVP_ERR_CONFIG = 1,      /* ConfigError      errors.hpp:13 */
    KVP_ERR_DIMENSION = 2,   /* DimensionError   errors.hpp:16 */
    KVP_ERR_CACHE = 3,       /* CacheError       errors.hpp:19 */
    KVP_ERR_INPUT = 4,       /* InputError       errors.hpp:22 */
    KVP_ERR_PARTITION = 5,   /* PartitionError   errors.hpp:25 */
    KVP_ERR_PROTOCOL = 6,    /* ProtocolError    errors.hpp:28 */
    KVP_ERR_ASSEMBLY = 7,    /* AssemblyError    errors.hpp:31 */
    KVP_ERR_LOOKUP = 8,      /* LookupError      errors.hpp:34 */
    KVP_ERR_SEARCH = 9,      /* SearchError      errors.hpp:37 */
    KVP_ERR_BUDGET = 10,     /* BudgetError      errors.hpp:40 */
    KVP_ERR_CALIBRATION = 11,/* CalibrationError errors.hpp:43 */
    KVP_ERR_IO = 12,         /* IoError          errors.hpp:46 */
    KVP_ERR_CUDA = 100,      /* device / driver failure (no reference equivalent) */
    KVP_ERR_NCCL = 101
} kvp_status;

/* Precision (config.hpp:10) plus the additive bf16 mode. */
typedef enum { KVP_F32 = 0, KVP_F64 = 1, KVP_BF16 = 2 } kvp_precision;
/* Strategy (engine.hpp:21). */
typedef enum { KVP_SERIAL = 0, KVP_TSP = 1, KVP_KVR = 2 } kvp_strategy;
/* FaultInjection::Kind (engine.hpp:50-55). */
typedef enum {
    KVP_FAULT_NONE = 0,
    KVP_FAULT_CORRUPT_LAYER_TAG = 1,
    KVP_FAULT_DROP_MESSAGE = 2,
    KVP_FAULT_DUPLICATE_MESSAGE = 3
} kvp_fault_kind;

/* ModelConfig (config.hpp:22-47). */
typedef struct kvp_model_config {
    int64_t d_model, n_heads, n_kv_heads, n_layers;
    uint64_t seed;
    int32_t precision; /* kvp_precision */
    int32_t rms_norm;  /* 0/1 */
} kvp_model_config;

/* FaultInjection (engine.hpp:50-55). */
typedef struct kvp_fault {
    int32_t kind; /* kvp_fault_kind */
    int64_t rank, layer;
} kvp_fault;

/* ExecutionMetrics (engine.hpp:61-83), per rank summed over layers. */
typedef struct kvp_metrics {
    int64_t n_layers, barrier_count, p;
    int64_t dot_products[KVP_MAX_RANKS];
    int64_t kv_pairs_sent[KVP_MAX_RANKS];
    int64_t kv_pairs_received[KVP_MAX_RANKS];
    int64_t wait_events[KVP_MAX_RANKS];
} kvp_metrics;

/* CostModel / NetworkModel (simnet.hpp:27-63); bandwidth in (K,V) pairs per second. */
typedef struct kvp_cost_model { double alpha, proj_coeff, softmax_coeff, fixed_overhead; } kvp_cost_model;
typedef struct kvp_network_model { double bandwidth, latency; } kvp_network_model;
/* SearchConfig (search.hpp:20-41) without the evaluator. */
typedef struct kvp_search_config { int64_t grid_width, initial_stride, min_stride; } kvp_search_config;
/* SearchResult (search.hpp:43-48); the partition goes to a caller array of p+1. */
typedef struct kvp_search_result { double ttft; int64_t evaluations, levels; } kvp_search_result;
/* TtftEvaluator (search.hpp:16) as a C callback over boundaries[0..p]. */
typedef double (*kvp_evaluator)(const int64_t* boundaries, int64_t p, void* user);

typedef struct kvp_engine kvp_engine;

/* ---------------------------------------------------------------- library */
int32_t kvp_abi_version(void);
const char* kvp_last_error(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int32_t kvp_device_count(void);

/* ------------------------------------------------------- engine (run<T>) */
/* Creates the in-process prefill engine: weights from init_weights (weights.hpp:54-83)
 * generated bit-exactly ON each device in `devices` (SplitMix64 streams keyed by
 * (seed, layer, role)); bf16 mode rounds those f32 values RNE and stores them
 * pre-transposed K-major.  Rank r of a run executes on devices[r % n_devices]. */
kvp_status kvp_engine_create(const kvp_model_config* cfg, const int32_t* devices, int32_t n_devices,
                             kvp_engine** out);
/* Replaces layer `layer`'s weights on every device with caller matrices (reference
 * [in x out] layout, f32): wq d x q, wk d x kv, wv d x kv, wo q x d, w1 d x 2d, w2 2d x d. */
kvp_status kvp_engine_load_layer(kvp_engine* e, int64_t layer, const float* wq, const float* wk,
                                 const float* wv, const float* wo, const float* w1, const float* w2);
kvp_status kvp_engine_destroy(kvp_engine* e);

/* run<T>(strategy, context, partition, weights, fault) (engine.hpp:186-318).
 * context: C x d host f32.  boundaries: p+1 entries (ContextPartition, partition.hpp:17).
 * hidden_out (nullable): C x d, rank order (assemble_output, engine.hpp:124-139).
 * first_token (nullable): d floats, row C-1 (engine.hpp:88,315).  fault nullable. */
kvp_status kvp_engine_run(kvp_engine* e, int32_t strategy, const float* context, int64_t C,
                          const int64_t* boundaries, int64_t p, const kvp_fault* fault,
                          float* hidden_out, float* first_token, kvp_metrics* metrics);
/* forward_serial (model.hpp:197-211): the single-rank prompt phase.  hidden_out (nullable):
 * C x d.  kv_out (nullable): the per-layer KVCacheSegment{layer, 0, C, K, V} rows
 * (kv_cache.hpp:14-31) as [n_layers][2][C][kv] f32, K before V. */
kvp_status kvp_forward_serial(kvp_engine* e, const float* context, int64_t C, float* hidden_out,
                              float* kv_out);
/* Same, but context / hidden_out / first_token are device pointers on devices[0]
 * (inputs already resident in HBM). */
kvp_status kvp_engine_run_device(kvp_engine* e, int32_t strategy, const float* context_dev,
                                 int64_t C, const int64_t* boundaries, int64_t p,
                                 const kvp_fault* fault, float* hidden_out_dev,
                                 float* first_token_dev, kvp_metrics* metrics);
/* Per-rank, per-layer device times of the last run (CUDA events on the rank's compute
 * stream), milliseconds: proj_ms = norm+QKV, rest_ms = attention..FFN (after the KV
 * prefix is available), wait_ms = time the rank's stream waited for its prefix.
 * Each array holds n_layers entries.  Feeds the load balancer (kvp_fit_cost_model). */
kvp_status kvp_engine_layer_times(kvp_engine* e, int64_t rank, float* proj_ms, float* rest_ms,
                                  float* wait_ms);
/* Device time of the last run, max over ranks, from the first launch to the first-token
 * readout (ms). */
kvp_status kvp_engine_last_ttft_ms(kvp_engine* e, float* ms);
/* Number of kernels this library launched during the last run (all ranks). */
kvp_status kvp_engine_last_launch_count(kvp_engine* e, int64_t* count);

/* Per-kernel-class device timing (profiling mode: CUDA events around every launch on the
 * launching stream).  Classes: "norm", "gemm_qkv", "attention", "gemm_o", "gemm_ffn1",
 * "gemm_ffn2".  flops / bytes are ALGORITHMIC per class summed over the last run's launches
 * (GEMM 2*M*N*K; attention 4*head_dim*heads per causal-visible (query,key) pair; norm reads
 * 4 B and writes 2-4 B per element). */
typedef struct kvp_kernel_stats {
    char name[32];
    int64_t launches;
    double total_ms, flops, bytes;
} kvp_kernel_stats;
kvp_status kvp_engine_set_profiling(kvp_engine* e, int32_t on);
kvp_status kvp_engine_kernel_stats(kvp_engine* e, kvp_kernel_stats* out, int32_t max_entries, int32_t* n_out);

/* Calibration for the load balancer: times ONE rank's layer executor in isolation on
 * devices[0] for `rows` local tokens after a prefix of `offset` tokens (held = offset + rows
 * keys), median of `reps` runs of layer 0 with synthetic activations.  proj_ms = norm+QKV
 * GEMM, rest_ms = attention + O-proj + FFN (the terms of CostModel::layer_time,
 * simnet.hpp:39-43). */
kvp_status kvp_engine_profile_layer(kvp_engine* e, int64_t rows, int64_t offset, int32_t reps, float* proj_ms,
                                    float* rest_ms);

/* Kernel microbenchmark (tuning / ncu target): the tcgen05 GEMM D[M x N] = A[M x K] B[N x K]^T
 * on devices[0] with random bf16 operands and epilogue kind epi (0 QKV-split, 1 residual,
 * 2 ReLU, 3 store); median device ms over reps (CUDA events); bn_out = tile width used. */
kvp_status kvp_bench_gemm(kvp_engine* e, int64_t M, int64_t N, int64_t K, int32_t epi, int32_t reps, float* ms,
                          int32_t* bn_out);

/* Kernel microbenchmark: the bf16 prefix-causal attention of q_rows queries at absolute
 * positions [offset, offset + q_rows) over offset + q_rows keys (random bf16 Q/K/V, head_dim
 * 64 or 128) on devices[0]; median device ms over reps (CUDA events). */
kvp_status kvp_bench_attn(kvp_engine* e, int64_t q_rows, int64_t offset, int32_t n_heads, int32_t n_kv_heads,
                          int32_t head_dim, int32_t reps, float* ms);

/* ------------------------------------------- one rank of a multi-process run */
/* One process per GPU: the caller owns the transport (e.g. NCCL p2p via torch.distributed)
 * and drives one rank's per-layer schedule -- the worker loop of run<T>
 * (engine.hpp:223-296) with the Channel send/recv replaced by the caller's transport.
 * kv_bufs: 2*n_layers device pointers (K_0, V_0, K_1, V_1, ...), each [held x kv] in the
 * engine's element type (bf16 or f32), owned by the caller (so the transport can address
 * them); NULL = engine-owned buffers.  rows: the rank's context rows [start, start+n_rows)
 * (host f32, or device f32 when rows_on_device).  Work is enqueued on the engine stream
 * returned by kvp_rank_stream; the caller orders its transport on that stream. */
kvp_status kvp_rank_begin(kvp_engine* e, const float* rows, int64_t n_rows, int64_t start, int64_t held,
                          int32_t rows_on_device, void* const* kv_bufs);
kvp_status kvp_rank_stream(kvp_engine* e, void** stream);
kvp_status kvp_rank_kv(kvp_engine* e, int64_t layer, void** K, void** V);
/* layer_qkv for the local rows: K/V rows land at [start, start+n_rows) of layer `layer`. */
kvp_status kvp_rank_qkv(kvp_engine* e, int64_t layer);
/* layer_finish over keys [0, k_rows) of layer `layer` with mask offset = start. */
kvp_status kvp_rank_finish(kvp_engine* e, int64_t layer, int64_t k_rows);
/* Synchronises, writes the final hidden rows (n_rows x d; host or device per out_on_device,
 * nullable) and the last local row (d floats, host, nullable); *ms = device time of the rank
 * from kvp_rank_begin to the last layer (nullable). */
kvp_status kvp_rank_end(kvp_engine* e, float* out_rows, int32_t out_on_device, float* last_row, float* ms);
/* Switch the open session to the decode kernels (bf16: HBM-bound GEMV + split-key attention;
 * at most 8 rows).  f32 engines keep the ordered SIMT kernels.  New (no reference
 * counterpart). */
kvp_status kvp_rank_set_decode(kvp_engine* e, int32_t on);

/* ------------------------------------------- fused KV handoff over peer memory */
/* The KV handoff of KVR (rank i -> i+1, engine.hpp:283-288) and the TSP all-gather
 * (engine.hpp:239-260) fused into the QKV projection: after kvp_rank_set_mirrors, the QKV
 * GEMM epilogue of every following kvp_rank_qkv stores this rank's K/V rows [start,
 * start+n_rows) ALSO into n_mirrors other buffers (other ranks' KV caches, mapped with
 * kvp_ipc_open: NVLink stores, tile by tile, while the projection runs).  mirror_bufs:
 * n_mirrors * 2*n_layers device pointers (per mirror the same K_0, V_0, K_1, ... layout as
 * kv_bufs of kvp_rank_begin); n_mirrors <= 8; bf16 only (f32 engines: KVP_ERR_CONFIG).
 * Cleared by kvp_rank_begin. */
kvp_status kvp_rank_set_mirrors(kvp_engine* e, int32_t n_mirrors, void* const* mirror_bufs);

/* Cross-process device memory (CUDA IPC): export the allocation holding dev_ptr as a
 * 64-byte handle plus dev_ptr's byte offset inside it; open a peer's handle in this process
 * (*dev_ptr = mapped base + offset); close a mapping opened with kvp_ipc_open. */
kvp_status kvp_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset);
kvp_status kvp_ipc_open(const void* handle64, int64_t offset, void** dev_ptr);
kvp_status kvp_ipc_close(void* dev_ptr, int64_t offset);

/* Stream-ordered 32-bit signals (the handoff's "message arrived" in device memory):
 * kvp_stream_signal writes value to *flag once all earlier work of the stream is done and
 * visible system-wide (flag may be a peer's memory); kvp_stream_wait holds the stream until
 * *flag >= value (flag in this device's memory, written by a peer).  kvp_stream_copy is an
 * async device copy on the stream (peer / IPC pointers allowed). */
kvp_status kvp_stream_signal(void* stream, void* flag, uint32_t value);
kvp_status kvp_stream_wait(void* stream, const void* flag, uint32_t value);
kvp_status kvp_stream_copy(void* stream, void* dst, const void* src, int64_t bytes);

/* ------------------------------------------- KV cache + decode */
/* The reference stops at the first token (engine.hpp:88); its natural consumer is a decode
 * step on the last rank's full KV cache.  A kvp_kv_cache owns per-layer K/V
 * device buffers of `capacity` rows; kvp_prefill_cached runs the single-rank prompt phase
 * into it (length := C; hidden_out C x d and first_token_hidden d floats are host, nullable)
 * and kvp_decode appends n_rows (<= 8) new rows at positions [length, length + n_rows)
 * attending to the whole cache (layer_qkv + layer_finish with offset = length), returning
 * their final hidden rows (host, n_rows x d). */
typedef struct kvp_kv_cache kvp_kv_cache;
kvp_status kvp_kv_cache_create(kvp_engine* e, int64_t capacity, kvp_kv_cache** out);
kvp_status kvp_kv_cache_destroy(kvp_kv_cache* c);
kvp_status kvp_kv_cache_length(const kvp_kv_cache* c, int64_t* length);
/* Truncate to `length` rows (e.g. to re-decode from an earlier position). */
kvp_status kvp_kv_cache_reset(kvp_kv_cache* c, int64_t length);
kvp_status kvp_prefill_cached(kvp_engine* e, kvp_kv_cache* c, const float* context, int64_t C, float* hidden_out,
                              float* first_token_hidden, float* ms);
kvp_status kvp_decode(kvp_engine* e, kvp_kv_cache* c, const float* rows, int64_t n_rows, float* out_rows,
                      float* ms);

/* ------------------------------------------- per-rank layer executor pieces */
/* layer_qkv (model.hpp:189-192): hidden rows x d -> Q rows x q, K/V rows x kv. */
kvp_status kvp_layer_qkv(kvp_engine* e, int64_t layer, const float* hidden, int64_t rows, float* Q,
                         float* K, float* V);
/* causal_attention (model.hpp:112-158) with CausalMask{offset, q_rows} (kv_cache.hpp:34). */
kvp_status kvp_causal_attention(kvp_engine* e, const float* Q, int64_t q_rows, const float* K,
                                const float* V, int64_t k_rows, int64_t offset, float* A);
/* layer_finish (model.hpp:164-175). */
kvp_status kvp_layer_finish(kvp_engine* e, int64_t layer, const float* hidden, int64_t rows,
                            const float* Q, const float* K, const float* V, int64_t k_rows,
                            int64_t offset, float* out);

/* Opt-in rotary position embedding (an extension: the reference model has no positional
 * encoding, so it is OFF by default and unavailable in the f32 parity mode).  theta > 0
 * enables it for bf16 engines with head_dim % 32 == 0: pairs (2i, 2i+1) of every Q and K
 * head of the token at absolute position t rotate by t * theta^(-2i/head_dim), fused into the
 * QKV projection epilogue (prefill, every strategy and rank, and decode); theta <= 0 disables.
 * The per-op helpers (kvp_layer_qkv) never apply it. */
kvp_status kvp_engine_set_rope(kvp_engine* e, double theta);

/* ------------------------------------------------ synthetic inputs */
/* random_context<float>(rows, d_model, seed) (weights.hpp:86-89): uniform [-1, 1) from the
 * SplitMix64 stream mix_seed(seed, 0xc7, 17) (rng.hpp:10-37), value = float((2u - 1) * 1.0)
 * computed in double -- bit-identical to the reference.  Host: out is rows x d_model f32. */
kvp_status kvp_random_context(int64_t rows, int64_t d_model, uint64_t seed, float* out);
/* Same values generated on devices[0] of the engine into a device buffer (the counter
 * generator runs one thread per element); synchronous. */
kvp_status kvp_random_context_device(kvp_engine* e, int64_t rows, uint64_t seed, float* out_dev);

/* ------------------------------------------------ partition plan (host) */
kvp_status kvp_validate_partition(int64_t C, const int64_t* boundaries, int64_t p);
/* even_partition (partition.hpp:59-69) */
kvp_status kvp_even_partition(int64_t C, int64_t p, int64_t* boundaries_out);
/* partition_from_ratios (partition.hpp:76-120) */
kvp_status kvp_partition_from_ratios(int64_t C, const double* ratios, int64_t p, int64_t* boundaries_out);
/* dot_product_counts / traffic_pairs (engine.hpp:95-121) */
kvp_status kvp_dot_product_counts(int32_t strategy, int64_t C, const int64_t* boundaries, int64_t p,
                                  int64_t* counts_out);
kvp_status kvp_traffic_pairs(int32_t strategy, int64_t C, const int64_t* boundaries, int64_t p,
                             int64_t* pairs_out);

/* ------------------------------------------- load balancer (host, bit-exact) */
/* simulate_ttft (simnet.hpp:164-278), quiet network. */
kvp_status kvp_simulate_ttft(int32_t strategy, int64_t C, const int64_t* boundaries, int64_t p,
                             int64_t n_layers, const kvp_cost_model* cost,
                             const kvp_network_model* net, double* ttft_out);
/* ttft_star (simnet.hpp:282-287) */
kvp_status kvp_ttft_star(int64_t C, int64_t p, double alpha, double* out);
/* calibrate_alpha (simnet.hpp:356-366) */
kvp_status kvp_calibrate_alpha(const int64_t* Cs, const double* times, int64_t n, double* alpha_out);
/* hierarchical_grid_search (search.hpp:156-207) / binary_search_two (search.hpp:92-150)
 * with a caller evaluator. */
kvp_status kvp_hierarchical_grid_search(int64_t C, int64_t p, const kvp_search_config* cfg,
                                        kvp_evaluator ev, void* user, int64_t* boundaries_out,
                                        kvp_search_result* res);
kvp_status kvp_binary_search_two(int64_t C, const kvp_search_config* cfg, kvp_evaluator ev,
                                 void* user, int64_t* boundaries_out, kvp_search_result* res);
/* The balancer proper (commands.hpp:252-278 Search branch): grid search scored by
 * simulate_ttft(KVR, .) under (cost, net) -- KVR-S. */
kvp_status kvp_search_partition(int64_t C, int64_t p, int64_t n_layers, const kvp_cost_model* cost,
                                const kvp_network_model* net, const kvp_search_config* cfg,
                                int64_t* boundaries_out, kvp_search_result* res);
/* practical_bound (simnet.hpp:297-316). */
kvp_status kvp_practical_bound(int64_t C, int64_t p, int64_t n_layers, const kvp_cost_model* cost,
                               int64_t* boundaries_out, double* ttft_out);
/* Extension (not in the reference): simulate_ttft with the attention term priced on the
 * CAUSAL-VISIBLE pairs the B200 kernels actually compute -- alpha * c_i * (b_i + (c_i+1)/2) for
 * both KVR and TSP (tile-skipping) -- instead of the reference's alpha*c_i*b_{i+1} (KVR) and
 * dense alpha*c_i*C (TSP).  Everything else (projection, softmax, wire, barriers) unchanged.
 * kvp_search_partition_causal = the grid search scored by it. */
kvp_status kvp_simulate_ttft_causal(int32_t strategy, int64_t C, const int64_t* boundaries, int64_t p,
                                    int64_t n_layers, const kvp_cost_model* cost, const kvp_network_model* net,
                                    double* ttft_out);
kvp_status kvp_search_partition_causal(int64_t C, int64_t p, int64_t n_layers, const kvp_cost_model* cost,
                                       const kvp_network_model* net, const kvp_search_config* cfg,
                                       int64_t* boundaries_out, kvp_search_result* res);
/* simulate_ttft with a NoiseSidecar{seed, slowdown_factor} (simnet.hpp:65-78,136-141). */
kvp_status kvp_simulate_ttft_noisy(int32_t strategy, int64_t C, const int64_t* boundaries, int64_t p,
                                   int64_t n_layers, const kvp_cost_model* cost, const kvp_network_model* net,
                                   uint64_t noise_seed, double slowdown_factor, double* ttft_out);
/* noise_study (simnet.hpp:332-353): per_trial (nullable) gets `trials` degradations. */
kvp_status kvp_noise_study(int32_t strategy, int64_t C, const int64_t* boundaries, int64_t p, int64_t n_layers,
                           const kvp_cost_model* cost, const kvp_network_model* net, double slowdown_factor,
                           int64_t trials, uint64_t seed, double* quiet_ttft, double* mean_degradation,
                           double* max_degradation, double* per_trial);
/* NoiseSidecar::degraded_link (simnet.hpp:71-75): the adjacent link (i -> i+1) a sidecar with
 * this seed slows in `layer`, -1 without links; noise_study's per-trial sidecar seed
 * mix_seed(seed, 0x7472, trial) (simnet.hpp:343).  Used by the physical sidecar of bench.py. */
kvp_status kvp_noise_degraded_link(uint64_t sidecar_seed, int64_t layer, int64_t link_count, int64_t* link_out);
kvp_status kvp_noise_trial_seed(uint64_t study_seed, int64_t trial, uint64_t* sidecar_seed_out);
/* KVR-P: PartitionLookupTable (lookup_table.hpp:22-39) given as n entries of
 * (context_lengths[i], ratios[i*p .. i*p+p)); interpolate_partition (lookup_table.hpp:44-64)
 * and partition_from_table (lookup_table.hpp:68-70). */
kvp_status kvp_interpolate_partition(const int64_t* context_lengths, const double* ratios, int64_t n, int64_t p,
                                     int64_t C, double* ratios_out);
kvp_status kvp_partition_from_table(const int64_t* context_lengths, const double* ratios, int64_t n, int64_t p,
                                    int64_t C, int64_t* boundaries_out);
/* Least-squares fit of CostModel{proj_coeff, alpha, softmax_coeff=0, fixed_overhead} from
 * measured per-layer times (new: the reference only fits alpha, simnet.hpp:356).
 * Samples i: local_rows[i], held_rows[i], proj_s[i] (norm+QKV seconds) and rest_s[i]
 * (attention..FFN seconds).  proj_coeff from proj_s ~ a*c; alpha/softmax/fixed from
 * rest_s ~ alpha*c*held + s*c + f (non-negative least squares). */
kvp_status kvp_fit_cost_model(const int64_t* local_rows, const int64_t* held_rows,
                              const double* proj_s, const double* rest_s, int64_t n,
                              kvp_cost_model* out);

#ifdef __cplusplus
}
#endif

#endif /* KVP_B200_H */
