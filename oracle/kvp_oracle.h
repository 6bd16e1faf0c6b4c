/*
 * kvp_oracle.h -- CPU restatement of the KV-Runahead reference (kvprefill) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the B200 product
 * in paper_2405_05329_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never links it.
 *
 * Every function restates one reference function operation-for-operation (same
 * accumulation order, same element type), so the f32/f64 results are bit-identical to
 * the reference compiled from /root/reference (checked in tests/test_oracle_pinned.py
 * against oracle/_ref and against tests/golden/*.json).  Citations are relative to
 * /root/reference/proj/include/kvprefill/.
 */
#ifndef KVP_ORACLE_H
#define KVP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: one per exception type in errors.hpp:8-46 (same numbering as the
 * product C-ABI in include/kvp_b200.h). */
enum {
    KVO_OK = 0,
    KVO_CONFIG = 1,
    KVO_DIMENSION = 2,
    KVO_CACHE = 3,
    KVO_INPUT = 4,
    KVO_PARTITION = 5,
    KVO_PROTOCOL = 6,
    KVO_ASSEMBLY = 7,
    KVO_LOOKUP = 8,
    KVO_SEARCH = 9,
    KVO_BUDGET = 10,
    KVO_CALIBRATION = 11,
    KVO_IO = 12
};

/* ModelConfig (config.hpp:22-47).  precision is informational here: the caller picks
 * the _f32 / _f64 entry point. */
typedef struct {
    int64_t d_model, n_heads, n_kv_heads, n_layers;
    uint64_t seed;
    int32_t precision; /* 0 f32, 1 f64 */
    int32_t rms_norm;
} kvo_config;

/* CostModel (simnet.hpp:27-44) and NetworkModel (simnet.hpp:48-63). */
typedef struct { double alpha, proj_coeff, softmax_coeff, fixed_overhead; } kvo_cost;
typedef struct { double bandwidth, latency; } kvo_net;

/* Strategy (engine.hpp:21). */
enum { KVO_SERIAL = 0, KVO_TSP = 1, KVO_KVR = 2 };

int kvo_validate_config(const kvo_config* c);

/* rng.hpp:10-37 */
uint64_t kvo_splitmix_next(uint64_t* state);
uint64_t kvo_mix_seed(uint64_t base, uint64_t a, uint64_t b);

/* weights.hpp:41-89.  Fills the six matrices of one layer (row-major, [in x out]). */
int kvo_layer_weights_f32(const kvo_config* c, int64_t layer, float* wq, float* wk, float* wv,
                          float* wo, float* w1, float* w2);
int kvo_layer_weights_f64(const kvo_config* c, int64_t layer, double* wq, double* wk, double* wv,
                          double* wo, double* w1, double* w2);
void kvo_random_context_f32(float* out, int64_t rows, int64_t d_model, uint64_t seed);
void kvo_random_context_f64(double* out, int64_t rows, int64_t d_model, uint64_t seed);
void kvo_seeded_matrix_f32(float* out, int64_t rows, int64_t cols, double scale, uint64_t stream);

/* Model core (model.hpp).  `weights` is 6*n_layers pointers: wq,wk,wv,wo,w1,w2 per layer. */
int kvo_layer_qkv_f32(const kvo_config* c, const float* const* weights, int64_t layer,
                      const float* hidden, int64_t rows, float* Q, float* K, float* V);
int kvo_layer_qkv_f64(const kvo_config* c, const double* const* weights, int64_t layer,
                      const double* hidden, int64_t rows, double* Q, double* K, double* V);
int kvo_causal_attention_f32(const kvo_config* c, const float* Q, int64_t q_rows, const float* K,
                             const float* V, int64_t k_rows, int64_t offset, float* A);
int kvo_causal_attention_f64(const kvo_config* c, const double* Q, int64_t q_rows, const double* K,
                             const double* V, int64_t k_rows, int64_t offset, double* A);
int kvo_layer_finish_f32(const kvo_config* c, const float* const* weights, int64_t layer,
                         const float* hidden, int64_t rows, const float* Q, const float* K,
                         const float* V, int64_t k_rows, int64_t offset, float* out);
int kvo_layer_finish_f64(const kvo_config* c, const double* const* weights, int64_t layer,
                         const double* hidden, int64_t rows, const double* Q, const double* K,
                         const double* V, int64_t k_rows, int64_t offset, double* out);
/* forward_serial (model.hpp:197-211).  kv_out (optional) receives per layer K then V,
 * each [C x kv_dim], layer-major. */
int kvo_forward_serial_f32(const kvo_config* c, const float* const* weights, const float* context,
                           int64_t C, float* hidden_out, float* kv_out);
int kvo_forward_serial_f64(const kvo_config* c, const double* const* weights, const double* context,
                           int64_t C, double* hidden_out, double* kv_out);
/* naive_causal_forward (oracle.hpp:34-111): independent f64 brute force. */
int kvo_naive_forward_f64(const kvo_config* c, const double* const* weights, const double* context,
                          int64_t C, double* hidden_out);

/* partition.hpp */
int kvo_validate_partition(int64_t C, const int64_t* boundaries, int64_t p);
int kvo_even_partition(int64_t C, int64_t p, int64_t* boundaries_out);
int kvo_partition_from_ratios(int64_t C, const double* ratios, int64_t p, int64_t* boundaries_out);
double kvo_table_build_cost(double T, int64_t N, int64_t C, int64_t grid_width);

/* engine.hpp:95-121 accounting */
int kvo_dot_product_counts(int strategy, int64_t C, const int64_t* boundaries, int64_t p,
                           int64_t* counts_out);
int kvo_traffic_pairs(int strategy, int64_t C, const int64_t* boundaries, int64_t p,
                      int64_t* pairs_out);

/* simnet.hpp:164-366 */
int kvo_simulate_ttft(int strategy, int64_t C, const int64_t* boundaries, int64_t p,
                      int64_t n_layers, const kvo_cost* cost, const kvo_net* net, double* ttft_out);
int kvo_ttft_star(int64_t C, int64_t p, double alpha, double* out);
int kvo_calibrate_alpha(const int64_t* Cs, const double* ts, int64_t n, double* alpha_out);

/* search.hpp:166-207 and oracle.hpp:117-158 */
typedef double (*kvo_evaluator)(const int64_t* boundaries, int64_t p, void* ctx);
typedef struct {
    int64_t grid_width, initial_stride, min_stride;
} kvo_search_config;
typedef struct {
    double ttft;
    int64_t evaluations, levels;
} kvo_search_result;
int kvo_hierarchical_grid_search(int64_t C, int64_t p, const kvo_search_config* cfg,
                                 kvo_evaluator ev, void* ctx, int64_t* boundaries_out,
                                 kvo_search_result* res);
int kvo_binary_search_two(int64_t C, const kvo_search_config* cfg, kvo_evaluator ev, void* ctx,
                          int64_t* boundaries_out, kvo_search_result* res);
int kvo_exhaustive_partition_search(int64_t C, int64_t p, kvo_evaluator ev, void* ctx,
                                    int64_t budget, int64_t* boundaries_out, kvo_search_result* res);
int64_t kvo_resolve_initial_stride(const kvo_search_config* cfg, int64_t C, int64_t p);

/* Convenience evaluator: simulate_ttft(KVR, part, model, cost, net).ttft
 * (the evaluator commands.hpp:558-562 builds).  ctx -> kvo_sim_ctx. */
typedef struct {
    int64_t n_layers;
    kvo_cost cost;
    kvo_net net;
    int strategy;
} kvo_sim_ctx;
double kvo_sim_evaluator(const int64_t* boundaries, int64_t p, void* ctx);
int kvo_practical_bound(int64_t C, int64_t p, int64_t n_layers, const kvo_cost* cost,
                        int64_t* boundaries_out, double* ttft_out);

#ifdef __cplusplus
}
#endif

#endif
