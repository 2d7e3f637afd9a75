/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the GAS training hot path.
 *
 * A plain-C restatement of the reference's algorithms (GNNAutoScale CPU re-creation,
 * /root/reference/proj). Every function cites the reference file:line it restates.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. The product (paper_2106_05609_b200/) never links or calls it.
 *
 * Parity of this restatement is PINNED against the reference itself: tests/test_oracle_pin.py
 * compares it with oracle/_ref/libref.so (the reference sources compiled in place) and with
 * the committed fixtures in tests/golden/ generated from that build.
 */
#ifndef GAS_ORACLE_H
#define GAS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- include/gas/rng.hpp ---------------------------------------------------------- */
uint64_t go_mix64(uint64_t x);                                           /* rng.hpp:11-16 */
uint64_t go_derive_seed(uint64_t s, uint64_t a, uint64_t b, uint64_t c); /* rng.hpp:18-21 */
void go_glorot(int64_t rows, int64_t cols, uint64_t seed, float* out);   /* nn.cpp:65-70 */
void go_epoch_order(int32_t nb, uint64_t model_seed, int64_t epoch, int32_t* out); /* trainer.cpp:395-400 */

/* ---- src/graph.cpp:25-61  build_graph ------------------------------------------------
 * row_offsets: caller array of n+1. *cols_out: malloc'd, free with go_free. Returns 0 or
 * 1 (invalid argument: negative n / edge out of range). */
int go_build_graph(const int32_t* u, const int32_t* v, int64_t m, int32_t n, int symmetrize,
                   int64_t* row_offsets, int32_t** cols_out, int64_t* nnz_out);
void go_free(void* p);

/* ---- src/graph.cpp:78-134 make_batch_plan + src/layers.cpp:42-70 build_plan_aggregation */
typedef struct {
    int32_t nb, next, nhalo;
    int32_t* batch;             /* nb, sorted global ids */
    int32_t* extended;          /* next, sorted global ids */
    int32_t* halo;              /* nhalo */
    uint8_t* is_halo;           /* next */
    int32_t* batch_local_rows;  /* nb */
    int32_t* halo_local_rows;   /* nhalo */
    int64_t* local_rowptr;      /* next+1 */
    int32_t* local_cols;
    int64_t* gcn_rowptr;        /* nb+1 */
    int32_t* gcn_cols;          /* local ids */
    float* gcn_coeffs;
    int64_t* sum_rowptr;        /* nb+1 */
    int32_t* sum_cols;
    float* sum_coeffs;
} go_plan;

/* 0 ok, 1 invalid argument (empty / unsorted / out-of-range batch). */
int go_plan_make(int32_t n, const int64_t* row_offsets, const int32_t* cols, const int32_t* batch,
                 int64_t nb, go_plan* out);
void go_plan_free(go_plan* p);

/* ---- src/tensor.cpp ops ------------------------------------------------------------- */
void go_aggregate_fwd(const int64_t* rowptr, int64_t m, const int32_t* cols, const float* coeffs,
                      const float* x, int64_t d, float* y);                 /* tensor.cpp:514-530 */
void go_aggregate_bwd(const int64_t* rowptr, int64_t m, const int32_t* cols, const float* coeffs,
                      const float* gy, int64_t d, float* gx);               /* tensor.cpp:531-549 (accumulates) */
void go_matmul_fwd(const float* a, int64_t m, int64_t k, const float* b, int64_t n, float* y); /* :148-167 */
void go_matmul_bwd(const float* a, const float* b, const float* gy, int64_t m, int64_t k, int64_t n,
                   float* ga, float* gb);                                  /* :169-204 (accumulates) */
/* Returns the float loss; accumulates d loss/d logits into glogits when non-null. :597-647 */
float go_softmax_ce(const float* logits, int64_t m, int64_t n, const int32_t* rows, const int32_t* labels,
                    int64_t r, float* glogits);

/* ---- src/nn.cpp --------------------------------------------------------------------- */
typedef struct { float lr, beta1, beta2, eps; } go_adam_cfg;
/* One AdamState::step (nn.cpp:20-41) for one tensor at step t (1-based). */
void go_adam_step(float* p, float* m, float* v, const float* g, int64_t size, int64_t t, go_adam_cfg cfg);
double go_grad_clip(float* g, int64_t size, double max_norm);              /* nn.cpp:47-63 */

/* ---- src/trainer.cpp: GAS session (Model::build, Model::forward, run_batch, gas_epoch) */
typedef struct {
    int32_t kind;  /* 0 gcn (restated); 2 appnp, 3 gcnii restated in go_session too */
    int32_t num_layers, hidden;
    float dropout, alpha, beta, l2_weight, clip_max_norm;
    float lr, beta1, beta2, eps;
    uint64_t seed;
} go_spec;

typedef struct go_session go_session;

/* 0 ok, 1 invalid argument. Inputs are copied. Only dropout == 0 is restated. */
int go_session_create(int32_t n, const int64_t* row_offsets, const int32_t* cols, const float* features,
                      int32_t in_dim, const int32_t* labels, const uint8_t* train_mask, int32_t num_classes,
                      const int32_t* assignment, int32_t num_parts, const go_spec* spec, go_session** out);
void go_session_free(go_session* s);
int64_t go_session_num_param_floats(const go_session* s);
void go_session_get_params(const go_session* s, float* out);
void go_session_set_params(go_session* s, const float* in);
int32_t go_session_history_dim(const go_session* s);
void go_session_get_history(const go_session* s, int32_t layer, float* out);
void go_session_set_history(go_session* s, int32_t layer, const float* in);
int64_t go_session_store_step(const go_session* s);
/* Same contract as ref_session_batch in ref_harness.cpp. */
int go_session_batch(go_session* s, int32_t part, int64_t epoch, int train, int push, float* acts,
                     float* logits, double* loss, float* grads, int* stepped);
/* One gas_epoch; *loss = mean batch loss. */
int go_session_epoch(go_session* s, int64_t epoch, int shuffle, double* loss);
/* data-parallel GAS step semantics (gas_oracle.c). k = 1 == go_session_epoch. */
int go_session_dp_batch(go_session* s, int32_t part, float* grads_out, float* acts_out, double* loss, int* stepped);
void go_session_dp_commit(go_session* s, int32_t part, const float* acts);
void go_session_dp_apply(go_session* s, const float* grad_sum, int32_t count, int32_t batches);
int go_session_dp_epoch(go_session* s, int64_t epoch, int shuffle, int32_t k, double* loss);

/* ---- bench input generator (same streams as gasb_synth_pairs / gasb_synth_features) -- */
int go_synth_pairs(int32_t n, int32_t communities, int64_t num_pairs, double intra_fraction, double gamma,
                   double min_weight, double max_weight, uint64_t seed, int32_t* src, int32_t* dst,
                   int32_t* community);
void go_synth_features(int64_t n, int32_t dim, int64_t ld, uint64_t seed, float* out);

#ifdef __cplusplus
}
#endif
#endif
