/* gasb.h — C ABI of the B200-native GNNAutoScale (GAS) training hot path.
 *
 * This is the drop-in boundary: libgasb.so exports exactly these `extern "C"` entry points
 * (plain pointers, sizes and status codes; no C++ or torch types). Each entry point names
 * the reference interface it replaces (/root/reference/proj, file:line). The C++ shim that
 * keeps the reference's class names on top of this ABI is include/gasb/gas.hpp; a
 * reference-side binding is shown in INTEGRATION.md.
 *
 * Conventions
 *  - Every call returns gasb_status. Exceptions never cross the ABI; the message of the last
 *    failure on the calling thread is gasb_last_error(). Status values map 1:1 onto the
 *    reference's exception types: INVALID_ARGUMENT = std::invalid_argument,
 *    LOGIC_ERROR = std::logic_error, RUNTIME_ERROR = std::runtime_error.
 *  - `d_` pointers are device (HBM) pointers, `h_` pointers host pointers. Device calls are
 *    stream-ordered on the given stream (NULL = legacy default stream) and asynchronous
 *    unless stated otherwise.
 *  - Layers are 1-based as in the reference (history layer l feeds layer l+1).
 *  - Handles own their HBM; nothing is freed across the ABI except by *_destroy.
 */
#ifndef GASB_H
#define GASB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* gasb_stream; /* cudaStream_t */

typedef enum {
    GASB_OK = 0,
    GASB_INVALID_ARGUMENT = 1,
    GASB_LOGIC_ERROR = 2,
    GASB_RUNTIME_ERROR = 3,
    GASB_CUDA_ERROR = 4
} gasb_status;

const char* gasb_last_error(void);
int32_t gasb_abi_version(void);

/* ==================================================================================== */
/* graph-core: include/gas/graph.hpp                                                     */
/* ==================================================================================== */
typedef struct gasb_graph_s* gasb_graph;

/* build_graph (include/gas/graph.hpp:46, src/graph.cpp:25-61): CSR of in-neighbours, rows
 * sorted and deduplicated, reverse edges added when symmetrize != 0, self-loops kept once.
 * Host arrays; OpenMP-parallel; result is the reference's canonical CSR bit for bit. */
gasb_status gasb_graph_build(const int32_t* h_src, const int32_t* h_dst, int64_t num_edges,
                             int32_t num_nodes, int32_t symmetrize, gasb_graph* out);
/* Adopts a CSR (validated: monotone offsets, sorted unique in-range rows). */
gasb_status gasb_graph_from_csr(int32_t num_nodes, const int64_t* h_row_offsets, const int32_t* h_cols,
                                int32_t symmetric, gasb_graph* out);
gasb_status gasb_graph_info(gasb_graph g, int32_t* num_nodes, int64_t* num_edges);
/* Borrowed host pointers, valid until gasb_graph_destroy. */
gasb_status gasb_graph_csr(gasb_graph g, const int64_t** h_row_offsets, const int32_t** h_cols);
gasb_status gasb_graph_destroy(gasb_graph g);

/* Synthetic power-law graph with planted communities (SURVEY §8d "Synthetic inputs"):
 * node weights w ~ Pareto(gamma) clipped to [min_weight, max_weight]; communities are a
 * seeded balanced random split; each of num_pairs undirected pairs picks u ~ w globally,
 * then v ~ w inside u's community with probability intra_fraction, else v ~ w globally.
 * Counter-based RNG per pair: output independent of thread count. Outputs host arrays
 * (num_pairs each) and the community of every node. */
typedef struct {
    int32_t num_nodes;
    int32_t num_communities;
    int64_t num_pairs;
    double intra_fraction;
    double gamma;
    double min_weight;
    double max_weight;
    uint64_t seed;
} gasb_synth_params;
gasb_status gasb_synth_pairs(const gasb_synth_params* p, int32_t* h_src, int32_t* h_dst, int32_t* h_community);
/* N(0,1) fp32 features (Box-Muller over a counter-based stream), rows padded to ld with 0. */
gasb_status gasb_synth_features(int64_t num_nodes, int32_t dim, int64_t ld, uint64_t seed, float* h_out);

/* ==================================================================================== */
/* partition-batch loader: make_batch_plan (graph.hpp:88, graph.cpp:78-134),              */
/* build_plan_aggregation (layers.hpp:38, layers.cpp:42-70), BatchSchedule::build         */
/* (trainer.hpp:91-96, trainer.cpp:253-262)                                              */
/* ==================================================================================== */
typedef struct gasb_schedule_s* gasb_schedule;

/* Plans every part of `assignment` (part ids in [0, num_parts), every part non-empty).
 * flags & GASB_PLAN_FULL also materializes plan.local_graph and the `sum` stencil (only
 * needed for parity checks / GIN); the GCN stencil and node lists are always built. */
#define GASB_PLAN_FULL 1
/* flags & GASB_PLAN_DEVICE builds every plan on the current CUDA device (GPU batch-plan
 * builder: part x node bitmaps + popcount scans, bit-exact with the host
 * builder) and copies the results into the schedule; same errors. */
#define GASB_PLAN_DEVICE 2
gasb_status gasb_schedule_build(gasb_graph g, const int32_t* h_assignment, int32_t num_parts, int32_t flags,
                                gasb_schedule* out);
/* Build timing: device_ms = GPU time of the device builder (-1 for host builds), total_ms =
 * wall time of gasb_schedule_build (inputs, kernels and copies into the host plans). */
gasb_status gasb_schedule_timing(gasb_schedule s, double* device_ms, double* total_ms);
/* Single plan for an explicit sorted batch (make_batch_plan semantics and errors). */
gasb_status gasb_schedule_build_batches(gasb_graph g, const int32_t* const* h_batches, const int64_t* sizes,
                                        int32_t num_batches, int32_t flags, gasb_schedule* out);
gasb_status gasb_schedule_num_parts(gasb_schedule s, int32_t* out);
/* sizes[6] = {num_batch, num_extended, num_halo, local_nnz, gcn_nnz, sum_nnz} */
gasb_status gasb_plan_sizes(gasb_schedule s, int32_t part, int64_t* sizes);
/* Copies plan arrays into caller host buffers (any may be NULL). Layouts as BatchPlan. */
gasb_status gasb_plan_copy(gasb_schedule s, int32_t part, int32_t* extended, int32_t* halo, uint8_t* is_halo,
                           int32_t* batch_local_rows, int32_t* halo_local_rows, int64_t* local_rowptr,
                           int32_t* local_cols, int64_t* gcn_rowptr, int32_t* gcn_cols, float* gcn_coeffs,
                           int64_t* sum_rowptr, int32_t* sum_cols, float* sum_coeffs);
gasb_status gasb_schedule_destroy(gasb_schedule s);
/* save_partition / load_partition (io.hpp:40-41, io.cpp:187-217): the reference's
 * "node part" text format (# comments, blank lines); load validates as
 * partition_from_assignment (partition.cpp:314-328) and reports num_parts = max part + 1. */
gasb_status gasb_partition_save(const char* path, const int32_t* h_assignment, int32_t num_nodes);
gasb_status gasb_partition_load(const char* path, int32_t num_nodes, int32_t* h_assignment, int32_t* num_parts);
/* random_partition (partition.hpp:23, partition.cpp:330-342), bit-exact (seeded shuffle). */
gasb_status gasb_random_partition(int32_t num_nodes, int32_t num_parts, uint64_t seed, int32_t* h_assignment);
/* cluster_partition (partition.hpp, partition.cpp:344-388): the reference's multilevel
 * partitioner (heavy-edge matching, greedy growth, boundary refinement, balance repair),
 * restated with sparse per-node connectivity and a one-pass balance repair: the SAME
 * assignment as the reference for the same graph, part count and seed, far faster. Host. */
gasb_status gasb_cluster_partition(gasb_graph g, int32_t num_parts, uint64_t seed, int32_t* h_assignment);

/* ==================================================================================== */
/* history-store: HistoryStore (include/gas/history.hpp:29-66, src/history.cpp:10-178)   */
/* L-1 fp32 tables of num_nodes x dim in HBM (row pitch ld >= dim, 16 B aligned), zero-   */
/* initialized; int64 last-push stamps (-1 = never pushed); a device step counter.        */
/* ==================================================================================== */
typedef struct gasb_history_s* gasb_history;

gasb_status gasb_history_create(int32_t num_layers, int32_t num_nodes, int32_t dim, gasb_history* out);
gasb_status gasb_history_destroy(gasb_history h);
gasb_status gasb_history_info(gasb_history h, int32_t* num_layers, int32_t* num_nodes, int32_t* dim, int64_t* ld);
/* HistoryStore::push (history.cpp:28-42): table[d_ids[i]] = d_rows[i*ld_rows : +dim],
 * stamp = current step. Ids are checked on device; an out-of-range id skips its row and
 * latches an error that the next synchronizing call (gasb_history_check) reports as
 * INVALID_ARGUMENT, the reference's exception for the same input. */
gasb_status gasb_history_push(gasb_history h, int32_t layer, const int32_t* d_ids, int64_t count,
                              const float* d_rows, int64_t ld_rows, gasb_stream stream);
/* HistoryStore::pull (history.cpp:44-55): d_out[i*ld_out : +dim] = table[d_ids[i]]. */
gasb_status gasb_history_pull(gasb_history h, int32_t layer, const int32_t* d_ids, int64_t count, float* d_out,
                              int64_t ld_out, gasb_stream stream);
/* Host-buffer variants: ids validated on the host first (exception-exact), then H2D/D2H
 * copies through pinned staging on `stream`; synchronous on return. */
gasb_status gasb_history_push_host(gasb_history h, int32_t layer, const int32_t* h_ids, int64_t count,
                                   const float* h_rows, gasb_stream stream);
gasb_status gasb_history_pull_host(gasb_history h, int32_t layer, const int32_t* h_ids, int64_t count,
                                   float* h_out, gasb_stream stream);
/* Synchronizes and reports (then clears) the device-side id check latched by push/pull. */
gasb_status gasb_history_check(gasb_history h);
gasb_status gasb_history_advance_step(gasb_history h, gasb_stream stream); /* advance_step() */
gasb_status gasb_history_step(gasb_history h, int64_t* out);               /* step() (syncs) */
gasb_status gasb_history_last_push_step(gasb_history h, int32_t layer, int32_t v, int64_t* out);
/* layer_matrix (history.cpp:57-60): borrowed device pointer + row pitch. */
gasb_status gasb_history_layer(gasb_history h, int32_t layer, float** d_table, int64_t* ld);
/* fill_layer (history.cpp:61-67) from host values (num_nodes x dim, dense). */
gasb_status gasb_history_fill_layer(gasb_history h, int32_t layer, const float* h_values);
gasb_status gasb_history_read_layer(gasb_history h, int32_t layer, float* h_values);
gasb_status gasb_history_read_stamps(gasb_history h, int32_t layer, int64_t* h_stamps);
gasb_status gasb_history_reset(gasb_history h); /* reset() (history.cpp:114-118) */
/* measure_staleness (history.hpp:51, history.cpp:77-112): per layer l (index l-1), against
 * the device reference matrix d_reference[l-1] (num_nodes x dim, pitch ld_reference[l-1]):
 * eps = per-row L2 distance (max, mean), age = steps since the row's last push (never
 * pushed: step + 1; max, mean). Row norms on the GPU, ordered sums on the host: bit-exact
 * with the reference. Synchronous. */
gasb_status gasb_history_staleness(gasb_history h, const float* const* d_reference, const int64_t* ld_reference,
                                   double* h_eps_max, double* h_eps_mean, int64_t* h_age_max, double* h_age_mean);
/* save_checkpoint / load_checkpoint (history.hpp:55-56, history.cpp:130-178): the
 * reference's GASH file format (magic, u32 layers/nodes/dim, dense fp32 tables), so a
 * checkpoint written by either side loads in the other. load creates a new store with
 * every stamp 0 and step 0, as the reference. */
gasb_status gasb_history_save(gasb_history h, const char* path);
gasb_status gasb_history_load(const char* path, gasb_history* out);

/* Prefetcher / PrefetchHandle (history.hpp:73-111, history.cpp:184-252) as stream work:
 * begin() snapshots all L-1 layers' halo rows on the prefetcher's side stream after an
 * event recorded on `compute`; wait(layer) makes `compute` wait for that layer's copy and
 * returns the device buffer (valid until the next begin). A stale generation is a
 * LOGIC_ERROR, an out-of-range layer an INVALID_ARGUMENT, as in the reference. */
typedef struct gasb_prefetcher_s* gasb_prefetcher;
gasb_status gasb_prefetcher_create(gasb_history h, gasb_prefetcher* out);
gasb_status gasb_prefetcher_destroy(gasb_prefetcher p);
gasb_status gasb_prefetch_begin(gasb_prefetcher p, const int32_t* d_halo, int64_t count, gasb_stream compute,
                                uint64_t* generation);
gasb_status gasb_prefetch_wait(gasb_prefetcher p, uint64_t generation, int32_t layer, gasb_stream compute,
                               const float** d_rows, int64_t* ld);

/* ==================================================================================== */
/* message-passing ops (src/tensor.cpp)                                                  */
/* ==================================================================================== */
/* aggregate forward (tensor.cpp:514-530): y[r,:] = sum_e coeffs[e] * x[cols[e],:],
 * e in [rowptr[r], rowptr[r+1]); fp64 accumulation, rounded to fp32.
 * seg_edges == 0: one warp per row in CSR order -> bit-exact with the reference.
 * seg_edges  > 0: rows split into segments of <= seg_edges edges whose fp64 partials are
 * combined in segment order (deterministic; differs from sequential fp64 only below fp32
 * resolution). Device int32 rowptr (relative), int32 cols into x's num_src rows. */
gasb_status gasb_spmm_fwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols, const float* d_coeffs,
                          const float* d_x, int32_t num_src, int64_t ldx, int32_t dim, float* d_y, int64_t ldy,
                          int32_t seg_edges, gasb_stream stream);
/* aggregate backward closure (tensor.cpp:531-549) restricted to the given targets, as a
 * gather over the transposed stencil: gx[t,:] = sum over (r, c) in CSC row t, r ascending,
 * of c * gy[r,:] with fp32 multiply-then-add -> bit-exact. Optional mask: gx[t,j] = 0
 * where d_mask[t*ldm + j] <= 0 (fused relu backward, tensor.cpp:363-369). */
gasb_status gasb_spmm_bwd(const int32_t* d_t_rowptr, int32_t num_targets, const int32_t* d_t_src,
                          const float* d_t_coeffs, const float* d_gy, int64_t ldgy, int32_t num_src, int32_t dim,
                          const float* d_mask, int64_t ldm, float* d_gx, int64_t ldgx, gasb_stream stream);
/* max and mean aggregation (north_star 3: sum/mean/max SpMM) over the same CSR stencils
 * (device int32 rowptr starting at 0, int32 cols into x's num_src rows). The reference has
 * only weighted sums (aggregate, tensor.cpp:514-549), so these are pinned to their
 * definitions (oracle/aggregators.py), not to a reference function:
 *  max_fwd : y[r,j] = the first edge's x[c,j], replaced in CSR order by any strictly greater
 *            value; d_argmax[r,j] (optional) = that edge's index; empty rows give 0 and -1;
 *  max_bwd : gx[s,j] = fp32 sum over rows r ascending of gy[r,j] for the edges (r -> s) that
 *            are argmax[r,j] (deterministic; overwrites gx's num_src rows);
 *  mean_fwd: y[r,j] = float(fp64 CSR-order sum of x[c,j] / deg r), 0 for an empty row;
 *  mean backward = gasb_spmm_bwd with the coefficients gasb_mean_coefficients writes
 *            (float(1.0 / deg r) per edge, host arrays).
 * Range errors raise the reference's aggregate message (tensor.cpp:515). */
gasb_status gasb_spmm_max_fwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols, const float* d_x,
                              int32_t num_src, int64_t ldx, int32_t dim, float* d_y, int64_t ldy, int32_t* d_argmax,
                              int64_t ld_arg, gasb_stream stream);
gasb_status gasb_spmm_max_bwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols,
                              const int32_t* d_argmax, int64_t ld_arg, const float* d_gy, int64_t ldgy,
                              int32_t num_src, int32_t dim, float* d_gx, int64_t ldgx, gasb_stream stream);
gasb_status gasb_spmm_mean_fwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols, const float* d_x,
                               int32_t num_src, int64_t ldx, int32_t dim, float* d_y, int64_t ldy,
                               gasb_stream stream);
gasb_status gasb_mean_coefficients(const int32_t* h_rowptr, int32_t num_dst, float* h_coeffs);
/* matmul (tensor.cpp:148-204) on fp32 row-major operands, fp32 accumulation:
 * op = 0: C = A[m,k] B[k,n]; 1: C = A[m,k] B[n,k]^T; 2: C = A[k,m]^T B[k,n].
 * beta == 0 overwrites C, beta == 1 accumulates. */
gasb_status gasb_gemm(int32_t op, int32_t m, int32_t n, int32_t k, const float* d_a, int64_t lda, const float* d_b,
                      int64_t ldb, float* d_c, int64_t ldc, float beta, gasb_stream stream);

/* AdamState::step (nn.hpp:21-38, nn.cpp:20-41) on one flat parameter tensor: `step` is the
 * step count t after the increment (1-based); bias corrections 1 - beta^t via host
 * std::pow, moment/update math in fp64 with the reference's rounding sequence -> bit-exact
 * with the reference given identical gradients and state. Synchronous. */
gasb_status gasb_adam_step(float* d_params, float* d_m, float* d_v, const float* d_grads, int64_t size, int64_t step,
                           float lr, float beta1, float beta2, float eps, gasb_stream stream);
/* grad_clip (nn.hpp:41, nn.cpp:47-63): global L2 norm in fp64; if norm > max_norm every
 * gradient is multiplied by float(max_norm / norm). *h_norm = the pre-clip norm (its fp64
 * sum runs in a fixed tree order, not the reference's sequential order). max_norm <= 0 is
 * INVALID_ARGUMENT. Synchronous. */
gasb_status gasb_grad_clip(float* d_grads, int64_t size, double max_norm, double* h_norm, gasb_stream stream);

/* ==================================================================================== */
/* layer-level ops: Layer::forward and its tape backward (layers.hpp:51-72,               */
/* layers.cpp:120-168) over one batch plan, for callers with their own Model::forward     */
/* ==================================================================================== */
/* One plan's device stencils (gcn stencil over local ids with segment tables, its
 * transpose over every extended row, batch_local_rows), built once from the schedule;
 * layers up to max_dim wide. */
typedef struct gasb_batch_ops_s* gasb_batch_ops;
gasb_status gasb_batch_ops_create(gasb_schedule s, int32_t part, int32_t max_dim, gasb_batch_ops* out);
gasb_status gasb_batch_ops_sizes(gasb_batch_ops b, int32_t* num_batch, int32_t* num_extended);
gasb_status gasb_batch_ops_destroy(gasb_batch_ops b);
/* LayerConfig (layers.hpp:17-27) without GIN: kind 0 GCN, 2 APPNP, 3 GCNII. */
typedef struct {
    int32_t kind;
    int32_t in_dim, out_dim;
    float alpha, beta;
} gasb_layer_config;
/* Layer::forward (LayerContext{plan, agg, h_in, h0}, layers.hpp:40-45): h_in is |V_b| x
 * in_dim in the plan's extended-node order (halo rows included), h0 (APPNP / GCNII) |V_b| x
 * out_dim, W in_dim x out_dim (GCN, GCNII). out = |B_b| x out_dim. d_saved (|B_b| x in_dim)
 * receives what the backward needs (GCN: the aggregation; GCNII: the mixed rows). The
 * aggregation is the exact-fp64 SpMM; mixing and W~ = (1-beta) I + beta W follow the
 * reference's rounding sequence. Stream-ordered, capturable. Same errors as the reference
 * ("APPNP: missing h0", dimension checks). */
gasb_status gasb_layer_fwd(gasb_batch_ops b, const gasb_layer_config* cfg, const float* d_h_in, int64_t ld_in,
                           const float* d_h0, int64_t ld_h0, const float* d_w, int64_t ld_w, float* d_out,
                           int64_t ld_out, float* d_saved, int64_t ld_saved, gasb_stream stream);
/* The tape backward of that forward given gy = d loss / d out (|B_b| x out_dim): ACCUMULATES
 * into gh_in (|V_b| x in_dim, every extended row, tensor.cpp:531-549), gh0 (|V_b| x out_dim,
 * batch rows, APPNP / GCNII) and gW (in_dim x out_dim, GCN / GCNII); NULL outputs are
 * skipped. d_scratch: |B_b| x max(in_dim, out_dim). Stream-ordered, capturable. */
gasb_status gasb_layer_bwd(gasb_batch_ops b, const gasb_layer_config* cfg, const float* d_gy, int64_t ld_gy,
                           const float* d_saved, int64_t ld_saved, const float* d_w, int64_t ld_w, float* d_gh_in,
                           int64_t ld_gh_in, float* d_gh0, int64_t ld_gh0, float* d_gw, int64_t ld_gw,
                           float* d_scratch, int64_t ld_scratch, gasb_stream stream);

/* ==================================================================================== */
/* gas-trainer: Model (trainer.hpp:45-88), gas_epoch (trainer.hpp:124-126,               */
/* trainer.cpp:386-442), run_batch (trainer.cpp:295-339), AdamState (nn.hpp:21-38)       */
/* ==================================================================================== */
typedef struct {
    int32_t kind; /* 0 GCN, 2 APPNP, 3 GCNII (LayerKind order, layers.hpp:12) */
    int32_t num_layers;
    int32_t hidden;
    float dropout, alpha, beta, l2_weight, clip_max_norm;
    float lr, beta1, beta2, eps;
    uint64_t seed;
} gasb_model_spec;

typedef struct {
    int32_t seg_edges;     /* SpMM row segmentation (0 = bit-exact sequential rows) */
    int32_t fused;         /* 1: pull-free SpMM reads histories in place (default);
                              0: reference-structured pull + compose (materialized halos) */
    int32_t prefetch;      /* materialized mode: pull batch b+1's halos on a side stream */
    int32_t use_graphs;    /* capture each batch into a CUDA graph */
    int32_t hoist_layer1;  /* compute layer-1 aggregation of all batches up front per epoch */
    int32_t device;        /* CUDA device ordinal */
    int32_t dropout_rng;   /* ModelSpec.dropout > 0 (tensor.cpp:374-401): the keep-mask stream.
                              GASB_DROPOUT_EXACT: the reference's own, Rng(derive_seed(seed ^
                              "drop", epoch, part, slot)).next_double() >= p element by element
                              (host mt19937_64, copied per batch) -> bit-exact, host-bound;
                              GASB_DROPOUT_PHILOX: Philox4x32-10 on the device keyed by the same
                              derive_seed value -> same keep rate, different masks, no host work */
    int32_t cross_batch;   /* the paper's concurrent execution across batches (GCN, fused,
                              segmented, no dropout; gas_epoch only). 0: off. 1: batch b+1's
                              halo aggregation (every history layer: the in-edges from rows
                              outside V_b+1, which only earlier batches' pushes write) runs on a
                              background stream while batch b runs its backward and Adam; the
                              batch's own forward aggregates only its intra-batch edges and adds
                              the halo fp64 partial. 2: as 1, and batch b+1's layer-1
                              aggregation also runs per batch on the background stream (instead
                              of the up-front hoisted launch), overlapped with batch b. Same
                              results up to fp64 summation order (the segmented mode's class). */
} gasb_trainer_options;
#define GASB_DROPOUT_EXACT 0
#define GASB_DROPOUT_PHILOX 1

typedef struct gasb_trainer_s* gasb_trainer;

/* Uploads features (n x in_dim host fp32), the schedule's stencils and labels to HBM and
 * builds the model (Model::build, trainer.cpp:55-129: seeded Glorot init identical to the
 * reference), AdamState and HistoryStore(L-1, n, history_dim). */
gasb_status gasb_trainer_create(gasb_schedule s, const float* h_features, int32_t in_dim, const int32_t* h_labels,
                                const uint8_t* h_train_mask, int32_t num_classes, const gasb_model_spec* spec,
                                const gasb_trainer_options* opt, gasb_trainer* out);
gasb_status gasb_trainer_destroy(gasb_trainer t);
/* gas_epoch with EpochOptions{evaluate=false, measure_staleness=false}: seeded batch order
 * (trainer.cpp:395-400), one optimizer step per batch with training rows, advance_step per
 * batch. Synchronous; *mean_loss as EpochReport.loss. */
gasb_status gasb_gas_epoch(gasb_trainer t, int64_t epoch, int32_t shuffle, double* mean_loss);
/* Enqueue-only variant for timing: no host synchronization, losses stay on device. */
gasb_status gasb_gas_epoch_async(gasb_trainer t, int64_t epoch, int32_t shuffle);
/* The batches order[begin, end) of gas_epoch's seeded order for `epoch` (same kernels,
 * graphs and hoisting as gasb_gas_epoch_async; end == num_parts is the whole epoch). */
gasb_status gasb_gas_epoch_range_async(gasb_trainer t, int64_t epoch, int32_t shuffle, int32_t begin, int32_t end);
/* Per-part batch objective (num_parts doubles, part order) as last computed: the loss of
 * every batch with training rows that ran (synchronizes). */
gasb_status gasb_trainer_part_losses(gasb_trainer t, double* h_losses);
/* EpochReport (trainer.hpp:107-115) of one gas_epoch (EpochOptions{evaluate = false}):
 *  loss            mean batch objective (as gasb_gas_epoch);
 *  edges_per_layer sum over batches of plan.local_graph.num_edges() (stored in-edges of the
 *                  batch rows), exactly as the reference;
 *  peak_floats / h_batch_peak_floats (num_parts, epoch order): the activation floats each
 *                  batch's device step writes (forward agg_l / act_l / logits and their
 *                  gradients over the batch rows). This stands in for the reference's
 *                  activation_meter (tensor.cpp:12-25), which counts its CPU tensors: the fused
 *                  path materializes no V_b-row tensors, so the figure is linear in L and in
 *                  B_b (SPEC A8), not equal to the reference's;
 *  device_bytes    HBM the trainer holds (free-memory drop since its construction);
 *  measure_staleness != 0: the frozen snapshot pass (gas_forward_snapshot, no push, no step)
 *                  then measure_staleness (trainer.cpp:434-438): h_eps_max[L-1], per layer. */
typedef struct {
    int64_t epoch;
    double loss;
    int64_t peak_floats;
    int64_t edges_per_layer;
    int64_t device_bytes;
    int32_t num_batches;
    int32_t staleness_layers; /* L - 1 when measured, else 0 */
} gasb_epoch_report;
gasb_status gasb_gas_epoch_report(gasb_trainer t, int64_t epoch, int32_t shuffle, int32_t measure_staleness,
                                  gasb_epoch_report* out, int64_t* h_batch_peak_floats, double* h_eps_max);
/* The keep mask of dropout slot `layer` (the layer-`layer` input, V_b x d_{layer-1} elements,
 * row-major; bit i % 32 of word i / 32) that batch `part` uses in `epoch`, under the
 * trainer's dropout_rng. LOGIC_ERROR when dropout == 0. Synchronous. */
gasb_status gasb_trainer_dropout_mask(gasb_trainer t, int32_t part, int64_t epoch, int32_t layer, uint32_t* h_words);
/* Mean loss of the last epoch enqueued with gasb_gas_epoch_async (synchronizes). */
gasb_status gasb_trainer_last_loss(gasb_trainer t, double* mean_loss);
/* One batch with capture (same contract as the oracle's session_batch): acts = pushed rows
 * per history layer ((L-1) x nb x hist_dim), logits nb x C, grads = flat pre-clip
 * parameter gradients in Model::params() order. Synchronous. */
gasb_status gasb_trainer_batch(gasb_trainer t, int32_t part, int64_t epoch, int32_t train, int32_t push,
                               float* h_acts, float* h_logits, double* loss, float* h_grads, int32_t* stepped);
gasb_status gasb_trainer_num_param_floats(gasb_trainer t, int64_t* out);
gasb_status gasb_trainer_get_params(gasb_trainer t, float* h_out);
gasb_status gasb_trainer_set_params(gasb_trainer t, const float* h_in);
gasb_status gasb_trainer_history(gasb_trainer t, gasb_history* out); /* borrowed */
gasb_status gasb_trainer_stream(gasb_trainer t, gasb_stream* out);
/* Replaces the device feature matrix from host memory (n x in_dim, dense), stream-ordered
 * on the trainer's stream (asynchronous when h_features is pinned, see gasb_host_register). */
gasb_status gasb_trainer_set_features(gasb_trainer t, const float* h_features);
/* set_features in two halves, so a step's input copy overlaps the previous step's compute:
 * stage = asynchronous H2D (pinned h_features) on the trainer's copy stream after the last
 * commit consumed the staging buffer; commit = the trainer's stream waits for the staged copy
 * and installs it as X. set_features == stage + commit. */
gasb_status gasb_trainer_stage_features(gasb_trainer t, const float* h_features);
gasb_status gasb_trainer_commit_features(gasb_trainer t);
/* Times `iters` back-to-back launches of one SpMM of the training step with CUDA events on
 * the trainer's stream: part >= 0 -> the per-batch aggregation of `layer` for that part;
 * part < 0 -> the hoisted whole-epoch layer-1 aggregation. Writes only scratch buffers. */
gasb_status gasb_trainer_profile_spmm(gasb_trainer t, int32_t part, int32_t layer, int32_t iters, float* avg_ms);
/* Page-locks host memory for asynchronous copies (cudaHostRegister / Unregister). */
gasb_status gasb_host_register(void* h_ptr, size_t bytes);
gasb_status gasb_host_unregister(void* h_ptr);
/* evaluate (trainer.hpp:131, trainer.cpp:444-464): the model's full-batch forward over
 * every node (BatchSchedule::full_batch: no halos) with the current parameters; acc3 =
 * fraction of each mask's nodes (train, val, test; host uint8[n], NULL = 0) whose argmax
 * logit (first maximum, nn.cpp:117-122) equals the label. GCN; synchronous. */
gasb_status gasb_trainer_evaluate(gasb_trainer t, const uint8_t* h_train, const uint8_t* h_val, const uint8_t* h_test,
                                  double* acc3);
/* Logits (n x C, global node order) of the last evaluate / infer_from_history. */
gasb_status gasb_trainer_full_logits(gasb_trainer t, float* h_logits);
/* infer_from_history (trainer.hpp:150, trainer.cpp:501-536): one final-layer application
 * over the layer-(L-1) histories for every node; predictions (argmax, n) and stale = some
 * layer-(L-1) row was never pushed. GCN; synchronous. */
gasb_status gasb_trainer_infer_from_history(gasb_trainer t, int32_t* h_predictions, int32_t* stale);
/* Kernel launches per epoch (counted by the host driver while enqueueing). */
gasb_status gasb_trainer_launch_count(gasb_trainer t, int64_t* out);

/* ==================================================================================== */
/* data-parallel training over k GPUs of one node (no reference counterpart: */
/* the reference is single-process). One process per GPU. A step runs k consecutive      */
/* batches of gas_epoch's seeded order (trainer.cpp:395-400), rank j the j-th, against    */
/* start-of-step parameters and histories; pushes are committed to every replica after    */
/* the step; gradients are summed in rank order over the batches with training rows,      */
/* divided by their count, clipped and applied once (oracle: go_session_dp_epoch).        */
/* Exchange over peer memory: each rank exports one HBM region (CUDA IPC handle); peers   */
/* map it (NVLink P2P) and read gradients and pushed rows directly.                       */
/* ==================================================================================== */
#define GASB_DP_HANDLE_BYTES 64
typedef struct gasb_dp_s* gasb_dp;
/* Turns a trainer into rank `rank` of `world` (1..8): allocates the exchange region and
 * makes the trainer's gradient and pushed-row buffers views into it. */
gasb_status gasb_dp_create(gasb_trainer t, int32_t rank, int32_t world, gasb_dp* out);
/* History placement of a data-parallel group.
 * REPLICATED: every rank keeps the whole HistoryStore; a step's pushed rows are committed
 *   into every replica (graphs whose tables fit one GPU: C3 716 MB).
 * SHARDED: partition p's rows belong to rank p mod world; each rank keeps only its rows
 *   (L-1 layers x its nodes, in its exported region; the trainer's full tables are freed).
 *   Batches pull their halo rows from the owners' shards (NVLink P2P loads) into the
 *   reference-structured compose -> SpMM path and push nothing; after the step barrier every
 *   rank commits the step's rows it owns from all ranks' act slots. Same step semantics,
 *   so the result is bit-identical to REPLICATED (C5: 2 x 111M x 256 tables need it). */
#define GASB_DP_REPLICATED 0
#define GASB_DP_SHARDED 1
gasb_status gasb_dp_create_ex(gasb_trainer t, int32_t rank, int32_t world, int32_t placement, gasb_dp* out);
/* This rank's region handle (GASB_DP_HANDLE_BYTES), to be all-gathered by the caller. */
gasb_status gasb_dp_export(gasb_dp d, uint8_t* h_handle);
/* Maps every peer's region from the gathered handles (world x GASB_DP_HANDLE_BYTES). */
gasb_status gasb_dp_connect(gasb_dp d, const uint8_t* h_handles);
/* Enqueues one data-parallel epoch on the trainer's stream (all ranks must call it). */
gasb_status gasb_dp_epoch_async(gasb_dp d, int64_t epoch, int32_t shuffle);
/* Synchronizes; a cross-rank barrier that timed out is a RUNTIME_ERROR. */
gasb_status gasb_dp_check(gasb_dp d);
/* Per-part losses of the last epoch for the parts THIS rank ran (0 elsewhere): summing
 * the arrays over ranks gives every part's loss exactly. Synchronizes. */
gasb_status gasb_dp_last_losses(gasb_dp d, double* h_losses);
gasb_status gasb_dp_launch_count(gasb_dp d, int64_t* out);
/* SHARDED: gathers history layer `layer` (n x hist_dim, host) from every rank's shard
 * (synchronizes; the trainer's own HistoryStore raises logic_error once its tables are
 * sharded). */
gasb_status gasb_dp_read_history(gasb_dp d, int32_t layer, float* h_out);
/* Bytes of the last epoch: NVLink = peer gradient slots read by the reduce + peer act rows
 * read by the commits + (sharded) halo rows read from peer shards; local_pull = halo rows
 * this rank read from its own shard; shard_rows = history rows this rank holds per layer. */
gasb_status gasb_dp_traffic(gasb_dp d, int64_t* nvlink_bytes, int64_t* local_pull_bytes, int64_t* shard_rows);
/* The SHARDED row ownership (host): owner_local[v] = owner << 29 | row in the owner's
 * shard (n entries), rows_per_rank[world]. */
gasb_status gasb_dp_shard_map(gasb_schedule s, int32_t world, uint32_t* h_owner_local, int64_t* h_rows_per_rank);
gasb_status gasb_dp_destroy(gasb_dp d);
/* gas_epoch's batch order (trainer.cpp:395-400) for `epoch` (host only). */
gasb_status gasb_epoch_order(int32_t num_parts, uint64_t seed, int64_t epoch, int32_t shuffle, int32_t* h_order);

#ifdef __cplusplus
}
#endif
#endif /* GASB_H */
