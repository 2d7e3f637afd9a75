// gas.hpp — C++20 shim keeping the reference's operator surface (namespace gas, class and
// function names of /root/reference/proj/include/gas/*.hpp) on top of the C ABI in gasb.h.
//
// A reference maintainer swaps the host HistoryStore / Prefetcher / gas_epoch for these by
// including this header and linking libgasb.so. Semantics follow the
// reference; differences are listed per class. Errors: every gasb_status is rethrown as
// the reference's exception type, so the reference's error tests port as-is:
//   GASB_INVALID_ARGUMENT -> std::invalid_argument, GASB_LOGIC_ERROR -> std::logic_error,
//   GASB_RUNTIME_ERROR / GASB_CUDA_ERROR -> std::runtime_error.
#ifndef GASB_GAS_HPP
#define GASB_GAS_HPP

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../gasb.h"

namespace gas::b200 {

using NodeId = std::int32_t;

inline void check(gasb_status s) {
    switch (s) {
        case GASB_OK: return;
        case GASB_INVALID_ARGUMENT: throw std::invalid_argument(gasb_last_error());
        case GASB_LOGIC_ERROR: throw std::logic_error(gasb_last_error());
        default: throw std::runtime_error(gasb_last_error());
    }
}

// Same layout as gas::DenseMatrix (include/gas/matrix.hpp:13-30): row-major, dense.
struct DenseMatrix {
    std::int64_t rows = 0;
    std::int64_t cols = 0;
    std::vector<float> values;
    DenseMatrix() = default;
    DenseMatrix(std::int64_t r, std::int64_t c, float fill = 0.0f)
        : rows(r), cols(c), values(static_cast<std::size_t>(r * c), fill) {}
    float* row(std::int64_t r) { return values.data() + r * cols; }
    const float* row(std::int64_t r) const { return values.data() + r * cols; }
};

// Move-only owner of one gasb handle.
template <class H, gasb_status (*Destroy)(H)>
class Handle {
  public:
    Handle() = default;
    explicit Handle(H h) : h_(h) {}
    Handle(Handle&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Handle& operator=(Handle&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;
    ~Handle() { reset(); }
    H get() const { return h_; }

  private:
    void reset() {
        if (h_) Destroy(h_);
        h_ = nullptr;
    }
    H h_ = nullptr;
};

// gas::Graph + build_graph (include/gas/graph.hpp:46, src/graph.cpp:25-61): in-neighbour CSR,
// sorted, deduplicated, optionally symmetrized. Host-resident (the loader is host code).
class Graph {
  public:
    static Graph build(std::span<const NodeId> src, std::span<const NodeId> dst, NodeId num_nodes,
                       bool symmetrize = true) {
        if (src.size() != dst.size()) throw std::invalid_argument("build_graph: src/dst size mismatch");
        gasb_graph g = nullptr;
        check(gasb_graph_build(src.data(), dst.data(), static_cast<std::int64_t>(src.size()), num_nodes,
                               symmetrize ? 1 : 0, &g));
        return Graph(g);
    }
    NodeId num_nodes() const {
        std::int32_t n = 0;
        std::int64_t e = 0;
        check(gasb_graph_info(h_.get(), &n, &e));
        return n;
    }
    std::int64_t num_edges() const {
        std::int32_t n = 0;
        std::int64_t e = 0;
        check(gasb_graph_info(h_.get(), &n, &e));
        return e;
    }
    std::span<const std::int64_t> row_offsets() const {
        const std::int64_t* ro = nullptr;
        const std::int32_t* c = nullptr;
        check(gasb_graph_csr(h_.get(), &ro, &c));
        return {ro, static_cast<std::size_t>(num_nodes()) + 1};
    }
    std::span<const NodeId> cols() const {
        const std::int64_t* ro = nullptr;
        const std::int32_t* c = nullptr;
        check(gasb_graph_csr(h_.get(), &ro, &c));
        return {c, static_cast<std::size_t>(num_edges())};
    }
    gasb_graph raw() const { return h_.get(); }

  private:
    explicit Graph(gasb_graph g) : h_(g) {}
    Handle<gasb_graph, gasb_graph_destroy> h_;
};

// The per-part BatchPlan fields a caller reads (include/gas/graph.hpp:60-88).
struct BatchPlan {
    std::vector<NodeId> batch_nodes, extended_nodes, halo_nodes;
    std::vector<std::uint8_t> is_halo;
    std::vector<std::int32_t> batch_local_rows, halo_local_rows;
    // gcn stencil of build_plan_aggregation (src/layers.cpp:42-70)
    std::vector<std::int64_t> gcn_row_ptr;
    std::vector<NodeId> gcn_cols;
    std::vector<float> gcn_coeffs;
};

// cluster_partition (include/gas/partition.hpp, src/partition.cpp:344-388): the reference's
// multilevel partitioner, same assignment (host); random_partition (:330-342).
inline std::vector<std::int32_t> cluster_partition(const Graph& g, std::int32_t num_parts, std::uint64_t seed = 0) {
    std::vector<std::int32_t> a(static_cast<std::size_t>(g.num_nodes()));
    check(gasb_cluster_partition(g.raw(), num_parts, seed, a.data()));
    return a;
}
inline std::vector<std::int32_t> random_partition(NodeId num_nodes, std::int32_t num_parts, std::uint64_t seed = 0) {
    std::vector<std::int32_t> a(static_cast<std::size_t>(num_nodes));
    check(gasb_random_partition(num_nodes, num_parts, seed, a.data()));
    return a;
}

// BatchSchedule::build (include/gas/trainer.hpp:91-96, src/trainer.cpp:253-262): one plan +
// stencil per part of the partitioning, in part order. Plans stay host-side until a
// Trainer uploads them.
class BatchSchedule {
  public:
    // device = true: the GPU batch-plan builder on the current CUDA device (plan_dev.cu),
    // bit-identical plans
    static BatchSchedule build(const Graph& g, std::span<const std::int32_t> assignment, std::int32_t num_parts,
                               bool full = false, bool device = false) {
        if (static_cast<std::int64_t>(assignment.size()) != g.num_nodes())
            throw std::invalid_argument("BatchSchedule::build: assignment size != num_nodes");
        gasb_schedule s = nullptr;
        check(gasb_schedule_build(g.raw(), assignment.data(), num_parts,
                                  (full ? GASB_PLAN_FULL : 0) | (device ? GASB_PLAN_DEVICE : 0), &s));
        return BatchSchedule(s);
    }
    std::int32_t num_parts() const {
        std::int32_t p = 0;
        check(gasb_schedule_num_parts(h_.get(), &p));
        return p;
    }
    BatchPlan plan(std::int32_t part) const {
        std::int64_t sz[6];
        check(gasb_plan_sizes(h_.get(), part, sz));
        BatchPlan p;
        p.extended_nodes.resize(static_cast<std::size_t>(sz[1]));
        p.halo_nodes.resize(static_cast<std::size_t>(sz[2]));
        p.is_halo.resize(static_cast<std::size_t>(sz[1]));
        p.batch_local_rows.resize(static_cast<std::size_t>(sz[0]));
        p.halo_local_rows.resize(static_cast<std::size_t>(sz[2]));
        p.gcn_row_ptr.resize(static_cast<std::size_t>(sz[0]) + 1);
        p.gcn_cols.resize(static_cast<std::size_t>(sz[4]));
        p.gcn_coeffs.resize(static_cast<std::size_t>(sz[4]));
        check(gasb_plan_copy(h_.get(), part, p.extended_nodes.data(), p.halo_nodes.data(), p.is_halo.data(),
                             p.batch_local_rows.data(), p.halo_local_rows.data(), nullptr, nullptr,
                             p.gcn_row_ptr.data(), p.gcn_cols.data(), p.gcn_coeffs.data(), nullptr, nullptr,
                             nullptr));
        p.batch_nodes.reserve(p.batch_local_rows.size());
        for (std::int32_t r : p.batch_local_rows) p.batch_nodes.push_back(p.extended_nodes[static_cast<std::size_t>(r)]);
        return p;
    }
    gasb_schedule raw() const { return h_.get(); }

  private:
    explicit BatchSchedule(gasb_schedule s) : h_(s) {}
    Handle<gasb_schedule, gasb_schedule_destroy> h_;
};

// gas::HistoryStore (include/gas/history.hpp:29-66) with the tables in HBM.
// Host-span push/pull keep the reference's signatures and exceptions (ids validated on
// the host before any copy). *_device variants take device ids/rows and are stream-ordered.
// Difference: layer_matrix returns a host copy (the table itself lives in HBM; its device
// pointer is layer_device()).
class HistoryStore {
  public:
    HistoryStore(std::int32_t num_layers, NodeId num_nodes, std::int32_t dim) {
        gasb_history h = nullptr;
        check(gasb_history_create(num_layers, num_nodes, dim, &h));
        h_ = Handle<gasb_history, gasb_history_destroy>(h);
    }
    explicit HistoryStore(gasb_history adopted) { h_ = Handle<gasb_history, gasb_history_destroy>(adopted); }
    std::int32_t num_layers() const { return info().l; }
    NodeId num_nodes() const { return info().n; }
    std::int32_t dim() const { return info().d; }

    void push(std::int32_t layer, std::span<const NodeId> node_ids, std::span<const float> embeddings) {
        if (embeddings.size() != node_ids.size() * static_cast<std::size_t>(dim()))
            throw std::invalid_argument("HistoryStore::push: embeddings size != ids * dim");
        check(gasb_history_push_host(h_.get(), layer, node_ids.data(), static_cast<std::int64_t>(node_ids.size()),
                                     embeddings.data(), nullptr));
    }
    DenseMatrix pull(std::int32_t layer, std::span<const NodeId> node_ids) const {
        DenseMatrix out(static_cast<std::int64_t>(node_ids.size()), dim());
        check(gasb_history_pull_host(h_.get(), layer, node_ids.data(), static_cast<std::int64_t>(node_ids.size()),
                                     out.values.data(), nullptr));
        return out;
    }
    void push_device(std::int32_t layer, const NodeId* d_ids, std::int64_t count, const float* d_rows,
                     std::int64_t ld_rows, gasb_stream stream) {
        check(gasb_history_push(h_.get(), layer, d_ids, count, d_rows, ld_rows, stream));
    }
    void pull_device(std::int32_t layer, const NodeId* d_ids, std::int64_t count, float* d_out, std::int64_t ld_out,
                     gasb_stream stream) const {
        check(gasb_history_pull(h_.get(), layer, d_ids, count, d_out, ld_out, stream));
    }
    // Reports (and clears) an out-of-range id latched by a device push/pull.
    void check_ids() const { check(gasb_history_check(h_.get())); }

    DenseMatrix layer_matrix(std::int32_t layer) const {
        DenseMatrix m(num_nodes(), dim());
        check(gasb_history_read_layer(h_.get(), layer, m.values.data()));
        return m;
    }
    std::pair<float*, std::int64_t> layer_device(std::int32_t layer) const {
        float* p = nullptr;
        std::int64_t ld = 0;
        check(gasb_history_layer(h_.get(), layer, &p, &ld));
        return {p, ld};
    }
    void fill_layer(std::int32_t layer, const DenseMatrix& values) {
        if (values.rows != num_nodes() || values.cols != dim())
            throw std::invalid_argument("HistoryStore::fill_layer: shape mismatch");
        check(gasb_history_fill_layer(h_.get(), layer, values.values.data()));
    }
    void advance_step(gasb_stream stream = nullptr) { check(gasb_history_advance_step(h_.get(), stream)); }
    std::int64_t step() const {
        std::int64_t s = 0;
        check(gasb_history_step(h_.get(), &s));
        return s;
    }
    std::int64_t last_push_step(std::int32_t layer, NodeId v) const {
        std::int64_t s = 0;
        check(gasb_history_last_push_step(h_.get(), layer, v, &s));
        return s;
    }
    void reset() { check(gasb_history_reset(h_.get())); }
    // measure_staleness (history.cpp:77-112) against device reference tables, one per layer
    struct LayerStats {
        double eps_max = 0.0, eps_mean = 0.0;
        std::int64_t age_max = 0;
        double age_mean = 0.0;
    };
    std::vector<LayerStats> measure_staleness(std::span<const float* const> d_reference,
                                              std::span<const std::int64_t> ld_reference) const {
        const std::int32_t L = num_layers();
        if (static_cast<std::int32_t>(d_reference.size()) != L || ld_reference.size() != d_reference.size())
            throw std::invalid_argument("measure_staleness: need one reference matrix per layer");
        std::vector<double> emax(L), emean(L), amean(L);
        std::vector<std::int64_t> amax(L);
        check(gasb_history_staleness(h_.get(), d_reference.data(), ld_reference.data(), emax.data(), emean.data(),
                                     amax.data(), amean.data()));
        std::vector<LayerStats> r(static_cast<std::size_t>(L));
        for (std::int32_t l = 0; l < L; ++l) r[l] = {emax[l], emean[l], amax[l], amean[l]};
        return r;
    }
    // save_checkpoint / load_checkpoint (history.cpp:130-178), the reference's GASH format
    void save_checkpoint(const std::string& path) const { check(gasb_history_save(h_.get(), path.c_str())); }
    static HistoryStore load_checkpoint(const std::string& path) {
        gasb_history h = nullptr;
        check(gasb_history_load(path.c_str(), &h));
        return HistoryStore(h);
    }
    gasb_history raw() const { return h_.get(); }

  private:
    struct Info {
        std::int32_t l, n, d;
        std::int64_t ld;
    };
    Info info() const {
        Info i{};
        check(gasb_history_info(h_.get(), &i.l, &i.n, &i.d, &i.ld));
        return i;
    }
    Handle<gasb_history, gasb_history_destroy> h_;
};

// gas::Prefetcher / PrefetchHandle (include/gas/history.hpp:73-111) as stream work: begin()
// snapshots every layer's halo rows on a side stream ordered after `compute`; wait(layer)
// orders `compute` after that layer's copy and returns the device rows (valid until the
// next begin). Stale handles -> std::logic_error, bad layer -> std::invalid_argument.
class Prefetcher;
class PrefetchHandle {
  public:
    struct Rows {
        const float* data;
        std::int64_t ld;
    };
    Rows wait(std::int32_t layer, gasb_stream compute) const;

  private:
    friend class Prefetcher;
    gasb_prefetcher owner_ = nullptr;
    std::uint64_t generation_ = 0;
};

class Prefetcher {
  public:
    explicit Prefetcher(const HistoryStore& store) {
        gasb_prefetcher p = nullptr;
        check(gasb_prefetcher_create(store.raw(), &p));
        h_ = Handle<gasb_prefetcher, gasb_prefetcher_destroy>(p);
    }
    PrefetchHandle begin(const NodeId* d_halo, std::int64_t count, gasb_stream compute) {
        PrefetchHandle ph;
        ph.owner_ = h_.get();
        check(gasb_prefetch_begin(h_.get(), d_halo, count, compute, &ph.generation_));
        return ph;
    }

  private:
    Handle<gasb_prefetcher, gasb_prefetcher_destroy> h_;
};

inline PrefetchHandle::Rows PrefetchHandle::wait(std::int32_t layer, gasb_stream compute) const {
    if (!owner_) throw std::logic_error("PrefetchHandle::wait: handle not issued by a Prefetcher");
    Rows r{nullptr, 0};
    check(gasb_prefetch_wait(owner_, generation_, layer, compute, &r.data, &r.ld));
    return r;
}

// aggregate (src/tensor.cpp:514-549) and matmul (src/tensor.cpp:148-204) on device buffers.
inline void aggregate_forward(const std::int32_t* d_rowptr, std::int32_t num_dst, const NodeId* d_cols,
                              const float* d_coeffs, const float* d_x, std::int32_t num_src, std::int64_t ldx,
                              std::int32_t dim, float* d_y, std::int64_t ldy, std::int32_t seg_edges,
                              gasb_stream stream) {
    check(gasb_spmm_fwd(d_rowptr, num_dst, d_cols, d_coeffs, d_x, num_src, ldx, dim, d_y, ldy, seg_edges, stream));
}
inline void aggregate_backward(const std::int32_t* d_t_rowptr, std::int32_t num_targets, const std::int32_t* d_t_src,
                               const float* d_t_coeffs, const float* d_gy, std::int64_t ldgy, std::int32_t num_src,
                               std::int32_t dim, const float* d_mask, std::int64_t ldm, float* d_gx,
                               std::int64_t ldgx, gasb_stream stream) {
    check(gasb_spmm_bwd(d_t_rowptr, num_targets, d_t_src, d_t_coeffs, d_gy, ldgy, num_src, dim, d_mask, ldm, d_gx,
                        ldgx, stream));
}
// max / mean neighbourhood aggregation (north_star's sum/mean/max SpMM; no reference
// counterpart, semantics fixed in gasb.h): forward with argmax, backward by argmax.
inline void aggregate_max_forward(const std::int32_t* d_rowptr, std::int32_t num_dst, const NodeId* d_cols,
                                  const float* d_x, std::int32_t num_src, std::int64_t ldx, std::int32_t dim,
                                  float* d_y, std::int64_t ldy, std::int32_t* d_argmax, std::int64_t ld_arg,
                                  gasb_stream stream) {
    check(gasb_spmm_max_fwd(d_rowptr, num_dst, d_cols, d_x, num_src, ldx, dim, d_y, ldy, d_argmax, ld_arg, stream));
}
inline void aggregate_max_backward(const std::int32_t* d_rowptr, std::int32_t num_dst, const NodeId* d_cols,
                                   const std::int32_t* d_argmax, std::int64_t ld_arg, const float* d_gy,
                                   std::int64_t ldgy, std::int32_t num_src, std::int32_t dim, float* d_gx,
                                   std::int64_t ldgx, gasb_stream stream) {
    check(gasb_spmm_max_bwd(d_rowptr, num_dst, d_cols, d_argmax, ld_arg, d_gy, ldgy, num_src, dim, d_gx, ldgx,
                            stream));
}
inline void aggregate_mean_forward(const std::int32_t* d_rowptr, std::int32_t num_dst, const NodeId* d_cols,
                                   const float* d_x, std::int32_t num_src, std::int64_t ldx, std::int32_t dim,
                                   float* d_y, std::int64_t ldy, gasb_stream stream) {
    check(gasb_spmm_mean_fwd(d_rowptr, num_dst, d_cols, d_x, num_src, ldx, dim, d_y, ldy, stream));
}
// float(1/deg) per edge: aggregate_backward with these coefficients is the mean's backward
inline std::vector<float> mean_coefficients(const std::vector<std::int32_t>& rowptr) {
    std::vector<float> c(rowptr.empty() ? 0 : static_cast<std::size_t>(rowptr.back()));
    check(gasb_mean_coefficients(rowptr.data(), static_cast<std::int32_t>(rowptr.size()) - 1, c.data()));
    return c;
}
enum class MatmulOp : std::int32_t { NN = 0, NT = 1, TN = 2 };
inline void matmul(MatmulOp op, std::int32_t m, std::int32_t n, std::int32_t k, const float* d_a, std::int64_t lda,
                   const float* d_b, std::int64_t ldb, float* d_c, std::int64_t ldc, bool accumulate,
                   gasb_stream stream) {
    check(gasb_gemm(static_cast<std::int32_t>(op), m, n, k, d_a, lda, d_b, ldb, d_c, ldc, accumulate ? 1.f : 0.f,
                    stream));
}

// AdamState::step / grad_clip (include/gas/nn.hpp:21-41) on device buffers.
inline void adam_step(float* d_params, float* d_m, float* d_v, const float* d_grads, std::int64_t size,
                      std::int64_t step, float lr = 0.01f, float beta1 = 0.9f, float beta2 = 0.999f,
                      float eps = 1e-8f, gasb_stream stream = nullptr) {
    check(gasb_adam_step(d_params, d_m, d_v, d_grads, size, step, lr, beta1, beta2, eps, stream));
}
inline double grad_clip(float* d_grads, std::int64_t size, double max_norm, gasb_stream stream = nullptr) {
    double n = 0.0;
    check(gasb_grad_clip(d_grads, size, max_norm, &n, stream));
    return n;
}

// Layer (include/gas/layers.hpp:51-72) over one batch plan: LayerContext{plan, agg} is a
// BatchOps (the plan's device stencils); forward / backward take device buffers
// (h_in |V_b| x in_dim, h0 for APPNP / GCNII, W, out |B_b| x out_dim; the backward
// ACCUMULATES into the gradient buffers, as the reference's tape does).
struct LayerConfig : gasb_layer_config {
    LayerConfig(std::int32_t kind, std::int32_t in_dim, std::int32_t out_dim, float alpha = 0.1f, float beta = 0.5f)
        : gasb_layer_config{kind, in_dim, out_dim, alpha, beta} {}
};
class BatchOps {
  public:
    BatchOps(gasb_schedule schedule, std::int32_t part, std::int32_t max_dim) {
        gasb_batch_ops b = nullptr;
        check(gasb_batch_ops_create(schedule, part, max_dim, &b));
        h_ = Handle<gasb_batch_ops, gasb_batch_ops_destroy>(b);
        check(gasb_batch_ops_sizes(b, &nb_, &ne_));
    }
    std::int32_t num_batch() const { return nb_; }
    std::int32_t num_extended() const { return ne_; }
    void forward(const LayerConfig& c, const float* h_in, std::int64_t ld_in, const float* h0, std::int64_t ld_h0,
                 const float* w, std::int64_t ld_w, float* out, std::int64_t ld_out, float* saved,
                 std::int64_t ld_saved, gasb_stream stream = nullptr) const {
        check(gasb_layer_fwd(h_.get(), &c, h_in, ld_in, h0, ld_h0, w, ld_w, out, ld_out, saved, ld_saved, stream));
    }
    void backward(const LayerConfig& c, const float* gy, std::int64_t ld_gy, const float* saved, std::int64_t ld_saved,
                  const float* w, std::int64_t ld_w, float* gh_in, std::int64_t ld_gh_in, float* gh0,
                  std::int64_t ld_gh0, float* gw, std::int64_t ld_gw, float* scratch, std::int64_t ld_scratch,
                  gasb_stream stream = nullptr) const {
        check(gasb_layer_bwd(h_.get(), &c, gy, ld_gy, saved, ld_saved, w, ld_w, gh_in, ld_gh_in, gh0, ld_gh0, gw, ld_gw,
                             scratch, ld_scratch, stream));
    }

  private:
    Handle<gasb_batch_ops, gasb_batch_ops_destroy> h_;
    std::int32_t nb_ = 0, ne_ = 0;
};

// EpochReport (include/gas/trainer.hpp:107-115); batch_peak_floats is the device step's
// activation floats (gasb.h), not the reference's CPU activation_meter.
struct EpochReport {
    std::int64_t epoch = 0;
    double loss = 0.0;
    std::int64_t peak_floats = 0;
    std::vector<std::int64_t> batch_peak_floats;
    std::vector<double> eps_max;
    std::int64_t edges_per_layer = 0;
    std::int64_t device_bytes = 0;
};

// Model + AdamState + HistoryStore + gas_epoch (include/gas/trainer.hpp:45-126) as one
// device-resident training context. gas_epoch has EpochOptions{evaluate=false,
// measure_staleness=false} semantics and returns EpochReport.loss.
struct ModelSpec : gasb_model_spec {
    ModelSpec() : gasb_model_spec{0, 2, 16, 0.f, 0.1f, 0.5f, 0.f, 0.f, 0.01f, 0.9f, 0.999f, 1e-8f, 0} {}
};
struct TrainerOptions : gasb_trainer_options {
    TrainerOptions() : gasb_trainer_options{128, 1, 0, 1, 1, 0, GASB_DROPOUT_EXACT} {}
};

class Trainer {
  public:
    Trainer(const BatchSchedule& schedule, std::span<const float> features, std::int32_t in_dim,
            std::span<const std::int32_t> labels, std::span<const std::uint8_t> train_mask, std::int32_t num_classes,
            const ModelSpec& spec, const TrainerOptions& opt = TrainerOptions()) {
        if (labels.size() != train_mask.size() || features.size() != labels.size() * static_cast<std::size_t>(in_dim))
            throw std::invalid_argument("Trainer: features/labels/train_mask sizes disagree");
        gasb_trainer t = nullptr;
        check(gasb_trainer_create(schedule.raw(), features.data(), in_dim, labels.data(), train_mask.data(),
                                  num_classes, &spec, &opt, &t));
        h_ = Handle<gasb_trainer, gasb_trainer_destroy>(t);
    }
    double gas_epoch(std::int64_t epoch, bool shuffle = true) {
        double loss = 0.0;
        check(gasb_gas_epoch(h_.get(), epoch, shuffle ? 1 : 0, &loss));
        return loss;
    }
    // gas_epoch with the EpochReport fields; measure_staleness runs the frozen snapshot pass
    EpochReport gas_epoch_report(std::int64_t epoch, std::int32_t num_parts, std::int32_t history_layers,
                                 bool shuffle = true, bool measure_staleness = false) {
        gasb_epoch_report r{};
        EpochReport out;
        out.batch_peak_floats.resize(static_cast<std::size_t>(num_parts));
        out.eps_max.resize(static_cast<std::size_t>(history_layers > 0 ? history_layers : 0));
        check(gasb_gas_epoch_report(h_.get(), epoch, shuffle ? 1 : 0, measure_staleness ? 1 : 0, &r,
                                    out.batch_peak_floats.data(), out.eps_max.empty() ? nullptr : out.eps_max.data()));
        out.epoch = r.epoch;
        out.loss = r.loss;
        out.peak_floats = r.peak_floats;
        out.edges_per_layer = r.edges_per_layer;
        out.device_bytes = r.device_bytes;
        out.batch_peak_floats.resize(static_cast<std::size_t>(r.num_batches));
        out.eps_max.resize(static_cast<std::size_t>(r.staleness_layers));
        return out;
    }
    std::vector<float> params() const {
        std::int64_t n = 0;
        check(gasb_trainer_num_param_floats(h_.get(), &n));
        std::vector<float> p(static_cast<std::size_t>(n));
        check(gasb_trainer_get_params(h_.get(), p.data()));
        return p;
    }
    void set_params(std::span<const float> p) { check(gasb_trainer_set_params(h_.get(), p.data())); }
    // evaluate (trainer.cpp:444-464): full-batch accuracy over host masks (nullptr = 0)
    struct Accuracy {
        double train = 0.0, val = 0.0, test = 0.0;
    };
    Accuracy evaluate(const std::uint8_t* train_mask, const std::uint8_t* val_mask,
                      const std::uint8_t* test_mask) {
        double a[3] = {0.0, 0.0, 0.0};
        check(gasb_trainer_evaluate(h_.get(), train_mask, val_mask, test_mask, a));
        return {a[0], a[1], a[2]};
    }
    // infer_from_history (trainer.cpp:501-536)
    struct InferenceResult {
        std::vector<std::int32_t> predictions;
        bool stale = false;
    };
    InferenceResult infer_from_history(NodeId num_nodes) {
        InferenceResult r;
        r.predictions.resize(static_cast<std::size_t>(num_nodes));
        std::int32_t st = 0;
        check(gasb_trainer_infer_from_history(h_.get(), r.predictions.data(), &st));
        r.stale = st != 0;
        return r;
    }
    gasb_trainer raw() const { return h_.get(); }

  private:
    Handle<gasb_trainer, gasb_trainer_destroy> h_;
};

// Data-parallel epochs over the GPUs of one node (no reference counterpart; csrc/dp.cu):
// one process per GPU; the caller all-gathers export() from every rank (any transport)
// and passes the concatenation to connect(). Replicas stay bit-identical.
class DataParallel {
  public:
    // placement: GASB_DP_REPLICATED or GASB_DP_SHARDED (partition-sharded histories, gasb.h)
    DataParallel(Trainer& t, std::int32_t rank, std::int32_t world, std::int32_t placement = GASB_DP_REPLICATED) {
        gasb_dp d = nullptr;
        check(gasb_dp_create_ex(t.raw(), rank, world, placement, &d));
        h_ = Handle<gasb_dp, gasb_dp_destroy>(d);
    }
    // sharded placement: one history layer gathered from every rank's shard
    DenseMatrix history_layer(std::int32_t layer, NodeId num_nodes, std::int32_t dim) const {
        DenseMatrix m(num_nodes, dim);
        check(gasb_dp_read_history(h_.get(), layer, m.values.data()));
        return m;
    }
    std::vector<std::uint8_t> export_handle() const {
        std::vector<std::uint8_t> h(GASB_DP_HANDLE_BYTES);
        check(gasb_dp_export(h_.get(), h.data()));
        return h;
    }
    void connect(std::span<const std::uint8_t> all_handles) { check(gasb_dp_connect(h_.get(), all_handles.data())); }
    // enqueues one epoch (every rank calls it); check() synchronizes and reports barrier timeouts
    void epoch_async(std::int64_t epoch, bool shuffle = true) { check(gasb_dp_epoch_async(h_.get(), epoch, shuffle)); }
    void check_done() const { check(gasb_dp_check(h_.get())); }
    // per-part losses of the parts this rank ran (0 elsewhere): sum over ranks for all parts
    std::vector<double> part_losses(std::int32_t num_parts) const {
        std::vector<double> l(static_cast<std::size_t>(num_parts));
        check(gasb_dp_last_losses(h_.get(), l.data()));
        return l;
    }

  private:
    Handle<gasb_dp, gasb_dp_destroy> h_;
};

}  // namespace gas::b200

#endif  // GASB_GAS_HPP
