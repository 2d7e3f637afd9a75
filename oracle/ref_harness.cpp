// TEST INFRASTRUCTURE ONLY. C-ABI harness over the UNMODIFIED reference library
// (/root/reference/proj, compiled in place by oracle/Makefile into _ref/libref.so).
//
// It exposes the reference's own public API (include/gas/*.hpp) to ctypes so that the
// tests can (1) pin the C restatement in oracle/gas_oracle.c against the real thing and
// (2) serve as `cpu_baseline.kind = "reference"` in bench.py. Nothing in the product
// (paper_2106_05609_b200/) links or loads this file.
//
// run_batch is file-local in the reference (src/trainer.cpp:295-339), so ref_session_batch
// reconstructs it from the public API: Model::forward + softmax_cross_entropy (+ l2_penalty)
// + Tape::backward + grad_clip + AdamState::step + HistoryStore::advance_step, in the same
// order as gas_epoch (src/trainer.cpp:386-442).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "gas/graph.hpp"
#include "gas/history.hpp"
#include "gas/io.hpp"
#include "gas/layers.hpp"
#include "gas/nn.hpp"
#include "gas/partition.hpp"
#include "gas/rng.hpp"
#include "gas/tensor.hpp"
#include "gas/trainer.hpp"

using namespace gas;

namespace {
thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 logic_error, 3 runtime_error / other
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

struct RefSpec {
    std::int32_t kind;  // 0 gcn, 1 gin, 2 appnp, 3 gcnii
    std::int32_t num_layers;
    std::int32_t hidden;
    float dropout, alpha, beta, l2_weight, clip_max_norm;
    float lr, beta1, beta2, eps;
    std::uint64_t seed;
};

struct Session {
    Dataset ds;
    BatchSchedule sched;
    std::vector<std::int32_t> sched_parts;  // part id of each schedule slot
    std::optional<Model> model;
    std::optional<AdamState> opt;
    HistoryStore store;
    std::optional<Prefetcher> prefetcher;
};

LayerKind to_kind(std::int32_t k) {
    switch (k) {
        case 0: return LayerKind::kGcn;
        case 1: return LayerKind::kGin;
        case 2: return LayerKind::kAppnp;
        case 3: return LayerKind::kGcnii;
    }
    throw std::invalid_argument("ref: bad layer kind");
}

void set_pattern(AggPattern& p, const std::int64_t* row_ptr, std::int64_t m, const std::int32_t* cols,
                 const float* coeffs) {
    p.row_ptr.assign(row_ptr, row_ptr + m + 1);
    p.cols.assign(cols, cols + row_ptr[m]);
    p.coeffs.assign(coeffs, coeffs + row_ptr[m]);
}

Tensor tensor_from(const float* v, std::int64_t r, std::int64_t c, bool rg) {
    Tensor t = Tensor::zeros(r, c, rg);
    std::memcpy(t.data(), v, sizeof(float) * static_cast<std::size_t>(r * c));
    return t;
}

// Records a closure that seeds `y`'s gradient with an arbitrary matrix, so that a single
// backward() exercises exactly one op's backward closure with a chosen upstream grad.
void seed_grad(Tape& tape, Tensor y, const float* gy) {
    tape.record([y, gy]() mutable {
        y.ensure_grad();
        std::memcpy(y.grad(), gy, sizeof(float) * static_cast<std::size_t>(y.size()));
    });
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_derive_seed(std::uint64_t s, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
    return derive_seed(s, a, b, c);
}

// ---- graph-core (src/graph.cpp) ----------------------------------------------------
int ref_graph_build(const std::int32_t* u, const std::int32_t* v, std::int64_t m, std::int32_t n,
                    int symmetrize, void** out) {
    return guard([&] {
        std::vector<Edge> edges(static_cast<std::size_t>(m));
        for (std::int64_t i = 0; i < m; ++i) edges[i] = {u[i], v[i]};
        *out = new Graph(build_graph(edges, n, symmetrize != 0));
    });
}

// Adopts an already-canonical CSR (sorted, deduplicated rows) without re-sorting; used for
// the large bench graphs where build_graph's per-row vectors would dominate setup time.
int ref_graph_from_csr(std::int32_t n, const std::int64_t* row_offsets, const std::int32_t* cols,
                       int symmetric, void** out) {
    return guard([&] {
        auto* g = new Graph();
        g->num_nodes = n;
        g->is_symmetric = symmetric != 0;
        g->row_offsets.assign(row_offsets, row_offsets + n + 1);
        g->col_indices.assign(cols, cols + row_offsets[n]);
        *out = g;
    });
}

std::int64_t ref_graph_num_edges(const void* g) { return static_cast<const Graph*>(g)->num_edges(); }

void ref_graph_copy(const void* gp, std::int64_t* row_offsets, std::int32_t* cols) {
    const Graph* g = static_cast<const Graph*>(gp);
    std::memcpy(row_offsets, g->row_offsets.data(), sizeof(std::int64_t) * g->row_offsets.size());
    std::memcpy(cols, g->col_indices.data(), sizeof(std::int32_t) * g->col_indices.size());
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

struct RefPlan {
    BatchPlan plan;
    PlanAggregation agg;
};

int ref_plan_make(const void* gp, const std::int32_t* batch, std::int64_t nb, void** out) {
    return guard([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        auto* p = new RefPlan();
        try {
            p->plan = make_batch_plan(g, std::span<const NodeId>(batch, static_cast<std::size_t>(nb)));
            p->agg = build_plan_aggregation(g, p->plan);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

// sizes: [num_batch, num_extended, num_halo, local_nnz, gcn_nnz, sum_nnz]
void ref_plan_sizes(const void* pp, std::int64_t* s) {
    const RefPlan* p = static_cast<const RefPlan*>(pp);
    s[0] = p->plan.num_batch();
    s[1] = p->plan.num_extended();
    s[2] = p->plan.num_halo();
    s[3] = p->plan.local_graph.num_edges();
    s[4] = static_cast<std::int64_t>(p->agg.gcn.cols.size());
    s[5] = static_cast<std::int64_t>(p->agg.sum.cols.size());
}

void ref_plan_copy(const void* pp, std::int32_t* extended, std::int32_t* halo, std::uint8_t* is_halo,
                   std::int32_t* batch_local_rows, std::int32_t* halo_local_rows,
                   std::int64_t* local_rowptr, std::int32_t* local_cols, std::int64_t* gcn_rowptr,
                   std::int32_t* gcn_cols, float* gcn_coeffs, std::int64_t* sum_rowptr,
                   std::int32_t* sum_cols, float* sum_coeffs) {
    const RefPlan* p = static_cast<const RefPlan*>(pp);
    const BatchPlan& pl = p->plan;
    auto cp = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
    };
    cp(extended, pl.extended_nodes);
    cp(halo, pl.halo_nodes);
    cp(is_halo, pl.is_halo);
    cp(batch_local_rows, pl.batch_local_rows);
    cp(halo_local_rows, pl.halo_local_rows);
    cp(local_rowptr, pl.local_graph.row_offsets);
    cp(local_cols, pl.local_graph.col_indices);
    cp(gcn_rowptr, p->agg.gcn.row_ptr);
    cp(gcn_cols, p->agg.gcn.cols);
    cp(gcn_coeffs, p->agg.gcn.coeffs);
    cp(sum_rowptr, p->agg.sum.row_ptr);
    cp(sum_cols, p->agg.sum.cols);
    cp(sum_coeffs, p->agg.sum.coeffs);
}

void ref_plan_free(void* p) { delete static_cast<RefPlan*>(p); }

// ---- partitioner (src/partition.cpp) -----------------------------------------------
int ref_cluster_partition(const void* gp, std::int32_t parts, std::uint64_t seed, std::int32_t* assignment) {
    return guard([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        Partitioning p = cluster_partition(g, parts, seed);
        std::memcpy(assignment, p.assignment.data(), sizeof(std::int32_t) * p.assignment.size());
    });
}

int ref_random_partition(const void* gp, std::int32_t parts, std::uint64_t seed, std::int32_t* assignment) {
    return guard([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        Partitioning p = random_partition(g, parts, seed);
        std::memcpy(assignment, p.assignment.data(), sizeof(std::int32_t) * p.assignment.size());
    });
}

// io.cpp:187-217 partition files
int ref_partition_save(const char* path, const std::int32_t* assignment, std::int32_t n, std::int32_t parts) {
    return guard([&] {
        std::vector<std::int32_t> a(assignment, assignment + n);
        save_partition(path, partition_from_assignment(a, parts));
    });
}
int ref_partition_load(const char* path, std::int32_t n, std::int32_t* assignment, std::int32_t* parts) {
    return guard([&] {
        Partitioning p = load_partition(path, n);
        std::memcpy(assignment, p.assignment.data(), sizeof(std::int32_t) * p.assignment.size());
        *parts = p.num_parts;
    });
}

double ref_inter_intra_ratio(const void* gp, const std::int32_t* assignment, std::int32_t parts) {
    const Graph& g = *static_cast<const Graph*>(gp);
    std::vector<std::int32_t> a(assignment, assignment + g.num_nodes);
    return inter_intra_ratio(g, partition_from_assignment(a, parts));
}

// ---- nn-core ops (src/tensor.cpp, src/nn.cpp) ---------------------------------------
// aggregate fwd (tensor.cpp:514-530) and, when gy != null, its backward closure (:531-549).
int ref_aggregate(const std::int64_t* row_ptr, std::int64_t m, const std::int32_t* cols,
                  const float* coeffs, const float* x, std::int64_t xrows, std::int64_t d, float* y,
                  const float* gy, float* gx) {
    return guard([&] {
        AggPattern pat;
        set_pattern(pat, row_ptr, m, cols, coeffs);
        Tape tape;
        Tensor X = tensor_from(x, xrows, d, gy != nullptr);
        Tensor Y = aggregate(gy ? &tape : nullptr, pat, X);
        std::memcpy(y, Y.data(), sizeof(float) * static_cast<std::size_t>(Y.size()));
        if (gy) {
            Tensor loss = Tensor::scalar(0.0f, true);
            seed_grad(tape, Y, gy);
            tape.backward(loss);
            DenseMatrix g = X.grad_matrix();
            std::memcpy(gx, g.values.data(), sizeof(float) * g.values.size());
        }
    });
}

// matmul fwd (tensor.cpp:148-167) and backward closure (:169-204).
int ref_matmul(const float* a, std::int64_t m, std::int64_t k, const float* b, std::int64_t n, float* y,
               const float* gy, float* ga, float* gb) {
    return guard([&] {
        Tape tape;
        Tensor A = tensor_from(a, m, k, gy != nullptr);
        Tensor B = tensor_from(b, k, n, gy != nullptr);
        Tensor Y = matmul(gy ? &tape : nullptr, A, B);
        std::memcpy(y, Y.data(), sizeof(float) * static_cast<std::size_t>(Y.size()));
        if (gy) {
            Tensor loss = Tensor::scalar(0.0f, true);
            seed_grad(tape, Y, gy);
            tape.backward(loss);
            DenseMatrix g1 = A.grad_matrix(), g2 = B.grad_matrix();
            std::memcpy(ga, g1.values.data(), sizeof(float) * g1.values.size());
            std::memcpy(gb, g2.values.data(), sizeof(float) * g2.values.size());
        }
    });
}

// softmax_cross_entropy (tensor.cpp:597-647): loss value and d loss / d logits.
int ref_softmax_ce(const float* logits, std::int64_t m, std::int64_t n, const std::int32_t* rows,
                   const std::int32_t* labels, std::int64_t r, float* loss, float* glogits) {
    return guard([&] {
        Tape tape;
        Tensor L = tensor_from(logits, m, n, true);
        Tensor y = softmax_cross_entropy(&tape, L, std::span<const std::int32_t>(rows, r),
                                         std::span<const std::int32_t>(labels, r));
        *loss = y.scalar_value();
        tape.backward(y);
        DenseMatrix g = L.grad_matrix();
        std::memcpy(glogits, g.values.data(), sizeof(float) * g.values.size());
    });
}

// AdamState::step (nn.cpp:20-41) over one tensor for `steps` consecutive grads.
int ref_adam(float* p, std::int64_t size, const float* grads, std::int32_t steps, float lr, float b1,
             float b2, float eps) {
    return guard([&] {
        Tensor P = tensor_from(p, 1, size, true);
        AdamState opt({P}, AdamConfig{lr, b1, b2, eps});
        for (std::int32_t s = 0; s < steps; ++s) {
            P.ensure_grad();
            std::memcpy(P.grad(), grads + s * size, sizeof(float) * static_cast<std::size_t>(size));
            opt.step();
        }
        std::memcpy(p, P.data(), sizeof(float) * static_cast<std::size_t>(size));
    });
}

// grad_clip (nn.cpp:47-63) on one flat gradient vector; returns the pre-clip norm.
double ref_grad_clip(float* g, std::int64_t size, double max_norm) {
    Tensor P = Tensor::zeros(1, size, true);
    P.ensure_grad();
    std::memcpy(P.grad(), g, sizeof(float) * static_cast<std::size_t>(size));
    std::vector<Tensor> ps{P};
    double norm = grad_clip(std::span<Tensor>(ps), max_norm);
    std::memcpy(g, P.grad(), sizeof(float) * static_cast<std::size_t>(size));
    return norm;
}

void ref_glorot(std::int64_t rows, std::int64_t cols, std::uint64_t seed, float* out) {
    Tensor w = Tensor::zeros(rows, cols, true);
    glorot_init(w, seed);
    std::memcpy(out, w.data(), sizeof(float) * static_cast<std::size_t>(w.size()));
}

// Epoch batch order of gas_epoch (trainer.cpp:395-400).
void ref_epoch_order(std::int32_t num_batches, std::uint64_t model_seed, std::int64_t epoch, std::int32_t* out) {
    std::vector<std::int32_t> order(static_cast<std::size_t>(num_batches));
    std::iota(order.begin(), order.end(), 0);
    Rng rng(derive_seed(model_seed ^ 0x6f726472ull, static_cast<std::uint64_t>(epoch)));
    rng.shuffle(order);
    std::memcpy(out, order.data(), sizeof(std::int32_t) * order.size());
}

// ---- history-store (src/history.cpp) -----------------------------------------------
int ref_history_create(std::int32_t layers, std::int32_t n, std::int32_t d, void** out) {
    return guard([&] { *out = new HistoryStore(layers, n, d); });
}
void ref_history_free(void* h) { delete static_cast<HistoryStore*>(h); }
int ref_history_push(void* h, std::int32_t layer, const std::int32_t* ids, std::int64_t k, const float* rows) {
    return guard([&] {
        auto* s = static_cast<HistoryStore*>(h);
        s->push(layer, std::span<const NodeId>(ids, static_cast<std::size_t>(k)),
                std::span<const float>(rows, static_cast<std::size_t>(k * s->dim())));
    });
}
int ref_history_pull(void* h, std::int32_t layer, const std::int32_t* ids, std::int64_t k, float* out) {
    return guard([&] {
        auto* s = static_cast<HistoryStore*>(h);
        DenseMatrix m = s->pull(layer, std::span<const NodeId>(ids, static_cast<std::size_t>(k)));
        if (!m.values.empty()) std::memcpy(out, m.values.data(), sizeof(float) * m.values.size());
    });
}
void ref_history_advance(void* h) { static_cast<HistoryStore*>(h)->advance_step(); }
int ref_history_stamp(void* h, std::int32_t layer, std::int32_t v, std::int64_t* out) {
    return guard([&] { *out = static_cast<HistoryStore*>(h)->last_push_step(layer, v); });
}
int ref_history_fill(void* h, std::int32_t layer, const float* values) {
    return guard([&] {
        auto* s = static_cast<HistoryStore*>(h);
        DenseMatrix m(s->num_nodes(), s->dim());
        std::memcpy(m.values.data(), values, sizeof(float) * m.values.size());
        s->fill_layer(layer, m);
    });
}
int ref_history_layer(void* h, std::int32_t layer, float* out) {
    return guard([&] {
        const DenseMatrix& m = static_cast<HistoryStore*>(h)->layer_matrix(layer);
        std::memcpy(out, m.values.data(), sizeof(float) * m.values.size());
    });
}
// out: per layer [eps_max, eps_mean, age_max, age_mean]
int ref_history_staleness(void* h, const float* reference, double* out) {
    return guard([&] {
        auto* s = static_cast<HistoryStore*>(h);
        std::vector<DenseMatrix> refs;
        const std::int64_t per = static_cast<std::int64_t>(s->num_nodes()) * s->dim();
        for (std::int32_t l = 0; l < s->num_layers(); ++l) {
            DenseMatrix m(s->num_nodes(), s->dim());
            std::memcpy(m.values.data(), reference + l * per, sizeof(float) * m.values.size());
            refs.push_back(std::move(m));
        }
        StalenessReport r = s->measure_staleness(refs);
        for (std::size_t l = 0; l < r.layers.size(); ++l) {
            out[4 * l + 0] = r.layers[l].eps_max;
            out[4 * l + 1] = r.layers[l].eps_mean;
            out[4 * l + 2] = static_cast<double>(r.layers[l].age_max);
            out[4 * l + 3] = r.layers[l].age_mean;
        }
    });
}
int ref_history_save(void* h, const char* path) {
    return guard([&] { static_cast<HistoryStore*>(h)->save_checkpoint(path); });
}
int ref_history_load(const char* path, void** out) {
    return guard([&] { *out = new HistoryStore(HistoryStore::load_checkpoint(path)); });
}

// ---- gas-trainer session (src/trainer.cpp) -------------------------------------------
// Builds Dataset + BatchSchedule (+ Model, AdamState, HistoryStore) as train_model does
// (trainer.cpp:538-574), from an explicit partition assignment. When sample_parts is
// non-null only those parts are planned (bench: bounded CPU sample of the workload).
int ref_session_create(const void* gp, const float* features, std::int32_t in_dim, const std::int32_t* labels,
                       const std::uint8_t* train_mask, std::int32_t num_classes, const std::int32_t* assignment,
                       std::int32_t num_parts, const std::int32_t* sample_parts, std::int32_t num_sample,
                       const RefSpec* spec, void** out) {
    return guard([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        auto s = std::make_unique<Session>();
        s->ds.graph = g;
        const std::int64_t n = g.num_nodes;
        s->ds.features = DenseMatrix(n, in_dim);
        std::memcpy(s->ds.features.values.data(), features, sizeof(float) * static_cast<std::size_t>(n * in_dim));
        s->ds.labels.labels.assign(labels, labels + n);
        s->ds.labels.num_classes = num_classes;
        s->ds.labels.train_mask.assign(train_mask, train_mask + n);
        s->ds.labels.val_mask.assign(static_cast<std::size_t>(n), 0);
        s->ds.labels.test_mask.assign(static_cast<std::size_t>(n), 0);
        std::vector<std::int32_t> a(assignment, assignment + n);
        Partitioning parts = partition_from_assignment(a, num_parts);
        if (sample_parts && num_sample > 0) {
            for (std::int32_t i = 0; i < num_sample; ++i) {
                const auto& nodes = parts.parts.at(static_cast<std::size_t>(sample_parts[i]));
                s->sched.plans.push_back(make_batch_plan(s->ds.graph, nodes));
                s->sched.aggs.push_back(build_plan_aggregation(s->ds.graph, s->sched.plans.back()));
                s->sched_parts.push_back(sample_parts[i]);
            }
        } else {
            s->sched = BatchSchedule::build(s->ds.graph, parts);
            for (std::int32_t i = 0; i < num_parts; ++i) s->sched_parts.push_back(i);
        }
        ModelSpec ms;
        ms.kind = to_kind(spec->kind);
        ms.num_layers = spec->num_layers;
        ms.hidden = spec->hidden;
        ms.dropout = spec->dropout;
        ms.alpha = spec->alpha;
        ms.beta = spec->beta;
        ms.l2_weight = spec->l2_weight;
        ms.clip_max_norm = spec->clip_max_norm;
        ms.opt = AdamConfig{spec->lr, spec->beta1, spec->beta2, spec->eps};
        ms.seed = spec->seed;
        s->model.emplace(Model::build(ms, in_dim, num_classes));
        s->opt.emplace(s->model->params(), ms.opt);
        s->store = HistoryStore(std::max(0, ms.num_layers - 1), g.num_nodes, s->model->history_dim());
        *out = s.release();
    });
}

void ref_session_free(void* s) { delete static_cast<Session*>(s); }

std::int32_t ref_session_num_params(void* sp) {
    return static_cast<std::int32_t>(static_cast<Session*>(sp)->model->params().size());
}
void ref_session_param_shape(void* sp, std::int32_t i, std::int64_t* rows, std::int64_t* cols) {
    auto ps = static_cast<Session*>(sp)->model->params();
    *rows = ps.at(static_cast<std::size_t>(i)).rows();
    *cols = ps.at(static_cast<std::size_t>(i)).cols();
}
// Parameters flattened in Model::params() order (trainer.cpp:122-127).
void ref_session_get_params(void* sp, float* out) {
    for (Tensor t : static_cast<Session*>(sp)->model->params()) {
        std::memcpy(out, t.data(), sizeof(float) * static_cast<std::size_t>(t.size()));
        out += t.size();
    }
}
void ref_session_set_params(void* sp, const float* in) {
    for (Tensor t : static_cast<Session*>(sp)->model->params()) {
        std::memcpy(t.data(), in, sizeof(float) * static_cast<std::size_t>(t.size()));
        in += t.size();
    }
}
std::int32_t ref_session_history_dim(void* sp) { return static_cast<Session*>(sp)->model->history_dim(); }
int ref_session_get_history(void* sp, std::int32_t layer, float* out) {
    return ref_history_layer(&static_cast<Session*>(sp)->store, layer, out);
}
int ref_session_set_history(void* sp, std::int32_t layer, const float* in) {
    return ref_history_fill(&static_cast<Session*>(sp)->store, layer, in);
}
std::int64_t ref_session_store_step(void* sp) { return static_cast<Session*>(sp)->store.step(); }
std::int64_t ref_session_adam_steps(void* sp) { return static_cast<Session*>(sp)->opt->step_count(); }

// One gas_epoch (trainer.cpp:386-442) with evaluate/staleness off, as in gas_main.cpp:274-277.
int ref_session_epoch(void* sp, std::int64_t epoch, int shuffle, int use_prefetch, double* loss, double* seconds) {
    return guard([&] {
        Session* s = static_cast<Session*>(sp);
        EpochOptions o;
        o.evaluate = false;
        o.measure_staleness = false;
        o.shuffle = shuffle != 0;
        if (use_prefetch && !s->prefetcher) s->prefetcher.emplace(s->store);
        o.prefetcher = use_prefetch ? &*s->prefetcher : nullptr;
        auto t0 = std::chrono::steady_clock::now();
        EpochReport r = gas_epoch(*s->model, *s->opt, s->ds, s->sched, s->store, epoch, o);
        auto t1 = std::chrono::steady_clock::now();
        *loss = r.loss;
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// gas_epoch with the report fields (EpochReport, trainer.hpp:107-115): measure_staleness runs
// the frozen gas_forward_snapshot pass and measure_staleness after the epoch (trainer.cpp:434-438).
int ref_session_epoch_report(void* sp, std::int64_t epoch, int shuffle, int measure_staleness, double* loss,
                             std::int64_t* peak_floats, std::int64_t* edges_per_layer, std::int64_t* batch_peak,
                             double* eps_max) {
    return guard([&] {
        Session* s = static_cast<Session*>(sp);
        EpochOptions o;
        o.evaluate = false;
        o.measure_staleness = measure_staleness != 0;
        o.shuffle = shuffle != 0;
        EpochReport r = gas_epoch(*s->model, *s->opt, s->ds, s->sched, s->store, epoch, o);
        *loss = r.loss;
        *peak_floats = r.peak_floats;
        *edges_per_layer = r.edges_per_layer;
        if (batch_peak) std::copy(r.batch_peak_floats.begin(), r.batch_peak_floats.end(), batch_peak);
        if (eps_max) std::copy(r.eps_max.begin(), r.eps_max.end(), eps_max);
    });
}

// One batch exactly as gas_epoch runs it (run_batch without capture, trainer.cpp:295-339,
// then advance_step :426), timed with steady_clock: the reference arm's unit of work.
int ref_session_run(void* sp, std::int32_t slot, std::int64_t epoch, double* loss_out, double* seconds) {
    return guard([&] {
        Session* s = static_cast<Session*>(sp);
        Model& model = *s->model;
        const BatchPlan& plan = s->sched.plans.at(static_cast<std::size_t>(slot));
        const PlanAggregation& agg = s->sched.aggs.at(static_cast<std::size_t>(slot));
        auto t0 = std::chrono::steady_clock::now();
        Model::ForwardOptions fwd;
        fwd.training = true;
        fwd.epoch = epoch;
        fwd.batch_index = s->sched_parts.at(static_cast<std::size_t>(slot));
        fwd.store = &s->store;
        fwd.push = true;
        Tape tape;
        Tensor logits = model.forward(&tape, s->ds.features, plan, agg, fwd);
        std::vector<std::int32_t> rows, lab;
        for (std::size_t i = 0; i < plan.batch_nodes.size(); ++i) {
            const NodeId v = plan.batch_nodes[i];
            if (s->ds.labels.train_mask[v]) {
                rows.push_back(static_cast<std::int32_t>(i));
                lab.push_back(s->ds.labels.labels[v]);
            }
        }
        *loss_out = 0.0;
        if (!rows.empty()) {
            Tensor loss = softmax_cross_entropy(&tape, logits, rows, lab);
            *loss_out = loss.scalar_value();
            tape.backward(loss);
            auto params = model.params();
            if (model.spec().clip_max_norm > 0.0f) grad_clip(std::span<Tensor>(params), model.spec().clip_max_norm);
            s->opt->step();
            s->opt->zero_grad();
        }
        s->store.advance_step();
        tape.reset();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// One batch of gas_epoch with full capture. slot = schedule index (== part id when the
// whole partition is planned). Outputs (batch rows, in plan.batch_nodes order):
//   acts   : (L-1) x nb x hist_dim   pushed (post-activation) rows per history layer
//   logits : nb x C
//   grads  : flat parameter gradients BEFORE clipping (Model::params() order)
// *stepped = 1 when an optimizer step happened (batch had training rows and train != 0).
int ref_session_batch(void* sp, std::int32_t slot, std::int64_t epoch, int train, int push, float* acts,
                      float* logits_out, double* loss_out, float* grads, int* stepped) {
    return guard([&] {
        Session* s = static_cast<Session*>(sp);
        Model& model = *s->model;
        const BatchPlan& plan = s->sched.plans.at(static_cast<std::size_t>(slot));
        const PlanAggregation& agg = s->sched.aggs.at(static_cast<std::size_t>(slot));
        const std::int32_t L = model.num_layers();
        const std::int64_t n = s->ds.graph.num_nodes;

        std::vector<DenseMatrix> cap(static_cast<std::size_t>(std::max(0, L - 1)),
                                     DenseMatrix(n, model.history_dim()));
        DenseMatrix fin(n, model.num_classes());
        Model::ForwardOptions fwd;
        fwd.training = train != 0;
        fwd.epoch = epoch;
        fwd.batch_index = s->sched_parts.at(static_cast<std::size_t>(slot));
        fwd.store = &s->store;
        fwd.push = push != 0;
        fwd.capture.layer_out = &cap;
        fwd.capture.final_out = &fin;
        Tape tape;
        Tape* tp = train ? &tape : nullptr;
        Tensor logits = model.forward(tp, s->ds.features, plan, agg, fwd);

        const std::int64_t nb = plan.num_batch();
        const std::int32_t hd = model.history_dim();
        if (acts)
            for (std::int32_t l = 0; l < L - 1; ++l)
                for (std::int64_t i = 0; i < nb; ++i)
                    std::memcpy(acts + (static_cast<std::int64_t>(l) * nb + i) * hd,
                                cap[l].row(plan.batch_nodes[i]), sizeof(float) * hd);
        if (logits_out) std::memcpy(logits_out, logits.data(), sizeof(float) * static_cast<std::size_t>(logits.size()));

        std::vector<std::int32_t> rows, lab;
        for (std::size_t i = 0; i < plan.batch_nodes.size(); ++i) {
            const NodeId v = plan.batch_nodes[i];
            if (s->ds.labels.train_mask[v]) {
                rows.push_back(static_cast<std::int32_t>(i));
                lab.push_back(s->ds.labels.labels[v]);
            }
        }
        *stepped = 0;
        *loss_out = 0.0;
        if (!rows.empty()) {
            Tensor loss = softmax_cross_entropy(tp, logits, rows, lab);
            auto params = model.params();
            if (train && model.spec().l2_weight > 0.0f)
                loss = add(tp, loss, l2_penalty(tp, params, model.spec().l2_weight));
            *loss_out = loss.scalar_value();
            if (train) {
                tape.backward(loss);
                if (grads) {
                    float* g = grads;
                    for (Tensor t : params) {
                        DenseMatrix gm = t.grad_matrix();
                        std::memcpy(g, gm.values.data(), sizeof(float) * gm.values.size());
                        g += t.size();
                    }
                }
                if (model.spec().clip_max_norm > 0.0f)
                    grad_clip(std::span<Tensor>(params), model.spec().clip_max_norm);
                s->opt->step();
                s->opt->zero_grad();
                *stepped = 1;
            }
        }
        s->store.advance_step();
    });
}

// evaluate (trainer.cpp:444-464) with the session's params: accuracy over the given masks
// (train mask: the session's) and the full-batch logits (n x C, global order).
int ref_session_evaluate(void* sp, const std::uint8_t* val_mask, const std::uint8_t* test_mask, double* acc3,
                         float* logits_out) {
    return guard([&] {
        Session* s = static_cast<Session*>(sp);
        const std::size_t n = static_cast<std::size_t>(s->ds.graph.num_nodes);
        s->ds.labels.val_mask.assign(val_mask, val_mask + n);
        s->ds.labels.test_mask.assign(test_mask, test_mask + n);
        BatchSchedule full = BatchSchedule::full_batch(s->ds.graph);
        Accuracy a = evaluate(*s->model, s->ds, full);
        acc3[0] = a.train;
        acc3[1] = a.val;
        acc3[2] = a.test;
        if (logits_out) {
            Model::ForwardOptions fwd;
            Tensor lg = s->model->forward(nullptr, s->ds.features, full.plans[0], full.aggs[0], fwd);
            std::memcpy(logits_out, lg.data(), sizeof(float) * static_cast<std::size_t>(lg.size()));
        }
    });
}

// infer_from_history (trainer.cpp:501-536) over the session's store.
int ref_session_infer(void* sp, std::int32_t* predictions, int* stale) {
    return guard([&] {
        Session* s = static_cast<Session*>(sp);
        InferenceResult r = infer_from_history(*s->model, s->store, s->ds);
        std::memcpy(predictions, r.predictions.data(), sizeof(std::int32_t) * r.predictions.size());
        *stale = r.stale ? 1 : 0;
    });
}

}  // extern "C"
