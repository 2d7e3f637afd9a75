// Internal definition of the single-GPU trainer (trainer.cu), shared with the
// data-parallel exchange (dp.cu).
#pragma once

#include <algorithm>
#include <cmath>
#include <memory>
#include <utility>
#include <vector>

#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {
const Schedule& schedule_of(gasb_schedule s);
gasb_history history_create(int32_t layers, int32_t n, int32_t dim);
void history_destroy(gasb_history h);
float* history_table(gasb_history h, int32_t layer);
int64_t history_ld(gasb_history h);
int64_t* history_stamps(gasb_history h, int32_t layer);
int64_t* history_step_ptr(gasb_history h);
int32_t* history_flags(gasb_history h, int32_t layer);
void history_release_tables(gasb_history h);

// Partition-sharded history tables of a data-parallel group (dp.cu): node v's rows live in
// rank owner(v)'s shard (in its peer-mapped exchange region) at row local(v).
constexpr int kShardMaxWorld = 8;
constexpr int kShardLocalBits = 29;
struct ShardView {
    const uint32_t* owner_local = nullptr;  // per global node: owner << 29 | row in the owner's shard
    const float* tables[kShardMaxWorld] = {};  // rank j's shard of H_1 (layer l at + (l-1) * layer_stride[j])
    int64_t layer_stride[kShardMaxWorld] = {};
    int64_t ld = 0;
    int32_t world = 0;  // 0: the trainer's histories are local tables
};
// dst[i] = H_layer[ids[i]] read from the owners' shards (NVLink P2P loads for remote rows).
void launch_shard_pull(const ShardView& s, int32_t layer, const int32_t* ids, int64_t count, float* dst,
                       int64_t ldd, int32_t dim, cudaStream_t st);

// Host staging vectors whose elements are default-initialised (not zeroed): the setup loops
// write every element from OpenMP threads, so the pages are first touched in parallel
// instead of by a serial zero-fill on the constructing thread.
template <class T>
struct UninitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = UninitAlloc<U>;
    };
    UninitAlloc() = default;
    template <class U>
    UninitAlloc(const UninitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* q) noexcept {
        ::new (static_cast<void*>(q)) U;
    }
    template <class U, class... A>
    void construct(U* q, A&&... a) {
        ::new (static_cast<void*>(q)) U(std::forward<A>(a)...);
    }
};
template <class T>
using HVec = std::vector<T, UninitAlloc<T>>;

template <class T>
struct DevBuf {
    T* p = nullptr;
    int64_t n = 0;
    void alloc(int64_t count) {
        free();
        n = count;
        GASB_CUDA(cudaMalloc(&p, sizeof(T) * std::max<int64_t>(count, 1)));
    }
    template <class V>
    void upload(const V& v) {
        alloc(static_cast<int64_t>(v.size()));
        if (!v.empty()) GASB_CUDA(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    }
    // stream-ordered upload that reallocates only to grow (per-epoch tables); the host
    // vector must stay alive until the copy ran (the caller keeps it as a member)
    void upload_async(const std::vector<T>& v, cudaStream_t st) {
        if (n < static_cast<int64_t>(v.size())) {
            GASB_CUDA(cudaStreamSynchronize(st));
            alloc(static_cast<int64_t>(v.size()));
        }
        if (!v.empty()) GASB_CUDA(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
    }
    void zero() {
        if (n) GASB_CUDA(cudaMemset(p, 0, sizeof(T) * n));
    }
    bool owned = true;  // false: a view into memory owned elsewhere (the DP exchange region)
    void adopt(T* q, int64_t count) {
        free();
        p = q;
        n = count;
        owned = false;
    }
    void free() {
        if (p && owned) cudaFree(p);
        p = nullptr;
        n = 0;
        owned = true;
    }
    ~DevBuf() { free(); }
};

struct SegTable {
    DevBuf<int64_t> seg_beg;
    DevBuf<int32_t> seg_row, seg_slot, row_seg0, row_nseg;
    DevBuf<int32_t> ranges;  // per group: nranges + 1 work-range boundaries (split_ranges)
    int32_t nranges = 0;
    bool split = false;  // rows cut at range boundaries (not the bit-exact sequential mode)
    std::vector<int64_t> group_seg0, group_nseg;  // per group (batch) range of segments
    int64_t max_group_slots = 0, total_slots = 0;
    DevBuf<int32_t> row_slots;  // source-blocked tables: each row's partial slots in combine order
    SpmmSegs segs(int64_t g) const {
        SpmmSegs s{seg_beg.p, seg_row.p, seg_slot.p, row_seg0.p, row_nseg.p, ranges.p + g * (nranges + 1), nranges,
                   split ? 0 : 1};
        s.row_slots = row_slots.p;
        return s;
    }
};

}  // namespace gasb

using namespace gasb;  // internal header: the trainer is written against gasb's helpers

struct gasb_trainer_s {
    gasb_model_spec spec{};
    gasb_trainer_options opt{};
    int32_t n = 0, F = 0, C = 0, L = 0, H = 0, hist_dim = 0, num_parts = 0;
    int64_t ldF = 0, ldH = 0, ldC = 0;
    const Schedule* sched = nullptr;
    cudaStream_t stream = nullptr, side = nullptr;
    // host-input pipeline (set_features): H2D into x_stage on copy_stream, re-pitched into X
    // on `stream`; ev_staged / ev_stage_free order the two so a step's H2D overlaps the
    // previous step's compute
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_staged = nullptr, ev_stage_free = nullptr;
    gasb_history hist = nullptr;

    // per part (host)
    std::vector<int32_t> nb, ne, nh, ntrain;
    std::vector<int64_t> row_off, edge_off, t_off, tr_off, ext_off;
    int32_t nb_max = 0, ne_max = 0;

    // device data
    DevBuf<float> X, x_stage;  // x_stage: dense host-layout copy for set_features
    DevBuf<int32_t> batch_nodes, cols_g, cols_l, t_src, train_rows, train_labels, extended, compose_idx, halo_ids;
    DevBuf<double> coef64;
    DevBuf<float> t_cf;
    DevBuf<int64_t> t_rowptr;
    DevBuf<int32_t> t_order;  // per part: intra-batch targets by descending entry count
    // spmm_bwd2 plan (GCN layers with d >= 64): per part, per (CTA split, source phase) blobs
    DevBuf<int64_t> bwd2_boff;
    DevBuf<unsigned char> bwd2_blobs;
    std::vector<int64_t> bwd2_off;  // per part: index of its first blob offset in bwd2_boff
    std::vector<char> bwd2_ok;      // per part: every blob fits shared memory
    int32_t bwd2_splits = 0;
    bool use_bwd2 = false;
    // aggregate backward of a batch layer (intra-batch targets): spmm_bwd2 where planned, else spmm_bwd
    void spmm_bwd_batch(int32_t p, const float* gy, int64_t ldgy, int32_t dim, const float* mask, int64_t ldm,
                        float* gx, int64_t ldgx, cudaStream_t st);
    SegTable seg_batch, seg_all;
    DevBuf<int32_t> counters, row_label, xflags, ce_done;  // xflags: value flags of X (kernels.cuh)
    DevBuf<double> partial_batch, partial_all;
    int32_t max_chunks = 0;
    int64_t pld = 0, pld_all = 0;

    // model
    // per parameter tensor: device offset, rows, cols, row pitch (cols rounded up to 4 floats
    // so every weight is a TMA-describable GEMM operand; pads are 0 and stay 0 under Adam)
    std::vector<int64_t> poff, prow, pcol, ppitch;
    int64_t nparam_dense = 0;  // Model::params() floats (the API's flat layout)
    std::vector<int32_t> layer_param;       // param index of W_l (GCN) per layer 1..L
    int64_t nparam = 0;
    std::vector<float> h_params_init;
    DevBuf<float> params, grads, adam_m, adam_v;
    DevBuf<int64_t> t_counter;
    DevBuf<int32_t> adam_done;  // Adam's fused end-of-batch arrival counter
    DevBuf<double> bc, norm_scratch;
    int64_t bc_cap = 0, t_host = 0;

    // activations
    std::vector<int32_t> dims;    // d[0..L]
    DevBuf<float> agg_all;        // hoisted layer-1 aggregation, n x ldF
    std::vector<DevBuf<float>> agg, act;
    DevBuf<float> logits, glogits, g_agg, g_out, x_ext, h_ext, halo_buf;
    // TMA tensor maps of the SpMM source tables (tile::gather4 staging, spmm.cu)
    CUtensorMap tm_x{}, tm_xext{}, tm_hext{};
    std::vector<CUtensorMap> tm_hist;
    bool tm_ok[4] = {false, false, false, false};  // x, hist, x_ext, h_ext
    const CUtensorMap* source_tmap(int32_t l) const {
        if (l == 1) return tm_ok[0] ? &tm_x : nullptr;
        return tm_ok[1] ? &tm_hist[l - 2] : nullptr;
    }
    void build_tmaps() {
        tm_ok[0] = make_row_tmap(X.p, n, F, ldF, spmm_box_cols(F), &tm_x);
        tm_hist.resize(static_cast<size_t>(std::max(0, L - 1)));
        tm_ok[1] = L >= 2;
        for (int32_t l = 1; l < L; ++l)
            tm_ok[1] = tm_ok[1] && make_row_tmap(history_table(hist, l), n, hist_dim, history_ld(hist), spmm_box_cols(hist_dim),
                                                 &tm_hist[l - 1]);
        if (x_ext.p) tm_ok[2] = make_row_tmap(x_ext.p, ne_max, F, ldF, spmm_box_cols(F), &tm_xext);
        const int32_t hdim = residual ? D : H;
        if (h_ext.p) tm_ok[3] = make_row_tmap(h_ext.p, ne_max, hdim, ld_of(hdim), spmm_box_cols(hdim), &tm_hext);
        if (residual && h0.p) tm_h0_ok = make_row_tmap(h0.p, ne_max, D, ldD, spmm_box_cols(D), &tm_h0);
    }
    DevBuf<double> loss, row_scratch;

    DevBuf<float> gemm_ws;  // split-K scratch of the tensor-core GEMM (gemm_tc.cu)
    // GCN backward: the weight-gradient GEMMs run on `side` (own split-K scratch), overlapped
    // with the dgrad -> SpMM-backward chain; g_out is double-buffered so a wgrad still
    // reading layer l's gradient never races the SpMM backward of layer l - 1
    DevBuf<float> gemm_ws2, g_out2;
    std::vector<cudaEvent_t> ev_fork, ev_wdone;
    cudaEvent_t ev_join = nullptr;
    // reference-structured mode with opt.prefetch (the Prefetcher, history.cpp:184-252, and
    // the paper's concurrent execution): every history layer's halo rows of the batch are
    // pulled on `side` at batch start, overlapped with layer-1 compute; layer l waits only
    // for its own copy (the batch's pushes never touch its halo rows)
    DevBuf<float> halo_pf;
    int64_t halo_pf_ld = 0, halo_pf_rows = 0;
    cudaEvent_t ev_pf_start = nullptr;
    std::vector<cudaEvent_t> ev_pf;
    void enqueue_prefetch(int32_t p);
    // sharded data-parallel mode: halo rows come from the owners' shards, batches push
    // nothing (the group commits the step's rows to their owners after the step barrier)
    ShardView shard{};
    bool sharded_dp = false;
    void pull_halo(int32_t p, int32_t layer, float* dst, int64_t ldd, int32_t dim) {
        const int32_t* ids = halo_ids.p + (ext_off[p] - row_off[p]);
        if (shard.world > 0) launch_shard_pull(shard, layer, ids, nh[p], dst, ldd, dim, stream);
        else
            launch_rows(1, ids, nh[p], history_table(hist, layer), history_ld(hist), dst, ldd, dim, n, nullptr,
                        nullptr, nullptr, stream);
    }
    DevBuf<double> colsum_ws;  // row-block partials of the bias-gradient column sums
    struct WsGuard {        // scopes the thread's GEMM / column-sum workspaces to one enqueue
        explicit WsGuard(DevBuf<float>& w, DevBuf<double>* c = nullptr) {
            set_gemm_workspace(w.p, kGemmWsFloats);
            if (c && c->p) set_colsum_workspace(c->p, c->n);
        }
        ~WsGuard() {
            set_gemm_workspace(nullptr, 0);
            set_colsum_workspace(nullptr, 0);
        }
    };

    // ---- residual models: APPNP (kind 2) / GCNII (kind 3) ----
    bool residual = false;
    int32_t D = 0;      // width of every propagation layer and of the histories (GCNII: H, APPNP: C)
    int64_t ldD = 0, ldA = 0;  // ldA: row pitch of act[l] (GCN: ldH)
    int32_t p_hw1 = -1, p_hb1 = -1, p_hw2 = -1, p_hb2 = -1, p_ow = -1, p_ob = -1;  // param indices
    DevBuf<int32_t> brow;                  // batch_local_rows per part, at row_off
    DevBuf<int64_t> a_rowptr;              // CSC over ALL edges of a batch (targets = V_b local rows)
    DevBuf<int32_t> a_src;                 //   entries: batch row r, ascending r per target
    DevBuf<float> a_cf;
    std::vector<int64_t> a_off;            // per part: offset of its ne+1 row pointers
    DevBuf<float> h0, z, h0g, zg, wt, prop, gmix, dprop, gout;
    std::vector<DevBuf<float>> mixed;      // GCNII: mixed_l (needed for dW~_l)
    CUtensorMap tm_h0{};
    bool tm_h0_ok = false;
    float* P(int32_t i) { return params.p + poff[i]; }
    float* G(int32_t i) { return grads.p + poff[i]; }
    int32_t add_param(int64_t r, int64_t c) {
        poff.push_back(nparam);
        prow.push_back(r);
        pcol.push_back(c);
        ppitch.push_back(round_up(c, 4));
        nparam += r * ppitch.back();
        nparam_dense += r * c;
        return static_cast<int32_t>(poff.size()) - 1;
    }
    int64_t pp(int32_t i) const { return ppitch[i]; }
    // dense (Model::params() order) <-> padded device layout
    void params_to_dense(const float* dev, float* host) const {
        int64_t o = 0;
        for (size_t i = 0; i < poff.size(); ++i) {
            GASB_CUDA(cudaMemcpy2D(host + o, sizeof(float) * pcol[i], dev + poff[i], sizeof(float) * ppitch[i],
                                   sizeof(float) * pcol[i], prow[i], cudaMemcpyDeviceToHost));
            o += prow[i] * pcol[i];
        }
    }
    void params_from_dense(const float* host, float* dev) const {
        int64_t o = 0;
        for (size_t i = 0; i < poff.size(); ++i) {
            GASB_CUDA(cudaMemcpy2D(dev + poff[i], sizeof(float) * ppitch[i], host + o, sizeof(float) * pcol[i],
                                   sizeof(float) * pcol[i], prow[i], cudaMemcpyHostToDevice));
            o += prow[i] * pcol[i];
        }
    }
    void build_residual(const std::vector<int64_t>& h_arp, const HVec<int32_t>& h_asrc,
                        const HVec<float>& h_acf, const std::vector<int32_t>& h_brow);
    void enqueue_batch_res(int32_t p, bool train, bool push, bool fused, bool dp = false);

    // ---- cross-batch concurrent execution (opt.cross_batch; the paper's concurrent pulls,
    // SURVEY north_star 5): batch b+1's halo aggregations run on the low-priority stream `bg`
    // while batch b runs its backward; batch b+1's forward then aggregates only its intra-batch
    // edges and adds the halo fp64 partials (one segment table over both launches) ----
    int32_t xmode = 0;          // 0 off, 1 halo on bg (layer 1 hoisted), 2 + per-batch layer 1 on bg
    int32_t bg_ctas = 0;        // grid cap of the bg launches (0: full grid)
    int32_t xphase = 0;         // enqueue_batch: 0 whole batch, 1 forward only, 2 loss + backward only
    cudaStream_t bg = nullptr;
    cudaEvent_t ev_xstart = nullptr, ev_xfwd = nullptr, ev_xbg = nullptr;
    DevBuf<int32_t> xcols;      // per part, edges re-laid [halo-source block | intra-source block],
    DevBuf<double> xcoef;       //   each row-major in CSR order (same offsets as cols_g)
    SegTable seg_xh, seg_xi;    // per part: the halo block's / the intra block's segments
    DevBuf<double> partial_x;   // per history layer: xslots x pldx fp64 partials
    DevBuf<int32_t> counters_x; // per history layer: R x cxld arrival counters (self-resetting)
    DevBuf<double> xsum;        // per history layer: the halo block's fp64 row sums (nb_max x pldx)
    int64_t pldx = 0, xslots = 0;
    int32_t cxld = 0;
    std::vector<cudaGraphExec_t> graphs_xf, graphs_xb;
    std::vector<int64_t> graph_launches_xf, graph_launches_xb;
    void build_xbatch(const std::vector<int64_t>& rp, const HVec<int32_t>& cg, const HVec<double>& cf);
    void enqueue_bg(int32_t q, bool wait_fwd);
    int64_t launch_x_graph(int32_t p, int32_t phase);
    void run_epoch_x(const std::vector<int32_t>& order);
    SpmmSegs xsegs(int32_t p, bool halo) const { return (halo ? seg_xh : seg_xi).segs(p); }
    double* xsums(int32_t l) { return xsum.p + static_cast<int64_t>(l - 2) * nb_max * pldx; }
    void build_block_segments(const std::vector<int64_t>& row_start, const std::vector<int64_t>& part_end,
                              SegTable& t);
    double* xpartial(int32_t l) { return partial_x.p + static_cast<int64_t>(l - 2) * xslots * pldx; }
    int32_t* xcounters(int32_t l) { return counters_x.p + static_cast<int64_t>(l - 2) * row_off[num_parts] * cxld; }

    // graphs
    std::vector<cudaGraphExec_t> graphs;
    std::vector<int64_t> graph_launches;
    int64_t epoch_launches = 0;
    std::vector<int32_t> last_order;
    std::vector<uint8_t> last_stepped;

    ~gasb_trainer_s() {
        if (stream) cudaStreamSynchronize(stream);
        for (auto g : graphs)
            if (g) cudaGraphExecDestroy(g);
        for (auto g : graphs_dp)
            if (g) cudaGraphExecDestroy(g);
        for (auto g : graphs_xf)
            if (g) cudaGraphExecDestroy(g);
        for (auto g : graphs_xb)
            if (g) cudaGraphExecDestroy(g);
        if (bg) cudaStreamSynchronize(bg);
        for (auto e : {ev_xstart, ev_xfwd, ev_xbg})
            if (e) cudaEventDestroy(e);
        if (bg) cudaStreamDestroy(bg);
        if (hist) history_destroy(hist);
        for (auto e : ev_fork) cudaEventDestroy(e);
        for (auto e : ev_wdone) cudaEventDestroy(e);
        if (ev_join) cudaEventDestroy(ev_join);
        if (ev_pf_start) cudaEventDestroy(ev_pf_start);
        if (ev_sub_uploaded) cudaEventDestroy(ev_sub_uploaded);
        if (sub_pinned) cudaFreeHost(sub_pinned);
        for (auto e : ev_pf) cudaEventDestroy(e);
        if (copy_stream) cudaStreamSynchronize(copy_stream);
        if (ev_staged) cudaEventDestroy(ev_staged);
        if (ev_stage_free) cudaEventDestroy(ev_stage_free);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        for (int i = 0; i < 2; ++i) {
            if (dmask_done[i]) cudaEventDestroy(dmask_done[i]);
            if (dmask_host[i]) cudaFreeHost(dmask_host[i]);
        }
        if (side) cudaStreamDestroy(side);
        if (stream) cudaStreamDestroy(stream);
    }

    int64_t ld_of(int32_t d) const { return round_up(std::max(d, 1), 8); }
    // value flags of the table layer l's aggregation reads: X for l = 1, H_{l-1} otherwise
    const int32_t* source_flags(int32_t l) const { return l == 1 ? xflags.p : history_flags(hist, l - 1); }
    float* W(int32_t l) { return params.p + poff[layer_param[l]]; }
    float* gW(int32_t l) { return grads.p + poff[layer_param[l]]; }

    // Adam bias corrections 1 - beta^t (nn.cpp:23-24), host std::pow as the reference, as a
    // device table indexed by the device step counter. The captured batch graphs bake the
    // table's address into their Adam node, so it must never move: build() sizes it once up
    // to the saturation step T (the first t with both corrections == 1.0 exactly; pow is
    // monotone, so every later t gives 1.0 too) and the kernel clamps t to T, held in bc[0].
    // Betas that never saturate (beta -> 1) grow the table, and a move re-captures the graphs.
    bool bc_saturated = false;
    void ensure_bc(int64_t t_max) {
        if (bc_saturated || t_max < bc_cap) return;
        const double b1 = spec.beta1, b2 = spec.beta2;
        auto sat = [&](int64_t t) {
            return 1.0 - std::pow(b1, static_cast<double>(t)) == 1.0 && 1.0 - std::pow(b2, static_cast<double>(t)) == 1.0;
        };
        constexpr int64_t kMaxTable = int64_t(1) << 22;  // 64 MB of corrections
        int64_t cap = std::max<int64_t>(1024, bc_cap), tsat = 0;
        if (bc_cap == 0)
            for (int64_t t = 1; t < kMaxTable; ++t)
                if (sat(t)) {
                    tsat = t;
                    break;
                }
        if (tsat > 0) cap = tsat + 1;
        else
            while (cap <= t_max) cap *= 2;
        std::vector<double> h(static_cast<size_t>(2 * cap));
        for (int64_t t = 1; t < cap; ++t) {
            h[2 * t] = 1.0 - std::pow(b1, static_cast<double>(t));
            h[2 * t + 1] = 1.0 - std::pow(b2, static_cast<double>(t));
        }
        h[0] = static_cast<double>(tsat > 0 ? tsat : int64_t(1) << 52);  // clamp step
        GASB_CUDA(cudaStreamSynchronize(stream));
        const bool moved = bc.p != nullptr;
        bc.upload(h);
        bc_cap = cap;
        bc_saturated = tsat > 0;
        if (moved) drop_graphs();  // their Adam nodes hold the old address
    }
    void drop_graphs() {
        for (auto& g : graphs)
            if (g) cudaGraphExecDestroy(g), g = nullptr;
        for (auto& g : graphs_dp)
            if (g) cudaGraphExecDestroy(g), g = nullptr;
        for (auto& g : graphs_xf)
            if (g) cudaGraphExecDestroy(g), g = nullptr;
        for (auto& g : graphs_xb)
            if (g) cudaGraphExecDestroy(g), g = nullptr;
    }

    // dropout (ModelSpec.dropout > 0, GCN): per-layer keep masks of the running batch (bit
    // words over the layer input's V_b x d_{l-1} elements) at dmask + dmask_off[l], refilled
    // before every training batch (philox kernels, or the reference's mt19937_64 stream from
    // the host through a 2-slot page-locked ring); the batch runs the materialized path
    bool drop = false;
    float inv_keep = 1.0f;
    DevBuf<uint32_t> dmask;
    // the model's dropout sites (trainer.cpp:142-163, 181-227): seed slot (derive_seed's last
    // argument), width, and whether the input is the B_b batch rows (else all V_b rows)
    std::vector<uint64_t> dslot;
    std::vector<int32_t> dslot_w;
    std::vector<uint8_t> dslot_batch;
    std::vector<int64_t> dmask_off;  // word offset of each site's mask (+ total)
    DevBuf<float> dtmp;              // residual models: layer-1 input gradient before dropout bwd
    const uint32_t* mask_of(uint64_t slot) const {
        for (size_t i = 0; i < dslot.size(); ++i)
            if (dslot[i] == slot) return dmask.p + dmask_off[i];
        throw std::logic_error("dropout: no such site");
    }
    uint32_t* dmask_host[2] = {nullptr, nullptr};
    cudaEvent_t dmask_done[2] = {nullptr, nullptr};
    int dmask_slot = 0;
    void enqueue_masks(int32_t p, int64_t epoch);
    // EpochReport (trainer.hpp:107-115): per part, the stored in-edges of its batch rows
    // (plan.local_graph.num_edges(), summed into edges_per_layer) and the activation floats
    // its step writes; the frozen snapshot tables of the staleness pass (gas_forward_snapshot,
    // trainer.cpp:466-483), allocated on first use
    std::vector<int64_t> part_edges, part_act_floats;
    DevBuf<float> snap;
    size_t mem_free_at_build = 0;
    void enqueue_snapshot();
    void build(const float* h_features, const int32_t* h_labels, const uint8_t* h_train);
    void enqueue_batch(int32_t p, bool train, bool push, bool use_hoisted, bool fused, bool dp = false);
    void enqueue_hoisted();
    // source-blocked hoisted layer 1 (GASB_HOIST_BLOCKS = B > 1, segmented mode): the epoch's
    // edges reordered block-major by source id range, so a chunk pass walks one 1/B slice of X at
    // a time (an L2-sized working set); every row's per-block pieces are fp64 partials combined in
    // block order
    SegTable seg_hoist;
    DevBuf<int32_t> hoist_cols;
    DevBuf<double> hoist_coef, partial_hoist;
    void build_hoist_blocked(const std::vector<int64_t>& rp, const HVec<int32_t>& cg, const HVec<double>& cf,
                             int32_t blocks);
    void run_epoch(int64_t epoch, bool shuffle, int32_t begin = 0, int32_t end = -1);
    // data-parallel mode (dp.cu): batches skip Adam and the step counters (applied after
    // the cross-rank exchange) and have their own per-part graphs
    std::vector<cudaGraphExec_t> graphs_dp;
    DevBuf<char> dp_region;
    // data-parallel layer-1 hoisting over this rank's parts of the epoch (enqueue_hoisted_parts):
    // the parts' stencils are copied contiguously, their segment tables rebuilt per epoch
    std::vector<int64_t> h_rowptr;  // absolute row pointers of the concatenated stencils (R + 1)
    DevBuf<int32_t> sub_cols;
    DevBuf<double> sub_coef;
    DevBuf<int64_t> sub_seg_beg;
    DevBuf<int32_t> sub_seg_row, sub_seg_slot, sub_row_seg0, sub_row_nseg, sub_ranges;
    DevBuf<double> sub_partial;
    std::vector<int64_t> hs_beg;
    std::vector<int32_t> hs_row, hs_slot, hs_r0, hs_rn, hs_ranges;
    // page-locked staging of those tables (asynchronous H2D; reused once the previous
    // epoch's copies, which ran first in that epoch, are done)
    char* sub_pinned = nullptr;
    size_t sub_pinned_bytes = 0;
    cudaEvent_t ev_sub_uploaded = nullptr;
    void enqueue_hoisted_parts(const std::vector<int32_t>& parts);
    // full-graph forward (evaluate / infer_from_history, trainer.cpp:444-536): every row of
    // every part in one launch per layer over the whole-epoch segment table; layer outputs
    // scattered by global id into ping-pong tables the next layer gathers in place
    DevBuf<int32_t> labels_all, eval_flags;
    DevBuf<uint8_t> eval_masks;
    DevBuf<int64_t> eval_counts;
    DevBuf<float> eval_agg, eval_act, eval_tab[2], eval_logits, eval_h0, eval_z, eval_mixed;
    DevBuf<double> eval_partial;
    int64_t eval_pld = 0;
    void ensure_eval();
    void enqueue_full_forward(int32_t first_layer);
    void enqueue_full_forward_res(int32_t first_layer);  // the DP exchange region (grads and act_l are views into it)
    std::vector<int64_t> graph_launches_dp;
    int64_t launch_batch_graph(int32_t p, bool dp);
    void capture_batch_graph(int32_t p, bool dp);
};
