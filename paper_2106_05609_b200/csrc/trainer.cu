// GAS training driver on one B200: Model::build, Model::forward, run_batch and gas_epoch
// of the reference (src/trainer.cpp:55-129, :174-251, :295-339, :386-442) re-designed
// around HBM-resident state and per-batch CUDA graphs.
//
// Data layout in HBM:
//  X        n x ldF fp32 features (ldF = F rounded up to 8 floats: 32 B aligned rows)
//  H_l      HistoryStore tables (history.cu), l = 1..L-1
//  stencils all batches concatenated in part order: cols (int32 global node ids), coeffs
//           (fp64 copies of the reference's fp32 coefficients), row pointers (int64)
//  segments per-batch and whole-epoch segment tables for the SpMM (spmm.cu)
//  CSC      per batch, the intra-batch transposed stencil for the backward gather
//  params   one flat fp32 vector in Model::params() order (+ grads, Adam m, v)
//
// Forward, fused mode (default): after layer l pushes act_l into H_l (fused into the GEMM
// epilogue), H_l[v] for v in V_b equals compose_rows(act_l, pull(halo)) row for row, so
// layer l+1's SpMM gathers H_l in place by global id: no pull, no compose, no x_ext
// gather (value-identical to the reference). Materialized mode keeps the reference's
// structure (gather/pull -> compose -> SpMM over local ids) and optionally prefetches
// the next batch's halos on a side stream (the paper's concurrent execution, §5).
//
// Layer-1 hoisting: agg_1 = A_b X depends on neither parameters nor histories, so when
// dropout == 0 each epoch first runs layer 1's aggregation of ALL batches as one
// chunk-major launch (X streams through L2 once instead of once per batch). Same values,
// same FLOPs, recomputed every epoch.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <type_traits>

#include "trainer_impl.hpp"

namespace gasb {
namespace {

// ---- host RNG exactly as gas::Rng (include/gas/rng.hpp) -------------------------------
uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t s, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
    return mix64(mix64(mix64(s ^ mix64(a)) ^ mix64(b)) ^ mix64(c));
}
struct Rng {
    std::mt19937_64 gen;
    explicit Rng(uint64_t s) : gen(s) {}
    double next_double() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    uint64_t next_below(uint64_t n) {
        if (n <= 1) return 0;
        const uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % n);
        uint64_t x;
        do {
            x = gen();
        } while (x >= limit);
        return x % n;
    }
};
void glorot_init(float* w, int64_t rows, int64_t cols, uint64_t seed) {  // nn.cpp:65-70
    const double bound = std::sqrt(6.0 / static_cast<double>(rows + cols));
    Rng rng(seed);
    for (int64_t i = 0; i < rows * cols; ++i) w[i] = static_cast<float>((rng.next_double() * 2.0 - 1.0) * bound);
}

// Segments each group (batch) of rows of the absolute row pointer `rp` for one SpMM launch
// per group (segment_launch, spmm.cu): split = false keeps rows whole (bit-exact mode).
// Partial slots restart at 0 per group when per_group_slots (one launch at a time).
void build_segments(const std::vector<int64_t>& rp, const std::vector<int64_t>& group_rows, bool split,
                    bool per_group_slots, SegTable& t) {
    const int64_t ngroups = static_cast<int64_t>(group_rows.size()) - 1;
    const int64_t nrows = group_rows.back();
    std::vector<int64_t> sb;
    std::vector<int32_t> sr, ss, r0(static_cast<size_t>(nrows)), rn(static_cast<size_t>(nrows));
    t.group_seg0.assign(static_cast<size_t>(ngroups), 0);
    t.group_nseg.assign(static_cast<size_t>(ngroups), 0);
    t.nranges = spmm_ranges_per_launch();
    t.split = split;
    std::vector<int32_t> rs(static_cast<size_t>(ngroups) * (t.nranges + 1));
    int64_t slot = 0;
    t.max_group_slots = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
        if (per_group_slots) slot = 0;
        t.group_seg0[g] = static_cast<int64_t>(sr.size());
        if (!sb.empty()) sb.pop_back();  // previous group's sentinel
        segment_launch(rp.data(), group_rows[g], group_rows[g + 1], split, t.nranges, sb, sr, ss, r0.data(),
                       rn.data(), slot, rs.data() + g * (t.nranges + 1));
        t.group_nseg[g] = static_cast<int64_t>(sr.size()) - t.group_seg0[g];
        t.max_group_slots = std::max(t.max_group_slots, slot);
    }
    t.total_slots = per_group_slots ? t.max_group_slots : slot;
    t.ranges.upload(rs);
    t.seg_beg.upload(sb);
    t.seg_row.upload(sr);
    t.seg_slot.upload(ss);
    t.row_seg0.upload(r0);
    t.row_nseg.upload(rn);
}

__global__ void end_batch_kernel(int64_t* step, int64_t* t_counter, int stepped) {
    *step += 1;
    if (stepped) *t_counter += 1;
}

// h_ext[i] = is_halo ? halo_rows[k] : act[j]  — compose_rows (tensor.cpp:459-512) for the
// materialized path, one warp per extended row.
__global__ void compose_kernel(const int32_t* __restrict__ src_index, const float* __restrict__ act, int64_t lda,
                               const float* __restrict__ halo, int64_t ldh, int32_t ne, int32_t dim,
                               float* __restrict__ out, int64_t ldo) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= ne) return;
    const int32_t s = src_index[w];  // >= 0: batch index into act, < 0: -(halo index)-1
    const float* src = s >= 0 ? act + static_cast<int64_t>(s) * lda : halo + static_cast<int64_t>(-s - 1) * ldh;
    for (int c = lane; c < dim; c += 32) out[w * ldo + c] = src[c];
}

// evaluate's count (trainer.cpp:449-462): row i (part order) is node v = nodes[i]; its
// prediction is argmax_row (nn.cpp:117-122: first maximum, strict >) of logits row i.
// counts[2k] = rows in mask k, counts[2k+1] = correct rows; preds[v] = prediction.
__global__ void __launch_bounds__(256) argmax_count_kernel(const float* __restrict__ logits, int64_t ldl,
                                                           int64_t rows, int32_t C, const int32_t* __restrict__ nodes,
                                                           const int32_t* __restrict__ labels,
                                                           const uint8_t* __restrict__ masks, int64_t n,
                                                           unsigned long long* __restrict__ counts,
                                                           int32_t* __restrict__ preds) {
    __shared__ unsigned long long sc[6];
    if (threadIdx.x < 6) sc[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < rows) {
        const float* r = logits + i * ldl;
        int32_t best = 0;
        for (int32_t j = 1; j < C; ++j)
            if (r[j] > r[best]) best = j;
        const int32_t v = nodes[i];
        if (preds) preds[v] = best;
        if (masks)
            for (int k = 0; k < 3; ++k)
                if (masks[k * n + v]) {
                    atomicAdd(&sc[2 * k], 1ull);
                    if (best == labels[v]) atomicAdd(&sc[2 * k + 1], 1ull);
                }
    }
    __syncthreads();
    if (threadIdx.x < 6 && sc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], sc[threadIdx.x]);
}

// X[r, :F] = dense[r, :] (row pitch F -> ldF) and flags |= table_flag_of over the values:
// one warp per row, one atomic per CTA.
__global__ void __launch_bounds__(256) repitch_flags_kernel(const float* __restrict__ dense, int64_t rows, int32_t F,
                                                            float* __restrict__ X, int64_t ldF, int32_t* flags) {
    __shared__ int32_t sf;
    if (threadIdx.x == 0) sf = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int32_t f = 0;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const float* src = dense + r * F;
        float* dst = X + r * ldF;
        for (int32_t c = lane; c < F; c += 32) {
            const float v = src[c];
            dst[c] = v;
            f |= table_flag_of(v);
        }
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0 && f) atomicOr(&sf, f);
    __syncthreads();
    if (threadIdx.x == 0 && sf) atomicOr(flags, sf);
}

}  // namespace
}  // namespace gasb
using namespace gasb;

void gasb_trainer_s::build(const float* h_features, const int32_t* h_labels, const uint8_t* h_train) {
    // GASB_TRACE_SETUP=1: wall time of each setup phase on stderr
    const bool trace_on = std::getenv("GASB_TRACE_SETUP") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto trace = [&](const char* what) {
        if (!trace_on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[setup] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const Graph& g = *sched->graph;
    n = g.num_nodes;
    num_parts = sched->num_parts;
    L = spec.num_layers;
    H = spec.hidden;
    require(spec.kind == 0 || spec.kind == 2 || spec.kind == 3,
            "trainer: the device path implements GCN, APPNP and GCNII (GIN is out of scope)");
    require(L >= 1 && H > 0 && F > 0 && C > 0, "trainer: bad model dims");
    drop = spec.dropout > 0.0f;
    require(opt.dropout_rng == GASB_DROPOUT_EXACT || opt.dropout_rng == GASB_DROPOUT_PHILOX,
            "trainer: unknown dropout_rng");
    inv_keep = 1.0f / (1.0f - spec.dropout);  // tensor.cpp:380
    require(spec.l2_weight >= 0.0f, "l2_penalty: negative weight");
    residual = spec.kind != 0;
    D = spec.kind == 2 ? C : H;  // Model::history_dim (trainer.cpp:130-140)
    hist_dim = L >= 2 ? (residual ? D : H) : 0;
    dims.assign(static_cast<size_t>(L) + 1, residual ? D : H);
    dims[0] = F;
    if (!residual) dims[L] = C;
    ldF = ld_of(F);
    ldH = ld_of(H);
    ldC = ld_of(C);
    ldD = ld_of(D);
    ldA = residual ? ldD : ldH;

    // ---- per-part sizes and offsets ----
    nb.resize(num_parts);
    ne.resize(num_parts);
    nh.resize(num_parts);
    ntrain.resize(num_parts);
    row_off.assign(num_parts + 1, 0);
    edge_off.assign(num_parts + 1, 0);
    t_off.assign(num_parts + 1, 0);
    tr_off.assign(num_parts + 1, 0);
    ext_off.assign(num_parts + 1, 0);
    std::vector<int64_t> nintra(num_parts, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t p = 0; p < num_parts; ++p) {
        const HostPlan& P = sched->plans[p];
        nb[p] = static_cast<int32_t>(P.batch.size());
        ne[p] = static_cast<int32_t>(P.extended.size());
        nh[p] = static_cast<int32_t>(P.halo.size());
        int32_t tr = 0;
        for (int32_t v : P.batch) tr += h_train[v] ? 1 : 0;
        ntrain[p] = tr;
        int64_t intra = 0;
        for (int32_t c : P.gcn_cols) intra += P.is_halo[c] ? 0 : 1;
        nintra[p] = intra;
    }
    for (int32_t p = 0; p < num_parts; ++p) {
        row_off[p + 1] = row_off[p] + nb[p];
        edge_off[p + 1] = edge_off[p] + static_cast<int64_t>(sched->plans[p].gcn_cols.size());
        t_off[p + 1] = t_off[p] + nintra[p];
        tr_off[p + 1] = tr_off[p] + ntrain[p];
        ext_off[p + 1] = ext_off[p] + ne[p];
        nb_max = std::max(nb_max, nb[p]);
        ne_max = std::max(ne_max, ne[p]);
    }
    const int64_t R = row_off[num_parts], E = edge_off[num_parts], T = t_off[num_parts], NE = ext_off[num_parts];
    trace("sizes");

    // ---- host staging of the concatenated stencils ----
    std::vector<int32_t> h_bn(R), h_trr(tr_off[num_parts]), h_trl(tr_off[num_parts]);
    HVec<int32_t> h_cg(E), h_cl(E), h_tsrc(T), h_ext(NE), h_cidx(NE);
    std::vector<int32_t> h_rlab(R);
    HVec<double> h_cf(E);
    HVec<float> h_tcf(T);
    std::vector<int64_t> h_rp(R + 1), h_trp(R + num_parts);
    h_rp[R] = E;
    // residual models: batch_local_rows, and the all-edge CSC for the layer-1 backward
    std::vector<int32_t> h_brow;
    HVec<int32_t> h_asrc;
    HVec<float> h_acf;
    std::vector<int64_t> h_arp;
    if (residual || drop) h_brow.resize(R);
    if (residual) {
        h_asrc.resize(E);
        h_acf.resize(E);
        h_arp.resize(NE + num_parts);
        a_off.resize(num_parts);
        for (int32_t p = 0; p < num_parts; ++p) a_off[p] = ext_off[p] + p;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t p = 0; p < num_parts; ++p) {
        const HostPlan& P = sched->plans[p];
        const int64_t r0 = row_off[p], e0 = edge_off[p];
        std::vector<int32_t> local2batch(P.extended.size(), -1);
        for (int32_t i = 0; i < nb[p]; ++i) {
            h_bn[r0 + i] = P.batch[i];
            local2batch[P.batch_local_rows[i]] = i;
            h_rp[r0 + i] = e0 + P.gcn_rowptr[i];
        }
        for (size_t e = 0; e < P.gcn_cols.size(); ++e) {
            h_cg[e0 + e] = P.extended[P.gcn_cols[e]];
            h_cl[e0 + e] = P.gcn_cols[e];
            h_cf[e0 + e] = static_cast<double>(P.gcn_coeffs[e]) * kCoeffScale;  // exact (see spmm.cu)
        }
        // transposed intra-batch stencil: target = batch index of the source row, entries
        // in ascending dst row r (the reference's scatter order, tensor.cpp:540-547)
        std::vector<int64_t> cnt(static_cast<size_t>(nb[p]) + 1, 0);
        for (size_t e = 0; e < P.gcn_cols.size(); ++e) {
            const int32_t t = local2batch[P.gcn_cols[e]];
            if (t >= 0) cnt[t + 1]++;
        }
        for (int32_t t = 0; t < nb[p]; ++t) cnt[t + 1] += cnt[t];
        int64_t* trp = h_trp.data() + r0 + p;  // nb+1 entries per part
        for (int32_t t = 0; t <= nb[p]; ++t) trp[t] = t_off[p] + cnt[t];
        std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
        for (int32_t r = 0; r < nb[p]; ++r)
            for (int64_t e = P.gcn_rowptr[r]; e < P.gcn_rowptr[r + 1]; ++e) {
                const int32_t t = local2batch[P.gcn_cols[e]];
                if (t < 0) continue;
                const int64_t k = t_off[p] + fill[t]++;
                h_tsrc[k] = r;
                h_tcf[k] = P.gcn_coeffs[e];
            }
        int32_t k = 0;
        for (int32_t i = 0; i < nb[p]; ++i) {
            h_rlab[r0 + i] = h_train[P.batch[i]] ? h_labels[P.batch[i]] : -1;
            if (h_train[P.batch[i]]) {
                h_trr[tr_off[p] + k] = i;
                h_trl[tr_off[p] + k] = h_labels[P.batch[i]];
                ++k;
            }
        }
        int32_t hk = 0;
        for (int32_t i = 0; i < ne[p]; ++i) {
            h_ext[ext_off[p] + i] = P.extended[i];
            h_cidx[ext_off[p] + i] = P.is_halo[i] ? -(hk++) - 1 : local2batch[i];
        }
        if (residual || drop)
            for (int32_t i = 0; i < nb[p]; ++i) h_brow[r0 + i] = P.batch_local_rows[i];
        if (residual) {
            // transposed stencil over every V_b target (tensor.cpp:531-549 writes all rows of
            // h_in; layer 1 of APPNP/GCNII keeps the halo rows)
            std::vector<int64_t> ac(static_cast<size_t>(ne[p]) + 1, 0);
            for (int32_t c : P.gcn_cols) ac[c + 1]++;
            for (int32_t t = 0; t < ne[p]; ++t) ac[t + 1] += ac[t];
            int64_t* arp = h_arp.data() + a_off[p];
            for (int32_t t = 0; t <= ne[p]; ++t) arp[t] = e0 + ac[t];
            for (int32_t r = 0; r < nb[p]; ++r)
                for (int64_t e = P.gcn_rowptr[r]; e < P.gcn_rowptr[r + 1]; ++e) {
                    const int64_t k = e0 + ac[P.gcn_cols[e]]++;
                    h_asrc[k] = r;
                    h_acf[k] = P.gcn_coeffs[e];
                }
        }
    }
    for (int32_t i = 0; i < static_cast<int32_t>(h_trl.size()); ++i)
        require(h_trl[i] >= 0 && h_trl[i] < C, "softmax_cross_entropy: label out of range");
    trace("host staging");

    GASB_CUDA(cudaSetDevice(opt.device));
    {
        size_t fr = 0, tot = 0;
        GASB_CUDA(cudaMemGetInfo(&fr, &tot));
        mem_free_at_build = fr;
    }
    // cross-batch mode (gasb.h cross_batch; GASB_XBATCH overrides): GCN over the fused,
    // segmented path without dropout
    {
        const char* xe = getenv("GASB_XBATCH");
        xmode = xe ? atoi(xe) : opt.cross_batch;
        const bool ok = !residual && opt.fused && !drop && L >= 2 && opt.seg_edges > 0;
        xmode = ok ? std::max(0, std::min(2, xmode)) : 0;
        if (xmode == 1 && !opt.hoist_layer1) xmode = 2;  // layer 1 per batch then
        const char* be = getenv("GASB_BG_CTAS");
        bg_ctas = be ? std::max(0, atoi(be)) : 148;
    }
    if (xmode) {
        // the batch chain (stream, side) outranks the background aggregations at CTA dispatch
        int least = 0, greatest = 0;
        GASB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        GASB_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, greatest));
        GASB_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, greatest));
        GASB_CUDA(cudaStreamCreateWithPriority(&bg, cudaStreamNonBlocking, least));
        for (cudaEvent_t* e : {&ev_xstart, &ev_xfwd, &ev_xbg})
            GASB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    } else {
        GASB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        GASB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    }
    GASB_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    GASB_CUDA(cudaEventCreateWithFlags(&ev_staged, cudaEventDisableTiming));
    GASB_CUDA(cudaEventCreateWithFlags(&ev_stage_free, cudaEventDisableTiming));
    trace("cuda context + streams");
    batch_nodes.upload(h_bn);
    cols_g.upload(h_cg);
    cols_l.upload(h_cl);
    coef64.upload(h_cf);
    t_src.upload(h_tsrc);
    t_cf.upload(h_tcf);
    t_rowptr.upload(h_trp);
    {  // per part: intra-batch targets heaviest first (spmm_bwd claims them in this order)
        std::vector<int32_t> h_ord(static_cast<size_t>(R));
#pragma omp parallel for schedule(dynamic, 1)
        for (int32_t p = 0; p < num_parts; ++p) {
            int32_t* o = h_ord.data() + row_off[p];
            const int64_t* trp = h_trp.data() + row_off[p] + p;
            std::iota(o, o + nb[p], 0);
            std::stable_sort(o, o + nb[p], [&](int32_t a, int32_t b) {
                return trp[a + 1] - trp[a] > trp[b + 1] - trp[b];
            });
        }
        t_order.upload(h_ord);
    }
    {  // spmm_bwd2 plans (GASB_BWD2=0: the one-column-per-lane kernel everywhere)
        const char* e = getenv("GASB_BWD2");
        use_bwd2 = (!e || atoi(e) != 0) && H >= 64;
        if (use_bwd2) {
            std::vector<int64_t> boff;
            std::vector<unsigned char> blobs;
            bwd2_splits = spmm_bwd2_splits(H);
            bwd2_off.resize(num_parts);
            bwd2_ok.resize(num_parts);
            for (int32_t p = 0; p < num_parts; ++p) {
                bwd2_off[p] = static_cast<int64_t>(boff.size());
                bwd2_ok[p] = build_bwd2_plan(h_trp.data() + row_off[p] + p, h_tsrc.data(), h_tcf.data(), nb[p], nb[p],
                                             bwd2_splits, boff, blobs);
                boff.push_back(static_cast<int64_t>(blobs.size()));  // the part's end offset
            }
            bwd2_boff.upload(boff);
            bwd2_blobs.upload(blobs);
        }
    }
    trace("stencil uploads + t_order");
    train_rows.upload(h_trr);
    train_labels.upload(h_trl);
    row_label.upload(h_rlab);
    labels_all.upload(std::vector<int32_t>(h_labels, h_labels + n));
    extended.upload(h_ext);
    compose_idx.upload(h_cidx);
    {
        std::vector<int64_t> grp(num_parts + 1);
        for (int32_t p = 0; p <= num_parts; ++p) grp[p] = row_off[p];
        build_segments(h_rp, grp, opt.seg_edges > 0, true, seg_batch);
        h_rowptr = h_rp;
        std::vector<int64_t> one{0, R};
        build_segments(h_rp, one, opt.seg_edges > 0, false, seg_all);
    }
    trace("segments");
    if (xmode) {
        build_xbatch(h_rp, h_cg, h_cf);
        trace("cross-batch tables");
    }
    max_chunks = static_cast<int32_t>(ceil_div(std::max(F, H), 64));
    counters.alloc(R * max_chunks);
    counters.zero();
    pld = round_up(std::max(F, H), 256);  // fp64 partial row width, any SpMM chunk width (64 | 128 | 256)
    pld_all = round_up(F, 256);
    partial_batch.alloc(std::max<int64_t>(seg_batch.max_group_slots, 1) * pld);
    partial_all.alloc(std::max<int64_t>(seg_all.total_slots, 1) * pld_all);
    {
        // GASB_HOIST_BLOCKS: source blocks of the hoisted layer 1 (1 = off)
        const char* hbe = getenv("GASB_HOIST_BLOCKS");
        const int32_t hb = hbe ? std::max(1, std::min(64, atoi(hbe))) : 1;
        if (hb > 1 && opt.hoist_layer1 && opt.fused && !residual && opt.seg_edges > 0) {
            build_hoist_blocked(h_rp, h_cg, h_cf, hb);
            trace("blocked hoist table");
        }
    }

    // ---- features ----
    X.alloc(static_cast<int64_t>(n) * ldF);
    GASB_CUDA(cudaMemcpy2D(X.p, sizeof(float) * ldF, h_features, sizeof(float) * F, sizeof(float) * F, n,
                           cudaMemcpyHostToDevice));
    if (ldF > F)
        GASB_CUDA(cudaMemset2D(X.p + F, sizeof(float) * ldF, 0, sizeof(float) * (ldF - F), n));
    // SpMM source tables free of denormal / non-finite values take the integer widening path
    xflags.alloc(1);
    xflags.zero();
    launch_scan_special(X.p, n, ldF, F, xflags.p, nullptr);
    ce_done.alloc(1);
    ce_done.zero();
    trace("features");

    // ---- Model::build (trainer.cpp:55-129); params in Model::params() order ----
    layer_param.assign(static_cast<size_t>(L) + 1, -1);
    if (!residual) {  // GCN: W_l (d_{l-1} x d_l)
        for (int32_t l = 1; l <= L; ++l) layer_param[l] = add_param(dims[l - 1], dims[l]);
    } else {  // head_w1, head_b1, [head_w2, head_b2], [W_l], [out_w, out_b]
        p_hw1 = add_param(F, H);
        p_hb1 = add_param(1, H);
        if (spec.kind == 2) {
            p_hw2 = add_param(H, C);
            p_hb2 = add_param(1, C);
        } else {
            for (int32_t l = 1; l <= L; ++l) layer_param[l] = add_param(H, H);
            p_ow = add_param(H, C);
            p_ob = add_param(1, C);
        }
    }
    h_params_init.assign(static_cast<size_t>(nparam), 0.0f);
    auto glorot_at = [&](int32_t i, uint64_t seed) {
        std::vector<float> w(static_cast<size_t>(prow[i] * pcol[i]));
        glorot_init(w.data(), prow[i], pcol[i], seed);
        for (int64_t r = 0; r < prow[i]; ++r)
            std::copy(w.begin() + r * pcol[i], w.begin() + (r + 1) * pcol[i],
                      h_params_init.begin() + poff[i] + r * ppitch[i]);
    };
    for (int32_t l = 1; l <= L; ++l)  // Layer::build(cfg, derive_seed(seed,10,l)) -> glorot(derive_seed(.,1))
        if (layer_param[l] >= 0)
            glorot_at(layer_param[l], derive_seed(derive_seed(spec.seed, 10, static_cast<uint64_t>(l)), 1));
    if (p_hw1 >= 0) glorot_at(p_hw1, derive_seed(spec.seed, 20, 1));  // seed_for(20, 1)
    if (p_hw2 >= 0) glorot_at(p_hw2, derive_seed(spec.seed, 20, 2));
    if (p_ow >= 0) glorot_at(p_ow, derive_seed(spec.seed, 30, 1));
    params.upload(h_params_init);
    grads.alloc(nparam);
    grads.zero();
    adam_m.alloc(nparam);
    adam_m.zero();
    adam_v.alloc(nparam);
    adam_v.zero();
    t_counter.alloc(1);
    t_counter.zero();
    adam_done.alloc(1);
    adam_done.zero();
    norm_scratch.alloc(512);  // [0, 256): clip norm, [256, 512): l2 penalty
    ensure_bc(4096);

    // ---- HistoryStore(L-1, n, H) ----
    hist = history_create(std::max(0, L - 1), n, hist_dim);
    trace("params + history");

    // ---- activations ----
    agg.resize(static_cast<size_t>(L) + 1);
    act.resize(static_cast<size_t>(L) + 1);
    if (!residual) {
        for (int32_t l = 1; l <= L; ++l) agg[l].alloc(static_cast<int64_t>(nb_max) * ld_of(dims[l - 1]));
        for (int32_t l = 1; l < L; ++l) act[l].alloc(static_cast<int64_t>(nb_max) * ldH);
        if (opt.hoist_layer1 || xmode) agg_all.alloc(R * ldF);
    } else {
        build_residual(h_arp, h_asrc, h_acf, h_brow);
    }
    logits.alloc(static_cast<int64_t>(nb_max) * ldC);
    glogits.alloc(static_cast<int64_t>(nb_max) * ldC);
    g_agg.alloc(static_cast<int64_t>(nb_max) * std::max(ldH, ldC));
    g_out.alloc(static_cast<int64_t>(nb_max) * ldH);
    loss.alloc(num_parts);
    loss.zero();
    if (residual) colsum_ws.alloc(kColsumWsDoubles);
    gemm_ws.alloc(kGemmWsFloats + kGemmTileCounters);  // split-K slices + tile counters
    gemm_ws.zero();
    if (!residual) {
        gemm_ws2.alloc(kGemmWsFloats + kGemmTileCounters);
        gemm_ws2.zero();
        g_out2.alloc(static_cast<int64_t>(nb_max) * ldH);
        ev_fork.assign(static_cast<size_t>(L) + 1, nullptr);
        ev_wdone.assign(static_cast<size_t>(L) + 1, nullptr);
        for (int32_t l = 0; l <= L; ++l) {
            GASB_CUDA(cudaEventCreateWithFlags(&ev_fork[l], cudaEventDisableTiming));
            GASB_CUDA(cudaEventCreateWithFlags(&ev_wdone[l], cudaEventDisableTiming));
        }
        GASB_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    row_scratch.alloc(nb_max);
    if (drop) {
        if (!residual) brow.upload(h_brow);
        // dropout sites in the reference's forward order
        auto site = [&](uint64_t slot, int32_t w, bool batch_rows) {
            dslot.push_back(slot);
            dslot_w.push_back(w);
            dslot_batch.push_back(batch_rows ? 1 : 0);
        };
        if (residual) {
            site(100, F, false);  // head input x_ext (trainer.cpp:149/158)
            if (spec.kind == 2) site(101, H, false);  // APPNP head hidden (:151)
        }
        for (int32_t l = 1; l <= L; ++l) site(static_cast<uint64_t>(l), dims[l - 1], false);  // layer inputs (:203-204)
        if (spec.kind == 3) site(9000, H, true);  // GCNII output head input (:222-223)
        dmask_off.assign(dslot.size() + 1, 0);
        for (size_t i = 0; i < dslot.size(); ++i)
            dmask_off[i + 1] = dmask_off[i] + round_up(ceil_div(static_cast<int64_t>(dslot_batch[i] ? nb_max : ne_max) *
                                                                    dslot_w[i], 32), 32);
        const int64_t words = dmask_off.back();
        dmask.alloc(words);
        if (residual) dtmp.alloc(static_cast<int64_t>(ne_max) * ldD);
        if (opt.dropout_rng == GASB_DROPOUT_EXACT)
            for (int i = 0; i < 2; ++i) {
                GASB_CUDA(cudaHostAlloc(&dmask_host[i], sizeof(uint32_t) * words, cudaHostAllocDefault));
                GASB_CUDA(cudaEventCreateWithFlags(&dmask_done[i], cudaEventDisableTiming));
                GASB_CUDA(cudaEventRecord(dmask_done[i], stream));
            }
    }
    // EpochReport bookkeeping (host): stored in-edges of each batch's rows, and the activation
    // floats of its step: every forward layer input/output over the batch rows (+ the residual
    // heads over all V_b rows) and their gradients (GCN's layer-1 input has none)
    part_edges.assign(num_parts, 0);
    part_act_floats.assign(num_parts, 0);
    for (int32_t p = 0; p < num_parts; ++p) {
        const Graph& G = *sched->graph;
        for (int32_t v : sched->plans[p].batch) part_edges[p] += G.row_offsets[v + 1] - G.row_offsets[v];
        int64_t fwd = 0;
        for (int32_t l = 1; l <= L; ++l) fwd += static_cast<int64_t>(nb[p]) * (dims[l - 1] + dims[l]);
        if (residual) fwd += static_cast<int64_t>(ne[p]) * (F + H + D);
        part_act_floats[p] = 2 * fwd - (residual ? 0 : static_cast<int64_t>(nb[p]) * F);
    }
    graphs.assign(num_parts, nullptr);
    graph_launches.assign(num_parts, 0);
    GASB_CUDA(cudaDeviceSynchronize());
    trace("activations + sync");
}

// Layer 1 hoisted over a subset of parts (one data-parallel rank's batches of an epoch):
// the parts' edges are copied into one contiguous stream, segments / ranges are built on the
// host over that stream (rows keep their absolute ids, so the output lands in agg_all where
// the per-part graphs read it), and one chunk-major launch aggregates them all.
void gasb_trainer_s::enqueue_hoisted_parts(const std::vector<int32_t>& parts) {
    std::vector<int64_t> vrp(1, 0);  // virtual (contiguous) row pointers
    std::vector<int32_t> vrow;       // virtual row -> absolute row
    int64_t E = 0;
    for (int32_t p : parts) {
        for (int64_t r = row_off[p]; r < row_off[p + 1]; ++r) {
            E += h_rowptr[r + 1] - h_rowptr[r];
            vrp.push_back(E);
            vrow.push_back(static_cast<int32_t>(r));
        }
    }
    const int64_t R = row_off[num_parts], rows = static_cast<int64_t>(vrow.size());
    if (rows == 0) return;
    hs_beg.clear();
    hs_row.clear();
    hs_slot.clear();
    std::vector<int32_t> r0(static_cast<size_t>(rows)), rn(static_cast<size_t>(rows));
    const int32_t nr = spmm_ranges_per_launch();
    hs_ranges.assign(static_cast<size_t>(nr) + 1, 0);
    int64_t slot = 0;
    segment_launch(vrp.data(), 0, rows, opt.seg_edges > 0, nr, hs_beg, hs_row, hs_slot, r0.data(), rn.data(), slot,
                   hs_ranges.data());
    for (auto& r : hs_row) r = vrow[r];  // segments name absolute rows
    hs_r0.assign(static_cast<size_t>(R), 0);
    hs_rn.assign(static_cast<size_t>(R), 0);
    for (int64_t v = 0; v < rows; ++v) {
        hs_r0[vrow[v]] = r0[v];
        hs_rn[vrow[v]] = rn[v];
    }
    if (sub_cols.n < E) {
        GASB_CUDA(cudaStreamSynchronize(stream));
        sub_cols.alloc(E);
        sub_coef.alloc(E);
    }
    int64_t off = 0;
    for (int32_t p : parts) {
        const int64_t e0 = h_rowptr[row_off[p]], e1 = h_rowptr[row_off[p + 1]];
        GASB_CUDA(cudaMemcpyAsync(sub_cols.p + off, cols_g.p + e0, sizeof(int32_t) * (e1 - e0),
                                  cudaMemcpyDeviceToDevice, stream));
        GASB_CUDA(cudaMemcpyAsync(sub_coef.p + off, coef64.p + e0, sizeof(double) * (e1 - e0),
                                  cudaMemcpyDeviceToDevice, stream));
        off += e1 - e0;
    }
    // tables -> page-locked staging -> device, all stream-ordered (no host synchronisation)
    auto bytes_of = [](const auto& v) { return (sizeof(v[0]) * v.size() + 255) / 256 * 256; };
    const size_t total = bytes_of(hs_beg) + bytes_of(hs_row) + bytes_of(hs_slot) + bytes_of(hs_r0) + bytes_of(hs_rn) +
                         bytes_of(hs_ranges);
    if (!ev_sub_uploaded) GASB_CUDA(cudaEventCreateWithFlags(&ev_sub_uploaded, cudaEventDisableTiming));
    GASB_CUDA(cudaEventSynchronize(ev_sub_uploaded));  // the previous epoch's copies (long done)
    if (sub_pinned_bytes < total) {
        if (sub_pinned) GASB_CUDA(cudaFreeHost(sub_pinned));
        GASB_CUDA(cudaHostAlloc(&sub_pinned, total, cudaHostAllocDefault));
        sub_pinned_bytes = total;
    }
    size_t po = 0;
    auto stage = [&](auto& dev, const auto& v) {
        using T = std::decay_t<decltype(v[0])>;
        if (dev.n < static_cast<int64_t>(v.size())) {
            GASB_CUDA(cudaStreamSynchronize(stream));
            dev.alloc(static_cast<int64_t>(v.size()));
        }
        std::memcpy(sub_pinned + po, v.data(), sizeof(T) * v.size());
        GASB_CUDA(cudaMemcpyAsync(dev.p, sub_pinned + po, sizeof(T) * v.size(), cudaMemcpyHostToDevice, stream));
        po += bytes_of(v);
    };
    stage(sub_seg_beg, hs_beg);
    stage(sub_seg_row, hs_row);
    stage(sub_seg_slot, hs_slot);
    stage(sub_row_seg0, hs_r0);
    stage(sub_row_nseg, hs_rn);
    stage(sub_ranges, hs_ranges);
    GASB_CUDA(cudaEventRecord(ev_sub_uploaded, stream));
    const int64_t need = std::max<int64_t>(slot, 1) * pld_all;
    if (sub_partial.n < need) {
        GASB_CUDA(cudaStreamSynchronize(stream));
        sub_partial.alloc(need);
    }
    SpmmSegs segs{sub_seg_beg.p, sub_seg_row.p, sub_seg_slot.p, sub_row_seg0.p, sub_row_nseg.p, sub_ranges.p, nr,
                  opt.seg_edges > 0 ? 0 : 1};
    launch_spmm_fwd(segs, sub_cols.p, sub_coef.p, X.p, ldF, F, agg_all.p, ldF, 0, sub_partial.p, pld_all, counters.p,
                    max_chunks, stream, source_flags(1), source_tmap(1));
}

void gasb_trainer_s::enqueue_hoisted() {
    if (hoist_cols.p) {
        launch_spmm_fwd(seg_hoist.segs(0), hoist_cols.p, hoist_coef.p, X.p, ldF, F, agg_all.p, ldF, 0,
                        partial_hoist.p, pld_all, counters.p, max_chunks, stream, source_flags(1), source_tmap(1));
        return;
    }
    launch_spmm_fwd(seg_all.segs(0), cols_g.p, coef64.p, X.p, ldF, F, agg_all.p, ldF, 0, partial_all.p, pld_all,
                    counters.p, max_chunks, stream, source_flags(1), source_tmap(1));
}

void gasb_trainer_s::spmm_bwd_batch(int32_t p, const float* gy, int64_t ldgy, int32_t dim, const float* mask,
                                    int64_t ldm, float* gx, int64_t ldgx, cudaStream_t st) {
    const int64_t r0 = row_off[p];
    const int32_t m = nb[p];
    if (use_bwd2 && bwd2_ok[p] && dim == H &&
        launch_spmm_bwd2(bwd2_boff.p + bwd2_off[p], bwd2_blobs.p, bwd2_splits, gy, ldgy, dim, mask, ldm, gx, ldgx, st,
                         m, false))
        return;
    launch_spmm_bwd(t_rowptr.p + r0 + p, m, t_src.p, t_cf.p, gy, ldgy, dim, mask, ldm, gx, ldgx, st, m, false,
                    t_order.p + r0);
}

void gasb_trainer_s::build_hoist_blocked(const std::vector<int64_t>& rp, const HVec<int32_t>& cg,
                                         const HVec<double>& cf, int32_t B) {
    const int64_t R = static_cast<int64_t>(rp.size()) - 1, E = rp[R];
    auto blk = [&](int32_t c) { return static_cast<int32_t>(static_cast<int64_t>(c) * B / n); };
    // pieces (block, row) laid out block-major; piece offsets by an exclusive scan in that order
    std::vector<int64_t> off(static_cast<size_t>(B) * R + 1, 0);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < R; ++r)
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) ++off[static_cast<size_t>(blk(cg[e])) * R + r + 1];
    for (size_t i = 1; i < off.size(); ++i) off[i] += off[i - 1];
    HVec<int32_t> hc(static_cast<size_t>(E));
    HVec<double> hf(static_cast<size_t>(E));
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < R; ++r) {
        int64_t pos[64];
        for (int32_t b = 0; b < B; ++b) pos[b] = off[static_cast<size_t>(b) * R + r];
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {  // CSR order within each piece
            const int32_t b = blk(cg[e]);
            hc[pos[b]] = cg[e];
            hf[pos[b]] = cf[e];
            ++pos[b];
        }
    }
    // ranges: each block's edges cut into one range per resident warp, so that the persistent
    // grid (warp w takes ranges w, w + W, ...) walks the blocks roughly in lockstep and the
    // concurrently gathered source rows stay within one block. Segments: the pieces in
    // sequence, cut where a range boundary falls inside
    const int32_t W = spmm_ranges_per_launch(), nr = W * B;
    std::vector<int64_t> bnd(static_cast<size_t>(nr) + 1);
    for (int32_t b = 0; b < B; ++b) {
        const int64_t e0 = off[static_cast<size_t>(b) * R], e1 = off[static_cast<size_t>(b + 1) * R];
        for (int32_t q = 0; q < W; ++q) bnd[static_cast<size_t>(b) * W + q] = e0 + (e1 - e0) * q / W;
    }
    bnd[nr] = E;
    auto bound = [&](int64_t k) { return bnd[static_cast<size_t>(k)]; };
    std::vector<int64_t> sb;
    std::vector<int32_t> sr;
    sb.reserve(static_cast<size_t>(B) * R + nr + 1);
    sr.reserve(static_cast<size_t>(B) * R + nr + 1);
    int64_t k = 1;
    for (int64_t i = 0; i < static_cast<int64_t>(B) * R; ++i) {
        const int64_t b0 = off[i], b1 = off[i + 1];
        if (b0 == b1) continue;
        const int32_t row = static_cast<int32_t>(i % R);
        while (k < nr && bound(k) <= b0) ++k;
        sb.push_back(b0);
        sr.push_back(row);
        for (; k < nr && bound(k) < b1; ++k)
            if (sb.back() != bound(k)) {
                sb.push_back(bound(k));
                sr.push_back(row);
            }
    }
    const int64_t nseg = static_cast<int64_t>(sr.size());
    sb.push_back(E);
    // slots: rows with more than one segment get one per segment; the row's slot list in
    // sequence (block) order
    std::vector<int32_t> rn(static_cast<size_t>(R), 0), r0(static_cast<size_t>(R), 0), ss(static_cast<size_t>(nseg));
    for (int64_t s = 0; s < nseg; ++s) ++rn[sr[s]];
    int64_t slots = 0, acc = 0;
    for (int64_t r = 0; r < R; ++r) {
        r0[r] = static_cast<int32_t>(acc);
        acc += rn[r];
    }
    std::vector<int32_t> fill(r0), rs(static_cast<size_t>(acc));
    for (int64_t s = 0; s < nseg; ++s) {
        const int32_t r = sr[s];
        ss[s] = rn[r] == 1 ? -1 : static_cast<int32_t>(slots++);
        rs[fill[r]++] = ss[s];
    }
    std::vector<int32_t> ranges(static_cast<size_t>(nr) + 1);
    {
        int64_t s = 0;
        ranges[0] = 0;
        for (int32_t q = 1; q < nr; ++q) {
            const int64_t t = bound(q);
            while (s < nseg && sb[s] < t) ++s;
            ranges[q] = static_cast<int32_t>(s);
        }
        ranges[nr] = static_cast<int32_t>(nseg);
    }
    seg_hoist.nranges = nr;
    seg_hoist.split = true;
    seg_hoist.total_slots = slots;
    seg_hoist.seg_beg.upload(sb);
    seg_hoist.seg_row.upload(sr);
    seg_hoist.seg_slot.upload(ss);
    seg_hoist.row_seg0.upload(r0);
    seg_hoist.row_nseg.upload(rn);
    seg_hoist.row_slots.upload(rs);
    seg_hoist.ranges.upload(ranges);
    hoist_cols.upload(hc);
    hoist_coef.upload(hf);
    partial_hoist.alloc(std::max<int64_t>(slots, 1) * pld_all);
}

void gasb_trainer_s::build_residual(const std::vector<int64_t>& h_arp, const HVec<int32_t>& h_asrc,
                                    const HVec<float>& h_acf, const std::vector<int32_t>& h_brow) {
    brow.upload(h_brow);
    a_rowptr.upload(h_arp);
    a_src.upload(h_asrc);
    a_cf.upload(h_acf);
    const int64_t nbm = nb_max, nem = ne_max;
    h0.alloc(nem * ldD);
    h0g.alloc(nem * ldD);
    if (spec.kind == 2) {
        z.alloc(nem * ldH);
        zg.alloc(nem * ldH);
    } else {
        wt.alloc(static_cast<int64_t>(L) * H * round_up(H, 4));
        mixed.resize(static_cast<size_t>(L) + 1);
        for (int32_t l = 1; l <= L; ++l) mixed[l].alloc(nbm * ldD);
    }
    for (int32_t l = 1; l <= L; ++l)
        if (l < L || spec.kind == 3) act[l].alloc(nbm * ldD);
    prop.alloc(nbm * ldD);
    gmix.alloc(nbm * ldD);
    dprop.alloc(nbm * ldD);
    gout.alloc(nbm * ldD);
}

void gasb_trainer_s::enqueue_prefetch(int32_t p) {
    GASB_CUDA(cudaEventRecord(ev_pf_start, stream));  // after the previous batch's pushes
    GASB_CUDA(cudaStreamWaitEvent(side, ev_pf_start, 0));
    for (int32_t l = 1; l < L; ++l) {
        launch_rows(1, halo_ids.p + (ext_off[p] - row_off[p]), nh[p], history_table(hist, l), history_ld(hist),
                    halo_pf.p + static_cast<int64_t>(l - 1) * halo_pf_rows * halo_pf_ld, halo_pf_ld, hist_dim, n,
                    nullptr, nullptr, nullptr, side);
        GASB_CUDA(cudaEventRecord(ev_pf[l], side));
    }
}

// APPNP / GCNII batch: Model::forward (trainer.cpp:174-251) with head_forward over all V_b
// rows (:142-163), appnp/gcnii layers (layers.cpp:150-168), the GCNII output head
// (:221-227), then run_batch's backward (halo rows of h0 receive the layer-1 aggregation
// gradient) and Adam.
void gasb_trainer_s::enqueue_batch_res(int32_t p, bool train, bool push, bool fused, bool dp) {
    const int32_t m = nb[p], me = ne[p];
    const int64_t r0 = row_off[p];
    const SpmmSegs segs = seg_batch.segs(p);
    const int32_t* bn = batch_nodes.p + r0;
    const int32_t* br = brow.p + r0;
    const bool gcnii = spec.kind == 3;
    const bool dr = drop && train;  // dropout only while training (ForwardOptions.training)
    require(!dr || !fused, "trainer: dropout batches run the materialized path");
    if (!fused && halo_pf.p) enqueue_prefetch(p);
    // ---- head_forward over the extended rows: x_ext = X[V_b] (gather_features, trainer.cpp:20-27)
    launch_rows(1, extended.p + ext_off[p], me, X.p, ldF, x_ext.p, ldF, F, n, nullptr, nullptr, nullptr, stream);
    if (dr) launch_dropout_apply(x_ext.p, ldF, me, F, mask_of(100), inv_keep, stream);  // trainer.cpp:149/158
    {
        GemmEpilogue e1;
        e1.bias = P(p_hb1);
        e1.relu = 1;
        launch_gemm(0, me, H, F, x_ext.p, ldF, P(p_hw1), pp(p_hw1), gcnii ? h0.p : z.p, gcnii ? ldD : ldH, e1, stream);
        // APPNP head hidden (trainer.cpp:151): dropped in place — dropped z > 0 exactly where the
        // relu mask and the keep mask both hold, so the backward's relu mask reads it as well
        if (!gcnii && dr) launch_dropout_apply(z.p, ldH, me, H, mask_of(101), inv_keep, stream);
        if (!gcnii) {
            GemmEpilogue e2;
            e2.bias = P(p_hb2);
            launch_gemm(0, me, C, H, z.p, ldH, P(p_hw2), pp(p_hw2), h0.p, ldD, e2, stream);
        }
    }
    if (gcnii) launch_wtilde(P(layer_param[1]), wt.p, L, H, pp(layer_param[1]), spec.beta, stream);
    // ---- propagation layers ----
    for (int32_t l = 1; l <= L; ++l) {
        if (l == 1 && dr) {  // input = dropout(h0) over V_b (trainer.cpp:203-204; h0 itself feeds the mixing)
            GASB_CUDA(cudaMemcpy2DAsync(h_ext.p, sizeof(float) * ldD, h0.p, sizeof(float) * ldD, sizeof(float) * D, me,
                                        cudaMemcpyDeviceToDevice, stream));
            launch_dropout_apply(h_ext.p, ldD, me, D, mask_of(1), inv_keep, stream);
            launch_spmm_fwd(segs, cols_l.p, coef64.p, h_ext.p, ldD, D, prop.p, ldD, r0, partial_batch.p, pld,
                            counters.p, max_chunks, stream, nullptr, tm_ok[3] ? &tm_hext : nullptr);
        } else if (l == 1) {  // input = h0 over V_b (local ids)
            launch_spmm_fwd(segs, cols_l.p, coef64.p, h0.p, ldD, D, prop.p, ldD, r0, partial_batch.p, pld, counters.p,
                            max_chunks, stream, nullptr, tm_h0_ok ? &tm_h0 : nullptr);
        } else if (fused) {  // pull-free: H_{l-1} by global id
            launch_spmm_fwd(segs, cols_g.p, coef64.p, history_table(hist, l - 1), history_ld(hist), D, prop.p, ldD, r0,
                            partial_batch.p, pld, counters.p, max_chunks, stream, source_flags(l), source_tmap(l));
        } else {  // pull halos (or wait for the prefetched copy), compose_rows, SpMM over local ids
            const float* halo = halo_buf.p;
            int64_t ldh = ldD;
            if (halo_pf.p) {
                GASB_CUDA(cudaStreamWaitEvent(stream, ev_pf[l - 1], 0));
                halo = halo_pf.p + static_cast<int64_t>(l - 2) * halo_pf_rows * halo_pf_ld;
                ldh = halo_pf_ld;
            } else {
                pull_halo(p, l - 1, halo_buf.p, ldD, D);
            }
            const int64_t blocks = ceil_div(static_cast<int64_t>(me) * 32, 256);
            compose_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(compose_idx.p + ext_off[p],
                                                                               act[l - 1].p, ldD, halo, ldh, me,
                                                                               D, h_ext.p, ldD);
            ++t_launches;
            GASB_CUDA(cudaGetLastError());
            if (dr) launch_dropout_apply(h_ext.p, ldD, me, D, mask_of(l), inv_keep, stream);
            launch_spmm_fwd(segs, cols_l.p, coef64.p, h_ext.p, ldD, D, prop.p, ldD, r0, partial_batch.p, pld,
                            counters.p, max_chunks, stream, (push && !dr) ? source_flags(l) : nullptr,
                            tm_ok[3] ? &tm_hext : nullptr);
        }
        PushEpilogue pe{history_table(hist, l), history_ld(hist), bn, history_stamps(hist, l),
                        history_step_ptr(hist), history_flags(hist, l)};
        const bool do_push = push && l < L;
        if (gcnii) {
            launch_mix(h0.p, ldD, br, prop.p, ldD, m, D, spec.alpha, mixed[l].p, ldD, nullptr, stream);
            GemmEpilogue e;  // act_l = relu(mixed_l . W~_l), pushed for l < L
            e.relu = 1;
            if (do_push) e.push = pe;
            launch_gemm(0, m, H, H, mixed[l].p, ldD, wt.p + static_cast<int64_t>(l - 1) * H * pp(layer_param[1]),
                        pp(layer_param[1]), act[l].p, ldD, e,
                        stream);
            if (l == L) {  // relu -> [dropout] -> out_w, out_b (trainer.cpp:221-227)
                if (dr) launch_dropout_apply(act[L].p, ldD, m, H, mask_of(9000), inv_keep, stream);
                GemmEpilogue eo;
                eo.bias = P(p_ob);
                launch_gemm(0, m, C, H, act[L].p, ldD, P(p_ow), pp(p_ow), logits.p, ldC, eo, stream);
            }
        } else {  // APPNP: out = alpha h0[B] + (1 - alpha) prop, pushed raw (no relu)
            launch_mix(h0.p, ldD, br, prop.p, ldD, m, D, spec.alpha, l < L ? act[l].p : logits.p, l < L ? ldD : ldC,
                       do_push ? &pe : nullptr, stream);
        }
    }
    // ---- loss + backward ----
    const bool stepped = ntrain[p] > 0 && train;
    if (ntrain[p] > 0)
        launch_softmax_ce(logits.p, ldC, m, C, row_label.p + r0, ntrain[p], glogits.p, ldC, loss.p + p,
                          row_scratch.p, ce_done.p, stream);
    if (stepped) {
        const GemmEpilogue plain;
        const float* dout = glogits.p;
        int64_t ldo = ldC;
        if (gcnii) {  // output head: d out_w, d out_b, then relu backward into d act_L
            launch_gemm(2, H, C, m, act[L].p, ldD, glogits.p, ldC, G(p_ow), pp(p_ow), plain, stream);
            launch_colsum(glogits.p, ldC, m, C, G(p_ob), stream);
            launch_gemm(1, m, H, C, glogits.p, ldC, P(p_ow), pp(p_ow), gout.p, ldD, plain, stream);
            if (dr) launch_dropout_apply(gout.p, ldD, m, H, mask_of(9000), inv_keep, stream);  // dropout bwd
            launch_mask(gout.p, ldD, act[L].p, ldD, m, H, stream);
            dout = gout.p;
            ldo = ldD;
        }
        launch_zero(h0g.p, static_cast<int64_t>(me) * ldD, stream);
        for (int32_t l = L; l >= 1; --l) {
            const float* dmix = dout;
            int64_t ldm = ldo;
            if (gcnii) {  // out_l = mixed_l . W~_l
                GemmEpilogue ew;  // dW_l = beta * (mixed_l^T dout) (scale bwd of W~)
                ew.post_scale = spec.beta;
                launch_gemm(2, H, H, m, mixed[l].p, ldD, dout, ldo, G(layer_param[l]), pp(layer_param[l]), ew, stream);
                launch_gemm(1, m, H, H, dout, ldo, wt.p + static_cast<int64_t>(l - 1) * H * pp(layer_param[1]),
                            pp(layer_param[1]), gmix.p, ldD, plain, stream);
                dmix = gmix.p;
                ldm = ldD;
            }
            launch_mix_bwd(dmix, ldm, m, D, spec.alpha, br, h0g.p, ldD, dprop.p, ldD, stream);
            if (l >= 2) {  // to act_{l-1}'s batch rows (compose bwd), relu mask for GCNII
                launch_spmm_bwd(t_rowptr.p + r0 + p, m, t_src.p, t_cf.p, dprop.p, ldD, D, gcnii ? act[l - 1].p : nullptr,
                                ldD, gout.p, ldD, stream, m, false, t_order.p + r0);
                if (dr) launch_dropout_rows_bwd(gout.p, ldD, m, D, br, mask_of(l), inv_keep, stream);
                dout = gout.p;
                ldo = ldD;
            } else if (dr) {  // layer 1 input = dropout(h0): its gradient, then the dropout bwd into h0g
                launch_spmm_bwd(a_rowptr.p + a_off[p], me, a_src.p, a_cf.p, dprop.p, ldD, D, nullptr, 0, dtmp.p, ldD,
                                stream, m, false);
                launch_dropout_bwd_acc(h0g.p, ldD, me, D, dtmp.p, ldD, mask_of(1), inv_keep, stream);
            } else {  // layer 1: every V_b row of h0, accumulated onto the residual terms
                launch_spmm_bwd(a_rowptr.p + a_off[p], me, a_src.p, a_cf.p, dprop.p, ldD, D, nullptr, 0, h0g.p, ldD,
                                stream, m, true);
            }
        }
        // head backward (x_ext carries no gradient)
        if (gcnii) {
            launch_mask(h0g.p, ldD, h0.p, ldD, me, H, stream);
            launch_colsum(h0g.p, ldD, me, H, G(p_hb1), stream);
            launch_gemm(2, F, H, me, x_ext.p, ldF, h0g.p, ldD, G(p_hw1), pp(p_hw1), plain, stream);
        } else {
            launch_colsum(h0g.p, ldD, me, C, G(p_hb2), stream);
            launch_gemm(2, H, C, me, z.p, ldH, h0g.p, ldD, G(p_hw2), pp(p_hw2), plain, stream);
            launch_gemm(1, me, H, C, h0g.p, ldD, P(p_hw2), pp(p_hw2), zg.p, ldH, plain, stream);
            if (dr) launch_dropout_apply(zg.p, ldH, me, H, mask_of(101), inv_keep, stream);  // dropout bwd
            launch_mask(zg.p, ldH, z.p, ldH, me, H, stream);
            launch_colsum(zg.p, ldH, me, H, G(p_hb1), stream);
            launch_gemm(2, F, H, me, x_ext.p, ldF, zg.p, ldH, G(p_hw1), pp(p_hw1), plain, stream);
        }
        if (spec.l2_weight > 0.0f)  // l2_penalty (tensor.cpp:649-678): loss term + 2 w p on every gradient
            launch_l2_penalty(params.p, grads.p, nparam, spec.l2_weight, loss.p + p, norm_scratch.p + 256, stream);
        if (!dp) {  // data-parallel: Adam runs on the cross-rank gradient sum (dp.cu)
            launch_adam(params.p, adam_m.p, adam_v.p, grads.p, nparam, t_counter.p, bc.p, spec.lr, spec.beta1,
                        spec.beta2, spec.eps, spec.clip_max_norm, norm_scratch.p, stream, history_step_ptr(hist),
                        adam_done.p);  // + the end of the batch
            return;
        }
    }
    if (dp) return;
    end_batch_kernel<<<1, 1, 0, stream>>>(history_step_ptr(hist), t_counter.p, stepped ? 1 : 0);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

namespace {
// Restores the thread's flat-SpMM launch state (grid cap, row-sum hand-off) on every exit path,
// so an exception between setting and clearing it cannot leak into later launches.
struct SpmmLaunchState {
    ~SpmmLaunchState() {
        set_spmm_grid_cap(0);
        set_spmm_row_sums(nullptr, nullptr, 0);
    }
};
}  // namespace

void gasb_trainer_s::enqueue_batch(int32_t p, bool train, bool push, bool use_hoisted, bool fused, bool dp) {
    WsGuard ws(gemm_ws, &colsum_ws);
    if (residual) {
        enqueue_batch_res(p, train, push, fused, dp);
        return;
    }
    const int32_t m = nb[p];
    const int64_t r0 = row_off[p];
    const SpmmSegs segs = seg_batch.segs(p);
    const int32_t* bn = batch_nodes.p + r0;
    const bool dr = drop && train;  // dropout only while training (ForwardOptions.training)
    require(!dr || !fused, "trainer: dropout batches run the materialized path");
    if (!fused && halo_pf.p && xphase != 2) enqueue_prefetch(p);
    // cross-batch phases (run_epoch_x): the forward, or the loss + backward, of the batch;
    // the forward's history layers aggregate only the intra-batch block (enqueue_bg ran the halo)
    const bool xsplit = xphase != 0;
    require(!xsplit || (fused && use_hoisted && !dr), "trainer: cross-batch phases need the fused hoisted path");
    // ---------------- forward (Model::forward, trainer.cpp:174-251) ----------------
    for (int32_t l = 1; l <= L && xphase != 2; ++l) {
        const int32_t din = dims[l - 1], dout = dims[l];
        const int64_t lda = ld_of(din);
        float* a = agg[l].p;
        if (l == 1 && use_hoisted) {
            a = agg_all.p + r0 * ldF;
        } else if (xsplit) {
            SpmmLaunchState restore;
            set_spmm_row_sums(nullptr, xsums(l), pldx);  // y = float(intra sum + halo sum)
            launch_spmm_fwd(xsegs(p, false), xcols.p, xcoef.p, history_table(hist, l - 1), history_ld(hist), din, a,
                            lda, r0, xpartial(l), pldx, xcounters(l), cxld, stream, source_flags(l), source_tmap(l));
        } else if (fused) {
            const float* src = l == 1 ? X.p : history_table(hist, l - 1);
            const int64_t lds = l == 1 ? ldF : history_ld(hist);
            launch_spmm_fwd(segs, cols_g.p, coef64.p, src, lds, din, a, lda, r0, partial_batch.p, pld, counters.p,
                            max_chunks, stream, source_flags(l), source_tmap(l));
        } else {
            // reference structure: x_ext / compose over V_b local rows, SpMM by local ids
            const int64_t ldx = ld_of(din);
            const float* hsrc;
            if (l == 1) {
                launch_rows(1, extended.p + ext_off[p], ne[p], X.p, ldF, x_ext.p, ldx, din, n, nullptr, nullptr,
                            nullptr, stream);  // gather_features (trainer.cpp:20-27)
                hsrc = x_ext.p;
                if (dr) launch_dropout_apply(x_ext.p, ldx, ne[p], din, mask_of(l), inv_keep, stream);
            } else {
                // HistoryStore::pull of the halo rows, then compose_rows (tensor.cpp:459-512)
                const float* halo = halo_buf.p;
                int64_t ldh = ldx;
                if (halo_pf.p) {  // Prefetcher::wait(l - 1): the side-stream copy of this layer
                    GASB_CUDA(cudaStreamWaitEvent(stream, ev_pf[l - 1], 0));
                    halo = halo_pf.p + static_cast<int64_t>(l - 2) * halo_pf_rows * halo_pf_ld;
                    ldh = halo_pf_ld;
                } else {
                    pull_halo(p, l - 1, halo_buf.p, ldx, din);
                }
                const int64_t blocks = ceil_div(static_cast<int64_t>(ne[p]) * 32, 256);
                compose_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
                    compose_idx.p + ext_off[p], act[l - 1].p, ldH, halo, ldh, ne[p], din, h_ext.p, ldx);
                ++t_launches;
                GASB_CUDA(cudaGetLastError());
                hsrc = h_ext.p;
                // dropout of the layer input, every V_b row (trainer.cpp:203-204)
                if (dr) launch_dropout_apply(h_ext.p, ldx, ne[p], din, mask_of(l), inv_keep, stream);
            }
            // the composed rows come from X / H_{l-1} (+ act_{l-1}, pushed to H_{l-1} when push);
            // without push the act rows are unflagged, so take the exact F2F widening (as after
            // dropout's scaling, which may overflow a finite value)
            launch_spmm_fwd(segs, cols_l.p, coef64.p, hsrc, ldx, din, a, lda, r0, partial_batch.p, pld, counters.p,
                            max_chunks, stream, ((push || l == 1) && !dr) ? source_flags(l) : nullptr,
                            l == 1 ? (tm_ok[2] ? &tm_xext : nullptr) : (tm_ok[3] ? &tm_hext : nullptr));
        }
        float* Wl = W(l);
        if (l < L) {
            // HistoryStore::push fused into the epilogue (stamps + the table's value flags)
            PushEpilogue pe{history_table(hist, l), history_ld(hist), bn, history_stamps(hist, l),
                            history_step_ptr(hist), history_flags(hist, l)};
            launch_gemm(0, m, dout, din, a, lda, Wl, pp(layer_param[l]), act[l].p, ldH, 0.f, true, push ? &pe : nullptr,
                        stream);
        } else {
            launch_gemm(0, m, dout, din, a, lda, Wl, pp(layer_param[l]), logits.p, ldC, 0.f, false, nullptr, stream);
        }
    }
    if (xphase == 1) return;
    // ---------------- loss + backward (run_batch, trainer.cpp:295-339) ----------------
    const bool stepped = ntrain[p] > 0 && train;
    if (ntrain[p] > 0)
        launch_softmax_ce(logits.p, ldC, m, C, row_label.p + r0, ntrain[p], glogits.p, ldC, loss.p + p,
                          row_scratch.p, ce_done.p, stream);
    if (stepped) {
        float* g = glogits.p;
        int64_t ldg = ldC;
        float* gbuf[2] = {g_out.p, g_out2.p};
        for (int32_t l = L; l >= 1; --l) {
            const int32_t din = dims[l - 1], dout = dims[l];
            const int64_t lda = ld_of(din);
            const float* a = (l == 1 && use_hoisted) ? agg_all.p + r0 * ldF : agg[l].p;
            // matmul backward (tensor.cpp:169-204): dW = agg^T g on the side stream (fork
            // after g is complete) ; dagg = g W^T on the main stream
            GASB_CUDA(cudaEventRecord(ev_fork[l], stream));
            GASB_CUDA(cudaStreamWaitEvent(side, ev_fork[l], 0));
            // Split-K CTAs spin until every slice of their tile arrived, which is only safe while
            // one split-K grid is in flight: the side-stream wgrads may split, the main-stream
            // dgrads overlapping them run unsplit (no workspace) and never wait, so they always
            // drain and the wgrad's slices become resident (at C3 the dgrads have 8 k-blocks and
            // would not split anyway)
            set_gemm_workspace(gemm_ws2.p, kGemmWsFloats);
            launch_gemm(2, din, dout, m, a, lda, g, ldg, gW(l), pp(layer_param[l]), 0.f, false, nullptr, side);
            set_gemm_workspace(nullptr, 0);
            GASB_CUDA(cudaEventRecord(ev_wdone[l], side));
            if (l == 1) break;  // x_ext carries no gradient
            // into the buffer the wgrad of layer l + 1 read: wait for it
            float* go = gbuf[l & 1];
            if (l + 1 <= L - 1) GASB_CUDA(cudaStreamWaitEvent(stream, ev_wdone[l + 1], 0));
            if (dout < din) {
                // narrow layer (the classifier, 41 < 256 at C3): aggregate backward on the dout-wide
                // gradient first, then the dgrad GEMM and the relu mask: A^T (g W^T) == (A^T g) W^T,
                // dout/din of the gather work (reassociation only; within the 1e-5 grad contract)
                launch_spmm_bwd(t_rowptr.p + r0 + p, m, t_src.p, t_cf.p, g, ldg, dout, nullptr, 0, g_agg.p, ldC,
                                stream, m, false, t_order.p + r0);
                launch_gemm(1, m, din, dout, g_agg.p, ldC, W(l), pp(layer_param[l]), go, ldH, 0.f, false, nullptr,
                            stream);
                launch_mask(go, ldH, act[l - 1].p, ldH, m, din, stream);  // relu backward (mask = act_{l-1})
            } else {
                launch_gemm(1, m, din, dout, g, ldg, W(l), pp(layer_param[l]), g_agg.p, ldH, 0.f, false, nullptr,
                            stream);
                // aggregate backward over intra-batch edges + compose bwd + relu bwd (mask = act)
                spmm_bwd_batch(p, g_agg.p, ldH, din, act[l - 1].p, ldH, go, ldH, stream);
            }
            // dropout backward on the batch rows of the layer input (tensor.cpp:390-397)
            if (dr) launch_dropout_rows_bwd(go, ldH, m, din, brow.p + r0, mask_of(l), inv_keep, stream);
            g = go;
            ldg = ldH;
        }
        set_gemm_workspace(gemm_ws.p, kGemmWsFloats);
        GASB_CUDA(cudaEventRecord(ev_join, side));  // every weight gradient is complete
        GASB_CUDA(cudaStreamWaitEvent(stream, ev_join, 0));
        if (spec.l2_weight > 0.0f)  // l2_penalty (tensor.cpp:649-678): loss term + 2 w p on every gradient
            launch_l2_penalty(params.p, grads.p, nparam, spec.l2_weight, loss.p + p, norm_scratch.p + 256, stream);
        if (!dp) {  // data-parallel: Adam runs on the cross-rank gradient sum (dp.cu)
            launch_adam(params.p, adam_m.p, adam_v.p, grads.p, nparam, t_counter.p, bc.p, spec.lr, spec.beta1,
                        spec.beta2, spec.eps, spec.clip_max_norm, norm_scratch.p, stream, history_step_ptr(hist),
                        adam_done.p);  // + the end of the batch
            return;
        }
    }
    if (dp) return;
    end_batch_kernel<<<1, 1, 0, stream>>>(history_step_ptr(hist), t_counter.p, stepped ? 1 : 0);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

// Keep masks of every dropout site of batch p in epoch `epoch` (row-major over the site's
// input; seed derive_seed(seed ^ "drop", epoch, p, slot): trainer.cpp:144-147, 181-184 —
// batch_index = the partition id).
void gasb_trainer_s::enqueue_masks(int32_t p, int64_t epoch) {
    const uint64_t base = spec.seed ^ 0x64726f70ull;  // kDropTag
    const size_t ns = dslot.size();
    auto count = [&](size_t i) { return static_cast<int64_t>(dslot_batch[i] ? nb[p] : ne[p]) * dslot_w[i]; };
    if (opt.dropout_rng == GASB_DROPOUT_PHILOX) {
        for (size_t i = 0; i < ns; ++i)
            launch_philox_mask(dmask.p + dmask_off[i], count(i),
                               derive_seed(base, static_cast<uint64_t>(epoch), static_cast<uint64_t>(p), dslot[i]),
                               spec.dropout, stream);
        return;
    }
    // the reference's stream (Rng(seed).next_double() >= p per element, in order), one host
    // thread per site, into the page-locked slot not read by the copy still in flight
    const int s = dmask_slot;
    dmask_slot ^= 1;
    GASB_CUDA(cudaEventSynchronize(dmask_done[s]));
    uint32_t* h = dmask_host[s];
    const double pd = spec.dropout;
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t i = 0; i < ns; ++i) {
        Rng rng(derive_seed(base, static_cast<uint64_t>(epoch), static_cast<uint64_t>(p), dslot[i]));
        const int64_t cnt = count(i);
        uint32_t* w = h + dmask_off[i];
        for (int64_t i0 = 0; i0 < cnt; i0 += 32) {
            uint32_t bits = 0;
            const int e = static_cast<int>(std::min<int64_t>(32, cnt - i0));
            for (int b = 0; b < e; ++b) bits |= static_cast<uint32_t>(rng.next_double() >= pd) << b;
            w[i0 >> 5] = bits;
        }
    }
    GASB_CUDA(cudaMemcpyAsync(dmask.p, h, sizeof(uint32_t) * dmask_off[ns], cudaMemcpyHostToDevice, stream));
    GASB_CUDA(cudaEventRecord(dmask_done[s], stream));
}

void gasb_trainer_s::run_epoch(int64_t epoch, bool shuffle, int32_t begin, int32_t end) {
    // batch order (trainer.cpp:395-400)
    std::vector<int32_t> order(static_cast<size_t>(num_parts));
    std::iota(order.begin(), order.end(), 0);
    if (shuffle) {
        Rng rng(derive_seed(spec.seed ^ 0x6f726472ull, static_cast<uint64_t>(epoch)));
        for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[rng.next_below(i)]);
    }
    // [begin, end) of the order: a window of the epoch's batches (the timed configuration's
    // parity test runs the first batches of an epoch; gas_epoch is the whole range)
    begin = std::max(0, begin);
    end = std::min(end < 0 ? num_parts : end, num_parts);
    order = std::vector<int32_t>(order.begin() + std::min(begin, end), order.begin() + end);
    int64_t steps = 0;
    for (int32_t p : order) steps += ntrain[p] > 0 ? 1 : 0;
    ensure_bc(t_host + steps + 2);
    if (xmode) {
        run_epoch_x(order);
        t_host += steps;
        last_order = order;
        return;
    }
    const bool hoisted = opt.hoist_layer1 && opt.fused && !residual && !drop;
    const int64_t l0 = t_launches;
    if (hoisted) enqueue_hoisted();
    epoch_launches = t_launches - l0;
    for (int32_t p : order) {
        if (drop) {
            const int64_t c0 = t_launches;
            enqueue_masks(p, epoch);
            epoch_launches += t_launches - c0;
        }
        epoch_launches += launch_batch_graph(p, false);
    }
    t_host += steps;
    last_order = order;
}

// ---------------- cross-batch concurrent execution (opt.cross_batch) ----------------
// The reference overlaps batch b+1's history pulls with batch b's compute (Prefetcher,
// history.cpp:184-252; trainer.cpp:416-418). The fused path has no pulls: batch b+1's halo
// rows are read in place by its aggregations. What can move is the aggregation over the halo
// in-edges itself: they read H_{l-1} rows of nodes outside V_{b+1}, which only earlier
// batches' pushes write, and batch b's last push is in its forward. So right after batch b's
// forward, the background stream aggregates every history layer's halo block of batch b+1
// into fp64 partials, overlapped with batch b's backward and Adam; batch b+1's forward then
// aggregates its intra-batch block and the last-arriving segment of each row combines the
// row's partials in segment order (halo block first) and stores the fp32 row.
//
// Edge layout: per part, the edges are re-laid as [halo-source block | intra-source block],
// each row-major and in CSR order inside a row; every row gets >= 1 segment in each block
// (possibly empty), all with partial slots, so the store is always made by the intra launch.
void gasb_trainer_s::build_xbatch(const std::vector<int64_t>& rp, const HVec<int32_t>& cg, const HVec<double>& cf) {
    const int64_t R = row_off[num_parts], E = edge_off[num_parts];
    HVec<int32_t> xc(static_cast<size_t>(E));
    HVec<double> xf(static_cast<size_t>(E));
    std::vector<int64_t> rph(static_cast<size_t>(R)), rpi(static_cast<size_t>(R)), hend(num_parts);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t p = 0; p < num_parts; ++p) {
        const HostPlan& P = sched->plans[p];
        const int64_t e0 = edge_off[p];
        int64_t nhal = 0;
        for (int32_t c : P.gcn_cols) nhal += P.is_halo[c] ? 1 : 0;
        int64_t kh = e0, ki = e0 + nhal;
        for (int64_t r = row_off[p]; r < row_off[p + 1]; ++r) {
            rph[r] = kh;
            rpi[r] = ki;
            for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                if (P.is_halo[P.gcn_cols[e - e0]]) {
                    xc[kh] = cg[e];
                    xf[kh++] = cf[e];
                } else {
                    xc[ki] = cg[e];
                    xf[ki++] = cf[e];
                }
            }
        }
        hend[p] = e0 + nhal;
    }
    xcols.upload(xc);
    xcoef.upload(xf);
    std::vector<int64_t> iend(num_parts);
    for (int32_t p = 0; p < num_parts; ++p) iend[p] = edge_off[p + 1];
    build_block_segments(rph, hend, seg_xh);
    build_block_segments(rpi, iend, seg_xi);
    xslots = std::max(seg_xh.max_group_slots, seg_xi.max_group_slots);
    pldx = round_up(std::max(H, 1), 256);
    cxld = static_cast<int32_t>(ceil_div(std::max(H, 1), 64));
    partial_x.alloc(static_cast<int64_t>(L - 1) * std::max<int64_t>(xslots, 1) * pldx);
    counters_x.alloc(static_cast<int64_t>(L - 1) * R * cxld);
    counters_x.zero();
    xsum.alloc(static_cast<int64_t>(L - 1) * nb_max * pldx);
}

// Segment table of one block per part (rows' edges at row_start[r] .., the part's block ending
// at part_end[p]): the split segmentation of segment_launch, one launch (group) per part. A
// zero-length gap segment after each part keeps seg_beg[group end] at the block's end (the
// next part's block starts elsewhere).
void gasb_trainer_s::build_block_segments(const std::vector<int64_t>& row_start, const std::vector<int64_t>& part_end,
                                          SegTable& t) {
    const int64_t R = row_off[num_parts];
    const int32_t nr = spmm_ranges_per_launch();
    t.nranges = nr;
    t.split = true;
    std::vector<int64_t> sb, tmp(static_cast<size_t>(R) + 1);
    std::vector<int32_t> sr, ss, r0(R), rn(R), rs(static_cast<size_t>(num_parts) * (nr + 1));
    t.group_seg0.assign(num_parts, 0);
    t.group_nseg.assign(num_parts, 0);
    t.max_group_slots = 0;
    for (int32_t p = 0; p < num_parts; ++p) {
        const int64_t lo = row_off[p], hi = row_off[p + 1];
        for (int64_t r = lo; r < hi; ++r) tmp[r] = row_start[r];
        tmp[hi] = part_end[p];
        t.group_seg0[p] = static_cast<int64_t>(sr.size());
        int64_t slot = 0;
        segment_launch(tmp.data(), lo, hi, true, nr, sb, sr, ss, r0.data(), rn.data(), slot,
                       rs.data() + static_cast<int64_t>(p) * (nr + 1));
        t.group_nseg[p] = static_cast<int64_t>(sr.size()) - t.group_seg0[p];
        t.max_group_slots = std::max(t.max_group_slots, slot);
        sr.push_back(static_cast<int32_t>(lo));  // the gap segment (sb's sentinel stays as its start)
        ss.push_back(-1);
    }
    sb.push_back(sb.empty() ? 0 : sb.back());
    t.total_slots = t.max_group_slots;
    t.ranges.upload(rs);
    t.seg_beg.upload(sb);
    t.seg_row.upload(sr);
    t.seg_slot.upload(ss);
    t.row_seg0.upload(r0);
    t.row_nseg.upload(rn);
}

// Background work of batch q on `bg`: (xmode 2) its layer-1 rows of agg_all, then — after the
// previous batch's forward (ev_xfwd) when wait_fwd — the halo block of every history layer.
void gasb_trainer_s::enqueue_bg(int32_t q, bool wait_fwd) {
    SpmmLaunchState restore;
    set_spmm_grid_cap(bg_ctas);
    if (xmode == 2)
        launch_spmm_fwd(seg_batch.segs(q), cols_g.p, coef64.p, X.p, ldF, F, agg_all.p, ldF, 0, partial_batch.p, pld,
                        counters.p, max_chunks, bg, source_flags(1), source_tmap(1));
    if (wait_fwd) GASB_CUDA(cudaStreamWaitEvent(bg, ev_xfwd, 0));
    for (int32_t l = 2; l <= L; ++l) {  // fp64 row sums of the halo block (the intra launch stores the rows)
        set_spmm_row_sums(xsums(l), nullptr, pldx);
        launch_spmm_fwd(xsegs(q, true), xcols.p, xcoef.p, history_table(hist, l - 1), history_ld(hist), dims[l - 1],
                        agg[l].p, ld_of(dims[l - 1]), row_off[q], xpartial(l), pldx, xcounters(l), cxld, bg,
                        source_flags(l), source_tmap(l));
    }
}

// One phase (1 forward, 2 loss + backward + Adam) of batch p on `stream`, through its captured
// graph when use_graphs. Returns the kernels its graph launches.
int64_t gasb_trainer_s::launch_x_graph(int32_t p, int32_t phase) {
    if (!opt.use_graphs) {  // (direct launches: counted by t_launches)
        xphase = phase;
        enqueue_batch(p, true, true, true, true, false);
        xphase = 0;
        return 0;
    }
    std::vector<cudaGraphExec_t>& gs = phase == 1 ? graphs_xf : graphs_xb;
    std::vector<int64_t>& gl = phase == 1 ? graph_launches_xf : graph_launches_xb;
    if (gs.empty()) {
        gs.assign(num_parts, nullptr);
        gl.assign(num_parts, 0);
    }
    if (!gs[p]) {
        cudaGraph_t graph;
        const int64_t c0 = t_launches;
        xphase = phase;
        GASB_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        enqueue_batch(p, true, true, true, true, false);
        GASB_CUDA(cudaStreamEndCapture(stream, &graph));
        xphase = 0;
        gl[p] = t_launches - c0;
        t_launches = c0;
        GASB_CUDA(cudaGraphInstantiate(&gs[p], graph, 0));
        GASB_CUDA(cudaGraphDestroy(graph));
    }
    GASB_CUDA(cudaGraphLaunch(gs[p], stream));
    return gl[p];
}

// The epoch's batches with batch i+1's background work overlapped with batch i:
//   bg:     [L1(o0)] halo(o0) | [L1(o1)] .. wait fwd(o0) .. halo(o1) | [L1(o2)] .. wait fwd(o1) ..
//   stream: wait bg | fwd(o0) bwd(o0) | wait bg | fwd(o1) bwd(o1) | ...
void gasb_trainer_s::run_epoch_x(const std::vector<int32_t>& order) {
    const int64_t l0 = t_launches;
    int64_t launches = 0;
    if (xmode == 1) enqueue_hoisted();
    GASB_CUDA(cudaEventRecord(ev_xstart, stream));  // X (set_features), the hoisted layer 1, the last epoch
    GASB_CUDA(cudaStreamWaitEvent(bg, ev_xstart, 0));
    const size_t nbat = order.size();
    if (nbat > 0) {
        enqueue_bg(order[0], false);
        GASB_CUDA(cudaEventRecord(ev_xbg, bg));
        GASB_CUDA(cudaStreamWaitEvent(stream, ev_xbg, 0));
    }
    for (size_t i = 0; i < nbat; ++i) {
        const int32_t p = order[i];
        launches += launch_x_graph(p, 1);
        const bool next = i + 1 < nbat;
        if (next) {
            GASB_CUDA(cudaEventRecord(ev_xfwd, stream));
            enqueue_bg(order[i + 1], true);
            GASB_CUDA(cudaEventRecord(ev_xbg, bg));
        }
        launches += launch_x_graph(p, 2);
        if (next) GASB_CUDA(cudaStreamWaitEvent(stream, ev_xbg, 0));
    }
    epoch_launches = t_launches - l0 + launches;
}

// gas_forward_snapshot (trainer.cpp:466-483): every batch in PART order, forward only against
// the frozen store (no push, no step: the reference-structured path composes the batch's
// fresh rows with pulled halos), each history layer's batch rows scattered by global id into
// the snapshot tables (layer_values) that measure_staleness compares the store with.
void gasb_trainer_s::enqueue_snapshot() {
    if (L < 2) return;
    const int64_t ldh = history_ld(hist), tab = static_cast<int64_t>(n) * ldh;
    if (!snap.p) {
        snap.alloc(static_cast<int64_t>(L - 1) * tab);
        GASB_CUDA(cudaMemsetAsync(snap.p, 0, sizeof(float) * snap.n, stream));
    }
    for (int32_t p = 0; p < num_parts; ++p) {
        enqueue_batch(p, false, false, false, false, /*dp: no Adam, no step*/ true);
        for (int32_t l = 1; l < L; ++l)
            launch_rows(0, batch_nodes.p + row_off[p], nb[p], act[l].p, ldA, snap.p + (l - 1) * tab, ldh, hist_dim,
                        n, nullptr, nullptr, nullptr, stream);
    }
}

// Enqueues one training batch (forward, push, loss, backward; + Adam and the step counters
// unless dp) on `stream`, through its captured per-part graph when use_graphs. Returns the
// number of kernels it launches.
int64_t gasb_trainer_s::launch_batch_graph(int32_t p, bool dp) {
    const bool hoisted = opt.hoist_layer1 && opt.fused && !residual && !drop;
    const bool push = !sharded_dp, fused = opt.fused != 0 && !sharded_dp && !drop;
    if (!opt.use_graphs) {
        const int64_t c0 = t_launches;
        enqueue_batch(p, true, push, hoisted, fused, dp);
        return t_launches - c0;
    }
    std::vector<cudaGraphExec_t>& gs = dp ? graphs_dp : graphs;
    std::vector<int64_t>& gl = dp ? graph_launches_dp : graph_launches;
    if (gs.empty()) {
        gs.assign(num_parts, nullptr);
        gl.assign(num_parts, 0);
    }
    if (!gs[p]) capture_batch_graph(p, dp);
    GASB_CUDA(cudaGraphLaunch(gs[p], stream));
    return gl[p];
}

// Captures (without launching) the per-part batch graph of part p.
void gasb_trainer_s::capture_batch_graph(int32_t p, bool dp) {
    const bool hoisted = opt.hoist_layer1 && opt.fused && !residual && !drop;
    std::vector<cudaGraphExec_t>& gs = dp ? graphs_dp : graphs;
    std::vector<int64_t>& gl = dp ? graph_launches_dp : graph_launches;
    if (gs.empty()) {
        gs.assign(num_parts, nullptr);
        gl.assign(num_parts, 0);
    }
    if (!gs[p]) {
        cudaGraph_t graph;
        const int64_t c0 = t_launches;
        GASB_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        enqueue_batch(p, true, !sharded_dp, hoisted, opt.fused != 0 && !sharded_dp && !drop, dp);
        GASB_CUDA(cudaStreamEndCapture(stream, &graph));
        gl[p] = t_launches - c0;
        t_launches = c0;
        GASB_CUDA(cudaGraphInstantiate(&gs[p], graph, 0));
        GASB_CUDA(cudaGraphDestroy(graph));
    }
}

void gasb_trainer_s::ensure_eval() {
    if (eval_agg.p) return;
    const int64_t R = row_off[num_parts];
    const int64_t ldT = residual ? ldD : ldH;  // width of the layer tables
    eval_agg.alloc(R * ld_of(std::max(F, residual ? D : H)));
    eval_act.alloc(R * ldT);
    for (auto& b : eval_tab) {
        b.alloc(static_cast<int64_t>(n) * ldT);
        b.zero();
    }
    if (residual) {
        eval_h0.alloc(static_cast<int64_t>(n) * ldD);
        if (spec.kind == 2) eval_z.alloc(static_cast<int64_t>(n) * ldH);
        else eval_mixed.alloc(R * ldD);
    }
    eval_logits.alloc(R * ldC);
    eval_flags.alloc(2);
    eval_flags.zero();
    eval_masks.alloc(3LL * n);
    eval_counts.alloc(6);
    eval_pld = round_up(std::max(F, H), 256);
    eval_partial.alloc(std::max<int64_t>(seg_all.total_slots, 1) * eval_pld);
}

// Model::forward over BatchSchedule::full_batch (every node, no halos): the whole-graph
// stencil is the concatenation of the parts' stencils (each row's coefficients depend only
// on global degrees), so the layer-l SpMM is one launch over the whole-epoch segment table
// gathering the previous layer's table by global id. first_layer = L: infer_from_history's
// final layer over H_{L-1} (trainer.cpp:512-520).
void gasb_trainer_s::enqueue_full_forward(int32_t first_layer) {
    WsGuard ws(gemm_ws, &colsum_ws);
    const SpmmSegs segs = seg_all.segs(0);
    const int64_t R = row_off[num_parts];
    GASB_CUDA(cudaMemsetAsync(eval_flags.p, 0, 2 * sizeof(int32_t), stream));
    for (int32_t l = first_layer; l <= L; ++l) {
        const int32_t din = dims[l - 1], dout = dims[l];
        const int64_t lda = ld_of(din);
        const float* src;
        int64_t lds;
        const int32_t* flags;
        const CUtensorMap* tm = nullptr;
        if (l == 1) {
            src = X.p, lds = ldF, flags = xflags.p, tm = source_tmap(1);
        } else if (l == first_layer) {  // pulled layer-(L-1) histories
            src = history_table(hist, l - 1), lds = history_ld(hist), flags = source_flags(l), tm = source_tmap(l);
        } else {
            src = eval_tab[(l - 1) & 1].p, lds = ldH, flags = eval_flags.p + ((l - 1) & 1);
        }
        launch_spmm_fwd(segs, cols_g.p, coef64.p, src, lds, din, eval_agg.p, lda, 0, eval_partial.p, eval_pld,
                        counters.p, max_chunks, stream, flags, tm);
        if (l < L) {
            PushEpilogue pe{eval_tab[l & 1].p, ldH, batch_nodes.p, nullptr, nullptr, eval_flags.p + (l & 1)};
            launch_gemm(0, static_cast<int>(R), dout, din, eval_agg.p, lda, W(l), pp(layer_param[l]), eval_act.p, ldH,
                        0.f, true, &pe, stream);
        } else {
            launch_gemm(0, static_cast<int>(R), dout, din, eval_agg.p, lda, W(l), pp(layer_param[l]), eval_logits.p,
                        ldC, 0.f, false, nullptr, stream);
        }
    }
}

// APPNP / GCNII over the full graph: head MLP over every node in global order (the h0
// table the layer-1 SpMM gathers by global id), then per layer SpMM -> alpha-mixing with
// h0[v] (-> GCNII: relu(mixed . W~_l)) -> scatter into the next layer's table; GCNII's
// output head on the last layer (trainer.cpp:142-163, :221-227; layers.cpp:150-168).
void gasb_trainer_s::enqueue_full_forward_res(int32_t first_layer) {
    WsGuard ws(gemm_ws, &colsum_ws);
    const SpmmSegs segs = seg_all.segs(0);
    const int64_t R = row_off[num_parts];
    const bool gcnii = spec.kind == 3;
    GASB_CUDA(cudaMemsetAsync(eval_flags.p, 0, 2 * sizeof(int32_t), stream));
    {  // head over all n nodes (X in global order)
        GemmEpilogue e1;
        e1.bias = P(p_hb1);
        e1.relu = 1;
        launch_gemm(0, n, H, F, X.p, ldF, P(p_hw1), pp(p_hw1), gcnii ? eval_h0.p : eval_z.p, gcnii ? ldD : ldH, e1,
                    stream);
        if (!gcnii) {
            GemmEpilogue e2;
            e2.bias = P(p_hb2);
            launch_gemm(0, n, C, H, eval_z.p, ldH, P(p_hw2), pp(p_hw2), eval_h0.p, ldD, e2, stream);
        }
    }
    if (gcnii) launch_wtilde(P(layer_param[1]), wt.p, L, H, pp(layer_param[1]), spec.beta, stream);
    // the h0 table's value flags (the SpMM widening path): unknown sign, finite
    int32_t* h0_flags = eval_flags.p;  // reuse slot 0 for layer 1's source, reset below
    GASB_CUDA(cudaMemsetAsync(h0_flags, 0, sizeof(int32_t), stream));
    launch_scan_special(eval_h0.p, n, ldD, D, h0_flags, stream);
    for (int32_t l = first_layer; l <= L; ++l) {
        const float* src;
        int64_t lds;
        const int32_t* flags;
        const CUtensorMap* tm = nullptr;
        if (l == 1) {
            src = eval_h0.p, lds = ldD, flags = h0_flags;
        } else if (l == first_layer) {
            src = history_table(hist, l - 1), lds = history_ld(hist), flags = source_flags(l), tm = source_tmap(l);
        } else {
            src = eval_tab[(l - 1) & 1].p, lds = ldD, flags = eval_flags.p + ((l - 1) & 1);
        }
        launch_spmm_fwd(segs, cols_g.p, coef64.p, src, lds, D, eval_agg.p, ldD, 0, eval_partial.p, eval_pld,
                        counters.p, max_chunks, stream, flags, tm);
        int32_t* out_flags = eval_flags.p + (l & 1);
        if (l < L) GASB_CUDA(cudaMemsetAsync(out_flags, 0, sizeof(int32_t), stream));
        PushEpilogue pe{eval_tab[l & 1].p, ldD, batch_nodes.p, nullptr, nullptr, out_flags};
        if (gcnii) {
            launch_mix(eval_h0.p, ldD, batch_nodes.p, eval_agg.p, ldD, static_cast<int32_t>(R), D, spec.alpha,
                       eval_mixed.p, ldD, nullptr, stream);
            GemmEpilogue e;
            e.relu = 1;
            if (l < L) e.push = pe;
            launch_gemm(0, static_cast<int>(R), H, H, eval_mixed.p, ldD,
                        wt.p + static_cast<int64_t>(l - 1) * H * pp(layer_param[1]), pp(layer_param[1]), eval_act.p,
                        ldD, e, stream);
            if (l == L) {
                GemmEpilogue eo;
                eo.bias = P(p_ob);
                launch_gemm(0, static_cast<int>(R), C, H, eval_act.p, ldD, P(p_ow), pp(p_ow), eval_logits.p, ldC, eo,
                            stream);
            }
        } else {
            launch_mix(eval_h0.p, ldD, batch_nodes.p, eval_agg.p, ldD, static_cast<int32_t>(R), D, spec.alpha,
                       l < L ? eval_act.p : eval_logits.p, l < L ? ldD : ldC, l < L ? &pe : nullptr, stream);
        }
    }
}

extern "C" {

gasb_status gasb_trainer_evaluate(gasb_trainer t, const uint8_t* h_train, const uint8_t* h_val, const uint8_t* h_test,
                                  double* acc3) {
    return guard([&] {
        require(t && acc3, "evaluate: null argument");
        GASB_CUDA(cudaSetDevice(t->opt.device));
        t->ensure_eval();
        const int64_t n = t->n;
        const uint8_t* hm[3] = {h_train, h_val, h_test};
        for (int k = 0; k < 3; ++k) {
            if (hm[k]) GASB_CUDA(cudaMemcpyAsync(t->eval_masks.p + k * n, hm[k], n, cudaMemcpyHostToDevice, t->stream));
            else GASB_CUDA(cudaMemsetAsync(t->eval_masks.p + k * n, 0, n, t->stream));
        }
        GASB_CUDA(cudaMemsetAsync(t->eval_counts.p, 0, 6 * sizeof(int64_t), t->stream));
        if (t->residual) t->enqueue_full_forward_res(1);
        else t->enqueue_full_forward(1);
        const int64_t R = t->row_off[t->num_parts];
        argmax_count_kernel<<<static_cast<unsigned>(ceil_div(R, 256)), 256, 0, t->stream>>>(
            t->eval_logits.p, t->ldC, R, t->C, t->batch_nodes.p, t->labels_all.p, t->eval_masks.p, n,
            reinterpret_cast<unsigned long long*>(t->eval_counts.p), nullptr);
        GASB_CUDA(cudaGetLastError());
        int64_t c[6];
        GASB_CUDA(cudaMemcpyAsync(c, t->eval_counts.p, sizeof(c), cudaMemcpyDeviceToHost, t->stream));
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        for (int k = 0; k < 3; ++k)
            acc3[k] = c[2 * k] == 0 ? 0.0 : static_cast<double>(c[2 * k + 1]) / static_cast<double>(c[2 * k]);
    });
}

gasb_status gasb_trainer_full_logits(gasb_trainer t, float* h_logits) {
    return guard([&] {
        require(t && h_logits, "full_logits: null argument");
        if (!t->eval_logits.p) throw std::logic_error("full_logits: no evaluate / infer has run");
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        const int64_t R = t->row_off[t->num_parts];
        std::vector<float> rows(static_cast<size_t>(R) * t->C);
        std::vector<int32_t> nodes(static_cast<size_t>(R));
        GASB_CUDA(cudaMemcpy2D(rows.data(), sizeof(float) * t->C, t->eval_logits.p, sizeof(float) * t->ldC,
                               sizeof(float) * t->C, R, cudaMemcpyDeviceToHost));
        GASB_CUDA(cudaMemcpy(nodes.data(), t->batch_nodes.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < R; ++i)
            std::copy(rows.begin() + i * t->C, rows.begin() + (i + 1) * t->C,
                      h_logits + static_cast<int64_t>(nodes[i]) * t->C);
    });
}

gasb_status gasb_trainer_infer_from_history(gasb_trainer t, int32_t* h_predictions, int32_t* stale) {
    return guard([&] {
        require(t && h_predictions && stale, "infer_from_history: null argument");
        GASB_CUDA(cudaSetDevice(t->opt.device));
        t->ensure_eval();
        const int64_t n = t->n;
        if (t->residual) t->enqueue_full_forward_res(t->L >= 2 ? t->L : 1);
        else t->enqueue_full_forward(t->L >= 2 ? t->L : 1);
        const int64_t R = t->row_off[t->num_parts];
        DevBuf<int32_t> preds;
        preds.alloc(n);
        argmax_count_kernel<<<static_cast<unsigned>(ceil_div(R, 256)), 256, 0, t->stream>>>(
            t->eval_logits.p, t->ldC, R, t->C, t->batch_nodes.p, t->labels_all.p, nullptr, n, nullptr, preds.p);
        GASB_CUDA(cudaGetLastError());
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        GASB_CUDA(cudaMemcpy(h_predictions, preds.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
        *stale = 0;
        if (t->L >= 2) {  // some layer-(L-1) row never pushed (trainer.cpp:521-525)
            std::vector<int64_t> st(static_cast<size_t>(n));
            GASB_CUDA(cudaMemcpy(st.data(), history_stamps(t->hist, t->L - 1), sizeof(int64_t) * n,
                                 cudaMemcpyDeviceToHost));
            for (int64_t v = 0; v < n && !*stale; ++v) *stale = st[v] < 0;
        }
    });
}

gasb_status gasb_trainer_create(gasb_schedule s, const float* h_features, int32_t in_dim, const int32_t* h_labels,
                                const uint8_t* h_train_mask, int32_t num_classes, const gasb_model_spec* spec,
                                const gasb_trainer_options* opt, gasb_trainer* out) {
    return guard([&] {
        require(s && h_features && h_labels && h_train_mask && spec && out, "trainer: null argument");
        require(in_dim > 0 && num_classes > 0, "Model: in_dim and num_classes must be positive");
        require(spec->num_layers >= 1, "ModelSpec: need at least one layer");
        require(spec->hidden > 0, "ModelSpec: hidden must be positive");
        require(spec->dropout >= 0.0f && spec->dropout < 1.0f, "ModelSpec: dropout must be in [0,1)");
        auto t = std::make_unique<gasb_trainer_s>();
        t->spec = *spec;
        if (opt) t->opt = *opt;
        else t->opt = gasb_trainer_options{128, 1, 0, 1, 1, 0, GASB_DROPOUT_EXACT};
        t->sched = &schedule_of(s);
        t->F = in_dim;
        t->C = num_classes;
        t->build(h_features, h_labels, h_train_mask);
        {  // V_b-row buffers: the reference-structured path, push = 0 batches and the residual heads
            const int64_t ldmax = t->ld_of(std::max(t->F, t->H));
            t->x_ext.alloc(static_cast<int64_t>(t->ne_max) * ldmax);
            t->h_ext.alloc(static_cast<int64_t>(t->ne_max) * ldmax);
            t->halo_buf.alloc(static_cast<int64_t>(t->ne_max) * ldmax);
            // halo ids per part, concatenated at ext_off - row_off
            std::vector<int32_t> hid(static_cast<size_t>(t->ext_off[t->num_parts] - t->row_off[t->num_parts]));
            for (int32_t p = 0; p < t->num_parts; ++p) {
                const HostPlan& P = t->sched->plans[p];
                std::copy(P.halo.begin(), P.halo.end(), hid.begin() + (t->ext_off[p] - t->row_off[p]));
            }
            t->halo_ids.upload(hid);
        }
        if (!t->opt.fused && t->opt.prefetch && t->L >= 2) {
            int64_t nh_max = 0;
            for (int32_t p = 0; p < t->num_parts; ++p) nh_max = std::max<int64_t>(nh_max, t->nh[p]);
            t->halo_pf_ld = t->ld_of(t->hist_dim);
            t->halo_pf_rows = std::max<int64_t>(nh_max, 1);
            t->halo_pf.alloc(static_cast<int64_t>(t->L - 1) * t->halo_pf_rows * t->halo_pf_ld);
            GASB_CUDA(cudaEventCreateWithFlags(&t->ev_pf_start, cudaEventDisableTiming));
            t->ev_pf.assign(static_cast<size_t>(t->L), nullptr);
            for (auto& e : t->ev_pf) GASB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        t->build_tmaps();
        *out = t.release();
    });
}

gasb_status gasb_trainer_destroy(gasb_trainer t) {
    delete t;
    return GASB_OK;
}

gasb_status gasb_gas_epoch_async(gasb_trainer t, int64_t epoch, int32_t shuffle) {
    return guard([&] {
        require(t, "trainer: null handle");
        t->run_epoch(epoch, shuffle != 0);
    });
}

gasb_status gasb_gas_epoch_range_async(gasb_trainer t, int64_t epoch, int32_t shuffle, int32_t begin, int32_t end) {
    return guard([&] {
        require(t, "trainer: null handle");
        require(begin >= 0 && begin <= end && end <= t->num_parts, "gas_epoch_range: need 0 <= begin <= end <= parts");
        t->run_epoch(epoch, shuffle != 0, begin, end);
    });
}

gasb_status gasb_trainer_dropout_mask(gasb_trainer t, int32_t part, int64_t epoch, int32_t layer, uint32_t* h_words) {
    return guard([&] {
        require(t && h_words, "trainer: null argument");
        if (!t->drop) throw std::logic_error("dropout_mask: the model has dropout == 0");
        require(part >= 0 && part < t->num_parts && layer >= 1 && layer <= t->L, "dropout_mask: part/layer out of range");
        t->enqueue_masks(part, epoch);
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        const int64_t words = ceil_div(static_cast<int64_t>(t->ne[part]) * t->dims[layer - 1], 32);
        GASB_CUDA(cudaMemcpy(h_words, t->mask_of(static_cast<uint64_t>(layer)), sizeof(uint32_t) * words,
                             cudaMemcpyDeviceToHost));
    });
}

gasb_status gasb_trainer_part_losses(gasb_trainer t, double* h_losses) {
    return guard([&] {
        require(t && h_losses, "trainer: null argument");
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        GASB_CUDA(cudaMemcpy(h_losses, t->loss.p, sizeof(double) * t->num_parts, cudaMemcpyDeviceToHost));
    });
}

gasb_status gasb_gas_epoch_report(gasb_trainer t, int64_t epoch, int32_t shuffle, int32_t measure_staleness,
                                  gasb_epoch_report* out, int64_t* h_batch_peak_floats, double* h_eps_max) {
    return guard([&] {
        require(t && out, "trainer: null argument");
        t->run_epoch(epoch, shuffle != 0);
        gasb_epoch_report r{};
        r.epoch = epoch;
        r.num_batches = static_cast<int32_t>(t->last_order.size());
        {
            GASB_CUDA(cudaStreamSynchronize(t->stream));
            std::vector<double> l(static_cast<size_t>(t->num_parts));
            GASB_CUDA(cudaMemcpy(l.data(), t->loss.p, sizeof(double) * l.size(), cudaMemcpyDeviceToHost));
            double sum = 0.0;
            int64_t cnt = 0;
            for (int32_t p : t->last_order)
                if (t->ntrain[p] > 0) {
                    sum += l[p];
                    ++cnt;
                }
            r.loss = cnt > 0 ? sum / static_cast<double>(cnt) : 0.0;
        }
        for (size_t i = 0; i < t->last_order.size(); ++i) {  // epoch order, as batch_peak_floats
            const int32_t p = t->last_order[i];
            r.peak_floats = std::max(r.peak_floats, t->part_act_floats[p]);
            r.edges_per_layer += t->part_edges[p];
            if (h_batch_peak_floats) h_batch_peak_floats[i] = t->part_act_floats[p];
        }
        size_t fr = 0, tot = 0;
        GASB_CUDA(cudaMemGetInfo(&fr, &tot));
        r.device_bytes = t->mem_free_at_build > fr ? static_cast<int64_t>(t->mem_free_at_build - fr) : 0;
        if (measure_staleness && t->L >= 2) {  // trainer.cpp:434-438
            t->enqueue_snapshot();
            GASB_CUDA(cudaStreamSynchronize(t->stream));
            const int64_t ldh = history_ld(t->hist), tab = static_cast<int64_t>(t->n) * ldh;
            std::vector<const float*> refs(static_cast<size_t>(t->L - 1));
            std::vector<int64_t> lds(refs.size(), ldh), amax(refs.size());
            std::vector<double> emax(refs.size()), emean(refs.size()), amean(refs.size());
            for (int32_t l = 1; l < t->L; ++l) refs[l - 1] = t->snap.p + (l - 1) * tab;
            const gasb_status st = gasb_history_staleness(t->hist, refs.data(), lds.data(), emax.data(), emean.data(),
                                                          amax.data(), amean.data());
            if (st != GASB_OK) throw std::runtime_error(gasb_last_error());
            r.staleness_layers = t->L - 1;
            if (h_eps_max) std::copy(emax.begin(), emax.end(), h_eps_max);
        }
        *out = r;
    });
}

gasb_status gasb_trainer_last_loss(gasb_trainer t, double* mean_loss) {
    return guard([&] {
        require(t && mean_loss, "trainer: null argument");
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        std::vector<double> l(static_cast<size_t>(t->num_parts));
        GASB_CUDA(cudaMemcpy(l.data(), t->loss.p, sizeof(double) * l.size(), cudaMemcpyDeviceToHost));
        double sum = 0.0;
        int64_t cnt = 0;
        for (int32_t p : t->last_order)  // EpochReport.loss: mean over stepped batches, epoch order
            if (t->ntrain[p] > 0) {
                sum += l[p];
                ++cnt;
            }
        *mean_loss = cnt > 0 ? sum / static_cast<double>(cnt) : 0.0;
    });
}

gasb_status gasb_gas_epoch(gasb_trainer t, int64_t epoch, int32_t shuffle, double* mean_loss) {
    gasb_status s = gasb_gas_epoch_async(t, epoch, shuffle);
    if (s != GASB_OK) return s;
    double l = 0.0;
    s = gasb_trainer_last_loss(t, &l);
    if (mean_loss) *mean_loss = l;
    return s;
}

gasb_status gasb_trainer_batch(gasb_trainer t, int32_t part, int64_t epoch, int32_t train, int32_t push,
                               float* h_acts, float* h_logits, double* loss, float* h_grads, int32_t* stepped) {
    return guard([&] {
        require(t, "trainer: null handle");
        require(part >= 0 && part < t->num_parts, "trainer: part out of range");
        const bool tr = train != 0;
        t->ensure_bc(t->t_host + 2);
        const bool dr = t->drop && tr;
        if (dr) t->enqueue_masks(part, epoch);
        t->enqueue_batch(part, tr, push != 0, false, push != 0 && t->opt.fused != 0 && !dr);
        const bool st = tr && t->ntrain[part] > 0;
        if (st) t->t_host++;
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        const int32_t m = t->nb[part];
        const int32_t hd = t->hist_dim;
        if (h_acts && hd > 0)
            for (int32_t l = 1; l < t->L; ++l)
                GASB_CUDA(cudaMemcpy2D(h_acts + static_cast<int64_t>(l - 1) * m * hd, sizeof(float) * hd, t->act[l].p,
                                       sizeof(float) * t->ldA, sizeof(float) * hd, m, cudaMemcpyDeviceToHost));
        if (h_logits)
            GASB_CUDA(cudaMemcpy2D(h_logits, sizeof(float) * t->C, t->logits.p, sizeof(float) * t->ldC,
                                   sizeof(float) * t->C, m, cudaMemcpyDeviceToHost));
        if (loss) {
            double l = 0.0;
            if (t->ntrain[part] > 0) GASB_CUDA(cudaMemcpy(&l, t->loss.p + part, sizeof(double), cudaMemcpyDeviceToHost));
            *loss = l;
        }
        if (h_grads && st)
            t->params_to_dense(t->grads.p, h_grads);
        if (stepped) *stepped = st ? 1 : 0;
    });
}

gasb_status gasb_trainer_num_param_floats(gasb_trainer t, int64_t* out) {
    return guard([&] {
        require(t && out, "trainer: null argument");
        *out = t->nparam_dense;
    });
}

gasb_status gasb_trainer_get_params(gasb_trainer t, float* h) {
    return guard([&] {
        require(t && h, "trainer: null argument");
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        t->params_to_dense(t->params.p, h);
    });
}

gasb_status gasb_trainer_set_params(gasb_trainer t, const float* h) {
    return guard([&] {
        require(t && h, "trainer: null argument");
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        t->params_from_dense(h, t->params.p);
    });
}

gasb_status gasb_trainer_history(gasb_trainer t, gasb_history* out) {
    return guard([&] {
        require(t && out, "trainer: null argument");
        *out = t->hist;
    });
}

gasb_status gasb_trainer_stream(gasb_trainer t, gasb_stream* out) {
    return guard([&] {
        require(t && out, "trainer: null argument");
        *out = t->stream;
    });
}

gasb_status gasb_trainer_stage_features(gasb_trainer t, const float* h) {
    return guard([&] {
        require(t && h, "trainer: null argument");
        // one contiguous DMA at full link rate into a dense staging copy, on the copy stream,
        // after the previous staged copy has been consumed
        const int64_t cnt = static_cast<int64_t>(t->n) * t->F;
        if (t->x_stage.n < cnt) {
            GASB_CUDA(cudaStreamSynchronize(t->stream));
            t->x_stage.alloc(cnt);
            GASB_CUDA(cudaEventRecord(t->ev_stage_free, t->stream));
        }
        GASB_CUDA(cudaStreamWaitEvent(t->copy_stream, t->ev_stage_free, 0));
        GASB_CUDA(cudaMemcpyAsync(t->x_stage.p, h, sizeof(float) * cnt, cudaMemcpyHostToDevice, t->copy_stream));
        GASB_CUDA(cudaEventRecord(t->ev_staged, t->copy_stream));
    });
}

gasb_status gasb_trainer_commit_features(gasb_trainer t) {
    return guard([&] {
        require(t, "trainer: null argument");
        if (!t->x_stage.p) throw std::logic_error("commit_features: nothing staged");
        // one device pass re-pitches the rows into X and rebuilds X's value flags (X is
        // replaced whole), ordered after the staged copy
        GASB_CUDA(cudaStreamWaitEvent(t->stream, t->ev_staged, 0));
        GASB_CUDA(cudaMemsetAsync(t->xflags.p, 0, sizeof(int32_t), t->stream));
        repitch_flags_kernel<<<1184, 256, 0, t->stream>>>(t->x_stage.p, t->n, t->F, t->X.p, t->ldF, t->xflags.p);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        GASB_CUDA(cudaEventRecord(t->ev_stage_free, t->stream));
    });
}

gasb_status gasb_trainer_set_features(gasb_trainer t, const float* h) {
    const gasb_status s = gasb_trainer_stage_features(t, h);
    return s != GASB_OK ? s : gasb_trainer_commit_features(t);
}

gasb_status gasb_trainer_profile_spmm(gasb_trainer t, int32_t part, int32_t layer, int32_t iters, float* avg_ms) {
    return guard([&] {
        require(t && avg_ms && iters > 0, "trainer: bad argument");
        require(part < t->num_parts && layer >= 1 && layer <= t->L, "trainer: part/layer out of range");
        require(part >= 0 || (layer == 1 && t->agg_all.p), "trainer: hoisted profile needs hoist_layer1");
        require(!t->residual || layer >= 2, "trainer: APPNP/GCNII layer 1 aggregates the per-batch head output");
        cudaEvent_t a, b;
        GASB_CUDA(cudaEventCreate(&a));
        GASB_CUDA(cudaEventCreate(&b));
        auto once = [&] {
            if (part < 0) {
                t->enqueue_hoisted();
                return;
            }
            const int32_t din = t->dims[layer - 1];
            const SpmmSegs segs = t->seg_batch.segs(part);
            const float* src = layer == 1 ? t->X.p : history_table(t->hist, layer - 1);
            const int64_t lds = layer == 1 ? t->ldF : history_ld(t->hist);
            float* out = t->residual ? t->prop.p : t->agg[layer].p;
            launch_spmm_fwd(segs, t->cols_g.p, t->coef64.p, src, lds, din, out, t->ld_of(din),
                            t->row_off[part], t->partial_batch.p, t->pld,
                            t->counters.p, t->max_chunks, t->stream, t->source_flags(layer),
                            t->source_tmap(layer));
        };
        once();  // warm
        GASB_CUDA(cudaEventRecord(a, t->stream));
        for (int32_t i = 0; i < iters; ++i) once();
        GASB_CUDA(cudaEventRecord(b, t->stream));
        GASB_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        GASB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *avg_ms = ms / static_cast<float>(iters);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

gasb_status gasb_host_register(void* h, size_t bytes) {
    return guard([&] { GASB_CUDA(cudaHostRegister(h, bytes, cudaHostRegisterDefault)); });
}

gasb_status gasb_host_unregister(void* h) {
    return guard([&] { GASB_CUDA(cudaHostUnregister(h)); });
}

gasb_status gasb_trainer_launch_count(gasb_trainer t, int64_t* out) {
    return guard([&] {
        require(t && out, "trainer: null argument");
        *out = t->epoch_launches;
    });
}

}  // extern "C"
