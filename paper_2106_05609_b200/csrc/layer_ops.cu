// Layer-level entry points: Layer::forward and its tape backward over one batch plan
// (include/gas/layers.hpp:51-72, src/layers.cpp:120-168), for callers that keep the
// reference's layer-by-layer structure (a Model::forward of their own) instead of the fused
// trainer. A gasb_batch_ops handle holds one plan's device stencils, built once:
//   gcn stencil   rows = the batch rows, cols = extended-node local ids (make_batch_plan order),
//                 fp64 coefficients pre-scaled by 2^896 (the SpMM's exact widening, spmm.cu),
//                 segment / range tables of one launch (rows cut at equal-edge boundaries)
//   CSC           the transposed stencil over EVERY extended row (tensor.cpp:531-549 writes
//                 all rows of h_in's gradient; the trainer needs only batch rows for GCN
//                 layers >= 2, this op keeps the reference's full contract)
//   batch_local_rows (select_rows of h0 for APPNP / GCNII)
// All calls are stream-ordered and capturable (no host synchronization).
#include <algorithm>
#include <cmath>
#include <vector>

#include "trainer_impl.hpp"  // DevBuf, schedule_of

struct gasb_batch_ops_s {
    int32_t nb = 0, ne = 0, max_dim = 0, nchunks = 0;
    int64_t nnz = 0;
    DevBuf<int32_t> cols, brow, t_src, ranges, seg_row, seg_slot, row_seg0, row_nseg, counters;
    DevBuf<int64_t> seg_beg, t_rowptr;
    DevBuf<double> coef64, partial;
    DevBuf<float> t_cf, wt;
    DevBuf<int32_t> special;
    int32_t nranges = 0;
    int64_t pld = 0;
    SpmmSegs segs() const {
        return SpmmSegs{seg_beg.p, seg_row.p, seg_slot.p, row_seg0.p, row_nseg.p, ranges.p, nranges, 0};
    }
    // y = A x (x: ne rows of width dim, pitch ldx); exact fp64 accumulation, rows segmented
    void aggregate(const float* x, int64_t ldx, int32_t dim, float* y, int64_t ldy, cudaStream_t st) {
        GASB_CUDA(cudaMemsetAsync(special.p, 0, sizeof(int32_t), st));
        launch_scan_special(x, ne, ldx, dim, special.p, st);  // selects the SpMM's widening path
        CUtensorMap tm;
        const bool have_tm = make_row_tmap(x, ne, dim, ldx, spmm_box_cols(dim), &tm);
        launch_spmm_fwd(segs(), cols.p, coef64.p, x, ldx, dim, y, ldy, 0, partial.p, pld, counters.p, nchunks, st,
                        special.p, have_tm ? &tm : nullptr);
    }
};

namespace {
void check_cfg(const gasb_layer_config* c, const gasb_batch_ops_s* b) {
    require(c != nullptr && b != nullptr, "Layer: null argument");
    require(c->kind == 0 || c->kind == 2 || c->kind == 3, "Layer: kind must be gcn (0), appnp (2) or gcnii (3)");
    require(c->in_dim > 0 && c->out_dim > 0, "LayerConfig: in_dim and out_dim must be positive");
    require(c->kind == 0 || c->in_dim == c->out_dim, "LayerConfig: appnp/gcnii need in_dim == out_dim");
    require(std::max(c->in_dim, c->out_dim) <= b->max_dim, "Layer: width exceeds the batch ops' max_dim");
}
}  // namespace

extern "C" {

gasb_status gasb_batch_ops_create(gasb_schedule s, int32_t part, int32_t max_dim, gasb_batch_ops* out) {
    return guard([&] {
        require(s && out, "batch_ops: null argument");
        const Schedule& S = schedule_of(s);
        require(part >= 0 && part < S.num_parts, "batch_ops: part out of range");
        require(max_dim > 0, "batch_ops: max_dim must be positive");
        const HostPlan& P = S.plans[part];
        auto b = std::make_unique<gasb_batch_ops_s>();
        b->nb = static_cast<int32_t>(P.batch.size());
        b->ne = static_cast<int32_t>(P.extended.size());
        b->nnz = static_cast<int64_t>(P.gcn_cols.size());
        b->max_dim = max_dim;
        b->nchunks = static_cast<int32_t>(ceil_div(max_dim, 64));
        std::vector<double> cd(P.gcn_coeffs.size());
        for (size_t e = 0; e < cd.size(); ++e) cd[e] = static_cast<double>(P.gcn_coeffs[e]) * kCoeffScale;
        b->cols.upload(P.gcn_cols);
        b->coef64.upload(cd);
        b->brow.upload(P.batch_local_rows);
        // segments of one launch over the batch rows (row pointers as absolute edge offsets)
        std::vector<int64_t> sb;
        std::vector<int32_t> sr, ss, r0(static_cast<size_t>(b->nb)), rn(static_cast<size_t>(b->nb));
        b->nranges = spmm_ranges_per_launch();
        std::vector<int32_t> rs(static_cast<size_t>(b->nranges) + 1);
        int64_t slots = 0;
        segment_launch(P.gcn_rowptr.data(), 0, b->nb, true, b->nranges, sb, sr, ss, r0.data(), rn.data(), slots,
                       rs.data());
        b->seg_beg.upload(sb);
        b->seg_row.upload(sr);
        b->seg_slot.upload(ss);
        b->row_seg0.upload(r0);
        b->row_nseg.upload(rn);
        b->ranges.upload(rs);
        b->pld = round_up(max_dim, 256);
        b->partial.alloc(std::max<int64_t>(slots, 1) * b->pld);
        b->counters.alloc(static_cast<int64_t>(std::max(b->nb, 1)) * b->nchunks);
        b->counters.zero();
        b->special.alloc(1);
        // CSC over every extended row: entries (batch row r, coeff), r ascending per target
        std::vector<int64_t> trp(static_cast<size_t>(b->ne) + 1, 0);
        for (int32_t c : P.gcn_cols) trp[c + 1]++;
        for (int32_t t = 0; t < b->ne; ++t) trp[t + 1] += trp[t];
        std::vector<int32_t> tsrc(static_cast<size_t>(b->nnz));
        std::vector<float> tcf(static_cast<size_t>(b->nnz));
        std::vector<int64_t> fill(trp.begin(), trp.end() - 1);
        for (int32_t r = 0; r < b->nb; ++r)
            for (int64_t e = P.gcn_rowptr[r]; e < P.gcn_rowptr[r + 1]; ++e) {
                const int64_t k = fill[P.gcn_cols[e]]++;
                tsrc[k] = r;
                tcf[k] = P.gcn_coeffs[e];
            }
        b->t_rowptr.upload(trp);
        b->t_src.upload(tsrc);
        b->t_cf.upload(tcf);
        b->wt.alloc(static_cast<int64_t>(max_dim) * round_up(max_dim, 4));
        GASB_CUDA(cudaDeviceSynchronize());
        *out = b.release();
    });
}

gasb_status gasb_batch_ops_sizes(gasb_batch_ops b, int32_t* num_batch, int32_t* num_extended) {
    return guard([&] {
        require(b, "batch_ops: null handle");
        if (num_batch) *num_batch = b->nb;
        if (num_extended) *num_extended = b->ne;
    });
}

gasb_status gasb_batch_ops_destroy(gasb_batch_ops b) {
    if (b) cudaDeviceSynchronize();
    delete b;
    return GASB_OK;
}

gasb_status gasb_layer_fwd(gasb_batch_ops b, const gasb_layer_config* cfg, const float* d_h_in, int64_t ld_in,
                           const float* d_h0, int64_t ld_h0, const float* d_w, int64_t ld_w, float* d_out,
                           int64_t ld_out, float* d_saved, int64_t ld_saved, gasb_stream stream) {
    return guard([&] {
        check_cfg(cfg, b);
        require(d_h_in && d_out && d_saved, "Layer: null buffer");
        require(ld_in >= cfg->in_dim && ld_out >= cfg->out_dim && ld_saved >= cfg->in_dim, "Layer: bad pitch");
        require(cfg->kind == 0 || d_h0, cfg->kind == 2 ? "APPNP: missing h0" : "GCNII: missing h0");
        require(cfg->kind == 2 || d_w, "Layer: missing weight");
        cudaStream_t st = as_stream(stream);
        set_gemm_workspace(nullptr, 0);
        const int32_t din = cfg->in_dim, dout = cfg->out_dim;
        switch (cfg->kind) {
            case 0:  // gcn_forward: matmul(aggregate(gcn, h), W)        (layers.cpp:138-141)
                b->aggregate(d_h_in, ld_in, din, d_saved, ld_saved, st);
                launch_gemm(0, b->nb, dout, din, d_saved, ld_saved, d_w, ld_w, d_out, ld_out, 0.f, false, nullptr, st);
                break;
            case 2:  // appnp_forward: alpha h0[B] + (1 - alpha) A h     (layers.cpp:150-157)
                b->aggregate(d_h_in, ld_in, din, d_saved, ld_saved, st);
                launch_mix(d_h0, ld_h0, b->brow.p, d_saved, ld_saved, b->nb, dout, cfg->alpha, d_out, ld_out, nullptr,
                           st);
                break;
            default: {  // gcnii_forward: mixed W~, W~ = (1 - beta) I + beta W   (layers.cpp:159-168)
                b->aggregate(d_h_in, ld_in, din, d_out, ld_out, st);  // prop (scratch in out)
                launch_mix(d_h0, ld_h0, b->brow.p, d_out, ld_out, b->nb, dout, cfg->alpha, d_saved, ld_saved, nullptr,
                           st);  // mixed (saved for the backward)
                const int64_t pw = round_up(dout, 4);
                GASB_CUDA(cudaMemcpy2DAsync(b->wt.p, sizeof(float) * pw, d_w, sizeof(float) * ld_w,
                                            sizeof(float) * dout, din, cudaMemcpyDeviceToDevice, st));
                launch_wtilde(b->wt.p, b->wt.p, 1, dout, pw, cfg->beta, st);
                launch_gemm(0, b->nb, dout, din, d_saved, ld_saved, b->wt.p, pw, d_out, ld_out, 0.f, false, nullptr,
                            st);
            }
        }
    });
}

gasb_status gasb_layer_bwd(gasb_batch_ops b, const gasb_layer_config* cfg, const float* d_gy, int64_t ld_gy,
                           const float* d_saved, int64_t ld_saved, const float* d_w, int64_t ld_w, float* d_gh_in,
                           int64_t ld_gh_in, float* d_gh0, int64_t ld_gh0, float* d_gw, int64_t ld_gw,
                           float* d_scratch, int64_t ld_scratch, gasb_stream stream) {
    return guard([&] {
        check_cfg(cfg, b);
        require(d_gy && d_scratch, "Layer backward: null buffer");
        require(ld_scratch >= std::max(cfg->in_dim, cfg->out_dim), "Layer backward: bad scratch pitch");
        cudaStream_t st = as_stream(stream);
        set_gemm_workspace(nullptr, 0);
        const int32_t din = cfg->in_dim, dout = cfg->out_dim;
        GemmEpilogue acc;
        acc.beta = 1.f;
        const float* gprop = d_gy;  // gradient of the aggregation output
        int64_t ldp = ld_gy;
        switch (cfg->kind) {
            case 0:
                // matmul backward (tensor.cpp:169-204): gW += agg^T gy, gagg = gy W^T
                if (d_gw) launch_gemm(2, din, dout, b->nb, d_saved, ld_saved, d_gy, ld_gy, d_gw, ld_gw, acc, st);
                if (d_gh_in) {
                    launch_gemm(1, b->nb, din, dout, d_gy, ld_gy, d_w, ld_w, d_scratch, ld_scratch, 0.f, false, nullptr,
                                st);
                    gprop = d_scratch;
                    ldp = ld_scratch;
                }
                break;
            case 2:
                // add/scale backward: h0[B] += alpha gy ; dprop = (1 - alpha) gy
                launch_mix_bwd(d_gy, ld_gy, b->nb, dout, cfg->alpha, b->brow.p, d_gh0, ld_gh0, d_scratch, ld_scratch,
                               st);
                gprop = d_scratch;
                ldp = ld_scratch;
                break;
            default: {
                // W~ = (1 - beta) I + beta W: gW += beta (mixed^T gy); dmixed = gy W~^T
                const int64_t pw = round_up(dout, 4);
                GASB_CUDA(cudaMemcpy2DAsync(b->wt.p, sizeof(float) * pw, d_w, sizeof(float) * ld_w,
                                            sizeof(float) * dout, din, cudaMemcpyDeviceToDevice, st));
                launch_wtilde(b->wt.p, b->wt.p, 1, dout, pw, cfg->beta, st);
                if (d_gw) {
                    GemmEpilogue e;
                    e.beta = 1.f;
                    e.post_scale = cfg->beta;
                    launch_gemm(2, din, dout, b->nb, d_saved, ld_saved, d_gy, ld_gy, d_gw, ld_gw, e, st);
                }
                // dmixed into the scratch, then the mixing backward in place (dprop = (1-a) dmixed)
                launch_gemm(1, b->nb, din, dout, d_gy, ld_gy, b->wt.p, pw, d_scratch, ld_scratch, 0.f, false, nullptr,
                            st);
                launch_mix_bwd(d_scratch, ld_scratch, b->nb, din, cfg->alpha, b->brow.p, d_gh0, ld_gh0, d_scratch,
                               ld_scratch, st);
                gprop = d_scratch;
                ldp = ld_scratch;
            }
        }
        // aggregate backward (tensor.cpp:531-549): h_in.grad[t] += sum c * gprop[r], every V_b row
        if (d_gh_in)
            launch_spmm_bwd(b->t_rowptr.p, b->ne, b->t_src.p, b->t_cf.p, gprop, ldp, din, nullptr, 0, d_gh_in,
                            ld_gh_in, st, b->nb, /*accumulate=*/true);
    });
}

}  // extern "C"
