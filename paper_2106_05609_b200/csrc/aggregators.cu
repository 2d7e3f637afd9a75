// max and mean neighbourhood aggregation (north_star item 3: "sum/mean/max SpMM"), forward
// and backward, over the same CSR batch stencils as the weighted-sum aggregate (spmm.cu).
//
// The reference implements only weighted sums (`aggregate`, src/tensor.cpp:514-549, with the
// gcn and sum stencils of src/layers.cpp:42-70), so these two have no reference counterpart:
// they are pinned to their definitions (oracle/aggregators.py), which fix every rounding:
//   max  : y[r,j] = x[c_b, j] for the first edge b of row r, then replaced in CSR order by any
//          strictly greater value (the first occurrence of the maximum wins; a NaN survives only
//          as the first value); argmax[r,j] = that edge's index; an empty row gives 0 and -1.
//          Backward: gx[s,j] = sum, rows ascending, of gy[r,j] over the edges (r -> s) that are
//          argmax[r,j] (fp32 adds) — deterministic, no atomics.
//   mean : y[r,j] = float(fp64 CSR-order sum of x[c,j] / deg r) (0 for an empty row).
//          Backward: gasb_spmm_bwd with coefficients float(1.0 / deg r) (gasb_mean_coefficients).
// Layout: lanes over 32 consecutive columns of a row, one warp per (row, 32-column chunk) —
// each edge is one coalesced 128 B row-slice load; rows run in parallel across warps. These
// are op-level kernels (the trainer's GCN path uses the weighted-sum SpMM), so they favour a
// simple, exactly specified order over the flat engine's segmentation.
#include <algorithm>
#include <vector>

#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {
namespace {

constexpr int kAggWarps = 8;

__global__ void __launch_bounds__(kAggWarps * 32) max_fwd_kernel(const int32_t* __restrict__ rp, int32_t m,
                                                                 const int32_t* __restrict__ cols,
                                                                 const float* __restrict__ x, int64_t ldx, int32_t dim,
                                                                 float* __restrict__ y, int64_t ldy,
                                                                 int32_t* __restrict__ arg, int64_t lda) {
    const int lane = threadIdx.x & 31;
    const int32_t nchunks = (dim + 31) / 32;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kAggWarps + (threadIdx.x >> 5);
    if (w >= static_cast<int64_t>(m) * nchunks) return;
    const int32_t r = static_cast<int32_t>(w / nchunks), j = static_cast<int32_t>(w % nchunks) * 32 + lane;
    const int32_t b = rp[r], e = rp[r + 1];
    float best = 0.0f;
    int32_t bi = -1;
    if (j < dim && b < e) {
        best = __ldg(x + static_cast<int64_t>(cols[b]) * ldx + j);
        bi = b;
#pragma unroll 4
        for (int32_t k = b + 1; k < e; ++k) {
            const float v = __ldg(x + static_cast<int64_t>(cols[k]) * ldx + j);
            if (v > best) {
                best = v;
                bi = k;
            }
        }
    }
    if (j < dim) {
        y[static_cast<int64_t>(r) * ldy + j] = best;
        if (arg) arg[static_cast<int64_t>(r) * lda + j] = bi;
    }
}

// t_rp / t_edge / t_row: the stencil transposed by source (entries in ascending row, then edge).
__global__ void __launch_bounds__(kAggWarps * 32) max_bwd_kernel(const int32_t* __restrict__ t_rp, int32_t ns,
                                                                 const int32_t* __restrict__ t_edge,
                                                                 const int32_t* __restrict__ t_row,
                                                                 const int32_t* __restrict__ arg, int64_t lda,
                                                                 const float* __restrict__ gy, int64_t ldgy,
                                                                 int32_t dim, float* __restrict__ gx, int64_t ldgx) {
    const int lane = threadIdx.x & 31;
    const int32_t nchunks = (dim + 31) / 32;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kAggWarps + (threadIdx.x >> 5);
    if (w >= static_cast<int64_t>(ns) * nchunks) return;
    const int32_t s = static_cast<int32_t>(w / nchunks), j = static_cast<int32_t>(w % nchunks) * 32 + lane;
    if (j >= dim) return;
    float acc = 0.0f;
    for (int32_t k = t_rp[s]; k < t_rp[s + 1]; ++k) {
        const int32_t r = t_row[k];
        if (arg[static_cast<int64_t>(r) * lda + j] == t_edge[k]) acc = __fadd_rn(acc, gy[static_cast<int64_t>(r) * ldgy + j]);
    }
    gx[static_cast<int64_t>(s) * ldgx + j] = acc;
}

__global__ void __launch_bounds__(kAggWarps * 32) mean_fwd_kernel(const int32_t* __restrict__ rp, int32_t m,
                                                                  const int32_t* __restrict__ cols,
                                                                  const float* __restrict__ x, int64_t ldx,
                                                                  int32_t dim, float* __restrict__ y, int64_t ldy) {
    const int lane = threadIdx.x & 31;
    const int32_t nchunks = (dim + 31) / 32;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kAggWarps + (threadIdx.x >> 5);
    if (w >= static_cast<int64_t>(m) * nchunks) return;
    const int32_t r = static_cast<int32_t>(w / nchunks), j = static_cast<int32_t>(w % nchunks) * 32 + lane;
    if (j >= dim) return;
    const int32_t b = rp[r], e = rp[r + 1];
    double acc = 0.0;
#pragma unroll 4
    for (int32_t k = b; k < e; ++k) acc = __dadd_rn(acc, static_cast<double>(__ldg(x + static_cast<int64_t>(cols[k]) * ldx + j)));
    y[static_cast<int64_t>(r) * ldy + j] = e > b ? static_cast<float>(__ddiv_rn(acc, static_cast<double>(e - b))) : 0.0f;
}

unsigned blocks_for(int64_t warps) { return static_cast<unsigned>((warps + kAggWarps - 1) / kAggWarps); }

void check_stencil(const std::vector<int32_t>& rp, const std::vector<int32_t>& cols, int32_t num_src) {
    for (size_t r = 1; r < rp.size(); ++r) require(rp[r] >= rp[r - 1], "aggregate: row pointer not monotone");
    require(rp.empty() || rp[0] == 0, "aggregate: row pointer must start at 0");
    for (int32_t c : cols) require(c >= 0 && c < num_src, "aggregate: source row out of range");
}

}  // namespace
}  // namespace gasb

using namespace gasb;

extern "C" gasb_status gasb_spmm_max_fwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols,
                                         const float* d_x, int32_t num_src, int64_t ldx, int32_t dim, float* d_y,
                                         int64_t ldy, int32_t* d_argmax, int64_t ld_arg, gasb_stream stream) {
    return guard([&] {
        require(num_dst >= 0 && num_src >= 0 && dim >= 0, "aggregate: bad shape");
        require(ldx >= dim && ldy >= dim && (!d_argmax || ld_arg >= dim), "aggregate: leading dimension < dim");
        if (num_dst == 0 || dim == 0) return;
        cudaStream_t st = as_stream(stream);
        std::vector<int32_t> rp(static_cast<size_t>(num_dst) + 1);
        GASB_CUDA(cudaMemcpyAsync(rp.data(), d_rowptr, sizeof(int32_t) * rp.size(), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> cols(static_cast<size_t>(std::max(rp.back(), 0)));
        if (!cols.empty())
            GASB_CUDA(cudaMemcpyAsync(cols.data(), d_cols, sizeof(int32_t) * cols.size(), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        check_stencil(rp, cols, num_src);  // the reference's aggregate range check (tensor.cpp:515)
        const int64_t warps = static_cast<int64_t>(num_dst) * ((dim + 31) / 32);
        max_fwd_kernel<<<blocks_for(warps), kAggWarps * 32, 0, st>>>(d_rowptr, num_dst, d_cols, d_x, ldx, dim, d_y,
                                                                      ldy, d_argmax, ld_arg);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
    });
}

extern "C" gasb_status gasb_spmm_max_bwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols,
                                         const int32_t* d_argmax, int64_t ld_arg, const float* d_gy, int64_t ldgy,
                                         int32_t num_src, int32_t dim, float* d_gx, int64_t ldgx,
                                         gasb_stream stream) {
    return guard([&] {
        require(num_dst >= 0 && num_src >= 0 && dim >= 0, "aggregate: bad shape");
        require(ld_arg >= dim && ldgy >= dim && ldgx >= dim, "aggregate: leading dimension < dim");
        if (num_src == 0 || dim == 0) return;
        cudaStream_t st = as_stream(stream);
        std::vector<int32_t> rp(static_cast<size_t>(num_dst) + 1);
        GASB_CUDA(cudaMemcpyAsync(rp.data(), d_rowptr, sizeof(int32_t) * rp.size(), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        const int64_t nnz = std::max(rp.back(), 0);
        std::vector<int32_t> cols(static_cast<size_t>(nnz));
        if (nnz) GASB_CUDA(cudaMemcpyAsync(cols.data(), d_cols, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        check_stencil(rp, cols, num_src);
        // transpose by source: entries in ascending row (then edge) order
        std::vector<int32_t> t_rp(static_cast<size_t>(num_src) + 1, 0), t_edge(static_cast<size_t>(nnz)),
            t_row(static_cast<size_t>(nnz));
        for (int32_t c : cols) ++t_rp[c + 1];
        for (int32_t s = 0; s < num_src; ++s) t_rp[s + 1] += t_rp[s];
        std::vector<int32_t> fill(t_rp.begin(), t_rp.end() - 1);
        for (int32_t r = 0; r < num_dst; ++r)
            for (int32_t k = rp[r]; k < rp[r + 1]; ++k) {
                const int32_t q = fill[cols[k]]++;
                t_edge[q] = k;
                t_row[q] = r;
            }
        int32_t *d_trp = nullptr, *d_te = nullptr, *d_tr = nullptr;
        GASB_CUDA(cudaMallocAsync(&d_trp, sizeof(int32_t) * t_rp.size(), st));
        GASB_CUDA(cudaMallocAsync(&d_te, sizeof(int32_t) * std::max<int64_t>(nnz, 1), st));
        GASB_CUDA(cudaMallocAsync(&d_tr, sizeof(int32_t) * std::max<int64_t>(nnz, 1), st));
        GASB_CUDA(cudaMemcpyAsync(d_trp, t_rp.data(), sizeof(int32_t) * t_rp.size(), cudaMemcpyHostToDevice, st));
        if (nnz) {
            GASB_CUDA(cudaMemcpyAsync(d_te, t_edge.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
            GASB_CUDA(cudaMemcpyAsync(d_tr, t_row.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
        }
        const int64_t warps = static_cast<int64_t>(num_src) * ((dim + 31) / 32);
        max_bwd_kernel<<<blocks_for(warps), kAggWarps * 32, 0, st>>>(d_trp, num_src, d_te, d_tr, d_argmax, ld_arg,
                                                                      d_gy, ldgy, dim, d_gx, ldgx);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        GASB_CUDA(cudaFreeAsync(d_trp, st));
        GASB_CUDA(cudaFreeAsync(d_te, st));
        GASB_CUDA(cudaFreeAsync(d_tr, st));
        GASB_CUDA(cudaStreamSynchronize(st));  // the host staging vectors die here
    });
}

extern "C" gasb_status gasb_spmm_mean_fwd(const int32_t* d_rowptr, int32_t num_dst, const int32_t* d_cols,
                                          const float* d_x, int32_t num_src, int64_t ldx, int32_t dim, float* d_y,
                                          int64_t ldy, gasb_stream stream) {
    return guard([&] {
        require(num_dst >= 0 && num_src >= 0 && dim >= 0, "aggregate: bad shape");
        require(ldx >= dim && ldy >= dim, "aggregate: leading dimension < dim");
        if (num_dst == 0 || dim == 0) return;
        cudaStream_t st = as_stream(stream);
        std::vector<int32_t> rp(static_cast<size_t>(num_dst) + 1);
        GASB_CUDA(cudaMemcpyAsync(rp.data(), d_rowptr, sizeof(int32_t) * rp.size(), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> cols(static_cast<size_t>(std::max(rp.back(), 0)));
        if (!cols.empty())
            GASB_CUDA(cudaMemcpyAsync(cols.data(), d_cols, sizeof(int32_t) * cols.size(), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        check_stencil(rp, cols, num_src);
        const int64_t warps = static_cast<int64_t>(num_dst) * ((dim + 31) / 32);
        mean_fwd_kernel<<<blocks_for(warps), kAggWarps * 32, 0, st>>>(d_rowptr, num_dst, d_cols, d_x, ldx, dim, d_y,
                                                                       ldy);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
    });
}

extern "C" gasb_status gasb_mean_coefficients(const int32_t* h_rowptr, int32_t num_dst, float* h_coeffs) {
    return guard([&] {
        require(num_dst >= 0 && h_rowptr && (num_dst == 0 || h_coeffs), "mean_coefficients: null argument");
        for (int32_t r = 0; r < num_dst; ++r) {
            const int32_t b = h_rowptr[r], e = h_rowptr[r + 1];
            require(e >= b, "aggregate: row pointer not monotone");
            const float c = static_cast<float>(1.0 / static_cast<double>(e - b));
            for (int32_t k = b; k < e; ++k) h_coeffs[k] = c;
        }
    });
}
