// Message-passing aggregation: the reference's `aggregate` (src/tensor.cpp:514-549) as
// sm_100a kernels over per-batch CSR stencils.
//
// Forward (tensor.cpp:519-529): y[r,:] = sum_e double(c_e) * double(x[col_e,:]) in CSR
// order, rounded once to fp32. The product of two fp32 values is exact in fp64, so
// fma(c, x, acc) == acc + c*x rounded once == the reference's `acc += c * src` -> the
// sequential mode (one segment per row) is bit-exact. Work item = (segment, 64-column
// chunk) per warp; lanes own 2 adjacent columns (float2 loads, 256 B per row per warp);
// the grid is chunk-major so all resident warps gather the same 256 B column slice and
// the slice of the source table stays L2-resident (column chunking).
// Power-law rows are split into segments of <= S edges; their fp64 partials are summed in
// segment order by the last-arriving warp (deterministic, no float atomics).
//
// Backward (tensor.cpp:531-549): the scatter gx[col_e] += c_e * gy[r] becomes a gather
// over the transposed stencil, entries of each target in ascending r with fp32
// multiply-then-add -> bit-exact; relu backward (tensor.cpp:363-369) fused as a mask.
#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {

constexpr int kChunk = 64;  // columns per warp work item
constexpr int kUnroll = 8;  // edges in flight per lane

__global__ void __launch_bounds__(256) spmm_fwd_kernel(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, int64_t nseg, int64_t seg_base,
    const int32_t* __restrict__ cols, const double* __restrict__ coeffs, const float* __restrict__ x, int64_t ldx,
    int32_t dim, int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base, double* __restrict__ partial,
    int64_t pld, int32_t* __restrict__ counters, int32_t cld) {
    const int lane = threadIdx.x & 31;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= nseg * nchunks) return;
    const int32_t chunk = static_cast<int32_t>(w / nseg);
    const int64_t s = seg_base + (w - static_cast<int64_t>(chunk) * nseg);
    const int32_t col = chunk * kChunk + lane * 2;
    const bool active = col < dim;
    const float* xc = x + col;
    const int64_t e0 = seg_beg[s], e1 = seg_beg[s + 1];
    double a0 = 0.0, a1 = 0.0;
    for (int64_t eb = e0; eb < e1; eb += 32) {
        const int cnt = static_cast<int>((e1 - eb) < 32 ? (e1 - eb) : 32);
        const int32_t my_col = lane < cnt ? __ldg(cols + eb + lane) : 0;
        const double my_cf = lane < cnt ? __ldg(coeffs + eb + lane) : 0.0;
        int j = 0;
        for (; j + kUnroll <= cnt; j += kUnroll) {
            float2 v[kUnroll];
            double cf[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int32_t cc = __shfl_sync(0xffffffffu, my_col, j + u);
                cf[u] = __shfl_sync(0xffffffffu, my_cf, j + u);
                v[u] = active ? __ldg(reinterpret_cast<const float2*>(xc + static_cast<int64_t>(cc) * ldx))
                              : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                a0 = __fma_rn(cf[u], static_cast<double>(v[u].x), a0);
                a1 = __fma_rn(cf[u], static_cast<double>(v[u].y), a1);
            }
        }
        for (; j < cnt; ++j) {
            const int32_t cc = __shfl_sync(0xffffffffu, my_col, j);
            const double cf = __shfl_sync(0xffffffffu, my_cf, j);
            const float2 v = active ? __ldg(reinterpret_cast<const float2*>(xc + static_cast<int64_t>(cc) * ldx))
                                    : make_float2(0.f, 0.f);
            a0 = __fma_rn(cf, static_cast<double>(v.x), a0);
            a1 = __fma_rn(cf, static_cast<double>(v.y), a1);
        }
    }
    const int32_t row = seg_row[s];
    const int32_t slot = seg_slot[s];
    float* yr = y + (static_cast<int64_t>(row) - row_base) * ldy;
    if (slot < 0) {
        if (col + 1 < dim) *reinterpret_cast<float2*>(yr + col) = make_float2(static_cast<float>(a0), static_cast<float>(a1));
        else if (active) yr[col] = static_cast<float>(a0);
        return;
    }
    // multi-segment row: publish the fp64 partial, last arriving warp combines in order
    *reinterpret_cast<double2*>(partial + static_cast<int64_t>(slot) * pld + col) = make_double2(a0, a1);
    __threadfence();
    __syncwarp();
    int last = 0;
    const int32_t k = row_nseg[row];
    if (lane == 0) last = atomicAdd(counters + static_cast<int64_t>(row) * cld + chunk, 1) == k - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    const int32_t s0 = row_seg0[row];
    double b0 = 0.0, b1 = 0.0;
    for (int32_t i = 0; i < k; ++i) {
        const int32_t sl = seg_slot[s0 + i];
        const double2 p = __ldcg(reinterpret_cast<const double2*>(partial + static_cast<int64_t>(sl) * pld + col));
        b0 += p.x;
        b1 += p.y;
    }
    if (col + 1 < dim) *reinterpret_cast<float2*>(yr + col) = make_float2(static_cast<float>(b0), static_cast<float>(b1));
    else if (active) yr[col] = static_cast<float>(b0);
    if (lane == 0) counters[static_cast<int64_t>(row) * cld + chunk] = 0;  // self-reset for the next launch
}

void launch_spmm_fwd(const SpmmSegs& s, const int32_t* cols, const double* coeffs, const float* x, int64_t ldx,
                     int32_t dim, float* y, int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld,
                     int32_t* counters, int32_t counters_ld, cudaStream_t st) {
    if (s.nseg <= 0 || dim <= 0) return;
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kChunk));
    require(ldx % 2 == 0 && ldy % 2 == 0, "spmm_fwd: leading dimensions must be even");
    require(nchunks <= counters_ld, "spmm_fwd: counters too narrow");
    const int64_t warps = s.nseg * nchunks;
    const int64_t blocks = ceil_div(warps, 8);
    spmm_fwd_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        s.seg_beg, s.seg_row, s.seg_slot, s.row_seg0, s.row_nseg, s.nseg, s.seg_base, cols, coeffs, x, ldx, dim,
        nchunks, y, ldy, row_base, partial, partial_ld, counters, counters_ld);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(256) spmm_bwd_kernel(const int64_t* __restrict__ rp, int32_t nt,
                                                       const int32_t* __restrict__ src, const float* __restrict__ cf,
                                                       const float* __restrict__ gy, int64_t ldgy, int32_t dim,
                                                       int32_t nchunks, const float* __restrict__ mask, int64_t ldm,
                                                       float* __restrict__ gx, int64_t ldgx) {
    const int lane = threadIdx.x & 31;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= static_cast<int64_t>(nt) * nchunks) return;
    const int32_t chunk = static_cast<int32_t>(w / nt);
    const int32_t t = static_cast<int32_t>(w - static_cast<int64_t>(chunk) * nt);
    const int32_t col = chunk * kChunk + lane * 2;
    const bool active = col < dim;
    const float* gc = gy + col;
    float a0 = 0.0f, a1 = 0.0f;
    const int64_t e0 = rp[t], e1 = rp[t + 1];
    for (int64_t eb = e0; eb < e1; eb += 32) {
        const int cnt = static_cast<int>((e1 - eb) < 32 ? (e1 - eb) : 32);
        const int32_t my_r = lane < cnt ? __ldg(src + eb + lane) : 0;
        const float my_c = lane < cnt ? __ldg(cf + eb + lane) : 0.0f;
        int j = 0;
        for (; j + kUnroll <= cnt; j += kUnroll) {
            float2 v[kUnroll];
            float c[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int32_t r = __shfl_sync(0xffffffffu, my_r, j + u);
                c[u] = __shfl_sync(0xffffffffu, my_c, j + u);
                v[u] = active ? __ldg(reinterpret_cast<const float2*>(gc + static_cast<int64_t>(r) * ldgy))
                              : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                a0 = __fadd_rn(a0, __fmul_rn(c[u], v[u].x));
                a1 = __fadd_rn(a1, __fmul_rn(c[u], v[u].y));
            }
        }
        for (; j < cnt; ++j) {
            const int32_t r = __shfl_sync(0xffffffffu, my_r, j);
            const float c = __shfl_sync(0xffffffffu, my_c, j);
            const float2 v = active ? __ldg(reinterpret_cast<const float2*>(gc + static_cast<int64_t>(r) * ldgy))
                                    : make_float2(0.f, 0.f);
            a0 = __fadd_rn(a0, __fmul_rn(c, v.x));
            a1 = __fadd_rn(a1, __fmul_rn(c, v.y));
        }
    }
    if (!active) return;
    if (mask) {
        const float* mr = mask + static_cast<int64_t>(t) * ldm + col;
        if (!(mr[0] > 0.0f)) a0 = 0.0f;
        if (col + 1 < dim && !(mr[1] > 0.0f)) a1 = 0.0f;
    }
    float* o = gx + static_cast<int64_t>(t) * ldgx + col;
    if (col + 1 < dim) *reinterpret_cast<float2*>(o) = make_float2(a0, a1);
    else o[0] = a0;
}

void launch_spmm_bwd(const int64_t* t_rowptr, int32_t nt, const int32_t* t_src, const float* t_coeffs,
                     const float* gy, int64_t ldgy, int32_t dim, const float* mask, int64_t ldm, float* gx,
                     int64_t ldgx, cudaStream_t st) {
    if (nt <= 0 || dim <= 0) return;
    require(ldgy % 2 == 0 && ldgx % 2 == 0 && (!mask || ldm % 2 == 0), "spmm_bwd: leading dimensions must be even");
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kChunk));
    const int64_t blocks = ceil_div(static_cast<int64_t>(nt) * nchunks, 8);
    spmm_bwd_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(t_rowptr, nt, t_src, t_coeffs, gy, ldgy, dim,
                                                                   nchunks, mask, ldm, gx, ldgx);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

}  // namespace gasb

using namespace gasb;

// ---- standalone C-ABI entry points (op-level parity tests) ---------------------------
namespace {
struct SegScratch {
    int64_t* seg_beg = nullptr;
    int32_t *seg_row = nullptr, *seg_slot = nullptr, *row_seg0 = nullptr, *row_nseg = nullptr, *counters = nullptr;
    double* partial = nullptr;
    int64_t* rp64 = nullptr;
};
}  // namespace

extern "C" gasb_status gasb_spmm_fwd(const int32_t* d_rowptr, int32_t m, const int32_t* d_cols, const float* d_coeffs,
                                     const float* d_x, int64_t ldx, int32_t dim, float* d_y, int64_t ldy,
                                     int32_t seg_edges, gasb_stream stream) {
    return guard([&] {
        require(m >= 0 && dim >= 0 && seg_edges >= 0, "aggregate: bad shape");
        if (m == 0 || dim == 0) return;
        cudaStream_t st = as_stream(stream);
        // Segmentation is host work: read the row pointer, build segments, upload.
        std::vector<int32_t> rp(static_cast<size_t>(m) + 1);
        GASB_CUDA(cudaMemcpyAsync(rp.data(), d_rowptr, sizeof(int32_t) * (m + 1), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        const int64_t nnz = rp[m];
        std::vector<int64_t> sb;
        std::vector<int32_t> sr, ss, r0(static_cast<size_t>(m)), rn(static_cast<size_t>(m));
        int32_t slots = 0;
        for (int32_t r = 0; r < m; ++r) {
            require(rp[r + 1] >= rp[r], "aggregate: row pointer not monotone");
            const int64_t deg = rp[r + 1] - rp[r];
            const int64_t k = (seg_edges == 0 || deg <= seg_edges) ? 1 : ceil_div(deg, seg_edges);
            r0[r] = static_cast<int32_t>(sr.size());
            rn[r] = static_cast<int32_t>(k);
            for (int64_t i = 0; i < k; ++i) {
                sb.push_back(rp[r] + i * (k == 1 ? 0 : seg_edges));
                sr.push_back(r);
                ss.push_back(k == 1 ? -1 : slots++);
            }
        }
        sb.push_back(nnz);
        const int64_t nseg = static_cast<int64_t>(sr.size());
        const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kChunk));
        SegScratch z;
        double* coeffs64 = nullptr;
        GASB_CUDA(cudaMallocAsync(&z.seg_beg, sizeof(int64_t) * (nseg + 1), st));
        GASB_CUDA(cudaMallocAsync(&z.seg_row, sizeof(int32_t) * nseg, st));
        GASB_CUDA(cudaMallocAsync(&z.seg_slot, sizeof(int32_t) * nseg, st));
        GASB_CUDA(cudaMallocAsync(&z.row_seg0, sizeof(int32_t) * m, st));
        GASB_CUDA(cudaMallocAsync(&z.row_nseg, sizeof(int32_t) * m, st));
        GASB_CUDA(cudaMallocAsync(&z.counters, sizeof(int32_t) * m * nchunks, st));
        GASB_CUDA(cudaMallocAsync(&z.partial, sizeof(double) * std::max<int64_t>(slots, 1) * nchunks * kChunk, st));
        GASB_CUDA(cudaMallocAsync(&coeffs64, sizeof(double) * std::max<int64_t>(nnz, 1), st));
        GASB_CUDA(cudaMemcpyAsync(z.seg_beg, sb.data(), sizeof(int64_t) * (nseg + 1), cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemcpyAsync(z.seg_row, sr.data(), sizeof(int32_t) * nseg, cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemcpyAsync(z.seg_slot, ss.data(), sizeof(int32_t) * nseg, cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemcpyAsync(z.row_seg0, r0.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemcpyAsync(z.row_nseg, rn.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemsetAsync(z.counters, 0, sizeof(int32_t) * m * nchunks, st));
        {
            std::vector<float> cf(static_cast<size_t>(nnz));
            std::vector<double> cd(static_cast<size_t>(nnz));
            GASB_CUDA(cudaMemcpyAsync(cf.data(), d_coeffs, sizeof(float) * nnz, cudaMemcpyDeviceToHost, st));
            GASB_CUDA(cudaStreamSynchronize(st));
            for (int64_t e = 0; e < nnz; ++e) cd[e] = cf[e];
            GASB_CUDA(cudaMemcpyAsync(coeffs64, cd.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
            SpmmSegs segs{z.seg_beg, z.seg_row, z.seg_slot, z.row_seg0, z.row_nseg, nseg, 0};
            launch_spmm_fwd(segs, d_cols, coeffs64, d_x, ldx, dim, d_y, ldy, 0, z.partial,
                            static_cast<int64_t>(nchunks) * kChunk, z.counters, nchunks, st);
            GASB_CUDA(cudaStreamSynchronize(st));
        }
        cudaFreeAsync(z.seg_beg, st);
        cudaFreeAsync(z.seg_row, st);
        cudaFreeAsync(z.seg_slot, st);
        cudaFreeAsync(z.row_seg0, st);
        cudaFreeAsync(z.row_nseg, st);
        cudaFreeAsync(z.counters, st);
        cudaFreeAsync(z.partial, st);
        cudaFreeAsync(coeffs64, st);
        GASB_CUDA(cudaStreamSynchronize(st));
    });
}

extern "C" gasb_status gasb_spmm_bwd(const int32_t* d_t_rowptr, int32_t nt, const int32_t* d_t_src,
                                     const float* d_t_coeffs, const float* d_gy, int64_t ldgy, int32_t dim,
                                     const float* d_mask, int64_t ldm, float* d_gx, int64_t ldgx, gasb_stream stream) {
    return guard([&] {
        require(nt >= 0 && dim >= 0, "aggregate backward: bad shape");
        if (nt == 0 || dim == 0) return;
        cudaStream_t st = as_stream(stream);
        int64_t* rp64 = nullptr;
        std::vector<int32_t> rp(static_cast<size_t>(nt) + 1);
        GASB_CUDA(cudaMemcpyAsync(rp.data(), d_t_rowptr, sizeof(int32_t) * (nt + 1), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> r64(rp.begin(), rp.end());
        GASB_CUDA(cudaMallocAsync(&rp64, sizeof(int64_t) * (nt + 1), st));
        GASB_CUDA(cudaMemcpyAsync(rp64, r64.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, st));
        launch_spmm_bwd(rp64, nt, d_t_src, d_t_coeffs, d_gy, ldgy, dim, d_mask, ldm, d_gx, ldgx, st);
        cudaFreeAsync(rp64, st);
        GASB_CUDA(cudaStreamSynchronize(st));
    });
}
