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

// ---- pipelined forward (cp.async staging) ----------------------------------------------
// Work item = (segment, chunk of 32*CPL columns) per warp; each lane owns CPL adjacent
// columns. Edges go in stages of 64/CPL; for each stage the source-row slices (8 KB) are
// copied global->shared with cp.async (LDGSTS.128, zero-fill past the row pitch) kStages
// stages ahead of the FMAs, and the stage's fp64 coefficients go to shared memory for
// broadcast reads. The FMAs walk the stage's rows in order, so the fp64 accumulation is
// exactly the CSR order of the segment (bit-exact per segment).
//
// Widening fp32 -> fp64 without F2F. F2F.F64.F32 issues to the XU pipe, which ncu showed
// saturated (94%) in this kernel. Instead the coefficients are stored pre-scaled by 2^896
// (exact) and the source value x is re-laid-out as the double D = x * 2^-896 (exact for
// every finite float, zeros and denormals included):
//   non-negative x : hi = u >> 3,                               lo = u << 29   (2 int ops)
//   signed x       : hi = ((u & 0x7fffffff) >> 3) | (u & sign), lo = u << 29   (4 int ops)
// so fma(c * 2^896, D, acc) == acc + c*x rounded once — the reference's `acc += c * src`.
// A per-table flag word (kTableNeg / kTableNonFinite) selects the path; tables holding
// inf/nan take F2F (D = double(x) * 2^-896, also exact).
constexpr int kStages = 3;
constexpr int kPipeWarps = 4;
constexpr int kStageDataBytes = 8192;

enum WidenMode { kWidenF2F = 0, kWidenSigned = 1, kWidenNonNeg = 2 };

template <int MODE>
__device__ __forceinline__ double widen_scaled(float f) {
    const uint32_t u = __float_as_uint(f);
    if (MODE == kWidenNonNeg)
        return __hiloint2double(static_cast<int>(u >> 3), static_cast<int>(u << 29));
    if (MODE == kWidenSigned)
        return __hiloint2double(static_cast<int>(((u & 0x7fffffffu) >> 3) | (u & 0x80000000u)),
                                static_cast<int>(u << 29));
    return __dmul_rn(static_cast<double>(f), 0x1.0p-896);
}

__device__ __forceinline__ int widen_mode(const int32_t* flags) {
    const int32_t f = flags ? *flags : kTableNonFinite;
    return (f & kTableNonFinite) ? kWidenF2F : (f & kTableNeg) ? kWidenSigned : kWidenNonNeg;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int CPL>
struct PipeCfg {
    static constexpr int kCols = 32 * CPL;                       // columns per work item
    static constexpr int kEdges = kStageDataBytes / (kCols * 4);  // edges per stage (32 | 16)
    static constexpr int kPieces = kCols / 4;                     // 16 B pieces per row slice
    static constexpr int kRowsPerIssue = 32 / kPieces;            // rows per LDGSTS instruction
    static constexpr int kStageBytes = kStageDataBytes + kEdges * 8;
    static constexpr int kSmem = kPipeWarps * kStages * kStageBytes;
};

// One stage of FMAs: rows of the stage in CSR order, CPL fp64 accumulators per lane.
template <int CPL, int MODE>
__device__ __forceinline__ void stage_fma(const float* rows, const double* cf, int cnt, double (&acc)[CPL]) {
    constexpr int kCols = 32 * CPL;
#pragma unroll 8
    for (int j = 0; j < cnt; ++j) {
        const double c = cf[j];
        if constexpr (CPL == 4) {
            const float4 v = *reinterpret_cast<const float4*>(rows + j * kCols);
            acc[0] = __fma_rn(c, widen_scaled<MODE>(v.x), acc[0]);
            acc[1] = __fma_rn(c, widen_scaled<MODE>(v.y), acc[1]);
            acc[2] = __fma_rn(c, widen_scaled<MODE>(v.z), acc[2]);
            acc[3] = __fma_rn(c, widen_scaled<MODE>(v.w), acc[3]);
        } else {
            const float2 v = *reinterpret_cast<const float2*>(rows + j * kCols);
            acc[0] = __fma_rn(c, widen_scaled<MODE>(v.x), acc[0]);
            acc[1] = __fma_rn(c, widen_scaled<MODE>(v.y), acc[1]);
        }
    }
}

// coeffs are the stencil coefficients pre-scaled by 2^896 (see widen_scaled).
template <int CPL>
__global__ void __launch_bounds__(kPipeWarps * 32, 2) spmm_fwd_pipe_kernel(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, int64_t nseg, int64_t seg_base,
    const int32_t* __restrict__ cols, const double* __restrict__ coeffs, const float* __restrict__ x, int64_t ldx,
    int32_t dim, int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base, double* __restrict__ partial,
    int64_t pld, int32_t* __restrict__ counters, int32_t cld, const int32_t* __restrict__ table_flags) {
    using Cfg = PipeCfg<CPL>;
    constexpr int KE = Cfg::kEdges;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kPipeWarps + warp;
    if (w >= nseg * nchunks) return;  // warps are independent: no block-wide barriers below
    const int mode = widen_mode(table_flags);
    unsigned char* wbase = smem_raw + static_cast<size_t>(warp) * kStages * Cfg::kStageBytes;
    const int32_t chunk = static_cast<int32_t>(w / nseg);
    const int64_t s = seg_base + (w - static_cast<int64_t>(chunk) * nseg);
    const int32_t col = chunk * Cfg::kCols + lane * CPL;
    const bool active = col < dim;
    const int64_t e0 = seg_beg[s], e1 = seg_beg[s + 1];
    const int nblk = static_cast<int>((e1 - e0 + KE - 1) / KE);
    const int rsub = lane / Cfg::kPieces, q = lane % Cfg::kPieces;
    const int32_t colq = chunk * Cfg::kCols + q * 4;  // first float of this lane's 16 B piece
    const bool qok = colq + 4 <= ldx;                 // pieces past the row pitch are zero-filled

    auto issue = [&](int b, int32_t mc, double mf) {
        unsigned char* st = wbase + (b % kStages) * Cfg::kStageBytes;
        float* rows = reinterpret_cast<float*>(st);
        if (lane < KE) reinterpret_cast<double*>(st + kStageDataBytes)[lane] = mf;
#pragma unroll
        for (int i = 0; i < KE / Cfg::kRowsPerIssue; ++i) {
            const int j = i * Cfg::kRowsPerIssue + rsub;
            const int32_t c = __shfl_sync(0xffffffffu, mc, j);
            const bool ok = c >= 0 && qok;
            const float* src = ok ? x + static_cast<int64_t>(c) * ldx + colq : x;
            cp_async16(rows + j * Cfg::kCols + q * 4, src, ok ? 16 : 0);
        }
    };
    auto meta = [&](int b, int32_t& mc, double& mf) {
        const int64_t e = e0 + static_cast<int64_t>(KE) * b + lane;
        const bool ok = lane < KE && e < e1;
        mc = ok ? __ldg(cols + e) : -1;
        mf = ok ? __ldg(coeffs + e) : 0.0;
    };

    int32_t mc;
    double mf;
#pragma unroll
    for (int b = 0; b < kStages; ++b) {
        if (b < nblk) {
            meta(b, mc, mf);
            issue(b, mc, mf);
        }
        cp_async_commit();
    }
    int32_t nc = -1;
    double nf = 0.0;
    if (kStages < nblk) meta(kStages, nc, nf);
    double acc[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
    for (int b = 0; b < nblk; ++b) {
        cp_async_wait<kStages - 1>();
        __syncwarp();
        const unsigned char* st = wbase + (b % kStages) * Cfg::kStageBytes;
        const float* rows = reinterpret_cast<const float*>(st) + lane * CPL;
        const double* cf = reinterpret_cast<const double*>(st + kStageDataBytes);
        const int64_t rem = e1 - e0 - static_cast<int64_t>(KE) * b;
        const int cnt = static_cast<int>(rem < KE ? rem : KE);
        if (active) {
            if (mode == kWidenNonNeg) stage_fma<CPL, kWidenNonNeg>(rows, cf, cnt, acc);
            else if (mode == kWidenSigned) stage_fma<CPL, kWidenSigned>(rows, cf, cnt, acc);
            else stage_fma<CPL, kWidenF2F>(rows, cf, cnt, acc);
        }
        __syncwarp();
        const int bn = b + kStages;
        if (bn < nblk) issue(bn, nc, nf);
        cp_async_commit();
        if (bn + 1 < nblk) meta(bn + 1, nc, nf);
    }
    cp_async_wait<0>();
    const int32_t row = seg_row[s];
    const int32_t slot = seg_slot[s];
    float* yr = y + (static_cast<int64_t>(row) - row_base) * ldy;
    if (slot >= 0) {  // multi-segment row: publish the fp64 partial, last arriving warp combines
        double* pp = partial + static_cast<int64_t>(slot) * pld + col;
#pragma unroll
        for (int k = 0; k < CPL; ++k) pp[k] = acc[k];
        __threadfence();
        __syncwarp();
        int last = 0;
        const int32_t nk = row_nseg[row];
        if (lane == 0) last = atomicAdd(counters + static_cast<int64_t>(row) * cld + chunk, 1) == nk - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) return;
        __threadfence();
        const int32_t s0 = row_seg0[row];
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
        for (int32_t i = 0; i < nk; ++i) {
            const double* q2 = partial + static_cast<int64_t>(seg_slot[s0 + i]) * pld + col;
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[k] += __ldcg(q2 + k);
        }
        if (lane == 0) counters[static_cast<int64_t>(row) * cld + chunk] = 0;  // self-reset
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k)
        if (col + k < dim) yr[col + k] = static_cast<float>(acc[k]);
}

static int g_pipe_smem_set[2] = {};

template <int CPL>
static void launch_pipe(const SpmmSegs& s, const int32_t* cols, const double* coeffs, const float* x, int64_t ldx,
                        int32_t dim, float* y, int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld,
                        int32_t* counters, int32_t counters_ld, cudaStream_t st, const int32_t* special) {
    using Cfg = PipeCfg<CPL>;
    auto kern = spmm_fwd_pipe_kernel<CPL>;
    int& set = g_pipe_smem_set[CPL == 4];
    if (!set) {
        GASB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
        set = 1;
    }
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, Cfg::kCols));
    require(nchunks <= counters_ld && static_cast<int64_t>(nchunks) * Cfg::kCols <= partial_ld,
            "spmm_fwd: counters / partials too narrow");
    const int64_t warps = s.nseg * nchunks;
    kern<<<static_cast<unsigned>(ceil_div(warps, kPipeWarps)), kPipeWarps * 32, Cfg::kSmem, st>>>(
        s.seg_beg, s.seg_row, s.seg_slot, s.row_seg0, s.row_nseg, s.nseg, s.seg_base, cols, coeffs, x, ldx, dim,
        nchunks, y, ldy, row_base, partial, partial_ld, counters, counters_ld, special);
}

// Columns per lane of the pipelined SpMM (tuning knob GASB_SPMM_CPL = 2 | 4, default 4:
// 128-column chunks, measured fastest on the Reddit-shaped workload).
static int spmm_cpl() {
    static int v = [] {
        const char* e = getenv("GASB_SPMM_CPL");
        return e && atoi(e) == 2 ? 2 : 4;
    }();
    return v;
}

// flags[0] |= kTableNeg / kTableNonFinite for the values of x[rows x dim] (pitch ld).
__global__ void scan_special_kernel(const float* __restrict__ x, int64_t rows, int64_t ld, int32_t dim,
                                    int32_t* __restrict__ special) {
    int found = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * dim;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        found |= table_flag_of(x[(i / dim) * ld + (i % dim)]);
    found = __reduce_or_sync(0xffffffffu, found);
    if ((threadIdx.x & 31) == 0 && found) atomicOr(special, found);
}

void launch_scan_special(const float* x, int64_t rows, int64_t ld, int32_t dim, int32_t* special, cudaStream_t st) {
    if (rows <= 0 || dim <= 0) return;
    scan_special_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(rows * dim, 256), 2048)), 256, 0, st>>>(
        x, rows, ld, dim, special);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_spmm_fwd(const SpmmSegs& s, const int32_t* cols, const double* coeffs, const float* x, int64_t ldx,
                     int32_t dim, float* y, int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld,
                     int32_t* counters, int32_t counters_ld, cudaStream_t st, const int32_t* special) {
    if (s.nseg <= 0 || dim <= 0) return;
    require(ldx % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0,
            "spmm_fwd: source rows must be 16 B aligned (ldx % 4 == 0)");
    if (spmm_cpl() == 2)
        launch_pipe<2>(s, cols, coeffs, x, ldx, dim, y, ldy, row_base, partial, partial_ld, counters, counters_ld, st,
                       special);
    else
        launch_pipe<4>(s, cols, coeffs, x, ldx, dim, y, ldy, row_base, partial, partial_ld, counters, counters_ld, st,
                       special);
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

// Shared-memory staged variant: the gathered rows gy[0..nsrc) are few (one batch), so a CTA
// stages the 32-column slice gy[:, chunk] (nsrc x 128 B) in smem once and every target of
// its range gathers from smem; lane = column, entries in order -> same rounding sequence.
constexpr int kBwdCW = 32;
constexpr int kBwdThreads = 512;

__global__ void __launch_bounds__(kBwdThreads) spmm_bwd_smem_kernel(
    const int64_t* __restrict__ rp, int32_t nt, const int32_t* __restrict__ src, const float* __restrict__ cf,
    const float* __restrict__ gy, int64_t ldgy, int32_t nsrc, int32_t dim, const float* __restrict__ mask,
    int64_t ldm, float* __restrict__ gx, int64_t ldgx, int32_t targets_per_cta) {
    extern __shared__ float sg[];  // nsrc x kBwdCW
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int32_t col0 = blockIdx.x * kBwdCW;
    const int32_t ncol = min(kBwdCW, dim - col0);
    // stage gy[:, col0 : col0+ncol] (zero-padded to 32 columns)
    {  // 8 lanes x float4 per 128 B row slice, 8 rows in flight per thread
        const int c4 = (threadIdx.x & 7) * 4;
        const bool vec = (ldgy % 4 == 0) && ((reinterpret_cast<uintptr_t>(gy) & 15) == 0);
        for (int64_t r0 = threadIdx.x >> 3; r0 < nsrc; r0 += 8 * (blockDim.x >> 3)) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t r = r0 + static_cast<int64_t>(u) * (blockDim.x >> 3);
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (r < nsrc) {
                    const float* p = gy + r * ldgy + col0 + c4;
                    if (vec && c4 + 4 <= ncol) v[u] = __ldg(reinterpret_cast<const float4*>(p));
                    else {
                        if (c4 + 0 < ncol) v[u].x = __ldg(p + 0);
                        if (c4 + 1 < ncol) v[u].y = __ldg(p + 1);
                        if (c4 + 2 < ncol) v[u].z = __ldg(p + 2);
                        if (c4 + 3 < ncol) v[u].w = __ldg(p + 3);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t r = r0 + static_cast<int64_t>(u) * (blockDim.x >> 3);
                if (r < nsrc) *reinterpret_cast<float4*>(sg + r * kBwdCW + c4) = v[u];
            }
        }
    }
    __syncthreads();
    const int32_t t_lo = blockIdx.y * targets_per_cta;
    const int32_t t_hi = min(nt, t_lo + targets_per_cta);
    for (int32_t t = t_lo + warp; t < t_hi; t += nwarps) {
        const int64_t e0 = rp[t], e1 = rp[t + 1];
        float a = 0.0f;
        for (int64_t eb = e0; eb < e1; eb += 32) {
            const int cnt = static_cast<int>((e1 - eb) < 32 ? (e1 - eb) : 32);
            const int32_t my_r = lane < cnt ? __ldg(src + eb + lane) : 0;
            const float my_c = lane < cnt ? __ldg(cf + eb + lane) : 0.0f;
#pragma unroll 8
            for (int j = 0; j < cnt; ++j) {
                const int32_t r = __shfl_sync(0xffffffffu, my_r, j);
                const float c = __shfl_sync(0xffffffffu, my_c, j);
                a = __fadd_rn(a, __fmul_rn(c, sg[r * kBwdCW + lane]));
            }
        }
        if (lane < ncol) {
            const int32_t col = col0 + lane;
            if (mask && !(mask[static_cast<int64_t>(t) * ldm + col] > 0.0f)) a = 0.0f;
            gx[static_cast<int64_t>(t) * ldgx + col] = a;
        }
    }
}

static int g_bwd_smem_set = 0;

void launch_spmm_bwd(const int64_t* t_rowptr, int32_t nt, const int32_t* t_src, const float* t_coeffs,
                     const float* gy, int64_t ldgy, int32_t dim, const float* mask, int64_t ldm, float* gx,
                     int64_t ldgx, cudaStream_t st, int32_t nsrc) {
    if (nt <= 0 || dim <= 0) return;
    const int64_t smem = static_cast<int64_t>(nsrc) * kBwdCW * sizeof(float);
    if (nsrc > 0 && smem <= 200 * 1024) {
        if (!g_bwd_smem_set) {
            GASB_CUDA(cudaFuncSetAttribute(spmm_bwd_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           200 * 1024));
            g_bwd_smem_set = 1;
        }
        const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kBwdCW));
        // ~148 CTAs in total, at least one warp-round of targets each
        const int32_t splits = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(148, nchunks),
                                                                                        ceil_div(nt, 16))));
        const int32_t per = static_cast<int32_t>(ceil_div(nt, splits));
        dim3 grid(static_cast<unsigned>(nchunks), static_cast<unsigned>(ceil_div(nt, per)));
        spmm_bwd_smem_kernel<<<grid, kBwdThreads, smem, st>>>(t_rowptr, nt, t_src, t_coeffs, gy, ldgy, nsrc, dim,
                                                             mask, ldm, gx, ldgx, per);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return;
    }
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
                                     const float* d_x, int32_t num_src, int64_t ldx, int32_t dim, float* d_y,
                                     int64_t ldy, int32_t seg_edges, gasb_stream stream) {
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
        GASB_CUDA(cudaMallocAsync(&z.partial, sizeof(double) * std::max<int64_t>(slots, 1) * round_up(dim, 128), st));
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
            for (int64_t e = 0; e < nnz; ++e) {  // scaled by 2^896: exact while |c| < 2^127
                require(std::fabs(cf[e]) < 0x1.0p+126f, "aggregate: |coefficient| must be < 2^126");
                cd[e] = static_cast<double>(cf[e]) * kCoeffScale;
            }
            GASB_CUDA(cudaMemcpyAsync(coeffs64, cd.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
            int32_t* special = nullptr;
            GASB_CUDA(cudaMallocAsync(&special, sizeof(int32_t), st));
            GASB_CUDA(cudaMemsetAsync(special, 0, sizeof(int32_t), st));
            launch_scan_special(d_x, num_src, ldx, dim, special, st);
            SpmmSegs segs{z.seg_beg, z.seg_row, z.seg_slot, z.row_seg0, z.row_nseg, nseg, 0};
            launch_spmm_fwd(segs, d_cols, coeffs64, d_x, ldx, dim, d_y, ldy, 0, z.partial,
                            round_up(dim, 128), z.counters, nchunks, st, special);
            GASB_CUDA(cudaStreamSynchronize(st));
            cudaFreeAsync(special, st);
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
                                     const float* d_t_coeffs, const float* d_gy, int64_t ldgy, int32_t num_src,
                                     int32_t dim, const float* d_mask, int64_t ldm, float* d_gx, int64_t ldgx,
                                     gasb_stream stream) {
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
        launch_spmm_bwd(rp64, nt, d_t_src, d_t_coeffs, d_gy, ldgy, dim, d_mask, ldm, d_gx, ldgx, st, num_src);
        cudaFreeAsync(rp64, st);
        GASB_CUDA(cudaStreamSynchronize(st));
    });
}
