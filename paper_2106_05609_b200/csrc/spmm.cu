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
#include <algorithm>
#include <cstring>

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
//   signed x       : hi = ((u & 0x7fffffff) >> 3) | (u & sign), lo = u << 29   (IMAD.WIDE + LOP3)
// so fma(c * 2^896, D, acc) == acc + c*x rounded once — the reference's `acc += c * src`.
// A per-table flag word (kTableNeg / kTableNonFinite) selects the path; tables holding
// inf/nan take F2F (D = double(x) * 2^-896, also exact).
#ifndef GASB_SPMM_STAGES
#define GASB_SPMM_STAGES 2
#endif
#ifndef GASB_SPMM_STAGE_BYTES
#define GASB_SPMM_STAGE_BYTES 8192
#endif
#ifndef GASB_SPMM_CTAS
#define GASB_SPMM_CTAS 3
#endif
constexpr int kStages = GASB_SPMM_STAGES;      // stages in flight per warp
constexpr int kPipeCtas = GASB_SPMM_CTAS;      // resident CTAs per SM (persistent grid)
#ifndef GASB_SPMM_WARPS
#define GASB_SPMM_WARPS 4
#endif
constexpr int kPipeWarps = GASB_SPMM_WARPS;    // warps per CTA
constexpr int kStageDataBytes = GASB_SPMM_STAGE_BYTES;

enum WidenMode { kWidenF2F = 0, kWidenSigned = 1, kWidenNonNeg = 2 };

// The bit pattern {hi = u >> 3, lo = u << 29} is the 64-bit product u * 2^29: one
// IMAD.WIDE.U32. Signed tables use the signed product and one LOP3 (widen_scaled).
__device__ __forceinline__ uint64_t mul_wide_2p29(uint32_t u) {
    uint64_t d;
    asm("mul.wide.u32 %0, %1, 536870912;" : "=l"(d) : "r"(u));
    return d;
}

template <int MODE>
__device__ __forceinline__ double widen_scaled(float f) {
    const uint32_t u = __float_as_uint(f);
    if (MODE == kWidenNonNeg) return __longlong_as_double(static_cast<long long>(mul_wide_2p29(u)));
    if (MODE == kWidenSigned) {
        // signed product u * 2^29 (u read as int32): for a negative x the sign extension sets
        // hi bits 28..31; clearing bits 28..30 leaves the sign at bit 31 and the exponent
        // field untouched. IMAD.WIDE + LOP3.
        long long d;
        asm("mul.wide.s32 %0, %1, 536870912;" : "=l"(d) : "r"(u));
        const uint32_t hi = static_cast<uint32_t>(static_cast<unsigned long long>(d) >> 32) & 0x8FFFFFFFu;
        return __hiloint2double(static_cast<int>(hi), static_cast<int>(static_cast<uint32_t>(d)));
    }
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
__device__ __forceinline__ void cp_async_ca4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_ca8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
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
    static constexpr int kHdrBytes = 16;                          // stage descriptor
    // 128 B aligned: TMA destinations must be 128 B aligned
    // data | fp64 coeffs | header | int32 source rows (TMA gather coordinates)
    static constexpr int kStageBytes = (kStageDataBytes + kEdges * 8 + kHdrBytes + kEdges * 4 + 127) / 128 * 128;
    static constexpr int kSmem = kPipeWarps * kStages * kStageBytes;
};
// TMA mode: per-warp ring of kMetaWin windows of 32 edges (int32 col + fp64 coeff each),
// prefetched with cp.async kMetaWin windows ahead of the gather issue, so the row indices a
// tile::gather4 needs are in shared memory (not a dependent global load) when it is issued.
constexpr int kMetaWin = 4;
constexpr int kMetaRingBytes = kMetaWin * 32 * (4 + 8);

// Stage descriptor (shared memory): edges of ONE segment, so the FMA loop needs no
// boundary tests; `ends` marks the segment's last stage (then it is finalized).
struct StageHdr {
    int32_t cnt, ends, row, slot;
};

// All KE edges of a stage (predicated on j < cnt, warp-uniform), CSR order, CPL fp64
// accumulators per lane.
template <int CPL, int MODE>
__device__ __forceinline__ void edge_fma(const float* rows, const double* cf, int j, double (&acc)[CPL]) {
    constexpr int kCols = 32 * CPL;
    const double c = cf[j];
    if constexpr (CPL == 8) {  // lane owns columns [4 lane, +4) and [128 + 4 lane, +4): conflict-free LDS.128
        const float4 v = *reinterpret_cast<const float4*>(rows + j * kCols);
        const float4 w = *reinterpret_cast<const float4*>(rows + j * kCols + 128);
        acc[0] = __fma_rn(c, widen_scaled<MODE>(v.x), acc[0]);
        acc[1] = __fma_rn(c, widen_scaled<MODE>(v.y), acc[1]);
        acc[2] = __fma_rn(c, widen_scaled<MODE>(v.z), acc[2]);
        acc[3] = __fma_rn(c, widen_scaled<MODE>(v.w), acc[3]);
        acc[4] = __fma_rn(c, widen_scaled<MODE>(w.x), acc[4]);
        acc[5] = __fma_rn(c, widen_scaled<MODE>(w.y), acc[5]);
        acc[6] = __fma_rn(c, widen_scaled<MODE>(w.z), acc[6]);
        acc[7] = __fma_rn(c, widen_scaled<MODE>(w.w), acc[7]);
    } else if constexpr (CPL == 4) {
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

template <int CPL, int MODE, int KE>
__device__ __forceinline__ void stage_fma(const float* rows, const double* cf, int cnt, double (&acc)[CPL]) {
    if (cnt == KE) {  // full stage (the common case): straight-line code, loads hoisted freely
#pragma unroll
        for (int j = 0; j < KE; ++j) edge_fma<CPL, MODE>(rows, cf, j, acc);
    } else {
#pragma unroll 4
        for (int j = 0; j < cnt; ++j) edge_fma<CPL, MODE>(rows, cf, j, acc);
    }
}

// Persistent streaming SpMM. The launch's segments are pre-split (host) into `nranges`
// contiguous ranges of ~equal edge count (range_seg[r] .. range_seg[r+1]); work item =
// (chunk, range), chunk-major, handed to warps grid-stride. A warp streams its range as a
// sequence of stages of <= KE edges of a single segment through the cp.async pipeline
// (kStages deep, no drain at row boundaries); after a segment's last stage it stores the
// row, or publishes an fp64 partial and the last-arriving warp of the row combines the
// partials in segment order. coeffs are pre-scaled by 2^896 (see widen_scaled).
// ---- TMA (tile::gather4) + mbarrier helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// Bounded wait: a barrier that never completes traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    for (uint32_t spins = 0;; ++spins) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (spins > (1u << 26)) __trap();
    }
}
// 4 rows x box-width columns of a 2-D row-major table -> shared memory (rows contiguous);
// out-of-range rows / columns are zero-filled; completes `bytes` on the mbarrier.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int32_t c0, int32_t r0, int32_t r1,
                                            int32_t r2, int32_t r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

template <int CPL, bool TMA>
__global__ void __launch_bounds__(kPipeWarps * 32, kPipeCtas) spmm_fwd_pipe_kernel(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, const int32_t* __restrict__ range_seg,
    int32_t nranges, const int32_t* __restrict__ cols, const double* __restrict__ coeffs, const float* __restrict__ x,
    int64_t ldx, int32_t dim, int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base,
    double* __restrict__ partial, int64_t pld, int32_t* __restrict__ counters, int32_t cld,
    const int32_t* __restrict__ table_flags, const __grid_constant__ CUtensorMap tmap) {
    using Cfg = PipeCfg<CPL>;
    constexpr int KE = Cfg::kEdges;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kPipeWarps;
    const int mode = widen_mode(table_flags);
    unsigned char* wbase = smem_raw + static_cast<size_t>(warp) * kStages * Cfg::kStageBytes;
    const int rsub = lane / Cfg::kPieces, q = lane % Cfg::kPieces;
    // TMA: one mbarrier per stage slot (after all stage buffers), phase bit per slot
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kPipeWarps * kStages * Cfg::kStageBytes) + warp * kStages;
    unsigned char* ring = smem_raw + kPipeWarps * kStages * Cfg::kStageBytes + kPipeWarps * kStages * 8 +
                          warp * kMetaRingBytes;
    int32_t* ring_c = reinterpret_cast<int32_t*>(ring);
    double* ring_f = reinterpret_cast<double*>(ring + kMetaWin * 32 * 4);
    uint32_t phases = 0;
    if constexpr (TMA) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
            for (int k = 0; k < kStages; ++k) mbar_init(bars + k, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncwarp();
    }
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * kPipeWarps + warp;
         item < static_cast<int64_t>(nchunks) * nranges; item += nwarps) {
        const int32_t chunk = static_cast<int32_t>(item / nranges);
        const int32_t r = static_cast<int32_t>(item - static_cast<int64_t>(chunk) * nranges);
        const int32_t s_lo = range_seg[r], s_hi = range_seg[r + 1];
        if (s_lo >= s_hi) continue;
        const int32_t col = chunk * Cfg::kCols + lane * CPL;
        const int32_t colq = chunk * Cfg::kCols + q * 4;  // first float of this lane's 16 B piece
        const bool qok = colq + 4 <= ldx;                 // pieces past the row pitch are zero-filled

        // ---- issue-side cursor over the range's segments (window of 32 segment records)
        int32_t iseg = s_lo, wbase_seg = s_lo, w_row = 0, w_slot = -1;
        int64_t ipos = seg_beg[s_lo], w_end = 0;
        auto load_window = [&](int32_t from) {
            wbase_seg = from;
            const int32_t sg = from + lane;
            w_end = sg < s_hi ? seg_beg[sg + 1] : 0;
            w_row = sg < s_hi ? seg_row[sg] : 0;
            w_slot = sg < s_hi ? seg_slot[sg] : -1;
        };
        load_window(s_lo);
        // ---- edge-metadata ring (TMA mode): window q = edges [e_lo + 32q, +32) in slot q % kMetaWin
        const int64_t e_lo = seg_beg[s_lo], e_hi = seg_beg[s_hi];
        int w_issued = 0;
        auto prefetch_win = [&] {
            const int slot = w_issued % kMetaWin;
            const int64_t e = e_lo + 32LL * w_issued + lane;
            if (e < e_hi) {
                cp_async_ca4(ring_c + slot * 32 + lane, cols + e);
                cp_async_ca8(ring_f + slot * 32 + lane, coeffs + e);
            }
            cp_async_commit();
            ++w_issued;
        };
        // make the windows holding edges [e_first, e_first + c) resident; recycle older slots
        auto ensure_meta = [&](int64_t e_first, int c) {
            const int q0 = static_cast<int>((e_first - e_lo) >> 5);
            const int q1 = static_cast<int>((e_first + c - 1 - e_lo) >> 5);
            while (w_issued < q0 + kMetaWin && e_lo + 32LL * w_issued < e_hi) prefetch_win();
            const int allowed = w_issued - (q1 + 1);  // cp.async groups that may stay in flight
            if (allowed >= 3) cp_async_wait<3>();
            else if (allowed == 2) cp_async_wait<2>();
            else if (allowed == 1) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncwarp();
        };
        if constexpr (TMA) {
#pragma unroll
            for (int k = 0; k < kMetaWin; ++k)
                if (e_lo + 32LL * w_issued < e_hi) prefetch_win();
        }
        // describe the next stage (edges [ipos, ipos + cnt) of segment iseg) and advance
        auto next_stage = [&](StageHdr& h, int64_t& e_first) -> bool {
            if (iseg >= s_hi) return false;
            if (iseg - wbase_seg >= 32) load_window(iseg);
            const int k = iseg - wbase_seg;
            const int64_t end = __shfl_sync(0xffffffffu, w_end, k);
            const int64_t c = end - ipos < KE ? end - ipos : KE;
            h.cnt = static_cast<int32_t>(c);
            h.ends = ipos + c == end;
            h.row = __shfl_sync(0xffffffffu, w_row, k);
            h.slot = __shfl_sync(0xffffffffu, w_slot, k);
            e_first = ipos;
            ipos += c;
            if (h.ends) ++iseg;
            return true;
        };
        auto meta = [&](const StageHdr& h, int64_t e_first, int32_t& mc, double& mf) {
            const bool ok = lane < h.cnt;
            if constexpr (TMA) {
                if (h.cnt > 0) ensure_meta(e_first, h.cnt);
                const int64_t o = e_first - e_lo + lane;
                const int idx = static_cast<int>(((o >> 5) % kMetaWin) * 32 + (o & 31));
                mc = ok ? ring_c[idx] : -1;
                mf = ok ? ring_f[idx] : 0.0;
            } else {
                mc = ok ? __ldg(cols + e_first + lane) : -1;
                mf = ok ? __ldg(coeffs + e_first + lane) : 0.0;
            }
        };
        auto issue = [&](int slot_idx, const StageHdr& h, int32_t mc, double mf) {
            unsigned char* st = wbase + slot_idx * Cfg::kStageBytes;
            float* rows = reinterpret_cast<float*>(st);
            if (lane < KE) reinterpret_cast<double*>(st + kStageDataBytes)[lane] = mf;
            if (lane == 0) *reinterpret_cast<StageHdr*>(st + kStageDataBytes + KE * 8) = h;
            if constexpr (TMA) {
                // rows of stage i go to rows + i*kCols; unused slots (mc = -1) are zero-filled.
                // The warp parks the stage's source rows in shared memory; lane 0 reads them
                // back four at a time (one LDS.128 per gather4, no shuffles).
                int32_t* srow = reinterpret_cast<int32_t*>(st + kStageDataBytes + KE * 8 + Cfg::kHdrBytes);
                if (lane < KE) srow[lane] = mc;
                __syncwarp();
                if (lane == 0) {
                    const int ng = (h.cnt + 3) >> 2;
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // after the warp's reads
                    mbar_expect_tx(bars + slot_idx, static_cast<uint32_t>(ng) * 4u * Cfg::kCols * 4u);
                    const int32_t c0 = chunk * Cfg::kCols;
                    for (int i = 0; i < ng; ++i) {
                        const int4 r = reinterpret_cast<const int4*>(srow)[i];
                        tma_gather4(rows + 4 * i * Cfg::kCols, &tmap, c0, r.x, r.y, r.z, r.w, bars + slot_idx);
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < KE / Cfg::kRowsPerIssue; ++i) {
                    const int j = i * Cfg::kRowsPerIssue + rsub;
                    if (i * Cfg::kRowsPerIssue < h.cnt) {  // warp-uniform
                        const int32_t c = __shfl_sync(0xffffffffu, mc, j);
                        const bool ok = c >= 0 && qok;
                        const float* src = ok ? x + static_cast<int64_t>(c) * ldx + colq : x;
                        cp_async16(rows + j * Cfg::kCols + q * 4, src, ok ? 16 : 0);
                    }
                }
            }
        };

        // ---- prologue: up to kStages stages in flight, metadata of the next one prefetched
        int issued = 0;
        StageHdr nh;
        int64_t ne_first = 0;
        int32_t nmc = -1;
        double nmf = 0.0;
        bool have_next = next_stage(nh, ne_first);
        if (have_next) meta(nh, ne_first, nmc, nmf);
#pragma unroll
        for (int k = 0; k < kStages; ++k) {
            if (have_next) {
                issue(k, nh, nmc, nmf);
                ++issued;
                have_next = next_stage(nh, ne_first);
                if (have_next) meta(nh, ne_first, nmc, nmf);
            }
            if constexpr (!TMA) cp_async_commit();
        }
        double acc[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
        for (int b = 0; b < issued; ++b) {
            if constexpr (TMA) {
                const int sl = b % kStages;
                mbar_wait(bars + sl, (phases >> sl) & 1u);
                phases ^= 1u << sl;
            } else {
                cp_async_wait<kStages - 1>();
            }
            __syncwarp();
            const unsigned char* st = wbase + (b % kStages) * Cfg::kStageBytes;
            const float* rows = reinterpret_cast<const float*>(st) + lane * CPL;
            const double* cf = reinterpret_cast<const double*>(st + kStageDataBytes);
            const StageHdr h = *reinterpret_cast<const StageHdr*>(st + kStageDataBytes + KE * 8);
            if (mode == kWidenNonNeg) stage_fma<CPL, kWidenNonNeg, KE>(rows, cf, h.cnt, acc);
            else if (mode == kWidenSigned) stage_fma<CPL, kWidenSigned, KE>(rows, cf, h.cnt, acc);
            else stage_fma<CPL, kWidenF2F, KE>(rows, cf, h.cnt, acc);
            __syncwarp();
            if (have_next) {  // refill the slot just consumed
                issue(b % kStages, nh, nmc, nmf);
                ++issued;
                have_next = next_stage(nh, ne_first);
                if (have_next) meta(nh, ne_first, nmc, nmf);
            }
            if constexpr (!TMA) cp_async_commit();
            if (h.ends) {  // end of segment: store the row, or publish the partial and combine
                float* yr = y + (static_cast<int64_t>(h.row) - row_base) * ldy;
                bool store = true;
                if (h.slot >= 0) {
                    double* pp = partial + static_cast<int64_t>(h.slot) * pld + col;
#pragma unroll
                    for (int k = 0; k < CPL; ++k) pp[k] = acc[k];
                    __threadfence();
                    __syncwarp();
                    int last = 0;
                    const int32_t nk = row_nseg[h.row];
                    if (lane == 0)
                        last = atomicAdd(counters + static_cast<int64_t>(h.row) * cld + chunk, 1) == nk - 1;
                    store = __shfl_sync(0xffffffffu, last, 0) != 0;
                    if (store) {
                        __threadfence();
                        const int32_t s0 = row_seg0[h.row];
#pragma unroll
                        for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
                        for (int32_t i = 0; i < nk; ++i) {
                            const double* q2 = partial + static_cast<int64_t>(seg_slot[s0 + i]) * pld + col;
#pragma unroll
                            for (int k = 0; k < CPL; ++k) acc[k] += __ldcg(q2 + k);
                        }
                        if (lane == 0) counters[static_cast<int64_t>(h.row) * cld + chunk] = 0;  // self-reset
                    }
                }
                if (store) {
#pragma unroll
                    for (int k = 0; k < CPL; ++k)
                        if (col + k < dim) yr[col + k] = static_cast<float>(acc[k]);
                }
#pragma unroll
                for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
            }
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

// ---- direct-load forward (no shared-memory staging) ------------------------------------
// Same work decomposition, segment tables and fp64 partial protocol as the pipelined
// kernel, but each lane gathers its 16 B piece of every source row straight into
// registers (LDG.128, L1 no-allocate): KD independent row loads in flight per warp, no
// stage bookkeeping, and the edge stream runs across segment (row) boundaries without
// draining. Small register footprint -> 16 warps per SM hide the L2/HBM latency.
constexpr int kDirectKD = 8;      // row loads in flight per warp
constexpr int kDirectWarps = 8;   // warps per CTA (2 CTAs per SM)

__device__ __forceinline__ float4 ldg_row_piece(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// Column of accumulator k of a lane whose first column is `col` (CPL = 8: two 4-column
// groups 128 apart, see edge_fma).
template <int CPL>
__device__ __forceinline__ int32_t col_of(int32_t col, int k) {
    return CPL == 8 ? col + (k & 3) + ((k >> 2) << 7) : col + k;
}

// Optional row-sum hand-off between two launches over the same rows (cross-batch mode):
// out != nullptr: a finished row's fp64 sum goes to out[row - row_base] (ld doubles per row)
// instead of y; in != nullptr: the stored fp32 row is float(sum + in[row - row_base]).
struct RowSums {
    double* out = nullptr;
    const double* in = nullptr;
    int64_t ld = 0;
};

// Ends segment `k` of the warp's window: store the row (single-segment row) or publish an
// fp64 partial, the last-arriving warp of the row summing the partials in segment order.
template <int CPL>
__device__ __forceinline__ void seg_finish(double (&acc)[CPL], int32_t row, int32_t slot, int lane, int32_t col,
                                           int32_t chunk, int32_t dim, float* __restrict__ y, int64_t ldy,
                                           int64_t row_base, double* __restrict__ partial, int64_t pld,
                                           int32_t* __restrict__ counters, int32_t cld,
                                           const int32_t* __restrict__ seg_slot,
                                           const int32_t* __restrict__ row_seg0,
                                           const int32_t* __restrict__ row_nseg, const RowSums& rs = RowSums{}) {
    bool store = true;
    if (slot >= 0) {
        double* pp = partial + static_cast<int64_t>(slot) * pld;
#pragma unroll
        for (int k = 0; k < CPL; ++k) pp[col_of<CPL>(col, k)] = acc[k];
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // publish the partial before arriving
        __syncwarp();
        int last = 0;
        const int32_t nk = row_nseg[row];
        if (lane == 0) last = atomicAdd(counters + static_cast<int64_t>(row) * cld + chunk, 1) == nk - 1;
        store = __shfl_sync(0xffffffffu, last, 0) != 0;
        if (store) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // see every peer's published partial
            const int32_t s0 = row_seg0[row];
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
            for (int32_t i = 0; i < nk; ++i) {
                const double* q2 = partial + static_cast<int64_t>(seg_slot[s0 + i]) * pld;
#pragma unroll
                for (int k = 0; k < CPL; ++k) acc[k] += __ldcg(q2 + col_of<CPL>(col, k));
            }
            if (lane == 0) counters[static_cast<int64_t>(row) * cld + chunk] = 0;  // self-reset
        }
    }
    if (store) {
        if (rs.out) {  // the row's fp64 sum for a later launch (no fp32 row)
            double* o = rs.out + (static_cast<int64_t>(row) - row_base) * rs.ld;
#pragma unroll
            for (int k = 0; k < CPL; ++k)
                if (col_of<CPL>(col, k) < dim) o[col_of<CPL>(col, k)] = acc[k];
        } else {
            float* yr = y + (static_cast<int64_t>(row) - row_base) * ldy;
            const double* si = rs.in ? rs.in + (static_cast<int64_t>(row) - row_base) * rs.ld : nullptr;
#pragma unroll
            for (int k = 0; k < CPL; ++k)
                if (col_of<CPL>(col, k) < dim)
                    yr[col_of<CPL>(col, k)] =
                        static_cast<float>(si ? __dadd_rn(acc[k], __ldcg(si + col_of<CPL>(col, k))) : acc[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
}

__device__ __forceinline__ void direct_finish(double a0, double a1, double a2, double a3, int32_t row, int32_t slot, int lane, int32_t col,
                                              int32_t chunk, int32_t dim, float* __restrict__ y, int64_t ldy,
                                              int64_t row_base, double* __restrict__ partial, int64_t pld,
                                              int32_t* __restrict__ counters, int32_t cld,
                                              const int32_t* __restrict__ seg_slot,
                                              const int32_t* __restrict__ row_seg0,
                                              const int32_t* __restrict__ row_nseg) {
    double acc[4] = {a0, a1, a2, a3};
    bool store = true;
    if (slot >= 0) {
        double* pp = partial + static_cast<int64_t>(slot) * pld + col;
#pragma unroll
        for (int k = 0; k < 4; ++k) pp[k] = acc[k];
        __threadfence();
        __syncwarp();
        int last = 0;
        const int32_t nk = row_nseg[row];
        if (lane == 0) last = atomicAdd(counters + static_cast<int64_t>(row) * cld + chunk, 1) == nk - 1;
        store = __shfl_sync(0xffffffffu, last, 0) != 0;
        if (store) {
            __threadfence();
            const int32_t s0 = row_seg0[row];
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = 0.0;
            for (int32_t i = 0; i < nk; ++i) {
                const double* q2 = partial + static_cast<int64_t>(seg_slot[s0 + i]) * pld + col;
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[k] += __ldcg(q2 + k);
            }
            if (lane == 0) counters[static_cast<int64_t>(row) * cld + chunk] = 0;  // self-reset
        }
    }
    if (store) {
        float* yr = y + (static_cast<int64_t>(row) - row_base) * ldy;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (col + k < dim) yr[col + k] = static_cast<float>(acc[k]);
    }
}

template <int MODE>
__device__ __forceinline__ void direct_items(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, const int32_t* __restrict__ range_seg,
    int32_t nranges, const int32_t* __restrict__ cols, const double* __restrict__ coeffs, const float* __restrict__ x,
    int64_t ldx, int32_t dim, int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base,
    double* __restrict__ partial, int64_t pld, int32_t* __restrict__ counters, int32_t cld) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         item < static_cast<int64_t>(nchunks) * nranges; item += nwarps) {
        const int32_t chunk = static_cast<int32_t>(item / nranges);
        const int32_t r = static_cast<int32_t>(item - static_cast<int64_t>(chunk) * nranges);
        const int32_t s_lo = range_seg[r], s_hi = range_seg[r + 1];
        if (s_lo >= s_hi) continue;
        const int32_t col = chunk * 128 + lane * 4;
        const bool colok = col < dim;  // col % 4 == 0 and ldx % 4 == 0: the whole piece is inside the pitch
        const float* xc = x + (colok ? col : 0);
        // window of 32 segment records (end offset, row, slot), lane k holds segment wseg + k
        int32_t wseg = s_lo, cur = s_lo;
        int64_t w_end = 0;
        int32_t w_row = 0, w_slot = -1;
        auto load_window = [&](int32_t from) {
            wseg = from;
            const int32_t sg = from + lane;
            w_end = sg < s_hi ? seg_beg[sg + 1] : 0;
            w_row = sg < s_hi ? seg_row[sg] : 0;
            w_slot = sg < s_hi ? seg_slot[sg] : -1;
        };
        load_window(s_lo);
        int64_t cur_end = __shfl_sync(0xffffffffu, w_end, 0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        auto finish = [&] {
            const int k = cur - wseg;
            const int32_t row = __shfl_sync(0xffffffffu, w_row, k);
            const int32_t slot = __shfl_sync(0xffffffffu, w_slot, k);
            direct_finish(acc[0], acc[1], acc[2], acc[3], row, slot, lane, col, chunk, dim, y, ldy, row_base, partial, pld, counters, cld,
                          seg_slot, row_seg0, row_nseg);
            acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
            ++cur;
            if (cur < s_hi) {
                if (cur - wseg >= 32) load_window(cur);
                cur_end = __shfl_sync(0xffffffffu, w_end, cur - wseg);
            }
        };
        const int64_t E_lo = seg_beg[s_lo], E_hi = seg_beg[s_hi];
        for (int64_t e = E_lo; e < E_hi; e += 32) {
            const int n = static_cast<int>(E_hi - e < 32 ? E_hi - e : 32);
            const int32_t mc = lane < n ? __ldg(cols + e + lane) : 0;
            const double mf = lane < n ? __ldg(coeffs + e + lane) : 0.0;
            for (int j = 0; j < n; j += kDirectKD) {
                float4 v[kDirectKD];
#pragma unroll
                for (int k = 0; k < kDirectKD; ++k) {
                    const int32_t c = __shfl_sync(0xffffffffu, mc, j + k);
                    v[k] = (j + k < n && colok) ? ldg_row_piece(xc + static_cast<int64_t>(c) * ldx)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int k = 0; k < kDirectKD; ++k) {
                    const double f = __shfl_sync(0xffffffffu, mf, j + k);
                    if (j + k < n) {  // warp-uniform
                        while (e + j + k == cur_end && cur < s_hi) finish();
                        acc[0] = __fma_rn(f, widen_scaled<MODE>(v[k].x), acc[0]);
                        acc[1] = __fma_rn(f, widen_scaled<MODE>(v[k].y), acc[1]);
                        acc[2] = __fma_rn(f, widen_scaled<MODE>(v[k].z), acc[2]);
                        acc[3] = __fma_rn(f, widen_scaled<MODE>(v[k].w), acc[3]);
                    }
                }
            }
        }
        while (cur < s_hi) finish();  // the last segment (and any empty trailing ones)
    }
}

__global__ void __launch_bounds__(kDirectWarps * 32, 2) spmm_fwd_direct_kernel(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, const int32_t* __restrict__ range_seg,
    int32_t nranges, const int32_t* __restrict__ cols, const double* __restrict__ coeffs, const float* __restrict__ x,
    int64_t ldx, int32_t dim, int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base,
    double* __restrict__ partial, int64_t pld, int32_t* __restrict__ counters, int32_t cld,
    const int32_t* __restrict__ table_flags) {
    const int mode = widen_mode(table_flags);
#define GASB_DIRECT(M)                                                                                           \
    direct_items<M>(seg_beg, seg_row, seg_slot, row_seg0, row_nseg, range_seg, nranges, cols, coeffs, x, ldx, dim, \
                    nchunks, y, ldy, row_base, partial, pld, counters, cld)
    if (mode == kWidenNonNeg) GASB_DIRECT(kWidenNonNeg);
    else if (mode == kWidenSigned) GASB_DIRECT(kWidenSigned);
    else GASB_DIRECT(kWidenF2F);
#undef GASB_DIRECT
}

static void launch_direct(const SpmmSegs& s, const int32_t* cols, const double* coeffs, const float* x, int64_t ldx,
                          int32_t dim, float* y, int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld,
                          int32_t* counters, int32_t counters_ld, cudaStream_t st, const int32_t* special) {
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, 128));
    require(nchunks <= counters_ld && static_cast<int64_t>(nchunks) * 128 <= partial_ld,
            "spmm_fwd: counters / partials too narrow");
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        GASB_CUDA(cudaGetDevice(&dev));
        GASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int64_t items = static_cast<int64_t>(nchunks) * s.nranges;
    const int64_t blocks = std::min<int64_t>(ceil_div(items, kDirectWarps), 2LL * sms);
    spmm_fwd_direct_kernel<<<static_cast<unsigned>(blocks), kDirectWarps * 32, 0, st>>>(
        s.seg_beg, s.seg_row, s.seg_slot, s.row_seg0, s.row_nseg, s.range_seg, s.nranges, cols, coeffs, x, ldx, dim,
        nchunks, y, ldy, row_base, partial, partial_ld, counters, counters_ld, special);
}

// SpMM gather engine (GASB_SPMM_ENGINE = flat | tma | cp | direct; default flat): the
// flat-stream TMA kernel, the segment-staged TMA / cp.async pipeline, or direct register
// loads. All produce identical values (same segments and accumulation order).
static int spmm_engine() {
    static int v = [] {
        const char* e = getenv("GASB_SPMM_ENGINE");
        if (!e) return 3;
        if (!strcmp(e, "direct")) return 2;
        if (!strcmp(e, "cp")) return 1;
        if (!strcmp(e, "flat")) return 3;
        return 0;
    }();
    return v;
}

// ---- flat-stream forward (TMA tile::gather4) -------------------------------------------
// The pipelined kernel above cuts stages at segment boundaries, so every row costs at least
// one (often short) stage and each stage walks the segment cursor. Here a stage is a fixed
// 16-edge slice of the work range's flat edge stream: the edge metadata arrives in 32-edge
// windows (cp.async ring, kMetaWin ahead), a stage is exactly half a window, and segment
// (row) ends are handled inside the FMA loop — a stage with no segment end (the common
// case: rows average hundreds of edges) runs the 16 FMAs straight. Same segments, ranges,
// fp64 partials and accumulation order as the pipelined kernel (bit-identical results).
template <int CPL, int MODE, bool DUAL>
__device__ __forceinline__ void flat_items(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, const int32_t* __restrict__ range_seg,
    int32_t nranges, const int32_t* __restrict__ cols, const double* __restrict__ coeffs, int32_t dim,
    int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base, double* __restrict__ partial, int64_t pld,
    int32_t* __restrict__ counters, int32_t cld, const int32_t* __restrict__ slot_list, const CUtensorMap* tmap,
    unsigned char* wbase, uint64_t* bars,
    int32_t* ring_c, double* ring_f, const RowSums& rsum) {
    using Cfg = PipeCfg<CPL>;
    constexpr int KE = Cfg::kEdges;
    static_assert(KE == 8 || KE == 16 || KE == 32, "a flat stage is a quarter, half or all of a 32-edge window");
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kPipeWarps;
    uint32_t phases = 0;
    for (int64_t item = static_cast<int64_t>(blockIdx.x) * kPipeWarps + (threadIdx.x >> 5);
         item < static_cast<int64_t>(nchunks) * nranges; item += nwarps) {
        const int32_t chunk = static_cast<int32_t>(item / nranges);
        const int32_t r = static_cast<int32_t>(item - static_cast<int64_t>(chunk) * nranges);
        const int32_t s_lo = range_seg[r], s_hi = range_seg[r + 1];
        if (s_lo >= s_hi) continue;
        const int32_t col = chunk * Cfg::kCols + lane * (CPL == 8 ? 4 : CPL);
        const int64_t e_lo = seg_beg[s_lo], e_hi = seg_beg[s_hi];
        const int32_t nst = static_cast<int32_t>((e_hi - e_lo + KE - 1) / KE);
        // consumer-side window of 32 segment records (end offset, row, slot)
        int32_t wseg = s_lo, cur = s_lo;
        int64_t w_end = 0;
        int32_t w_row = 0, w_slot = -1;
        auto load_window = [&](int32_t from) {
            wseg = from;
            const int32_t sg = from + lane;
            w_end = sg < s_hi ? seg_beg[sg + 1] : 0;
            w_row = sg < s_hi ? seg_row[sg] : 0;
            w_slot = sg < s_hi ? seg_slot[sg] : -1;
        };
        load_window(s_lo);
        int64_t cur_end = __shfl_sync(0xffffffffu, w_end, 0);
        // edge-metadata ring: window q = edges [e_lo + 32q, +32) in ring slot q % kMetaWin
        int w_issued = 0;
        auto prefetch_win = [&] {
            const int slot = w_issued % kMetaWin;
            const int64_t e = e_lo + 32LL * w_issued + lane;
            if (e < e_hi) {
                cp_async_ca4(ring_c + slot * 32 + lane, cols + e);
                cp_async_ca8(ring_f + slot * 32 + lane, coeffs + e);
            }
            cp_async_commit();
            ++w_issued;
        };
#pragma unroll
        for (int k = 0; k < kMetaWin; ++k)
            if (e_lo + 32LL * w_issued < e_hi) prefetch_win();
        auto issue = [&](int32_t k, int slot_idx) {
            const int q = (k * KE) >> 5;  // metadata window of this stage
            while (w_issued < q + kMetaWin && e_lo + 32LL * w_issued < e_hi) prefetch_win();
            const int allowed = w_issued - (q + 1);  // groups that may stay in flight
            if (allowed >= 3) cp_async_wait<3>();
            else if (allowed == 2) cp_async_wait<2>();
            else if (allowed == 1) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncwarp();
            const int64_t e0 = e_lo + static_cast<int64_t>(k) * KE;
            const int cnt = static_cast<int>(e_hi - e0 < KE ? e_hi - e0 : KE);
            unsigned char* st = wbase + slot_idx * Cfg::kStageBytes;
            int32_t* srow = reinterpret_cast<int32_t*>(st + kStageDataBytes + KE * 8 + Cfg::kHdrBytes);
            if (lane < KE) {
                const int ridx = (q % kMetaWin) * 32 + ((k * KE) & 31) + lane;
                const bool ok = lane < cnt;
                reinterpret_cast<double*>(st + kStageDataBytes)[lane] = ok ? ring_f[ridx] : 0.0;
                srow[lane] = ok ? ring_c[ridx] : -1;  // row -1: zero-filled by TMA
            }
            __syncwarp();
            if (lane == 0) {
                const int ng = (cnt + 3) >> 2;
                float* rows = reinterpret_cast<float*>(st);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // after the warp's reads
                mbar_expect_tx(bars + slot_idx, static_cast<uint32_t>(ng) * 4u * Cfg::kCols * 4u);
                const int32_t c0 = chunk * Cfg::kCols;
                for (int i = 0; i < ng; ++i) {
                    const int4 rr = reinterpret_cast<const int4*>(srow)[i];
                    tma_gather4(rows + 4 * i * Cfg::kCols, tmap, c0, rr.x, rr.y, rr.z, rr.w, bars + slot_idx);
                }
            }
        };
        double acc[CPL], acc2[CPL];  // acc2: odd stage edges when DUAL (added at the row end)
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = acc2[k] = 0.0;
        auto finish = [&] {
            const int kk = cur - wseg;
            const int32_t row = __shfl_sync(0xffffffffu, w_row, kk);
            const int32_t slot = __shfl_sync(0xffffffffu, w_slot, kk);
            if constexpr (DUAL) {
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    acc[k] = __dadd_rn(acc[k], acc2[k]);
                    acc2[k] = 0.0;
                }
            }
            seg_finish<CPL>(acc, row, slot, lane, col, chunk, dim, y, ldy, row_base, partial, pld, counters, cld,
                            slot_list, row_seg0, row_nseg, rsum);
            ++cur;
            if (cur < s_hi) {
                if (cur - wseg >= 32) load_window(cur);
                cur_end = __shfl_sync(0xffffffffu, w_end, cur - wseg);
            }
        };
        int32_t issued = 0;
#pragma unroll
        for (int k = 0; k < kStages; ++k)
            if (issued < nst) {
                issue(issued, k);
                ++issued;
            }
        for (int32_t b = 0; b < nst; ++b) {
            const int sl = b % kStages;
            mbar_wait(bars + sl, (phases >> sl) & 1u);
            phases ^= 1u << sl;
            const unsigned char* st = wbase + sl * Cfg::kStageBytes;
            const float* rows = reinterpret_cast<const float*>(st) + lane * (CPL == 8 ? 4 : CPL);
            const double* cf = reinterpret_cast<const double*>(st + kStageDataBytes);
            const int64_t eb = e_lo + static_cast<int64_t>(b) * KE;
            const int cnt = static_cast<int>(e_hi - eb < KE ? e_hi - eb : KE);
#ifdef GASB_SPMM_NOFMA  // timing probe only (wrong values): the gathers without the FMAs
            if (cnt == KE && cur_end >= eb + KE) {
                acc[0] += cf[lane & 15] * rows[0];
            } else
#endif
            if (cnt == KE && cur_end >= eb + KE) {  // no segment ends inside: straight FMAs
                if constexpr (DUAL) {
#pragma unroll
                    for (int j = 0; j < KE; j += 2) {
                        edge_fma<CPL, MODE>(rows, cf, j, acc);
                        edge_fma<CPL, MODE>(rows, cf, j + 1, acc2);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < KE; ++j) edge_fma<CPL, MODE>(rows, cf, j, acc);
                }
            } else {
                for (int j = 0; j < cnt; ++j) {
                    while (eb + j == cur_end && cur < s_hi) finish();
                    if (DUAL && (j & 1)) edge_fma<CPL, MODE>(rows, cf, j, acc2);
                    else edge_fma<CPL, MODE>(rows, cf, j, acc);
                }
            }
            __syncwarp();
            if (issued < nst) {  // refill the slot just consumed
                issue(issued, sl);
                ++issued;
            }
        }
        while (cur < s_hi) finish();
        cp_async_wait<0>();
        __syncwarp();
    }
}

template <int CPL, bool DUAL>
__global__ void __launch_bounds__(kPipeWarps * 32, kPipeCtas) spmm_fwd_flat_kernel(
    const int64_t* __restrict__ seg_beg, const int32_t* __restrict__ seg_row, const int32_t* __restrict__ seg_slot,
    const int32_t* __restrict__ row_seg0, const int32_t* __restrict__ row_nseg, const int32_t* __restrict__ range_seg,
    int32_t nranges, const int32_t* __restrict__ cols, const double* __restrict__ coeffs, int32_t dim,
    int32_t nchunks, float* __restrict__ y, int64_t ldy, int64_t row_base, double* __restrict__ partial, int64_t pld,
    int32_t* __restrict__ counters, int32_t cld, const int32_t* __restrict__ table_flags,
    const int32_t* __restrict__ slot_list, const __grid_constant__ CUtensorMap tmap, const RowSums rsum) {
    using Cfg = PipeCfg<CPL>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    pdl_trigger();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* wbase = smem_raw + static_cast<size_t>(warp) * kStages * Cfg::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kPipeWarps * kStages * Cfg::kStageBytes) + warp * kStages;
    unsigned char* ring = smem_raw + kPipeWarps * kStages * Cfg::kStageBytes + kPipeWarps * kStages * 8 +
                          warp * kMetaRingBytes;
    int32_t* ring_c = reinterpret_cast<int32_t*>(ring);
    double* ring_f = reinterpret_cast<double*>(ring + kMetaWin * 32 * 4);
    if (lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (int k = 0; k < kStages; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    pdl_wait();  // (PDL) everything below reads the previous kernels' outputs
    const int mode = widen_mode(table_flags);
#define GASB_FLAT(M)                                                                                              \
    flat_items<CPL, M, DUAL>(seg_beg, seg_row, seg_slot, row_seg0, row_nseg, range_seg, nranges, cols, coeffs, dim, nchunks, \
                  y, ldy, row_base, partial, pld, counters, cld, slot_list, &tmap, wbase, bars, ring_c, ring_f, rsum)
    if (mode == kWidenNonNeg) GASB_FLAT(kWidenNonNeg);
    else if (mode == kWidenSigned) GASB_FLAT(kWidenSigned);
    else GASB_FLAT(kWidenF2F);
#undef GASB_FLAT
}

// Grid cap of the flat SpMM launches enqueued by this thread (set_spmm_grid_cap): the
// background stream's launches leave SMs to the batch chain running beside them.
static thread_local int32_t t_spmm_grid_cap = 0;
void set_spmm_grid_cap(int32_t ctas) { t_spmm_grid_cap = ctas; }
// Row-sum hand-off of this thread's next flat SpMM launches (set_spmm_row_sums).
static thread_local RowSums t_row_sums{};
void set_spmm_row_sums(double* out, const double* in, int64_t ld) { t_row_sums = RowSums{out, in, ld}; }

template <int CPL, bool DUAL>
static void launch_flat(const SpmmSegs& s, const int32_t* cols, const double* coeffs, int32_t dim, float* y,
                        int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld, int32_t* counters,
                        int32_t counters_ld, cudaStream_t st, const int32_t* special, const CUtensorMap* tmap) {
    using Cfg = PipeCfg<CPL>;
    constexpr int kSmem = Cfg::kSmem + kPipeWarps * kStages * 8 + kPipeWarps * kMetaRingBytes;
    static int set = 0;
    if (!set) {
        GASB_CUDA(cudaFuncSetAttribute(spmm_fwd_flat_kernel<CPL, DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmem));
        set = 1;
    }
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, Cfg::kCols));
    require(nchunks <= counters_ld && static_cast<int64_t>(nchunks) * Cfg::kCols <= partial_ld,
            "spmm_fwd: counters / partials too narrow");
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        GASB_CUDA(cudaGetDevice(&dev));
        GASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int64_t items = static_cast<int64_t>(nchunks) * s.nranges;
    int64_t blocks = std::min<int64_t>(ceil_div(items, kPipeWarps), static_cast<int64_t>(kPipeCtas) * sms);
    if (t_spmm_grid_cap > 0) blocks = std::min<int64_t>(blocks, t_spmm_grid_cap);
    launch_pdl(spmm_fwd_flat_kernel<CPL, DUAL>, dim3(static_cast<unsigned>(blocks)), dim3(kPipeWarps * 32), kSmem, st,
               s.seg_beg, s.seg_row, s.seg_slot, s.row_seg0, s.row_nseg, s.range_seg, s.nranges, cols, coeffs, dim,
               nchunks, y, ldy, row_base, partial, partial_ld, counters, counters_ld, special,
               s.row_slots ? s.row_slots : s.seg_slot, *tmap, t_row_sums);
}

static int g_pipe_smem_set[2][2] = {};

template <int CPL, bool TMA>
static void launch_pipe(const SpmmSegs& s, const int32_t* cols, const double* coeffs, const float* x, int64_t ldx,
                        int32_t dim, float* y, int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld,
                        int32_t* counters, int32_t counters_ld, cudaStream_t st, const int32_t* special,
                        const CUtensorMap* tmap) {
    using Cfg = PipeCfg<CPL>;
    auto kern = spmm_fwd_pipe_kernel<CPL, TMA>;
    constexpr int kSmem = Cfg::kSmem + kPipeWarps * kStages * 8 + (TMA ? kPipeWarps * kMetaRingBytes : 0);
    int& set = g_pipe_smem_set[CPL == 4][TMA];
    if (!set) {
        GASB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        set = 1;
    }
    CUtensorMap tm{};
    if (tmap) tm = *tmap;
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, Cfg::kCols));
    require(nchunks <= counters_ld && static_cast<int64_t>(nchunks) * Cfg::kCols <= partial_ld,
            "spmm_fwd: counters / partials too narrow");
    // persistent grid: 2 CTAs (8 warps) per SM — the shared-memory bound — over (chunk, range)
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        GASB_CUDA(cudaGetDevice(&dev));
        GASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int64_t items = static_cast<int64_t>(nchunks) * s.nranges;
    const int64_t blocks = std::min<int64_t>(ceil_div(items, kPipeWarps), static_cast<int64_t>(kPipeCtas) * sms);
    kern<<<static_cast<unsigned>(blocks), kPipeWarps * 32, kSmem, st>>>(
        s.seg_beg, s.seg_row, s.seg_slot, s.row_seg0, s.row_nseg, s.range_seg, s.nranges, cols, coeffs, x, ldx, dim,
        nchunks, y, ldy, row_base, partial, partial_ld, counters, counters_ld, special, tm);
}

// Tensor map of a row-major fp32 table (rows x dim, pitch ld floats) for tile::gather4:
// box = {box_cols, 1}; columns >= dim and rows outside [0, rows) read as zero.
bool make_row_tmap(const float* base, int64_t rows, int32_t dim, int64_t ld, int32_t box_cols, CUtensorMap* out) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (rows <= 0 || dim <= 0 || (ld * 4) % 16 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(rows)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 1};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box,
                              estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// SpMM gather engine (tuning knob GASB_SPMM_TMA = 0 | 1, default 1: TMA tile::gather4).
bool spmm_use_tma() {
    static int v = [] {
        const char* e = getenv("GASB_SPMM_TMA");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

// Columns per lane of the flat SpMM for a table of width dim (tuning knob GASB_SPMM_CPL =
// 2 | 4 | 8 forces one). Default: 2 (64-column chunks) up to 64 columns (products-shape
// APPNP 381 -> 377 ms, PubMed GCNII 30.5 -> 30.2 ms per epoch); 8 (256-column chunks, 1 KB
// TMA rows) when the 256-column rounding wastes no more than the 128-column one plus 64
// columns; else 4. Fewer, wider
// gathered rows: a probe timing the gathers alone (FMAs removed) fitted
// t = 35 us per (rows of a 512 B batch) + 29 us per 573 MB at C3, i.e. a per-row TMA cost
// next to the L2 -> SM byte rate (19.6 TB/s measured by tools/l2bw).
int32_t spmm_cpl_for(int32_t dim) {
    static const int forced = [] {
        const char* e = getenv("GASB_SPMM_CPL");
        const int v = e ? atoi(e) : 0;
        return v == 2 || v == 4 || v == 8 ? v : 0;
    }();
    if (forced) return forced;
    if (dim <= 64) return 2;  // narrow tables (APPNP's C-wide histories, GCNII h = 64): no idle lanes
    const int32_t r = dim % 256;
    return (dim >= 192 && (r == 0 || r > 192)) ? 8 : 4;
}

int32_t spmm_box_cols(int32_t dim) { return 32 * spmm_cpl_for(dim); }

int32_t spmm_ranges_per_launch() {
    static int32_t v = 0;
    if (!v) {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
            sms = 148;
        v = kPipeCtas * kPipeWarps * sms;
        if (const char* e = getenv("GASB_SPMM_RANGES_PER_SM")) v = std::max(1, atoi(e)) * sms;  // (the reg engine)
    }
    return v;
}

// Splits segments [g0, g1) (edges seg_beg[g0] .. seg_beg[g1]) into `nranges` contiguous
// ranges of ~equal edge count; out receives nranges + 1 absolute segment boundaries.
void split_ranges(const int64_t* seg_beg, int64_t g0, int64_t g1, int32_t nranges, int32_t* out) {
    const int64_t E0 = seg_beg[g0], E = seg_beg[g1] - E0;
    int64_t s = g0;
    out[0] = static_cast<int32_t>(g0);
    for (int32_t r = 1; r < nranges; ++r) {
        const int64_t target = E0 + E * r / nranges;
        while (s < g1 && seg_beg[s] < target) ++s;
        out[r] = static_cast<int32_t>(s);
    }
    out[nranges] = static_cast<int32_t>(g1);
}

// Segments the rows [r_lo, r_hi) of one launch (rp: absolute edge offsets). split = false:
// one segment per row (the bit-exact sequential mode) and ranges at row boundaries.
// split = true: the launch's edges are cut into nranges ranges of EXACTLY equal size and a
// row is split only where a range boundary falls inside it (<= nranges - 1 extra segments
// per launch, each an fp64 partial); all other rows are one segment with no partial.
void segment_launch(const int64_t* rp, int64_t r_lo, int64_t r_hi, bool split, int32_t nranges,
                    std::vector<int64_t>& sb, std::vector<int32_t>& sr, std::vector<int32_t>& ss, int32_t* r0,
                    int32_t* rn, int64_t& slot, int32_t* ranges) {
    const int64_t g0 = static_cast<int64_t>(sr.size());
    const int64_t E0 = rp[r_lo], E = rp[r_hi] - E0;
    auto bound = [&](int64_t k) { return E0 + E * k / nranges; };
    int64_t k = 1;  // next interior boundary
    std::vector<int64_t> cuts;
    for (int64_t r = r_lo; r < r_hi; ++r) {
        const int64_t b = rp[r], e = rp[r + 1];
        while (k < nranges && bound(k) <= b) ++k;
        cuts.clear();
        if (split)
            for (; k < nranges && bound(k) < e; ++k)
                if (cuts.empty() || cuts.back() != bound(k)) cuts.push_back(bound(k));
        const int64_t pieces = 1 + static_cast<int64_t>(cuts.size());
        r0[r] = static_cast<int32_t>(sr.size());
        rn[r] = static_cast<int32_t>(pieces);
        for (int64_t i = 0; i < pieces; ++i) {
            sb.push_back(i == 0 ? b : cuts[static_cast<size_t>(i - 1)]);
            sr.push_back(static_cast<int32_t>(r));
            ss.push_back(pieces == 1 ? -1 : static_cast<int32_t>(slot++));
        }
    }
    const int64_t g1 = static_cast<int64_t>(sr.size());
    sb.push_back(rp[r_hi]);  // sentinel (popped by the caller when appending more launches)
    if (!split) {
        split_ranges(sb.data(), g0, g1, nranges, ranges);
        return;
    }
    int64_t s = g0;  // ranges: first segment starting at or after each boundary
    ranges[0] = static_cast<int32_t>(g0);
    for (int32_t q = 1; q < nranges; ++q) {
        const int64_t t = bound(q);
        while (s < g1 && sb[s] < t) ++s;
        ranges[q] = static_cast<int32_t>(s);
    }
    ranges[nranges] = static_cast<int32_t>(g1);
}

// Two interleaved fp64 chains per column in the segmented (non-exact) mode (GASB_SPMM_DUAL
// = 1 enables; measured no faster at C3, so off by default).
static bool spmm_dual() {
    static int v = [] {
        const char* e = getenv("GASB_SPMM_DUAL");
        return e ? atoi(e) : 0;
    }();
    return v != 0;
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
                     int32_t* counters, int32_t counters_ld, cudaStream_t st, const int32_t* special,
                     const CUtensorMap* tmap) {
    if (s.nranges <= 0 || dim <= 0) return;
    require(ldx % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0,
            "spmm_fwd: source rows must be 16 B aligned (ldx % 4 == 0)");
    if (spmm_engine() == 3 && tmap && spmm_use_tma()) {
#define GASB_FLAT_LAUNCH(C, D) \
    launch_flat<C, D>(s, cols, coeffs, dim, y, ldy, row_base, partial, partial_ld, counters, counters_ld, st, special, tmap)
        const bool dual = !s.exact && spmm_dual();
        const int cpl = spmm_cpl_for(dim);  // must match the tensor map's box (spmm_box_cols(dim))
        if (cpl == 8) {
            GASB_FLAT_LAUNCH(8, false);
        } else if (cpl == 2) {
            if (dual) GASB_FLAT_LAUNCH(2, true);
            else GASB_FLAT_LAUNCH(2, false);
        } else {
            if (dual) GASB_FLAT_LAUNCH(4, true);
            else GASB_FLAT_LAUNCH(4, false);
        }
#undef GASB_FLAT_LAUNCH
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return;
    }
    require(!s.row_slots, "spmm_fwd: a slot-list segment table needs the flat TMA engine");
    if (spmm_engine() == 2) {
        launch_direct(s, cols, coeffs, x, ldx, dim, y, ldy, row_base, partial, partial_ld, counters, counters_ld, st,
                      special);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return;
    }
    // (a 256-column tensor map belongs to the flat kernel: the staged kernels use cp.async then)
    const bool tma = tmap != nullptr && spmm_use_tma() && spmm_engine() == 0 && spmm_cpl_for(dim) != 8;
#define GASB_PIPE(C, T)                                                                                               \
    launch_pipe<C, T>(s, cols, coeffs, x, ldx, dim, y, ldy, row_base, partial, partial_ld, counters, counters_ld, st, \
                      special, tmap)
    if (spmm_cpl_for(dim) == 2) {  // (the staged kernels run 2 or 4 columns per lane)
        if (tma) GASB_PIPE(2, true);
        else GASB_PIPE(2, false);
    } else {
        if (tma) GASB_PIPE(4, true);
        else GASB_PIPE(4, false);
    }
#undef GASB_PIPE
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(256) spmm_bwd_kernel(const int64_t* __restrict__ rp, int32_t nt,
                                                       const int32_t* __restrict__ src, const float* __restrict__ cf,
                                                       const float* __restrict__ gy, int64_t ldgy, int32_t dim,
                                                       int32_t nchunks, const float* __restrict__ mask, int64_t ldm,
                                                       float* __restrict__ gx, int64_t ldgx, int accumulate) {
    const int lane = threadIdx.x & 31;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= static_cast<int64_t>(nt) * nchunks) return;
    const int32_t chunk = static_cast<int32_t>(w / nt);
    const int32_t t = static_cast<int32_t>(w - static_cast<int64_t>(chunk) * nt);
    const int32_t col = chunk * kChunk + lane * 2;
    const bool active = col < dim;
    const float* gc = gy + col;
    float a0 = 0.0f, a1 = 0.0f;
    if (accumulate && active) {
        const float* o = gx + static_cast<int64_t>(t) * ldgx + col;
        a0 = o[0];
        a1 = col + 1 < dim ? o[1] : 0.0f;
    }
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
constexpr int kBwdRing = 8;  // metadata windows in flight per warp (spmm_bwd_smem_kernel)
constexpr int kBwdThreads = 1024;
#ifdef GASB_BWD_TIMING  // per-CTA globaltimer stamps of the last launch (timing probe builds only)
__device__ unsigned long long g_bwd_stamps[512 * 4];  // [0, 256): spmm_bwd_smem, [256, 512): spmm_bwd2
extern "C" void gasb_debug_bwd_stamps(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_bwd_stamps, sizeof(unsigned long long) * 512 * 4);
}
__device__ unsigned long long g_bwd_end[512];
__device__ unsigned long long g_bwd_warp[64 * 3];  // spmm_bwd2, CTA (0, 0), phase 0: per warp entries, targets, end
extern "C" void gasb_debug_bwd_warp(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_bwd_warp, sizeof(unsigned long long) * 64 * 3);
}
extern "C" void gasb_debug_bwd_end(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_bwd_end, sizeof(unsigned long long) * 512);
}
__device__ __forceinline__ unsigned long long bwd_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

__global__ void __launch_bounds__(kBwdThreads) spmm_bwd_smem_kernel(
    const int64_t* __restrict__ rp, int32_t nt, const int32_t* __restrict__ src, const float* __restrict__ cf,
    const float* __restrict__ gy, int64_t ldgy, int32_t nsrc, int32_t dim, const float* __restrict__ mask,
    int64_t ldm, float* __restrict__ gx, int64_t ldgx, int32_t targets_per_cta, int accumulate, const int32_t* __restrict__ order) {
    extern __shared__ float sg[];  // nsrc x kBwdCW, then 32 (offset, coeff) pairs per warp
    __shared__ int32_t s_next;
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x == 0) s_next = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#ifdef GASB_BWD_TIMING
    const int cta = blockIdx.x + gridDim.x * blockIdx.y;
    if (threadIdx.x == 0 && cta < 256) {
        g_bwd_stamps[cta * 4] = bwd_now();
        g_bwd_stamps[cta * 4 + 2] = 0;
        g_bwd_stamps[cta * 4 + 3] = 0;
    }
    unsigned long long my_entries = 0;
#endif
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
#ifdef GASB_BWD_TIMING
    if (threadIdx.x == 0 && cta < 256) g_bwd_stamps[cta * 4 + 1] = bwd_now();
#endif
    // targets t = blockIdx.y + splits * k; warps claim k dynamically (power-law in-degrees)
    const int32_t splits = targets_per_cta;
    // per-warp ring of kBwdRing 32-entry windows of (source row, coeff), filled by cp.async
    // kBwdRing windows ahead: a hub target (~1,100 intra-batch entries at C3) costs one
    // metadata latency, not one per window
    // (row, coeff) pairs interleaved so an entry is one broadcast LDS.64
    int2* ring = reinterpret_cast<int2*>(sg + static_cast<int64_t>(nsrc) * kBwdCW) + warp * kBwdRing * 32;
    auto claim = [&]() -> int32_t {
        int32_t k = 0;
        if (lane == 0) k = atomicAdd(&s_next, 1);
        const int32_t i = static_cast<int32_t>(blockIdx.y) + splits * __shfl_sync(0xffffffffu, k, 0);
        return (order && i < nt) ? __ldg(order + i) : i;
    };
    // software-pipelined over targets: the next target is claimed and its row pointers loaded
    // while the current one accumulates
    int32_t t = claim();
    int64_t e0n = t < nt ? rp[t] : 0, e1n = t < nt ? rp[t + 1] : 0;
    for (;;) {
        if (t >= nt) break;
        const int64_t e0 = e0n, e1 = e1n;
        const bool keep = !mask || lane >= ncol || mask[static_cast<int64_t>(t) * ldm + col0 + lane] > 0.0f;
        float a = (accumulate && lane < ncol) ? gx[static_cast<int64_t>(t) * ldgx + col0 + lane] : 0.0f;
        const int32_t tn = claim();
        if (tn < nt) {
            e0n = rp[tn];
            e1n = rp[tn + 1];
        }
        const int32_t nw = static_cast<int32_t>((e1 - e0 + 31) >> 5);
        int32_t issued = 0;
        auto prefetch = [&] {
            const int slot = issued % kBwdRing;
            const int64_t e = e0 + 32LL * issued + lane;
            if (e < e1) {
                int2* dst = ring + slot * 32 + lane;
                cp_async_ca4(&dst->x, src + e);
                cp_async_ca4(&dst->y, cf + e);
            }
            cp_async_commit();
            ++issued;
        };
#pragma unroll
        for (int k = 0; k < kBwdRing; ++k)
            if (issued < nw) prefetch();
        const float* sgl = sg + lane;
        for (int32_t q = 0; q < nw; ++q) {
            const int pending = issued - q - 1;  // windows after q that may still be in flight
            if (pending >= 7) cp_async_wait<7>();
            else if (pending == 6) cp_async_wait<6>();
            else if (pending == 5) cp_async_wait<5>();
            else if (pending == 4) cp_async_wait<4>();
            else if (pending == 3) cp_async_wait<3>();
            else if (pending == 2) cp_async_wait<2>();
            else if (pending == 1) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncwarp();
            const int slot = q % kBwdRing;
            const int2* w = ring + slot * 32;
            const int64_t eb = e0 + 32LL * q;
            const int cnt = static_cast<int>(e1 - eb < 32 ? e1 - eb : 32);
            if (cnt == 32) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int2 rc = w[j];
                    a = __fadd_rn(a, __fmul_rn(__int_as_float(rc.y), sgl[rc.x * kBwdCW]));
                }
            } else {
                for (int j = 0; j < cnt; ++j) {
                    const int2 rc = w[j];
                    a = __fadd_rn(a, __fmul_rn(__int_as_float(rc.y), sgl[rc.x * kBwdCW]));
                }
            }
            __syncwarp();  // the slot is free again
            if (issued < nw) prefetch();
        }
        if (lane < ncol) gx[static_cast<int64_t>(t) * ldgx + col0 + lane] = keep ? a : 0.0f;
#ifdef GASB_BWD_TIMING
        my_entries += static_cast<unsigned long long>(e1 - e0);
#endif
        t = tn;
    }
#ifdef GASB_BWD_TIMING
    if (lane == 0 && cta < 256) {
        atomicMax(&g_bwd_stamps[cta * 4 + 2], bwd_now());
        atomicMax(&g_bwd_stamps[cta * 4 + 3], my_entries);
    }
#endif
}

static int g_bwd_smem_set = 0;

void launch_spmm_bwd(const int64_t* t_rowptr, int32_t nt, const int32_t* t_src, const float* t_coeffs,
                     const float* gy, int64_t ldgy, int32_t dim, const float* mask, int64_t ldm, float* gx,
                     int64_t ldgx, cudaStream_t st, int32_t nsrc, bool accumulate, const int32_t* order) {
    if (nt <= 0 || dim <= 0) return;
    const int64_t smem = static_cast<int64_t>(nsrc) * kBwdCW * sizeof(float) + (kBwdThreads / 32) * kBwdRing * 32 * 8;
    if (nsrc > 0 && smem <= 216 * 1024) {
        auto kern = spmm_bwd_smem_kernel;
        if (!g_bwd_smem_set) {
            GASB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024));
            g_bwd_smem_set = 1;
        }
        const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kBwdCW));
        // one CTA per SM (the staged slice fills shared memory): a single wave of <= #SMs CTAs
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            GASB_CUDA(cudaGetDevice(&dev));
            GASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        }
        const int32_t splits = static_cast<int32_t>(
            std::max<int64_t>(1, std::min<int64_t>(sms / nchunks, ceil_div(nt, kBwdThreads / 32))));
        dim3 grid(static_cast<unsigned>(nchunks), static_cast<unsigned>(splits));
        launch_pdl(kern, grid, dim3(kBwdThreads), smem, st, t_rowptr, nt, t_src, t_coeffs, gy, ldgy, nsrc, dim, mask,
                   ldm, gx, ldgx, splits, accumulate ? 1 : 0, order);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return;
    }
    require(ldgy % 2 == 0 && ldgx % 2 == 0 && (!mask || ldm % 2 == 0), "spmm_bwd: leading dimensions must be even");
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kChunk));
    const int64_t blocks = ceil_div(static_cast<int64_t>(nt) * nchunks, 8);
    spmm_bwd_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(t_rowptr, nt, t_src, t_coeffs, gy, ldgy, dim,
                                                                   nchunks, mask, ldm, gx, ldgx, accumulate ? 1 : 0);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

// ---- aggregate backward, two columns per lane (spmm_bwd2) ---------------------------------
// Same per-target sums as spmm_bwd_smem_kernel (entries in ascending source row, fp32 multiply
// then add -> bit-exact) at half the instructions per column: each lane owns two adjacent
// columns of a 64-column chunk and does both with one packed multiply and one packed add
// (FFMA2 / FADD2). The multiply is fma.rn.f32x2(c, x, z) with z = -0.0 held in a kernel
// parameter: exactly c * x rounded once for every input, and opaque, so ptxas cannot contract
// the following add into an FMA (it does contract mul.rn.f32x2 + add.rn.f32x2, even with
// --fmad=false).
// A 64-column slice of every source row does not fit shared memory next to the metadata, so
// the sources are staged in phases of kBwd2Rows rows. The plan (build_bwd2_plan) is laid out
// per (CTA split, phase) as one contiguous blob: a target table {t, first entry, count} in
// claim order (heaviest first), then each target's entries of that phase (ascending source,
// padded to a multiple of 8 with (zero row, -0.0), which add exactly nothing: a + (-0.0 *
// 0.0) == a for every a). At each phase one thread issues the TMA loads of the source slice
// and one bulk copy of the blob, so no warp waits on a dependent global load afterwards.
// Between phases the running fp32 sums live in gx: the accumulation sequence is unchanged.
constexpr int kBwd2CW = 64;
constexpr int kBwd2Rows = 608;                   // source rows per phase (a multiple of the TMA box)
#ifndef GASB_BWD2_BOX
#define GASB_BWD2_BOX 32
#endif
constexpr int kBwd2Box = GASB_BWD2_BOX;          // rows per TMA box
constexpr int kBwd2Threads = 1024;
constexpr int kBwd2SliceBytes = (kBwd2Rows + 1) * kBwd2CW * 4;  // + the zero row
constexpr int kBwd2BlobBytes = 52 * 1024;        // per (split, phase) plan blob
constexpr int kBwd2Slots = 48;                   // targets per split: running sums kept in shared memory
constexpr int kBwd2MaxPhases = 8;
// + 64 B for the mbarrier and the claim counter, + 128 B to align the TMA destination
constexpr int kBwd2Smem = kBwd2SliceBytes + kBwd2BlobBytes + kBwd2Slots * kBwd2CW * 4 + 64 + 128;

__device__ __forceinline__ uint64_t f2_mulz(float c, uint64_t x, uint64_t negz) {
    uint64_t d;
    const uint64_t cc = (static_cast<uint64_t>(__float_as_uint(c)) << 32) | __float_as_uint(c);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(cc), "l"(x), "l"(negz));
    return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// blob_off: (splits * phases + 1) byte offsets into blobs, (split, phase) major.
__global__ void __launch_bounds__(kBwd2Threads) spmm_bwd2_kernel(
    const int64_t* __restrict__ blob_off, const unsigned char* __restrict__ blobs, int32_t phases, int32_t nsrc,
    int32_t dim, const float* __restrict__ mask, int64_t ldm, float* __restrict__ gx, int64_t ldgx, int accumulate,
    uint64_t negz, const __grid_constant__ CUtensorMap gy_map) {
    extern __shared__ __align__(128) unsigned char smem_raw2[];
    __shared__ int64_t s_off[kBwd2MaxPhases + 1];
    // (pointer arithmetic on the __shared__ array, so the compiler keeps LDS/STS for it)
    unsigned char* base =
        smem_raw2 + ((128u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw2)) & 127u)) & 127u);
    float* sg = reinterpret_cast<float*>(base);  // (kBwd2Rows + 1) x 64: the phase's rows, then a zero row
    unsigned char* blob = base + kBwd2SliceBytes;
    float2* run = reinterpret_cast<float2*>(blob + kBwd2BlobBytes);  // [slot][32 lanes]: sums between phases
    uint64_t* bar = reinterpret_cast<uint64_t*>(blob + kBwd2BlobBytes + kBwd2Slots * kBwd2CW * 4);
    int32_t* s_next = reinterpret_cast<int32_t*>(bar + 1);
    const int lane = threadIdx.x & 31;
    const int32_t col0 = blockIdx.x * kBwd2CW;
    const int32_t ncol = min(kBwd2CW, dim - col0);
    const int32_t c = col0 + 2 * lane;  // this lane's columns c, c + 1
    const bool has0 = 2 * lane < ncol, has1 = 2 * lane + 1 < ncol;
    const bool vec_gx = (ldgx % 2 == 0) && ((reinterpret_cast<uintptr_t>(gx) & 7) == 0);
    const bool vec_m = !mask || ((ldm % 2 == 0) && ((reinterpret_cast<uintptr_t>(mask) & 7) == 0));
    const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    // the plan is static data (not produced by the preceding kernels): its offsets and the first
    // blob are fetched before pdl_wait; the source slice only after it
    auto issue_slice = [&](int32_t q) {
        const int32_t r0 = q * kBwd2Rows, rows = min(kBwd2Rows, nsrc - r0);
        for (int32_t b = 0; b < (rows + kBwd2Box - 1) / kBwd2Box; ++b)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sg + b * kBwd2Box * kBwd2CW))),
                "l"(reinterpret_cast<uint64_t>(&gy_map)), "r"(col0), "r"(r0 + b * kBwd2Box), "r"(bar_s)
                : "memory");
    };
    auto expect_and_issue_blob = [&](int32_t q) {  // thread 0: this phase's transaction bytes, then the blob
        const int32_t rows = min(kBwd2Rows, nsrc - q * kBwd2Rows);
        const uint32_t blob_bytes = static_cast<uint32_t>(s_off[q + 1] - s_off[q]);
        mbar_expect_tx(bar, static_cast<uint32_t>((rows + kBwd2Box - 1) / kBwd2Box) * kBwd2Box * kBwd2CW * 4u + blob_bytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(blob))), "l"(blobs + s_off[q]),
                     "r"(blob_bytes), "r"(bar_s)
                     : "memory");
    };
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&gy_map)) : "memory");
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int32_t q = 0; q <= phases; ++q) s_off[q] = blob_off[static_cast<int64_t>(blockIdx.y) * phases + q];
        *s_next = 0;
        expect_and_issue_blob(0);
    }
    if (threadIdx.x < kBwd2CW) sg[kBwd2Rows * kBwd2CW + threadIdx.x] = 0.0f;  // the padding entries' row
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x == 0) issue_slice(0);
    __syncthreads();  // the zero row
    const unsigned char* sgl = reinterpret_cast<const unsigned char*>(sg) + 8 * lane;  // this lane's 2 columns
    const int4* hdr = reinterpret_cast<const int4*>(blob);
#ifdef GASB_BWD_TIMING
    const int cta = 256 + blockIdx.x + gridDim.x * blockIdx.y;
    if (threadIdx.x == 0 && cta < 512) {
        g_bwd_stamps[cta * 4] = bwd_now();
        g_bwd_stamps[cta * 4 + 2] = 0;
    }
#endif
    for (int32_t q = 0; q < phases; ++q) {
        if (q > 0) {
            __syncthreads();  // every warp is done with the previous phase's slice and blob
            if (threadIdx.x == 0) {
                *s_next = 0;  // (published by the mbarrier arrive below)
                expect_and_issue_blob(q);
                issue_slice(q);
            }
        }
        mbar_wait(bar, static_cast<uint32_t>(q & 1));
#ifdef GASB_BWD_TIMING
        if (threadIdx.x == 0 && cta < 512 && q < 2) g_bwd_stamps[cta * 4 + 1 + 2 * q] = bwd_now();
#endif
        const bool last_phase = q + 1 == phases;
        const int32_t ntq = hdr[0].x;
#ifdef GASB_BWD_TIMING
        unsigned long long w_ent = 0, w_tg = 0;
        const unsigned long long w_t0 = bwd_now();
#endif
        for (;;) {
            int32_t k = 0;
            if (lane == 0) k = atomicAdd(s_next, 1);
            k = __shfl_sync(0xffffffffu, k, 0);
            if (k >= ntq) break;
            const int4 d = hdr[1 + k];  // {target, entry offset (bytes, in the blob), entries, slot}
            const int32_t t = d.x;
            float* gp = gx + static_cast<int64_t>(t) * ldgx + c;
            float2 mv = make_float2(1.0f, 1.0f);
            if (last_phase && mask) {  // issued now, used after the entries
                const float* mp = mask + static_cast<int64_t>(t) * ldm + c;
                if (vec_m && has1) mv = *reinterpret_cast<const float2*>(mp);
                else {
                    if (has0) mv.x = mp[0];
                    if (has1) mv.y = mp[1];
                }
            }
            float2 a = make_float2(0.0f, 0.0f);
            if (q > 0) a = run[d.w * 32 + lane];
            else if (accumulate) {
                if (vec_gx && has1) a = *reinterpret_cast<const float2*>(gp);
                else {
                    if (has0) a.x = gp[0];
                    if (has1) a.y = gp[1];
                }
            }
            uint64_t acc = (static_cast<uint64_t>(__float_as_uint(a.y)) << 32) | __float_as_uint(a.x);
            const int4* ent = reinterpret_cast<const int4*>(blob + d.y);  // 2 entries per int4
#ifdef GASB_BWD_TIMING
            w_ent += d.z;
            ++w_tg;
#endif
            // 8 entries per step, software-pipelined: the next step's metadata is loaded while this
            // step's source values are loaded and multiplied (the products are independent; only
            // the adds form the ordered chain)
            int4 m[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) m[u] = ent[u];
            for (int32_t j = 0; j < d.z; j += 8) {
                uint64_t x[8];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    x[2 * u] = *reinterpret_cast<const uint64_t*>(sgl + m[u].x);
                    x[2 * u + 1] = *reinterpret_cast<const uint64_t*>(sgl + m[u].z);
                }
                float cf[8];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    cf[2 * u] = __int_as_float(m[u].y);
                    cf[2 * u + 1] = __int_as_float(m[u].w);
                }
                if (j + 8 < d.z) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) m[u] = ent[((j + 8) >> 1) + u];
                }
                uint64_t pr[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) pr[v] = f2_mulz(cf[v], x[v], negz);
#pragma unroll
                for (int v = 0; v < 8; ++v) acc = f2_add(acc, pr[v]);
            }
            float2 r;
            r.x = __uint_as_float(static_cast<uint32_t>(acc));
            r.y = __uint_as_float(static_cast<uint32_t>(acc >> 32));
            if (!last_phase) {
                run[d.w * 32 + lane] = r;
                continue;
            }
            if (!(mv.x > 0.0f)) r.x = 0.0f;
            if (!(mv.y > 0.0f)) r.y = 0.0f;
            if (vec_gx && has1) *reinterpret_cast<float2*>(gp) = r;
            else {
                if (has0) gp[0] = r.x;
                if (has1) gp[1] = r.y;
            }
        }
#ifdef GASB_BWD_TIMING
        if (lane == 0 && cta < 512 && q == 0) atomicMax(&g_bwd_stamps[cta * 4 + 2], bwd_now());
        if (lane == 0 && q == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
            const int w = threadIdx.x >> 5;
            g_bwd_warp[w * 3] = w_ent;
            g_bwd_warp[w * 3 + 1] = w_tg;
            g_bwd_warp[w * 3 + 2] = bwd_now() - w_t0;
        }
#endif
    }
#ifdef GASB_BWD_TIMING
    __syncthreads();
    if (threadIdx.x == 0 && cta < 512) g_bwd_end[cta] = bwd_now();
#endif
}

int32_t spmm_bwd2_splits(int32_t dim) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms = 148;
    return std::max<int32_t>(1, sms / static_cast<int32_t>(ceil_div(dim, kBwd2CW)));
}

// Blobs of one part: targets t = 0 .. nt-1 dealt round-robin to `splits` CTAs (t mod splits);
// per (split, phase): int4 {targets, 0, 0, 0}, then per target (heaviest first) int4
// {t, entry offset in bytes from the blob start, entries, 0}, then the entries as int2
// {byte offset of the source row in the staged slice, coefficient bits}, per target padded to a
// multiple of 8. Appends to blobs (16 B aligned) and to off (splits * phases offsets, plus the
// end offset when `last`). Returns false if some blob exceeds the shared-memory budget.
bool build_bwd2_plan(const int64_t* trp, const int32_t* tsrc, const float* tcf, int32_t nt, int32_t nsrc,
                     int32_t splits, std::vector<int64_t>& off, std::vector<unsigned char>& blobs) {
    const int32_t phases = std::max<int32_t>(1, static_cast<int32_t>(ceil_div(nsrc, kBwd2Rows)));
    const int2 pad{kBwd2Rows * kBwd2CW * 4, static_cast<int>(0x80000000u)};
    bool ok = phases <= kBwd2MaxPhases && ceil_div(nt, splits) <= kBwd2Slots;
    std::vector<int64_t> split_at(static_cast<size_t>(nt) * (phases + 1));  // per target: phase boundaries
    for (int32_t t = 0; t < nt; ++t) {
        int64_t e = trp[t];
        for (int32_t q = 0; q <= phases; ++q) {
            const int32_t lo = q * kBwd2Rows;
            while (e < trp[t + 1] && tsrc[e] < lo) ++e;
            split_at[static_cast<size_t>(t) * (phases + 1) + q] = q == phases ? trp[t + 1] : e;
        }
    }
    for (int32_t s = 0; s < splits; ++s)
        for (int32_t q = 0; q < phases; ++q) {
            std::vector<int32_t> ts;
            for (int32_t t = s; t < nt; t += splits) ts.push_back(t);
            auto cnt_of = [&](int32_t t) {
                return split_at[static_cast<size_t>(t) * (phases + 1) + q + 1] - split_at[static_cast<size_t>(t) * (phases + 1) + q];
            };
            std::stable_sort(ts.begin(), ts.end(), [&](int32_t a, int32_t b) { return cnt_of(a) > cnt_of(b); });
            const size_t b0 = blobs.size();
            off.push_back(static_cast<int64_t>(b0));
            const size_t hdr_bytes = 16 * (ts.size() + 1);
            blobs.resize(b0 + hdr_bytes, 0);
            int32_t h0[4] = {static_cast<int32_t>(ts.size()), 0, 0, 0};
            std::memcpy(blobs.data() + b0, h0, 16);
            for (size_t k = 0; k < ts.size(); ++k) {
                const int32_t t = ts[k];
                const int64_t e0 = split_at[static_cast<size_t>(t) * (phases + 1) + q], e1 = e0 + cnt_of(t);
                const int64_t n8 = (e1 - e0 + 7) / 8 * 8;
                int32_t h[4] = {t, static_cast<int32_t>(blobs.size() - b0), static_cast<int32_t>(n8), t / splits};
                std::memcpy(blobs.data() + b0 + 16 * (k + 1), h, 16);
                for (int64_t i = 0; i < n8; ++i) {
                    int2 m = pad;
                    if (e0 + i < e1) {
                        m.x = (tsrc[e0 + i] - q * kBwd2Rows) * kBwd2CW * 4;
                        std::memcpy(&m.y, &tcf[e0 + i], 4);
                    }
                    const size_t at = blobs.size();
                    blobs.resize(at + 8);
                    std::memcpy(blobs.data() + at, &m, 8);
                }
            }
            if (blobs.size() - b0 > static_cast<size_t>(kBwd2BlobBytes)) ok = false;
        }
    return ok;
}

static int g_bwd2_smem_set = 0;

bool launch_spmm_bwd2(const int64_t* blob_off, const unsigned char* blobs, int32_t splits, const float* gy,
                      int64_t ldgy, int32_t dim, const float* mask, int64_t ldm, float* gx, int64_t ldgx,
                      cudaStream_t st, int32_t nsrc, bool accumulate) {
    if (dim < kBwd2CW || (ldgy * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(gy) & 15) != 0) return false;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult qr;
        void* fn = nullptr;
        GASB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
        require(qr == cudaDriverEntryPointSuccess && fn, "spmm_bwd2: cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    CUtensorMap map{};
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(nsrc)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ldgy) * 4};
    const cuuint32_t box[2] = {kBwd2CW, kBwd2Box};
    const cuuint32_t es[2] = {1, 1};
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gy), gdim, gstride, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (!g_bwd2_smem_set) {
        GASB_CUDA(cudaFuncSetAttribute(spmm_bwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwd2Smem));
        g_bwd2_smem_set = 1;
    }
    const int32_t phases = std::max<int32_t>(1, static_cast<int32_t>(ceil_div(nsrc, kBwd2Rows)));
    const int32_t nchunks = static_cast<int32_t>(ceil_div(dim, kBwd2CW));
    const uint64_t negz = 0x8000000080000000ull;
    launch_pdl(spmm_bwd2_kernel, dim3(static_cast<unsigned>(nchunks), static_cast<unsigned>(splits)),
               dim3(kBwd2Threads), kBwd2Smem, st, blob_off, blobs, phases, nsrc, dim, mask, ldm, gx, ldgx,
               accumulate ? 1 : 0, negz, map);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
    return true;
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
        std::vector<int64_t> rp64(static_cast<size_t>(m) + 1), sb;
        for (int32_t r = 0; r <= m; ++r) {
            require(r == 0 || rp[r] >= rp[r - 1], "aggregate: row pointer not monotone");
            rp64[r] = rp[r];
        }
        std::vector<int32_t> sr, ss, r0(static_cast<size_t>(m)), rn(static_cast<size_t>(m));
        const int32_t nranges = spmm_ranges_per_launch();
        std::vector<int32_t> rs(static_cast<size_t>(nranges) + 1);
        int64_t slot64 = 0;
        segment_launch(rp64.data(), 0, m, seg_edges > 0, nranges, sb, sr, ss, r0.data(), rn.data(), slot64, rs.data());
        const int64_t slots = slot64;
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
        GASB_CUDA(cudaMallocAsync(&z.partial, sizeof(double) * std::max<int64_t>(slots, 1) * round_up(dim, 256), st));
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
            int32_t* d_rs = nullptr;
            GASB_CUDA(cudaMallocAsync(&d_rs, sizeof(int32_t) * (nranges + 1), st));
            GASB_CUDA(cudaMemcpyAsync(d_rs, rs.data(), sizeof(int32_t) * (nranges + 1), cudaMemcpyHostToDevice, st));
            SpmmSegs segs{z.seg_beg, z.seg_row, z.seg_slot, z.row_seg0, z.row_nseg, d_rs, nranges};
            CUtensorMap tm;
            const bool have_tm = make_row_tmap(d_x, num_src, dim, ldx, spmm_box_cols(dim), &tm);
            launch_spmm_fwd(segs, d_cols, coeffs64, d_x, ldx, dim, d_y, ldy, 0, z.partial,
                            round_up(dim, 256), z.counters, nchunks, st, special, have_tm ? &tm : nullptr);
            GASB_CUDA(cudaStreamSynchronize(st));
            cudaFreeAsync(special, st);
            cudaFreeAsync(d_rs, st);
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
