// Device kernels of the GAS hot path (sm_100a). Declarations of launch helpers shared
// between translation units; the kernels live in history.cu, spmm.cu, gemm.cu, train_ops.cu.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace gasb {

constexpr int kWarp = 32;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Counts kernel launches issued through these helpers (gpu_launches evidence).
extern thread_local int64_t t_launches;

// Programmatic dependent launch (PDL). The kernels of the per-batch chain are launched with
// programmatic stream serialization: the next kernel's grid is set up, and its CTAs become
// resident as SMs free up (running any prologue that touches no global memory), while this
// one drains. Every kernel launched this way calls pdl_wait() in every CTA before its first
// global-memory access. pdl_wait() returns once the preceding grid has completed and its
// writes are visible, so the chain stays transitively ordered. pdl_trigger() lets the
// dependent grid launch. Both are no-ops for a normal launch. Opt-in (GASB_PDL=1): measured
// no faster at C3 (the per-batch graph's launch gaps are already small), GPU suite green with it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
bool pdl_enabled();
void check_launch(cudaError_t e, const char* what);
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    check_launch(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "launch_pdl");
}

// Per-table value flags (device int32, OR-accumulated by every producer of a table that the
// SpMM reads): they pick the fp32 -> fp64 widening path of the forward SpMM (spmm.cu).
constexpr int32_t kTableNeg = 1;        // some value has its sign bit set
constexpr int32_t kTableNonFinite = 2;  // some value is inf / nan
// Coefficients of the forward SpMM are stored multiplied by 2^896 (exact; see spmm.cu).
constexpr double kCoeffScale = 0x1.0p+896;

__host__ __device__ inline int32_t table_flag_of(float v) {
#ifdef __CUDA_ARCH__
    const uint32_t u = __float_as_uint(v);
#else
    uint32_t u;
    __builtin_memcpy(&u, &v, 4);
#endif
    return ((u >> 31) ? kTableNeg : 0) | (((u & 0x7fffffffu) >= 0x7f800000u) ? kTableNonFinite : 0);
}

// ---- history rows (history.cu) ------------------------------------------------------
// mode 0 = push: dst[ids[i]] = src[i] (+ stamps[ids[i]] = *step); mode 1 = pull: dst[i] = src[ids[i]].
// flags (push only, optional): the destination table's value-flag word.
void launch_rows(int mode, const int32_t* ids, int64_t count, const float* src, int64_t lds, float* dst,
                 int64_t ldd, int32_t dim, int32_t n, int64_t* stamps, const int64_t* step, int32_t* err,
                 cudaStream_t st, int32_t* flags = nullptr);
void launch_advance_step(int64_t* step, cudaStream_t st);

// ---- SpMM (spmm.cu) -------------------------------------------------------------------
// Segmented CSR SpMM with fp64 accumulation. Segments tile the edge range of the rows they
// cover in row order: segment s = edges [seg_beg[s], seg_beg[s+1]) of row seg_row[s] (rows
// absolute; the output row is seg_row[s] - row_base). Rows with more than one segment
// combine fp64 partials in segment order (slot[s] >= 0 indexes `partial`, counters are
// per (row, chunk) and self-reset).
struct SpmmSegs {
    const int64_t* seg_beg;   // nseg + 1, absolute edge offsets
    const int32_t* seg_row;   // nseg
    const int32_t* seg_slot;  // nseg: partial slot or -1 (single-segment row)
    const int32_t* row_seg0;  // per absolute row: first segment index (only multi-seg rows)
    const int32_t* row_nseg;  // per absolute row: number of segments
    const int32_t* range_seg; // nranges + 1 segment boundaries of this launch (split_ranges)
    int32_t nranges;
    // 1: one fp64 chain per column in CSR order (the bit-exact sequential mode); 0: rows may
    // be split anyway, so each row also runs two interleaved chains (even / odd edges of the
    // stage) added at the row end — twice the independent DFMAs, same fp64 accuracy class
    int32_t exact = 1;
    // optional: per row, the partial slots of its segments in combine order, indexed from
    // row_seg0[row] (tables whose rows' segments are not consecutive: the source-blocked
    // hoisted layer 1); nullptr: the row's segments are consecutive, seg_slot[row_seg0 + i]
    const int32_t* row_slots = nullptr;
};
// Host: splits segments [g0, g1) into nranges contiguous ranges of ~equal edges.
void split_ranges(const int64_t* seg_beg, int64_t g0, int64_t g1, int32_t nranges, int32_t* out);
// Host: segments + nranges+1 work ranges of one launch over rows [r_lo, r_hi) (spmm.cu).
// Appends to sb/sr/ss (plus a trailing sentinel in sb), fills r0/rn of those rows.
void segment_launch(const int64_t* rp, int64_t r_lo, int64_t r_hi, bool split, int32_t nranges,
                    std::vector<int64_t>& sb, std::vector<int32_t>& sr, std::vector<int32_t>& ss, int32_t* r0,
                    int32_t* rn, int64_t& slot, int32_t* ranges);
// Work ranges per SpMM launch: 8 resident warps per SM (2 CTAs of 4).
int32_t spmm_ranges_per_launch();
// coeffs: stencil coefficients as fp64 pre-multiplied by kCoeffScale. special: the source
// table's flag word (kTableNeg / kTableNonFinite); nullptr = assume anything (exact F2F).
// tmap (optional): tensor map of x for TMA tile::gather4 staging (make_row_tmap with
// box_cols = spmm_box_cols()); nullptr = cp.async staging.
void launch_spmm_fwd(const SpmmSegs& s, const int32_t* cols, const double* coeffs, const float* x, int64_t ldx,
                     int32_t dim, float* y, int64_t ldy, int64_t row_base, double* partial, int64_t partial_ld,
                     int32_t* counters, int32_t counters_ld, cudaStream_t st, const int32_t* special = nullptr,
                     const CUtensorMap* tmap = nullptr);
// Caps the grid of this thread's flat SpMM launches at `ctas` CTAs (0: the full persistent
// grid). Work items are grid-strided, so a capped launch does the same work on fewer SMs.
void set_spmm_grid_cap(int32_t ctas);
// Row-sum hand-off for this thread's next flat SpMM launches (reset with nullptrs): out: each
// finished row's fp64 sum is written to out[row - row_base] (ld doubles per row) instead of
// the fp32 row; in: the fp32 row stored is float(sum + in[row - row_base]).
void set_spmm_row_sums(double* out, const double* in, int64_t ld);
bool make_row_tmap(const float* base, int64_t rows, int32_t dim, int64_t ld, int32_t box_cols, CUtensorMap* out);
int32_t spmm_box_cols(int32_t dim);
int32_t spmm_cpl_for(int32_t dim);
// special[0] |= table_flag_of(v) over the values v of x[rows x dim] (pitch ld).
void launch_scan_special(const float* x, int64_t rows, int64_t ld, int32_t dim, int32_t* special, cudaStream_t st);
// Transposed (CSC) gather, fp32 multiply-then-add in entry order (bit-exact with the
// reference scatter). mask (optional): zero where mask <= 0 (relu backward).
// accumulate: gx[t] continues from its current value (the reference's `g += c * gy` into
// a grad buffer that already holds other contributions) instead of starting at 0.
// order (optional): the targets heaviest first (claimed in that order, so a hub's serial
// chain starts early instead of setting the tail).
void launch_spmm_bwd(const int64_t* t_rowptr, int32_t ntargets, const int32_t* t_src, const float* t_coeffs,
                     const float* gy, int64_t ldgy, int32_t dim, const float* mask, int64_t ldm, float* gx,
                     int64_t ldgx, cudaStream_t st, int32_t nsrc = 0, bool accumulate = false,
                     const int32_t* order = nullptr);

// Two-columns-per-lane variant (spmm.cu, spmm_bwd2_kernel): same results, bit for bit, over
// a per-(CTA split, source phase) plan of one part (build_bwd2_plan; false if a blob would
// not fit shared memory). launch_spmm_bwd2 returns false (nothing launched) when dim < 64 or
// gy cannot be described to TMA; callers then use launch_spmm_bwd.
int32_t spmm_bwd2_splits(int32_t dim);
bool build_bwd2_plan(const int64_t* trp, const int32_t* tsrc, const float* tcf, int32_t nt, int32_t nsrc,
                     int32_t splits, std::vector<int64_t>& off, std::vector<unsigned char>& blobs);
bool launch_spmm_bwd2(const int64_t* blob_off, const unsigned char* blobs, int32_t splits, const float* gy,
                      int64_t ldgy, int32_t dim, const float* mask, int64_t ldm, float* gx, int64_t ldgx,
                      cudaStream_t st, int32_t nsrc, bool accumulate = false);

// ---- GEMM (gemm.cu) -------------------------------------------------------------------
// op 0: C = A B ; 1: C = A B^T ; 2: C = A^T B.  Row-major fp32, fp32 accumulation.
// History push fused into the epilogue (op 0 only): rows also scattered to
// table[ids[i]] with stamps and the table's value flags.
struct PushEpilogue {
    float* table;
    int64_t ld;
    const int32_t* ids;
    int64_t* stamps;
    const int64_t* step;
    int32_t* special;  // the table's value flags: OR of table_flag_of(pushed values)
};
// Epilogue applied to each rounded fp32 result x, in the reference's op order (each step
// one fp32 rounding, no contraction):
//   x = x * post_scale   (scale(), tensor.cpp:254-275; 1 = skip)
//   x = x + beta * C     (gradient accumulation; beta is 0 or 1)
//   x = x + bias[col]    (add_rowvec, tensor.cpp:277-307; nullptr = skip)
//   x = relu(x)          (tensor.cpp:355-372)
//   C = x; push (table != nullptr)
struct GemmEpilogue {
    float beta = 0.f;
    float post_scale = 1.f;
    const float* bias = nullptr;
    int relu = 0;
    PushEpilogue push{};
};
void launch_gemm(int op, int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                 int64_t ldc, const GemmEpilogue& ep, cudaStream_t st);
// Split-K scratch for the tensor-core GEMM on this host thread (nullptr: no split-K). GEMMs
// enqueued afterwards on ONE stream may share it (they run in order). The buffer holds
// `floats` floats followed by kGemmTileCounters ints that must be zero initially.
constexpr int64_t kGemmTileCounters = 1024;
constexpr int64_t kGemmWsFloats = 148LL * 128 * 64 + 4096;
// serial_fixup: the last slice of a tile to arrive reduces it (no CTA waits, so any number of
// split-K grids may run concurrently); otherwise every slice CTA waits for its peers and
// reduces 1/S of the tile — faster, but only one such grid may be in flight at a time.
void set_gemm_workspace(float* ws, int64_t floats, bool serial_fixup = false);
void launch_gemm(int op, int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                 int64_t ldc, float beta, bool relu, const PushEpilogue* push, cudaStream_t st);
__device__ __forceinline__ float gemm_epilogue_value(const GemmEpilogue& ep, float x, const float* crow, int col) {
    if (ep.post_scale != 1.f) x = __fmul_rn(x, ep.post_scale);
    if (ep.beta != 0.f) x = __fadd_rn(x, crow[col]);
    if (ep.bias) x = __fadd_rn(x, ep.bias[col]);
    if (ep.relu) x = x > 0.f ? x : 0.f;
    return x;
}

// ---- training ops (train_ops.cu) ---------------------------------------------------
// Softmax cross-entropy over the training rows (row_label[i] >= 0; r of them) of an m-row
// batch: loss (double, written to *loss_out) and d loss / d logits into glogits (zero rows
// elsewhere), as tensor.cpp:597-647. row_scratch: m doubles; done: self-resetting counter.
void launch_softmax_ce(const float* logits, int64_t ldl, int32_t m, int32_t n, const int32_t* row_label, int32_t r,
                       float* glogits, int64_t ldg, double* loss_out, double* row_scratch, int32_t* done,
                       cudaStream_t st);
// AdamState::step (nn.cpp:20-41) over the flat parameter vector; bias corrections from
// bc[2*t], t = ++(*t_counter) on device. clip_max_norm > 0 applies grad_clip first.
// end_step (optional): the end of the batch fused in — the last block advances *end_step and
// *t_counter (end_done: a zero-initialised, self-resetting int).
void launch_adam(float* p, float* m, float* v, float* g, int64_t size, int64_t* t_counter, const double* bc,
                 float lr, float b1, float b2, float eps, float clip_max_norm, double* norm_scratch,
                 cudaStream_t st, int64_t* end_step = nullptr, int32_t* end_done = nullptr);
void launch_zero(float* p, int64_t count, cudaStream_t st);
// dropout (tensor.cpp:374-401) with bit-word keep masks over the row-major rows x dim input
void launch_dropout_apply(float* x, int64_t ldx, int64_t rows, int32_t dim, const uint32_t* mask, float inv_keep,
                          cudaStream_t st);
void launch_dropout_rows_bwd(float* g, int64_t ldg, int32_t m, int32_t dim, const int32_t* rows, const uint32_t* mask,
                             float inv_keep, cudaStream_t st);
void launch_philox_mask(uint32_t* mask, int64_t count, uint64_t key, float p, cudaStream_t st);
void launch_dropout_bwd_acc(float* g, int64_t ldg, int64_t rows, int32_t dim, const float* gin, int64_t ldi,
                            const uint32_t* mask, float inv_keep, cudaStream_t st);
// l2_penalty (tensor.cpp:649-678): g += 2 w p (before clip / Adam), *loss = float(*loss) + float(w sum p^2).
// scratch: kNormBlocks doubles.
void launch_l2_penalty(const float* p, float* g, int64_t size, float w, double* loss, double* scratch,
                       cudaStream_t st);

// ---- residual models: APPNP / GCNII (residual.cu) ---------------------------------------
// out[i] = alpha * h0[rows[i]] + (1 - alpha) * prop[i]  (+ optional history push of out)
void launch_mix(const float* h0, int64_t ldh0, const int32_t* rows, const float* prop, int64_t ldp, int32_t m,
                int32_t d, float alpha, float* out, int64_t ldo, const PushEpilogue* push, cudaStream_t st);
// wt[l] = (1 - beta) I + beta W[l], l < layers (d x d each, row pitch `pitch`)
void launch_wtilde(const float* w, float* wt, int32_t layers, int32_t d, int64_t pitch, float beta,
                   cudaStream_t st);
// dprop = (1 - alpha) dmix ; h0g[rows[i]] += alpha dmix[i]
void launch_mix_bwd(const float* dmix, int64_t ldd, int32_t m, int32_t d, float alpha, const int32_t* rows,
                    float* h0g, int64_t ldh, float* dprop, int64_t ldp, cudaStream_t st);
// out[j] = float(sum_i double(g[i, j]))
void launch_colsum(const float* g, int64_t ldg, int32_t m, int32_t n, float* out, cudaStream_t st);
// fp64 row-block partials for launch_colsum on this host thread (nullptr: single-level sum)
void set_colsum_workspace(double* ws, int64_t doubles);
constexpr int64_t kColsumWsDoubles = 148LL * 8 * 1024;
// g = mask > 0 ? g : 0
void launch_mask(float* g, int64_t ldg, const float* mask, int64_t ldm, int32_t m, int32_t n, cudaStream_t st);

}  // namespace gasb
