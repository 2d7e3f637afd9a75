// Dense feature transform (the reference's matmul, src/tensor.cpp:148-204) on the 5th-gen
// tensor cores: tcgen05.mma kind::tf32 with fp32 accumulators in TMEM, operands staged by
// TMA (128 B swizzle), 3xTF32 split for fp32-level accuracy (the reference accumulates in
// fp64; plain TF32 misses the 1e-5 normwise bound, 3xTF32 meets it — SURVEY §7.6).
//
//   op 0: C[m,n] = A[m,k] B[k,n]    (A K-major, B MN-major)   forward  X·W
//   op 1: C[m,n] = A[m,k] B[n,k]^T  (A K-major, B K-major)    dgrad    dY·W^T
//   op 2: C[m,n] = A[k,m]^T B[k,n]  (A MN-major, B MN-major)  wgrad    X^T·dY
//
// CTA = one 128 x BN output tile:
//   warp 4 (1 thread)   TMA producer: fp32 A/B tiles of BK=32 into a 3-stage ring
//   warps 0-3, 6-7      split each landed tile in place into hi = tf32(x) and lo = x - hi (exact)
//   warp 5 (1 thread)   MMA issuer: per k-step of 8, D += Ahi.Bhi + Ahi.Blo + Alo.Bhi
//   warps 8-11          drain: sum each accumulator group out of TMEM as soon as it is final,
//                       then the epilogue (staged through shared memory, coalesced stores)
//   (TALL kernels, 2 CTAs/SM: no drain warps; warps 0-3 drain and store after the mainloop)
// mbarriers: full (TMA -> split), split (split -> MMA), empty (tcgen05.commit -> TMA),
// accready[g] (group g's last commit -> drain). Waits are bounded (trap instead of hang).
#include <cstdlib>

#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {

// Workspace layout: ws_floats floats of slice partials, then kGemmTileCounters ints of
// per-tile arrival counters (zero-initialised by the owner, self-resetting).
thread_local float* t_gemm_ws = nullptr;
thread_local int64_t t_gemm_ws_floats = 0;
thread_local bool t_gemm_serial = false;
void set_gemm_workspace(float* ws, int64_t floats, bool serial_fixup) {
    t_gemm_ws = ws;
    t_gemm_ws_floats = ws ? floats : 0;
    t_gemm_serial = serial_fixup;
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        GASB_CUDA(cudaGetDevice(&dev));
        GASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return sms;
}

#ifdef GASB_GEMM_TIMING
__device__ uint64_t g_gemm_stamps[40 + 2 * 256];  // + per-CTA (x + gridDim.x * y) start / end
extern "C" void gasb_debug_gemm_stamps(uint64_t* out) {
    cudaMemcpyFromSymbol(out, g_gemm_stamps, sizeof(uint64_t) * (40 + 2 * 256));
}
#endif
namespace tc {

#ifndef GASB_GEMM_STAGES
#define GASB_GEMM_STAGES 3
#endif
#ifndef GASB_GEMM_MAXACC
#define GASB_GEMM_MAXACC 8
#endif
constexpr int BM = 128, BK = 32, kStagesTC = GASB_GEMM_STAGES;
#ifndef GASB_GEMM_SPLIT_HELPERS
#define GASB_GEMM_SPLIT_HELPERS 2  // 4 measured slower with the drain warps (14 warps cap registers at 128)
#endif
#ifndef GASB_GEMM_KSTEPS_PER_ACC
#define GASB_GEMM_KSTEPS_PER_ACC 1  // 16 cut the epilogue 3.8 -> 2.7 us but broke the 64-layer GCNII contract
#endif
constexpr int kSplitHelpers = GASB_GEMM_SPLIT_HELPERS;  // extra warps that only split tiles
constexpr int kSplitThreads = 128 + 32 * kSplitHelpers;  // warps 0-3 + helpers
// non-TALL kernels add 4 drain warps (6 + kSplitHelpers ..): they sum each accumulator out of
// TMEM as soon as the tensor core finishes it, concurrently with the split warps' shared-memory
// work, then run the epilogue. TALL kernels (2 CTAs/SM, ~100 registers) have warps 0-3 drain
// everything after the mainloop instead.
template <bool TALL>
__host__ __device__ constexpr int threads_of() {
    return 192 + 32 * kSplitHelpers + (TALL ? 0 : 128);
}
template <bool TALL>
__host__ __device__ constexpr int alloc_warp() {  // the warp that allocates (and frees) TMEM: an epilogue warp
    return TALL ? 0 : 6 + kSplitHelpers;
}
// The tensor core's fp32 accumulation truncates, so its error grows linearly with the number
// of k-steps; k-steps are interleaved over kAcc TMEM accumulators (kAcc * BN <= 512 columns)
// summed round-to-nearest in the epilogue, cutting that growth kAcc-fold.
// TALL variant (many output tiles, short K: e.g. the APPNP/GCNII heads over every V_b row):
// 2 stages and 4 accumulators so two CTAs share an SM (shared memory and TMEM), overlapping
// one CTA's epilogue with the other's mainloop.
template <int BN, bool TALL = false>
struct Acc {
    static constexpr int kMax = TALL ? 4 : GASB_GEMM_MAXACC;
    static constexpr int kAcc = 512 / BN < kMax ? 512 / BN : kMax;
    static constexpr int kCols = kAcc * BN;  // TMEM allocation (power of two)
};
template <bool TALL>
constexpr int stages_of() {
    return TALL ? 2 : kStagesTC;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    for (uint32_t spins = 0;; ++spins) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(su32(b)), "r"(parity)
            : "memory");
        if (done) return;
        if (spins > (1u << 26)) __trap();
    }
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int32_t c0, int32_t c1, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(su32(b))
        : "memory");
}

// UMMA shared-memory descriptor, version 1 (sm_100). layout 2 = SWIZZLE_128B (K-major
// operands); layout 1 = SWIZZLE_128B_BASE32B (32 B atoms), the only smem layout the tensor
// core accepts for MN-major tf32 operands.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

// Instruction descriptor: D f32, A/B tf32, majors, N, M = 128.
__host__ __device__ constexpr uint32_t instr_desc(int n, bool a_mn, bool b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b))
                 : "memory");
}

// round-to-nearest tf32 (low 13 mantissa bits zero) and the exact remainder
__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// truncated tf32: what the tensor core reads from an fp32 operand
__device__ __forceinline__ float tf32_tr(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
#ifndef GASB_GEMM_TRUNC_SPLIT
#define GASB_GEMM_TRUNC_SPLIT 0  // measured no faster: the mainloop is bound by shared-memory traffic overall
#endif

template <int BN, bool A_MN, bool B_MN, bool TALL = false>
struct Layout {
    static constexpr int kStages = stages_of<TALL>();
    static constexpr int kTileA = BM * BK * 4;  // bytes (16 KB)
    static constexpr int kTileB = BN * BK * 4;
    // stage: A, A_lo, B, B_lo (each 1024 B aligned: SW128 atoms)
    static constexpr int kStage = 2 * kTileA + 2 * kTileB;
    static constexpr int kBars = 8 * (3 * kStages + GASB_GEMM_MAXACC);
    static constexpr int kSmem = 1024 + kStages * kStage + kBars + 16;
};

template <int BN, bool A_MN, bool B_MN, bool TALL>
__global__ void __launch_bounds__(threads_of<TALL>(), TALL ? 2 : 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a,
                                                             const __grid_constant__ CUtensorMap tma_b, int M,
                                                             int N, int K, float* __restrict__ C, int64_t ldc,
                                                             GemmEpilogue ep, int kbs, float* __restrict__ ws,
                                                             int64_t ws_floats, int serial_fixup,
                                                             int acc_groups) {
    const PushEpilogue& push = ep.push;
    using Lay = Layout<BN, A_MN, B_MN, TALL>;
    constexpr int kStagesTC = Lay::kStages;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~1023ull);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + kStagesTC * Lay::kStage);
    uint64_t* full = bars;
    uint64_t* split = bars + kStagesTC;
    uint64_t* empty = bars + 2 * kStagesTC;
    uint64_t* accready = bars + 3 * kStagesTC;  // one per accumulator group: its last MMA completed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kStagesTC + Acc<BN, TALL>::kAcc);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
#ifdef GASB_GEMM_TIMING  // globaltimer stamps of CTA (0,0) into g_gemm_stamps (timing probe builds only)
    auto stamp = [&](int i) {
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            g_gemm_stamps[i] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);
#ifdef GASB_GEMM_TIMING
    const int cta_id = blockIdx.x + gridDim.x * blockIdx.y;
    if (threadIdx.x == 0 && blockIdx.z == 0 && cta_id < 256) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_gemm_stamps[40 + 2 * cta_id] = t;
    }
#endif
#else
    auto stamp = [](int) {};
#endif
    // split-K: this CTA covers k-blocks [kb0, kb0 + nk) (blockIdx.z = slice); with ws != nullptr
    // it writes its raw fp32 sums to ws[slice] and gemm_splitk_reduce applies the epilogue.
    const int kb0 = blockIdx.z * kbs;
    const int nk = min((K + BK - 1) / BK - kb0, kbs);
    // accumulators in use: one per GASB_GEMM_KSTEPS_PER_ACC k-steps (the fp32 accumulation
    // error grows with the k-steps an accumulator sums), at most Acc::kAcc; fewer accumulators
    // mean fewer TMEM reads in the epilogue
    const int nacc = min(Acc<BN, TALL>::kAcc, max(1, (nk * (BK / 8) + GASB_GEMM_KSTEPS_PER_ACC - 1) /
                                                         GASB_GEMM_KSTEPS_PER_ACC));
    // Accumulator groups: the k-steps are cut into `ng` contiguous blocks, and the k-steps of
    // block j are interleaved over the accumulators of group j (nacc / ng of them: consecutive
    // MMAs then write different accumulators, which keeps the tensor core's pipeline full).
    // A group is final once its last k-step's MMAs complete, so the drain warps sum it out of
    // TMEM (in accumulator order) while later groups are still in the tensor core, instead of
    // reading every accumulator after the last MMA (TMEM reads run at ~64 B/clk).
    const int nsteps_all = nk * (BK / 8);
    const int ng = (acc_groups > 0 && nacc % acc_groups == 0) ? acc_groups : 1;
    const int per_g = nacc / ng;
    auto group_first = [&](int j) { return (j * nsteps_all + ng - 1) / ng; };  // first k-step of block j

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesTC; ++s) {
            bar_init(full + s, 1);
            bar_init(split + s, kSplitThreads);
            bar_init(empty + s, 1);
        }
        for (int q = 0; q < Acc<BN, TALL>::kAcc; ++q) bar_init(accready + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == alloc_warp<TALL>()) {  // TMEM: kAcc accumulators of BN fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                     "r"(Acc<BN, TALL>::kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();
    pdl_wait();  // (PDL) the setup above touched no global memory; A and C belong to earlier kernels
    if (threadIdx.x == 0) stamp(1);

    const bool drainer = !TALL && warp >= 6 + kSplitHelpers;
    const int etid = (warp & 3) * 32 + lane;  // epilogue thread: TMEM lane == tile row
    if (warp == 4) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kStagesTC;
                bar_wait(empty + s, ((kb / kStagesTC) & 1) ^ 1);
                if (kb < 8) stamp(24 + kb);
                unsigned char* st = base + s * Lay::kStage;
                bar_expect(full + s, Lay::kTileA + Lay::kTileB);
                const int k0 = (kb0 + kb) * BK;
                if (A_MN) {  // A^T tile: K rows x 128 MN cols as 4 boxes of 32 cols
                    for (int j = 0; j < BM / 32; ++j) tma_2d(st + j * BK * 128, &tma_a, m0 + 32 * j, k0, full + s);
                } else {
                    tma_2d(st, &tma_a, k0, m0, full + s);
                }
                unsigned char* sb = st + 2 * Lay::kTileA;
                if (B_MN) {
                    for (int j = 0; j < BN / 32; ++j) tma_2d(sb + j * BK * 128, &tma_b, n0 + 32 * j, k0, full + s);
                } else {
                    tma_2d(sb, &tma_b, k0, n0, full + s);
                }
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = instr_desc(BN, A_MN, B_MN);
            // (group, position in group) tracked incrementally: the single issuing thread is on
            // the critical path, so no divisions per k-step
            int j = 0, r = 0, rq = 0, gnext = group_first(1);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kStagesTC;
                bar_wait(split + s, (kb / kStagesTC) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t sa = su32(base + s * Lay::kStage);
                const uint32_t sa_lo = sa + Lay::kTileA;
                const uint32_t sb = sa + 2 * Lay::kTileA;
                const uint32_t sb_lo = sb + Lay::kTileB;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    // K-major (SW128): +32 B per k-step inside the 128 B swizzle row; LBO unused,
                    // SBO = 1024 B between 8-row groups.
                    // MN-major (SW128_32B): +8 K-rows x 128 B per k-step; LBO = stride of the
                    // 32-column MN blocks (one TMA box each), SBO = 512 B between 4-row atoms.
                    const uint32_t offa = A_MN ? kk * 1024 : kk * 32;
                    const uint32_t offb = B_MN ? kk * 1024 : kk * 32;
                    const uint32_t lboa = A_MN ? BK * 128 : 16, lbob = B_MN ? BK * 128 : 16;
                    const uint32_t sboa = A_MN ? 512 : 1024, sbob = B_MN ? 512 : 1024;
                    const uint32_t lya = A_MN ? 1 : 2, lyb = B_MN ? 1 : 2;
                    const uint64_t ahi = smem_desc(sa + offa, lboa, sboa, lya);
                    const uint64_t alo = smem_desc(sa_lo + offa, lboa, sboa, lya);
                    const uint64_t bhi = smem_desc(sb + offb, lbob, sbob, lyb);
                    const uint64_t blo = smem_desc(sb_lo + offb, lbob, sbob, lyb);
                    const int g = kb * (BK / 8) + kk;  // global k-step: accumulator j * per_g + r % per_g
                    const uint32_t d = tmem + static_cast<uint32_t>((j * per_g + rq) * BN);
                    const uint32_t first = r < per_g ? 0u : 1u;
                    mma_tf32(d, ahi, bhi, idesc, first);
#ifndef GASB_GEMM_DBG_ONEMMA  // (timing experiments only: plain TF32)
                    mma_tf32(d, ahi, blo, idesc, 1u);
                    mma_tf32(d, alo, bhi, idesc, 1u);
#endif
                    ++r;
                    rq = rq + 1 == per_g ? 0 : rq + 1;
                    if (g + 1 == gnext) {  // the group's last k-step: final once these MMAs complete
                        mma_commit(accready + j);
                        ++j;
                        r = rq = 0;
                        gnext = group_first(j + 1);
                    }
                }
                mma_commit(empty + s);  // frees the stage once these MMAs have read it
            }
        }
    } else {
        // ------- split (warps 0-3 and the helper warps 6+); drain + epilogue (drain warps / TALL: 0-3) -------
        const int sid = warp < 4 ? threadIdx.x : threadIdx.x - 64;  // split thread 0 .. kSplitThreads-1
        // warps 0-3: the tile row's sums over the drained accumulators (TMEM lane == tile row).
        // TALL (2 CTAs/SM, ~100 registers): 32 columns at a time, all accumulators at the end
        constexpr int kSum = TALL ? 32 : BN;
        float sum[kSum];
        const uint32_t tlane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        auto drain = [&](int q, int cb) {  // sum[0 .. kSum) += accumulator q, columns cb ..
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            constexpr int kG = 32;  // columns per tcgen05.wait::ld (64 spills at 448 threads)
#pragma unroll
            for (int c0 = 0; c0 < kSum; c0 += kG) {
                uint32_t v[kG];
#pragma unroll
                for (int c1 = 0; c1 < kG; c1 += 32) {
                    const uint32_t taddr = tlane + static_cast<uint32_t>(q * BN + cb + c0 + c1);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                        : "=r"(v[c1 + 0]), "=r"(v[c1 + 1]), "=r"(v[c1 + 2]), "=r"(v[c1 + 3]), "=r"(v[c1 + 4]),
                          "=r"(v[c1 + 5]), "=r"(v[c1 + 6]), "=r"(v[c1 + 7]), "=r"(v[c1 + 8]), "=r"(v[c1 + 9]),
                          "=r"(v[c1 + 10]), "=r"(v[c1 + 11]), "=r"(v[c1 + 12]), "=r"(v[c1 + 13]), "=r"(v[c1 + 14]),
                          "=r"(v[c1 + 15]), "=r"(v[c1 + 16]), "=r"(v[c1 + 17]), "=r"(v[c1 + 18]), "=r"(v[c1 + 19]),
                          "=r"(v[c1 + 20]), "=r"(v[c1 + 21]), "=r"(v[c1 + 22]), "=r"(v[c1 + 23]), "=r"(v[c1 + 24]),
                          "=r"(v[c1 + 25]), "=r"(v[c1 + 26]), "=r"(v[c1 + 27]), "=r"(v[c1 + 28]), "=r"(v[c1 + 29]),
                          "=r"(v[c1 + 30]), "=r"(v[c1 + 31])
                        : "r"(taddr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < kG; ++j)
                    sum[c0 + j] = q == 0 ? __uint_as_float(v[j]) : __fadd_rn(sum[c0 + j], __uint_as_float(v[j]));
            }
        };
        for (int kb = 0; kb < (drainer ? 0 : nk); ++kb) {
            const int s = kb % kStagesTC;
            bar_wait(full + s, (kb / kStagesTC) & 1);
            if (threadIdx.x == 0 && kb == 0) stamp(2);
            if (threadIdx.x == 0 && kb < 8) stamp(8 + kb);
            float4* a = reinterpret_cast<float4*>(base + s * Lay::kStage);
            float4* alo = a + Lay::kTileA / 16;
            float4* b = a + 2 * Lay::kTileA / 16;
            float4* blo = b + Lay::kTileB / 16;
#if GASB_GEMM_TRUNC_SPLIT
            // hi = the raw fp32 tile itself (the tensor core reads tf32 by truncating the low 13
            // mantissa bits), lo = rn_tf32(x - trunc_tf32(x)) (x - trunc is exact): only the lo
            // tiles are written, a third of the shared-memory traffic of a hi + lo rewrite — the
            // split is the mainloop's serial step (tools/gemm_timing_probe.py). Dropped terms
            // ~2^-22 relative, as the round-to-nearest split.
            for (int i = sid; i < Lay::kTileA / 16; i += kSplitThreads) {
                const float4 v = a[i];
                alo[i] = make_float4(tf32_hi(v.x - tf32_tr(v.x)), tf32_hi(v.y - tf32_tr(v.y)), tf32_hi(v.z - tf32_tr(v.z)),
                                     tf32_hi(v.w - tf32_tr(v.w)));
            }
            for (int i = sid; i < Lay::kTileB / 16; i += kSplitThreads) {
                const float4 v = b[i];
                blo[i] = make_float4(tf32_hi(v.x - tf32_tr(v.x)), tf32_hi(v.y - tf32_tr(v.y)), tf32_hi(v.z - tf32_tr(v.z)),
                                     tf32_hi(v.w - tf32_tr(v.w)));
            }
#elif defined(GASB_GEMM_DBG_NOSPLIT)  // (timing experiments only: no split)
            (void)alo, (void)blo, (void)sid;
#else
            // hi = rn_tf32(x), lo = rn_tf32(x - hi): both exactly tf32, so the tensor core's
            // operand truncation changes nothing; dropped lo*lo term ~2^-22 relative
            for (int i = sid; i < Lay::kTileA / 16; i += kSplitThreads) {
                float4 v = a[i], h;
                h.x = tf32_hi(v.x), h.y = tf32_hi(v.y), h.z = tf32_hi(v.z), h.w = tf32_hi(v.w);
                a[i] = h;
                alo[i] = make_float4(tf32_hi(v.x - h.x), tf32_hi(v.y - h.y), tf32_hi(v.z - h.z), tf32_hi(v.w - h.w));
            }
            for (int i = sid; i < Lay::kTileB / 16; i += kSplitThreads) {
                float4 v = b[i], h;
                h.x = tf32_hi(v.x), h.y = tf32_hi(v.y), h.z = tf32_hi(v.z), h.w = tf32_hi(v.w);
                b[i] = h;
                blo[i] = make_float4(tf32_hi(v.x - h.x), tf32_hi(v.y - h.y), tf32_hi(v.z - h.z), tf32_hi(v.w - h.w));
            }
#endif
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core
            if (threadIdx.x == 0 && kb < 8) stamp(16 + kb);
            bar_arrive(split + s);
        }
        if (drainer || (TALL && warp < 4)) {
            for (int j = 0; j < ng; ++j) {  // in accumulator order, each group as soon as it is final
                bar_wait(accready + j, 0);  // (a backed-off poll measured the same)
                if (!TALL)
                    for (int q = j * per_g; q < (j + 1) * per_g; ++q) drain(q, 0);
            }
            if (etid == 0) stamp(3);
            // phase 1: each thread (= tile row) parks its raw sums in shared memory (the stage
            // buffers are free: every MMA has completed), 16 B chunk c of row r at chunk position
            // c ^ (r mod kChunks) so that 8 consecutive rows hit distinct banks
            constexpr int kChunks = BN / 4;
            float4* stg = reinterpret_cast<float4*>(base);
    #pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 32) {
                if (TALL)
                    for (int q = 0; q < nacc; ++q) drain(q, c0);
                const int cs = TALL ? 0 : c0;  // this chunk's offset in sum[]
    #pragma unroll
                for (int j = 0; j < 32; j += 4)
                    stg[etid * kChunks + (((c0 + j) >> 2) ^ (etid & (kChunks - 1)))] =
                        make_float4(sum[cs + j], sum[cs + j + 1], sum[cs + j + 2], sum[cs + j + 3]);
            }
            {
                const int row = m0 + etid;
                if (row < M && push.table && push.stamps && !ws && blockIdx.y == 0) push.stamps[push.ids[row]] = *push.step;
            }
            __syncwarp();
            // phase 2: the warp stores its 32 rows coalesced (kChunks lanes per row, 16 B each),
            // applying the epilogue (scale, beta, bias, relu) and the history push on the way
            int32_t flags = 0;
            {
                const bool v4 = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) &&
                                (!push.table || ((push.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(push.table) & 15) == 0));
                const int Np = (N + 3) & ~3;  // split-K partial row pitch
                const int ch = lane % kChunks, c = n0 + 4 * ch;
    #pragma unroll 2
                for (int i = lane / kChunks; i < 32; i += 32 / kChunks) {
                    const int lr = (warp & 3) * 32 + i, r = m0 + lr;
                    const float4 s4 = stg[lr * kChunks + (ch ^ (lr & (kChunks - 1)))];
                    if (r >= M) continue;
                    if (ws) {  // slice partial: raw sums
                        if (c < Np)
                            *reinterpret_cast<float4*>(ws + (static_cast<int64_t>(blockIdx.z) * M + r) * Np + c) = s4;
                        continue;
                    }
                    float* cr = C + static_cast<int64_t>(r) * ldc;
                    float* pr = push.table ? push.table + static_cast<int64_t>(push.ids[r]) * push.ld : nullptr;
                    if (v4 && c + 3 < N) {
                        float4 x;
                        x.x = gemm_epilogue_value(ep, s4.x, cr, c);
                        x.y = gemm_epilogue_value(ep, s4.y, cr, c + 1);
                        x.z = gemm_epilogue_value(ep, s4.z, cr, c + 2);
                        x.w = gemm_epilogue_value(ep, s4.w, cr, c + 3);
                        *reinterpret_cast<float4*>(cr + c) = x;
                        if (pr) {
                            *reinterpret_cast<float4*>(pr + c) = x;
                            flags |= table_flag_of(x.x) | table_flag_of(x.y) | table_flag_of(x.z) | table_flag_of(x.w);
                        }
                        continue;
                    }
                    const float xs[4] = {s4.x, s4.y, s4.z, s4.w};
    #pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (c + q < N) {
                            const float x = gemm_epilogue_value(ep, xs[q], cr, c + q);
                            cr[c + q] = x;
                            if (pr) {
                                pr[c + q] = x;
                                flags |= table_flag_of(x);
                            }
                        }
                    }
                }
            }
            if (ws) {
                // parallel split-K fixup: every CTA of the tile publishes its slice, frees its TMEM
                // (a peer CTA may be waiting for it on this SM), waits until all gridDim.z slices of
                // the tile are in, then reduces its own 1/S of the tile's rows, summing the slices
                // in slice order (deterministic, independent of arrival order)
                __threadfence();
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
                if (warp == alloc_warp<TALL>()) {
                    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                                 "r"(Acc<BN, TALL>::kCols));
                }
                const int S = static_cast<int>(gridDim.z);
                int* arrive = reinterpret_cast<int*>(ws + ws_floats) + 2 * (blockIdx.y * gridDim.x + blockIdx.x);
                __shared__ int last_flag;
                if (serial_fixup) {
                    // serial fixup: no CTA ever waits; the last slice to arrive reduces the whole
                    // tile (in slice order), so any number of split-K grids may be in flight
                    if (etid == 0) {
                        const int prev = atomicAdd(arrive, 1);
                        last_flag = prev == S - 1;
                        if (last_flag) __threadfence();
                    }
                    asm volatile("bar.sync 1, 128;\n" ::: "memory");
                    if (!last_flag) goto fixup_done;
                } else if (etid == 0) {
                    atomicAdd(arrive, 1);
                    for (uint32_t spins = 0;; ++spins) {
                        int v;
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(arrive) : "memory");
                        if (v >= S) break;
                        if (spins > (1u << 28)) __trap();  // grid <= #SMs and the only split-K grid in flight (launch_tc callers): every slice gets resident
                        __nanosleep(64);
                    }
                }
                if (!serial_fixup) asm volatile("bar.sync 1, 128;\n" ::: "memory");
                {
                const int Np = (N + 3) & ~3;
                const int64_t slice = static_cast<int64_t>(M) * Np;
                const int rows_per = serial_fixup ? BM : (BM + S - 1) / S;
                const int rlo = serial_fixup ? 0 : blockIdx.z * rows_per, rhi = min(BM, rlo + rows_per);
                constexpr int kQ = BN / 4;  // float4 quads per tile row
                for (int idx = etid; idx < (rhi - rlo) * kQ; idx += 128) {
                    const int r = m0 + rlo + idx / kQ, c = n0 + 4 * (idx % kQ);
                    if (r >= M || c >= N) continue;
                    const float4* wp = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(r) * Np + c);
                    float4 x = __ldcg(wp);
                    for (int z = 1; z < S; ++z) {
                        const float4 y = __ldcg(wp + z * (slice >> 2));
                        x = make_float4(__fadd_rn(x.x, y.x), __fadd_rn(x.y, y.y), __fadd_rn(x.z, y.z), __fadd_rn(x.w, y.w));
                    }
                    float* cr = C + static_cast<int64_t>(r) * ldc;
                    float* pr = push.table ? push.table + static_cast<int64_t>(push.ids[r]) * push.ld : nullptr;
                    const float xs[4] = {x.x, x.y, x.z, x.w};
    #pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (c + k >= N) break;
                        const float v = gemm_epilogue_value(ep, xs[k], cr, c + k);
                        cr[c + k] = v;
                        if (pr) {
                            pr[c + k] = v;
                            flags |= table_flag_of(v);
                        }
                    }
                    if (pr && c == 0 && push.stamps) push.stamps[push.ids[r]] = *push.step;
                }
                if (serial_fixup) {
                    if (etid == 0) arrive[0] = 0;  // the only CTA left on this tile
                } else if (etid == 0 && atomicAdd(arrive + 1, 1) == S - 1) {  // last to leave resets
                    arrive[0] = 0;
                    arrive[1] = 0;
                }
                }
            fixup_done:;
            }
            if (push.special) {
                flags = __reduce_or_sync(0xffffffffu, flags);
                if (lane == 0 && flags) atomicOr(push.special, flags);
            }
        }
    }
    if ((drainer || (TALL && warp < 4)) && etid == 0) stamp(4);
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == alloc_warp<TALL>() && !ws) {  // (split-K CTAs freed their TMEM before the fixup)
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(Acc<BN, TALL>::kCols));
    }
#ifdef GASB_GEMM_TIMING
    if (threadIdx.x == 0 && blockIdx.z == 0 && cta_id < 256) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_gemm_stamps[41 + 2 * cta_id] = t;
    }
#endif
}

// 2-D fp32 tensor map for TMA with 128 B swizzle: contiguous dim `inner` (elements), `outer`
// rows with pitch `ld` floats; box {32, box_outer}. mn_major selects the 32 B-atom swizzle.
static bool make_tmap(const float* p, int64_t inner, int64_t outer, int64_t ld, int box_outer, CUtensorMap* out,
                      bool mn_major) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // the 32-element box must fit the contiguous dimension (narrower tables read back zeros)
    if (inner < 32 || outer <= 0 || (ld * 4) % 16 != 0 || reinterpret_cast<uintptr_t>(p) % 16 != 0) return false;
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * 4};
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_outer)};
    const cuuint32_t es[2] = {1, 1};
    return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), gdim, gstride, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, bool TALL = false>
static bool launch_tc(int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                      int64_t ldc, const GemmEpilogue& ep, cudaStream_t st) {
    using Lay = Layout<BN, A_MN, B_MN, TALL>;
    CUtensorMap ta, tb;
    // A: K-major -> inner K, outer M (box 32 x 128); MN-major -> inner M, outer K (box 32 x 32)
    const bool ok_a = A_MN ? make_tmap(a, m, k, lda, BK, &ta, true) : make_tmap(a, k, m, lda, BM, &ta, false);
    const bool ok_b = B_MN ? make_tmap(b, n, k, ldb, BK, &tb, true) : make_tmap(b, k, n, ldb, BN, &tb, false);
    if (!ok_a || !ok_b) return false;  // pitch not 16 B aligned: caller uses the SIMT kernel
    static bool attr = false;
    if (!attr) {
        GASB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, A_MN, B_MN, TALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Lay::kSmem));
        attr = true;
    }
    // split-K over otherwise idle SMs (deterministic: slices reduced in order by a 2nd kernel)
    const int64_t tiles = ceil_div(m, BM) * ceil_div(n, BN);
    const int nkb = static_cast<int>(ceil_div(k, BK));
    int S = 1;
    static const int split_div = [] {  // GASB_GEMM_SPLITK_DIV: min k-blocks per split-K slice (0 = off)
        const char* e = getenv("GASB_GEMM_SPLITK_DIV");
        return e ? atoi(e) : 6;  // measured at C3 (ms/epoch): 4: 110.0, 6: 106.5, 8: 107.3, 12: 109.2, 16: 111.0
    }();
    if (!TALL && split_div > 0 && t_gemm_ws && tiles < num_sms()) {
        S = static_cast<int>(std::min<int64_t>(num_sms() / tiles, std::max(1, nkb / split_div)));
        while (S > 1 && static_cast<int64_t>(S) * m * round_up(n, 4) > t_gemm_ws_floats) --S;
        if (2 * tiles > kGemmTileCounters) S = 1;
    }
    static const int acc_groups = [] {  // GASB_GEMM_ACC_GROUPS: accumulator groups (1 = drain after the mainloop)
        const char* e = getenv("GASB_GEMM_ACC_GROUPS");
        return e ? std::max(1, atoi(e)) : 2;
    }();
    const int kbs = static_cast<int>(ceil_div(nkb, S));
    S = static_cast<int>(ceil_div(nkb, kbs));  // no empty slices
    dim3 grid(static_cast<unsigned>(ceil_div(m, BM)), static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(S));
    launch_pdl(gemm_tc_kernel<BN, A_MN, B_MN, TALL>, grid, dim3(threads_of<TALL>()), Lay::kSmem, st, ta, tb, m, n, k, c,
               ldc, ep, kbs, S > 1 ? t_gemm_ws : nullptr, t_gemm_ws_floats, t_gemm_serial ? 1 : 0, acc_groups);
    return true;
}

}  // namespace tc

// Tensor-core path of launch_gemm (gemm.cu) — same contract. Returns false (nothing
// launched) when an operand's row pitch cannot be described to TMA.
bool launch_gemm_tc(int op, int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                    int64_t ldc, const GemmEpilogue& ep, cudaStream_t st) {
    if (m <= 0 || n <= 0) return true;
    bool ok, n32 = false;
    // many tiles with a short K (the residual heads over every V_b row): two CTAs per SM
    const bool tall = ceil_div(m, tc::BM) * ceil_div(n, 64) >= 2LL * num_sms() && k <= 16 * tc::BK;
    if (tall && n > 32) {
        switch (op) {
            case 0: ok = tc::launch_tc<64, false, true, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st); break;
            case 1: ok = tc::launch_tc<64, false, false, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st); break;
            case 2: ok = tc::launch_tc<64, true, true, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st); break;
            default: throw std::invalid_argument("gemm: op must be 0, 1 or 2");
        }
        if (!ok) return false;
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return true;
    }
    // narrow N tiles keep enough CTAs in flight for the ~1K-row batch GEMMs
    static const int bn_thresh = [] {  // GASB_GEMM_BN32_BELOW: N-tile 32 while the 64-wide grid < this many CTAs
        const char* e = getenv("GASB_GEMM_BN32_BELOW");
        return e ? atoi(e) : 0;
    }();
    if (ceil_div(m, tc::BM) * ceil_div(n, 64) < bn_thresh) n32 = true;
    switch (op) {
        case 0:
            ok = (n <= 32 || n32) ? tc::launch_tc<32, false, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st)
                         : tc::launch_tc<64, false, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st);
            break;
        case 1:
            ok = (n <= 32 || n32) ? tc::launch_tc<32, false, false>(m, n, k, a, lda, b, ldb, c, ldc, ep, st)
                         : tc::launch_tc<64, false, false>(m, n, k, a, lda, b, ldb, c, ldc, ep, st);
            break;
        case 2:
            ok = (n <= 32 || n32) ? tc::launch_tc<32, true, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st)
                         : tc::launch_tc<64, true, true>(m, n, k, a, lda, b, ldb, c, ldc, ep, st);
            break;
        default: throw std::invalid_argument("gemm: op must be 0, 1 or 2");
    }
    if (!ok) return false;
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
    return true;
}

}  // namespace gasb
