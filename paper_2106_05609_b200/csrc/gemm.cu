// Dense feature transform (the reference's matmul, src/tensor.cpp:148-204) — dispatch to the
// tcgen05 3xTF32 kernel (gemm_tc.cu) and this FP32 SIMT fallback for pitches a TMA tensor map
// cannot describe (pitch not 16 B aligned or inner extent < 32). The reference accumulates in
// fp64; both engines stay ~1e-6 normwise, inside the 1e-5 contract.
//
// Tile 64x64x16, 256 threads, 4x4 outputs per thread in a strided (16-apart) pattern so
// that smem reads are conflict-free broadcasts; register double-buffering of the next
// k-tile. Epilogue for op 0 (forward): optional relu, optional row push into a history
// table (HistoryStore::push fused, history.cpp:28-42) with last-push stamps.
#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <int OP>
__device__ __forceinline__ void load_a(const float* __restrict__ A, int64_t lda, int M, int K, int m0, int k0, int tid,
                                       float (&ra)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int m, k;
        if (OP == 2) {  // A is [K, M]
            m = m0 + (tid & 63);
            k = k0 + (tid >> 6) + 4 * i;
            ra[i] = (m < M && k < K) ? __ldg(A + static_cast<int64_t>(k) * lda + m) : 0.f;
        } else {  // A is [M, K]
            k = k0 + (tid & 15);
            m = m0 + (tid >> 4) + 16 * i;
            ra[i] = (m < M && k < K) ? __ldg(A + static_cast<int64_t>(m) * lda + k) : 0.f;
        }
    }
}
template <int OP>
__device__ __forceinline__ void store_a(float (*As)[BM + 4], int tid, const float (&ra)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (OP == 2) As[(tid >> 6) + 4 * i][tid & 63] = ra[i];
        else As[tid & 15][(tid >> 4) + 16 * i] = ra[i];
    }
}
template <int OP>
__device__ __forceinline__ void load_b(const float* __restrict__ B, int64_t ldb, int N, int K, int n0, int k0, int tid,
                                       float (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int n, k;
        if (OP == 1) {  // B is [N, K]
            k = k0 + (tid & 15);
            n = n0 + (tid >> 4) + 16 * i;
            rb[i] = (n < N && k < K) ? __ldg(B + static_cast<int64_t>(n) * ldb + k) : 0.f;
        } else {  // B is [K, N]
            n = n0 + (tid & 63);
            k = k0 + (tid >> 6) + 4 * i;
            rb[i] = (n < N && k < K) ? __ldg(B + static_cast<int64_t>(k) * ldb + n) : 0.f;
        }
    }
}
template <int OP>
__device__ __forceinline__ void store_b(float (*Bs)[BN + 4], int tid, const float (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (OP == 1) Bs[tid & 15][(tid >> 4) + 16 * i] = rb[i];
        else Bs[(tid >> 6) + 4 * i][tid & 63] = rb[i];
    }
}
}  // namespace

template <int OP>
__global__ void __launch_bounds__(256) gemm_kernel(int M, int N, int K, const float* __restrict__ A, int64_t lda,
                                                   const float* __restrict__ B, int64_t ldb, float* __restrict__ C,
                                                   int64_t ldc, GemmEpilogue ep) {
    const PushEpilogue& push = ep.push;
    __shared__ float As[2][BK][BM + 4];
    __shared__ float Bs[2][BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    float acc[4][4] = {};
    float ra[4], rb[4];
    load_a<OP>(A, lda, M, K, m0, 0, tid, ra);
    load_b<OP>(B, ldb, N, K, n0, 0, tid, rb);
    store_a<OP>(As[0], tid, ra);
    store_b<OP>(Bs[0], tid, rb);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += BK) {
        const bool more = k0 + BK < K;
        if (more) {
            load_a<OP>(A, lda, M, K, m0, k0 + BK, tid, ra);
            load_b<OP>(B, ldb, N, K, n0, k0 + BK, tid, rb);
        }
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            store_a<OP>(As[buf ^ 1], tid, ra);
            store_b<OP>(Bs[buf ^ 1], tid, rb);
            __syncthreads();
            buf ^= 1;
        }
    }
    int32_t pushed_flags = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= M) continue;
        float* crow = C + static_cast<int64_t>(m) * ldc;
        float* prow = nullptr;
        if (push.table) {
            const int32_t id = push.ids[m];
            prow = push.table + static_cast<int64_t>(id) * push.ld;
            if (blockIdx.x == 0 && tx == 0 && push.stamps) push.stamps[id] = *push.step;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= N) continue;
            const float v = gemm_epilogue_value(ep, acc[i][j], crow, n);
            crow[n] = v;
            if (prow) {
                prow[n] = v;
                pushed_flags |= table_flag_of(v);
            }
        }
    }
    if (push.special) {  // the history table's value flags (spmm.cu widening paths)
        pushed_flags = __reduce_or_sync(0xffffffffu, pushed_flags);
        if ((tid & 31) == 0 && pushed_flags) atomicOr(push.special, pushed_flags);
    }
}

bool launch_gemm_tc(int op, int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                    int64_t ldc, const GemmEpilogue& ep, cudaStream_t st);

// GEMM engine (tuning knob GASB_GEMM_TC = 1 tcgen05 3xTF32 (default) | 0 FP32 SIMT).
static bool gemm_use_tc() {
    static int v = [] {
        const char* e = getenv("GASB_GEMM_TC");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

void launch_gemm(int op, int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                 int64_t ldc, const GemmEpilogue& ep, cudaStream_t st) {
    if (m <= 0 || n <= 0) return;
    require(op == 0 || !ep.push.table, "gemm: push epilogue only for op 0");
    if (gemm_use_tc() && k > 0 && launch_gemm_tc(op, m, n, k, a, lda, b, ldb, c, ldc, ep, st)) return;
    dim3 grid(static_cast<unsigned>(ceil_div(n, BN)), static_cast<unsigned>(ceil_div(m, BM)));
    switch (op) {
        case 0: gemm_kernel<0><<<grid, 256, 0, st>>>(m, n, k, a, lda, b, ldb, c, ldc, ep); break;
        case 1: gemm_kernel<1><<<grid, 256, 0, st>>>(m, n, k, a, lda, b, ldb, c, ldc, ep); break;
        case 2: gemm_kernel<2><<<grid, 256, 0, st>>>(m, n, k, a, lda, b, ldb, c, ldc, ep); break;
        default: throw std::invalid_argument("gemm: op must be 0, 1 or 2");
    }
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_gemm(int op, int m, int n, int k, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                 int64_t ldc, float beta, bool relu, const PushEpilogue* push, cudaStream_t st) {
    GemmEpilogue ep;
    ep.beta = beta;
    ep.relu = relu ? 1 : 0;
    if (push) ep.push = *push;
    launch_gemm(op, m, n, k, a, lda, b, ldb, c, ldc, ep, st);
}

}  // namespace gasb

extern "C" gasb_status gasb_gemm(int32_t op, int32_t m, int32_t n, int32_t k, const float* a, int64_t lda,
                                 const float* b, int64_t ldb, float* c, int64_t ldc, float beta, gasb_stream stream) {
    return gasb::guard([&] {
        gasb::require(m >= 0 && n >= 0 && k >= 0, "matmul: negative shape");
        gasb::require(beta == 0.f || beta == 1.f, "matmul: beta must be 0 or 1");
        // the standalone entry point may be called on several streams at once: a split-K
        // workspace of its own per call (stream-ordered allocation) and the serial fixup, in
        // which no CTA waits for its peer slices
        cudaStream_t st = gasb::as_stream(stream);
        constexpr int64_t total = gasb::kGemmWsFloats + gasb::kGemmTileCounters;
        float* ws = nullptr;
        GASB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(float) * total, st));
        GASB_CUDA(cudaMemsetAsync(ws + gasb::kGemmWsFloats, 0, sizeof(float) * gasb::kGemmTileCounters, st));
        gasb::set_gemm_workspace(ws, gasb::kGemmWsFloats, /*serial_fixup=*/true);
        struct Reset {
            float* ws;
            cudaStream_t st;
            ~Reset() {
                gasb::set_gemm_workspace(nullptr, 0);
                cudaFreeAsync(ws, st);
            }
        } reset{ws, st};
        gasb::launch_gemm(op, m, n, k, a, lda, b, ldb, c, ldc, beta, false, nullptr, st);
    });
}
