// TMA tile::gather4 throughput ceiling on this GPU: the gather engine of the flat SpMM
// (spmm.cu) without its FMAs, segments or metadata. Each warp's lane 0 keeps `stages`
// stages of 4-row x box-column gathers (one cp.async.bulk.tensor.2d...tile::gather4 per
// stage, mbarrier completion) in flight over pseudo-random rows of an fp32 table; the warp
// only waits and re-issues. Sweeps table size (L2-resident vs DRAM), row width (box 256 =
// 1 KB rows, 128 = 512 B), stages per warp and warps per SM (shared memory bounds the
// product, as in the SpMM). Prints one JSON line per point: gathered bytes / kernel time
// (CUDA events, best of 3).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/l2bw/tma_gather_bw.cu -o tools/l2bw/tma_gather_bw
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void gather_kernel(const __grid_constant__ CUtensorMap tm, int64_t rows, int box, int stages, int iters,
                              int* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int stage_bytes = 4 * box * 4;
    unsigned char* wbase = smem + static_cast<size_t>(warp) * stages * stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(nw) * stages * stage_bytes) + warp * stages;
    // rows is a power of two: a 32-bit LCG masked to it (cheap next to the TMA issue)
    uint32_t r = static_cast<uint32_t>((blockIdx.x * nw + warp) * 2654435761u + 12345u);
    const uint32_t mask = static_cast<uint32_t>(rows - 1);
    auto next_row = [&]() {
        r = r * 1664525u + 1013904223u;
        return static_cast<int32_t>((r >> 7) & mask);
    };
    if (lane == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + s)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int s) {
        const int32_t r0 = next_row(), r1 = next_row(), r2 = next_row(), r3 = next_row();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bars + s)), "r"(stage_bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(wbase + s * stage_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bars + s))
            : "memory");
    };
    uint32_t phase = 0;
    int sum = 0;
    if (lane == 0) {
        for (int s = 0; s < stages; ++s) issue(s);
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(su32(bars + s)), "r"((phase >> s) & 1u)
                    : "memory");
            phase ^= 1u << s;
            sum += reinterpret_cast<const int*>(wbase + s * stage_bytes)[0];
            if (i + stages < iters) issue(s);
        }
    }
    if (sum == 0x7fffffff) out[0] = sum;
}

int main() {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    int* out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int64_t mb : {32, 2048}) {
        const int dim = 256;
        const int64_t rows = (mb << 20) / (dim * 4);
        float* tab;
        cudaMalloc(&tab, rows * dim * 4);
        cudaMemset(tab, 0, rows * dim * 4);
        for (int box : {256, 128}) {
            CUtensorMap tm;
            const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(rows)};
            const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(dim) * 4};
            const cuuint32_t boxd[2] = {static_cast<cuuint32_t>(box), 1};
            const cuuint32_t es[2] = {1, 1};
            encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, gdim, gstride, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int stage_bytes = 4 * box * 4;
            for (int wps : {8, 12, 16, 24, 32})
                for (int stages : {1, 2, 3, 4, 6, 8}) {
                    const int threads = 128, ctas_per_sm = wps / 4;
                    const size_t smem = static_cast<size_t>(4) * stages * (stage_bytes + 8);
                    if (smem * ctas_per_sm > 220 * 1024 || smem > 220 * 1024) continue;
                    const int blocks = sms * ctas_per_sm;
                    const int iters = 2048;
                    float best = 1e30f;
                    for (int rep = 0; rep < 3; ++rep) {
                        cudaEventRecord(e0);
                        gather_kernel<<<blocks, threads, smem>>>(tm, rows, box, stages, iters, out);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        float ms = 0;
                        cudaEventElapsedTime(&ms, e0, e1);
                        if (ms < best) best = ms;
                    }
                    if (cudaGetLastError() != cudaSuccess) {
                        printf("{\"error\": \"launch failed\"}\n");
                        return 1;
                    }
                    const double bytes = static_cast<double>(blocks) * 4 * iters * stage_bytes;
                    printf("{\"table_mb\": %lld, \"row_bytes\": %d, \"warps_per_sm\": %d, \"stages\": %d, "
                           "\"inflight_kb_per_sm\": %d, \"gbs\": %.1f}\n",
                           static_cast<long long>(mb), box * 4, wps, stages, wps * stages * stage_bytes / 1024,
                           bytes / (best * 1e-3) / 1e9);
                    fflush(stdout);
                }
        }
        cudaFree(tab);
    }
    return 0;
}
