// L2 -> SM read throughput on this GPU: the ceiling for gathers whose rows are L2 hits.
// A buffer smaller than L2 (default 32 MB) is read repeatedly with 16 B ld.global.cg
// (L2, not L1) by a persistent grid, either streaming or as 1 KB rows gathered in a
// pseudo-random order (the SpMM's access shape: a warp reads one 1 KB row per step).
// Prints one JSON line per pattern: bytes moved / kernel time (CUDA events, best of 5).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2bw/l2_bw.cu -o tools/l2bw/l2_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ldcg(const float4* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// each warp: `iters` steps, each step reads one 1 KB row (64 lanes x 16 B? -> 32 lanes x 2 x 16 B)
template <bool GATHER>
__global__ void read_kernel(const float4* __restrict__ buf, int64_t rows, int iters, float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    float acc = 0.0f;
    uint64_t r = warp * 0x9E3779B97F4A7C15ull + 1;
    int64_t row = warp % rows;
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        if (GATHER) {
            r ^= r << 13;
            r ^= r >> 7;
            r ^= r << 17;
            row = static_cast<int64_t>((r >> 11) & static_cast<uint64_t>(rows - 1));  // rows: power of two
        } else {
            row += nwarps;
            if (row >= rows) row -= rows;
        }
        const float4* p = buf + row * 64;  // 1 KB row = 64 x 16 B
        const float4 a = ldcg(p + lane), b = ldcg(p + 32 + lane);
        acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
    }
    if (acc == 12345.678f) out[0] = acc;
}

int main(int argc, char** argv) {
    const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 32) << 20;  // power of two MB
    const int64_t rows = bytes / 1024;
    float4* buf;
    float* out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int pat = 0; pat < 2; ++pat) {
        for (int wps : {8, 16, 32, 64}) {  // warps per SM
            const int threads = 256, blocks = sms * wps / 8;
            float best = 1e30f;
            for (int rep = 0; rep < 6; ++rep) {
                cudaEventRecord(e0);
                if (pat) read_kernel<true><<<blocks, threads>>>(buf, rows, iters, out);
                else read_kernel<false><<<blocks, threads>>>(buf, rows, iters, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) best = ms < best ? ms : best;
            }
            const double moved = double(blocks) * threads / 32 * iters * 1024.0;
            printf("{\"pattern\": \"%s\", \"buffer_mb\": %lld, \"warps_per_sm\": %d, \"gbs\": %.1f}\n",
                   pat ? "gather_1kb_rows" : "stream_1kb_rows", (long long)(bytes >> 20), wps, moved / best / 1e6);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
