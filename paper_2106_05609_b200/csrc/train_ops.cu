// Loss and optimizer kernels of the GAS batch step.
//  softmax_cross_entropy  src/tensor.cpp:597-647  (fp64 row math, float gradient)
//  grad_clip              src/nn.cpp:47-63        (fp64 global norm, float scale)
//  AdamState::step        src/nn.cpp:20-41        (fp64 math, fp32 moments)
// Arithmetic is written with explicit _rn intrinsics so no FMA contraction changes the
// rounding sequence of the reference (built without -march: no FMA);
// Adam is therefore bit-exact given identical gradients and bias corrections.
#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {

// One block. Rows of the training mask are handled one per thread (sequential over the
// classes, as the reference); the per-row losses are summed in row order by thread 0.
__global__ void __launch_bounds__(256) softmax_ce_kernel(const float* __restrict__ logits, int64_t ldl, int32_t m,
                                                         int32_t n, const int32_t* __restrict__ rows,
                                                         const int32_t* __restrict__ labels, int32_t r,
                                                         float* __restrict__ gl, int64_t ldg,
                                                         double* __restrict__ loss_out, double* __restrict__ scratch) {
    for (int64_t i = threadIdx.x; i < static_cast<int64_t>(m) * n; i += blockDim.x)
        gl[(i / n) * ldg + (i % n)] = 0.0f;
    __syncthreads();
    const float inv_m = __frcp_rn(static_cast<float>(r));  // 1.0f / float(rows.size())
    for (int32_t i = threadIdx.x; i < r; i += blockDim.x) {
        const float* row = logits + static_cast<int64_t>(rows[i]) * ldl;
        float* g = gl + static_cast<int64_t>(rows[i]) * ldg;
        float mx = row[0];
        for (int32_t j = 1; j < n; ++j) mx = fmaxf(mx, row[j]);
        double denom = 0.0;
        for (int32_t j = 0; j < n; ++j) denom = __dadd_rn(denom, exp(__dsub_rn(static_cast<double>(row[j]), mx)));
        scratch[i] = __dsub_rn(log(denom), __dsub_rn(static_cast<double>(row[labels[i]]), mx));
        const float gy_inv = __fmul_rn(1.0f, inv_m);
        for (int32_t j = 0; j < n; ++j) {
            const double p = __ddiv_rn(exp(__dsub_rn(static_cast<double>(row[j]), mx)), denom);
            const double delta = (j == labels[i]) ? 1.0 : 0.0;
            g[j] = __fadd_rn(g[j], __fmul_rn(gy_inv, static_cast<float>(__dsub_rn(p, delta))));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int32_t i = 0; i < r; ++i) total = __dadd_rn(total, scratch[i]);
        *loss_out = static_cast<double>(static_cast<float>(__ddiv_rn(total, static_cast<double>(r))));
    }
}

void launch_softmax_ce(const float* logits, int64_t ldl, int32_t m, int32_t n, const int32_t* rows,
                       const int32_t* labels, int32_t r, float* glogits, int64_t ldg, double* loss_out,
                       double* row_scratch, cudaStream_t st) {
    softmax_ce_kernel<<<1, 256, 0, st>>>(logits, ldl, m, n, rows, labels, r, glogits, ldg, loss_out, row_scratch);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

// Global gradient norm: fixed-shape two-level reduction (deterministic run to run).
__global__ void __launch_bounds__(256) sumsq_kernel(const float* __restrict__ g, int64_t size,
                                                    double* __restrict__ partial) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < size;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = g[i];
        acc = __dadd_rn(acc, __dmul_rn(v, v));
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void finish_norm_kernel(double* partial, int nparts) {
    double acc = 0.0;
    for (int i = 0; i < nparts; ++i) acc = __dadd_rn(acc, partial[i]);
    partial[nparts] = __dsqrt_rn(acc);
}

constexpr int kNormBlocks = 128;

__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                                                   const float* __restrict__ g, int64_t size,
                                                   const int64_t* __restrict__ t_counter, const double* __restrict__ bc,
                                                   float lr, float b1, float b2, float eps, float clip,
                                                   const double* __restrict__ norm) {
    const int64_t t = *t_counter + 1;
    const double bc1 = bc[2 * t], bc2 = bc[2 * t + 1];
    float s = 1.0f;
    bool scale = false;
    if (clip > 0.0f) {
        const double nn = *norm;
        if (nn > static_cast<double>(clip)) {
            scale = true;
            s = static_cast<float>(__ddiv_rn(static_cast<double>(clip), nn));
        }
    }
    const double B1 = b1, B2 = b2, omb1 = __dsub_rn(1.0, B1), omb2 = __dsub_rn(1.0, B2), LR = lr, EPS = eps;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < size;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float gf = scale ? __fmul_rn(g[e], s) : g[e];
        const double ge = gf;
        const double mm = __dadd_rn(__dmul_rn(B1, static_cast<double>(m[e])), __dmul_rn(omb1, ge));
        const double vv = __dadd_rn(__dmul_rn(B2, static_cast<double>(v[e])), __dmul_rn(__dmul_rn(omb2, ge), ge));
        m[e] = static_cast<float>(mm);
        v[e] = static_cast<float>(vv);
        const double mhat = __ddiv_rn(mm, bc1), vhat = __ddiv_rn(vv, bc2);
        const double upd = __ddiv_rn(__dmul_rn(LR, mhat), __dadd_rn(__dsqrt_rn(vhat), EPS));
        p[e] = static_cast<float>(__dsub_rn(static_cast<double>(p[e]), upd));
    }
}

void launch_adam(float* p, float* m, float* v, float* g, int64_t size, int64_t* t_counter, const double* bc, float lr,
                 float b1, float b2, float eps, float clip_max_norm, double* norm_scratch, cudaStream_t st) {
    if (clip_max_norm > 0.0f) {
        sumsq_kernel<<<kNormBlocks, 256, 0, st>>>(g, size, norm_scratch);
        finish_norm_kernel<<<1, 1, 0, st>>>(norm_scratch, kNormBlocks);
        t_launches += 2;
    }
    const int64_t blocks = std::min<int64_t>(ceil_div(size, 256), 4 * 148);
    adam_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(p, m, v, g, size, t_counter, bc, lr, b1, b2, eps,
                                                               clip_max_norm, norm_scratch + kNormBlocks);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

__global__ void zero_kernel(float* p, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0.0f;
}

void launch_zero(float* p, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    zero_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 256), 1184)), 256, 0, st>>>(p, count);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

}  // namespace gasb
