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

// A warp per batch row (grid-wide), lanes over the classes. row_label[i] = label of batch row
// i when it is a training row, -1 otherwise (its gradient row is zeroed). Row max is exact in
// any order; the fp64 softmax denominator and the loss sum use a fixed shuffle / tree order
// (deterministic; differs from the reference's sequential fp64 sums only below the fp32
// resolution of the outputs). The last CTA to finish sums the per-row terms in row order.
constexpr int kCeThreads = 256;

__global__ void __launch_bounds__(kCeThreads) softmax_ce_kernel(const float* __restrict__ logits, int64_t ldl,
                                                                int32_t m, int32_t n,
                                                                const int32_t* __restrict__ row_label, int32_t r,
                                                                float* __restrict__ gl, int64_t ldg,
                                                                double* __restrict__ loss_out,
                                                                double* __restrict__ scratch,
                                                                int32_t* __restrict__ done) {
    __shared__ double red[kCeThreads];
    __shared__ int last;
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int32_t i = blockIdx.x * (kCeThreads / 32) + (threadIdx.x >> 5);
    const float inv_m = __frcp_rn(static_cast<float>(r));  // 1.0f / float(rows.size())
    const float gy_inv = __fmul_rn(1.0f, inv_m);            // gy * inv_m, gy = 1
    double term = 0.0;
    if (i < m) {
        const float* row = logits + static_cast<int64_t>(i) * ldl;
        float* g = gl + static_cast<int64_t>(i) * ldg;
        const int lab = row_label[i];
        if (lab < 0) {
            for (int j = lane; j < n; j += 32) g[j] = 0.0f;
        } else {
        float mx = -INFINITY;
        for (int j = lane; j < n; j += 32) mx = fmaxf(mx, row[j]);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double e[2] = {0.0, 0.0}, den = 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int j = lane + 32 * k;
            if (j < n) e[k] = exp(__dsub_rn(static_cast<double>(row[j]), static_cast<double>(mx)));
            den = __dadd_rn(den, e[k]);
        }
        for (int j = 64 + lane; j < n; j += 32) den = __dadd_rn(den, exp(__dsub_rn(static_cast<double>(row[j]), mx)));
        for (int o = 16; o > 0; o >>= 1) den = __dadd_rn(den, __shfl_xor_sync(0xffffffffu, den, o));
        term = __dsub_rn(log(den), __dsub_rn(static_cast<double>(row[lab]), mx));
        for (int j = lane; j < n; j += 32) {
            const double ej = j < 64 ? e[j >> 5] : exp(__dsub_rn(static_cast<double>(row[j]), mx));
            const double p = __ddiv_rn(ej, den);
            const double delta = (j == lab) ? 1.0 : 0.0;
            g[j] = __fmul_rn(gy_inv, static_cast<float>(__dsub_rn(p, delta)));
        }
        }
        if (lane == 0) scratch[i] = term;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1) == static_cast<int>(gridDim.x) - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double acc = 0.0;
    for (int32_t k = threadIdx.x; k < m; k += kCeThreads) acc = __dadd_rn(acc, __ldcg(scratch + k));
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kCeThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *loss_out = static_cast<double>(static_cast<float>(__ddiv_rn(red[0], static_cast<double>(r))));
        *done = 0;  // self-reset for the next launch / graph replay
    }
}

void launch_softmax_ce(const float* logits, int64_t ldl, int32_t m, int32_t n, const int32_t* row_label, int32_t r,
                       float* glogits, int64_t ldg, double* loss_out, double* row_scratch, int32_t* done,
                       cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>(ceil_div(m, kCeThreads / 32));
    launch_pdl(softmax_ce_kernel, dim3(blocks), dim3(kCeThreads), 0, st, logits, ldl, m, n, row_label, r, glogits, ldg,
               loss_out, row_scratch, done);
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
                                                   int64_t* t_counter, const double* __restrict__ bc,
                                                   float lr, float b1, float b2, float eps, float clip,
                                                   const double* __restrict__ norm, int64_t* __restrict__ end_step, int32_t* __restrict__ end_done) {
    pdl_trigger();
    pdl_wait();
    const int64_t t = min(*t_counter + 1, static_cast<int64_t>(bc[0]));  // bc[0]: saturation step
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
    if (end_step) {  // end of batch fused in: the last block to finish advances the counters
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(end_done, 1) == static_cast<int32_t>(gridDim.x) - 1) {
                *end_step += 1;  // HistoryStore::advance_step (trainer.cpp:426)
                *t_counter += 1;  // AdamState::step count
                *end_done = 0;
            }
        }
    }
}

void launch_adam(float* p, float* m, float* v, float* g, int64_t size, int64_t* t_counter, const double* bc, float lr,
                 float b1, float b2, float eps, float clip_max_norm, double* norm_scratch, cudaStream_t st,
                 int64_t* end_step, int32_t* end_done) {
    if (clip_max_norm > 0.0f) {
        sumsq_kernel<<<kNormBlocks, 256, 0, st>>>(g, size, norm_scratch);
        finish_norm_kernel<<<1, 1, 0, st>>>(norm_scratch, kNormBlocks);
        t_launches += 2;
    }
    const int64_t blocks = std::min<int64_t>(ceil_div(size, 256), 4 * 148);
    launch_pdl(adam_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, p, m, v, g, size, t_counter, bc, lr,
               b1, b2, eps, clip_max_norm, static_cast<const double*>(norm_scratch + kNormBlocks), end_step, end_done);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

// l2_penalty (tensor.cpp:649-678) as the reference's run_batch applies it (trainer.cpp:322-323):
// its backward closure runs first, so every parameter gradient is g = (2 w v) + (data
// gradient) — one fp32 rounding each, as `g[i] += gy * 2.0f * weight * v[i]` with gy = 1 —
// and the loss becomes float(ce) + float(w * sum double(v)^2).
__global__ void __launch_bounds__(256) l2_grad_kernel(const float* __restrict__ p, float* __restrict__ g,
                                                      int64_t size, float two_w) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < size;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        g[i] = __fadd_rn(__fmul_rn(two_w, p[i]), g[i]);
}

__global__ void l2_loss_kernel(const double* partial, int nparts, float w, double* loss) {
    double acc = 0.0;
    for (int i = 0; i < nparts; ++i) acc = __dadd_rn(acc, partial[i]);
    const float pen = static_cast<float>(__dmul_rn(static_cast<double>(w), acc));
    *loss = static_cast<double>(__fadd_rn(static_cast<float>(*loss), pen));
}

void launch_l2_penalty(const float* p, float* g, int64_t size, float w, double* loss, double* scratch,
                       cudaStream_t st) {
    sumsq_kernel<<<kNormBlocks, 256, 0, st>>>(p, size, scratch);
    l2_loss_kernel<<<1, 1, 0, st>>>(scratch, kNormBlocks, w, loss);
    const int64_t blocks = std::min<int64_t>(ceil_div(size, 256), 4 * 148);
    l2_grad_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(p, g, size, 2.0f * w);  // exact
    t_launches += 3;
    GASB_CUDA(cudaGetLastError());
}

__global__ void zero_kernel(float* p, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0.0f;
}

// ---- dropout (tensor.cpp:374-401): keep masks as bit words, element i = r * dim + c of the
// row-major rows x dim input (the reference's draw order), bit i%32 of word i/32 ----------
// y = keep ? x * inv_keep : 0  (one fp32 rounding, as `x.data()[i] * inv_keep`), in place.
__global__ void __launch_bounds__(256) dropout_apply_kernel(float* __restrict__ x, int64_t ldx, int64_t rows,
                                                            int32_t dim, const uint32_t* __restrict__ mask,
                                                            float inv_keep) {
    const int64_t total = rows * dim;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / dim;
        const int32_t c = static_cast<int32_t>(i - r * dim);
        const bool keep = (mask[i >> 5] >> (i & 31)) & 1u;
        float* p = x + r * ldx + c;
        *p = keep ? __fmul_rn(*p, inv_keep) : 0.0f;
    }
}

// The backward on a subset of the rows (the batch rows of the composed input, compose_rows'
// backward keeps only those): g[i, c] = keep(rows[i], c) ? g[i, c] * inv_keep : 0.
__global__ void __launch_bounds__(256) dropout_rows_bwd_kernel(float* __restrict__ g, int64_t ldg, int32_t m,
                                                               int32_t dim, const int32_t* __restrict__ rows,
                                                               const uint32_t* __restrict__ mask, float inv_keep) {
    const int64_t total = static_cast<int64_t>(m) * dim;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t r = static_cast<int32_t>(i / dim);
        const int32_t c = static_cast<int32_t>(i - static_cast<int64_t>(r) * dim);
        const int64_t e = static_cast<int64_t>(rows[r]) * dim + c;
        const bool keep = (mask[e >> 5] >> (e & 31)) & 1u;
        float* p = g + static_cast<int64_t>(r) * ldg + c;
        *p = keep ? __fmul_rn(*p, inv_keep) : 0.0f;
    }
}

// Philox4x32-10 keep masks: element i draws lane i%4 of philox(counter = i/4, key); keep =
// u >= p with u = (x >> 8) * 2^-24 (24-bit uniform, compared in double like next_double()).
__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
}
__global__ void __launch_bounds__(256) philox_mask_kernel(uint32_t* __restrict__ mask, int64_t count, uint64_t key,
                                                          double p) {
    const int64_t words = (count + 31) >> 5;
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t bits = 0;
        for (int q = 0; q < 8; ++q) {  // 8 philox calls x 4 lanes = 32 elements
            const uint64_t ctr = static_cast<uint64_t>(w) * 8 + q;
            uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32), c2 = 0, c3 = 0;
            uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
            for (int r = 0; r < 10; ++r) {
                philox_round(c0, c1, c2, c3, k0, k1);
                k0 += 0x9E3779B9u;
                k1 += 0xBB67AE85u;
            }
            const uint32_t x[4] = {c0, c1, c2, c3};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double u = static_cast<double>(x[j] >> 8) * 0x1.0p-24;
                if (u >= p) bits |= 1u << (q * 4 + j);
            }
        }
        if (w == words - 1 && (count & 31)) bits &= (1u << (count & 31)) - 1u;
        mask[w] = bits;
    }
}

// Dropout backward into an input that other ops also feed: g[i] += gin[i] * inv_keep where
// kept (tensor.cpp:393-396: `if (mask[i]) g[i] += gy[i] * inv_keep`, untouched otherwise).
__global__ void __launch_bounds__(256) dropout_bwd_acc_kernel(float* __restrict__ g, int64_t ldg, int64_t rows,
                                                              int32_t dim, const float* __restrict__ gin, int64_t ldi,
                                                              const uint32_t* __restrict__ mask, float inv_keep) {
    const int64_t total = rows * dim;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / dim;
        const int32_t c = static_cast<int32_t>(i - r * dim);
        if ((mask[i >> 5] >> (i & 31)) & 1u) {
            float* p = g + r * ldg + c;
            *p = __fadd_rn(*p, __fmul_rn(gin[r * ldi + c], inv_keep));
        }
    }
}

void launch_dropout_bwd_acc(float* g, int64_t ldg, int64_t rows, int32_t dim, const float* gin, int64_t ldi,
                            const uint32_t* mask, float inv_keep, cudaStream_t st) {
    const int64_t total = rows * dim;
    if (total <= 0) return;
    dropout_bwd_acc_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 8 * 148)), 256, 0, st>>>(
        g, ldg, rows, dim, gin, ldi, mask, inv_keep);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_dropout_apply(float* x, int64_t ldx, int64_t rows, int32_t dim, const uint32_t* mask, float inv_keep,
                          cudaStream_t st) {
    const int64_t total = rows * dim;
    if (total <= 0) return;
    dropout_apply_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 8 * 148)), 256, 0, st>>>(
        x, ldx, rows, dim, mask, inv_keep);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_dropout_rows_bwd(float* g, int64_t ldg, int32_t m, int32_t dim, const int32_t* rows, const uint32_t* mask,
                             float inv_keep, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(m) * dim;
    if (total <= 0) return;
    dropout_rows_bwd_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 8 * 148)), 256, 0, st>>>(
        g, ldg, m, dim, rows, mask, inv_keep);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_philox_mask(uint32_t* mask, int64_t count, uint64_t key, float p, cudaStream_t st) {
    const int64_t words = (count + 31) >> 5;
    if (words <= 0) return;
    philox_mask_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(words, 256), 8 * 148)), 256, 0, st>>>(
        mask, count, key, static_cast<double>(p));
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_zero(float* p, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    zero_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 256), 1184)), 256, 0, st>>>(p, count);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

}  // namespace gasb

// ---- op-level entry points: AdamState::step and grad_clip on caller buffers ------------
using namespace gasb;
namespace {
__global__ void scale_kernel(float* __restrict__ g, int64_t size, const double* __restrict__ norm, double max_norm) {
    const double nn = *norm;
    if (!(nn > max_norm)) return;
    const float s = static_cast<float>(__ddiv_rn(max_norm, nn));
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < size;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        g[i] = __fmul_rn(g[i], s);
}
}  // namespace

extern "C" gasb_status gasb_adam_step(float* d_p, float* d_m, float* d_v, const float* d_g, int64_t size, int64_t step,
                                      float lr, float beta1, float beta2, float eps, gasb_stream stream) {
    return guard([&] {
        require(size >= 0 && step >= 1, "adam_step: need size >= 0 and step >= 1");
        require(size == 0 || (d_p && d_m && d_v && d_g), "adam_step: null buffer");
        if (size == 0) return;
        cudaStream_t st = as_stream(stream);
        // bias corrections of step t on the host (std::pow, as nn.cpp:22-23), laid out for
        // adam_kernel: bc[0] = clamp step 1, bc[2..3] = (1 - b1^t, 1 - b2^t), counter 0
        double hb[4] = {1.0, 0.0, 1.0 - std::pow(static_cast<double>(beta1), static_cast<double>(step)),
                        1.0 - std::pow(static_cast<double>(beta2), static_cast<double>(step))};
        void* buf = nullptr;
        GASB_CUDA(cudaMallocAsync(&buf, 4 * sizeof(double) + sizeof(int64_t), st));
        double* bc = static_cast<double*>(buf);
        int64_t* counter = reinterpret_cast<int64_t*>(bc + 4);
        GASB_CUDA(cudaMemcpyAsync(bc, hb, sizeof(hb), cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemsetAsync(counter, 0, sizeof(int64_t), st));
        launch_adam(d_p, d_m, d_v, const_cast<float*>(d_g), size, counter, bc, lr, beta1, beta2, eps, 0.0f, nullptr,
                    st, nullptr, nullptr);
        GASB_CUDA(cudaFreeAsync(buf, st));
        GASB_CUDA(cudaStreamSynchronize(st));  // hb is a host stack buffer
    });
}

extern "C" gasb_status gasb_grad_clip(float* d_g, int64_t size, double max_norm, double* h_norm, gasb_stream stream) {
    return guard([&] {
        if (!(max_norm > 0.0)) throw std::invalid_argument("grad_clip: max_norm must be positive");
        require(size >= 0 && (size == 0 || d_g), "grad_clip: bad buffer");
        cudaStream_t st = as_stream(stream);
        double* scratch = nullptr;
        GASB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(double) * (kNormBlocks + 1), st));
        sumsq_kernel<<<kNormBlocks, 256, 0, st>>>(d_g, size, scratch);
        finish_norm_kernel<<<1, 1, 0, st>>>(scratch, kNormBlocks);
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(size, 256), 4 * 148));
        scale_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(d_g, size, scratch + kNormBlocks, max_norm);
        GASB_CUDA(cudaGetLastError());
        double nn = 0.0;
        GASB_CUDA(cudaMemcpyAsync(&nn, scratch + kNormBlocks, sizeof(double), cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaFreeAsync(scratch, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        if (h_norm) *h_norm = nn;
    });
}
