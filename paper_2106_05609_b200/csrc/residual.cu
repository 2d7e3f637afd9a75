// Elementwise ops of the residual GAS models — APPNP and GCNII (src/layers.cpp:150-168,
// src/trainer.cpp:142-163, :221-227) — with the reference's rounding sequence: every
// `scale` is one fp32 multiply and every `add` one fp32 add (built without FMA contraction,
// SURVEY App. A.8), so these kernels use __fmul_rn / __fadd_rn explicitly.
#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {

namespace {

// out[i,:] = alpha * h0[rows[i],:] + (1 - alpha) * prop[i,:]   (appnp/gcnii mixing)
// One warp per row; optional history push of the result (APPNP layers push `out` itself).
__global__ void __launch_bounds__(256) mix_kernel(const float* __restrict__ h0, int64_t ldh0,
                                                  const int32_t* __restrict__ rows, const float* __restrict__ prop,
                                                  int64_t ldp, int32_t m, int32_t d, float alpha, float one_m_alpha,
                                                  float* __restrict__ out, int64_t ldo, PushEpilogue push) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= m) return;
    const float* hr = h0 + static_cast<int64_t>(rows[w]) * ldh0;
    const float* pr = prop + w * ldp;
    float* orow = out + w * ldo;
    float* prow = nullptr;
    if (push.table) {
        const int32_t id = push.ids[w];
        prow = push.table + static_cast<int64_t>(id) * push.ld;
        if (lane == 0 && push.stamps) push.stamps[id] = *push.step;
    }
    int32_t flags = 0;
    for (int c = lane; c < d; c += 32) {
        const float v = __fadd_rn(__fmul_rn(hr[c], alpha), __fmul_rn(pr[c], one_m_alpha));
        orow[c] = v;
        if (prow) {
            prow[c] = v;
            flags |= table_flag_of(v);
        }
    }
    if (push.special) {
        flags = __reduce_or_sync(0xffffffffu, flags);
        if (lane == 0 && flags) atomicOr(push.special, flags);
    }
}

// wt[l] = (1 - beta) * I + beta * W[l] for all layers (gcnii W~, layers.cpp:166); d x d
// matrices with row pitch `pitch` (pad columns are 0 in W and stay 0 in wt)
__global__ void wtilde_kernel(const float* __restrict__ w, float* __restrict__ wt, int64_t total, int32_t d,
                              int64_t pitch, float beta, float one_m_beta) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e = i % (static_cast<int64_t>(d) * pitch);
        const float id = (e / pitch == e % pitch) ? 1.0f : 0.0f;
        wt[i] = __fadd_rn(__fmul_rn(id, one_m_beta), __fmul_rn(w[i], beta));
    }
}

// Backward of the mixing: dprop = (1 - alpha) * dmix; h0g[rows[i]] += alpha * dmix[i]
// (scale bwd then select_rows bwd, tensor.cpp:254-275, :434-457). Rows of one batch are
// distinct, so the read-modify-write of h0g is race-free.
// dmix and dprop may alias (in place: each element is read before it is written); h0g may be
// null (no h0 gradient wanted).
__global__ void __launch_bounds__(256) mix_bwd_kernel(const float* dmix, int64_t ldd, int32_t m, int32_t d,
                                                      float alpha, float one_m_alpha,
                                                      const int32_t* __restrict__ rows, float* __restrict__ h0g,
                                                      int64_t ldh, float* dprop, int64_t ldp) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= m) return;
    const float* g = dmix + w * ldd;
    float* hg = h0g ? h0g + static_cast<int64_t>(rows[w]) * ldh : nullptr;
    float* pg = dprop + w * ldp;
    for (int c = lane; c < d; c += 32) {
        const float v = g[c];
        pg[c] = __fmul_rn(one_m_alpha, v);
        if (hg) hg[c] = __fadd_rn(hg[c], __fmul_rn(alpha, v));
    }
}

// out[j] = float(sum_i double(g[i,j])) — add_rowvec's bias gradient (tensor.cpp:296-303).
// Block = 32 columns x 8 row groups; fp64 partials combined in a fixed order.
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ g, int64_t ldg, int32_t m, int32_t n,
                                                     float* __restrict__ out) {
    __shared__ double part[8][33];
    const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
    const int32_t col = blockIdx.x * 32 + cx;
    double acc = 0.0;
    if (col < n)
        for (int32_t i = ry; i < m; i += 8) acc += static_cast<double>(g[static_cast<int64_t>(i) * ldg + col]);
    part[ry][cx] = acc;
    __syncthreads();
    if (ry == 0 && col < n) {
        double s = part[0][cx];
        for (int k = 1; k < 8; ++k) s += part[k][cx];
        out[col] = static_cast<float>(s);
    }
}

// g = mask > 0 ? g : 0 (relu backward, tensor.cpp:363-369), in place.
__global__ void mask_kernel(float* __restrict__ g, int64_t ldg, const float* __restrict__ mask, int64_t ldm,
                            int32_t m, int32_t n) {
    // one warp per row (grid-stride), lanes across the columns: no per-element division
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < m;
         r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5)
        for (int32_t c = lane; c < n; c += 32)
            if (!(mask[r * ldm + c] > 0.0f)) g[r * ldg + c] = 0.0f;
}

unsigned grid_for(int64_t work, int threads) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads), 148 * 16)));
}

}  // namespace

void launch_mix(const float* h0, int64_t ldh0, const int32_t* rows, const float* prop, int64_t ldp, int32_t m,
                int32_t d, float alpha, float* out, int64_t ldo, const PushEpilogue* push, cudaStream_t st) {
    if (m <= 0) return;
    PushEpilogue pe{};
    if (push) pe = *push;
    const float one_m_alpha = 1.0f - alpha;  // float arithmetic, as `1.0f - cfg_.alpha`
    mix_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(m) * 32, 256)), 256, 0, st>>>(
        h0, ldh0, rows, prop, ldp, m, d, alpha, one_m_alpha, out, ldo, pe);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_wtilde(const float* w, float* wt, int32_t layers, int32_t d, int64_t pitch, float beta,
                   cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(layers) * d * pitch;
    if (total <= 0) return;
    wtilde_kernel<<<grid_for(total, 256), 256, 0, st>>>(w, wt, total, d, pitch, beta, 1.0f - beta);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_mix_bwd(const float* dmix, int64_t ldd, int32_t m, int32_t d, float alpha, const int32_t* rows,
                    float* h0g, int64_t ldh, float* dprop, int64_t ldp, cudaStream_t st) {
    if (m <= 0) return;
    mix_bwd_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(m) * 32, 256)), 256, 0, st>>>(
        dmix, ldd, m, d, alpha, 1.0f - alpha, rows, h0g, ldh, dprop, ldp);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

// Two-level column sum for tall inputs (APPNP/GCNII heads run over every V_b row: 585K rows
// at C4): CTA (x, y) sums rows y, y + R, ... of its 32 columns in fp64 (8 warps, fixed order),
// then one thread per column adds the R row-block partials in order. Deterministic.
__global__ void __launch_bounds__(256) colsum_partial_kernel(const float* __restrict__ g, int64_t ldg, int32_t m,
                                                             int32_t n, double* __restrict__ part) {
    __shared__ double sp[8][33];
    const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
    const int32_t col = blockIdx.x * 32 + cx;
    const int32_t R = gridDim.y;
    double acc = 0.0;
    if (col < n)
        for (int64_t i = static_cast<int64_t>(blockIdx.y) + static_cast<int64_t>(ry) * R; i < m;
             i += static_cast<int64_t>(8) * R)
            acc += static_cast<double>(g[i * ldg + col]);
    sp[ry][cx] = acc;
    __syncthreads();
    if (ry == 0 && col < n) {
        double s = sp[0][cx];
        for (int k = 1; k < 8; ++k) s += sp[k][cx];
        part[static_cast<int64_t>(blockIdx.y) * n + col] = s;
    }
}

__global__ void colsum_finish_kernel(const double* __restrict__ part, int32_t R, int32_t n, float* __restrict__ out) {
    const int32_t col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= n) return;
    double s = 0.0;
    for (int32_t r = 0; r < R; ++r) s += part[static_cast<int64_t>(r) * n + col];
    out[col] = static_cast<float>(s);
}

thread_local double* t_colsum_ws = nullptr;
thread_local int64_t t_colsum_ws_doubles = 0;
void set_colsum_workspace(double* ws, int64_t doubles) {
    t_colsum_ws = ws;
    t_colsum_ws_doubles = ws ? doubles : 0;
}

void launch_colsum(const float* g, int64_t ldg, int32_t m, int32_t n, float* out, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t cb = ceil_div(n, 32);
    int64_t R = std::min<int64_t>(ceil_div(m, 2048), std::max<int64_t>(1, 148 * 8 / cb));
    if (t_colsum_ws) R = std::min<int64_t>(R, t_colsum_ws_doubles / n);
    if (R <= 1 || !t_colsum_ws) {
        colsum_kernel<<<static_cast<unsigned>(cb), 256, 0, st>>>(g, ldg, m, n, out);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return;
    }
    colsum_partial_kernel<<<dim3(static_cast<unsigned>(cb), static_cast<unsigned>(R)), 256, 0, st>>>(g, ldg, m, n,
                                                                                                  t_colsum_ws);
    colsum_finish_kernel<<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, st>>>(t_colsum_ws,
                                                                                 static_cast<int32_t>(R), n, out);
    t_launches += 2;
    GASB_CUDA(cudaGetLastError());
}

void launch_mask(float* g, int64_t ldg, const float* mask, int64_t ldm, int32_t m, int32_t n, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(m) * n;
    if (total <= 0) return;
    launch_pdl(mask_kernel, dim3(grid_for(total, 256)), dim3(256), 0, st, g, ldg, mask, ldm, m, n);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

}  // namespace gasb
