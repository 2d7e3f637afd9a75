// History store in HBM: HistoryStore::push / pull (src/history.cpp:28-55) as vectorised,
// coalesced row scatter / gather kernels, plus the Prefetcher (history.cpp:184-252) as
// side-stream work ordered by CUDA events.
//
// Layout: L-1 tables, each num_nodes x ld fp32 (ld = dim rounded up to 4 floats, so every
// row starts 16 B aligned and moves as float4), one contiguous allocation; int64 stamps
// L-1 x num_nodes (-1 = never pushed); int64 step counter in device memory so that pushes
// captured into CUDA graphs stamp the live step.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>

#include "gasb_internal.hpp"
#include "kernels.cuh"

namespace gasb {

thread_local int64_t t_launches = 0;

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("GASB_PDL");  // off by default: C3 epoch 103.5 (off) vs 104.3 ms (on)
        return e && atoi(e) != 0;
    }();
    return on;
}
void check_launch(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// One warp moves R rows per round; each lane moves float4 (VEC=4) or float (VEC=1) columns.
// All loads of a round are issued before its stores to keep R*dim/128 requests in flight.
template <int VEC, int R>
__global__ void __launch_bounds__(256) rows_kernel(int mode, const int32_t* __restrict__ ids, int64_t count,
                                                   const float* __restrict__ src, int64_t lds,
                                                   float* __restrict__ dst, int64_t ldd, int32_t dim, int32_t n,
                                                   int64_t* __restrict__ stamps, const int64_t* __restrict__ step,
                                                   int32_t* __restrict__ err, int32_t* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t stamp = (mode == 0 && stamps) ? *step : 0;
    int32_t fl = 0;  // value flags of pushed rows (kernels.cuh kTableNeg / kTableNonFinite)
    for (int64_t base = warp * R; base < count; base += nwarps * R) {
        int64_t srow[R], drow[R];
        bool ok[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = base + r;
            ok[r] = i < count;
            int32_t id = ok[r] ? __ldg(ids + i) : 0;
            if (ok[r] && (id < 0 || id >= n)) {
                if (lane == 0) atomicAdd(err, 1);
                ok[r] = false;
            }
            srow[r] = mode == 0 ? i : id;
            drow[r] = mode == 0 ? id : i;
            if (ok[r] && mode == 0 && stamps && lane == 0) stamps[id] = stamp;
        }
        if constexpr (VEC == 4) {
            for (int c = lane * 4; c < dim; c += 128) {
                float4 v[R];
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (ok[r]) v[r] = __ldg(reinterpret_cast<const float4*>(src + srow[r] * lds + c));
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (ok[r]) {
                        *reinterpret_cast<float4*>(dst + drow[r] * ldd + c) = v[r];
                        if (flags)
                            fl |= table_flag_of(v[r].x) | table_flag_of(v[r].y) | table_flag_of(v[r].z) |
                                  table_flag_of(v[r].w);
                    }
            }
        } else {
            for (int c = lane; c < dim; c += 32) {
                float v[R];
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (ok[r]) v[r] = __ldg(src + srow[r] * lds + c);
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (ok[r]) {
                        dst[drow[r] * ldd + c] = v[r];
                        if (flags) fl |= table_flag_of(v[r]);
                    }
            }
        }
    }
    if (flags) {
        fl = __reduce_or_sync(0xffffffffu, fl);
        if (lane == 0 && fl) atomicOr(flags, fl);
    }
}

// Narrow rows (dim <= 64 floats, float4-aligned): a warp splits into 32 / LPR lane groups of
// LPR lanes, one row per group, so all 32 lanes move data (a 16-float row would otherwise
// leave 28 lanes idle).
template <int LPR, int R>
__global__ void __launch_bounds__(256) rows_narrow_kernel(int mode, const int32_t* __restrict__ ids, int64_t count,
                                                          const float* __restrict__ src, int64_t lds,
                                                          float* __restrict__ dst, int64_t ldd, int32_t dim, int32_t n,
                                                          int64_t* __restrict__ stamps,
                                                          const int64_t* __restrict__ step, int32_t* __restrict__ err,
                                                          int32_t* __restrict__ flags) {
    constexpr int G = 32 / LPR;  // rows per warp instruction
    const int lane = threadIdx.x & 31, grp = lane / LPR, sub = lane % LPR;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t stamp = (mode == 0 && stamps) ? *step : 0;
    int32_t fl = 0;
    for (int64_t base = warp * R * G; base < count; base += nwarps * R * G) {
        int64_t srow[R], drow[R];
        bool ok[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = base + r * G + grp;
            ok[r] = i < count;
            const int32_t id = ok[r] ? __ldg(ids + i) : 0;
            if (ok[r] && (id < 0 || id >= n)) {
                if (sub == 0) atomicAdd(err, 1);
                ok[r] = false;
            }
            srow[r] = mode == 0 ? i : id;
            drow[r] = mode == 0 ? id : i;
            if (ok[r] && mode == 0 && stamps && sub == 0) stamps[id] = stamp;
        }
        for (int c = sub * 4; c < dim; c += LPR * 4) {
            float4 v[R];
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (ok[r]) v[r] = __ldg(reinterpret_cast<const float4*>(src + srow[r] * lds + c));
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (ok[r]) {
                    *reinterpret_cast<float4*>(dst + drow[r] * ldd + c) = v[r];
                    if (flags)
                        fl |= table_flag_of(v[r].x) | table_flag_of(v[r].y) | table_flag_of(v[r].z) |
                              table_flag_of(v[r].w);
                }
        }
    }
    if (flags) {
        fl = __reduce_or_sync(0xffffffffu, fl);
        if (lane == 0 && fl) atomicOr(flags, fl);
    }
}

__global__ void advance_step_kernel(int64_t* step) { *step += 1; }

__global__ void fill_stamps_kernel(int64_t* stamps, int64_t n, const int64_t* step) {
    const int64_t s = *step;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        stamps[i] = s;
}

// measure_staleness (history.cpp:77-112), per row: norm[v] = sqrt(sum_j (double(a_j) -
// double(b_j))^2) in column order without contraction (the reference's loop, bit for bit),
// age[v] = stamp < 0 ? step + 1 : step - stamp. One thread per row: the row sum is
// sequential by definition; the cross-row sums are done on the host in row order.
__global__ void __launch_bounds__(256) staleness_rows_kernel(const float* __restrict__ a, int64_t lda,
                                                             const float* __restrict__ b, int64_t ldb, int32_t n,
                                                             int32_t dim, const int64_t* __restrict__ stamps,
                                                             const int64_t* __restrict__ step,
                                                             double* __restrict__ norm, int64_t* __restrict__ age) {
    const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const float* ra = a + v * lda;
    const float* rb = b + v * ldb;
    double acc = 0.0;
    for (int32_t j = 0; j < dim; ++j) {
        const double d = __dsub_rn(static_cast<double>(ra[j]), static_cast<double>(rb[j]));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    norm[v] = __dsqrt_rn(acc);
    const int64_t st = stamps[v], s = *step;
    age[v] = st < 0 ? s + 1 : s - st;
}

static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (!g_num_sms) g_num_sms = 148;
    }
    return g_num_sms;
}

void launch_rows(int mode, const int32_t* ids, int64_t count, const float* src, int64_t lds, float* dst, int64_t ldd,
                 int32_t dim, int32_t n, int64_t* stamps, const int64_t* step, int32_t* err, cudaStream_t st,
                 int32_t* flags) {
    if (count <= 0) return;
    const bool vec4 = (dim % 4 == 0) && (lds % 4 == 0) && (ldd % 4 == 0) &&
                      (reinterpret_cast<uintptr_t>(src) % 16 == 0) && (reinterpret_cast<uintptr_t>(dst) % 16 == 0);
    constexpr int R = 4;
    if (vec4 && dim <= 64) {
        const int lpr = dim <= 16 ? 4 : dim <= 32 ? 8 : 16;  // lanes per row (float4 each)
        const int64_t warps_needed = ceil_div(count, static_cast<int64_t>(R) * (32 / lpr));
        const int64_t blocks = std::min<int64_t>(ceil_div(warps_needed, 8), static_cast<int64_t>(num_sms()) * 8);
#define GASB_NARROW(L)                                                                                            \
    rows_narrow_kernel<L, R><<<static_cast<unsigned>(blocks), 256, 0, st>>>(mode, ids, count, src, lds, dst, ldd, \
                                                                            dim, n, stamps, step, err, flags)
        if (lpr == 4) GASB_NARROW(4);
        else if (lpr == 8) GASB_NARROW(8);
        else GASB_NARROW(16);
#undef GASB_NARROW
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        return;
    }
    const int64_t warps_needed = ceil_div(count, R);
    const int64_t blocks = std::min<int64_t>(ceil_div(warps_needed, 8), static_cast<int64_t>(num_sms()) * 8);
    if (vec4)
        rows_kernel<4, R><<<static_cast<unsigned>(blocks), 256, 0, st>>>(mode, ids, count, src, lds, dst, ldd, dim, n,
                                                                         stamps, step, err, flags);
    else
        rows_kernel<1, R><<<static_cast<unsigned>(blocks), 256, 0, st>>>(mode, ids, count, src, lds, dst, ldd, dim, n,
                                                                         stamps, step, err, flags);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

void launch_advance_step(int64_t* step, cudaStream_t st) {
    advance_step_kernel<<<1, 1, 0, st>>>(step);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

}  // namespace gasb

using namespace gasb;

struct gasb_history_s {
    int32_t layers = 0, n = 0, dim = 0;
    int64_t ld = 0;
    float* tables = nullptr;
    int64_t* stamps = nullptr;
    int64_t* step = nullptr;
    int32_t* err = nullptr;
    int32_t* flags = nullptr;  // per layer: OR of table_flag_of over every value ever stored

    bool released = false;  // tables handed over to a sharded data-parallel group (dp.cu)
    float* table(int32_t layer) const { return tables + static_cast<int64_t>(layer - 1) * n * ld; }
    int64_t* stamp(int32_t layer) const { return stamps + static_cast<int64_t>(layer - 1) * n; }
    int32_t* flag(int32_t layer) const { return flags + (layer - 1); }
    void check_layer(int32_t layer) const {
        if (released)
            throw std::logic_error("HistoryStore: the tables are sharded across a data-parallel group "
                                   "(read them through gasb_dp_read_history)");
        if (layer < 1 || layer > layers)
            throw std::invalid_argument("HistoryStore: layer " + std::to_string(layer) + " out of range [1," +
                                        std::to_string(layers) + "]");
    }
    ~gasb_history_s() {
        cudaFree(tables);
        cudaFree(stamps);
        cudaFree(step);
        cudaFree(err);
        cudaFree(flags);
    }
};

struct gasb_prefetcher_s {
    gasb_history h = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t start = nullptr;
    std::vector<cudaEvent_t> ready;
    std::vector<float*> bufs;
    int64_t capacity = 0;  // rows per layer buffer
    uint64_t generation = 0;
    ~gasb_prefetcher_s() {
        if (side) cudaStreamSynchronize(side);
        for (float* b : bufs) cudaFree(b);
        for (cudaEvent_t e : ready) cudaEventDestroy(e);
        if (start) cudaEventDestroy(start);
        if (side) cudaStreamDestroy(side);
    }
};

namespace gasb {
// Shared with trainer.cu: create a history store on the current device.
gasb_history history_create(int32_t layers, int32_t n, int32_t dim) {
    require(layers >= 0 && n >= 0 && dim >= 0, "HistoryStore: negative shape");
    auto* h = new gasb_history_s();
    try {
        h->layers = layers;
        h->n = n;
        h->dim = dim;
        h->ld = round_up(std::max<int64_t>(dim, 1), 4);
        const int64_t tab = static_cast<int64_t>(layers) * n * h->ld;
        GASB_CUDA(cudaMalloc(&h->tables, sizeof(float) * std::max<int64_t>(tab, 1)));
        GASB_CUDA(cudaMemset(h->tables, 0, sizeof(float) * std::max<int64_t>(tab, 1)));
        const int64_t ns = static_cast<int64_t>(layers) * n;
        GASB_CUDA(cudaMalloc(&h->stamps, sizeof(int64_t) * std::max<int64_t>(ns, 1)));
        GASB_CUDA(cudaMemset(h->stamps, 0xFF, sizeof(int64_t) * std::max<int64_t>(ns, 1)));
        GASB_CUDA(cudaMalloc(&h->step, sizeof(int64_t)));
        GASB_CUDA(cudaMemset(h->step, 0, sizeof(int64_t)));
        GASB_CUDA(cudaMalloc(&h->err, sizeof(int32_t)));
        GASB_CUDA(cudaMemset(h->err, 0, sizeof(int32_t)));
        GASB_CUDA(cudaMalloc(&h->flags, sizeof(int32_t) * std::max(layers, 1)));
        GASB_CUDA(cudaMemset(h->flags, 0, sizeof(int32_t) * std::max(layers, 1)));  // zero tables
        GASB_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}
float* history_table(gasb_history h, int32_t layer) { return h->table(layer); }
int64_t history_ld(gasb_history h) { return h->ld; }
int64_t* history_stamps(gasb_history h, int32_t layer) { return h->stamp(layer); }
int64_t* history_step_ptr(gasb_history h) { return h->step; }
int32_t* history_flags(gasb_history h, int32_t layer) { return h->flag(layer); }
void history_destroy(gasb_history h) { delete h; }
// Frees the tables (stamps, flags and the step counter stay): a sharded data-parallel group
// keeps each rank's rows in its exchange region instead.
void history_release_tables(gasb_history h) {
    cudaDeviceSynchronize();
    cudaFree(h->tables);
    h->tables = nullptr;
    h->released = true;
}
}  // namespace gasb

extern "C" {

gasb_status gasb_history_create(int32_t layers, int32_t n, int32_t dim, gasb_history* out) {
    return guard([&] {
        require(out != nullptr, "HistoryStore: null out");
        *out = history_create(layers, n, dim);
    });
}

gasb_status gasb_history_destroy(gasb_history h) {
    delete h;
    return GASB_OK;
}

gasb_status gasb_history_info(gasb_history h, int32_t* layers, int32_t* n, int32_t* dim, int64_t* ld) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        if (layers) *layers = h->layers;
        if (n) *n = h->n;
        if (dim) *dim = h->dim;
        if (ld) *ld = h->ld;
    });
}

gasb_status gasb_history_push(gasb_history h, int32_t layer, const int32_t* ids, int64_t count, const float* rows,
                              int64_t ld_rows, gasb_stream stream) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        h->check_layer(layer);
        require(count >= 0 && (count == 0 || (ids && rows)) && ld_rows >= h->dim,
                "HistoryStore::push: row count mismatch");
        launch_rows(0, ids, count, rows, ld_rows, h->table(layer), h->ld, h->dim, h->n, h->stamp(layer), h->step,
                    h->err, as_stream(stream), h->flag(layer));
    });
}

gasb_status gasb_history_pull(gasb_history h, int32_t layer, const int32_t* ids, int64_t count, float* out,
                              int64_t ld_out, gasb_stream stream) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        h->check_layer(layer);
        require(count >= 0 && (count == 0 || (ids && out)) && ld_out >= h->dim, "HistoryStore::pull: bad output");
        launch_rows(1, ids, count, h->table(layer), h->ld, out, ld_out, h->dim, h->n, nullptr, nullptr, h->err,
                    as_stream(stream));
    });
}

gasb_status gasb_history_check(gasb_history h) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        int32_t e = 0;
        GASB_CUDA(cudaDeviceSynchronize());
        GASB_CUDA(cudaMemcpy(&e, h->err, sizeof(e), cudaMemcpyDeviceToHost));
        if (e) {
            GASB_CUDA(cudaMemset(h->err, 0, sizeof(int32_t)));
            throw std::invalid_argument("HistoryStore: node id out of range (" + std::to_string(e) + " rows)");
        }
    });
}

static void host_ids_check(gasb_history h, const int32_t* ids, int64_t count, const char* what) {
    for (int64_t i = 0; i < count; ++i)
        if (ids[i] < 0 || ids[i] >= h->n) throw std::invalid_argument(std::string(what) + ": node id out of range");
}

gasb_status gasb_history_push_host(gasb_history h, int32_t layer, const int32_t* ids, int64_t count,
                                   const float* rows, gasb_stream stream) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        h->check_layer(layer);
        require(count >= 0, "HistoryStore::push: row count mismatch");
        host_ids_check(h, ids, count, "HistoryStore::push");
        if (count == 0) return;
        cudaStream_t st = as_stream(stream);
        int32_t* d_ids = nullptr;
        float* d_rows = nullptr;
        GASB_CUDA(cudaMallocAsync(&d_ids, sizeof(int32_t) * count, st));
        GASB_CUDA(cudaMallocAsync(&d_rows, sizeof(float) * count * h->dim, st));
        GASB_CUDA(cudaMemcpyAsync(d_ids, ids, sizeof(int32_t) * count, cudaMemcpyHostToDevice, st));
        GASB_CUDA(cudaMemcpyAsync(d_rows, rows, sizeof(float) * count * h->dim, cudaMemcpyHostToDevice, st));
        launch_rows(0, d_ids, count, d_rows, h->dim, h->table(layer), h->ld, h->dim, h->n, h->stamp(layer), h->step,
                    h->err, st, h->flag(layer));
        GASB_CUDA(cudaFreeAsync(d_ids, st));
        GASB_CUDA(cudaFreeAsync(d_rows, st));
        GASB_CUDA(cudaStreamSynchronize(st));
    });
}

gasb_status gasb_history_pull_host(gasb_history h, int32_t layer, const int32_t* ids, int64_t count, float* out,
                                   gasb_stream stream) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        h->check_layer(layer);
        require(count >= 0, "HistoryStore::pull: negative count");
        host_ids_check(h, ids, count, "HistoryStore::pull");
        if (count == 0) return;
        cudaStream_t st = as_stream(stream);
        int32_t* d_ids = nullptr;
        float* d_out = nullptr;
        GASB_CUDA(cudaMallocAsync(&d_ids, sizeof(int32_t) * count, st));
        GASB_CUDA(cudaMallocAsync(&d_out, sizeof(float) * count * h->dim, st));
        GASB_CUDA(cudaMemcpyAsync(d_ids, ids, sizeof(int32_t) * count, cudaMemcpyHostToDevice, st));
        launch_rows(1, d_ids, count, h->table(layer), h->ld, d_out, h->dim, h->dim, h->n, nullptr, nullptr, h->err, st);
        GASB_CUDA(cudaMemcpyAsync(out, d_out, sizeof(float) * count * h->dim, cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaFreeAsync(d_ids, st));
        GASB_CUDA(cudaFreeAsync(d_out, st));
        GASB_CUDA(cudaStreamSynchronize(st));
    });
}

gasb_status gasb_history_advance_step(gasb_history h, gasb_stream stream) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        launch_advance_step(h->step, as_stream(stream));
    });
}

gasb_status gasb_history_step(gasb_history h, int64_t* out) {
    return guard([&] {
        require(h && out, "HistoryStore: null argument");
        GASB_CUDA(cudaDeviceSynchronize());
        GASB_CUDA(cudaMemcpy(out, h->step, sizeof(int64_t), cudaMemcpyDeviceToHost));
    });
}

gasb_status gasb_history_last_push_step(gasb_history h, int32_t layer, int32_t v, int64_t* out) {
    return guard([&] {
        require(h && out, "HistoryStore: null argument");
        h->check_layer(layer);
        require(v >= 0 && v < h->n, "HistoryStore: node id out of range");
        GASB_CUDA(cudaDeviceSynchronize());
        GASB_CUDA(cudaMemcpy(out, h->stamp(layer) + v, sizeof(int64_t), cudaMemcpyDeviceToHost));
    });
}

gasb_status gasb_history_layer(gasb_history h, int32_t layer, float** table, int64_t* ld) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        h->check_layer(layer);
        if (table) *table = h->table(layer);
        if (ld) *ld = h->ld;
    });
}

gasb_status gasb_history_fill_layer(gasb_history h, int32_t layer, const float* values) {
    return guard([&] {
        require(h && values, "HistoryStore: null argument");
        h->check_layer(layer);
        GASB_CUDA(cudaDeviceSynchronize());
        GASB_CUDA(cudaMemcpy2D(h->table(layer), sizeof(float) * h->ld, values, sizeof(float) * h->dim,
                               sizeof(float) * h->dim, h->n, cudaMemcpyHostToDevice));
        if (h->n > 0) fill_stamps_kernel<<<256, 256>>>(h->stamp(layer), h->n, h->step);
        GASB_CUDA(cudaMemset(h->flag(layer), 0, sizeof(int32_t)));  // the table is replaced whole
        launch_scan_special(h->table(layer), h->n, h->ld, h->dim, h->flag(layer), nullptr);
        GASB_CUDA(cudaGetLastError());
        GASB_CUDA(cudaDeviceSynchronize());
    });
}

gasb_status gasb_history_read_layer(gasb_history h, int32_t layer, float* values) {
    return guard([&] {
        require(h && values, "HistoryStore: null argument");
        h->check_layer(layer);
        GASB_CUDA(cudaDeviceSynchronize());
        GASB_CUDA(cudaMemcpy2D(values, sizeof(float) * h->dim, h->table(layer), sizeof(float) * h->ld,
                               sizeof(float) * h->dim, h->n, cudaMemcpyDeviceToHost));
    });
}

gasb_status gasb_history_read_stamps(gasb_history h, int32_t layer, int64_t* stamps) {
    return guard([&] {
        require(h && stamps, "HistoryStore: null argument");
        h->check_layer(layer);
        GASB_CUDA(cudaDeviceSynchronize());
        GASB_CUDA(cudaMemcpy(stamps, h->stamp(layer), sizeof(int64_t) * h->n, cudaMemcpyDeviceToHost));
    });
}

gasb_status gasb_history_reset(gasb_history h) {
    return guard([&] {
        require(h, "HistoryStore: null handle");
        GASB_CUDA(cudaDeviceSynchronize());
        const int64_t tab = static_cast<int64_t>(h->layers) * h->n * h->ld;
        if (tab) GASB_CUDA(cudaMemset(h->tables, 0, sizeof(float) * tab));
        const int64_t ns = static_cast<int64_t>(h->layers) * h->n;
        if (ns) GASB_CUDA(cudaMemset(h->stamps, 0xFF, sizeof(int64_t) * ns));
        GASB_CUDA(cudaMemset(h->step, 0, sizeof(int64_t)));
        GASB_CUDA(cudaMemset(h->flags, 0, sizeof(int32_t) * std::max(h->layers, 1)));
        GASB_CUDA(cudaDeviceSynchronize());
    });
}

gasb_status gasb_prefetcher_create(gasb_history h, gasb_prefetcher* out) {
    return guard([&] {
        require(h && out, "Prefetcher: null argument");
        auto* p = new gasb_prefetcher_s();
        try {
            p->h = h;
            GASB_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
            GASB_CUDA(cudaEventCreateWithFlags(&p->start, cudaEventDisableTiming));
            p->ready.resize(static_cast<size_t>(h->layers));
            p->bufs.assign(static_cast<size_t>(h->layers), nullptr);
            for (auto& e : p->ready) GASB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

gasb_status gasb_prefetcher_destroy(gasb_prefetcher p) {
    delete p;
    return GASB_OK;
}

gasb_status gasb_prefetch_begin(gasb_prefetcher p, const int32_t* d_halo, int64_t count, gasb_stream compute,
                                uint64_t* generation) {
    return guard([&] {
        require(p && generation && count >= 0, "Prefetcher: bad argument");
        gasb_history h = p->h;
        if (count > p->capacity) {  // grow (synchronizes the side stream first)
            GASB_CUDA(cudaStreamSynchronize(p->side));
            for (auto& b : p->bufs) {
                cudaFree(b);
                b = nullptr;
                GASB_CUDA(cudaMalloc(&b, sizeof(float) * count * h->ld));
            }
            p->capacity = count;
        }
        ++p->generation;
        GASB_CUDA(cudaEventRecord(p->start, as_stream(compute)));
        GASB_CUDA(cudaStreamWaitEvent(p->side, p->start, 0));
        for (int32_t l = 1; l <= h->layers; ++l) {
            launch_rows(1, d_halo, count, h->table(l), h->ld, p->bufs[l - 1], h->ld, h->dim, h->n, nullptr, nullptr,
                        h->err, p->side);
            GASB_CUDA(cudaEventRecord(p->ready[l - 1], p->side));
        }
        *generation = p->generation;
    });
}

gasb_status gasb_prefetch_wait(gasb_prefetcher p, uint64_t generation, int32_t layer, gasb_stream compute,
                               const float** rows, int64_t* ld) {
    return guard([&] {
        require(p, "Prefetcher: null handle");
        if (layer < 1 || layer > p->h->layers)
            throw std::invalid_argument("Prefetcher: layer " + std::to_string(layer) + " was never requested");
        if (generation != p->generation)
            throw std::logic_error("Prefetcher: handle does not match the active batch");
        GASB_CUDA(cudaStreamWaitEvent(as_stream(compute), p->ready[layer - 1], 0));
        if (rows) *rows = p->bufs[layer - 1];
        if (ld) *ld = p->h->ld;
    });
}

/* measure_staleness (history.cpp:77-112). */
gasb_status gasb_history_staleness(gasb_history h, const float* const* d_reference, const int64_t* ld_reference,
                                   double* h_eps_max, double* h_eps_mean, int64_t* h_age_max, double* h_age_mean) {
    return guard([&] {
        require(h && d_reference && ld_reference, "measure_staleness: null argument");
        require(h_eps_max && h_eps_mean && h_age_max && h_age_mean, "measure_staleness: null argument");
        // as every other host accessor: the trainer's streams are non-blocking, so wait for its
        // in-flight pushes and step updates before reading the tables
        GASB_CUDA(cudaDeviceSynchronize());
        const int64_t n = h->n;
        double* d_norm = nullptr;
        int64_t* d_age = nullptr;
        GASB_CUDA(cudaMalloc(&d_norm, sizeof(double) * std::max<int64_t>(n, 1)));
        GASB_CUDA(cudaMalloc(&d_age, sizeof(int64_t) * std::max<int64_t>(n, 1)));
        std::vector<double> norm(static_cast<size_t>(n));
        std::vector<int64_t> age(static_cast<size_t>(n));
        try {
            for (int32_t l = 1; l <= h->layers; ++l) {
                require(d_reference[l - 1] != nullptr, "measure_staleness: need one reference matrix per layer");
                require(ld_reference[l - 1] >= h->dim, "measure_staleness: reference shape mismatch");
                if (n > 0) {
                    staleness_rows_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256>>>(
                        h->table(l), h->ld, d_reference[l - 1], ld_reference[l - 1], h->n, h->dim, h->stamp(l),
                        h->step, d_norm, d_age);
                    ++t_launches;
                    GASB_CUDA(cudaGetLastError());
                    GASB_CUDA(cudaMemcpy(norm.data(), d_norm, sizeof(double) * n, cudaMemcpyDeviceToHost));
                    GASB_CUDA(cudaMemcpy(age.data(), d_age, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
                }
                double sum = 0.0, mx = 0.0, age_sum = 0.0;  // row order, as the reference
                int64_t age_max = 0;
                for (int64_t v = 0; v < n; ++v) {
                    sum += norm[v];
                    mx = std::max(mx, norm[v]);
                    age_sum += static_cast<double>(age[v]);
                    age_max = std::max(age_max, age[v]);
                }
                h_eps_max[l - 1] = mx;
                h_eps_mean[l - 1] = n > 0 ? sum / static_cast<double>(n) : 0.0;
                h_age_max[l - 1] = age_max;
                h_age_mean[l - 1] = n > 0 ? age_sum / static_cast<double>(n) : 0.0;
            }
        } catch (...) {
            cudaFree(d_norm);
            cudaFree(d_age);
            throw;
        }
        cudaFree(d_norm);
        cudaFree(d_age);
    });
}

/* save_checkpoint (history.cpp:130-148): "GASH", u32 layers, u32 nodes, u32 dim, then each
 * layer's rows x dim fp32 values, row-major, dense (the reference's byte format). */
gasb_status gasb_history_save(gasb_history h, const char* path) {
    return guard([&] {
        require(h && path, "checkpoint: null argument");
        GASB_CUDA(cudaDeviceSynchronize());
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw std::runtime_error(std::string("checkpoint: cannot open ") + path);
        std::vector<float> buf(static_cast<size_t>(h->n) * h->dim);
        try {
            const uint32_t hdr[3] = {static_cast<uint32_t>(h->layers), static_cast<uint32_t>(h->n),
                                     static_cast<uint32_t>(h->dim)};
            if (std::fwrite("GASH", 1, 4, f) != 4 || std::fwrite(hdr, sizeof(uint32_t), 3, f) != 3)
                throw std::runtime_error("checkpoint: write failed");
            for (int32_t l = 1; l <= h->layers; ++l) {
                if (buf.empty()) continue;
                GASB_CUDA(cudaMemcpy2D(buf.data(), sizeof(float) * h->dim, h->table(l), sizeof(float) * h->ld,
                                       sizeof(float) * h->dim, h->n, cudaMemcpyDeviceToHost));
                if (std::fwrite(buf.data(), sizeof(float), buf.size(), f) != buf.size())
                    throw std::runtime_error("checkpoint: write failed");
            }
        } catch (...) {
            std::fclose(f);
            throw;
        }
        std::fclose(f);
    });
}

/* load_checkpoint (history.cpp:150-178): a new store with the file's tables, every stamp 0
 * and step 0; runtime_error for an unopenable file, bad magic or truncation. */
gasb_status gasb_history_load(const char* path, gasb_history* out) {
    return guard([&] {
        require(path && out, "checkpoint: null argument");
        std::FILE* f = std::fopen(path, "rb");
        if (!f) throw std::runtime_error(std::string("checkpoint: cannot open ") + path);
        gasb_history h = nullptr;
        try {
            char magic[4];
            if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "GASH", 4) != 0)
                throw std::runtime_error(std::string("checkpoint: bad magic in ") + path);
            uint32_t hdr[3];
            for (int i = 0; i < 3; ++i)
                if (std::fread(hdr + i, sizeof(uint32_t), 1, f) != 1)
                    throw std::runtime_error("checkpoint: truncated header");
            h = history_create(static_cast<int32_t>(hdr[0]), static_cast<int32_t>(hdr[1]),
                               static_cast<int32_t>(hdr[2]));
            std::vector<float> buf(static_cast<size_t>(h->n) * h->dim);
            for (int32_t l = 1; l <= h->layers; ++l) {
                if (!buf.empty()) {
                    if (std::fread(buf.data(), sizeof(float), buf.size(), f) != buf.size())
                        throw std::runtime_error(std::string("checkpoint: truncated matrix in ") + path);
                    GASB_CUDA(cudaMemcpy2D(h->table(l), sizeof(float) * h->ld, buf.data(), sizeof(float) * h->dim,
                                           sizeof(float) * h->dim, h->n, cudaMemcpyHostToDevice));
                    int32_t fl = 0;
                    for (float v : buf) fl |= table_flag_of(v);
                    GASB_CUDA(cudaMemcpy(h->flag(l), &fl, sizeof(fl), cudaMemcpyHostToDevice));
                }
                if (h->n > 0) GASB_CUDA(cudaMemset(h->stamp(l), 0, sizeof(int64_t) * h->n));
            }
        } catch (...) {
            std::fclose(f);
            if (h) history_destroy(h);
            throw;
        }
        std::fclose(f);
        *out = h;
    });
}

}  // extern "C"
