// GPU batch-plan builder: BatchSchedule::build for every part at once.
//
// Same outputs, bit for bit, as the host builder in graph_host.cpp (pinned against the
// reference's make_batch_plan, src/graph.cpp:78-134, and build_plan_aggregation,
// src/layers.cpp:42-70). The reference marks V_b in an O(n) flag array per batch
// (graph.cpp:92-99) and scans it in id order; here every part's flag array is one row of
// a part x n bitmap set by all batches concurrently, and the id-ordered scan becomes a
// popcount prefix over the bitmap words:
//
//   1. stable radix sort of (part, node) -> the batches, ids ascending inside a part
//      (partition_from_assignment, partition.cpp:314-328); part range / emptiness checks
//   2. bitmap[p][w] = w in V_b(p): one warp per batch row sets its node and its CSR row
//   3. popcount + exclusive scan over the words (part-major) -> ext offsets and, for any
//      (p, w) in V_b(p), local id lid(p, w) = wpre[word] - wpre[part start] + popc(prefix bits)
//   4. extended / is_halo / halo / halo_local_rows from the set bits in word order
//      (a halo's rank = local id - #batch nodes below it, a binary search in the batch)
//   5. gcn stencil rows in CSR order, coefficient float(1 / (sqrt(dw+1) * sqrt(dv+1))) in
//      fp64 (IEEE sqrt / mul / div: the host's values exactly), the self term appended at the
//      row end when the row has no stored self-loop; optional local graph and sum stencil.
//
// The bitmap is bounded (bitmap_budget()): parts are processed in groups when P x n bits
// exceed it (C5-sized graphs). Results land in device arrays and are copied into the
// schedule's HostPlans, so every consumer of a schedule (trainer, plan_copy) is unchanged.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gasb_internal.hpp"

namespace gasb {
namespace {

// bytes of part x node bitmap per group (GASB_PLAN_BITMAP_BYTES overrides it: tests force groups)
int64_t bitmap_budget() {
    const char* e = std::getenv("GASB_PLAN_BITMAP_BYTES");
    return e ? std::max<int64_t>(4, std::atoll(e)) : int64_t(1) << 30;
}

template <class T>
struct DArr {
    T* p = nullptr;
    int64_t n = 0;
    explicit DArr(int64_t count = 0) { alloc(count); }
    void alloc(int64_t count) {
        free();
        n = count;
        if (count > 0) GASB_CUDA(cudaMalloc(&p, sizeof(T) * count));
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DArr() { free(); }
    DArr(const DArr&) = delete;
    DArr& operator=(const DArr&) = delete;
};

__global__ void check_parts_kernel(const int32_t* __restrict__ asg, int32_t n, int32_t P, int32_t* bad) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
        const int32_t a = asg[v];
        if (a < 0 || a >= P) atomicOr(bad, 1);
    }
}

__global__ void iota_kernel(int32_t* __restrict__ out, int32_t n) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x)
        out[v] = static_cast<int32_t>(v);
}

// part_off[q] = first sorted index whose part >= q (q = 0 .. P)
__global__ void part_bounds_kernel(const int32_t* __restrict__ keys, int32_t n, int32_t P, int64_t* __restrict__ part_off) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q > P) return;
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = lo + (hi - lo) / 2;
        if (keys[mid] < q) lo = mid + 1;
        else hi = mid;
    }
    part_off[q] = lo;
}

// cs[v] = sqrt(double(degree(v)) + 1.0) (layers.cpp:42-70 via the host restatement)
__global__ void degree_sqrt_kernel(const int64_t* __restrict__ ro, int32_t n, double* __restrict__ cs) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
        const int32_t deg = static_cast<int32_t>(ro[v + 1] - ro[v]);
        cs[v] = __dsqrt_rn(static_cast<double>(deg) + 1.0);
    }
}

// Row lengths in sorted (batch) order: gcn = deg + [no stored self-loop], sum = deg.
__global__ void row_len_kernel(const int32_t* __restrict__ order, const int64_t* __restrict__ ro,
                               const int32_t* __restrict__ cols, int32_t n, int64_t* __restrict__ glen,
                               int64_t* __restrict__ slen) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t v = order[i];
        int64_t lo = ro[v], hi = ro[v + 1];
        const int64_t deg = hi - lo;
        while (lo < hi) {  // cols strictly increasing per row
            const int64_t mid = lo + (hi - lo) / 2;
            if (cols[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        const bool self = lo < ro[v + 1] && cols[lo] == v;
        glen[i] = deg + (self ? 0 : 1);
        if (slen) slen[i] = deg;
    }
}

// One warp per batch row of the group: set the row's node and its in-neighbours in its
// part's bitmap row.
__global__ void mark_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ asg,
                            const int64_t* __restrict__ ro, const int32_t* __restrict__ cols, int64_t i0, int64_t i1,
                            int32_t p0, int64_t W, uint32_t* __restrict__ bm) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = i0 + ((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5); i < i1; i += nwarps) {
        const int32_t v = order[i];
        uint32_t* row = bm + (asg[v] - p0) * W;
        if (lane == 0) atomicOr(row + (v >> 5), 1u << (v & 31));
        for (int64_t e = ro[v] + lane; e < ro[v + 1]; e += 32) {
            const int32_t w = cols[e];
            atomicOr(row + (w >> 5), 1u << (w & 31));
        }
    }
}

__global__ void popc_kernel(const uint32_t* __restrict__ bm, int64_t words, int64_t* __restrict__ cnt) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < words; k += int64_t(gridDim.x) * blockDim.x)
        cnt[k] = __popc(bm[k]);
}

struct GroupView {
    const uint32_t* bm;   // (p1 - p0) x W
    const int64_t* wpre;  // exclusive prefix of popcounts over the group's words (+ total)
    int64_t W;
    int32_t p0;
    __device__ __forceinline__ int32_t lid(int32_t p, int32_t w) const {
        const int64_t base = static_cast<int64_t>(p - p0) * W;
        const int64_t k = base + (w >> 5);
        return static_cast<int32_t>(wpre[k] - wpre[base] + __popc(bm[k] & ((1u << (w & 31)) - 1u)));
    }
};

__device__ __forceinline__ int32_t lower_bound_i32(const int32_t* a, int32_t n, int32_t x) {
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = lo + (hi - lo) / 2;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Step 4: one thread per bitmap word; set bits in ascending node order.
__global__ void emit_ext_kernel(GroupView g, int64_t words, int64_t ext_base, const int32_t* __restrict__ asg,
                                const int32_t* __restrict__ order, const int64_t* __restrict__ part_off,
                                int32_t* __restrict__ ext, uint8_t* __restrict__ is_halo, int32_t* __restrict__ halo,
                                int32_t* __restrict__ hlr) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < words; k += int64_t(gridDim.x) * blockDim.x) {
        uint32_t bits = g.bm[k];
        if (!bits) continue;
        const int32_t pl = static_cast<int32_t>(k / g.W);
        const int32_t p = g.p0 + pl;
        const int64_t pstart = g.wpre[pl * g.W];
        const int64_t ext_off = ext_base + pstart;          // global start of part p's extended list
        const int64_t halo_off = ext_off - part_off[p];     // sum over earlier parts of (ne - nb)
        const int32_t* batch = order + part_off[p];
        const int32_t nb = static_cast<int32_t>(part_off[p + 1] - part_off[p]);
        int32_t local = static_cast<int32_t>(g.wpre[k] - pstart);
        const int32_t wbase = static_cast<int32_t>((k - pl * g.W) << 5);
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int32_t w = wbase + b;
            const bool h = asg[w] != p;
            ext[ext_off + local] = w;
            is_halo[ext_off + local] = h ? 1 : 0;
            if (h) {
                const int64_t r = halo_off + (local - lower_bound_i32(batch, nb, w));
                halo[r] = w;
                hlr[r] = local;
            }
            ++local;
        }
    }
}

// Step 5: one warp per batch row. gcn stencil (+ sum stencil / local-graph columns), the
// batch_local_rows entry, and per-part local row pointers.
__global__ void emit_rows_kernel(GroupView g, const int32_t* __restrict__ order, const int32_t* __restrict__ asg,
                                 const int64_t* __restrict__ ro, const int32_t* __restrict__ cols,
                                 const double* __restrict__ cs, const int64_t* __restrict__ part_off, int64_t i0,
                                 int64_t i1, const int64_t* __restrict__ gpos, const int64_t* __restrict__ spos,
                                 int32_t* __restrict__ blr, int64_t* __restrict__ grp_local,
                                 int32_t* __restrict__ gcols, float* __restrict__ gco, int64_t* __restrict__ srp_local,
                                 int32_t* __restrict__ scols) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = i0 + ((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5); i < i1; i += nwarps) {
        const int32_t v = order[i];
        const int32_t p = asg[v];
        const int64_t e0 = ro[v], deg = ro[v + 1] - e0;
        const double cv = cs[v];
        const int64_t o = gpos[i];
        const int64_t pb = part_off[p];
        const int32_t j = static_cast<int32_t>(i - pb);  // batch index inside the part
        const int32_t lv = g.lid(p, v);
        for (int64_t e = lane; e < deg; e += 32) {
            const int32_t w = cols[e0 + e];
            const int32_t lw = g.lid(p, w);
            gcols[o + e] = lw;
            gco[o + e] = __double2float_rn(__ddiv_rn(1.0, __dmul_rn(cs[w], cv)));
            if (scols) scols[spos[i] + e] = lw;
        }
        if (lane == 0) {
            const int64_t glen = gpos[i + 1] - o;
            if (glen > deg) {  // no stored self-loop: (lv, 1/(cv*cv)) at the row end
                gcols[o + deg] = lv;
                gco[o + deg] = __double2float_rn(__ddiv_rn(1.0, __dmul_rn(cv, cv)));
            }
            blr[i] = lv;
            // local row pointers: nb + 1 entries per part at offset part_off[p] + p
            grp_local[pb + p + j] = o - gpos[pb];
            if (srp_local) srp_local[pb + p + j] = spos[i] - spos[pb];
            if (i + 1 == part_off[p + 1]) {
                grp_local[pb + p + j + 1] = gpos[i + 1] - gpos[pb];
                if (srp_local) srp_local[pb + p + j + 1] = spos[i + 1] - spos[pb];
            }
        }
    }
}

// plan.local_graph row pointers (GASB_PLAN_FULL): ne + 1 per part at ext_off[p] + p; a halo
// row is empty, so lrp[i] = sum_rowptr[#batch nodes below ext[i]].
__global__ void local_rowptr_kernel(const int32_t* __restrict__ ext, const int64_t* __restrict__ ext_off,
                                    const int32_t* __restrict__ order, const int64_t* __restrict__ part_off,
                                    const int64_t* __restrict__ srp_local, int32_t p0, int32_t p1,
                                    int64_t* __restrict__ lrp) {
    const int64_t lo = ext_off[p0], hi = ext_off[p1];
    for (int64_t x = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < hi; x += int64_t(gridDim.x) * blockDim.x) {
        int32_t a = p0, b = p1 - 1;  // part of position x
        while (a < b) {
            const int32_t m = (a + b + 1) / 2;
            if (ext_off[m] <= x) a = m;
            else b = m - 1;
        }
        const int32_t p = a;
        const int32_t nb = static_cast<int32_t>(part_off[p + 1] - part_off[p]);
        const int64_t* srp = srp_local + part_off[p] + p;
        const int32_t r = lower_bound_i32(order + part_off[p], nb, ext[x]);
        lrp[x + p] = srp[r];
        if (x + 1 == ext_off[p + 1]) lrp[x + 1 + p] = srp[nb];
    }
}

inline int grid_for(int64_t items, int per_block) {
    const int64_t b = (items + per_block - 1) / per_block;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

template <class T>
void download(std::vector<T>& dst, const T* src, int64_t count) {
    dst.resize(static_cast<size_t>(count));
    if (count > 0) GASB_CUDA(cudaMemcpy(dst.data(), src, sizeof(T) * count, cudaMemcpyDeviceToHost));
}

}  // namespace

void build_schedule_device(const Graph& G, const int32_t* h_asg, int32_t P, bool full, Schedule& s) {
    const int32_t n = G.num_nodes;
    const int64_t m = G.num_edges();
    require(n > 0, "partition_from_assignment: empty part");
    cudaStream_t st;
    GASB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // device time = the kernels' spans only: every allocation happens between spans
    struct Spans {
        cudaStream_t st;
        std::vector<cudaEvent_t> ev;
        void mark() {
            cudaEvent_t e;
            GASB_CUDA(cudaEventCreate(&e));
            GASB_CUDA(cudaEventRecord(e, st));
            ev.push_back(e);
        }
        float total() {
            GASB_CUDA(cudaStreamSynchronize(st));
            float ms = 0.0f;
            for (size_t i = 0; i + 1 < ev.size(); i += 2) {
                float x = 0.0f;
                GASB_CUDA(cudaEventElapsedTime(&x, ev[i], ev[i + 1]));
                ms += x;
            }
            return ms;
        }
        ~Spans() {
            for (auto e : ev) cudaEventDestroy(e);
            cudaStreamDestroy(st);
        }
    } spans{st, {}};

    const bool trace_on = std::getenv("GASB_TRACE_SETUP") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto trace = [&](const char* what) {  // GASB_TRACE_SETUP=1: phase wall times (synchronising)
        if (!trace_on) return;
        GASB_CUDA(cudaStreamSynchronize(st));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[plan_dev] %-22s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };

    // ---- inputs and every buffer whose size is known up front ----
    const int64_t W = (static_cast<int64_t>(n) + 31) / 32;
    const int32_t group = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(P, bitmap_budget() / (W * 4))));
    const int64_t gwords = static_cast<int64_t>(group) * W;
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < P) ++end_bit;
    DArr<int64_t> ro(n + 1);
    DArr<int32_t> cols(std::max<int64_t>(m, 1)), asg(n);
    GASB_CUDA(cudaMemcpyAsync(ro.p, G.row_offsets.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
    if (m) GASB_CUDA(cudaMemcpyAsync(cols.p, G.cols.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
    GASB_CUDA(cudaMemcpyAsync(asg.p, h_asg, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    DArr<int32_t> bad(1), ids(n), order(n), keys(n), blr(n);
    DArr<int64_t> part_off(P + 1), ext_off(P + 1), glen(n), gpos(n + 1), slen(full ? n : 0), spos(full ? n + 1 : 0);
    DArr<int64_t> grp_local(n + P), srp_local(full ? n + P : 0), wcnt(gwords), wpre(gwords + 1);
    DArr<double> cs(n);
    DArr<uint32_t> bm(gwords);
    size_t sort_tmp = 0, scan_tmp = 0;
    GASB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, asg.p, keys.p, ids.p, order.p, n, 0, end_bit, st));
    GASB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, scan_tmp, wcnt.p, wpre.p + 1, std::max<int64_t>(n, gwords), st));
    DArr<unsigned char> tmp(static_cast<int64_t>(std::max(sort_tmp, scan_tmp)));
    auto scan = [&](const int64_t* in, int64_t* out, int64_t count) {  // out[0] = 0, out[1..count] inclusive
        size_t t = tmp.n;
        GASB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, t, in, out + 1, count, st));
        GASB_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    };
    trace("inputs + allocs");

    // ---- 1. batches: stable sort of node ids by part ----
    spans.mark();
    GASB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st));
    check_parts_kernel<<<grid_for(n, 256), 256, 0, st>>>(asg.p, n, P, bad.p);
    int32_t h_bad = 0;
    GASB_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GASB_CUDA(cudaStreamSynchronize(st));
    require(h_bad == 0, "partition_from_assignment: part id out of range");
    iota_kernel<<<grid_for(n, 256), 256, 0, st>>>(ids.p, n);
    GASB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, sort_tmp, asg.p, keys.p, ids.p, order.p, n, 0, end_bit, st));
    part_bounds_kernel<<<(P + 1 + 255) / 256, 256, 0, st>>>(keys.p, n, P, part_off.p);
    std::vector<int64_t> h_poff(static_cast<size_t>(P) + 1);
    GASB_CUDA(cudaMemcpyAsync(h_poff.data(), part_off.p, sizeof(int64_t) * (P + 1), cudaMemcpyDeviceToHost, st));
    GASB_CUDA(cudaStreamSynchronize(st));
    for (int32_t p = 0; p < P; ++p) require(h_poff[p + 1] > h_poff[p], "partition_from_assignment: empty part");
    trace("sort + bounds");

    // ---- stencil row lengths and positions (sorted order) ----
    degree_sqrt_kernel<<<grid_for(n, 256), 256, 0, st>>>(ro.p, n, cs.p);
    row_len_kernel<<<grid_for(n, 256), 256, 0, st>>>(order.p, ro.p, cols.p, n, glen.p, full ? slen.p : nullptr);
    scan(glen.p, gpos.p, n);
    if (full) scan(slen.p, spos.p, n);
    int64_t Eg = 0, Es = 0;
    GASB_CUDA(cudaMemcpyAsync(&Eg, gpos.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (full) GASB_CUDA(cudaMemcpyAsync(&Es, spos.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    trace("row lengths + scans");

    // ---- 2-4. bitmaps and extended lists, in part groups ----
    std::vector<int64_t> h_eoff(static_cast<size_t>(P) + 1, 0);
    std::vector<std::pair<int32_t, int32_t>> groups;
    for (int32_t p0 = 0; p0 < P; p0 += group) groups.emplace_back(p0, std::min(P, p0 + group));
    auto fill_group = [&](int32_t p0, int32_t p1) {
        const int64_t words = static_cast<int64_t>(p1 - p0) * W;
        GASB_CUDA(cudaMemsetAsync(bm.p, 0, sizeof(uint32_t) * words, st));
        const int64_t i0 = h_poff[p0], i1 = h_poff[p1];
        mark_kernel<<<grid_for((i1 - i0) * 32, 256), 256, 0, st>>>(order.p, asg.p, ro.p, cols.p, i0, i1, p0, W, bm.p);
        popc_kernel<<<grid_for(words, 256), 256, 0, st>>>(bm.p, words, wcnt.p);
        scan(wcnt.p, wpre.p, words);
    };
    // extended sizes need the bitmaps first (a second fill per group when there are several)
    for (auto [p0, p1] : groups) {
        fill_group(p0, p1);
        std::vector<int64_t> wp(static_cast<size_t>(p1 - p0) + 1);
        for (int32_t p = p0; p <= p1; ++p)
            GASB_CUDA(cudaMemcpyAsync(&wp[p - p0], wpre.p + static_cast<int64_t>(p - p0) * W, sizeof(int64_t),
                                      cudaMemcpyDeviceToHost, st));
        GASB_CUDA(cudaStreamSynchronize(st));
        for (int32_t p = p0; p < p1; ++p) h_eoff[p + 1] = h_eoff[p] + (wp[p - p0 + 1] - wp[p - p0]);
    }
    spans.mark();
    trace("bitmap + popc scan");

    const int64_t NE = h_eoff[P], NH = NE - n;
    DArr<int32_t> ext(NE), halo(std::max<int64_t>(NH, 1)), hlr(std::max<int64_t>(NH, 1));
    DArr<int32_t> gcols(std::max<int64_t>(Eg, 1)), scols(full ? std::max<int64_t>(Es, 1) : 0);
    DArr<float> gco(std::max<int64_t>(Eg, 1));
    DArr<uint8_t> ish(NE);
    DArr<int64_t> lrp(full ? NE + P : 0);
    GASB_CUDA(cudaMemcpyAsync(ext_off.p, h_eoff.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, st));
    GASB_CUDA(cudaStreamSynchronize(st));
    trace("output allocs");

    spans.mark();
    for (auto [p0, p1] : groups) {
        if (groups.size() > 1) fill_group(p0, p1);
        const int64_t words = static_cast<int64_t>(p1 - p0) * W;
        GroupView gv{bm.p, wpre.p, W, p0};
        emit_ext_kernel<<<grid_for(words, 256), 256, 0, st>>>(gv, words, h_eoff[p0], asg.p, order.p, part_off.p, ext.p,
                                                             ish.p, halo.p, hlr.p);
        const int64_t i0 = h_poff[p0], i1 = h_poff[p1];
        emit_rows_kernel<<<grid_for((i1 - i0) * 32, 256), 256, 0, st>>>(
            gv, order.p, asg.p, ro.p, cols.p, cs.p, part_off.p, i0, i1, gpos.p, full ? spos.p : nullptr, blr.p,
            grp_local.p, gcols.p, gco.p, full ? srp_local.p : nullptr, full ? scols.p : nullptr);
        if (full)
            local_rowptr_kernel<<<grid_for(h_eoff[p1] - h_eoff[p0], 256), 256, 0, st>>>(
                ext.p, ext_off.p, order.p, part_off.p, srp_local.p, p0, p1, lrp.p);
    }
    GASB_CUDA(cudaGetLastError());
    spans.mark();
    const float dev_ms = spans.total();
    trace("emit");

    // ---- into the schedule's HostPlans (part order) ----
    std::vector<int64_t> h_gpos(static_cast<size_t>(P) + 1), h_spos(static_cast<size_t>(P) + 1, 0);
    for (int32_t p = 0; p <= P; ++p) {
        GASB_CUDA(cudaMemcpy(&h_gpos[p], gpos.p + h_poff[p], sizeof(int64_t), cudaMemcpyDeviceToHost));
        if (full) GASB_CUDA(cudaMemcpy(&h_spos[p], spos.p + h_poff[p], sizeof(int64_t), cudaMemcpyDeviceToHost));
    }
    s.graph = &G;
    s.num_parts = P;
    s.plans.assign(static_cast<size_t>(P), HostPlan{});
    // parts copied from OpenMP threads: the pageable copies and the first touch of the host
    // vectors overlap across parts
    int dev = 0;
    GASB_CUDA(cudaGetDevice(&dev));
    std::string err;
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t p = 0; p < P; ++p) {
      try {
        GASB_CUDA(cudaSetDevice(dev));
        HostPlan& hp = s.plans[p];
        const int64_t b0 = h_poff[p], nb = h_poff[p + 1] - b0;
        const int64_t x0 = h_eoff[p], ne = h_eoff[p + 1] - x0;
        const int64_t h0 = x0 - b0, nh = ne - nb;
        download(hp.batch, order.p + b0, nb);
        download(hp.extended, ext.p + x0, ne);
        download(hp.is_halo, ish.p + x0, ne);
        download(hp.halo, halo.p + h0, nh);
        download(hp.halo_local_rows, hlr.p + h0, nh);
        download(hp.batch_local_rows, blr.p + b0, nb);
        download(hp.gcn_rowptr, grp_local.p + b0 + p, nb + 1);
        download(hp.gcn_cols, gcols.p + h_gpos[p], h_gpos[p + 1] - h_gpos[p]);
        download(hp.gcn_coeffs, gco.p + h_gpos[p], h_gpos[p + 1] - h_gpos[p]);
        if (full) {
            download(hp.local_rowptr, lrp.p + x0 + p, ne + 1);
            download(hp.sum_rowptr, srp_local.p + b0 + p, nb + 1);
            download(hp.sum_cols, scols.p + h_spos[p], h_spos[p + 1] - h_spos[p]);
            hp.local_cols = hp.sum_cols;  // batch rows in ascending id order, halo rows empty
            hp.sum_coeffs.assign(hp.sum_cols.size(), 1.0f);
        }
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    }
    if (!err.empty()) throw CudaError(err);
    s.device_ms = dev_ms;
    trace("copies into host plans");
}

}  // namespace gasb
