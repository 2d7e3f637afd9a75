// Data-parallel GAS training over k GPUs of one node, one process per GPU.
//
// Step semantics (the oracle's go_session_dp_epoch, oracle/gas_oracle.c): a step takes k
// consecutive batches of the seeded epoch order (trainer.cpp:395-400); rank j runs the j-th.
// Every batch sees the start-of-step parameters and histories (Jacobi): its own rows are
// fresh (pushed into the rank's replica and read in place, as compose_rows does), every
// other row is the start-of-step history. After the step, each rank's pushed rows are
// committed into every replica, the gradients are summed in rank order over the batches
// that had training rows and divided by their count, then clipped and applied by Adam on
// every rank — so all replicas stay bit-identical without a broadcast. At k = 1 the step
// IS gas_epoch's batch.
//
// Exchange over peer memory (no NCCL on the data path). Each rank owns one HBM region,
// exported with CUDA IPC and mapped by every peer (NVLink P2P across GPUs):
//   [ signal words | gradient slot (trainer grads) | pushed-row slots (trainer act_l) ]
// The trainer's grads and act_l buffers ARE views into the region, so the batch graph
// writes them in place and peers read them directly:
//   barrier  -> every rank's batch is done (grads, act_l complete)
//   reduce   -> gsum = (sum over stepped ranks, rank order, of grads_j) / count: each rank
//               reads all k gradient slots over NVLink (1.2 MB each at C3) — the all-reduce
//               as one kernel, deterministic and identical on every rank
//   commit   -> H_l[batch_j] = act_l of rank j for every peer j (NVLink reads, local HBM
//               writes, stamps, table value flags)
//   barrier  -> every rank has read the step's slots (they are rewritten next step)
//   adam     -> on gsum; step counters advance by the step's batch count
// Barriers are release/acquire flag words in the peers' regions (st.release.sys /
// ld.acquire.sys), monotone sequence numbers, bounded spins (a timeout latches an error
// instead of hanging the GPU).
//
// Memory: histories are replicated (C3: 716 MB per GPU); broadcasting pushes costs
// (k-1)/k of n*d*4 bytes per layer-epoch per GPU, ~20x fewer NVLink bytes than sharded
// halo pulls at C3 (SURVEY §8e "Alternative").
#include <cstring>
#include <memory>
#include <random>

#include "trainer_impl.hpp"

namespace gasb {
namespace {

constexpr int kMaxWorld = 8;
constexpr size_t kAlign = 256;
constexpr int64_t kSpinTimeoutNs = 30LL * 1000 * 1000 * 1000;

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

struct PeerPtrs {
    uint64_t* flags[kMaxWorld];  // each rank's signal words (world entries, indexed by source rank)
};

// Thread j: publish `seq` into rank j's word for this rank, then wait for rank j's `seq`.
__global__ void dp_barrier_kernel(PeerPtrs peers, int rank, int world, uint64_t seq, int32_t* err) {
    const int j = threadIdx.x;
    if (j >= world) return;
    __threadfence_system();
    st_release_sys(peers.flags[j] + rank, seq);
    const uint64_t* mine = peers.flags[rank] + j;
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(mine) < seq) {
        if (globaltimer() - t0 > static_cast<uint64_t>(kSpinTimeoutNs)) {
            atomicOr(err, 1);
            break;
        }
        __nanosleep(256);
    }
}

struct GradSlots {
    const float* g[kMaxWorld];
};

// gsum[e] = (((0 + g_j0[e]) + g_j1[e]) + ...) / count over the stepped ranks j in rank
// order: go_session_dp_epoch's `gsum[e] += g[e]` then `gsum[e] / (float)count`.
__global__ void __launch_bounds__(256) dp_reduce_kernel(GradSlots slots, uint32_t stepped_mask, int world,
                                                        float count, int64_t n4, float* __restrict__ gsum) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < world; ++j) {
            if (!((stepped_mask >> j) & 1u)) continue;
            const float4 v = __ldcv(reinterpret_cast<const float4*>(slots.g[j]) + i);
            acc.x = __fadd_rn(acc.x, v.x);
            acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z);
            acc.w = __fadd_rn(acc.w, v.w);
        }
        acc.x = __fdiv_rn(acc.x, count);
        acc.y = __fdiv_rn(acc.y, count);
        acc.z = __fdiv_rn(acc.z, count);
        acc.w = __fdiv_rn(acc.w, count);
        reinterpret_cast<float4*>(gsum)[i] = acc;
    }
}

struct CommitJob {
    const float* acts;    // peer's act_1 slot (layer l at + (l-1) * layer_stride)
    const int32_t* ids;   // global ids of the peer's batch rows (local copy of the plan)
    int32_t nb;
    int32_t row0;         // prefix sum of nb over jobs (grid row space)
};
struct CommitJobs {
    CommitJob j[kMaxWorld];
    int32_t njobs;
};

// H_l[ids[i]] = acts_l[i] for every job (peer batch) and history layer; one warp per
// (job row, layer); float4 columns. Stamps = the start-of-step store step; the table's
// value flags OR the committed values' flags (the SpMM's widening path depends on them).
__global__ void __launch_bounds__(256) dp_commit_kernel(CommitJobs jobs, int32_t total_rows, int32_t layers,
                                                        int64_t layer_stride, int64_t lda, int32_t dim,
                                                        float* table0, int64_t table_layer_stride, int64_t ldt,
                                                        int64_t* stamps0, int64_t stamps_layer_stride,
                                                        const int64_t* step, int32_t* flags0, int32_t flags_stride) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= static_cast<int64_t>(total_rows) * layers) return;
    const int32_t l = static_cast<int32_t>(w / total_rows);
    const int32_t r = static_cast<int32_t>(w % total_rows);
    int jb = 0;
    while (jb + 1 < jobs.njobs && r >= jobs.j[jb + 1].row0) ++jb;
    const CommitJob& J = jobs.j[jb];
    const int32_t i = r - J.row0;
    const int32_t v = J.ids[i];
    const float* src = J.acts + l * layer_stride + static_cast<int64_t>(i) * lda;
    float* dst = table0 + l * table_layer_stride + static_cast<int64_t>(v) * ldt;
    int32_t f = 0;
    if ((dim & 3) == 0) {  // rows are 16 B aligned (lda, ldt multiples of 4)
        for (int c = lane; c < dim / 4; c += 32) {
            const float4 x = __ldcv(reinterpret_cast<const float4*>(src) + c);
            reinterpret_cast<float4*>(dst)[c] = x;
            f |= table_flag_of(x.x) | table_flag_of(x.y) | table_flag_of(x.z) | table_flag_of(x.w);
        }
    } else {
        for (int c = lane; c < dim; c += 32) {
            const float x = __ldcv(src + c);
            dst[c] = x;
            f |= table_flag_of(x);
        }
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0) {
        stamps0[l * stamps_layer_stride + v] = *step;
        if (f) atomicOr(flags0 + static_cast<int64_t>(l) * flags_stride, f);
    }
}

// ---- partition-sharded placement ---------------------------------------------------
// dst[i] = H_layer[ids[i]] from the owner's shard: one warp per row, float4 columns; rows
// owned by a peer are NVLink P2P loads through its IPC-mapped region.
__global__ void __launch_bounds__(256) shard_pull_kernel(ShardView s, int32_t layer, const int32_t* __restrict__ ids,
                                                         int64_t count, float* __restrict__ dst, int64_t ldd,
                                                         int32_t dim) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= count) return;
    const uint32_t ol = s.owner_local[ids ? ids[w] : w];
    const int32_t o = static_cast<int32_t>(ol >> kShardLocalBits);
    const int64_t li = ol & ((1u << kShardLocalBits) - 1);
    const float* src = s.tables[o] + (layer - 1) * s.layer_stride[o] + li * s.ld;
    float* d = dst + w * ldd;
    if ((dim & 3) == 0 && (ldd & 3) == 0) {
        for (int c = lane; c < dim / 4; c += 32)
            reinterpret_cast<float4*>(d)[c] = __ldcv(reinterpret_cast<const float4*>(src) + c);
    } else {
        for (int c = lane; c < dim; c += 32) d[c] = __ldcv(src + c);
    }
}

// Sharded commit: of every job's (rank's) batch rows, the ones this rank owns go into its
// shard (stamps = the start-of-step store step, the layer's value flags), from the job's
// act slot (a peer's over NVLink, or this rank's own).
__global__ void __launch_bounds__(256) dp_commit_sharded_kernel(CommitJobs jobs, int32_t total_rows, int32_t layers,
                                                                int64_t layer_stride, int64_t lda, int32_t dim,
                                                                const uint32_t* __restrict__ owner_local, int32_t me,
                                                                float* shard, int64_t shard_stride, int64_t ldt,
                                                                int64_t* stamps, int64_t n_owned, const int64_t* step,
                                                                int32_t* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= static_cast<int64_t>(total_rows) * layers) return;
    const int32_t l = static_cast<int32_t>(w / total_rows);
    const int32_t r = static_cast<int32_t>(w % total_rows);
    int jb = 0;
    while (jb + 1 < jobs.njobs && r >= jobs.j[jb + 1].row0) ++jb;
    const CommitJob& J = jobs.j[jb];
    const int32_t i = r - J.row0;
    const uint32_t ol = owner_local[J.ids[i]];
    if (static_cast<int32_t>(ol >> kShardLocalBits) != me) return;
    const int64_t li = ol & ((1u << kShardLocalBits) - 1);
    const float* src = J.acts + l * layer_stride + static_cast<int64_t>(i) * lda;
    float* dst = shard + l * shard_stride + li * ldt;
    int32_t f = 0;
    for (int c = lane; c < dim; c += 32) {
        const float x = __ldcv(src + c);
        dst[c] = x;
        f |= table_flag_of(x);
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0) {
        stamps[l * n_owned + li] = *step;
        if (f) atomicOr(flags + l, f);
    }
}

__global__ void dp_end_step_kernel(int64_t* step, int64_t* t_counter, int32_t batches, int32_t stepped) {
    *step += batches;
    if (stepped) *t_counter += 1;
}

uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t s, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
    return mix64(mix64(mix64(s ^ mix64(a)) ^ mix64(b)) ^ mix64(c));
}

}  // namespace

void launch_shard_pull(const ShardView& s, int32_t layer, const int32_t* ids, int64_t count, float* dst, int64_t ldd,
                       int32_t dim, cudaStream_t st) {
    if (count <= 0) return;
    shard_pull_kernel<<<static_cast<unsigned>(ceil_div(count * 32, 256)), 256, 0, st>>>(s, layer, ids, count, dst,
                                                                                        ldd, dim);
    ++t_launches;
    GASB_CUDA(cudaGetLastError());
}

// Row ownership of the sharded placement: partition p belongs to rank p mod world; a rank's
// rows are its parts' batch nodes in part order (then id order), packed owner << 29 | row.
void shard_map(const Schedule& S, int32_t world, std::vector<uint32_t>& owner_local, std::vector<int64_t>& n_owned) {
    owner_local.assign(static_cast<size_t>(S.graph->num_nodes), 0xffffffffu);
    n_owned.assign(static_cast<size_t>(world), 0);
    for (int32_t p = 0; p < S.num_parts; ++p) {
        const int32_t o = p % world;
        for (int32_t v : S.plans[p].batch) {
            require(n_owned[o] < (int64_t(1) << kShardLocalBits), "dp: shard exceeds 2^29 rows");
            owner_local[v] = (static_cast<uint32_t>(o) << kShardLocalBits) | static_cast<uint32_t>(n_owned[o]++);
        }
    }
}

// gas_epoch's batch order (trainer.cpp:395-400): Fisher-Yates with Rng(derive_seed(seed ^
// "ordr", epoch)).next_below (include/gas/rng.hpp), identity when !shuffle.
void epoch_order(int32_t num_parts, uint64_t seed, int64_t epoch, bool shuffle, std::vector<int32_t>& order) {
    order.resize(static_cast<size_t>(num_parts));
    for (int32_t i = 0; i < num_parts; ++i) order[i] = i;
    if (!shuffle) return;
    std::mt19937_64 gen(derive_seed(seed ^ 0x6f726472ull, static_cast<uint64_t>(epoch)));
    auto below = [&](uint64_t n) -> uint64_t {
        if (n <= 1) return 0;
        const uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % n);
        uint64_t x;
        do {
            x = gen();
        } while (x >= limit);
        return x % n;
    };
    for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[below(i)]);
}

}  // namespace gasb

using namespace gasb;

struct gasb_dp_s {
    gasb_trainer t = nullptr;
    int32_t rank = 0, world = 1;
    // sharded placement (GASB_DP_SHARDED): this rank's shard of every history layer sits in
    // its region at off_shard (n_owned[rank] rows per layer, pitch shard_ld); stamps / value
    // flags of the shard are local
    bool sharded = false;
    size_t off_shard = 0;
    int64_t shard_ld = 0;
    std::vector<int64_t> n_owned;
    std::vector<uint32_t> h_owner_local;
    DevBuf<uint32_t> owner_local;
    DevBuf<int64_t> shard_stamps;
    DevBuf<int32_t> shard_flags;
    // NVLink bytes of the last epoch (host-counted from the plans): halo rows read from peer
    // shards + peer act rows read by the commits (sharded), or peer act rows committed into
    // the replica (replicated); plus the gradient slots read by the reduce
    int64_t nvlink_bytes = 0, local_pull_bytes = 0;
    std::vector<int64_t> part_remote_halo, part_local_halo;
    char* region = nullptr;
    size_t off_flags = 0, off_grads = 0, off_acts = 0, bytes = 0;
    int64_t act_layer_stride = 0;  // floats between act_l slots
    int32_t hist_layers = 0;
    std::vector<char*> peer;  // region base of every rank (own = region)
    bool connected = false;
    uint64_t seq = 0;
    DevBuf<float> gsum;
    DevBuf<int32_t> err;
    std::vector<int32_t> last_order;
    std::vector<int32_t> last_parts;  // parts this rank ran in the last epoch
    int64_t epoch_launches = 0;

    ~gasb_dp_s() {
        if (t && t->stream) cudaStreamSynchronize(t->stream);
        for (int32_t j = 0; j < world; ++j)
            if (j != rank && j < static_cast<int32_t>(peer.size()) && peer[j]) cudaIpcCloseMemHandle(peer[j]);
    }
    uint64_t* flags_of(int32_t j) const { return reinterpret_cast<uint64_t*>(peer[j] + off_flags); }
    const float* grads_of(int32_t j) const { return reinterpret_cast<const float*>(peer[j] + off_grads); }
    const float* acts_of(int32_t j) const { return reinterpret_cast<const float*>(peer[j] + off_acts); }
    float* shard_of(int32_t j) const { return reinterpret_cast<float*>(peer[j] + off_shard); }
    void bind_shard_view() {
        ShardView v{};
        v.owner_local = owner_local.p;
        v.ld = shard_ld;
        v.world = world;
        for (int32_t j = 0; j < world; ++j) {
            v.tables[j] = shard_of(j);
            v.layer_stride[j] = n_owned[j] * shard_ld;
        }
        t->shard = v;
    }

    void barrier() {
        PeerPtrs pp{};
        for (int32_t j = 0; j < world; ++j) pp.flags[j] = flags_of(j);
        dp_barrier_kernel<<<1, 32, 0, t->stream>>>(pp, rank, world, ++seq, err.p);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
    }

    // One step over parts[0..kk): batch (if this rank has one), exchange, Adam.
    int64_t step(const int32_t* parts, int32_t kk, int64_t epoch) {
        gasb_trainer_s& T = *t;
        const int64_t c0 = t_launches;
        int64_t n = 0;
        if (rank < kk) {
            if (T.drop) {  // this batch's dropout masks (epoch, partition id), before its graph
                const int64_t c1 = t_launches;
                T.enqueue_masks(parts[rank], epoch);
                n += t_launches - c1;
            }
            n += T.launch_batch_graph(parts[rank], true);
        }
        barrier();
        uint32_t mask = 0;
        int32_t count = 0;
        for (int32_t j = 0; j < kk; ++j)
            if (T.ntrain[parts[j]] > 0) {
                mask |= 1u << j;
                ++count;
            }
        if (count > 0) {
            GradSlots gs{};
            for (int32_t j = 0; j < kk; ++j) gs.g[j] = grads_of(j);
            const int64_t n4 = T.nparam / 4;
            const int64_t blocks = std::min<int64_t>(ceil_div(n4, 256), 4 * 148);
            dp_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, T.stream>>>(gs, mask, kk,
                                                                                  static_cast<float>(count), n4, gsum.p);
            ++t_launches;
            GASB_CUDA(cudaGetLastError());
        }
        // NVLink traffic of the step (bookkeeping): gradient slots of the peers, halo rows from
        // peer shards (sharded), peer act rows read by the commit
        {
            const int64_t rowb = static_cast<int64_t>(T.hist_dim) * 4 * hist_layers;
            if (count > 0) nvlink_bytes += static_cast<int64_t>(T.nparam) * 4 * (count - ((mask >> rank) & 1u));
            for (int32_t j = 0; j < kk; ++j) {
                if (j == rank) {
                    if (sharded) {
                        nvlink_bytes += part_remote_halo[parts[j]] * rowb;
                        local_pull_bytes += part_local_halo[parts[j]] * rowb;
                    }
                    continue;
                }
                int64_t rows_in = T.nb[parts[j]];
                if (sharded) {
                    rows_in = 0;
                    for (int32_t v : T.sched->plans[parts[j]].batch)
                        rows_in += static_cast<int32_t>(h_owner_local[v] >> kShardLocalBits) == rank;
                }
                nvlink_bytes += rows_in * rowb;
            }
        }
        if (hist_layers > 0 && sharded) {
            CommitJobs jobs{};
            int32_t rows = 0;
            for (int32_t j = 0; j < kk; ++j) {  // every rank's batch, this rank's own included
                const int32_t p = parts[j];
                CommitJob& J = jobs.j[jobs.njobs++];
                J.acts = acts_of(j);
                J.ids = T.batch_nodes.p + T.row_off[p];
                J.nb = T.nb[p];
                J.row0 = rows;
                rows += T.nb[p];
            }
            if (rows > 0) {
                const int64_t warps = static_cast<int64_t>(rows) * hist_layers;
                dp_commit_sharded_kernel<<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, T.stream>>>(
                    jobs, rows, hist_layers, act_layer_stride, T.ldA, T.hist_dim, owner_local.p, rank,
                    shard_of(rank), n_owned[rank] * shard_ld, shard_ld, shard_stamps.p, n_owned[rank],
                    history_step_ptr(T.hist), shard_flags.p);
                ++t_launches;
                GASB_CUDA(cudaGetLastError());
            }
        } else if (hist_layers > 0) {
            CommitJobs jobs{};
            int32_t rows = 0;
            for (int32_t j = 0; j < kk; ++j) {
                if (j == rank) continue;
                const int32_t p = parts[j];
                CommitJob& J = jobs.j[jobs.njobs++];
                J.acts = acts_of(j);
                J.ids = T.batch_nodes.p + T.row_off[p];
                J.nb = T.nb[p];
                J.row0 = rows;
                rows += T.nb[p];
            }
            if (rows > 0) {
                const int64_t warps = static_cast<int64_t>(rows) * hist_layers;
                const int64_t ldt = history_ld(T.hist);
                const int64_t tstride = hist_layers > 1 ? history_table(T.hist, 2) - history_table(T.hist, 1) : 0;
                const int64_t sstride = hist_layers > 1 ? history_stamps(T.hist, 2) - history_stamps(T.hist, 1) : 0;
                const int32_t fstride = hist_layers > 1
                                            ? static_cast<int32_t>(history_flags(T.hist, 2) - history_flags(T.hist, 1))
                                            : 0;
                dp_commit_kernel<<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, T.stream>>>(
                    jobs, rows, hist_layers, act_layer_stride, T.ldA, T.hist_dim,
                    history_table(T.hist, 1), tstride, ldt, history_stamps(T.hist, 1), sstride,
                    history_step_ptr(T.hist), history_flags(T.hist, 1), fstride);
                ++t_launches;
                GASB_CUDA(cudaGetLastError());
            }
        }
        barrier();
        if (count > 0)
            launch_adam(T.params.p, T.adam_m.p, T.adam_v.p, gsum.p, T.nparam, T.t_counter.p, T.bc.p, T.spec.lr,
                        T.spec.beta1, T.spec.beta2, T.spec.eps, T.spec.clip_max_norm, T.norm_scratch.p, T.stream);
        dp_end_step_kernel<<<1, 1, 0, T.stream>>>(history_step_ptr(T.hist), T.t_counter.p, kk, count > 0 ? 1 : 0);
        ++t_launches;
        GASB_CUDA(cudaGetLastError());
        if (count > 0) T.t_host += 1;
        return n + (t_launches - c0);
    }
};

extern "C" {

gasb_status gasb_dp_create(gasb_trainer t, int32_t rank, int32_t world, gasb_dp* out) {
    return gasb_dp_create_ex(t, rank, world, GASB_DP_REPLICATED, out);
}

gasb_status gasb_dp_create_ex(gasb_trainer t, int32_t rank, int32_t world, int32_t placement, gasb_dp* out) {
    return guard([&] {
        require(placement == GASB_DP_REPLICATED || placement == GASB_DP_SHARDED, "dp: unknown history placement");
        require(t && out, "dp: null argument");
        require(world >= 1 && world <= kMaxWorld, "dp: world size must be in [1, 8]");
        require(rank >= 0 && rank < world, "dp: rank out of range");
        require(t->nparam % 4 == 0, "dp: parameter vector must be a multiple of 4 floats");
        GASB_CUDA(cudaSetDevice(t->opt.device));
        GASB_CUDA(cudaStreamSynchronize(t->stream));
        auto d = std::make_unique<gasb_dp_s>();
        d->t = t;
        d->rank = rank;
        d->world = world;
        d->hist_layers = t->hist_dim > 0 ? t->L - 1 : 0;
        d->act_layer_stride = static_cast<int64_t>(t->nb_max) * t->ldA;
        d->off_flags = 0;
        d->off_grads = align_up(sizeof(uint64_t) * kMaxWorld);
        d->off_acts = align_up(d->off_grads + sizeof(float) * static_cast<size_t>(t->nparam));
        d->bytes = align_up(d->off_acts + sizeof(float) * static_cast<size_t>(d->act_layer_stride) *
                                              static_cast<size_t>(std::max(d->hist_layers, 1)));
        d->sharded = placement == GASB_DP_SHARDED && d->hist_layers > 0;
        if (d->sharded) {
            if (t->opt.prefetch) throw std::invalid_argument("dp: the sharded placement has no prefetch mode");
            shard_map(*t->sched, world, d->h_owner_local, d->n_owned);
            d->shard_ld = round_up(t->hist_dim, 4);
            d->off_shard = d->bytes;
            d->bytes = align_up(d->off_shard + sizeof(float) * static_cast<size_t>(d->hist_layers) *
                                                   static_cast<size_t>(d->n_owned[rank] * d->shard_ld));
            d->owner_local.upload(d->h_owner_local);
            d->shard_stamps.alloc(static_cast<int64_t>(d->hist_layers) * std::max<int64_t>(d->n_owned[rank], 1));
            GASB_CUDA(cudaMemset(d->shard_stamps.p, 0xff, sizeof(int64_t) * d->shard_stamps.n));  // -1: never pushed
            d->shard_flags.alloc(d->hist_layers);
            d->shard_flags.zero();
            // halo rows per part by owner (this rank's view): remote = NVLink, local = HBM
            d->part_remote_halo.assign(t->num_parts, 0);
            d->part_local_halo.assign(t->num_parts, 0);
            for (int32_t p = 0; p < t->num_parts; ++p)
                for (int32_t v : t->sched->plans[p].halo)
                    (static_cast<int32_t>(d->h_owner_local[v] >> kShardLocalBits) == rank ? d->part_local_halo
                                                                                           : d->part_remote_halo)[p]++;
        }
        require(!t->dp_region.p, "dp: the trainer already belongs to a data-parallel group");
        t->dp_region.alloc(static_cast<int64_t>(d->bytes));  // owned by the trainer (its grads/act_l live there)
        d->region = t->dp_region.p;
        GASB_CUDA(cudaMemset(d->region, 0, d->bytes));
        // the trainer's gradient and pushed-row buffers become views into the region
        float* g = reinterpret_cast<float*>(d->region + d->off_grads);
        GASB_CUDA(cudaMemcpy(g, t->grads.p, sizeof(float) * t->nparam, cudaMemcpyDeviceToDevice));
        t->grads.adopt(g, t->nparam);
        for (int32_t l = 1; l <= d->hist_layers; ++l)
            t->act[l].adopt(reinterpret_cast<float*>(d->region + d->off_acts) + (l - 1) * d->act_layer_stride,
                            d->act_layer_stride);
        // graphs captured against the old buffers are stale
        for (auto& gx : t->graphs)
            if (gx) {
                cudaGraphExecDestroy(gx);
                gx = nullptr;
            }
        for (auto& gx : t->graphs_dp)
            if (gx) {
                cudaGraphExecDestroy(gx);
                gx = nullptr;
            }
        d->gsum.alloc(t->nparam);
        d->gsum.zero();
        d->err.alloc(1);
        d->err.zero();
        // every part can land on any rank (the epoch order is reshuffled): capture all the
        // data-parallel batch graphs now, not inside timed epochs
        if (t->opt.use_graphs && !d->sharded)  // (sharded: once the peers' shards are mapped)
            for (int32_t p = 0; p < t->num_parts; ++p) t->capture_batch_graph(p, true);
        d->peer.assign(static_cast<size_t>(world), nullptr);
        d->peer[rank] = d->region;
        if (d->sharded) {
            // the store's full tables are replaced by the group's shards (start: zeros, as the
            // fresh store), the batches pull halos from them and push nothing (see step())
            history_release_tables(t->hist);
            t->sharded_dp = true;
        }
        if (world == 1) {
            d->connected = true;
            if (d->sharded) d->bind_shard_view();
        }
        if (d->sharded && t->opt.use_graphs && world == 1)
            for (int32_t p = 0; p < t->num_parts; ++p) t->capture_batch_graph(p, true);
        *out = d.release();
    });
}

gasb_status gasb_dp_export(gasb_dp d, uint8_t* h_handle) {
    return guard([&] {
        require(d && h_handle, "dp: null argument");
        cudaIpcMemHandle_t h;
        GASB_CUDA(cudaIpcGetMemHandle(&h, d->region));
        static_assert(sizeof(h) == GASB_DP_HANDLE_BYTES, "IPC handle size");
        std::memcpy(h_handle, &h, sizeof(h));
    });
}

gasb_status gasb_dp_connect(gasb_dp d, const uint8_t* h_handles) {
    return guard([&] {
        require(d && h_handles, "dp: null argument");
        if (d->connected) throw std::logic_error("dp: already connected");
        GASB_CUDA(cudaSetDevice(d->t->opt.device));
        for (int32_t j = 0; j < d->world; ++j) {
            if (j == d->rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, h_handles + static_cast<size_t>(j) * GASB_DP_HANDLE_BYTES, sizeof(h));
            void* p = nullptr;
            GASB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            d->peer[j] = static_cast<char*>(p);
        }
        d->connected = true;
        if (d->sharded) {  // the batch graphs bake the peers' shard pointers: capture them now
            d->bind_shard_view();
            if (d->t->opt.use_graphs)
                for (int32_t p = 0; p < d->t->num_parts; ++p) d->t->capture_batch_graph(p, true);
        }
    });
}

gasb_status gasb_dp_epoch_async(gasb_dp d, int64_t epoch, int32_t shuffle) {
    return guard([&] {
        require(d, "dp: null handle");
        if (!d->connected) throw std::logic_error("dp: connect() before training");
        gasb_trainer_s& T = *d->t;
        GASB_CUDA(cudaSetDevice(T.opt.device));
        std::vector<int32_t> order;
        epoch_order(T.num_parts, T.spec.seed, epoch, shuffle != 0, order);
        int64_t steps = 0;
        for (int32_t s0 = 0; s0 < T.num_parts; s0 += d->world) ++steps;
        T.ensure_bc(T.t_host + steps + 2);
        d->epoch_launches = 0;
        d->nvlink_bytes = 0;
        d->local_pull_bytes = 0;
        d->last_parts.clear();
        for (int32_t s0 = 0; s0 < T.num_parts; s0 += d->world)
            if (d->rank < std::min(d->world, T.num_parts - s0)) d->last_parts.push_back(order[s0 + d->rank]);
        if (T.opt.hoist_layer1 && T.opt.fused && !T.residual && !T.drop && T.agg_all.p) {
            const int64_t c0 = t_launches;  // layer 1 of this rank's batches, one launch
            T.enqueue_hoisted_parts(d->last_parts);
            d->epoch_launches += t_launches - c0;
        }
        for (int32_t s0 = 0; s0 < T.num_parts; s0 += d->world) {
            const int32_t kk = std::min(d->world, T.num_parts - s0);
            d->epoch_launches += d->step(order.data() + s0, kk, epoch);
        }
        d->last_order = order;
        T.last_order = order;
        T.epoch_launches = d->epoch_launches;
    });
}

gasb_status gasb_dp_check(gasb_dp d) {
    return guard([&] {
        require(d, "dp: null handle");
        GASB_CUDA(cudaStreamSynchronize(d->t->stream));
        int32_t e = 0;
        GASB_CUDA(cudaMemcpy(&e, d->err.p, sizeof(e), cudaMemcpyDeviceToHost));
        if (e) {
            GASB_CUDA(cudaMemset(d->err.p, 0, sizeof(e)));
            throw std::runtime_error("dp: cross-rank barrier timed out (a peer did not arrive)");
        }
    });
}

gasb_status gasb_dp_last_losses(gasb_dp d, double* h_losses) {
    return guard([&] {
        require(d && h_losses, "dp: null argument");
        gasb_trainer_s& T = *d->t;
        GASB_CUDA(cudaStreamSynchronize(T.stream));
        std::vector<double> l(static_cast<size_t>(T.num_parts));
        GASB_CUDA(cudaMemcpy(l.data(), T.loss.p, sizeof(double) * l.size(), cudaMemcpyDeviceToHost));
        std::fill(h_losses, h_losses + T.num_parts, 0.0);
        for (int32_t p : d->last_parts)
            if (T.ntrain[p] > 0) h_losses[p] = l[p];
    });
}

gasb_status gasb_dp_launch_count(gasb_dp d, int64_t* out) {
    return guard([&] {
        require(d && out, "dp: null argument");
        *out = d->epoch_launches;
    });
}

gasb_status gasb_dp_read_history(gasb_dp d, int32_t layer, float* h_out) {
    return guard([&] {
        require(d && h_out, "dp: null argument");
        gasb_trainer_s& T = *d->t;
        if (!d->sharded) throw std::logic_error("dp: the replicated placement keeps the trainer's HistoryStore");
        if (!d->connected) throw std::logic_error("dp: connect() before reading the shards");
        require(layer >= 1 && layer <= d->hist_layers, "HistoryStore: layer out of range");
        GASB_CUDA(cudaStreamSynchronize(T.stream));
        DevBuf<float> full;
        full.alloc(static_cast<int64_t>(T.n) * d->shard_ld);
        launch_shard_pull(T.shard, layer, nullptr, T.n, full.p, d->shard_ld, T.hist_dim, T.stream);
        GASB_CUDA(cudaMemcpy2DAsync(h_out, sizeof(float) * T.hist_dim, full.p, sizeof(float) * d->shard_ld,
                                    sizeof(float) * T.hist_dim, T.n, cudaMemcpyDeviceToHost, T.stream));
        GASB_CUDA(cudaStreamSynchronize(T.stream));
    });
}

gasb_status gasb_dp_traffic(gasb_dp d, int64_t* nvlink_bytes, int64_t* local_pull_bytes, int64_t* shard_rows) {
    return guard([&] {
        require(d, "dp: null handle");
        if (nvlink_bytes) *nvlink_bytes = d->nvlink_bytes;
        if (local_pull_bytes) *local_pull_bytes = d->local_pull_bytes;
        if (shard_rows) *shard_rows = d->sharded ? d->n_owned[d->rank] : d->t->n;
    });
}

gasb_status gasb_dp_shard_map(gasb_schedule s, int32_t world, uint32_t* h_owner_local, int64_t* h_rows_per_rank) {
    return guard([&] {
        require(s && world >= 1 && world <= kMaxWorld, "dp: bad argument");
        std::vector<uint32_t> ol;
        std::vector<int64_t> no;
        shard_map(schedule_of(s), world, ol, no);
        if (h_owner_local) std::copy(ol.begin(), ol.end(), h_owner_local);
        if (h_rows_per_rank) std::copy(no.begin(), no.end(), h_rows_per_rank);
    });
}

gasb_status gasb_dp_destroy(gasb_dp d) {
    delete d;
    return GASB_OK;
}

gasb_status gasb_epoch_order(int32_t num_parts, uint64_t seed, int64_t epoch, int32_t shuffle, int32_t* h_order) {
    return guard([&] {
        require(num_parts > 0 && h_order, "epoch_order: bad argument");
        std::vector<int32_t> o;
        epoch_order(num_parts, seed, epoch, shuffle != 0, o);
        std::copy(o.begin(), o.end(), h_order);
    });
}

}  // extern "C"
