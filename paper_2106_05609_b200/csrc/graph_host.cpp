// Host side of the partition-batch loader: build_graph, make_batch_plan,
// build_plan_aggregation and BatchSchedule::build, plus the synthetic graph generator.
//
// All index work is bit-exact with the reference (SURVEY §8c parity contract):
//  - build_graph      src/graph.cpp:25-61   canonical CSR (per-row sort + unique)
//  - make_batch_plan  src/graph.cpp:78-134  V_b = B_b ∪ N(B_b) sorted, halos, local CSR
//  - build_plan_aggregation src/layers.cpp:42-70  gcn coeff float(1/(sqrt(dw+1)*sqrt(dv+1)))
//    in CSR order with the self term appended at the row end when no stored self-loop.
// Parallelism (OpenMP over rows / parts) never changes results: every output element is
// produced by exactly one thread in a fixed order.
#include <omp.h>

#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>

#include "gasb_internal.hpp"

struct gasb_graph_s {
    gasb::Graph g;
};
struct gasb_schedule_s {
    gasb::Schedule s;
};

namespace gasb {

static Graph build_graph_impl(const int32_t* src, const int32_t* dst, int64_t m, int32_t n, bool sym) {
    require(n >= 0, "build_graph: negative node count");
    int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t i = 0; i < m; ++i)
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) bad = std::max(bad, i);
    if (bad >= 0)
        throw std::invalid_argument("build_graph: edge (" + std::to_string(src[bad]) + "," +
                                    std::to_string(dst[bad]) + ") out of range for " + std::to_string(n) +
                                    " nodes");
    Graph g;
    g.num_nodes = n;
    g.symmetric = sym;
    // Row v collects sources w of edges w -> v (+ v into row u when symmetrizing, u != v).
    std::vector<int64_t> cnt(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        __atomic_fetch_add(&cnt[dst[i] + 1], 1, __ATOMIC_RELAXED);
        if (sym && src[i] != dst[i]) __atomic_fetch_add(&cnt[src[i] + 1], 1, __ATOMIC_RELAXED);
    }
    for (int32_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
    std::vector<int32_t> buf(static_cast<size_t>(cnt[n]));
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        buf[__atomic_fetch_add(&pos[dst[i]], 1, __ATOMIC_RELAXED)] = src[i];
        if (sym && src[i] != dst[i]) buf[__atomic_fetch_add(&pos[src[i]], 1, __ATOMIC_RELAXED)] = dst[i];
    }
    // Sort + dedup each row (order of insertion is irrelevant after sorting).
    std::vector<int64_t> uniq(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int32_t v = 0; v < n; ++v) {
        int32_t* b = buf.data() + cnt[v];
        int32_t* e = buf.data() + cnt[v + 1];
        std::sort(b, e);
        uniq[v + 1] = std::unique(b, e) - b;
    }
    g.row_offsets.assign(static_cast<size_t>(n) + 1, 0);
    for (int32_t v = 0; v < n; ++v) g.row_offsets[v + 1] = g.row_offsets[v] + uniq[v + 1];
    g.cols.resize(static_cast<size_t>(g.row_offsets[n]));
#pragma omp parallel for schedule(dynamic, 1024)
    for (int32_t v = 0; v < n; ++v)
        std::memcpy(g.cols.data() + g.row_offsets[v], buf.data() + cnt[v], sizeof(int32_t) * uniq[v + 1]);
    return g;
}

void build_plan(const Graph& g, const int32_t* batch, int64_t nb, bool full, HostPlan& p,
                std::vector<uint8_t>& mark, std::vector<int32_t>& g2l) {
    // graph.cpp:79-86: non-empty, in range, strictly increasing.
    require(nb > 0, "make_batch_plan: empty batch");
    for (int64_t i = 0; i < nb; ++i) {
        require(batch[i] >= 0 && batch[i] < g.num_nodes, "make_batch_plan: node id out of range");
        require(i == 0 || batch[i] > batch[i - 1], "make_batch_plan: batch nodes must be sorted and unique");
    }
    const int32_t n = g.num_nodes;
    if (static_cast<int32_t>(mark.size()) < n) mark.assign(static_cast<size_t>(n), 0);
    if (static_cast<int32_t>(g2l.size()) < n) g2l.assign(static_cast<size_t>(n), -1);
    // mark: 1 = halo candidate (in V_b), 2 = batch node.
    for (int64_t i = 0; i < nb; ++i) mark[batch[i]] = 2;
    std::vector<int32_t> touched;
    touched.reserve(static_cast<size_t>(nb) * 8);
    for (int64_t i = 0; i < nb; ++i)
        for (int64_t e = g.row_offsets[batch[i]]; e < g.row_offsets[batch[i] + 1]; ++e) {
            const int32_t w = g.cols[e];
            if (mark[w] == 0) {
                mark[w] = 1;
                touched.push_back(w);
            }
        }
    // V_b sorted = merge of the sorted batch and the sorted halo set (graph.cpp:101-112
    // scans 0..n-1; the merge yields the identical sequence in O(|V_b| log |V_b|)).
    std::sort(touched.begin(), touched.end());
    p.batch.assign(batch, batch + nb);
    p.halo = touched;
    const int64_t nh = static_cast<int64_t>(touched.size());
    const int64_t ne = nb + nh;
    p.extended.resize(static_cast<size_t>(ne));
    std::merge(p.batch.begin(), p.batch.end(), p.halo.begin(), p.halo.end(), p.extended.begin());
    p.is_halo.resize(static_cast<size_t>(ne));
    p.batch_local_rows.clear();
    p.halo_local_rows.clear();
    p.batch_local_rows.reserve(static_cast<size_t>(nb));
    p.halo_local_rows.reserve(static_cast<size_t>(nh));
    for (int64_t i = 0; i < ne; ++i) {
        const int32_t v = p.extended[i];
        const bool halo = mark[v] == 1;
        p.is_halo[i] = halo;
        g2l[v] = static_cast<int32_t>(i);
        (halo ? p.halo_local_rows : p.batch_local_rows).push_back(static_cast<int32_t>(i));
    }
    if (full) {  // local_graph: in-edges of batch rows only (graph.cpp:114-133)
        p.local_rowptr.assign(static_cast<size_t>(ne) + 1, 0);
        for (int64_t i = 0; i < ne; ++i)
            p.local_rowptr[i + 1] = p.local_rowptr[i] + (p.is_halo[i] ? 0 : g.degree(p.extended[i]));
        p.local_cols.resize(static_cast<size_t>(p.local_rowptr[ne]));
        for (int64_t i = 0; i < ne; ++i) {
            if (p.is_halo[i]) continue;
            int64_t pos = p.local_rowptr[i];
            const int32_t v = p.extended[i];
            for (int64_t e = g.row_offsets[v]; e < g.row_offsets[v + 1]; ++e) p.local_cols[pos++] = g2l[g.cols[e]];
        }
    }
    // build_plan_aggregation (layers.cpp:42-70).
    int64_t tot = 0;
    for (int64_t i = 0; i < nb; ++i) tot += g.degree(batch[i]);
    p.gcn_rowptr.assign(static_cast<size_t>(nb) + 1, 0);
    p.gcn_cols.resize(static_cast<size_t>(tot + nb));
    p.gcn_coeffs.resize(static_cast<size_t>(tot + nb));
    if (full) {
        p.sum_rowptr.assign(static_cast<size_t>(nb) + 1, 0);
        p.sum_cols.resize(static_cast<size_t>(tot));
        p.sum_coeffs.assign(static_cast<size_t>(tot), 1.0f);
    }
    int64_t eg = 0, es = 0;
    for (int64_t i = 0; i < nb; ++i) {
        const int32_t v = batch[i];
        const int32_t lv = p.batch_local_rows[i];
        const double cv = std::sqrt(static_cast<double>(g.degree(v)) + 1.0);
        bool self_seen = false;
        for (int64_t e = g.row_offsets[v]; e < g.row_offsets[v + 1]; ++e) {
            const int32_t w = g.cols[e];
            const double cw = std::sqrt(static_cast<double>(g.degree(w)) + 1.0);
            p.gcn_cols[eg] = g2l[w];
            p.gcn_coeffs[eg++] = static_cast<float>(1.0 / (cw * cv));
            if (full) p.sum_cols[es++] = g2l[w];
            if (w == v) self_seen = true;
        }
        if (!self_seen) {
            p.gcn_cols[eg] = lv;
            p.gcn_coeffs[eg++] = static_cast<float>(1.0 / (cv * cv));
        }
        p.gcn_rowptr[i + 1] = eg;
        if (full) p.sum_rowptr[i + 1] = es;
    }
    p.gcn_cols.resize(static_cast<size_t>(eg));
    p.gcn_coeffs.resize(static_cast<size_t>(eg));
    // restore scratch
    for (int64_t i = 0; i < nb; ++i) mark[batch[i]] = 0;
    for (int32_t w : touched) mark[w] = 0;
}

// ---- synthetic generator -----------------------------------------------------------
static inline uint64_t mix64(uint64_t x) {  // splitmix64 finalizer (as gas::mix64, rng.hpp:11-16)
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static inline double u01(uint64_t seed, uint64_t a, uint64_t b) {
    return static_cast<double>(mix64(mix64(seed ^ mix64(a)) ^ mix64(b)) >> 11) * 0x1.0p-53;
}

static int32_t sample_prefix(const double* cum, int64_t lo, int64_t hi, double target) {
    // smallest index i in [lo, hi) with cum[i+1] > target, cum[lo] = start
    int64_t a = lo, b = hi - 1;
    while (a < b) {
        int64_t mid = (a + b) >> 1;
        if (cum[mid + 1] > target) b = mid;
        else a = mid + 1;
    }
    return static_cast<int32_t>(a);
}

}  // namespace gasb

using namespace gasb;

namespace {
thread_local std::string t_last_error;
}
void gasb::set_last_error(const std::string& m) { t_last_error = m; }

extern "C" {

const char* gasb_last_error(void) { return t_last_error.c_str(); }
int32_t gasb_abi_version(void) { return 1; }

gasb_status gasb_graph_build(const int32_t* src, const int32_t* dst, int64_t m, int32_t n, int32_t sym,
                             gasb_graph* out) {
    return guard([&] {
        require(out != nullptr && (m == 0 || (src && dst)), "build_graph: null argument");
        require(m >= 0, "build_graph: negative edge count");
        auto* h = new gasb_graph_s{build_graph_impl(src, dst, m, n, sym != 0)};
        *out = h;
    });
}

gasb_status gasb_graph_from_csr(int32_t n, const int64_t* ro, const int32_t* cols, int32_t sym, gasb_graph* out) {
    return guard([&] {
        require(n >= 0 && ro && out, "graph_from_csr: bad argument");
        require(ro[0] == 0, "graph_from_csr: row_offsets[0] != 0");
        bool ok = true;
#pragma omp parallel for schedule(dynamic, 4096) reduction(&& : ok)
        for (int32_t v = 0; v < n; ++v) {
            if (ro[v + 1] < ro[v]) {
                ok = false;
                continue;
            }
            for (int64_t e = ro[v]; e < ro[v + 1]; ++e)
                if (cols[e] < 0 || cols[e] >= n || (e > ro[v] && cols[e] <= cols[e - 1])) ok = false;
        }
        require(ok, "graph_from_csr: CSR rows must be sorted, unique and in range");
        auto* h = new gasb_graph_s();
        h->g.num_nodes = n;
        h->g.symmetric = sym != 0;
        h->g.row_offsets.assign(ro, ro + n + 1);
        h->g.cols.assign(cols, cols + ro[n]);
        *out = h;
    });
}

gasb_status gasb_graph_info(gasb_graph g, int32_t* n, int64_t* m) {
    return guard([&] {
        require(g, "graph_info: null graph");
        if (n) *n = g->g.num_nodes;
        if (m) *m = g->g.num_edges();
    });
}

gasb_status gasb_graph_csr(gasb_graph g, const int64_t** ro, const int32_t** cols) {
    return guard([&] {
        require(g, "graph_csr: null graph");
        *ro = g->g.row_offsets.data();
        *cols = g->g.cols.data();
    });
}

gasb_status gasb_graph_destroy(gasb_graph g) {
    delete g;
    return GASB_OK;
}

gasb_status gasb_synth_pairs(const gasb_synth_params* p, int32_t* src, int32_t* dst, int32_t* community) {
    return guard([&] {
        require(p && src && dst, "synth_pairs: null argument");
        const int32_t n = p->num_nodes, K = p->num_communities;
        require(n > 0 && K > 0 && K <= n, "synth_pairs: need 0 < communities <= nodes");
        require(p->gamma > 1.0 && p->min_weight > 0.0 && p->max_weight >= p->min_weight, "synth_pairs: bad weights");
        const uint64_t seed = p->seed;
        // node weights (Pareto, exponent gamma)
        std::vector<double> w(static_cast<size_t>(n));
#pragma omp parallel for schedule(static)
        for (int32_t v = 0; v < n; ++v) {
            const double u = u01(seed, 0x77656967ull, static_cast<uint64_t>(v));  // "weig"
            w[v] = std::min(p->max_weight, p->min_weight * std::pow(1.0 - u, -1.0 / (p->gamma - 1.0)));
        }
        // balanced random communities: rank nodes by a hash key, community = rank mod K
        std::vector<std::pair<uint64_t, int32_t>> key(static_cast<size_t>(n));
        for (int32_t v = 0; v < n; ++v) key[v] = {mix64(seed ^ mix64(0x636f6d6dull ^ mix64(static_cast<uint64_t>(v)))), v};
        std::sort(key.begin(), key.end());
        std::vector<int32_t> comm(static_cast<size_t>(n));
        for (int32_t r = 0; r < n; ++r) comm[key[r].second] = r % K;
        // global prefix sums, and per-community prefix sums over members in id order
        std::vector<double> cum(static_cast<size_t>(n) + 1, 0.0);
        for (int32_t v = 0; v < n; ++v) cum[v + 1] = cum[v] + w[v];
        std::vector<int64_t> cstart(static_cast<size_t>(K) + 1, 0);
        for (int32_t v = 0; v < n; ++v) cstart[comm[v] + 1]++;
        for (int32_t c = 0; c < K; ++c) cstart[c + 1] += cstart[c];
        std::vector<int32_t> members(static_cast<size_t>(n));
        std::vector<double> ccum(static_cast<size_t>(n) + static_cast<size_t>(K), 0.0);
        {
            std::vector<int64_t> fill(cstart.begin(), cstart.end() - 1);
            for (int32_t v = 0; v < n; ++v) members[fill[comm[v]]++] = v;
            // ccum layout: community c occupies [cstart[c] + c, cstart[c+1] + c] (size+1)
            for (int32_t c = 0; c < K; ++c) {
                double* cc = ccum.data() + cstart[c] + c;
                cc[0] = 0.0;
                for (int64_t i = cstart[c]; i < cstart[c + 1]; ++i) cc[i - cstart[c] + 1] = cc[i - cstart[c]] + w[members[i]];
            }
        }
        const double W = cum[n];
        const int64_t m = p->num_pairs;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            const uint64_t ui = static_cast<uint64_t>(i);
            const int32_t u = sample_prefix(cum.data(), 0, n, u01(seed, ui, 1) * W);
            int32_t v;
            if (u01(seed, ui, 2) < p->intra_fraction) {
                const int32_t c = comm[u];
                const double* cc = ccum.data() + cstart[c] + c;
                const int64_t sz = cstart[c + 1] - cstart[c];
                const int32_t k = sample_prefix(cc, 0, sz, u01(seed, ui, 3) * cc[sz]);
                v = members[cstart[c] + k];
            } else {
                v = sample_prefix(cum.data(), 0, n, u01(seed, ui, 3) * W);
            }
            src[i] = u;
            dst[i] = v;
        }
        if (community) std::memcpy(community, comm.data(), sizeof(int32_t) * static_cast<size_t>(n));
    });
}

gasb_status gasb_synth_features(int64_t n, int32_t dim, int64_t ld, uint64_t seed, float* out) {
    return guard([&] {
        require(n >= 0 && dim >= 0 && ld >= dim && out, "synth_features: bad argument");
#pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < n; ++v) {
            float* row = out + v * ld;
            for (int32_t j = 0; j < dim; ++j) {
                const uint64_t c = static_cast<uint64_t>(v) * static_cast<uint64_t>(dim) + static_cast<uint64_t>(j);
                double u1 = u01(seed, c, 0x6e31ull);
                if (u1 <= 0.0) u1 = 0x1.0p-53;
                const double u2 = u01(seed, c, 0x6e32ull);
                row[j] = static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
            }
            for (int64_t j = dim; j < ld; ++j) row[j] = 0.0f;
        }
    });
}

static void build_schedule_from_batches(const Graph& g, const std::vector<std::vector<int32_t>>& batches, bool full,
                                        Schedule& s) {
    s.graph = &g;
    s.num_parts = static_cast<int32_t>(batches.size());
    s.plans.resize(batches.size());
    std::string err;
    bool failed = false;
#pragma omp parallel
    {
        std::vector<uint8_t> mark;
        std::vector<int32_t> g2l;
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < static_cast<int64_t>(batches.size()); ++b) {
            try {
                build_plan(g, batches[b].data(), static_cast<int64_t>(batches[b].size()), full, s.plans[b], mark, g2l);
            } catch (const std::exception& e) {
#pragma omp critical
                {
                    failed = true;
                    err = e.what();
                }
            }
        }
    }
    if (failed) throw std::invalid_argument(err);
}

gasb_status gasb_schedule_build(gasb_graph g, const int32_t* assignment, int32_t num_parts, int32_t flags,
                                gasb_schedule* out) {
    return guard([&] {
        require(g && assignment && out, "schedule_build: null argument");
        require(num_parts > 0, "schedule_build: num_parts must be positive");
        const Graph& G = g->g;
        if (flags & GASB_PLAN_DEVICE) {
            auto* h = new gasb_schedule_s();
            try {
                const auto t0 = std::chrono::steady_clock::now();
                build_schedule_device(G, assignment, num_parts, (flags & GASB_PLAN_FULL) != 0, h->s);
                h->s.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            } catch (...) {
                delete h;
                throw;
            }
            *out = h;
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        // partition_from_assignment (partition.cpp:314-328): parts sorted, non-empty.
        std::vector<std::vector<int32_t>> parts(static_cast<size_t>(num_parts));
        for (int32_t v = 0; v < G.num_nodes; ++v) {
            require(assignment[v] >= 0 && assignment[v] < num_parts, "partition_from_assignment: part id out of range");
            parts[assignment[v]].push_back(v);
        }
        for (const auto& p : parts) require(!p.empty(), "partition_from_assignment: empty part");
        auto* h = new gasb_schedule_s();
        try {
            build_schedule_from_batches(G, parts, (flags & GASB_PLAN_FULL) != 0, h->s);
        } catch (...) {
            delete h;
            throw;
        }
        h->s.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *out = h;
    });
}

gasb_status gasb_schedule_build_batches(gasb_graph g, const int32_t* const* batches, const int64_t* sizes,
                                        int32_t nbatches, int32_t flags, gasb_schedule* out) {
    return guard([&] {
        require(g && out && nbatches >= 0, "schedule_build_batches: bad argument");
        std::vector<std::vector<int32_t>> parts(static_cast<size_t>(nbatches));
        for (int32_t b = 0; b < nbatches; ++b) parts[b].assign(batches[b], batches[b] + sizes[b]);
        auto* h = new gasb_schedule_s();
        try {
            build_schedule_from_batches(g->g, parts, (flags & GASB_PLAN_FULL) != 0, h->s);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

gasb_status gasb_schedule_num_parts(gasb_schedule s, int32_t* out) {
    return guard([&] {
        require(s && out, "schedule: null argument");
        *out = s->s.num_parts;
    });
}

gasb_status gasb_schedule_timing(gasb_schedule s, double* device_ms, double* total_ms) {
    return guard([&] {
        require(s, "schedule: null argument");
        if (device_ms) *device_ms = s->s.device_ms;
        if (total_ms) *total_ms = s->s.total_ms;
    });
}

gasb_status gasb_plan_sizes(gasb_schedule s, int32_t part, int64_t* z) {
    return guard([&] {
        require(s && part >= 0 && part < s->s.num_parts, "plan_sizes: part out of range");
        const HostPlan& p = s->s.plans[part];
        z[0] = static_cast<int64_t>(p.batch.size());
        z[1] = static_cast<int64_t>(p.extended.size());
        z[2] = static_cast<int64_t>(p.halo.size());
        z[3] = p.local_rowptr.empty() ? -1 : p.local_rowptr.back();
        z[4] = static_cast<int64_t>(p.gcn_cols.size());
        z[5] = p.sum_rowptr.empty() ? -1 : static_cast<int64_t>(p.sum_cols.size());
    });
}

gasb_status gasb_plan_copy(gasb_schedule s, int32_t part, int32_t* extended, int32_t* halo, uint8_t* is_halo,
                           int32_t* blr, int32_t* hlr, int64_t* lrp, int32_t* lcols, int64_t* grp, int32_t* gcols,
                           float* gco, int64_t* srp, int32_t* scols, float* sco) {
    return guard([&] {
        require(s && part >= 0 && part < s->s.num_parts, "plan_copy: part out of range");
        const HostPlan& p = s->s.plans[part];
        auto cp = [](auto* dst, const auto& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
        };
        require(!(lrp || lcols) || !p.local_rowptr.empty(), "plan_copy: local graph not built (GASB_PLAN_FULL)");
        require(!(srp || scols || sco) || !p.sum_rowptr.empty(), "plan_copy: sum stencil not built (GASB_PLAN_FULL)");
        cp(extended, p.extended);
        cp(halo, p.halo);
        cp(is_halo, p.is_halo);
        cp(blr, p.batch_local_rows);
        cp(hlr, p.halo_local_rows);
        cp(lrp, p.local_rowptr);
        cp(lcols, p.local_cols);
        cp(grp, p.gcn_rowptr);
        cp(gcols, p.gcn_cols);
        cp(gco, p.gcn_coeffs);
        cp(srp, p.sum_rowptr);
        cp(scols, p.sum_cols);
        cp(sco, p.sum_coeffs);
    });
}

gasb_status gasb_schedule_destroy(gasb_schedule s) {
    delete s;
    return GASB_OK;
}

/* save_partition (io.cpp:187-192): one "node part" line per node, node order. */
gasb_status gasb_partition_save(const char* path, const int32_t* assignment, int32_t num_nodes) {
    return guard([&] {
        require(path && (assignment || num_nodes == 0), "save_partition: null argument");
        std::FILE* f = std::fopen(path, "w");
        if (!f) throw std::runtime_error(std::string("cannot write partition file: ") + path);
        for (int32_t v = 0; v < num_nodes; ++v) std::fprintf(f, "%d %d\n", v, assignment[v]);
        std::fclose(f);
    });
}

/* load_partition (io.cpp:194-217): '#' comments and blank lines skipped, "node part" per
 * line (later lines win), then partition_from_assignment (partition.cpp:314-328).
 * runtime_error: unopenable file, malformed line, node out of range, negative part,
 * unassigned node; invalid_argument: an empty part. */
gasb_status gasb_partition_load(const char* path, int32_t num_nodes, int32_t* assignment, int32_t* num_parts) {
    return guard([&] {
        require(path && num_parts && (assignment || num_nodes == 0), "load_partition: null argument");
        std::FILE* f = std::fopen(path, "r");
        if (!f) throw std::runtime_error(std::string("cannot open partition file: ") + path);
        std::vector<int32_t> a(static_cast<size_t>(num_nodes), -1);
        int32_t max_part = -1;
        std::string line;
        size_t lineno = 0;
        auto fail = [&](const char* what) {
            std::fclose(f);
            throw std::runtime_error(std::string(path) + ":" + std::to_string(lineno) + ": " + what);
        };
        char buf[4096];
        while (std::fgets(buf, sizeof(buf), f)) {
            line.assign(buf);
            while (!line.empty() && line.back() != '\n' && std::fgets(buf, sizeof(buf), f)) line += buf;
            ++lineno;
            const size_t hash = line.find('#');
            std::string body = hash == std::string::npos ? line : line.substr(0, hash);
            if (body.find_first_not_of(" \t\r\n") == std::string::npos) continue;
            long long node = 0, part = 0;
            char* end = nullptr;
            const char* p0 = body.c_str();
            errno = 0;
            node = std::strtoll(p0, &end, 10);
            if (end == p0 || errno) fail("expected 'node_id part_id'");
            const char* p1 = end;
            part = std::strtoll(p1, &end, 10);
            if (end == p1 || errno) fail("expected 'node_id part_id'");
            if (node < 0 || node >= num_nodes) fail("node id out of range");
            if (part < 0) fail("negative part id");
            a[static_cast<size_t>(node)] = static_cast<int32_t>(part);
            max_part = std::max(max_part, static_cast<int32_t>(part));
        }
        std::fclose(f);
        for (int32_t v = 0; v < num_nodes; ++v)
            if (a[v] < 0) throw std::runtime_error(std::string(path) + ": node " + std::to_string(v) + " unassigned");
        std::vector<int64_t> count(static_cast<size_t>(max_part + 1), 0);
        for (int32_t v : a) ++count[v];
        for (int64_t c : count) require(c > 0, "partition_from_assignment: empty part");
        std::copy(a.begin(), a.end(), assignment);
        *num_parts = max_part + 1;
    });
}

/* random_partition (partition.cpp:330-342): node order shuffled by Rng(derive_seed(seed,
 * "rand")) (rng.hpp shuffle), node order[i] -> part i % num_parts. Bit-exact. */
gasb_status gasb_random_partition(int32_t num_nodes, int32_t num_parts, uint64_t seed, int32_t* assignment) {
    return guard([&] {
        require(num_parts > 0, "random_partition: num_parts must be positive");
        require(num_parts <= num_nodes, "random_partition: more parts than nodes");
        require(assignment != nullptr, "random_partition: null argument");
        std::vector<int32_t> order(static_cast<size_t>(num_nodes));
        std::iota(order.begin(), order.end(), 0);
        const uint64_t s = mix64(mix64(mix64(seed ^ mix64(0x72616e64ull)) ^ mix64(0)) ^ mix64(0));
        std::mt19937_64 gen(s);
        for (size_t i = order.size(); i > 1; --i) {  // Rng::shuffle / next_below (rng.hpp:40-61)
            const uint64_t n = i, limit = ~uint64_t{0} - (~uint64_t{0} % n);
            uint64_t x;
            do {
                x = gen();
            } while (x >= limit);
            std::swap(order[i - 1], order[x % n]);
        }
        for (size_t i = 0; i < order.size(); ++i) assignment[order[i]] = static_cast<int32_t>(i % num_parts);
    });
}

gasb_status gasb_cluster_partition(gasb_graph g, int32_t num_parts, uint64_t seed, int32_t* assignment) {
    return guard([&] {
        require(g && assignment, "cluster_partition: null argument");
        cluster_partition(g->g, num_parts, seed, assignment);
    });
}

}  // extern "C"

namespace gasb {
const Schedule& schedule_of(gasb_schedule s) { return s->s; }
}  // namespace gasb
