// C++ shim (include/gasb/gas.hpp) compiled against libgasb.so and run on the host.
// Host-only parts run everywhere: Graph, BatchSchedule (plans + gcn stencil) and the error
// mapping. Device parts (HistoryStore, Trainer) run when a GPU is present; without one the
// constructor must fail with std::runtime_error (CUDA error), never silently.
//
// Known answers: SPEC.md:278-279 (GCN on the path P3, W = I, h = 1: node 0 -> 1/2 + 1/sqrt 6).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "gasb/gas.hpp"

using namespace gas::b200;

static int failures = 0;
#define EXPECT(c)                                                    \
    do {                                                             \
        if (!(c)) {                                                  \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                              \
        }                                                            \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // P3: 0 - 1 - 2 (undirected), symmetrized
    std::vector<NodeId> src{0, 1}, dst{1, 2};
    Graph g = Graph::build(src, dst, 3);
    EXPECT(g.num_nodes() == 3);
    EXPECT(g.num_edges() == 4);
    EXPECT(g.row_offsets()[3] == 4);

    // one part -> no halos; stencil of node 0 = [(1, 1/sqrt(2*3)), (0, 1/2)] (self term last)
    std::vector<std::int32_t> one{0, 0, 0};
    BatchSchedule s1 = BatchSchedule::build(g, one, 1);
    BatchPlan p = s1.plan(0);
    EXPECT(p.halo_nodes.empty());
    EXPECT(p.gcn_row_ptr.size() == 4 && p.gcn_row_ptr[1] == 2);
    EXPECT(p.gcn_cols[0] == 1 && p.gcn_cols[1] == 0);
    EXPECT(p.gcn_coeffs[0] == static_cast<float>(1.0 / (std::sqrt(2.0) * std::sqrt(3.0))));
    EXPECT(p.gcn_coeffs[1] == static_cast<float>(1.0 / (std::sqrt(2.0) * std::sqrt(2.0))));
    const double y0 = static_cast<double>(p.gcn_coeffs[0]) + p.gcn_coeffs[1];  // h = 1, W = I
    EXPECT(std::fabs(y0 - (0.5 + 1.0 / std::sqrt(6.0))) < 1e-7);

    // partitioners (host): every node assigned, every part non-empty, deterministic
    {
        std::vector<NodeId> rs, rd;
        for (NodeId v = 0; v < 60; ++v) {
            rs.push_back(v);
            rd.push_back((v * 7 + 3) % 60);
            rs.push_back(v);
            rd.push_back((v + 1) % 60);
        }
        Graph rg = Graph::build(rs, rd, 60);
        auto a = cluster_partition(rg, 4, 1);
        auto b = cluster_partition(rg, 4, 1);
        EXPECT(a == b && a.size() == 60);
        std::vector<int> cnt(4, 0);
        for (auto x : a) ++cnt[static_cast<std::size_t>(x)];
        EXPECT(cnt[0] > 0 && cnt[1] > 0 && cnt[2] > 0 && cnt[3] > 0);
        EXPECT(throws<std::invalid_argument>([&] { cluster_partition(rg, 0); }));
        EXPECT(random_partition(60, 4, 2).size() == 60);
    }

    // two parts {0,1} | {2}: part 0 sees node 2 as its halo
    std::vector<std::int32_t> two{0, 0, 1};
    BatchSchedule s2 = BatchSchedule::build(g, two, 2);
    EXPECT(s2.num_parts() == 2);
    BatchPlan q = s2.plan(0);
    EXPECT(q.batch_nodes == (std::vector<NodeId>{0, 1}));
    EXPECT(q.halo_nodes == (std::vector<NodeId>{2}));
    EXPECT(q.extended_nodes == (std::vector<NodeId>{0, 1, 2}));

    // error mapping (make_batch_plan / build_graph throw std::invalid_argument)
    std::vector<NodeId> bad_src{0}, bad_dst{7};
    EXPECT(throws<std::invalid_argument>([&] { Graph::build(bad_src, bad_dst, 3); }));
    std::vector<std::int32_t> bad_assign{0, 0, 5};
    EXPECT(throws<std::invalid_argument>([&] { BatchSchedule::build(g, bad_assign, 2); }));
    EXPECT(throws<std::invalid_argument>([&] { s2.plan(9); }));

    // device part: HistoryStore push -> pull identity, fresh rows are zeros
    bool have_gpu = true;
    try {
        HistoryStore h(3, 3, 4);
        std::vector<NodeId> ids{2, 0};
        std::vector<float> rows{1, 2, 3, 4, 5, 6, 7, 8};
        h.push(1, ids, rows);
        DenseMatrix got = h.pull(1, std::vector<NodeId>{0, 1, 2});
        EXPECT(got.row(0)[0] == 5 && got.row(1)[3] == 0 && got.row(2)[3] == 4);
        EXPECT(h.last_push_step(1, 2) == 0 && h.last_push_step(1, 1) == -1);
        h.advance_step();
        EXPECT(h.step() == 1);
        EXPECT(throws<std::invalid_argument>([&] { h.pull(4, ids); }));  // layer out of [1, 3]
        EXPECT(throws<std::invalid_argument>([&] { h.pull(0, ids); }));
        std::vector<NodeId> oob{3};
        EXPECT(throws<std::invalid_argument>([&] { h.pull(1, oob); }));  // id out of range
        // GPU batch-plan builder: same plan as the host builder, same errors
        BatchSchedule d2 = BatchSchedule::build(g, two, 2, false, true);
        BatchPlan dq = d2.plan(0);
        EXPECT(dq.extended_nodes == q.extended_nodes && dq.halo_nodes == q.halo_nodes);
        EXPECT(dq.gcn_cols == q.gcn_cols && dq.gcn_coeffs == q.gcn_coeffs && dq.gcn_row_ptr == q.gcn_row_ptr);
        EXPECT(throws<std::invalid_argument>([&] { BatchSchedule::build(g, bad_assign, 2, false, true); }));
        // GASH checkpoint round trip (history.cpp:130-178): tables kept, stamps 0, step 0
        const std::string path = "/tmp/gasb_shim_test.gash";
        h.save_checkpoint(path);
        HistoryStore back = HistoryStore::load_checkpoint(path);
        EXPECT(back.num_layers() == 3 && back.num_nodes() == 3 && back.dim() == 4);
        DenseMatrix b0 = back.pull(1, std::vector<NodeId>{0, 2});
        EXPECT(b0.row(0)[0] == 5 && b0.row(1)[3] == 4);
        EXPECT(back.step() == 0 && back.last_push_step(1, 1) == 0);
        EXPECT(throws<std::runtime_error>([&] { HistoryStore::load_checkpoint("/nonexistent/x.gash"); }));
        std::remove(path.c_str());
        // a world-1 data-parallel trainer over the P3 graph: one epoch, both parts' losses
        std::vector<float> feats{1.f, 0.f, 0.f, 1.f, 1.f, 1.f};
        std::vector<std::int32_t> labels{0, 1, 0};
        std::vector<std::uint8_t> mask{1, 1, 1};
        ModelSpec spec;
        spec.num_layers = 2;
        spec.hidden = 4;
        TrainerOptions topt;
        topt.use_graphs = 0;
        Trainer tr(s2, feats, 2, labels, mask, 2, spec, topt);
        DataParallel dp(tr, 0, 1);
        EXPECT(dp.export_handle().size() == GASB_DP_HANDLE_BYTES);
        dp.epoch_async(0);
        dp.check_done();
        const std::vector<double> pl = dp.part_losses(2);
        EXPECT(pl.size() == 2 && pl[0] > 0.0 && pl[1] > 0.0);
        EXPECT(throws<std::invalid_argument>([&] { DataParallel bad(tr, 1, 1); }));
    } catch (const std::runtime_error& e) {
        have_gpu = false;
        std::printf("no device: %s\n", e.what());
    }
    std::printf("%s %d failures\n", have_gpu ? "gpu" : "host-only", failures);
    return failures == 0 ? 0 : 1;
}
