"""The B200 path's host loader (build_graph, make_batch_plan, build_plan_aggregation,
BatchSchedule::build) is bit-exact with the reference. CPU only (host code of libgasb.so)."""
from pathlib import Path

import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset

G = Path(__file__).resolve().parent / "golden"
OPS = np.load(G / "ref_ops.npz")


def test_build_graph_golden():
    g = gb.build_graph(OPS["g_edges"], 120)
    ro, co = g.csr()
    assert np.array_equal(ro, OPS["g_ro"]) and np.array_equal(co, OPS["g_co"])
    ro, co = gb.build_graph(OPS["g_edges"], 120, symmetrize=False).csr()
    assert np.array_equal(ro, OPS["g_ro_directed"]) and np.array_equal(co, OPS["g_co_directed"])


def test_build_graph_edge_cases():
    g = gb.build_graph(np.zeros((0, 2), np.int32), 2)  # test_graph.cpp:25-30
    assert g.num_edges == 0 and np.array_equal(g.csr()[0], [0, 0, 0])
    g = gb.build_graph(np.array([[0, 1], [0, 1], [1, 0], [2, 2]]), 3)  # test_graph.cpp:36-42
    assert np.array_equal(np.diff(g.csr()[0]), [1, 1, 1])
    with pytest.raises(ValueError):
        gb.build_graph(np.array([[0, 5]]), 3)
    with pytest.raises(ValueError):
        gb.graph_from_csr(np.array([0, 2, 2]), np.array([1, 1]))  # unsorted / duplicate row


@pytest.mark.parametrize("name,batch", [("single", [0]), ("mid", list(range(10, 40, 3))), ("full", list(range(120)))])
def test_plans_golden(name, batch):
    g = gb.build_graph(OPS["g_edges"], 120)
    p = gb.make_batch_plan(g, batch)
    for k in ("extended_nodes", "halo_nodes", "is_halo", "batch_local_rows", "halo_local_rows", "gcn_row_ptr",
              "gcn_cols", "gcn_coeffs", "sum_row_ptr", "sum_cols", "sum_coeffs"):
        assert np.array_equal(getattr(p, k), OPS[f"plan_{name}_{k}"]), k
    assert np.array_equal(p.local_row_offsets, OPS[f"plan_{name}_local_row_offsets"])
    assert np.array_equal(p.local_col_indices, OPS[f"plan_{name}_local_col_indices"])


def test_plan_errors():
    g = gb.build_graph(OPS["g_edges"], 120)
    for bad in ([], [1, 0], [3, 3], [-1], [120]):
        with pytest.raises(ValueError):
            gb.make_batch_plan(g, bad)


def test_schedule_matches_oracle_on_cora_shape(oracle):
    ds = make_dataset("cora", with_features=False)
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, ds.workload.parts, full=True)
    ro_o, co_o = oracle.build_graph(*_edges_of(ds))
    assert np.array_equal(ro_o, ds.row_offsets) and np.array_equal(co_o, ds.cols)
    for p, nodes in enumerate(gb.partition_parts(ds.assignment, ds.workload.parts)):
        po, pg = oracle.make_plan(ds.row_offsets, ds.cols, nodes), sched.plan(p)
        for k, v in po.items():
            assert np.array_equal(v, getattr(pg, k)), (p, k)


def _edges_of(ds):
    # regenerate the undirected pair list the dataset was built from
    w = ds.workload
    e, _ = gb.synth_pairs(w.num_nodes, w.num_pairs, w.parts * w.comm_per_part, w.intra_fraction, 2.5, 1.0,
                          w.max_weight, w.seed)
    return e, w.num_nodes


def test_synth_is_deterministic():
    a = gb.synth_pairs(500, 3000, 5, 0.5, seed=9)
    b = gb.synth_pairs(500, 3000, 5, 0.5, seed=9)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    sizes = np.bincount(a[1])
    assert sizes.max() - sizes.min() <= 1
    x1, x2 = gb.synth_features(50, 7, 3), gb.synth_features(50, 7, 3)
    assert np.array_equal(x1, x2) and abs(float(x1.mean())) < 0.5
