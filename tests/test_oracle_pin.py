"""Pins the C restatement (oracle/gas_oracle.c) to the reference: against the committed
golden fixtures generated from the compiled reference (tests/golden/make_golden.py), and
live against oracle/_ref/libref.so when it is present. CPU only."""
from pathlib import Path

import numpy as np
import pytest

from pyoracle import make_spec

G = Path(__file__).resolve().parent / "golden"
OPS = np.load(G / "ref_ops.npz")
SES = np.load(G / "ref_sessions.npz")


def test_build_graph_golden(oracle):
    ro, co = oracle.build_graph(OPS["g_edges"], 120, True)
    assert np.array_equal(ro, OPS["g_ro"]) and np.array_equal(co, OPS["g_co"])
    ro, co = oracle.build_graph(OPS["g_edges"], 120, False)
    assert np.array_equal(ro, OPS["g_ro_directed"]) and np.array_equal(co, OPS["g_co_directed"])
    ro, co = oracle.build_graph(np.array([[0, 1], [1, 2]]), 3)
    assert np.array_equal(np.diff(ro), [1, 2, 1])  # test_graph.cpp:16-23
    assert np.array_equal(ro, OPS["p3_ro"]) and np.array_equal(co, OPS["p3_co"])


def test_build_graph_errors(oracle):
    with pytest.raises(ValueError):
        oracle.build_graph(np.array([[0, 5]]), 3)  # test_graph.cpp:31-33


@pytest.mark.parametrize("name,batch", [("single", [0]), ("mid", list(range(10, 40, 3))), ("full", list(range(120)))])
def test_plans_golden(oracle, name, batch):
    p = oracle.make_plan(OPS["g_ro"], OPS["g_co"], batch)
    for k, v in p.items():
        assert np.array_equal(v, OPS[f"plan_{name}_{k}"]), k


def test_plan_errors(oracle):
    with pytest.raises(ValueError):
        oracle.make_plan(OPS["g_ro"], OPS["g_co"], [])
    with pytest.raises(ValueError):
        oracle.make_plan(OPS["g_ro"], OPS["g_co"], [1, 0])


def test_ops_golden(oracle):
    pfx = "plan_mid_"
    y, gx = oracle.aggregate(OPS[pfx + "gcn_row_ptr"], OPS[pfx + "gcn_cols"], OPS[pfx + "gcn_coeffs"], OPS["agg_x"],
                             OPS["agg_gy"])
    assert np.array_equal(y, OPS["agg_y"]) and np.array_equal(gx, OPS["agg_gx"])
    y, ga, gb = oracle.matmul(OPS["mm_a"], OPS["mm_b"], OPS["mm_gy"])
    assert np.array_equal(y, OPS["mm_y"]) and np.array_equal(ga, OPS["mm_ga"]) and np.array_equal(gb, OPS["mm_gb"])
    loss, g = oracle.softmax_ce(OPS["ce_logits"], OPS["ce_rows"], OPS["ce_labels"])
    assert np.float32(loss) == OPS["ce_loss"] and np.array_equal(g, OPS["ce_grad"])
    assert np.array_equal(oracle.glorot(7, 5, 42), OPS["glorot_7x5_s42"])
    assert np.array_equal(oracle.epoch_order(10, 3, 4), OPS["order_10_s3_e4"])


@pytest.mark.parametrize("name,kind,L", [("gcn", 0, 3), ("appnp", 2, 3), ("gcnii", 3, 4)])
def test_sessions_golden(oracle, name, kind, L):
    """Full GAS batches (forward, pushes, loss, grads, clip, Adam) are bit-exact."""
    spec = make_spec(kind=kind, num_layers=L, hidden=8, seed=11, clip_max_norm=0.5 if kind == 3 else 0.0)
    comm = SES["s_comm"]
    s = oracle.session(SES["s_ro"], SES["s_co"], SES["s_feats"], SES["s_labels"], SES["s_train"], 4, comm, 4, spec)
    assert np.array_equal(s.get_params(), SES[f"{name}_params0"])
    for i in range(4):
        p = int(SES[f"{name}_b{i}_part"])
        acts, logits, loss, grads, stepped = s.batch(p, 0, nb=int((comm == p).sum()))
        assert np.array_equal(acts, SES[f"{name}_b{i}_acts"])
        assert np.array_equal(logits, SES[f"{name}_b{i}_logits"])
        assert loss == SES[f"{name}_b{i}_loss"]
        assert stepped == bool(SES[f"{name}_b{i}_stepped"])
        if stepped:
            assert np.array_equal(grads, SES[f"{name}_b{i}_grads"])
    assert np.array_equal(s.get_params(), SES[f"{name}_params1"])
    for l in range(1, L):
        assert np.array_equal(s.get_history(l), SES[f"{name}_hist{l}"])
    assert s.epoch(1)[0] == SES[f"{name}_epoch1_loss"]
    assert np.array_equal(s.get_params(), SES[f"{name}_params2"])


def test_live_against_reference(oracle, ref):
    """Random inputs, oracle vs the compiled reference, op by op and a whole epoch."""
    rng = np.random.default_rng(5)
    n = 150
    e = rng.integers(0, n, (600, 2)).astype(np.int32)
    assert all(np.array_equal(a, b) for a, b in zip(oracle.build_graph(e, n), ref.graph(e, n).csr()))
    ro, co = ref.graph(e, n).csr()
    rg = ref.graph(csr=(ro, co))
    batch = np.sort(rng.choice(n, 30, replace=False)).astype(np.int32)
    pr, po = rg.plan(batch), oracle.make_plan(ro, co, batch)
    for k in pr:
        assert np.array_equal(pr[k], po[k]), k
    x = rng.standard_normal((len(pr["extended_nodes"]), 33)).astype(np.float32)
    gy = rng.standard_normal((30, 33)).astype(np.float32)
    a1 = ref.aggregate(pr["gcn_row_ptr"], pr["gcn_cols"], pr["gcn_coeffs"], x, gy)
    a2 = oracle.aggregate(pr["gcn_row_ptr"], pr["gcn_cols"], pr["gcn_coeffs"], x, gy)
    assert np.array_equal(a1[0], a2[0]) and np.array_equal(a1[1], a2[1])
    comm = rng.integers(0, 5, n).astype(np.int32)
    comm[:5] = np.arange(5)
    feats = rng.standard_normal((n, 10)).astype(np.float32)
    labels = rng.integers(0, 3, n).astype(np.int32)
    train = (rng.random(n) < 0.5).astype(np.uint8)
    for kind, L in [(0, 2), (2, 2), (3, 3)]:
        spec = make_spec(kind=kind, num_layers=L, hidden=6, seed=2, l2_weight=1e-3)
        so = oracle.session(ro, co, feats, labels, train, 3, comm, 5, spec)
        sr = ref.session(ro, co, feats, labels, train, 3, comm, 5, spec)
        for ep in range(2):
            assert so.epoch(ep)[0] == sr.epoch(ep)[0]
        assert np.array_equal(so.get_params(), sr.get_params())
