"""Generates the golden fixtures in tests/golden/ from the REFERENCE ITSELF
(oracle/_ref/libref.so = /root/reference/proj/src compiled in place, see oracle/Makefile).

Run in the dev container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The fixtures are committed; the tests compare the C restatement (oracle/) and the B200
path against them on machines without the reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent / "oracle"))
from pyoracle import RefLib, make_spec  # noqa: E402


def small_graph(n=120, m=400, seed=0):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    e = np.stack([u, v], 1).astype(np.int32)
    e = np.concatenate([e, e[:7], np.array([[3, 3], [5, 5], [7, 7]], np.int32)])  # duplicates + self loops
    return e


def main():
    R = RefLib()
    out = {}
    # ---- graph-core known answers (tests/test_graph.cpp:16-42) + a random edge list ----
    p3 = R.graph(np.array([[0, 1], [1, 2]], np.int32), 3).csr()
    out["p3_ro"], out["p3_co"] = p3
    e = small_graph()
    ro, co = R.graph(e, 120).csr()
    out["g_edges"], out["g_ro"], out["g_co"] = e, ro, co
    ro_d, co_d = R.graph(e, 120, symmetrize=False).csr()
    out["g_ro_directed"], out["g_co_directed"] = ro_d, co_d
    rg = R.graph(csr=(ro, co))
    batches = {"single": np.array([0], np.int32), "mid": np.arange(10, 40, 3, dtype=np.int32),
               "full": np.arange(120, dtype=np.int32)}
    for name, b in batches.items():
        for k, v in rg.plan(b).items():
            out[f"plan_{name}_{k}"] = v
    # ---- op known answers on random inputs ----
    rng = np.random.default_rng(1)
    pl = rg.plan(batches["mid"])
    x = rng.standard_normal((len(pl["extended_nodes"]), 9)).astype(np.float32)
    gy = rng.standard_normal((len(pl["batch_nodes"]), 9)).astype(np.float32)
    y, gx = R.aggregate(pl["gcn_row_ptr"], pl["gcn_cols"], pl["gcn_coeffs"], x, gy)
    out.update(agg_x=x, agg_gy=gy, agg_y=y, agg_gx=gx)
    a = rng.standard_normal((13, 7)).astype(np.float32)
    a[a < -1.0] = 0.0  # exercise the zero-skip of the reference matmul
    b = rng.standard_normal((7, 5)).astype(np.float32)
    gm = rng.standard_normal((13, 5)).astype(np.float32)
    y, ga, gb = R.matmul(a, b, gm)
    out.update(mm_a=a, mm_b=b, mm_gy=gm, mm_y=y, mm_ga=ga, mm_gb=gb)
    lg = rng.standard_normal((11, 6)).astype(np.float32) * 3
    rows = np.array([0, 2, 3, 7, 10], np.int32)
    labs = np.array([1, 0, 5, 2, 2], np.int32)
    loss, g = R.softmax_ce(lg, rows, labs)
    out.update(ce_logits=lg, ce_rows=rows, ce_labels=labs, ce_loss=np.float32(loss), ce_grad=g)
    p0 = rng.standard_normal(50).astype(np.float32)
    grads = rng.standard_normal((5, 50)).astype(np.float32) * 0.1
    out.update(adam_p0=p0, adam_grads=grads, adam_p5=R.adam(p0, grads))
    out["glorot_7x5_s42"] = R.glorot(7, 5, 42)
    out["order_10_s3_e4"] = R.epoch_order(10, 3, 4)
    np.savez_compressed(HERE / "ref_ops.npz", **out)

    # ---- GAS sessions: GCN / APPNP / GCNII on a small planted-community graph ----
    n, parts, F, C = 200, 4, 12, 4
    rng = np.random.default_rng(7)
    comm = rng.integers(0, parts, n).astype(np.int32)
    comm[:parts] = np.arange(parts)
    pairs = []
    for _ in range(900):
        u = int(rng.integers(0, n))
        if rng.random() < 0.7:
            cands = np.flatnonzero(comm == comm[u])
            v = int(cands[rng.integers(0, len(cands))])
        else:
            v = int(rng.integers(0, n))
        pairs.append((u, v))
    edges = np.array(pairs, np.int32)
    ro, co = R.graph(edges, n).csr()
    feats = rng.standard_normal((n, F)).astype(np.float32)
    labels = (comm % C).astype(np.int32)
    train = (rng.random(n) < 0.6).astype(np.uint8)
    train[np.flatnonzero(comm == 3)] = 0  # one batch without training rows (no optimizer step)
    sess = dict(s_edges=edges, s_ro=ro, s_co=co, s_feats=feats, s_labels=labels, s_train=train, s_comm=comm)
    for name, kind, L in [("gcn", 0, 3), ("appnp", 2, 3), ("gcnii", 3, 4)]:
        spec = make_spec(kind=kind, num_layers=L, hidden=8, seed=11, clip_max_norm=0.5 if kind == 3 else 0.0)
        s = R.session(ro, co, feats, labels, train, C, comm, parts, spec)
        sess[f"{name}_params0"] = s.get_params()
        order = R.epoch_order(parts, 11, 0)
        for i, p in enumerate(order):
            nb = int((comm == p).sum())
            acts, logits, loss, grads, stepped = s.batch(int(p), 0, nb=nb)
            sess[f"{name}_b{i}_part"] = np.int32(p)
            sess[f"{name}_b{i}_acts"] = acts
            sess[f"{name}_b{i}_logits"] = logits
            sess[f"{name}_b{i}_loss"] = np.float64(loss)
            sess[f"{name}_b{i}_grads"] = grads if grads is not None else np.zeros(0, np.float32)
            sess[f"{name}_b{i}_stepped"] = np.int32(stepped)
        sess[f"{name}_params1"] = s.get_params()
        for l in range(1, L):
            sess[f"{name}_hist{l}"] = s.get_history(l)
        sess[f"{name}_epoch1_loss"] = np.float64(s.epoch(1)[0])
        sess[f"{name}_params2"] = s.get_params()
    np.savez_compressed(HERE / "ref_sessions.npz", **sess)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
