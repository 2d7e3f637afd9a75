"""Layer-level ABI (gasb_layer_fwd / gasb_layer_bwd): Layer::forward and its tape backward
(src/layers.cpp:120-168, tensor.cpp aggregate/matmul/scale/add/select_rows backward) over one
batch plan, against the C restatement's aggregate / matmul (pinned to the reference) and
float32 numpy for the mixing (one rounding per scale / add, as the reference)."""
import numpy as np
import pytest
import torch

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset

from conftest import normwise

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def cora():
    ds = make_dataset("cora", with_features=False)
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, ds.workload.parts)
    return ds, sched


def _t(a):
    """Device copy with a 16 B row pitch (the SpMM / TMA contract), as a strided view."""
    a = np.asarray(a, np.float32)
    t = torch.zeros(a.shape[0], (a.shape[1] + 3) // 4 * 4, device="cuda")
    t[:, :a.shape[1]] = torch.from_numpy(np.ascontiguousarray(a))
    return t[:, :a.shape[1]]


def _z(r, c):
    return _t(np.zeros((r, c), np.float32))


@pytest.mark.parametrize("kind,din,dout", [("gcn", 96, 40), ("gcn", 256, 256), ("appnp", 47, 47), ("gcnii", 64, 64)])
def test_layer_forward_backward(oracle, cora, kind, din, dout):
    ds, sched = cora
    p = 3
    plan = sched.plan(p)
    ops = gb.BatchOps(sched, p, max_dim=max(din, dout))
    nb, ne = ops.num_batch, ops.num_extended
    assert (nb, ne) == (len(plan.batch_nodes), len(plan.extended_nodes))
    rng = np.random.default_rng(11)
    h = rng.standard_normal((ne, din)).astype(np.float32)
    h0 = rng.standard_normal((ne, dout)).astype(np.float32)
    w = (rng.standard_normal((din, dout)) * 0.1).astype(np.float32)
    gy = rng.standard_normal((nb, dout)).astype(np.float32)
    cfg = gb.LayerConfig(kind, din, dout, alpha=0.1, beta=0.5)
    rp, cols, cf = plan.gcn_row_ptr, plan.gcn_cols, plan.gcn_coeffs
    brow = plan.batch_local_rows
    a, b = np.float32(cfg.alpha), np.float32(1.0) - np.float32(cfg.alpha)
    # ---- reference forward / backward ----
    prop = oracle.aggregate(rp, cols, cf, h)
    gw_ref = gh0_ref = None
    gh0_ref = np.zeros_like(h0)
    if kind == "gcn":
        y_ref, ga, gw_ref = oracle.matmul(prop, w, gy)
        _, gx_ref = oracle.aggregate(rp, cols, cf, h, ga)
    else:
        mixed = a * h0[brow] + b * prop
        if kind == "appnp":
            y_ref, dmix = mixed, gy
        else:
            bt = np.float32(cfg.beta)
            wt = (np.float32(1.0) - bt) * np.eye(din, dtype=np.float32) + bt * w
            y_ref, dmix, gwt = oracle.matmul(mixed, wt, gy)
            gw_ref = bt * gwt
        gh0_ref[brow] += a * dmix
        _, gx_ref = oracle.aggregate(rp, cols, cf, h, b * dmix)
    # ---- device ----
    H, H0, W, GY = _t(h), _t(h0), _t(w), _t(gy)
    out = _z(nb, dout)
    saved = _z(nb, din)
    gb.layer_forward(ops, cfg, H, out, saved, h0=H0 if kind != "gcn" else None, w=W if kind != "appnp" else None)
    ghin = _z(ne, din)
    gh0 = _z(ne, dout)
    gw = _z(din, dout)
    scratch = _z(nb, max(din, dout))
    gb.layer_backward(ops, cfg, GY, saved, scratch, w=W if kind != "appnp" else None, gh_in=ghin,
                      gh0=gh0 if kind != "gcn" else None, gw=gw if kind != "appnp" else None)
    torch.cuda.synchronize()
    assert normwise(out.cpu().numpy(), y_ref) <= TOL
    assert normwise(ghin.cpu().numpy(), gx_ref) <= TOL
    if kind != "gcn":
        assert normwise(gh0.cpu().numpy(), gh0_ref) <= TOL
    if gw_ref is not None:
        assert normwise(gw.cpu().numpy(), gw_ref) <= TOL
    # the backward accumulates (the reference's grads add into existing .grad buffers)
    gb.layer_backward(ops, cfg, GY, saved, scratch, w=W if kind != "appnp" else None, gh_in=ghin)
    torch.cuda.synchronize()
    assert normwise(ghin.cpu().numpy(), 2 * gx_ref) <= TOL


def test_layer_errors(cora):
    ds, sched = cora
    ops = gb.BatchOps(sched, 0, max_dim=64)
    x = torch.zeros(ops.num_extended, 64, device="cuda")
    o = torch.zeros(ops.num_batch, 64, device="cuda")
    with pytest.raises(ValueError, match="APPNP: missing h0"):
        gb.layer_forward(ops, gb.LayerConfig("appnp", 64, 64), x, o, o)
    with pytest.raises(ValueError, match="max_dim"):
        gb.layer_forward(ops, gb.LayerConfig("gcn", 128, 64), x, o, o, w=x)
