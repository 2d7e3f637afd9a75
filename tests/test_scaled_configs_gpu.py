"""Down-scaled parity for the configurations too large for the CPU reference at full size
(SURVEY §8 C4 / C5): graphs from the SAME generator parameters (feature
width, classes, hidden width, model, propagation depth, intra-community fraction, degree
scale) at 50K / 200K nodes, teacher-forced batch by batch against the reference compiled
from its own sources: pushed rows, logits, loss and parameter gradients within the 1e-5
normwise contract.

- C4 products_mini: APPNP K = 3, F = 100, C = 47 (47-wide histories: the CPL-2 SpMM chunks),
  h = 256 head, 20 parts.
- C5 papers_mini: GCN L = 3, F = 128, C = 172, h = 256, 16 parts; also run through the
  sharded data-parallel placement the full C5 shape needs (histories 2 x 111M x 256 fp32 =
  227 GB do not fit one B200): bit-identical to the replicated placement and to gas_epoch.
"""
import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset
from pyoracle import make_spec

from conftest import normwise

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _teacher_forced(ref, name, nbatches):
    ds = make_dataset(name)
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    spec = gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec, gb.TrainerOptions())
    order = [int(p) for p in ref.epoch_order(w.parts, 3, 0)[:nbatches]]
    rs = ref.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                     w.parts, make_spec(kind=gb.trainer.KINDS[w.kind], num_layers=w.num_layers, hidden=w.hidden,
                                        seed=3), sample_parts=order)
    assert np.array_equal(tr.get_params(), rs.get_params())
    worst = {}
    for slot, p in enumerate(order):
        rs.set_params(tr.get_params())
        for l in range(1, w.num_layers):
            rs.set_history(l, tr.history.layer_matrix(l))
        nb = int(sched.sizes(p)[0])
        ag, lg, lossg, gg, stg = tr.batch(p)
        ao, lo, losso, go, sto = rs.batch(slot, 0, nb=nb)
        assert stg == sto
        errs = {"acts": normwise(ag, ao), "logits": normwise(lg, lo)}
        if sto:
            errs["loss"] = abs(lossg - losso) / abs(losso)
            errs["grads"] = normwise(gg, go)
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
            assert v <= TOL, (name, p, k, v)
    print(name, f"nnz={len(ds.cols)}", worst)


def test_c4_products_shape_down_scaled(ref):
    _teacher_forced(ref, "products_mini", 3)


def test_c5_papers_shape_down_scaled(ref):
    _teacher_forced(ref, "papers_mini", 2)


def test_c5_papers_shape_sharded_world1_is_gas_epoch():
    ds = make_dataset("papers_mini")
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    mk = lambda: gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,  # noqa: E731
                               gb.ModelSpec(kind="gcn", num_layers=w.num_layers, hidden=w.hidden, seed=3),
                               gb.TrainerOptions())
    a, b = mk(), mk()
    dp = gb.DataParallelTrainer(b, 0, 1, placement="sharded")
    for e in range(2):
        assert a.gas_epoch(e) == dp.gas_epoch(e)
    assert np.array_equal(a.get_params(), b.get_params())
    for l in range(1, w.num_layers):
        assert np.array_equal(a.history.layer_matrix(l), dp.history_layer(l))
