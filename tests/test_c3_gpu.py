"""Parity at the headline configuration itself (BASELINE configs[2]): the
Reddit-shaped graph (232,965 nodes, 115M stored edges), 4-layer GCN h = 256, 200 parts,
default (segmented) SpMM mode, against the reference compiled from its own sources on two
batches of the seeded epoch order, teacher-forced: the reference gets our parameters and
history tables before each batch. Pushed rows, logits, loss and parameter gradients within
the 1e-5 normwise contract."""
import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset
from pyoracle import make_spec

from conftest import normwise

pytestmark = pytest.mark.gpu
TOL = 1e-5


def test_reddit_c3_teacher_forced_batches(ref):
    ds = make_dataset("reddit")
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    spec = gb.ModelSpec(kind="gcn", num_layers=w.num_layers, hidden=w.hidden, seed=3)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec,
                       gb.TrainerOptions(use_graphs=False))
    order = [int(p) for p in ref.epoch_order(w.parts, 3, 0)[:2]]
    rs = ref.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                     w.parts, make_spec(kind=0, num_layers=w.num_layers, hidden=w.hidden, seed=3),
                     sample_parts=order)
    assert np.array_equal(tr.get_params(), rs.get_params())  # Model::build init is bit-exact
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
            assert v <= TOL, (p, k, v)
    print("C3 teacher-forced worst normwise errors:", worst)
