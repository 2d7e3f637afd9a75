"""Dropout (tensor.cpp:374-401; applied to every layer input, trainer.cpp:181-184, 203-204).

- dropout_rng = "exact": the keep masks are the reference's own stream (Rng(derive_seed(seed ^
  "drop", epoch, part, layer)).next_double() >= p, element by element): the masks equal the
  reference's, and teacher-forced batches match the compiled reference within the 1e-5
  contract (forward with dropped inputs, backward through the masks).
- dropout_rng = "philox": device Philox4x32-10 masks keyed by the same derive_seed value —
  a different stream, so only statistical: keep rate 1 - p, independent of position,
  deterministic per (epoch, part, layer) and different across them.
"""
import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset
from pyoracle import make_spec

from conftest import normwise

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _setup(ref, p=0.5, rng="exact", hidden=64, name="cora"):
    ds = make_dataset(name)
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    spec = gb.ModelSpec(kind="gcn", num_layers=w.num_layers if name != "cora" else 3, hidden=hidden, seed=3,
                        dropout=p)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec,
                       gb.TrainerOptions(dropout_rng=rng))
    rs = None
    if ref is not None:
        rs = ref.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes,
                         ds.assignment, w.parts, make_spec(kind=0, num_layers=spec.num_layers, hidden=hidden, seed=3,
                                                           dropout=p))
    return ds, sched, tr, rs


@pytest.mark.parametrize("p", [0.5, 0.1])
def test_exact_dropout_teacher_forced_vs_reference(ref, p):
    ds, sched, tr, rs = _setup(ref, p)
    w = ds.workload
    worst = {}
    for epoch in (0, 1):
        for part in [int(x) for x in ref.epoch_order(w.parts, 3, epoch)[:5]]:
            rs.set_params(tr.get_params())
            for l in range(1, 3):
                rs.set_history(l, tr.history.layer_matrix(l))
            nb = int(sched.sizes(part)[0])
            ag, lg, lossg, gg, stg = tr.batch(part, epoch=epoch)
            ao, lo, losso, go, sto = rs.batch(part, epoch, nb=nb)
            assert stg == sto
            errs = {"acts": normwise(ag, ao), "logits": normwise(lg, lo)}
            if sto:
                errs["loss"] = abs(lossg - losso) / abs(losso)
                errs["grads"] = normwise(gg, go)
            for k, v in errs.items():
                worst[k] = max(worst.get(k, 0.0), v)
                assert v <= TOL, (epoch, part, k, v)
    print("dropout", p, worst)


def test_exact_dropout_free_running_epoch_vs_reference(ref):
    ds, sched, tr, rs = _setup(ref, 0.3)
    for e in range(2):
        lg = tr.gas_epoch(e)
        lo, _ = rs.epoch(e)
        assert abs(lg - lo) / abs(lo) <= 1e-4, (e, lg, lo)
    assert normwise(tr.get_params(), rs.get_params()) <= 2e-3


def test_exact_graphs_equal_eager():
    """Per-batch graphs replay the mask buffer the host refilled before each batch."""
    out = []
    for graphs in (True, False):
        ds = make_dataset("cora")
        w = ds.workload
        sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
        tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                           gb.ModelSpec(kind="gcn", num_layers=3, hidden=64, seed=3, dropout=0.4),
                           gb.TrainerOptions(use_graphs=graphs))
        for e in range(3):
            tr.gas_epoch(e)
        out.append(tr.get_params())
    assert np.array_equal(out[0], out[1])


def test_philox_masks_statistics():
    ds, sched, tr, _ = _setup(None, 0.3, rng="philox")
    m = tr.dropout_mask(2, 5, 1)
    keep = m.mean()
    n = m.size
    assert abs(keep - 0.7) < 5 * np.sqrt(0.21 / n), keep
    assert abs(m[:, : m.shape[1] // 2].mean() - m[:, m.shape[1] // 2:].mean()) < 0.01  # no column bias
    assert np.array_equal(m, tr.dropout_mask(2, 5, 1))  # deterministic
    assert not np.array_equal(m, tr.dropout_mask(2, 6, 1))  # per epoch
    m2 = tr.dropout_mask(2, 5, 2)  # per layer: agreement of two independent streams ~ 0.58
    k = min(m.size, m2.size)
    assert abs((m.reshape(-1)[:k] == m2.reshape(-1)[:k]).mean() - 0.58) < 0.02
    # lag-1 correlation of consecutive draws ~ 0
    f = m.reshape(-1).astype(np.float64) - keep
    assert abs(np.mean(f[1:] * f[:-1])) / 0.21 < 0.01
    losses = [tr.gas_epoch(e) for e in range(3)]
    assert np.isfinite(losses).all()


def test_exact_mask_keep_rate():
    ds, sched, tr, _ = _setup(None, 0.25)
    m = tr.dropout_mask(0, 0, 1)
    assert abs(m.mean() - 0.75) < 5 * np.sqrt(0.1875 / m.size)


@pytest.mark.parametrize("name", ["cora_appnp", "cora_gcnii"])
def test_exact_dropout_residual_teacher_forced_vs_reference(ref, name):
    """APPNP / GCNII sites too: the head input (slot 100), APPNP's head hidden (101), every
    layer input (slot l; layer 1 = dropout(h0) while h0 itself feeds the mixing) and the GCNII
    output head (9000), forward and backward (trainer.cpp:142-163, 203-204, 221-227)."""
    ds = make_dataset(name)
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    spec = gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3, dropout=0.3)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec, gb.TrainerOptions())
    rs = ref.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                     w.parts, make_spec(kind=gb.trainer.KINDS[w.kind], num_layers=w.num_layers, hidden=w.hidden,
                                        seed=3, dropout=0.3))
    worst = {}
    for epoch in (0, 1):
        for part in [int(x) for x in ref.epoch_order(w.parts, 3, epoch)[:4]]:
            rs.set_params(tr.get_params())
            for l in range(1, w.num_layers):
                rs.set_history(l, tr.history.layer_matrix(l))
            nb = int(sched.sizes(part)[0])
            ag, lg, lossg, gg, stg = tr.batch(part, epoch=epoch)
            ao, lo, losso, go, sto = rs.batch(part, epoch, nb=nb)
            assert stg == sto
            errs = {"acts": normwise(ag, ao), "logits": normwise(lg, lo)}
            if sto:
                errs["loss"] = abs(lossg - losso) / abs(losso)
                errs["grads"] = normwise(gg, go)
            for k, v in errs.items():
                worst[k] = max(worst.get(k, 0.0), v)
                assert v <= TOL, (name, epoch, part, k, v)
    print(name, "dropout 0.3", worst)


@pytest.mark.parametrize("name", ["cora_appnp", "cora_gcnii"])
def test_residual_dropout_graphs_equal_eager(name):
    out = []
    for graphs in (True, False):
        ds = make_dataset(name)
        w = ds.workload
        sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
        tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                           gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3, dropout=0.2),
                           gb.TrainerOptions(use_graphs=graphs, dropout_rng="philox"))
        for e in range(2):
            tr.gas_epoch(e)
        out.append(tr.get_params())
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("name,placement", [("cora", "replicated"), ("cora", "sharded"), ("cora_appnp", "replicated")])
def test_dropout_data_parallel_world1_is_gas_epoch(name, placement):
    """A data-parallel step draws its batch's masks like gas_epoch (epoch, partition id)."""
    ds = make_dataset(name)
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    mk = lambda: gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,  # noqa: E731
                               gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3,
                                            dropout=0.3), gb.TrainerOptions())
    a, b = mk(), mk()
    dp = gb.DataParallelTrainer(b, 0, 1, placement=placement)
    for e in range(2):
        assert a.gas_epoch(e) == dp.gas_epoch(e)
    assert np.array_equal(a.get_params(), b.get_params())
