"""GPU batch-plan builder (plan_dev.cu): every plan array of a
device-built schedule equals the host builder's bit for bit (the host builder is pinned
against the reference in test_loader.py / test_oracle_pin.py), including the multi-group
bitmap path and the reference's partition errors."""
import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset

pytestmark = pytest.mark.gpu

KEYS = ("batch_nodes", "extended_nodes", "halo_nodes", "is_halo", "batch_local_rows", "halo_local_rows",
        "local_row_offsets", "local_col_indices", "gcn_row_ptr", "gcn_cols", "gcn_coeffs", "sum_row_ptr",
        "sum_cols", "sum_coeffs")


def _same(host, dev, full=True):
    assert host.num_parts == dev.num_parts
    for p in range(host.num_parts):
        assert np.array_equal(host.sizes(p), dev.sizes(p)), p
        a, b = host.plan(p), dev.plan(p)
        for k in KEYS:
            x, y = getattr(a, k), getattr(b, k)
            if x is None:
                assert y is None or not full, (p, k)
                continue
            assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8)), (p, k)


def _graph_with_loops(n, m, seed):
    rng = np.random.default_rng(seed)
    e = rng.integers(0, n, size=(m, 2), dtype=np.int32)
    loops = rng.choice(n, size=n // 7, replace=False).astype(np.int32)  # stored self-loops on some rows
    e = np.concatenate([e, np.stack([loops, loops], 1)])
    return gb.build_graph(e, n)  # isolated nodes stay (degree 0 rows: only the self term)


@pytest.mark.parametrize("parts", [1, 3, 17])
def test_device_plans_equal_host_random_graph(parts):
    g = _graph_with_loops(5000, 40000, parts)
    asg = np.random.default_rng(parts).integers(0, parts, 5000).astype(np.int32)
    asg[:parts] = np.arange(parts)  # every part non-empty
    _same(gb.BatchSchedule.build(g, asg, parts, full=True), gb.BatchSchedule.build(g, asg, parts, full=True,
                                                                                  device=True))
    # without the local graph / sum stencil
    _same(gb.BatchSchedule.build(g, asg, parts), gb.BatchSchedule.build(g, asg, parts, device=True), full=False)


def test_device_plans_equal_host_multi_group(monkeypatch):
    """Bitmap budget of 3 parts' rows: the builder runs part groups [0,3), [3,6), ..."""
    n, parts = 3001, 10
    g = _graph_with_loops(n, 20000, 5)
    asg = (np.arange(n) * 7919 % parts).astype(np.int32)
    monkeypatch.setenv("GASB_PLAN_BITMAP_BYTES", str(3 * 4 * ((n + 31) // 32)))
    dev = gb.BatchSchedule.build(g, asg, parts, full=True, device=True)
    _same(gb.BatchSchedule.build(g, asg, parts, full=True), dev)


@pytest.mark.parametrize("name", ["cora", "reddit_mini"])
def test_device_plans_equal_host_workloads(name):
    ds = make_dataset(name, with_features=False)
    P = ds.workload.parts
    _same(gb.BatchSchedule.build(ds.graph, ds.assignment, P, full=True),
          gb.BatchSchedule.build(ds.graph, ds.assignment, P, full=True, device=True))


def test_device_builder_errors():
    g = _graph_with_loops(100, 400, 1)
    asg = np.zeros(100, np.int32)
    asg[5] = 4
    with pytest.raises(ValueError, match="out of range"):
        gb.BatchSchedule.build(g, asg, 3, device=True)
    asg[5] = 2  # part 1 empty
    with pytest.raises(ValueError, match="empty part"):
        gb.BatchSchedule.build(g, asg, 3, device=True)


def test_device_builder_reddit_shape():
    """C3 shape (200 parts, 115M stored edges): bit-exact with the host builder and timed."""
    ds = make_dataset("reddit", with_features=False)
    P = ds.workload.parts
    host = gb.BatchSchedule.build(ds.graph, ds.assignment, P)
    dev = gb.BatchSchedule.build(ds.graph, ds.assignment, P, device=True)
    _same(host, dev, full=False)
    d_ms, t_ms = dev.timing()
    print(f"\nplan builder C3: host {host.timing()[1]:.0f} ms, device {d_ms:.1f} ms GPU / {t_ms:.0f} ms incl. copies")
