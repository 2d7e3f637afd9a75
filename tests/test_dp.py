"""Data-parallel step semantics on CPU.

- gas_epoch's batch order from libgasb (host code) equals the oracle's and the compiled
  reference's (trainer.cpp:395-400), and step_plan tiles it into k-batch steps.
- The exchange protocol of dp.cu (per-rank batch against start-of-step state, gradient sum
  in rank order over the stepped ranks / count, pushes committed after the step) run as
  TWO gloo processes over the C oracle reproduces the oracle's single-process
  go_session_dp_epoch bit for bit, and k = 1 reproduces gas_epoch.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset
from pyoracle import make_spec

HERE = Path(__file__).resolve().parent


def test_epoch_order_matches_oracles(oracle, ref):
    for parts, seed in [(10, 3), (200, 3), (8, 0), (1, 5)]:
        for e in range(4):
            o = gb.epoch_order(parts, seed, e)
            assert np.array_equal(o, oracle.epoch_order(parts, seed, e))
            assert np.array_equal(o, ref.epoch_order(parts, seed, e))
    assert np.array_equal(gb.epoch_order(7, 3, 0, shuffle=False), np.arange(7))


@pytest.mark.parametrize("parts,k", [(10, 2), (10, 3), (200, 8), (5, 8)])
def test_step_plan_tiles_order(parts, k):
    plan = gb.step_plan(parts, 3, 1, k)
    assert plan.shape == (-(-parts // k), k)
    flat = plan.reshape(-1)
    assert np.array_equal(flat[:parts], gb.epoch_order(parts, 3, 1))
    assert (flat[parts:] == -1).all()


def _session(oracle, ds):
    w = ds.workload
    return oracle.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes,
                          ds.assignment, w.parts, make_spec(kind=0, num_layers=w.num_layers, hidden=w.hidden, seed=3))


def test_dp_k1_is_gas_epoch(oracle):
    ds = make_dataset("cora")
    a, b = _session(oracle, ds), _session(oracle, ds)
    for e in range(2):
        la, _ = a.epoch(e)
        lb = b.dp_epoch(e, 1)
        assert la == lb
    assert np.array_equal(a.get_params(), b.get_params())
    assert np.array_equal(a.get_history(1), b.get_history(1))


def test_dp_protocol_two_gloo_ranks(oracle, tmp_path):
    """Two processes exchange gradients (all_gather, summed in rank order) and pushed rows
    (all_gather_object) over gloo; their result equals go_session_dp_epoch(k=2) exactly."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 1000), WORLD_SIZE="2")
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, str(HERE / "helpers" / "dp_oracle_rank.py"), str(tmp_path)],
                                      env=e, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    ds = make_dataset("cora")
    s = _session(oracle, ds)
    losses = [s.dp_epoch(e, 2) for e in range(2)]
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(got["params"], s.get_params()), r
        assert np.array_equal(got["hist1"], s.get_history(1)), r
        assert np.allclose(got["losses"], losses, rtol=0, atol=0), (got["losses"], losses)


@pytest.mark.parametrize("name,k", [("cora", 2), ("cora", 3), ("cora_appnp", 2)])
def test_dp_sharded_protocol_gloo_ranks(oracle, tmp_path, name, k):
    """The SHARDED placement's protocol (libgasb's shard map: each rank holds only its parts'
    history rows; halo reads of start-of-step shards; owners commit the step's rows) run as
    k gloo processes over the C oracle equals go_session_dp_epoch(k) bit for bit."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(28500 + (os.getpid() + 7 * k) % 1000),
               WORLD_SIZE=str(k))
    procs = [subprocess.Popen([sys.executable, str(HERE / "helpers" / "dp_oracle_sharded_rank.py"), str(tmp_path), name],
                              env=dict(env, RANK=str(r)), stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(k)]
    outs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    ds = make_dataset(name)
    w = ds.workload
    s = oracle.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                       w.parts, make_spec(kind=gb.trainer.KINDS[w.kind], num_layers=w.num_layers, hidden=w.hidden,
                                          seed=3))
    losses = [s.dp_epoch(e, k) for e in range(2)]
    for r in range(k):
        got = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(got["params"], s.get_params()), r
        for l in range(1, w.num_layers):
            assert np.array_equal(got[f"hist{l}"], s.get_history(l)), (r, l)
        assert np.allclose(got["losses"], losses, rtol=0, atol=0)


def test_shard_map_partitions_rows():
    ds = make_dataset("cora", with_features=False)
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, ds.workload.parts)
    owner, local, rows = gb.shard_map(sched, 3)
    assert np.array_equal(owner, ds.assignment % 3)
    for j in range(3):
        assert np.array_equal(np.sort(local[owner == j]), np.arange(rows[j]))
