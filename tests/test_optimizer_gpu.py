"""AdamState::step (src/nn.cpp:20-41) and grad_clip (src/nn.cpp:47-63) as isolated device ops
against the reference compiled from its own sources, and the trainer's per-batch CUDA graphs
running past the Adam bias-correction table's initial capacity (the table must
never move under a captured graph)."""
import numpy as np
import pytest
import torch

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [dict(), dict(lr=0.003, beta1=0.8, beta2=0.99, eps=1e-6)])
def test_adam_bit_exact_vs_reference(ref, cfg):
    rng = np.random.default_rng(5)
    size, steps = 100_003, 7
    p0 = rng.standard_normal(size).astype(np.float32)
    g = (rng.standard_normal((steps, size)) * np.logspace(-9, 1, size)).astype(np.float32)
    g[:, :50] = 0.0  # zero gradients (ge = 0.0 path)
    want = ref.adam(p0, g, **{k.replace("beta", "b"): v for k, v in cfg.items()})
    p = torch.from_numpy(p0.copy()).cuda()
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    for t in range(steps):
        gb.adam_step(p, m, v, torch.from_numpy(g[t]).cuda(), t + 1, **cfg)
    got = p.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_grad_clip_vs_reference(ref):
    rng = np.random.default_rng(6)
    g0 = rng.standard_normal(300_001).astype(np.float32)
    for max_norm in (1.0, 1e4):
        want = g0.copy()
        nref = ref.lib.ref_grad_clip(want.ctypes.data, want.size, max_norm)
        gt = torch.from_numpy(g0.copy()).cuda()
        n = gb.grad_clip(gt, max_norm)
        assert abs(n - nref) <= 1e-13 * nref
        got = gt.cpu().numpy()
        # the scale float(max/norm) can differ by 1 ulp when the fp64 norm does
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-30)) <= 2.5e-7
    with pytest.raises(ValueError):
        gb.grad_clip(torch.zeros(4, device="cuda"), 0.0)


@pytest.mark.parametrize("beta2", [0.99, 0.9999999])
def test_graphs_past_bias_correction_capacity(beta2):
    """beta2 = 0.99 saturates (1 - beta2^t == 1.0 from t ~ 3.7K: the fixed-size table and the
    clamp); 0.9999999 never does within the run, so the table grows past its initial 8192
    entries and the captured graphs must be re-captured. Either way the graph replays must
    equal the eager path bit for bit after > 8192 optimizer steps."""
    ds = make_dataset("cora")
    w = ds.workload
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    spec = gb.ModelSpec(kind="gcn", num_layers=2, hidden=16, seed=3, opt=gb.AdamConfig(beta2=beta2))
    out = []
    for graphs in (True, False):
        tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec,
                           gb.TrainerOptions(use_graphs=graphs))
        for e in range(860):  # 10 batches per epoch -> 8600 steps
            tr.gas_epoch_async(e)
        tr.last_loss()
        out.append(tr.get_params())
    assert np.array_equal(out[0], out[1])
    assert np.isfinite(out[0]).all()
