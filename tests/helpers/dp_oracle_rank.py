"""One rank of the data-parallel exchange protocol (dp.cu) over the C oracle and gloo.
Test infrastructure for tests/test_dp.py; writes rank<r>.npz into argv[1]."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402
from pyoracle import Oracle, make_spec  # noqa: E402

out = Path(sys.argv[1])
dist.init_process_group("gloo")
rank, k = dist.get_rank(), dist.get_world_size()
ds = make_dataset("cora")
w = ds.workload
s = Oracle().session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                     w.parts, make_spec(kind=0, num_layers=w.num_layers, hidden=w.hidden, seed=3))
nb = np.bincount(ds.assignment, minlength=w.parts)
losses = []
for epoch in range(2):
    plan = gb.step_plan(w.parts, 3, epoch, k)
    lsum, lcnt = 0.0, 0
    for row in plan:
        kk = int((row >= 0).sum())
        p = int(row[rank]) if rank < kk else -1
        if p >= 0:
            g, acts, loss, st = s.dp_batch(p, int(nb[p]))
        else:
            g, acts, loss, st = np.zeros(s.nparam, np.float32), None, 0.0, False
        # gradient exchange: gather every rank's slot, sum in rank order over the stepped ones
        slots = [torch.zeros(s.nparam) for _ in range(k)]
        dist.all_gather(slots, torch.from_numpy(g))
        meta = [None] * k
        dist.all_gather_object(meta, (p, bool(st), float(loss), acts))
        gsum = np.zeros(s.nparam, np.float32)
        count = 0
        for j in range(kk):
            if meta[j][1]:
                gsum += slots[j].numpy()
                count += 1
                lsum += meta[j][2]
                lcnt += 1
        for j in range(kk):  # commit every rank's pushed rows (disjoint batches)
            s.dp_commit(meta[j][0], meta[j][3])
        s.dp_apply(gsum, count, kk)
    losses.append(lsum / lcnt if lcnt else 0.0)
np.savez(out / f"rank{rank}.npz", params=s.get_params(), hist1=s.get_history(1), losses=np.array(losses))
dist.destroy_process_group()
