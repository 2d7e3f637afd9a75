"""One rank of the SHARDED data-parallel protocol (dp.cu, GASB_DP_SHARDED) over the C oracle
and gloo. Test infrastructure for tests/test_dp.py; writes rank<r>.npz into argv[1].

Each rank keeps only the history rows it owns (libgasb's shard map: partition p -> rank
p mod k, rows in part order). Per step: halo reads = the start-of-step shards of every rank
(all_gather here, NVLink P2P loads on the GPU); the rank's batch runs against them; the
step's rows are committed only by their owners, from every rank's pushed rows."""
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

out, name = Path(sys.argv[1]), sys.argv[2]
dist.init_process_group("gloo")
rank, k = dist.get_rank(), dist.get_world_size()
ds = make_dataset(name)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
owner, local, rows = gb.shard_map(sched, k)
s = Oracle().session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment,
                     w.parts, make_spec(kind=gb.trainer.KINDS[w.kind], num_layers=w.num_layers, hidden=w.hidden,
                                        seed=3))
L = w.num_layers
shard = {l: np.zeros((int(rows[rank]), s.hist_dim), np.float32) for l in range(1, L)}
nb = np.bincount(ds.assignment, minlength=w.parts)


def assemble():
    """Every rank's shard -> the full start-of-step tables (the halo reads)."""
    got = [None] * k
    dist.all_gather_object(got, shard)
    full = {}
    for l in range(1, L):
        H = np.zeros((w.num_nodes, s.hist_dim), np.float32)
        for j in range(k):
            mine = owner == j
            H[mine] = got[j][l][local[mine]]
        full[l] = H
    return full


losses = []
for epoch in range(2):
    plan = gb.step_plan(w.parts, 3, epoch, k)
    lsum, lcnt = 0.0, 0
    for row in plan:
        for l, H in assemble().items():
            s.set_history(l, H)
        kk = int((row >= 0).sum())
        p = int(row[rank]) if rank < kk else -1
        if p >= 0:
            g, acts, loss, st = s.dp_batch(p, int(nb[p]))
        else:
            g, acts, loss, st = np.zeros(s.nparam, np.float32), None, 0.0, False
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
        for j in range(kk):  # commit: the rows this rank owns, from every rank's batch
            pj, acts_j = meta[j][0], meta[j][3]
            ids = sched.batch_nodes(pj)
            mine = owner[ids] == rank
            for l in range(1, L):
                shard[l][local[ids[mine]]] = acts_j[l - 1][mine]
        s.dp_apply(gsum, count, kk)
    losses.append(lsum / lcnt if lcnt else 0.0)
full = assemble()
np.savez(out / f"rank{rank}.npz", params=s.get_params(), losses=np.array(losses),
         **{f"hist{l}": full[l] for l in range(1, L)})
dist.destroy_process_group()
