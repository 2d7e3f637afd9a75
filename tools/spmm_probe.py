"""Times the SpMM of the training step for the current GASB_SPMM_VARIANT (env) on a workload:
per-batch layer-2 aggregation (avg over parts), the hoisted layer-1 aggregation, and whole
epochs. Prints one JSON line. Used to pick kernel variants; not part of the product."""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit")
ap.add_argument("--seg-edges", type=int, default=512)
ap.add_argument("--epochs", type=int, default=2)
a = ap.parse_args()
ds = make_dataset(a.workload)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3),
                   gb.TrainerOptions(seg_edges=a.seg_edges))
tr.gas_epoch(0)
parts = list(range(0, w.parts, max(1, w.parts // 20)))
l2 = sum(tr.profile_spmm(p, 2, 3) for p in parts) / len(parts)
l1 = tr.profile_spmm(-1, 1, 1)
torch.cuda.synchronize()
t = time.perf_counter()
for e in range(a.epochs):
    tr.gas_epoch(1 + e)
ep = (time.perf_counter() - t) / a.epochs
print(json.dumps({"variant": os.environ.get("GASB_SPMM_VARIANT", "default"), "seg": a.seg_edges, "l2_ms": l2,
                  "hoisted_l1_ms": l1, "epoch_ms": 1000 * ep, "loss": tr.last_loss()}))
