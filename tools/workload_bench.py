"""Device-timed GAS epochs on any workload of workloads.py (single GPU):
    python tools/workload_bench.py products_appnp [--epochs 3] [--warmup 2]
Prints one JSON line: epoch ms, nodes/s, stored nnz, setup seconds, final loss."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--epochs", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
t0 = time.time()
ds = make_dataset(a.workload)
w = ds.workload
t1 = time.time()
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
t2 = time.time()
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3))
t3 = time.time()
for e in range(a.warmup):
    tr.gas_epoch(e)
s = torch.cuda.ExternalStream(tr.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
for e in range(a.epochs):
    tr.gas_epoch_async(a.warmup + e)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.epochs
sizes = [sched.sizes(p) for p in range(w.parts)]
print(json.dumps({"workload": w.name, "kind": w.kind, "layers": w.num_layers, "hidden": w.hidden,
                  "num_nodes": w.num_nodes, "stored_nnz": int(len(ds.cols)), "parts": w.parts,
                  "mean_batch": float(sum(int(z[0]) for z in sizes) / w.parts),
                  "mean_extended": float(sum(int(z[1]) for z in sizes) / w.parts),
                  "epoch_ms": ms, "nodes_per_s": w.num_nodes / (ms / 1000), "final_loss": tr.last_loss(),
                  "setup_s": {"graph+features": t1 - t0, "schedule (host loader)": t2 - t1, "trainer upload": t3 - t2},
                  "launches_per_epoch": tr.launch_count()}))
