"""Per-batch loss trajectory of the GPU trainer (the bench configuration: hoisting, graphs,
segmented SpMM) over the first epochs of a workload, beside the reference's trajectory
(tools/ref_c3_trajectory.py output) when given.

    python tools/gpu_traj.py --out gpurun_out/gpu_traj.json [--ref profiles/r2_ref_c3_trajectory.json]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit")
ap.add_argument("--epochs", type=int, default=2)
ap.add_argument("--out", required=True)
ap.add_argument("--ref")
a = ap.parse_args()
ds = make_dataset(a.workload)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3,
                                opt=gb.AdamConfig(lr=w.lr)), gb.TrainerOptions())
out = {"workload": w.name, "impl": "B200 trainer (bench configuration)", "epochs": []}
ref = json.loads(Path(a.ref).read_text()) if a.ref else None
for e in range(a.epochs):
    order = [int(p) for p in gb.epoch_order(w.parts, 3, e)]
    losses = []
    for i, p in enumerate(order):  # one batch at a time through the epoch-range entry point
        tr.gas_epoch_range_async(e, i, i + 1)
        losses.append(float(tr.part_losses()[p]))
    rec = {"epoch": e, "order": order, "batch_loss": losses, "mean_loss": float(np.mean(losses))}
    if ref and e < len(ref["epochs"]):
        rl = np.array(ref["epochs"][e]["batch_loss"])
        rec["ref_mean_loss"] = float(rl.mean())
        rec["max_rel_diff_vs_ref"] = float(np.max(np.abs(np.array(losses) - rl) / np.abs(rl)))
    out["epochs"].append(rec)
    print(json.dumps({k: v for k, v in rec.items() if k not in ("order", "batch_loss")}), flush=True)
Path(a.out).write_text(json.dumps(out))
