"""One profiled GAS epoch (cudaProfilerStart/Stop around it) for ncu launch lists:
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python tools/profile_epoch.py
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit")
ap.add_argument("--epochs", type=int, default=1)
ap.add_argument("--seg-edges", type=int, default=128)
ap.add_argument("--no-hoist", action="store_true")
ap.add_argument("--no-graphs", action="store_true")
a = ap.parse_args()
ds = make_dataset(a.workload)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3),
                   gb.TrainerOptions(seg_edges=a.seg_edges, hoist_layer1=not a.no_hoist, use_graphs=not a.no_graphs))
tr.gas_epoch(0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for e in range(a.epochs):
    tr.gas_epoch(1 + e)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches/epoch", tr.launch_count())
