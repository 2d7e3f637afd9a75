"""Cross-batch concurrent execution at C3: device-timed epochs per (cross_batch, bg grid cap),
each against a fresh trainer from the same dataset/schedule; final loss and parameters
compared with the cross_batch = 0 run (same epochs).
    python tools/xbatch_probe.py [--epochs 3] [--warmup 3] [--configs 0:0,1:148,2:148,...]"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit")
ap.add_argument("--epochs", type=int, default=3)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--configs", default="0:0,1:148,1:296,2:148,2:296,1:0")
a = ap.parse_args()
ds = make_dataset(a.workload)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
spec = gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3, opt=gb.AdamConfig(lr=w.lr))
base = None
for cfg in a.configs.split(","):
    xm, cap = (int(v) for v in cfg.split(":"))
    os.environ["GASB_BG_CTAS"] = str(cap)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec,
                       gb.TrainerOptions(cross_batch=xm))
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
    params = tr.get_params()
    rec = {"cross_batch": xm, "bg_ctas": cap, "epoch_ms": round(ms, 3), "final_loss": tr.last_loss(),
           "launches": tr.launch_count()}
    if base is None:
        base = params
    else:
        rec["params_vs_first"] = float(np.linalg.norm(params.astype(np.float64) - base) / np.linalg.norm(base))
    print(json.dumps(rec), flush=True)
    del tr
