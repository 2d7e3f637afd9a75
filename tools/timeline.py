"""Kernel timeline of a window of C3 batches (torch.profiler / CUPTI: every kernel of the
process, graph nodes included, with its stream and device timestamps).
    GASB_XBATCH=1 GASB_BG_CTAS=148 python tools/timeline.py [--batches 12] [--out gpurun_out/tl.json]
Prints per-stream busy time over the window, the window span, and the per-kernel share."""
import argparse
import collections
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit")
ap.add_argument("--batches", type=int, default=12)
ap.add_argument("--out", default="")
a = ap.parse_args()
ds = make_dataset(a.workload)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
spec = gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3, opt=gb.AdamConfig(lr=w.lr))
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec, gb.TrainerOptions())
for e in range(2):
    tr.gas_epoch(e)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.gas_epoch_range_async(2, 20, 20 + a.batches)
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type.name != "CUDA" or e.device_resource_id is None:
        continue
    evs.append({"name": e.name[:70], "stream": int(e.device_resource_id), "t0": e.time_range.start,
                "t1": e.time_range.end})
evs.sort(key=lambda x: x["t0"])
t0, t1 = evs[0]["t0"], max(x["t1"] for x in evs)
span = (t1 - t0)
busy = collections.defaultdict(float)
per = collections.defaultdict(lambda: [0, 0.0])
for x in evs:
    busy[x["stream"]] += x["t1"] - x["t0"]
    k = x["name"].split("(")[0]
    per[k][0] += 1
    per[k][1] += x["t1"] - x["t0"]
# union of kernel intervals (GPU busy with >= 1 kernel)
u, cur0, cur1 = 0.0, None, None
for x in evs:
    if cur1 is None or x["t0"] > cur1:
        if cur1 is not None:
            u += cur1 - cur0
        cur0, cur1 = x["t0"], x["t1"]
    else:
        cur1 = max(cur1, x["t1"])
u += cur1 - cur0
env = {k: v for k, v in os.environ.items() if k.startswith("GASB_")}
print(json.dumps({"env": env, "batches": a.batches, "span_us": span, "per_batch_us": span / a.batches,
                  "gpu_busy_union_us": u, "stream_busy_us": {str(k): v for k, v in busy.items()}}))
for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k[:60]:60s} {c:5d} {t / a.batches:9.1f} us/batch {t / c:8.1f} us/launch")
if a.out:
    Path(a.out).write_text(json.dumps(evs))
