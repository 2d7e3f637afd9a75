"""SpMM engine probe at C3: per-batch layer-2 SpMM (avg over 20 parts), hoisted layer 1, one
epoch, and a parameter checksum after 2 epochs. Engine / tuning via environment variables:

    GASB_SPMM_ENGINE=reg GASB_REG_CPL=4 GASB_SPMM_RANGES_PER_SM=24 python tools/spmm_probe.py
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
ds = make_dataset(name)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3,
                                opt=gb.AdamConfig(lr=w.lr)), gb.TrainerOptions())
for e in range(2):
    tr.gas_epoch(e)
ck = float(np.abs(tr.get_params()).astype(np.float64).sum())
parts = list(range(0, w.parts, max(1, w.parts // 20)))
per = [tr.profile_spmm(p, 2, 5) for p in parts]
hoist = tr.profile_spmm(-1, 1, 3) if w.kind == "gcn" else float("nan")
import torch  # noqa: E402
s = torch.cuda.ExternalStream(tr.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for e in range(3):
    tr.gas_epoch_async(2 + e)
e1.record(s)
torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("GASB_")}
print(json.dumps({"env": env, "batch_spmm_us": 1000 * float(np.mean(per)), "hoisted_ms": hoist,
                  "epoch_ms": e0.elapsed_time(e1) / 3, "checksum": ck, "loss": tr.last_loss()}))
