"""Training-dynamics probe on the GPU trainer: per-epoch mean loss for workload variants.

    python tools/dyn_probe.py reddit 10 signal=0.5,comm_per_part=4 signal=1.0,comm_per_part=8
"""
import dataclasses
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import WORKLOADS, make_dataset  # noqa: E402

name, epochs = sys.argv[1], int(sys.argv[2])
for variant in sys.argv[3:]:
    kw = {}
    for kv in variant.split(","):
        k, v = kv.split("=")
        kw[k] = type(getattr(WORKLOADS[name], k))(v) if k != "lr" else float(v)
    lr = kw.pop("lr", 0.01)
    w = dataclasses.replace(WORKLOADS[name], **kw)
    t0 = time.time()
    ds = make_dataset(w)
    sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                       gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3,
                                    opt=gb.AdamConfig(lr=lr)), gb.TrainerOptions())
    ls = [round(tr.gas_epoch(e), 4) for e in range(epochs)]
    acc = tr.evaluate()[0] if w.kind == "gcn" else float("nan")
    print(f"{variant} lr={lr}: lnC={math.log(w.num_classes):.4f} losses={ls} train_acc={acc:.3f} "
          f"({time.time() - t0:.0f}s)", flush=True)
