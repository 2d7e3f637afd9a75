"""Per-batch loss trajectory of the REFERENCE (oracle/_ref: its own sources compiled in place)
over the first epochs of the C3 workload, for comparison with the GPU trainer's trajectory
(does the reference also collapse?). Test/measurement tooling only.

    python tools/ref_c3_trajectory.py [--workload reddit] [--epochs 2] --out profiles/r2_ref_c3_trajectory.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import importlib.util

spec = importlib.util.spec_from_file_location("wl", ROOT / "paper_2106_05609_b200" / "workloads.py")
wl = importlib.util.module_from_spec(spec)
sys.modules["wl"] = wl
spec.loader.exec_module(wl)
from pyoracle import OracleSynth, RefLib, make_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit")
ap.add_argument("--epochs", type=int, default=2)
ap.add_argument("--out", required=True)
a = ap.parse_args()
ds = wl.make_dataset(a.workload, backend=OracleSynth())
w = ds.workload
R = RefLib()
order0 = [int(p) for p in R.epoch_order(w.parts, 3, 0)]
slot_of = {p: i for i, p in enumerate(order0)}
kinds = {"gcn": 0, "appnp": 2, "gcnii": 3}
s = R.session(ds.row_offsets, ds.cols, ds.features, ds.labels, ds.train_mask, w.num_classes, ds.assignment, w.parts,
              make_spec(kind=kinds[w.kind], num_layers=w.num_layers, hidden=w.hidden, seed=3, lr=w.lr), sample_parts=order0)
out = {"workload": w.name, "impl": "reference (oracle/_ref, 1 thread)", "epochs": []}
t0 = time.time()
for e in range(a.epochs):
    order = [int(p) for p in R.epoch_order(w.parts, 3, e)]
    losses, secs = [], 0.0
    for p in order:
        l, dt = s.run(slot_of[p], e)
        losses.append(l)
        secs += dt
    out["epochs"].append({"epoch": e, "order": order, "batch_loss": losses, "seconds": secs})
    print(f"epoch {e}: mean loss {sum(losses) / len(losses):.6f}  ({secs:.0f} s)", flush=True)
    Path(a.out).write_text(json.dumps(out))
