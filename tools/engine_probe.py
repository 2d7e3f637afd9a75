"""SpMM engine comparison on the Reddit shape (GASB_SPMM_ENGINE read from the env):
per-batch layer-2 SpMM (d = 256) and hoisted layer-1 (d = 602) times, epoch time, and a
hash of the parameters after 2 epochs (engines must agree bit for bit)."""
import hashlib
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
ds = make_dataset(name)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3), gb.TrainerOptions())
tr.gas_epoch(0)
parts = list(range(0, w.parts, max(1, w.parts // 20)))
t2 = sum(tr.profile_spmm(p, 2, 5) for p in parts) / len(parts)
t1 = sum(tr.profile_spmm(p, 1, 3) for p in parts[:5]) / len(parts[:5])
th = tr.profile_spmm(-1, 1, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
tr.gas_epoch(1)
ep = time.perf_counter() - t0
h = hashlib.sha1(tr.get_params().tobytes()).hexdigest()[:12]
print(f"engine={os.environ.get('GASB_SPMM_ENGINE', 'default')} L2 per-batch {1000 * t2:.1f} us  "
      f"L1 per-batch {1000 * t1:.1f} us  hoisted L1 {th:.2f} ms  epoch {1000 * ep:.1f} ms  params {h}")
