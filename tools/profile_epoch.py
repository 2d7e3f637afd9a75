"""One profiled C3 epoch for ncu (`--profile-from-start off`): builds the bench workload, runs
two warm-up epochs (graphs captured, tables warm), then one epoch between cudaProfilerStart
and cudaProfilerStop.

    ncu --profile-from-start off ... python tools/profile_epoch.py [workload]
"""
import ctypes
import sys
from pathlib import Path

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
cudart = ctypes.CDLL("libcudart.so")
cudart.cudaProfilerStart()
tr.gas_epoch(2)
cudart.cudaProfilerStop()
print("profiled epoch, loss", tr.last_loss())
