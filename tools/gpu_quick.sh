python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 python -m pytest tests/test_trainer_gpu.py tests/test_history_gpu.py -x -q 2>&1 | tail -3
cat > /tmp/pf.py <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset
ds = make_dataset("reddit"); w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
for opt in (dict(), dict(fused=False, hoist_layer1=False), dict(fused=False, hoist_layer1=False, prefetch=True)):
    tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, gb.ModelSpec(kind="gcn", num_layers=4, hidden=256, seed=3), gb.TrainerOptions(**opt))
    tr.gas_epoch(0); tr.gas_epoch(1)
    torch.cuda.synchronize(); t = time.perf_counter()
    for e in range(3): tr.gas_epoch(2 + e)
    print(opt, "epoch ms %.1f" % (1000 * (time.perf_counter() - t) / 3), flush=True)
    del tr
PY
timeout 900 python /tmp/pf.py
