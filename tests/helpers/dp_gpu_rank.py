"""One rank of the data-parallel trainer (libgasb dp.cu) for tests/test_dp_gpu.py.

argv: out_dir workload world epochs [hoist|-] [replicated|sharded]. Every rank uses cuda:0 when only one GPU is visible
(two processes share it: the IPC exchange and the barriers work the same within one GPU),
else cuda:LOCAL_RANK. gloo is the control plane (IPC handle all-gather, loss sum)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

out, name, world, epochs = Path(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
dist.init_process_group("gloo")
rank = dist.get_rank()
dev = rank if torch.cuda.device_count() >= world else 0
torch.cuda.set_device(dev)
ds = make_dataset(name)
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
spec = gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes, spec,
                   gb.TrainerOptions(device=dev, hoist_layer1=len(sys.argv) > 5 and sys.argv[5] == "hoist"))
placement = sys.argv[6] if len(sys.argv) > 6 else "replicated"
dp = gb.DataParallelTrainer(tr, rank, world, group=dist.group.WORLD, placement=placement)
losses = [dp.gas_epoch(e) for e in range(epochs)]
hist = {f"hist{l}": dp.history_layer(l) for l in range(1, w.num_layers)}
tf = dp.traffic()
np.savez(out / f"rank{rank}.npz", params=tr.get_params(), losses=np.array(losses),
         step=np.array([tr.history.step()]), launches=np.array([dp.launch_count()]),
         traffic=np.array([tf["nvlink_bytes"], tf["local_pull_bytes"], tf["shard_rows"]]), **hist)
dist.barrier()
del dp
dist.destroy_process_group()
