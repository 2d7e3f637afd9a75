import time, sys, os
sys.path.insert(0, os.getcwd())
t=time.time()
import paper_2106_05609_b200 as gb
from paper_2106_05609_b200.workloads import make_dataset
from paper_2106_05609_b200.trainer import GasTrainer, ModelSpec, TrainerOptions
ds=make_dataset("reddit"); t1=time.time(); print("dataset", t1-t, flush=True)
P=ds.workload.parts
s=gb.BatchSchedule.build(ds.graph, ds.assignment, P); t2=time.time(); print("sched host", t2-t1, flush=True)
tr=GasTrainer(s, ds.features, ds.labels, ds.train_mask, ds.workload.num_classes, ModelSpec("gcn",4,256)); t3=time.time(); print("trainer create", t3-t2, flush=True)
tr.gas_epoch(0); t4=time.time(); print("first epoch", t4-t3, flush=True)
