"""Per-CTA phase timing of spmm_bwd_smem_kernel (GASB_LIB = a -DGASB_BWD_TIMING build): after one
C3 epoch, the last launch's stamps: start spread, staging time, finish spread, heaviest warp."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200._native import lib  # noqa: E402
from paper_2106_05609_b200.workloads import make_dataset  # noqa: E402

ds = make_dataset("reddit")
w = ds.workload
sched = gb.BatchSchedule.build(ds.graph, ds.assignment, w.parts)
tr = gb.GasTrainer(sched, ds.features, ds.labels, ds.train_mask, w.num_classes,
                   gb.ModelSpec(kind=w.kind, num_layers=w.num_layers, hidden=w.hidden, seed=3,
                                opt=gb.AdamConfig(lr=w.lr)), gb.TrainerOptions())
tr.gas_epoch(0)
lib.gasb_debug_bwd_stamps.argtypes = [ctypes.c_void_p]
raw = np.zeros(512 * 4, np.uint64)
lib.gasb_debug_bwd_stamps(raw.ctypes.data)
raw = raw.reshape(512, 4).astype(np.int64)
lib.gasb_debug_bwd_end.argtypes = [ctypes.c_void_p]
endv = np.zeros(512, np.uint64)
lib.gasb_debug_bwd_end(endv.ctypes.data)
endv = endv.astype(np.int64)
for name, s in (("spmm_bwd_smem (last launch)", raw[:256]), ("spmm_bwd2 (last launch)", raw[256:])):
    s = s[s[:, 0] > 0]
    if not len(s):
        continue
    t0 = s[:, 0].min()
    st = (s[:, 1] - s[:, 0]) / 1000
    en = (s[:, 2] - t0) / 1000
    print(f"{name}: {len(s)} CTAs: start spread {(s[:, 0].max() - t0) / 1000:.2f} us; first staging median {np.median(st):.2f} "
          f"max {st.max():.2f} us; end median {np.median(en):.2f} max {en.max():.2f} us")
    if name.startswith("spmm_bwd2"):
        e2 = endv[256:][raw[256:, 0] > 0]
        m = lambda v: np.round(np.median(v) / 1000, 2)  # noqa: E731
        print("   per CTA, median us after its start: phase-0 landed", m(s[:, 1] - s[:, 0]), "| phase-0 last warp done",
              m(s[:, 2] - s[:, 0]), "| phase-1 landed", m(s[:, 3] - s[:, 0]), "| end", m(e2 - s[:, 0]))
    else:
        print("   heaviest warp entries median", np.median(s[:, 3]), "max", s[:, 3].max())
try:
    lib.gasb_debug_bwd_warp.argtypes = [ctypes.c_void_p]
    wv = np.zeros(64 * 3, np.uint64)
    lib.gasb_debug_bwd_warp(wv.ctypes.data)
    wv = wv.reshape(64, 3)[:32].astype(np.int64)
    print("spmm_bwd2 CTA (0,0) phase 0 per warp (entries, targets, us):",
          [(int(a), int(b), round(c / 1000, 2)) for a, b, c in wv])
except AttributeError:
    pass
