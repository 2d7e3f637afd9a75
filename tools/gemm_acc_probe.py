"""tcgen05 GEMM accuracy (normwise vs fp64) and device time per launch for the C3 batch shapes;
run once per GASB_GEMM_* setting (they are read once per process)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402,F401
from paper_2106_05609_b200._native import check, lib  # noqa: E402

out = {"env": {k: v for k, v in os.environ.items() if k.startswith("GASB_GEMM")}}
g = torch.Generator(device="cpu").manual_seed(0)
for (M, N, K) in ((1165, 256, 256), (1165, 256, 602), (1165, 41, 256)):
    a = torch.rand(M, K, generator=g) * 2 - 1
    b = torch.rand(K, N, generator=g) * 2 - 1
    ref = a.double() @ b.double()
    ad, bd = a.cuda(), b.cuda()
    c = torch.empty(M, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    call = lambda: check(lib.gasb_gemm(0, M, N, K, ad.data_ptr(), K, bd.data_ptr(), N, c.data_ptr(), N, 0.0, st))  # noqa: E731
    for _ in range(5):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        call()
    e1.record()
    torch.cuda.synchronize()
    err = float(torch.linalg.norm(c.cpu().double() - ref) / torch.linalg.norm(ref))
    out[f"{M}x{N}x{K}"] = {"us": e0.elapsed_time(e1) * 1000 / 200, "normwise": err}
print(json.dumps(out))
