"""In-kernel phase timing of the tcgen05 GEMM (GASB_LIB = a -DGASB_GEMM_TIMING build): globaltimer
stamps of CTA (0,0,0): start, setup done (barriers, TMEM), first stage landed, mainloop done
(accumulator ready), epilogue done."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200._native import check, lib  # noqa: E402

lib.gasb_debug_gemm_stamps.argtypes = [ctypes.c_void_p]
M, N = 1165, 256
for K in (32, 256, 602):
    a = torch.randn(M, (K + 3) // 4 * 4, device="cuda")
    b = torch.randn(K, N, device="cuda")
    c = torch.empty(M, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for rep in range(4):
        check(lib.gasb_gemm(0, M, N, K, a.data_ptr(), a.stride(0), b.data_ptr(), N, c.data_ptr(), N, 0.0, st))
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    check(lib.gasb_gemm(0, M, N, K, a.data_ptr(), a.stride(0), b.data_ptr(), N, c.data_ptr(), N, 0.0, st))
    e1.record()
    torch.cuda.synchronize()
    s = np.zeros(40 + 2 * 256, np.uint64)
    lib.gasb_debug_gemm_stamps(s.ctypes.data)
    t0 = int(s[0])
    rel = lambda i: (int(s[i]) - t0) / 1000.0  # noqa: E731
    nk = min(8, (K + 31) // 32)
    print("  k-block: tma issue / stage landed / split done (us from start):",
          [(round(rel(24 + k), 2), round(rel(8 + k), 2), round(rel(16 + k), 2)) for k in range(nk)])
    nct = ((M + 127) // 128) * ((N + 63) // 64)
    cs = s[40:40 + 2 * nct].astype(np.int64).reshape(nct, 2)
    print(f"  {nct} CTAs: start spread {(cs[:, 0].max() - cs[:, 0].min()) / 1000:.2f} us, first start -> last end "
          f"{(cs[:, 1].max() - cs[:, 0].min()) / 1000:.2f} us, CTA durations {np.median(cs[:, 1] - cs[:, 0]) / 1000:.2f} "
          f"median / {(cs[:, 1] - cs[:, 0]).max() / 1000:.2f} max; event-timed launch {e0.elapsed_time(e1) * 1000:.2f} us")
    d = np.diff(s[:5].astype(np.int64)) / 1000.0
    print(f"K {K}: setup {d[0]:.2f} us, first stage {d[1]:.2f} us, mainloop {d[2]:.2f} us, epilogue {d[3]:.2f} us, "
          f"total {sum(d):.2f} us", flush=True)
x = torch.zeros(1024, device="cuda")
for _ in range(3):
    x.add_(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
x.add_(1)
e1.record()
torch.cuda.synchronize()
print(f"event-timed trivial kernel: {e0.elapsed_time(e1) * 1000:.2f} us")
