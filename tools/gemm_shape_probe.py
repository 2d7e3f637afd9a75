"""Per-launch time of the tcgen05 GEMM (standalone gasb_gemm, op 0) vs K at the C3 batch shape
(M = 1165, N = 256): intercept = fixed cost (launch, prologue, epilogue), slope = per k-block."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2106_05609_b200 as gb  # noqa: E402
from paper_2106_05609_b200._native import check, lib  # noqa: E402

M, N = 1165, 256
s = torch.cuda.current_stream()
for op in (0, 1):
    for K in (32, 64, 128, 256, 512, 1024):
        a = torch.randn(M, K, device="cuda")
        b = torch.randn(K, N, device="cuda") if op == 0 else torch.randn(N, K, device="cuda")
        c = torch.empty(M, N, device="cuda")
        for _ in range(3):
            check(lib.gasb_gemm(op, M, N, K, a.data_ptr(), K, b.data_ptr(), b.stride(0), c.data_ptr(), N, 0.0,
                                s.cuda_stream))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                check(lib.gasb_gemm(op, M, N, K, a.data_ptr(), K, b.data_ptr(), b.stride(0), c.data_ptr(), N, 0.0,
                                    torch.cuda.current_stream().cuda_stream))
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"op {op} M {M} N {N} K {K:5d}: {1000 * e0.elapsed_time(e1) / 100:7.2f} us per GEMM", flush=True)
