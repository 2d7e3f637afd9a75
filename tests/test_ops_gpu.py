"""Message-passing and transform kernels vs the CPU oracle (restating src/tensor.cpp).

aggregate forward: bit-exact in sequential mode (seg_edges=0) and in segmented mode on
these inputs (fp64 partial combination differs from sequential fp64 only below fp32
resolution; the test tolerates a vanishing fraction of 1-ulp differences).
aggregate backward: bit-exact (fp32 multiply-then-add in the reference's scatter order).
matmul: tcgen05 3xTF32 (fp32 SIMT where a pitch is not TMA-describable) vs the reference's
fp64 accumulation -> <= 1e-5 normwise per tensor (the stated contract).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200._native import check, lib

from conftest import normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def hub_plan():
    """A batch of a power-law graph with hub rows (degree >> segment size)."""
    edges, comm = gb.synth_pairs(20000, 400_000, 20, 0.3, gamma=2.2, min_weight=1.0, max_weight=400.0, seed=3)
    g = gb.build_graph(edges, 20000)
    parts = gb.partition_parts(comm, 20)
    p = gb.make_batch_plan(g, parts[4], full=False)
    assert np.diff(p.gcn_row_ptr).max() > 1000
    return p


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# widths cover every chunk layout of the flat kernel (spmm_cpl_for): 64-column chunks up to
# 64, 128-column chunks (65, 602), 256-column chunks / 1 KB rows (200, 256, 480, 512)
@pytest.mark.parametrize("d", [16, 47, 64, 65, 200, 256, 480, 512, 602])
@pytest.mark.parametrize("seg", [0, 64])
@pytest.mark.parametrize("nonneg", [False, True])
def test_aggregate_forward(torch, oracle, hub_plan, d, seg, nonneg):
    """nonneg: post-ReLU tables take the one-IMAD widening path, signed ones the IMAD.WIDE + LOP3 path."""
    p = hub_plan
    rng = np.random.default_rng(d)
    ne, nb = len(p.extended_nodes), len(p.batch_nodes)
    x = rng.standard_normal((ne, d)).astype(np.float32)
    if nonneg:
        x = np.abs(x)
    ld = (d + 3) // 4 * 4  # source rows 16 B aligned
    xp = np.zeros((ne, ld), np.float32)
    xp[:, :d] = x
    want = oracle.aggregate(p.gcn_row_ptr, p.gcn_cols, p.gcn_coeffs, x)
    d_rp = _dev(torch, p.gcn_row_ptr.astype(np.int32))
    d_cols, d_cf, d_x = _dev(torch, p.gcn_cols), _dev(torch, p.gcn_coeffs), _dev(torch, xp)
    d_y = torch.zeros(nb, ld, device="cuda")
    check(lib.gasb_spmm_fwd(d_rp.data_ptr(), nb, d_cols.data_ptr(), d_cf.data_ptr(), d_x.data_ptr(), ne, ld, d,
                            d_y.data_ptr(), ld, seg, None))
    got = d_y.cpu().numpy()[:, :d]
    mism = int((got != want).sum())
    if seg == 0:
        assert mism == 0
    else:
        assert mism <= max(2, want.size // 100000), mism
        assert normwise(got, want) < 1e-7


@pytest.mark.parametrize("special", [False, True])
def test_aggregate_forward_zeros_and_denormals(torch, oracle, hub_plan, special):
    """Sparse (relu-like) inputs take the integer widening path; a table holding a denormal
    switches to the exact F2F path — bit-exact either way."""
    p = hub_plan
    rng = np.random.default_rng(7)
    ne, nb, d = len(p.extended_nodes), len(p.batch_nodes), 64
    x = np.maximum(rng.standard_normal((ne, d)), 0).astype(np.float32)
    x[0, 1] = -0.0
    if special:
        x[3, 5] = np.float32(1e-40)  # denormal
        x[7, 9] = -np.float32(3e-39)
    want = oracle.aggregate(p.gcn_row_ptr, p.gcn_cols, p.gcn_coeffs, x)
    d_rp = _dev(torch, p.gcn_row_ptr.astype(np.int32))
    d_cols, d_cf, d_x = _dev(torch, p.gcn_cols), _dev(torch, p.gcn_coeffs), _dev(torch, x)
    d_y = torch.zeros(nb, d, device="cuda")
    check(lib.gasb_spmm_fwd(d_rp.data_ptr(), nb, d_cols.data_ptr(), d_cf.data_ptr(), d_x.data_ptr(), ne, d, d,
                            d_y.data_ptr(), d, 0, None))
    assert np.array_equal(d_y.cpu().numpy(), want)


@pytest.mark.parametrize("d", [64, 256, 602])
def test_aggregate_forward_signed_extremes(torch, oracle, hub_plan, d):
    """Signed tables (no denormals, no inf/nan) take the signed integer widening: -0.0, the
    smallest normal of either sign, values near FLT_MAX and every sign/exponent mix must
    widen exactly (the mask 0x8FFFFFFF keeps the sign and the exponent field)."""
    p = hub_plan
    rng = np.random.default_rng(900 + d)
    ne, nb = len(p.extended_nodes), len(p.batch_nodes)
    mant = rng.uniform(1.0, 2.0, (ne, d))
    expo = rng.integers(-126, 100, (ne, d))
    sign = np.where(rng.random((ne, d)) < 0.5, -1.0, 1.0)
    x = (sign * np.ldexp(mant, expo)).astype(np.float32)
    tiny = np.finfo(np.float32).tiny
    x[0, :4] = [-0.0, tiny, -tiny, 0.0]
    x[1, :2] = [np.float32(1e30), np.float32(-1e30)]
    assert not np.any((x != 0) & (np.abs(x) < tiny))
    ld = (d + 3) // 4 * 4
    xp = np.zeros((ne, ld), np.float32)
    xp[:, :d] = x
    want = oracle.aggregate(p.gcn_row_ptr, p.gcn_cols, p.gcn_coeffs, x)
    d_rp = _dev(torch, p.gcn_row_ptr.astype(np.int32))
    d_cols, d_cf, d_x = _dev(torch, p.gcn_cols), _dev(torch, p.gcn_coeffs), _dev(torch, xp)
    d_y = torch.zeros(nb, ld, device="cuda")
    check(lib.gasb_spmm_fwd(d_rp.data_ptr(), nb, d_cols.data_ptr(), d_cf.data_ptr(), d_x.data_ptr(), ne, ld, d,
                            d_y.data_ptr(), ld, 0, None))
    got = d_y.cpu().numpy()[:, :d]
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("d", [16, 64, 256])
def test_aggregate_backward_bit_exact(torch, oracle, hub_plan, d):
    p = hub_plan
    rng = np.random.default_rng(100 + d)
    ne, nb = len(p.extended_nodes), len(p.batch_nodes)
    gy = rng.standard_normal((nb, d)).astype(np.float32)
    x = np.zeros((ne, d), np.float32)
    _, want = oracle.aggregate(p.gcn_row_ptr, p.gcn_cols, p.gcn_coeffs, x, gy)
    # transposed stencil over all V_b targets, entries in ascending dst row (stable sort)
    rows = np.repeat(np.arange(nb, dtype=np.int32), np.diff(p.gcn_row_ptr))
    order = np.argsort(p.gcn_cols, kind="stable")
    t_src, t_cf = rows[order], p.gcn_coeffs[order]
    t_rp = np.zeros(ne + 1, np.int32)
    t_rp[1:] = np.cumsum(np.bincount(p.gcn_cols, minlength=ne))
    d_gy = _dev(torch, gy)
    d_gx = torch.zeros(ne, d, device="cuda")
    d_rp, d_src, d_cf = _dev(torch, t_rp), _dev(torch, t_src), _dev(torch, t_cf)  # keep alive across the call
    check(lib.gasb_spmm_bwd(d_rp.data_ptr(), ne, d_src.data_ptr(), d_cf.data_ptr(), d_gy.data_ptr(), d, nb, d, None, 0,
                            d_gx.data_ptr(), d, None))
    assert np.array_equal(d_gx.cpu().numpy(), want)


def _padded(torch, a, ld):
    """Device copy of a with row pitch ld (16 B aligned pitches take the tensor-core path)."""
    out = torch.zeros(a.shape[0], ld, device="cuda")
    out[:, : a.shape[1]] = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return out


@pytest.mark.parametrize("pad", [False, True])
@pytest.mark.parametrize("m,k,n", [(1165, 602, 256), (1165, 256, 41), (271, 1433, 16), (37, 5, 3), (300, 64, 96),
                                   (60000, 100, 256), (60000, 256, 47)])  # last two: TALL tiles, split-K wgrad
def test_matmul_forward_backward(torch, oracle, m, k, n, pad):
    rng = np.random.default_rng(m + k + n)
    a = rng.standard_normal((m, k)).astype(np.float32)
    a[a < -1.5] = 0.0
    b = (rng.standard_normal((k, n)) * 0.1).astype(np.float32)
    gy = rng.standard_normal((m, n)).astype(np.float32)
    y, ga, gbw = oracle.matmul(a, b, gy)
    lk, ln = ((k + 3) // 4 * 4, (n + 3) // 4 * 4) if pad else (k, n)
    da, db, dg = _padded(torch, a, lk), _padded(torch, b, ln), _padded(torch, gy, ln)
    dy = torch.empty(m, ln, device="cuda")
    dga = torch.empty(m, lk, device="cuda")
    dgb = torch.empty(k, ln, device="cuda")
    check(lib.gasb_gemm(0, m, n, k, da.data_ptr(), lk, db.data_ptr(), ln, dy.data_ptr(), ln, 0.0, None))
    check(lib.gasb_gemm(1, m, k, n, dg.data_ptr(), ln, db.data_ptr(), ln, dga.data_ptr(), lk, 0.0, None))
    check(lib.gasb_gemm(2, k, n, m, da.data_ptr(), lk, dg.data_ptr(), ln, dgb.data_ptr(), ln, 0.0, None))
    torch.cuda.synchronize()
    errs = [normwise(dy.cpu().numpy()[:, :n], y), normwise(dga.cpu().numpy()[:, :k], ga),
            normwise(dgb.cpu().numpy()[:, :n], gbw)]
    print("matmul normwise errors (fwd, dgrad, wgrad):", errs)
    assert max(errs) < 1e-5, errs  # the per-tensor contract; 3xTF32 measures ~1e-6
