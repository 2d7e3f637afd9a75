"""max / mean aggregation kernels (csrc/aggregators.cu) against their definitions
(oracle/aggregators.py) — bit-exact: max and its argmax are order-exact by definition, the
max backward adds in ascending row order, the mean sums in fp64 CSR order then divides.
The reference has no max / mean aggregate (only weighted sums), so these are
definition-pinned; the mean backward is the weighted-sum backward (bit-exact with the
reference's scatter) over gasb_mean_coefficients."""
import numpy as np
import pytest

import paper_2106_05609_b200 as gb
from paper_2106_05609_b200._native import check, lib
from aggregators import max_bwd, max_fwd, mean_coefficients, mean_fwd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _plan(n=3000, pairs=40_000, part=2):
    edges, comm = gb.synth_pairs(n, pairs, 8, 0.3, gamma=2.2, min_weight=1.0, max_weight=200.0, seed=5)
    g = gb.build_graph(edges, n)
    parts = gb.partition_parts(comm, 8)
    return gb.make_batch_plan(g, parts[part], full=False)


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _stencil(p):
    rp = np.asarray(p.gcn_row_ptr, np.int64).astype(np.int32)
    cols = np.asarray(p.gcn_cols, np.int32)
    return rp, cols


@pytest.mark.parametrize("d", [1, 31, 47, 64, 256])
@pytest.mark.parametrize("ties", [False, True])
def test_max_forward_backward_exact(torch, d, ties):
    p = _plan()
    rp, cols = _stencil(p)
    ne, nb = len(p.extended_nodes), len(p.batch_nodes)
    rng = np.random.default_rng(d)
    x = rng.standard_normal((ne, d)).astype(np.float32)
    if ties:  # few distinct values: many ties, first occurrence must win
        x = np.round(x).astype(np.float32)
    ld = d + 3  # odd pitches are fine: scalar column loads
    xp = np.zeros((ne, ld), np.float32)
    xp[:, :d] = x
    d_rp, d_cols, d_x = _dev(torch, rp), _dev(torch, cols), _dev(torch, xp)
    d_y = torch.full((nb, ld), 7.0, device="cuda")
    d_arg = torch.full((nb, ld), -7, dtype=torch.int32, device="cuda")
    check(lib.gasb_spmm_max_fwd(d_rp.data_ptr(), nb, d_cols.data_ptr(), d_x.data_ptr(), ne, ld, d, d_y.data_ptr(),
                                ld, d_arg.data_ptr(), ld, None))
    torch.cuda.synchronize()
    yo, ao = max_fwd(rp, cols, x)
    assert np.array_equal(d_y.cpu().numpy()[:, :d], yo)
    assert np.array_equal(d_arg.cpu().numpy()[:, :d], ao)
    gy = rng.standard_normal((nb, d)).astype(np.float32)
    d_gy = _dev(torch, gy)
    d_gx = torch.full((ne, d), 3.0, device="cuda")
    check(lib.gasb_spmm_max_bwd(d_rp.data_ptr(), nb, d_cols.data_ptr(), d_arg.data_ptr(), ld, d_gy.data_ptr(), d,
                                ne, d, d_gx.data_ptr(), d, None))
    torch.cuda.synchronize()
    assert np.array_equal(d_gx.cpu().numpy(), max_bwd(rp, cols, ao, gy, ne))


def test_max_empty_rows_and_nan_first(torch):
    rp = np.array([0, 0, 2, 2, 3], np.int32)  # rows 0 and 2 empty
    cols = np.array([1, 0, 1], np.int32)
    x = np.array([[np.nan, 2.0], [1.0, np.nan]], np.float32)
    d_y = torch.zeros((4, 2), device="cuda")
    d_arg = torch.zeros((4, 2), dtype=torch.int32, device="cuda")
    d_rp, d_cols, d_x = _dev(torch, rp), _dev(torch, cols), _dev(torch, x)  # (held: the call reads them)
    check(lib.gasb_spmm_max_fwd(d_rp.data_ptr(), 4, d_cols.data_ptr(), d_x.data_ptr(), 2, 2, 2, d_y.data_ptr(), 2,
                                d_arg.data_ptr(), 2, None))
    torch.cuda.synchronize()
    yo, ao = max_fwd(rp, cols, x)
    y = d_y.cpu().numpy()
    assert np.array_equal(np.isnan(y), np.isnan(yo)) and np.array_equal(np.nan_to_num(y), np.nan_to_num(yo))
    assert np.array_equal(d_arg.cpu().numpy(), ao)


def test_max_range_check(torch):
    rp = np.array([0, 1], np.int32)
    cols = np.array([5], np.int32)
    x = np.zeros((2, 4), np.float32)
    d_y = torch.zeros((1, 4), device="cuda")
    d_rp, d_cols, d_x = _dev(torch, rp), _dev(torch, cols), _dev(torch, x)
    st = lib.gasb_spmm_max_fwd(d_rp.data_ptr(), 1, d_cols.data_ptr(), d_x.data_ptr(), 2, 4, 4, d_y.data_ptr(), 4, None,
                               0, None)
    assert st == 1  # GASB_INVALID_ARGUMENT: aggregate's source range check (tensor.cpp:515)


@pytest.mark.parametrize("d", [1, 47, 256, 602])
def test_mean_forward_exact_and_backward(torch, d):
    p = _plan()
    rp, cols = _stencil(p)
    ne, nb = len(p.extended_nodes), len(p.batch_nodes)
    rng = np.random.default_rng(100 + d)
    x = rng.standard_normal((ne, d)).astype(np.float32)
    d_rp, d_cols, d_x = _dev(torch, rp), _dev(torch, cols), _dev(torch, x)
    d_y = torch.zeros((nb, d), device="cuda")
    check(lib.gasb_spmm_mean_fwd(d_rp.data_ptr(), nb, d_cols.data_ptr(), d_x.data_ptr(), ne, d, d, d_y.data_ptr(), d,
                                 None))
    torch.cuda.synchronize()
    assert np.array_equal(d_y.cpu().numpy(), mean_fwd(rp, cols, x))
    # backward: the weighted-sum backward over the transposed stencil with the mean coefficients
    cf = np.zeros(len(cols), np.float32)
    check(lib.gasb_mean_coefficients(rp.ctypes.data, nb, cf.ctypes.data))
    assert np.array_equal(cf, mean_coefficients(rp))
    order = np.argsort(cols, kind="stable")  # CSC by source, rows ascending within a source
    t_rp = np.zeros(ne + 1, np.int32)
    np.add.at(t_rp, cols + 1, 1)
    t_rp = np.cumsum(t_rp).astype(np.int32)
    rows = np.repeat(np.arange(nb, dtype=np.int32), np.diff(rp))
    t_src, t_cf = rows[order], cf[order]
    gy = rng.standard_normal((nb, d)).astype(np.float32)
    d_gx = torch.zeros((ne, d), device="cuda")
    d_trp, d_tsrc, d_tcf, d_gy = _dev(torch, t_rp), _dev(torch, t_src), _dev(torch, t_cf), _dev(torch, gy)
    check(lib.gasb_spmm_bwd(d_trp.data_ptr(), ne, d_tsrc.data_ptr(), d_tcf.data_ptr(), d_gy.data_ptr(), d, nb, d, None,
                            0, d_gx.data_ptr(), d, None))
    torch.cuda.synchronize()
    gx = np.zeros((ne, d), np.float32)
    for r in range(nb):  # the reference's scatter order: rows ascending, edges in row order
        for k in range(rp[r], rp[r + 1]):
            gx[cols[k]] = (gx[cols[k]] + (cf[k] * gy[r]).astype(np.float32)).astype(np.float32)
    assert np.array_equal(d_gx.cpu().numpy(), gx)
