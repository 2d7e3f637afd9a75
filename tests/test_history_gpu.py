"""History store in HBM vs the reference HistoryStore semantics (history.cpp:10-178).
SPEC.md:364-398 examples: fresh store = zeros, push-then-pull identity, overwrite,
stamps, layer range errors, prefetch == synchronous pull."""
import numpy as np
import pytest

import paper_2106_05609_b200 as gb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def test_fresh_store_is_zero_and_push_pull_identity():
    h = gb.HistoryStore(2, 50, 7)
    assert np.array_equal(h.pull(1, [3, 4, 49]), np.zeros((3, 7), np.float32))
    rows = np.arange(21, dtype=np.float32).reshape(3, 7)
    h.push(1, [4, 9, 0], rows)
    assert np.array_equal(h.pull(1, [0, 4, 9]), rows[[2, 0, 1]])
    h.push(1, [9], rows[:1] + 100)  # second value wins
    assert np.array_equal(h.pull(1, [9])[0], rows[0] + 100)
    assert np.array_equal(h.pull(2, [4]), np.zeros((1, 7), np.float32))
    assert h.pull(1, []).shape == (0, 7)


def test_stamps_and_steps(ref):
    h = gb.HistoryStore(1, 10, 4)
    r = ref.lib
    import ctypes as C
    rh = C.c_void_p()
    ref.check(r.ref_history_create(1, 10, 4, C.byref(rh)))
    for step in range(3):
        ids = np.array([step, step + 3], np.int32)
        rows = np.full((2, 4), step, np.float32)
        h.push(1, ids, rows)
        ref.check(r.ref_history_push(rh, 1, ids.ctypes.data, 2, rows.ctypes.data))
        h.advance_step()
        r.ref_history_advance(rh)
    assert h.step() == 3
    for v in range(10):
        s = C.c_int64()
        ref.check(r.ref_history_stamp(rh, 1, v, C.byref(s)))
        assert h.last_push_step(1, v) == s.value
    full = np.zeros((10, 4), np.float32)
    ref.check(r.ref_history_layer(rh, 1, full.ctypes.data))
    assert np.array_equal(h.layer_matrix(1), full)
    h.reset()
    assert h.step() == 0 and h.last_push_step(1, 0) == -1 and not h.layer_matrix(1).any()
    r.ref_history_free(rh)


def test_errors_match_reference():
    h = gb.HistoryStore(2, 10, 3)
    for bad_layer in (0, 3):
        with pytest.raises(ValueError):
            h.pull(bad_layer, [1])
        with pytest.raises(ValueError):
            h.push(bad_layer, [1], np.zeros((1, 3), np.float32))
    with pytest.raises(ValueError):
        h.pull(1, [10])
    with pytest.raises(ValueError):
        h.push(1, [1, 2], np.zeros((1, 3), np.float32))  # row count mismatch
    with pytest.raises(ValueError):
        h.fill_layer(1, np.zeros((9, 3), np.float32))


def test_device_push_pull_large_bit_exact(torch):
    n, d = 200_000, 256
    h = gb.HistoryStore(3, n, d)
    rng = np.random.default_rng(0)
    ids = np.sort(rng.choice(n, 60_000, replace=False)).astype(np.int32)
    rows = torch.randn(len(ids), d, device="cuda")
    d_ids = torch.from_numpy(ids).cuda()
    h.push_device(2, d_ids, len(ids), rows, d)
    halo = torch.from_numpy(rng.choice(n, 150_000).astype(np.int32)).cuda()
    out = torch.empty(len(halo), d, device="cuda")
    h.pull_device(2, halo, len(halo), out, d)
    torch.cuda.synchronize()
    h.check()
    table = torch.zeros(n, d, device="cuda")
    table[d_ids.long()] = rows
    assert torch.equal(out, table[halo.long()])


def test_device_bad_id_latches_error(torch):
    h = gb.HistoryStore(1, 10, 4)
    ids = torch.tensor([1, 11], dtype=torch.int32, device="cuda")
    out = torch.zeros(2, 4, device="cuda")
    h.pull_device(1, ids, 2, out, 4)
    with pytest.raises(ValueError):
        h.check()
    h.check()  # latch cleared


def test_odd_dim_scalar_path(torch):
    h = gb.HistoryStore(1, 100, 47)
    ids = np.arange(0, 100, 3, dtype=np.int32)
    rows = np.random.default_rng(1).standard_normal((len(ids), 47)).astype(np.float32)
    h.push(1, ids, rows)
    assert np.array_equal(h.pull(1, ids[::-1]), rows[::-1])


def test_prefetch_snapshot(torch):
    n, d = 5000, 64
    h = gb.HistoryStore(3, n, d)
    vals = [np.random.default_rng(l).standard_normal((n, d)).astype(np.float32) for l in range(3)]
    for l in range(3):
        h.fill_layer(l + 1, vals[l])
    assert h.last_push_step(2, 17) == 0  # fill_layer stamps every row with the current step
    pf = gb.Prefetcher(h)
    halo_np = np.random.default_rng(9).choice(n, 1234).astype(np.int32)
    halo = torch.from_numpy(halo_np).cuda()
    s = torch.cuda.Stream()
    handle = pf.begin(halo, len(halo), s)
    for l in (1, 2, 3):
        p, ld = handle.wait(l)
        s.synchronize()
        snap = _device_to_numpy(torch, p, len(halo), ld)[:, :d]
        assert np.array_equal(snap, vals[l - 1][halo_np])
    with pytest.raises(ValueError):
        handle.wait(4)
    pf.begin(halo, len(halo), s)
    with pytest.raises(RuntimeError):
        handle.wait(1)  # stale generation -> logic_error


def _device_to_numpy(torch, ptr, rows, ld):
    import ctypes
    out = np.empty((rows, ld), np.float32)
    cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
    cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    assert cudart.cudaMemcpy(out.ctypes.data, ptr, out.nbytes, 2) == 0
    return out


def _ref_store(ref, layers, n, d):
    import ctypes as C
    rh = C.c_void_p()
    ref.check(ref.lib.ref_history_create(layers, n, d, C.byref(rh)))
    return rh


def _drive_both(ref, h, rh, layers, n, d, seed=7):
    """Same pushes / steps into our store and the compiled reference's."""
    rng = np.random.default_rng(seed)
    for step in range(6):
        for layer in range(1, layers + 1):
            ids = np.sort(rng.choice(n, size=n // 5, replace=False)).astype(np.int32)
            rows = rng.standard_normal((len(ids), d)).astype(np.float32)
            h.push(layer, ids, rows)
            ref.check(ref.lib.ref_history_push(rh, layer, ids.ctypes.data, len(ids), rows.ctypes.data))
        h.advance_step()
        ref.lib.ref_history_advance(rh)


def test_measure_staleness_bit_exact(ref):
    """measure_staleness (history.cpp:77-112): eps (row L2 distances) and push ages."""
    layers, n, d = 2, 777, 13
    h = gb.HistoryStore(layers, n, d)
    rh = _ref_store(ref, layers, n, d)
    _drive_both(ref, h, rh, layers, n, d)
    refm = np.random.default_rng(1).standard_normal((layers, n, d)).astype(np.float32)
    got = h.measure_staleness([refm[l] for l in range(layers)])
    out = np.zeros(4 * layers)
    ref.check(ref.lib.ref_history_staleness(rh, refm.ctypes.data, out.ctypes.data))
    for l in range(layers):
        exp = out[4 * l:4 * l + 4]
        g = got[l]
        assert (g["eps_max"], g["eps_mean"], g["age_max"], g["age_mean"]) == (exp[0], exp[1], int(exp[2]), exp[3])
    with pytest.raises(ValueError):
        h.measure_staleness([refm[0]])
    ref.lib.ref_history_free(rh)


def test_gash_checkpoint_interop(ref, tmp_path):
    """save/load_checkpoint in the reference's GASH format, both directions."""
    import ctypes as C
    layers, n, d = 3, 100, 6
    h = gb.HistoryStore(layers, n, d)
    rh = _ref_store(ref, layers, n, d)
    _drive_both(ref, h, rh, layers, n, d, seed=3)
    ours, theirs = tmp_path / "ours.gash", tmp_path / "theirs.gash"
    h.save_checkpoint(ours)
    ref.check(ref.lib.ref_history_save(rh, str(theirs).encode()))
    assert ours.read_bytes() == theirs.read_bytes()  # byte-identical files
    loaded = gb.HistoryStore.load_checkpoint(theirs)
    assert (loaded.num_layers(), loaded.num_nodes(), loaded.dim()) == (layers, n, d)
    rl = C.c_void_p()
    ref.check(ref.lib.ref_history_load(str(ours).encode(), C.byref(rl)))
    for l in range(1, layers + 1):
        full = np.zeros((n, d), np.float32)
        ref.check(ref.lib.ref_history_layer(rl, l, full.ctypes.data))
        assert np.array_equal(loaded.layer_matrix(l), full)
        assert np.array_equal(loaded.layer_matrix(l), h.layer_matrix(l))
        assert (loaded.stamps(l) == 0).all()
    assert loaded.step() == 0
    bad = tmp_path / "bad.gash"
    bad.write_bytes(b"GASX" + ours.read_bytes()[4:])
    with pytest.raises(RuntimeError):
        gb.HistoryStore.load_checkpoint(bad)
    bad.write_bytes(ours.read_bytes()[:100])
    with pytest.raises(RuntimeError):
        gb.HistoryStore.load_checkpoint(bad)
    with pytest.raises(RuntimeError):
        gb.HistoryStore.load_checkpoint(tmp_path / "missing.gash")
    ref.lib.ref_history_free(rh)
    ref.lib.ref_history_free(rl)


@pytest.mark.parametrize("d", [4, 16, 32, 48, 64, 68, 256])
def test_push_pull_widths(d):
    """Every row-kernel variant (narrow lane groups for d <= 64, float4, scalar) moves rows
    exactly; stamps follow the pushes."""
    n = 5000
    h = gb.HistoryStore(1, n, d)
    rng = np.random.default_rng(d)
    ids = np.sort(rng.choice(n, size=1777, replace=False)).astype(np.int32)
    rows = rng.standard_normal((len(ids), d)).astype(np.float32)
    h.push(1, ids, rows)
    want = np.zeros((n, d), np.float32)
    want[ids] = rows
    assert np.array_equal(h.layer_matrix(1), want)
    q = rng.permutation(n)[:999].astype(np.int32)
    assert np.array_equal(h.pull(1, q), want[q])
    st = h.stamps(1)
    assert (st[ids] == 0).all() and (np.delete(st, ids) == -1).all()
