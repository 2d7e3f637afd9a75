"""Partition files (io.cpp:187-217) and random_partition (partition.cpp:330-342) vs the
compiled reference — host code, runs on CPU."""
import ctypes as C

import numpy as np
import pytest

import paper_2106_05609_b200 as gb


def _ref_random(ref, n, parts, seed):
    g = ref.graph(edges=np.array([[0, 1]], np.int32), n=n)
    a = np.zeros(n, np.int32)
    ref.check(ref.lib.ref_random_partition(g.h, parts, seed, a.ctypes.data))
    return a


@pytest.mark.parametrize("n,parts,seed", [(10, 3, 0), (2708, 10, 0), (1000, 7, 42), (5, 5, 9)])
def test_random_partition_bit_exact(ref, n, parts, seed):
    assert np.array_equal(gb.random_partition(n, parts, seed), _ref_random(ref, n, parts, seed))


def test_random_partition_errors():
    with pytest.raises(ValueError):
        gb.random_partition(5, 0)
    with pytest.raises(ValueError):
        gb.random_partition(5, 6)


def test_partition_file_round_trip_with_reference(ref, tmp_path):
    a = gb.random_partition(300, 7, 3)
    ours, theirs = tmp_path / "ours.part", tmp_path / "theirs.part"
    gb.save_partition(ours, a)
    ref.check(ref.lib.ref_partition_save(str(theirs).encode(), a.ctypes.data, len(a), 7))
    assert ours.read_bytes() == theirs.read_bytes()
    got, k = gb.load_partition(theirs, 300)
    assert k == 7 and np.array_equal(got, a)
    b = np.zeros(300, np.int32)
    kk = C.c_int32()
    ref.check(ref.lib.ref_partition_load(str(ours).encode(), 300, b.ctypes.data, C.byref(kk)))
    assert kk.value == 7 and np.array_equal(b, a)


@pytest.mark.parametrize("text,exc", [
    ("0 0\n1 x\n", RuntimeError),          # malformed line
    ("0 0\n5 1\n", RuntimeError),          # node out of range
    ("0 0\n1 -1\n", RuntimeError),         # negative part
    ("0 0\n", RuntimeError),               # node 1 unassigned
    ("0 0\n1 2\n", ValueError),            # part 1 empty (partition_from_assignment)
])
def test_partition_file_errors_match_reference(ref, tmp_path, text, exc):
    p = tmp_path / "bad.part"
    p.write_text(text)
    with pytest.raises(exc):
        gb.load_partition(p, 2)
    b = np.zeros(2, np.int32)
    kk = C.c_int32()
    with pytest.raises(exc):
        ref.check(ref.lib.ref_partition_load(str(p).encode(), 2, b.ctypes.data, C.byref(kk)))


def test_partition_file_comments_and_overrides(tmp_path):
    p = tmp_path / "c.part"
    p.write_text("# header\n0 1  # trailing comment\n\n1 1\n0 0\n")  # later lines win
    a, k = gb.load_partition(p, 2)
    assert k == 2 and list(a) == [0, 1]
    p.write_text("0 1\n1 0\n0 0\n")  # num_parts = max part ever read + 1 -> part 1 empty
    with pytest.raises(ValueError):
        gb.load_partition(p, 2)
    with pytest.raises(RuntimeError):
        gb.load_partition(tmp_path / "missing.part", 2)


@pytest.mark.parametrize("name,parts,seed", [("cora", 10, 0), ("cora", 7, 3), ("pubmed_gcnii", 8, 0),
                                             ("reddit_mini", 12, 1)])
def test_cluster_partition_equals_reference(ref, name, parts, seed):
    """cluster_partition (partition.cpp:344-388): the same assignment as the compiled
    reference (multilevel coarsening, growth, refinement, balance repair)."""
    from paper_2106_05609_b200.workloads import make_dataset
    ds = make_dataset(name, with_features=False)
    a = gb.cluster_partition(ds.graph, parts, seed)
    b = ref.graph(csr=(ds.row_offsets, ds.cols)).cluster_partition(parts, seed)
    assert np.array_equal(a, b)
    assert np.bincount(a, minlength=parts).min() > 0


def test_cluster_partition_errors():
    g = gb.build_graph(np.array([[0, 1], [1, 2]]), 3)
    with pytest.raises(ValueError):
        gb.cluster_partition(g, 0)
    with pytest.raises(ValueError):
        gb.cluster_partition(g, 4)
