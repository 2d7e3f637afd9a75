"""graph-core and the partition-batch loader (reference: include/gas/graph.hpp,
src/graph.cpp, src/layers.cpp:42-70, src/trainer.cpp:253-262), over the C ABI.

Names and error behaviour mirror the reference: invalid inputs raise ValueError
(std::invalid_argument)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._native import SynthParams, check, f64, i32, i64, lib, ptr, vp


class Graph:
    """CSR of in-neighbours (graph.hpp:19-41). Owns a gasb_graph handle."""

    def __init__(self, handle: int):
        self._h = vp(handle)
        n, m = i32(), i64()
        check(lib.gasb_graph_info(self._h, C.byref(n), C.byref(m)))
        self.num_nodes = n.value
        self.num_edges = m.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.gasb_graph_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def csr(self) -> tuple[np.ndarray, np.ndarray]:
        """(row_offsets int64[n+1], col_indices int32[nnz]) — copies."""
        ro, co = vp(), vp()
        check(lib.gasb_graph_csr(self._h, C.byref(ro), C.byref(co)))
        n, m = self.num_nodes, self.num_edges
        r = np.ctypeslib.as_array(C.cast(ro, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
        c = np.ctypeslib.as_array(C.cast(co, C.POINTER(C.c_int32)), shape=(max(m, 1),))[:m].copy() if m else \
            np.zeros(0, np.int32)
        return r, c

    def degrees(self) -> np.ndarray:
        ro, _ = self.csr()
        return np.diff(ro).astype(np.int64)


def build_graph(edges: np.ndarray, num_nodes: int, symmetrize: bool = True) -> Graph:
    """build_graph (graph.hpp:46): edges is an (m, 2) array of (src, dst) = (u, v) pairs."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    u = np.ascontiguousarray(e[:, 0])
    v = np.ascontiguousarray(e[:, 1])
    h = vp()
    check(lib.gasb_graph_build(ptr(u), ptr(v), len(u), int(num_nodes), int(bool(symmetrize)), C.byref(h)))
    return Graph(h.value)


def graph_from_csr(row_offsets: np.ndarray, cols: np.ndarray, symmetric: bool = True) -> Graph:
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    co = np.ascontiguousarray(cols, dtype=np.int32)
    h = vp()
    check(lib.gasb_graph_from_csr(len(ro) - 1, ptr(ro), ptr(co) if len(co) else None, int(symmetric), C.byref(h)))
    return Graph(h.value)


def synth_pairs(num_nodes: int, num_pairs: int, communities: int, intra_fraction: float, gamma: float = 2.5,
                min_weight: float = 1.0, max_weight: float = 1e9, seed: int = 1):
    """Seeded power-law + planted-community pair generator (include/gasb.h). Returns
    (edges (m,2) int32, community int32[n])."""
    p = SynthParams(num_nodes, communities, num_pairs, intra_fraction, gamma, min_weight, max_weight, seed)
    src = np.empty(num_pairs, np.int32)
    dst = np.empty(num_pairs, np.int32)
    comm = np.empty(num_nodes, np.int32)
    check(lib.gasb_synth_pairs(C.byref(p), ptr(src), ptr(dst), ptr(comm)))
    return np.stack([src, dst], axis=1), comm


def synth_features(num_nodes: int, dim: int, seed: int = 2) -> np.ndarray:
    out = np.empty((num_nodes, dim), np.float32)
    check(lib.gasb_synth_features(num_nodes, dim, dim, seed, ptr(out)))
    return out


@dataclass
class BatchPlan:
    """BatchPlan (graph.hpp:71-85) + PlanAggregation (layers.hpp:33-36), host copies."""

    batch_nodes: np.ndarray
    extended_nodes: np.ndarray
    halo_nodes: np.ndarray
    is_halo: np.ndarray
    batch_local_rows: np.ndarray
    halo_local_rows: np.ndarray
    local_row_offsets: np.ndarray | None
    local_col_indices: np.ndarray | None
    gcn_row_ptr: np.ndarray
    gcn_cols: np.ndarray
    gcn_coeffs: np.ndarray
    sum_row_ptr: np.ndarray | None
    sum_cols: np.ndarray | None
    sum_coeffs: np.ndarray | None


class BatchSchedule:
    """BatchSchedule::build (trainer.hpp:91-96): one plan per part, in part order."""

    def __init__(self, handle: int, graph: Graph):
        self._h = vp(handle)
        self.graph = graph  # keeps the graph alive (plans borrow it)
        n = i32()
        check(lib.gasb_schedule_num_parts(self._h, C.byref(n)))
        self.num_parts = n.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.gasb_schedule_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @staticmethod
    def build(graph: Graph, assignment: np.ndarray, num_parts: int, full: bool = False,
              device: bool = False) -> "BatchSchedule":
        """device=True runs the GPU batch-plan builder (plan_dev.cu) on the current CUDA
        device; the plans are bit-identical to the host builder's."""
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        if len(a) != graph.num_nodes:
            raise ValueError("partition: assignment length != num_nodes")
        h = vp()
        flags = (1 if full else 0) | (2 if device else 0)
        check(lib.gasb_schedule_build(graph.handle, ptr(a), int(num_parts), flags, C.byref(h)))
        return BatchSchedule(h.value, graph)

    def timing(self) -> tuple[float, float]:
        """(device_ms, total_ms) of the build; device_ms is -1 for host builds."""
        d, t = f64(), f64()
        check(lib.gasb_schedule_timing(self._h, C.byref(d), C.byref(t)))
        return d.value, t.value

    def sizes(self, part: int) -> np.ndarray:
        z = np.zeros(6, np.int64)
        check(lib.gasb_plan_sizes(self._h, int(part), ptr(z)))
        return z

    def batch_nodes(self, part: int) -> np.ndarray:
        """The part's batch node ids (sorted global ids), without copying its stencils."""
        nb, ne = (int(x) for x in self.sizes(part)[:2])
        ext, blr = np.empty(ne, np.int32), np.empty(nb, np.int32)
        check(lib.gasb_plan_copy(self._h, int(part), ptr(ext) if ne else None, None, None, ptr(blr) if nb else None,
                                 *([None] * 9)))
        return ext[blr] if nb else np.empty(0, np.int32)

    def plan(self, part: int) -> BatchPlan:
        nb, ne, nh, lnnz, gnnz, snnz = (int(x) for x in self.sizes(part))
        full = lnnz >= 0
        a = dict(
            extended_nodes=np.empty(ne, np.int32), halo_nodes=np.empty(nh, np.int32), is_halo=np.empty(ne, np.uint8),
            batch_local_rows=np.empty(nb, np.int32), halo_local_rows=np.empty(nh, np.int32),
            local_row_offsets=np.empty(ne + 1, np.int64) if full else None,
            local_col_indices=np.empty(max(lnnz, 0), np.int32) if full else None,
            gcn_row_ptr=np.empty(nb + 1, np.int64), gcn_cols=np.empty(gnnz, np.int32),
            gcn_coeffs=np.empty(gnnz, np.float32),
            sum_row_ptr=np.empty(nb + 1, np.int64) if full else None,
            sum_cols=np.empty(max(snnz, 0), np.int32) if full else None,
            sum_coeffs=np.empty(max(snnz, 0), np.float32) if full else None,
        )
        order = ["extended_nodes", "halo_nodes", "is_halo", "batch_local_rows", "halo_local_rows",
                 "local_row_offsets", "local_col_indices", "gcn_row_ptr", "gcn_cols", "gcn_coeffs",
                 "sum_row_ptr", "sum_cols", "sum_coeffs"]
        check(lib.gasb_plan_copy(self._h, int(part), *[ptr(a[k]) if a[k] is not None and a[k].size else None
                                                        for k in order]))
        batch = a["extended_nodes"][a["batch_local_rows"]] if nb else np.empty(0, np.int32)
        return BatchPlan(batch_nodes=batch, **a)


def make_batch_plan(graph: Graph, batch_nodes, full: bool = True) -> BatchPlan:
    """make_batch_plan (graph.hpp:88) + build_plan_aggregation (layers.hpp:38)."""
    b = np.ascontiguousarray(np.asarray(batch_nodes, dtype=np.int32))
    arr = (C.c_void_p * 1)(b.ctypes.data)
    sizes = np.array([len(b)], np.int64)
    h = vp()
    check(lib.gasb_schedule_build_batches(graph.handle, arr, ptr(sizes), 1, 1 if full else 0, C.byref(h)))
    return BatchSchedule(h.value, graph).plan(0)


def partition_parts(assignment: np.ndarray, num_parts: int) -> list[np.ndarray]:
    """partition_from_assignment (partition.cpp:314-328): sorted node list per part."""
    a = np.asarray(assignment)
    order = np.argsort(a, kind="stable")
    bounds = np.searchsorted(a[order], np.arange(num_parts + 1))
    return [order[bounds[p]:bounds[p + 1]].astype(np.int32) for p in range(num_parts)]


def save_partition(path: str, assignment) -> None:
    """save_partition (io.cpp:187-192)."""
    a = np.ascontiguousarray(assignment, dtype=np.int32)
    check(lib.gasb_partition_save(str(path).encode(), ptr(a) if len(a) else None, len(a)))


def load_partition(path: str, num_nodes: int) -> tuple[np.ndarray, int]:
    """load_partition (io.cpp:194-217): (assignment, num_parts)."""
    a = np.empty(num_nodes, np.int32)
    k = i32()
    check(lib.gasb_partition_load(str(path).encode(), int(num_nodes), ptr(a) if num_nodes else None, C.byref(k)))
    return a, k.value


def random_partition(num_nodes: int, num_parts: int, seed: int = 0) -> np.ndarray:
    """random_partition (partition.cpp:330-342), bit-exact with the reference."""
    a = np.empty(num_nodes, np.int32)
    check(lib.gasb_random_partition(int(num_nodes), int(num_parts), int(seed), ptr(a)))
    return a


def cluster_partition(graph: Graph, num_parts: int, seed: int = 0) -> np.ndarray:
    """cluster_partition (partition.cpp:344-388): the reference's multilevel partitioner,
    same assignment for the same graph / parts / seed."""
    a = np.empty(graph.num_nodes, np.int32)
    check(lib.gasb_cluster_partition(graph.handle, int(num_parts), int(seed), ptr(a)))
    return a
