"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracles.

  Oracle  : oracle/build/liboracle.so — the plain-C restatement (gas_oracle.c)
  RefLib  : oracle/_ref/libref.so     — the reference itself, compiled in place (ref_harness.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm import
this module, and only as the checker / CPU baseline; the product never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libref.so"

i32, i64, u64, f32, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_void_p
P = C.POINTER


def _p(a):
    if a is None:
        return None
    return a.ctypes.data


class Spec(C.Structure):  # go_spec / RefSpec (same layout)
    _fields_ = [("kind", i32), ("num_layers", i32), ("hidden", i32), ("dropout", f32), ("alpha", f32),
                ("beta", f32), ("l2_weight", f32), ("clip_max_norm", f32), ("lr", f32), ("beta1", f32),
                ("beta2", f32), ("eps", f32), ("seed", u64)]


def make_spec(kind=0, num_layers=2, hidden=16, dropout=0.0, alpha=0.1, beta=0.5, l2_weight=0.0, clip_max_norm=0.0,
              lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8, seed=0) -> Spec:
    return Spec(kind, num_layers, hidden, dropout, alpha, beta, l2_weight, clip_max_norm, lr, beta1, beta2, eps, seed)


class PlanArrays(C.Structure):  # go_plan
    _fields_ = [("nb", i32), ("next", i32), ("nhalo", i32)] + [(k, vp) for k in (
        "batch", "extended", "halo", "is_halo", "batch_local_rows", "halo_local_rows", "local_rowptr", "local_cols",
        "gcn_rowptr", "gcn_cols", "gcn_coeffs", "sum_rowptr", "sum_cols", "sum_coeffs")]


def _arr(p, dtype, n):
    if n == 0:
        return np.zeros(0, dtype)
    ct = {np.int32: C.c_int32, np.int64: C.c_int64, np.float32: C.c_float, np.uint8: C.c_uint8}[dtype]
    return np.ctypeslib.as_array(C.cast(p, P(ct)), shape=(n,)).copy()


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(str(path))
        L.go_build_graph.argtypes = [vp, vp, i64, i32, C.c_int, vp, P(vp), P(i64)]
        L.go_plan_make.argtypes = [i32, vp, vp, vp, i64, P(PlanArrays)]
        L.go_plan_free.argtypes = [P(PlanArrays)]
        L.go_free.argtypes = [vp]
        L.go_aggregate_fwd.argtypes = [vp, i64, vp, vp, vp, i64, vp]
        L.go_aggregate_bwd.argtypes = [vp, i64, vp, vp, vp, i64, vp]
        L.go_matmul_fwd.argtypes = [vp, i64, i64, vp, i64, vp]
        L.go_matmul_bwd.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp]
        L.go_softmax_ce.argtypes = [vp, i64, i64, vp, vp, i64, vp]
        L.go_softmax_ce.restype = f32
        L.go_glorot.argtypes = [i64, i64, u64, vp]
        L.go_epoch_order.argtypes = [i32, u64, i64, vp]
        L.go_derive_seed.argtypes = [u64, u64, u64, u64]
        L.go_derive_seed.restype = u64
        L.go_grad_clip.argtypes = [vp, i64, f64]
        L.go_grad_clip.restype = f64
        L.go_session_create.argtypes = [i32, vp, vp, vp, i32, vp, vp, i32, vp, i32, P(Spec), P(vp)]
        L.go_session_free.argtypes = [vp]
        L.go_session_num_param_floats.argtypes = [vp]
        L.go_session_num_param_floats.restype = i64
        L.go_session_get_params.argtypes = [vp, vp]
        L.go_session_set_params.argtypes = [vp, vp]
        L.go_session_history_dim.argtypes = [vp]
        L.go_session_history_dim.restype = i32
        L.go_session_get_history.argtypes = [vp, i32, vp]
        L.go_session_set_history.argtypes = [vp, i32, vp]
        L.go_session_batch.argtypes = [vp, i32, i64, C.c_int, C.c_int, vp, vp, P(f64), vp, P(C.c_int)]
        L.go_session_epoch.argtypes = [vp, i64, C.c_int, P(f64)]
        L.go_session_dp_batch.argtypes = [vp, i32, vp, vp, P(f64), P(C.c_int)]
        L.go_session_dp_commit.argtypes = [vp, i32, vp]
        L.go_session_dp_apply.argtypes = [vp, vp, i32, i32]
        L.go_session_dp_epoch.argtypes = [vp, i64, C.c_int, i32, P(f64)]
        L.go_synth_pairs.argtypes = [i32, i32, i64, f64, f64, f64, f64, u64, vp, vp, vp]
        L.go_synth_features.argtypes = [i64, i32, i64, u64, vp]

    def build_graph(self, edges: np.ndarray, n: int, symmetrize=True):
        e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
        u, v = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
        ro = np.zeros(n + 1, np.int64)
        cols, nnz = vp(), i64()
        rc = self.lib.go_build_graph(_p(u), _p(v), len(u), n, int(symmetrize), _p(ro), C.byref(cols), C.byref(nnz))
        if rc:
            raise ValueError("build_graph: invalid argument")
        out = _arr(cols.value, np.int32, nnz.value)
        self.lib.go_free(cols)
        return ro, out

    def make_plan(self, ro, cols, batch) -> dict:
        b = np.ascontiguousarray(batch, np.int32)
        pa = PlanArrays()
        rc = self.lib.go_plan_make(len(ro) - 1, _p(ro), _p(np.ascontiguousarray(cols, np.int32)), _p(b), len(b),
                                   C.byref(pa))
        if rc:
            raise ValueError("make_batch_plan: invalid argument")
        nb, ne, nh = pa.nb, pa.next, pa.nhalo
        lrp = _arr(pa.local_rowptr, np.int64, ne + 1)
        grp = _arr(pa.gcn_rowptr, np.int64, nb + 1)
        srp = _arr(pa.sum_rowptr, np.int64, nb + 1)
        d = dict(batch_nodes=_arr(pa.batch, np.int32, nb), extended_nodes=_arr(pa.extended, np.int32, ne),
                 halo_nodes=_arr(pa.halo, np.int32, nh), is_halo=_arr(pa.is_halo, np.uint8, ne),
                 batch_local_rows=_arr(pa.batch_local_rows, np.int32, nb),
                 halo_local_rows=_arr(pa.halo_local_rows, np.int32, nh), local_row_offsets=lrp,
                 local_col_indices=_arr(pa.local_cols, np.int32, int(lrp[-1])), gcn_row_ptr=grp,
                 gcn_cols=_arr(pa.gcn_cols, np.int32, int(grp[-1])), gcn_coeffs=_arr(pa.gcn_coeffs, np.float32,
                                                                                      int(grp[-1])),
                 sum_row_ptr=srp, sum_cols=_arr(pa.sum_cols, np.int32, int(srp[-1])),
                 sum_coeffs=_arr(pa.sum_coeffs, np.float32, int(srp[-1])))
        self.lib.go_plan_free(C.byref(pa))
        return d

    def aggregate(self, rp, cols, coeffs, x, gy=None):
        rp = np.ascontiguousarray(rp, np.int64)
        m, d = len(rp) - 1, x.shape[1]
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros((m, d), np.float32)
        self.lib.go_aggregate_fwd(_p(rp), m, _p(np.ascontiguousarray(cols, np.int32)),
                                  _p(np.ascontiguousarray(coeffs, np.float32)), _p(x), d, _p(y))
        if gy is None:
            return y
        gx = np.zeros_like(x)
        self.lib.go_aggregate_bwd(_p(rp), m, _p(np.ascontiguousarray(cols, np.int32)),
                                  _p(np.ascontiguousarray(coeffs, np.float32)),
                                  _p(np.ascontiguousarray(gy, np.float32)), d, _p(gx))
        return y, gx

    def matmul(self, a, b, gy=None):
        a, b = np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        y = np.zeros((m, n), np.float32)
        self.lib.go_matmul_fwd(_p(a), m, k, _p(b), n, _p(y))
        if gy is None:
            return y
        ga, gb = np.zeros_like(a), np.zeros_like(b)
        self.lib.go_matmul_bwd(_p(a), _p(b), _p(np.ascontiguousarray(gy, np.float32)), m, k, n, _p(ga), _p(gb))
        return y, ga, gb

    def softmax_ce(self, logits, rows, labels):
        lg = np.ascontiguousarray(logits, np.float32)
        g = np.zeros_like(lg)
        r = np.ascontiguousarray(rows, np.int32)
        lab = np.ascontiguousarray(labels, np.int32)
        loss = self.lib.go_softmax_ce(_p(lg), lg.shape[0], lg.shape[1], _p(r), _p(lab), len(r), _p(g))
        return loss, g

    def glorot(self, rows, cols, seed):
        out = np.zeros(rows * cols, np.float32)
        self.lib.go_glorot(rows, cols, seed, _p(out))
        return out.reshape(rows, cols)

    def epoch_order(self, nb, seed, epoch):
        out = np.zeros(nb, np.int32)
        self.lib.go_epoch_order(nb, seed, epoch, _p(out))
        return out

    def session(self, ro, cols, features, labels, train_mask, num_classes, assignment, num_parts, spec: Spec):
        return Session(self, "go", ro, cols, features, labels, train_mask, num_classes, assignment, num_parts, spec)


class OracleSynth:
    """The bench input generator restated in the oracle (go_synth_*; go_build_graph restates
    build_graph, src/graph.cpp:25-61): the `backend` of workloads.make_dataset for bench.py's
    reference arm, which must not load the product library. Graph handle = None."""

    def __init__(self, oracle: "Oracle | None" = None):
        self.o = oracle or Oracle()

    def synth_pairs(self, w):
        src, dst = np.empty(w.num_pairs, np.int32), np.empty(w.num_pairs, np.int32)
        comm = np.empty(w.num_nodes, np.int32)
        if self.o.lib.go_synth_pairs(w.num_nodes, w.parts * w.comm_per_part, w.num_pairs, w.intra_fraction, 2.5, 1.0, w.max_weight,
                                     w.seed, _p(src), _p(dst), _p(comm)):
            raise ValueError("synth_pairs: bad argument")
        return np.stack([src, dst], axis=1), comm

    def build_graph(self, edges, n):
        ro, co = self.o.build_graph(edges, n, symmetrize=True)
        return None, ro, co

    def synth_features(self, n, dim, seed):
        out = np.empty((n, dim), np.float32)
        self.o.lib.go_synth_features(n, dim, dim, seed, _p(out))
        return out


class RefLib:
    """The reference compiled from /root/reference/proj (oracle/_ref/libref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_build.argtypes = [vp, vp, i64, i32, C.c_int, P(vp)]
        L.ref_graph_from_csr.argtypes = [i32, vp, vp, C.c_int, P(vp)]
        L.ref_graph_num_edges.argtypes = [vp]
        L.ref_graph_num_edges.restype = i64
        L.ref_graph_copy.argtypes = [vp, vp, vp]
        L.ref_graph_free.argtypes = [vp]
        L.ref_plan_make.argtypes = [vp, vp, i64, P(vp)]
        L.ref_plan_sizes.argtypes = [vp, vp]
        L.ref_plan_copy.argtypes = [vp] + [vp] * 13
        L.ref_plan_free.argtypes = [vp]
        L.ref_cluster_partition.argtypes = [vp, i32, u64, vp]
        L.ref_random_partition.argtypes = [vp, i32, u64, vp]
        L.ref_partition_save.argtypes = [C.c_char_p, vp, i32, i32]
        L.ref_partition_load.argtypes = [C.c_char_p, i32, vp, P(i32)]
        L.ref_inter_intra_ratio.argtypes = [vp, vp, i32]
        L.ref_inter_intra_ratio.restype = f64
        L.ref_aggregate.argtypes = [vp, i64, vp, vp, vp, i64, i64, vp, vp, vp]
        L.ref_matmul.argtypes = [vp, i64, i64, vp, i64, vp, vp, vp, vp]
        L.ref_softmax_ce.argtypes = [vp, i64, i64, vp, vp, i64, vp, vp]
        L.ref_adam.argtypes = [vp, i64, vp, i32, f32, f32, f32, f32]
        L.ref_grad_clip.argtypes = [vp, i64, f64]
        L.ref_grad_clip.restype = f64
        L.ref_glorot.argtypes = [i64, i64, u64, vp]
        L.ref_epoch_order.argtypes = [i32, u64, i64, vp]
        L.ref_derive_seed.argtypes = [u64, u64, u64, u64]
        L.ref_derive_seed.restype = u64
        L.ref_history_create.argtypes = [i32, i32, i32, P(vp)]
        L.ref_history_free.argtypes = [vp]
        L.ref_history_push.argtypes = [vp, i32, vp, i64, vp]
        L.ref_history_pull.argtypes = [vp, i32, vp, i64, vp]
        L.ref_history_advance.argtypes = [vp]
        L.ref_history_stamp.argtypes = [vp, i32, i32, P(i64)]
        L.ref_history_fill.argtypes = [vp, i32, vp]
        L.ref_history_layer.argtypes = [vp, i32, vp]
        L.ref_history_staleness.argtypes = [vp, vp, vp]
        L.ref_history_save.argtypes = [vp, C.c_char_p]
        L.ref_history_load.argtypes = [C.c_char_p, P(vp)]
        L.ref_session_create.argtypes = [vp, vp, i32, vp, vp, i32, vp, i32, vp, i32, P(Spec), P(vp)]
        L.ref_session_free.argtypes = [vp]
        L.ref_session_num_params.argtypes = [vp]
        L.ref_session_param_shape.argtypes = [vp, i32, P(i64), P(i64)]
        L.ref_session_get_params.argtypes = [vp, vp]
        L.ref_session_set_params.argtypes = [vp, vp]
        L.ref_session_history_dim.argtypes = [vp]
        L.ref_session_history_dim.restype = i32
        L.ref_session_get_history.argtypes = [vp, i32, vp]
        L.ref_session_set_history.argtypes = [vp, i32, vp]
        L.ref_session_store_step.argtypes = [vp]
        L.ref_session_store_step.restype = i64
        L.ref_session_adam_steps.argtypes = [vp]
        L.ref_session_adam_steps.restype = i64
        L.ref_session_epoch.argtypes = [vp, i64, C.c_int, C.c_int, P(f64), P(f64)]
        L.ref_session_batch.argtypes = [vp, i32, i64, C.c_int, C.c_int, vp, vp, P(f64), vp, P(C.c_int)]
        L.ref_session_run.argtypes = [vp, i32, i64, P(f64), P(f64)]
        L.ref_session_epoch_report.argtypes = [vp, i64, C.c_int, C.c_int, P(f64), P(i64), P(i64), vp, vp]
        L.ref_session_evaluate.argtypes = [vp, vp, vp, vp, vp]
        L.ref_session_infer.argtypes = [vp, vp, P(C.c_int)]

    def check(self, rc):
        if rc == 0:
            return
        msg = self.lib.ref_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    def graph(self, edges=None, n=None, symmetrize=True, csr=None):
        g = vp()
        if csr is not None:
            ro, co = (np.ascontiguousarray(csr[0], np.int64), np.ascontiguousarray(csr[1], np.int32))
            self.check(self.lib.ref_graph_from_csr(len(ro) - 1, _p(ro), _p(co), 1, C.byref(g)))
        else:
            e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
            u, v = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
            self.check(self.lib.ref_graph_build(_p(u), _p(v), len(u), n, int(symmetrize), C.byref(g)))
        return RefGraph(self, g, n if n is not None else len(csr[0]) - 1)

    def aggregate(self, rp, cols, coeffs, x, gy=None):
        rp = np.ascontiguousarray(rp, np.int64)
        x = np.ascontiguousarray(x, np.float32)
        m, d = len(rp) - 1, x.shape[1]
        y = np.zeros((m, d), np.float32)
        gx = np.zeros_like(x) if gy is not None else None
        self.check(self.lib.ref_aggregate(_p(rp), m, _p(np.ascontiguousarray(cols, np.int32)),
                                          _p(np.ascontiguousarray(coeffs, np.float32)), _p(x), x.shape[0], d, _p(y),
                                          _p(np.ascontiguousarray(gy, np.float32)) if gy is not None else None,
                                          _p(gx)))
        return y if gy is None else (y, gx)

    def matmul(self, a, b, gy=None):
        a, b = np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        y = np.zeros((m, n), np.float32)
        ga = np.zeros_like(a) if gy is not None else None
        gb = np.zeros_like(b) if gy is not None else None
        self.check(self.lib.ref_matmul(_p(a), m, k, _p(b), n, _p(y),
                                       _p(np.ascontiguousarray(gy, np.float32)) if gy is not None else None, _p(ga),
                                       _p(gb)))
        return y if gy is None else (y, ga, gb)

    def softmax_ce(self, logits, rows, labels):
        lg = np.ascontiguousarray(logits, np.float32)
        g = np.zeros_like(lg)
        loss = f32()
        r = np.ascontiguousarray(rows, np.int32)
        lab = np.ascontiguousarray(labels, np.int32)
        self.check(self.lib.ref_softmax_ce(_p(lg), lg.shape[0], lg.shape[1], _p(r), _p(lab), len(r), C.byref(loss),
                                           _p(g)))
        return loss.value, g

    def adam(self, p, grads, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
        p = np.ascontiguousarray(p, np.float32).copy()
        g = np.ascontiguousarray(grads, np.float32)
        self.check(self.lib.ref_adam(_p(p), p.size, _p(g), g.shape[0], lr, b1, b2, eps))
        return p

    def glorot(self, rows, cols, seed):
        out = np.zeros(rows * cols, np.float32)
        self.lib.ref_glorot(rows, cols, seed, _p(out))
        return out.reshape(rows, cols)

    def epoch_order(self, nb, seed, epoch):
        out = np.zeros(nb, np.int32)
        self.lib.ref_epoch_order(nb, seed, epoch, _p(out))
        return out

    def session(self, ro, cols, features, labels, train_mask, num_classes, assignment, num_parts, spec: Spec,
                sample_parts=None):
        return Session(self, "ref", ro, cols, features, labels, train_mask, num_classes, assignment, num_parts, spec,
                       sample_parts)


class RefGraph:
    def __init__(self, ref: RefLib, h, n):
        self.ref, self.h, self.n = ref, h, n

    def __del__(self):
        if self.h:
            self.ref.lib.ref_graph_free(self.h)
            self.h = None

    def csr(self):
        m = self.ref.lib.ref_graph_num_edges(self.h)
        ro = np.zeros(self.n + 1, np.int64)
        co = np.zeros(max(m, 1), np.int32)
        self.ref.lib.ref_graph_copy(self.h, _p(ro), _p(co))
        return ro, co[:m]

    def plan(self, batch) -> dict:
        b = np.ascontiguousarray(batch, np.int32)
        h = vp()
        self.ref.check(self.ref.lib.ref_plan_make(self.h, _p(b), len(b), C.byref(h)))
        z = np.zeros(6, np.int64)
        self.ref.lib.ref_plan_sizes(h, _p(z))
        nb, ne, nh, lnnz, gnnz, snnz = (int(x) for x in z)
        d = dict(extended_nodes=np.zeros(ne, np.int32), halo_nodes=np.zeros(nh, np.int32),
                 is_halo=np.zeros(ne, np.uint8), batch_local_rows=np.zeros(nb, np.int32),
                 halo_local_rows=np.zeros(nh, np.int32), local_row_offsets=np.zeros(ne + 1, np.int64),
                 local_col_indices=np.zeros(lnnz, np.int32), gcn_row_ptr=np.zeros(nb + 1, np.int64),
                 gcn_cols=np.zeros(gnnz, np.int32), gcn_coeffs=np.zeros(gnnz, np.float32),
                 sum_row_ptr=np.zeros(nb + 1, np.int64), sum_cols=np.zeros(snnz, np.int32),
                 sum_coeffs=np.zeros(snnz, np.float32))
        self.ref.lib.ref_plan_copy(h, *[_p(a) if a.size else None for a in d.values()])
        self.ref.lib.ref_plan_free(h)
        d["batch_nodes"] = b.copy()
        return d

    def cluster_partition(self, parts, seed=0):
        a = np.zeros(self.n, np.int32)
        self.ref.check(self.ref.lib.ref_cluster_partition(self.h, parts, seed, _p(a)))
        return a

    def inter_intra_ratio(self, assignment, parts):
        a = np.ascontiguousarray(assignment, np.int32)
        return self.ref.lib.ref_inter_intra_ratio(self.h, _p(a), parts)


class Session:
    """Model + Adam + HistoryStore + BatchSchedule in either oracle (same contract)."""

    def __init__(self, owner, kind, ro, cols, features, labels, train_mask, num_classes, assignment, num_parts, spec,
                 sample_parts=None):
        self.owner, self.kind, self.spec = owner, kind, spec
        self.n = len(ro) - 1
        self.num_classes = num_classes
        self._x = np.ascontiguousarray(features, np.float32)
        lab = np.ascontiguousarray(labels, np.int32)
        tm = np.ascontiguousarray(train_mask, np.uint8)
        asg = np.ascontiguousarray(assignment, np.int32)
        ro = np.ascontiguousarray(ro, np.int64)
        co = np.ascontiguousarray(cols, np.int32)
        h = vp()
        L = owner.lib
        if kind == "go":
            rc = L.go_session_create(self.n, _p(ro), _p(co), _p(self._x), self._x.shape[1], _p(lab), _p(tm),
                                     num_classes, _p(asg), num_parts, C.byref(spec), C.byref(h))
            if rc:
                raise ValueError("go_session_create: invalid argument")
            self.nparam = L.go_session_num_param_floats(h)
            self.hist_dim = L.go_session_history_dim(h)
        else:
            self._g = owner.graph(csr=(ro, co))
            sp = np.ascontiguousarray(sample_parts, np.int32) if sample_parts is not None else None
            owner.check(L.ref_session_create(self._g.h, _p(self._x), self._x.shape[1], _p(lab), _p(tm), num_classes,
                                             _p(asg), num_parts, _p(sp), len(sp) if sp is not None else 0,
                                             C.byref(spec), C.byref(h)))
            k = L.ref_session_num_params(h)
            tot = 0
            for i in range(k):
                r, c = i64(), i64()
                L.ref_session_param_shape(h, i, C.byref(r), C.byref(c))
                tot += r.value * c.value
            self.nparam = tot
            self.hist_dim = L.ref_session_history_dim(h)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            (self.owner.lib.go_session_free if self.kind == "go" else self.owner.lib.ref_session_free)(self.h)
            self.h = None

    def _fn(self, name):
        return getattr(self.owner.lib, ("go_session_" if self.kind == "go" else "ref_session_") + name)

    def get_params(self):
        out = np.zeros(self.nparam, np.float32)
        self._fn("get_params")(self.h, _p(out))
        return out

    def set_params(self, v):
        v = np.ascontiguousarray(v, np.float32)
        self._fn("set_params")(self.h, _p(v))

    def get_history(self, layer):
        out = np.zeros((self.n, self.hist_dim), np.float32)
        self._fn("get_history")(self.h, layer, _p(out))
        return out

    def set_history(self, layer, v):
        v = np.ascontiguousarray(v, np.float32)
        self._fn("set_history")(self.h, layer, _p(v))

    def batch(self, part, epoch=0, train=True, push=True, nb=None):
        """(acts[(L-1), nb, hd], logits[nb, C], loss, grads|None, stepped)"""
        L = self.spec.num_layers
        acts = np.zeros((max(L - 1, 0), nb, self.hist_dim), np.float32)
        logits = np.zeros((nb, self.num_classes), np.float32)
        grads = np.zeros(self.nparam, np.float32)
        loss, stepped = f64(), C.c_int()
        rc = self._fn("batch")(self.h, part, epoch, int(train), int(push), _p(acts) if acts.size else None,
                               _p(logits), C.byref(loss), _p(grads), C.byref(stepped))
        if self.kind == "ref":
            self.owner.check(rc)
        elif rc:
            raise ValueError("go_session_batch failed")
        return acts, logits, loss.value, (grads if stepped.value else None), bool(stepped.value)

    def evaluate(self, val_mask, test_mask):
        """Reference only: evaluate (trainer.cpp:444-464) -> ((train, val, test), logits n x C)."""
        vm = np.ascontiguousarray(val_mask, np.uint8)
        tm = np.ascontiguousarray(test_mask, np.uint8)
        acc = np.zeros(3)
        logits = np.zeros((self.n, self.num_classes), np.float32)
        self.owner.check(self.owner.lib.ref_session_evaluate(self.h, _p(vm), _p(tm), _p(acc), _p(logits)))
        return tuple(float(a) for a in acc), logits

    def infer(self):
        """Reference only: infer_from_history (trainer.cpp:501-536) -> (predictions, stale)."""
        pred = np.zeros(self.n, np.int32)
        st = C.c_int()
        self.owner.check(self.owner.lib.ref_session_infer(self.h, _p(pred), C.byref(st)))
        return pred, bool(st.value)

    def run(self, slot, epoch=0):
        """Reference only: one gas_epoch batch without capture; returns (loss, seconds)."""
        loss, secs = f64(), f64()
        self.owner.check(self.owner.lib.ref_session_run(self.h, slot, epoch, C.byref(loss), C.byref(secs)))
        return loss.value, secs.value

    def epoch(self, epoch, shuffle=True, prefetch=False):
        loss, secs = f64(), f64()
        if self.kind == "go":
            rc = self.owner.lib.go_session_epoch(self.h, epoch, int(shuffle), C.byref(loss))
            if rc:
                raise ValueError("go_session_epoch failed")
            return loss.value, None
        self.owner.check(self.owner.lib.ref_session_epoch(self.h, epoch, int(shuffle), int(prefetch), C.byref(loss),
                                                          C.byref(secs)))
        return loss.value, secs.value

    def epoch_report(self, epoch, num_parts, measure_staleness=True, shuffle=True):
        """Reference only: gas_epoch's EpochReport (loss, peak_floats, edges_per_layer,
        batch_peak_floats, eps_max) with EpochOptions{evaluate=false}."""
        loss, pk, epl = f64(), i64(), i64()
        bp = np.zeros(num_parts, np.int64)
        eps = np.zeros(max(self.spec.num_layers - 1, 1), np.float64)
        self.owner.check(self.owner.lib.ref_session_epoch_report(self.h, epoch, int(shuffle), int(measure_staleness),
                                                                 C.byref(loss), C.byref(pk), C.byref(epl), _p(bp),
                                                                 _p(eps)))
        return dict(loss=loss.value, peak_floats=pk.value, edges_per_layer=epl.value, batch_peak_floats=bp,
                    eps_max=eps[:max(self.spec.num_layers - 1, 0)] if measure_staleness else np.zeros(0))

    # ---- data-parallel step semantics (C restatement only) ----
    def dp_epoch(self, epoch, k, shuffle=True):
        """Mean loss of one data-parallel epoch with k batches per step (k = 1: gas_epoch)."""
        assert self.kind == "go"
        loss = f64()
        if self.owner.lib.go_session_dp_epoch(self.h, epoch, int(shuffle), int(k), C.byref(loss)):
            raise ValueError("go_session_dp_epoch failed")
        return loss.value

    def dp_batch(self, part, nb):
        """(grads, acts[(L-1), nb, hd], loss, stepped) against the current params/histories; no push, no step."""
        assert self.kind == "go"
        g = np.zeros(self.nparam, np.float32)
        acts = np.zeros((max(self.spec.num_layers - 1, 0), nb, self.hist_dim), np.float32)
        loss, st = f64(), C.c_int()
        if self.owner.lib.go_session_dp_batch(self.h, int(part), _p(g), _p(acts) if acts.size else None,
                                              C.byref(loss), C.byref(st)):
            raise ValueError("go_session_dp_batch failed")
        return g, acts, loss.value, bool(st.value)

    def dp_commit(self, part, acts):
        a = np.ascontiguousarray(acts, np.float32)
        self.owner.lib.go_session_dp_commit(self.h, int(part), _p(a) if a.size else None)

    def dp_apply(self, grad_sum, count, batches):
        g = np.ascontiguousarray(grad_sum, np.float32)
        self.owner.lib.go_session_dp_apply(self.h, _p(g), int(count), int(batches))

