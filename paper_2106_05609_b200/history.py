"""HistoryStore / Prefetcher (include/gas/history.hpp:29-111) with HBM-resident tables.

Host-buffer methods (`push`, `pull`) keep the reference's span-based signatures and
exceptions; `push_device` / `pull_device` take device tensors (torch CUDA tensors, or raw
device pointers) and are stream-ordered."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import check, i32, i64, lib, ptr, u64, vp


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


class HistoryStore:
    def __init__(self, num_layers: int, num_nodes: int, dim: int, *, _handle=None, _owned=True):
        if _handle is None:
            h = vp()
            check(lib.gasb_history_create(int(num_layers), int(num_nodes), int(dim), C.byref(h)))
            _handle = h.value
        self._h = vp(_handle)
        self._owned = _owned
        L, n, d, ld = i32(), i32(), i32(), i64()
        check(lib.gasb_history_info(self._h, C.byref(L), C.byref(n), C.byref(d), C.byref(ld)))
        self._layers, self._n, self._dim, self.ld = L.value, n.value, d.value, ld.value

    def __del__(self):
        if getattr(self, "_h", None) and self._owned:
            lib.gasb_history_destroy(self._h)
        self._h = None

    @property
    def handle(self):
        return self._h

    def num_layers(self) -> int:
        return self._layers

    def num_nodes(self) -> int:
        return self._n

    def dim(self) -> int:
        return self._dim

    # ---- reference-shaped API (host spans) ----
    def push(self, layer: int, node_ids, embeddings) -> None:
        ids = np.ascontiguousarray(node_ids, dtype=np.int32)
        emb = np.ascontiguousarray(embeddings, dtype=np.float32)
        if emb.size != ids.size * self._dim:
            raise ValueError("HistoryStore::push: row count mismatch")
        check(lib.gasb_history_push_host(self._h, int(layer), ptr(ids), len(ids), ptr(emb), None))

    def pull(self, layer: int, node_ids) -> np.ndarray:
        ids = np.ascontiguousarray(node_ids, dtype=np.int32)
        out = np.empty((len(ids), self._dim), np.float32)
        check(lib.gasb_history_pull_host(self._h, int(layer), ptr(ids), len(ids), ptr(out), None))
        return out

    # ---- device API ----
    def push_device(self, layer: int, d_ids, count: int, d_rows, ld_rows: int, stream=None) -> None:
        check(lib.gasb_history_push(self._h, int(layer), ptr(d_ids) if hasattr(d_ids, "data_ptr") else d_ids, count,
                                    ptr(d_rows) if hasattr(d_rows, "data_ptr") else d_rows, ld_rows,
                                    _stream_ptr(stream)))

    def pull_device(self, layer: int, d_ids, count: int, d_out, ld_out: int, stream=None) -> None:
        check(lib.gasb_history_pull(self._h, int(layer), ptr(d_ids) if hasattr(d_ids, "data_ptr") else d_ids, count,
                                    ptr(d_out) if hasattr(d_out, "data_ptr") else d_out, ld_out, _stream_ptr(stream)))

    def check(self) -> None:
        check(lib.gasb_history_check(self._h))

    def layer_matrix(self, layer: int) -> np.ndarray:
        out = np.empty((self._n, self._dim), np.float32)
        check(lib.gasb_history_read_layer(self._h, int(layer), ptr(out)))
        return out

    def layer_pointer(self, layer: int) -> tuple[int, int]:
        p, ld = vp(), i64()
        check(lib.gasb_history_layer(self._h, int(layer), C.byref(p), C.byref(ld)))
        return p.value, ld.value

    def fill_layer(self, layer: int, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.shape != (self._n, self._dim):
            raise ValueError("HistoryStore::fill_layer: shape mismatch")
        check(lib.gasb_history_fill_layer(self._h, int(layer), ptr(v)))

    def advance_step(self, stream=None) -> None:
        check(lib.gasb_history_advance_step(self._h, _stream_ptr(stream)))

    def step(self) -> int:
        s = i64()
        check(lib.gasb_history_step(self._h, C.byref(s)))
        return s.value

    def last_push_step(self, layer: int, v: int) -> int:
        s = i64()
        check(lib.gasb_history_last_push_step(self._h, int(layer), int(v), C.byref(s)))
        return s.value

    def stamps(self, layer: int) -> np.ndarray:
        out = np.empty(self._n, np.int64)
        check(lib.gasb_history_read_stamps(self._h, int(layer), ptr(out)))
        return out

    def reset(self) -> None:
        check(lib.gasb_history_reset(self._h))

    def measure_staleness(self, reference) -> list[dict]:
        """measure_staleness (history.cpp:77-112): one reference matrix per layer (host arrays
        n x dim, or CUDA tensors); per layer eps_max / eps_mean / age_max / age_mean."""
        if len(reference) != self._layers:
            raise ValueError("measure_staleness: need one reference matrix per layer")
        import torch  # device staging of host references (plumbing)
        dev = []
        for r in reference:
            t = r if hasattr(r, "data_ptr") else torch.from_numpy(np.ascontiguousarray(r, np.float32))
            if tuple(t.shape) != (self._n, self._dim):
                raise ValueError("measure_staleness: reference shape mismatch")
            dev.append(t.cuda().contiguous())
        L = self._layers
        ptrs = (C.c_void_p * max(L, 1))(*[t.data_ptr() for t in dev])
        lds = np.array([self._dim] * max(L, 1), np.int64)
        emax, emean, amean = (np.zeros(max(L, 1)) for _ in range(3))
        amax = np.zeros(max(L, 1), np.int64)
        check(lib.gasb_history_staleness(self._h, ptrs, ptr(lds), ptr(emax), ptr(emean), ptr(amax), ptr(amean)))
        return [dict(eps_max=float(emax[l]), eps_mean=float(emean[l]), age_max=int(amax[l]),
                     age_mean=float(amean[l])) for l in range(L)]

    def save_checkpoint(self, path: str) -> None:
        """save_checkpoint (history.cpp:130-148): the reference's GASH format."""
        check(lib.gasb_history_save(self._h, str(path).encode()))

    @staticmethod
    def load_checkpoint(path: str) -> "HistoryStore":
        """load_checkpoint (history.cpp:150-178): new store, stamps 0, step 0."""
        h = vp()
        check(lib.gasb_history_load(str(path).encode(), C.byref(h)))
        return HistoryStore(0, 0, 0, _handle=h.value)


class PrefetchHandle:
    def __init__(self, owner: "Prefetcher", generation: int, stream):
        self._owner, self._generation, self._stream = owner, generation, stream

    def wait(self, layer: int) -> tuple[int, int]:
        """Orders the compute stream after layer's snapshot; returns (device ptr, ld)."""
        return self._owner._wait(self._generation, layer, self._stream)


class Prefetcher:
    def __init__(self, store: HistoryStore):
        self.store = store
        h = vp()
        check(lib.gasb_prefetcher_create(store.handle, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.gasb_prefetcher_destroy(self._h)
            self._h = None

    def begin(self, d_halo, count: int, stream=None) -> PrefetchHandle:
        gen = u64()
        check(lib.gasb_prefetch_begin(self._h, ptr(d_halo) if hasattr(d_halo, "data_ptr") else d_halo, count,
                                      _stream_ptr(stream), C.byref(gen)))
        return PrefetchHandle(self, gen.value, stream)

    def _wait(self, generation: int, layer: int, stream):
        p, ld = vp(), i64()
        check(lib.gasb_prefetch_wait(self._h, generation, int(layer), _stream_ptr(stream), C.byref(p), C.byref(ld)))
        return p.value, ld.value
