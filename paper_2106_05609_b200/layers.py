"""Layer-level ops (reference: include/gas/layers.hpp:17-72, src/layers.cpp:120-168) over the
C ABI: Layer::forward over one batch plan and its tape backward, on device tensors (torch
CUDA float32, row-major with any row pitch). For callers that drive their own
Model::forward layer by layer; the fused trainer (trainer.py) does not go through here."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._native import LayerConfigC, check, i32, lib, ptr, vp
from .graph import BatchSchedule

KINDS = {"gcn": 0, "appnp": 2, "gcnii": 3}


@dataclass
class LayerConfig:  # layers.hpp:17-27 (GIN fields out of scope)
    kind: str = "gcn"
    in_dim: int = 0
    out_dim: int = 0
    alpha: float = 0.1
    beta: float = 0.5

    def to_c(self) -> LayerConfigC:
        return LayerConfigC(KINDS[self.kind], self.in_dim, self.out_dim, self.alpha, self.beta)


class BatchOps:
    """One plan's device stencils (gasb_batch_ops): the LayerContext{plan, agg} of a batch."""

    def __init__(self, schedule: BatchSchedule, part: int, max_dim: int):
        h = vp()
        check(lib.gasb_batch_ops_create(schedule.handle, int(part), int(max_dim), C.byref(h)))
        self._h = h
        self.schedule = schedule
        nb, ne = i32(), i32()
        check(lib.gasb_batch_ops_sizes(self._h, C.byref(nb), C.byref(ne)))
        self.num_batch, self.num_extended = nb.value, ne.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.gasb_batch_ops_destroy(self._h)
            self._h = None


def _ld(t):
    return int(t.stride(0)) if t is not None else 0


def layer_forward(ops: BatchOps, cfg: LayerConfig, h_in, out, saved, h0=None, w=None, stream=None) -> None:
    """Layer::forward: out (|B_b| x out_dim) from h_in (|V_b| x in_dim); `saved` receives what
    layer_backward needs."""
    c = cfg.to_c()
    check(lib.gasb_layer_fwd(ops._h, C.byref(c), ptr(h_in), _ld(h_in), ptr(h0), _ld(h0), ptr(w), _ld(w), ptr(out),
                             _ld(out), ptr(saved), _ld(saved), stream))


def layer_backward(ops: BatchOps, cfg: LayerConfig, gy, saved, scratch, w=None, gh_in=None, gh0=None, gw=None,
                   stream=None) -> None:
    """Tape backward of layer_forward; ACCUMULATES into gh_in / gh0 / gw (None = skipped)."""
    c = cfg.to_c()
    check(lib.gasb_layer_bwd(ops._h, C.byref(c), ptr(gy), _ld(gy), ptr(saved), _ld(saved), ptr(w), _ld(w),
                             ptr(gh_in), _ld(gh_in), ptr(gh0), _ld(gh0), ptr(gw), _ld(gw), ptr(scratch),
                             _ld(scratch), stream))
