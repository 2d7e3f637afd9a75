"""GAS trainer (reference: include/gas/trainer.hpp — ModelSpec, Model, gas_epoch) over the
C ABI. All compute runs in libgasb.so on the GPU; this module only marshals arguments."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._native import EpochReportC, ModelSpecC, TrainerOptionsC, check, f64, i32, i64, lib, ptr, vp  # noqa: F401
from .graph import BatchSchedule
from .history import HistoryStore

KINDS = {"gcn": 0, "gin": 1, "appnp": 2, "gcnii": 3}


@dataclass
class AdamConfig:  # include/gas/nn.hpp:11-16
    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


@dataclass
class ModelSpec:  # include/gas/trainer.hpp:16-33 (GIN / Lipschitz fields are out of scope)
    kind: str = "gcn"
    num_layers: int = 2
    hidden: int = 16
    dropout: float = 0.0
    alpha: float = 0.1
    beta: float = 0.5
    l2_weight: float = 0.0
    clip_max_norm: float = 0.0
    opt: AdamConfig = field(default_factory=AdamConfig)
    seed: int = 0

    def to_c(self) -> ModelSpecC:
        return ModelSpecC(KINDS[self.kind], self.num_layers, self.hidden, self.dropout, self.alpha, self.beta,
                          self.l2_weight, self.clip_max_norm, self.opt.lr, self.opt.beta1, self.opt.beta2,
                          self.opt.eps, self.seed)


@dataclass
class TrainerOptions:
    seg_edges: int = 128      # SpMM row segmentation (0 = sequential rows, bit-exact)
    fused: bool = True        # pull-free SpMM over in-place histories
    prefetch: bool = False
    use_graphs: bool = True
    hoist_layer1: bool = True
    device: int = 0
    dropout_rng: str = "exact"  # "exact" (the reference's mt19937_64 masks) or "philox" (gasb.h)
    cross_batch: int = 0      # 1: batch b+1's halo aggregation overlapped with batch b (gasb.h); 2: + layer 1

    def to_c(self) -> TrainerOptionsC:
        return TrainerOptionsC(self.seg_edges, int(self.fused), int(self.prefetch), int(self.use_graphs),
                               int(self.hoist_layer1), self.device, {"exact": 0, "philox": 1}[self.dropout_rng],
                               int(self.cross_batch))


class GasTrainer:
    """Model + AdamState + HistoryStore on one GPU, driven by gas_epoch."""

    def __init__(self, schedule: BatchSchedule, features: np.ndarray, labels: np.ndarray, train_mask: np.ndarray,
                 num_classes: int, spec: ModelSpec, options: TrainerOptions | None = None):
        x = np.ascontiguousarray(features, dtype=np.float32)
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        tm = np.ascontiguousarray(train_mask, dtype=np.uint8)
        self.schedule = schedule
        self.spec = spec
        self.options = options or TrainerOptions()
        s, o = spec.to_c(), self.options.to_c()
        h = vp()
        check(lib.gasb_trainer_create(schedule.handle, ptr(x), x.shape[1], ptr(lab), ptr(tm), int(num_classes),
                                      C.byref(s), C.byref(o), C.byref(h)))
        self._h = h
        n = i64()
        check(lib.gasb_trainer_num_param_floats(self._h, C.byref(n)))
        self.num_param_floats = n.value
        hh = vp()
        check(lib.gasb_trainer_history(self._h, C.byref(hh)))
        self.history = HistoryStore(0, 0, 0, _handle=hh.value, _owned=False) if spec.num_layers >= 1 else None
        self.num_classes = num_classes
        self._in_dim = x.shape[1]
        self.train_mask = tm.astype(bool)
        self._part_train = None

    def part_train_rows(self) -> np.ndarray:
        """Training rows per part (parts without any take no optimizer step, trainer.cpp:313-317)."""
        if self._part_train is None:
            self._part_train = np.array([int(self.train_mask[self.schedule.batch_nodes(p)].sum())
                                         for p in range(self.schedule.num_parts)], np.int64)
        return self._part_train

    def __del__(self):
        if getattr(self, "_h", None):
            self.history = None
            lib.gasb_trainer_destroy(self._h)
            self._h = None

    def gas_epoch(self, epoch: int, shuffle: bool = True) -> float:
        loss = f64()
        check(lib.gasb_gas_epoch(self._h, int(epoch), int(shuffle), C.byref(loss)))
        return loss.value

    def gas_epoch_async(self, epoch: int, shuffle: bool = True) -> None:
        check(lib.gasb_gas_epoch_async(self._h, int(epoch), int(shuffle)))

    def gas_epoch_range_async(self, epoch: int, begin: int, end: int, shuffle: bool = True) -> None:
        """Batches order[begin:end] of gas_epoch's seeded order (same kernels and graphs)."""
        check(lib.gasb_gas_epoch_range_async(self._h, int(epoch), int(shuffle), int(begin), int(end)))

    def dropout_mask(self, part: int, epoch: int, layer: int) -> np.ndarray:
        """Keep mask (bool, V_b x d_{layer-1}) of the layer-`layer` input dropout of batch `part`."""
        ne = int(self.schedule.sizes(part)[1])
        d = self._in_dim if layer == 1 else (self.num_classes if self.spec.kind == "appnp" else self.spec.hidden)
        words = np.zeros((ne * d + 31) // 32, np.uint32)
        check(lib.gasb_trainer_dropout_mask(self._h, int(part), int(epoch), int(layer), ptr(words)))
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:ne * d]
        return bits.reshape(ne, d).astype(bool)

    def part_losses(self) -> np.ndarray:
        """Per-part batch objective as last computed (part order)."""
        out = np.zeros(self.schedule.num_parts, np.float64)
        check(lib.gasb_trainer_part_losses(self._h, ptr(out)))
        return out

    def gas_epoch_report(self, epoch: int, shuffle: bool = True, measure_staleness: bool = False) -> dict:
        """gas_epoch returning EpochReport's fields (trainer.hpp:107-115; gasb.h explains
        batch_peak_floats); measure_staleness runs the frozen snapshot pass (trainer.cpp:434-438)."""
        r = EpochReportC()
        bp = np.zeros(self.schedule.num_parts, np.int64)
        eps = np.zeros(max(self.spec.num_layers - 1, 1), np.float64)
        check(lib.gasb_gas_epoch_report(self._h, int(epoch), int(shuffle), int(measure_staleness), C.byref(r),
                                        ptr(bp), ptr(eps)))
        return dict(epoch=r.epoch, loss=r.loss, peak_floats=r.peak_floats, edges_per_layer=r.edges_per_layer,
                    device_bytes=r.device_bytes, batch_peak_floats=bp[:r.num_batches],
                    eps_max=eps[:r.staleness_layers])

    def last_loss(self) -> float:
        loss = f64()
        check(lib.gasb_trainer_last_loss(self._h, C.byref(loss)))
        return loss.value

    def launch_count(self) -> int:
        n = i64()
        check(lib.gasb_trainer_launch_count(self._h, C.byref(n)))
        return n.value

    def stream(self) -> int:
        s = vp()
        check(lib.gasb_trainer_stream(self._h, C.byref(s)))
        return s.value or 0

    def batch(self, part: int, epoch: int = 0, train: bool = True, push: bool = True):
        """One batch with capture: (acts[(L-1), nb, hd], logits[nb, C], loss, grads|None, stepped)."""
        nb = int(self.schedule.sizes(part)[0])
        L = self.spec.num_layers
        hd = self.num_classes if self.spec.kind == "appnp" else self.spec.hidden  # Model::history_dim
        acts = np.zeros((max(L - 1, 0), nb, hd), np.float32)
        logits = np.zeros((nb, self.num_classes), np.float32)
        grads = np.zeros(self.num_param_floats, np.float32)
        loss, stepped = f64(), i32()
        check(lib.gasb_trainer_batch(self._h, int(part), int(epoch), int(train), int(push), ptr(acts) if acts.size else
                                     None, ptr(logits), C.byref(loss), ptr(grads), C.byref(stepped)))
        return acts, logits, loss.value, (grads if stepped.value else None), bool(stepped.value)

    def set_features(self, features: np.ndarray) -> None:
        x = np.ascontiguousarray(features, dtype=np.float32)
        check(lib.gasb_trainer_set_features(self._h, ptr(x)))

    def stage_features(self, features: np.ndarray) -> None:
        """Asynchronous H2D of the next step's features (page-locked host memory) on the copy
        stream; the array must stay alive and unmodified until commit_features ran."""
        check(lib.gasb_trainer_stage_features(self._h, ptr(features)))

    def commit_features(self) -> None:
        """Installs the staged features as X (stream-ordered before the next epoch)."""
        check(lib.gasb_trainer_commit_features(self._h))

    def profile_spmm(self, part: int, layer: int, iters: int = 5) -> float:
        ms = C.c_float()
        check(lib.gasb_trainer_profile_spmm(self._h, int(part), int(layer), int(iters), C.byref(ms)))
        return ms.value

    def evaluate(self, train_mask=None, val_mask=None, test_mask=None) -> tuple[float, float, float]:
        """evaluate (trainer.cpp:444-464): full-batch accuracy (train, val, test); the train
        mask defaults to the trainer's."""
        masks = [np.ascontiguousarray(m, np.uint8) if m is not None else None
                 for m in (self.train_mask if train_mask is None else train_mask, val_mask, test_mask)]
        acc = np.zeros(3)
        check(lib.gasb_trainer_evaluate(self._h, *[ptr(m) for m in masks], ptr(acc)))
        return float(acc[0]), float(acc[1]), float(acc[2])

    def full_logits(self) -> np.ndarray:
        """Logits (n x C, global order) of the last evaluate / infer_from_history."""
        out = np.empty((len(self.train_mask), self.num_classes), np.float32)
        check(lib.gasb_trainer_full_logits(self._h, ptr(out)))
        return out

    def infer_from_history(self) -> tuple[np.ndarray, bool]:
        """infer_from_history (trainer.cpp:501-536): (predictions, stale)."""
        pred = np.empty(len(self.train_mask), np.int32)
        st = i32()
        check(lib.gasb_trainer_infer_from_history(self._h, ptr(pred), C.byref(st)))
        return pred, bool(st.value)

    def get_params(self) -> np.ndarray:
        out = np.empty(self.num_param_floats, np.float32)
        check(lib.gasb_trainer_get_params(self._h, ptr(out)))
        return out

    def set_params(self, values: np.ndarray) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32)
        check(lib.gasb_trainer_set_params(self._h, ptr(v)))


def adam_step(params, m, v, grads, step: int, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8, stream=None) -> None:
    """AdamState::step (nn.cpp:20-41) in place on device tensors (torch CUDA float32)."""
    check(lib.gasb_adam_step(ptr(params), ptr(m), ptr(v), ptr(grads), int(params.numel()), int(step), lr, beta1,
                             beta2, eps, stream))


def grad_clip(grads, max_norm: float, stream=None) -> float:
    """grad_clip (nn.cpp:47-63) in place on a device tensor; returns the pre-clip norm."""
    nn = f64()
    check(lib.gasb_grad_clip(ptr(grads), int(grads.numel()), float(max_norm), C.byref(nn), stream))
    return nn.value
