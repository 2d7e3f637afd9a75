"""Data-parallel GAS training over the GPUs of one node, one process per GPU.

The exchange (gradient all-reduce, history-push commit, cross-rank barriers) runs in
libgasb.so over peer memory (dp.cu); torch.distributed is only the control plane that
all-gathers the ranks' CUDA IPC handles once and combines the per-part losses.

Step semantics: the oracle's go_session_dp_epoch (oracle/gas_oracle.c) — k consecutive
batches of gas_epoch's seeded order per step (trainer.cpp:395-400), rank j runs the j-th,
start-of-step parameters and histories, pushes committed after the step, gradients summed
in rank order over the batches with training rows and divided by their count.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import DP_HANDLE_BYTES, check, i64, lib, ptr, vp
from .trainer import GasTrainer


def epoch_order(num_parts: int, seed: int, epoch: int, shuffle: bool = True) -> np.ndarray:
    """gas_epoch's batch order (trainer.cpp:395-400)."""
    out = np.empty(num_parts, np.int32)
    check(lib.gasb_epoch_order(int(num_parts), int(seed), int(epoch), int(shuffle), ptr(out)))
    return out


def step_plan(num_parts: int, seed: int, epoch: int, world: int, shuffle: bool = True) -> np.ndarray:
    """[steps, world] part run by each rank in each step (-1: idle in a short last step)."""
    order = epoch_order(num_parts, seed, epoch, shuffle)
    steps = -(-num_parts // world)
    plan = np.full((steps, world), -1, np.int32)
    plan.reshape(-1)[:num_parts] = order
    return plan


class DataParallelTrainer:
    """Wraps a GasTrainer as rank `rank` of `world`. `group`: a torch.distributed process
    group (any backend) used to all-gather the IPC handles and to sum the per-part losses;
    None for world == 1."""

    PLACEMENTS = {"replicated": 0, "sharded": 1}

    def __init__(self, trainer: GasTrainer, rank: int, world: int, group=None, placement: str = "replicated"):
        """placement: "replicated" (every rank holds every history row) or "sharded" (rank j
        holds the rows of partitions p with p mod world == j; halo rows are read from the
        owners over NVLink, the step's rows are committed to their owners; gasb.h)."""
        self.trainer = trainer
        self.rank, self.world, self.group = rank, world, group
        self.placement = placement
        h = vp()
        check(lib.gasb_dp_create_ex(trainer._h, int(rank), int(world), self.PLACEMENTS[placement], C.byref(h)))
        self._h = h
        if world > 1:
            import torch.distributed as dist
            mine = np.zeros(DP_HANDLE_BYTES, np.uint8)
            check(lib.gasb_dp_export(self._h, ptr(mine)))
            got = [None] * world
            dist.all_gather_object(got, bytes(mine), group=group)
            handles = np.frombuffer(b"".join(got), np.uint8).copy()
            check(lib.gasb_dp_connect(self._h, ptr(handles)))
        self.num_parts = trainer.schedule.num_parts

    def __del__(self):
        if getattr(self, "_h", None):
            lib.gasb_dp_destroy(self._h)
            self._h = None

    def epoch_async(self, epoch: int, shuffle: bool = True) -> None:
        check(lib.gasb_dp_epoch_async(self._h, int(epoch), int(shuffle)))

    def check(self) -> None:
        check(lib.gasb_dp_check(self._h))

    def part_losses(self) -> np.ndarray:
        """Every part's loss of the last epoch (0 for parts without training rows)."""
        out = np.zeros(self.num_parts, np.float64)
        check(lib.gasb_dp_last_losses(self._h, ptr(out)))
        if self.world > 1:
            import torch
            import torch.distributed as dist
            t = torch.from_numpy(out)
            if dist.get_backend(self.group) == "nccl":
                t = t.cuda()
            dist.all_reduce(t, group=self.group)  # one non-zero entry per part: exact
            out = t.cpu().numpy()
        return out

    def gas_epoch(self, epoch: int, shuffle: bool = True) -> float:
        """One data-parallel epoch; EpochReport.loss = mean over the stepped parts in epoch order."""
        self.epoch_async(epoch, shuffle)
        self.check()
        losses = self.part_losses()
        order = epoch_order(self.num_parts, self.trainer.spec.seed, epoch, shuffle)
        train = self.trainer.part_train_rows()
        stepped = [p for p in order if train[p] > 0]
        return float(sum(losses[p] for p in stepped) / len(stepped)) if stepped else 0.0

    def launch_count(self) -> int:
        n = i64()
        check(lib.gasb_dp_launch_count(self._h, C.byref(n)))
        return n.value

    def history_layer(self, layer: int) -> np.ndarray:
        """History layer `layer` (n x hist_dim): the trainer's table when replicated, gathered
        from every rank's shard when sharded."""
        if self.placement == "replicated":
            return self.trainer.history.layer_matrix(layer)
        n = len(self.trainer.train_mask)
        hd = self.trainer.num_classes if self.trainer.spec.kind == "appnp" else self.trainer.spec.hidden
        out = np.empty((n, hd), np.float32)
        check(lib.gasb_dp_read_history(self._h, int(layer), ptr(out)))
        return out

    def traffic(self) -> dict:
        """Bytes of the last epoch (gasb_dp_traffic): NVLink (peer gradients, peer act rows,
        halo rows from peer shards), halo rows from this rank's own shard, rows held per layer."""
        a, b, c = i64(), i64(), i64()
        check(lib.gasb_dp_traffic(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"nvlink_bytes": a.value, "local_pull_bytes": b.value, "shard_rows": c.value}


def shard_map(schedule, world: int) -> tuple[np.ndarray, np.ndarray]:
    """The sharded placement's row ownership: (owner[n], row-in-owner's-shard[n]), rows per rank."""
    n = schedule.graph.num_nodes
    ol = np.empty(n, np.uint32)
    rows = np.empty(world, np.int64)
    check(lib.gasb_dp_shard_map(schedule.handle, int(world), ptr(ol), ptr(rows)))
    return (ol >> 29).astype(np.int32), (ol & ((1 << 29) - 1)).astype(np.int64), rows
