"""B200-native GNNAutoScale (GAS) training hot path.

History tables in HBM, pull/push and message passing as sm_100a kernels, per-batch CUDA
graphs — behind the reference's operator surface (include/gas/{graph,history,trainer}.hpp).
The native library is libgasb.so (C ABI: include/gasb.h); importing this package fails
loudly when it has not been built.
"""
from ._native import LIB_PATH, lib  # noqa: F401  (raises ImportError when unbuilt)
from .graph import (BatchPlan, BatchSchedule, Graph, build_graph, cluster_partition, graph_from_csr,  # noqa: F401
                    make_batch_plan,
                    load_partition, partition_parts, random_partition, save_partition, synth_features,
                    synth_pairs)
from .history import HistoryStore, Prefetcher, PrefetchHandle  # noqa: F401
from .trainer import AdamConfig, GasTrainer, ModelSpec, TrainerOptions, adam_step, grad_clip  # noqa: F401
from .layers import BatchOps, LayerConfig, layer_backward, layer_forward  # noqa: F401
from .dp import DataParallelTrainer, epoch_order, shard_map, step_plan  # noqa: F401

__all__ = [
    "Graph", "build_graph", "graph_from_csr", "make_batch_plan", "BatchPlan", "BatchSchedule", "partition_parts",
    "synth_pairs", "synth_features", "cluster_partition", "save_partition", "load_partition", "random_partition", "HistoryStore", "Prefetcher", "PrefetchHandle", "ModelSpec", "AdamConfig",
    "TrainerOptions", "GasTrainer", "adam_step", "grad_clip", "BatchOps", "LayerConfig", "layer_forward",
    "layer_backward", "DataParallelTrainer", "epoch_order", "step_plan", "shard_map",
]
