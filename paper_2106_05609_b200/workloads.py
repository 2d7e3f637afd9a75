"""Synthetic workloads of BASELINE.json `configs`.

One seeded generator (power-law weights + planted communities, include/gasb.h
gasb_synth_pairs) feeds BOTH the B200 path and the CPU oracles; the CSR goes through
build_graph semantics on both sides, so the stored graph is identical. The planted
communities are the partition (the reference's own bench uses the natural partition,
tools/gas_main.cpp:251-254). Calibrated here (stored nnz / inter-intra ratio):

  C1 cora     n=2,708    nnz=10,554  ratio 0.150 (paper METIS Cora 0.14)   10 parts
  C2 pubmed   n=19,717   nnz=88,722  ratio 0.215                          8 parts
  C3 reddit   n=232,965  nnz=114.23M ratio 2.800 (paper METIS Reddit 2.80) 200 parts,
              mean degree 490.4 (Reddit 492), max degree 14.3K
  C4 products n=2.45M    nnz=122.5M  ratio 1.938 (paper METIS products 1.94) 100 parts

Labels = community mod C; each partition is `comm_per_part` planted communities (so a batch
holds several labels, as a METIS part of real Reddit does, instead of one). Features = N(0,1)
noise + `signal` x the label's centroid (a seeded N(0,1) vector per class), so the labels
are learnable and the trained network stays live. Round 1 used one community per part and
pure-noise features: every batch had a single label and the bias-free 4-layer GCN at C3
collapsed to all-dead ReLUs (loss exactly ln C); profiles/r2_c3_dynamics_probe.txt has the
variants measured on the GPU. Train mask: seeded 66% of nodes.

This module is data-only at import time: `make_dataset` takes a generator backend, the
product library's by default. bench.py's reference arm loads this file by path and passes
the oracle's restatement of the same generator (oracle/pyoracle.py OracleSynth), so the
reference arm never loads libgasb.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    num_nodes: int
    num_pairs: int
    parts: int
    intra_fraction: float
    max_weight: float
    in_dim: int
    num_classes: int
    kind: str
    num_layers: int
    hidden: int
    seed: int = 1
    train_frac: float = 0.66
    signal: float = 0.5  # centroid scale in the features (0 = pure noise, round-1 data)
    comm_per_part: int = 4  # planted communities per partition (labels = community mod C)
    lr: float = 0.01  # Adam learning rate of the workload's model (AdamConfig default 0.01)


WORKLOADS = {
    "cora": Workload("cora", 2708, 6150, 10, 0.88, 60.0, 1433, 7, "gcn", 2, 16),
    "pubmed_gcnii": Workload("pubmed_gcnii", 19717, 45700, 8, 0.8, 60.0, 500, 3, "gcnii", 64, 64),
    # lr 1e-3: at the AdamConfig default (1e-2) the bias-free 4-layer GCN diverges on this data
    # (profiles/r2_c3_dynamics_probe.txt: loss 3.2 -> 148 in 12 epochs; 1e-3: 3.4 -> 0.15)
    "reddit": Workload("reddit", 232965, 82_000_000, 200, 0.475, 120.0, 602, 41, "gcn", 4, 256, lr=1e-3),
    # C4: ogbn-products shape (61.9M raw undirected edges -> ~123.7M stored nnz), APPNP with
    # K = 3 propagation layers over 47-wide histories, inter/intra ~1.94
    "products_appnp": Workload("products_appnp", 2449029, 61_859_140, 100, 0.34, 120.0, 100, 47, "appnp", 3, 256),
    # C5: ogbn-papers100M shape (111M nodes, 1.6B raw edges -> ~3.2B stored nnz), GCN L = 3,
    # F = 128, 172 classes; needs the sharded history placement across GPUs
    "papers100m": Workload("papers100m", 111_059_956, 1_615_685_872, 8192, 0.5, 2000.0, 128, 172, "gcn", 3, 256),
    # down-scaled shapes for fast parity runs
    "cora_appnp": Workload("cora_appnp", 2708, 6150, 10, 0.88, 60.0, 1433, 7, "appnp", 3, 64),
    "cora_gcnii": Workload("cora_gcnii", 2708, 6150, 10, 0.88, 60.0, 1433, 7, "gcnii", 8, 64),
    "reddit_mini": Workload("reddit_mini", 12000, 1_200_000, 12, 0.4, 60.0, 602, 41, "gcn", 4, 256),
    # C4 down-scaled: the products_appnp generator parameters (F, C, h, K, intra, weights)
    # at 50K nodes and the same mean degree (~50), 20 parts (~2.5K-node batches)
    "products_mini": Workload("products_mini", 50_000, 1_262_840, 20, 0.34, 120.0, 100, 47, "appnp", 3, 256),
    # C5 down-scaled: the papers100m generator parameters at 200K nodes, same mean degree
    # (~29), 16 parts
    "papers_mini": Workload("papers_mini", 200_000, 2_909_600, 16, 0.5, 2000.0, 128, 172, "gcn", 3, 256),
}


@dataclass
class Dataset:
    workload: Workload
    graph: object
    row_offsets: np.ndarray
    cols: np.ndarray
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    assignment: np.ndarray


class ProductSynth:
    """The generator as the product library exports it (gasb_synth_*, gasb_graph_build)."""

    def synth_pairs(self, w: Workload):
        from .graph import synth_pairs
        return synth_pairs(w.num_nodes, w.num_pairs, w.parts * w.comm_per_part, w.intra_fraction, gamma=2.5,
                           min_weight=1.0,
                           max_weight=w.max_weight, seed=w.seed)

    def build_graph(self, edges, n):
        from .graph import build_graph
        g = build_graph(edges, n, symmetrize=True)
        ro, co = g.csr()
        return g, ro, co

    def synth_features(self, n, dim, seed):
        from .graph import synth_features
        return synth_features(n, dim, seed=seed)


def add_signal(x: np.ndarray, labels: np.ndarray, centroids: np.ndarray, signal: float) -> np.ndarray:
    """x += signal * centroids[label], in place, in row blocks (fp32, one rounding each)."""
    if signal == 0.0:
        return x
    c = (np.float32(signal) * centroids.astype(np.float32)).astype(np.float32)
    step = 1 << 16
    for r0 in range(0, len(x), step):
        x[r0:r0 + step] += c[labels[r0:r0 + step]]
    return x


def make_dataset(w: Workload | str, with_features: bool = True, backend=None) -> Dataset:
    if isinstance(w, str):
        w = WORKLOADS[w]
    be = backend or ProductSynth()
    edges, comm = be.synth_pairs(w)
    g, ro, co = be.build_graph(edges, w.num_nodes)
    del edges
    rng = np.random.default_rng(w.seed + 2)
    labels = (comm % w.num_classes).astype(np.int32)
    part = (comm // w.comm_per_part).astype(np.int32)  # comm = rank mod K: parts stay balanced
    train = (rng.random(w.num_nodes) < w.train_frac).astype(np.uint8)
    x = None
    if with_features:
        x = be.synth_features(w.num_nodes, w.in_dim, w.seed + 1)
        if w.signal:
            add_signal(x, labels, be.synth_features(w.num_classes, w.in_dim, w.seed + 3), w.signal)
    return Dataset(w, g, ro, co, x, labels, train, part)
