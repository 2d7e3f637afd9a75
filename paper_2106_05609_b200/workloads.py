"""Synthetic workloads of BASELINE.json `configs`.

One seeded generator (power-law weights + planted communities, include/gasb.h
gasb_synth_pairs) feeds BOTH the B200 path and the CPU oracles; the CSR goes through
build_graph semantics on both sides, so the stored graph is identical. The planted
communities are the partition (the reference's own bench uses the natural partition,
tools/gas_main.cpp:251-254). Calibrated here (stored nnz / inter-intra ratio):

  C1 cora     n=2,708    nnz≈10.5K  ratio≈0.15 (paper METIS Cora 0.14)   10 parts
  C2 pubmed   n=19,717   nnz≈88.6K  ratio≈0.21                           8 parts
  C3 reddit   n=232,965  nnz=114.97M ratio=2.82 (paper METIS Reddit 2.80) 200 parts,
              mean degree 493.5 (Reddit 492), max degree 15.2K
Labels = community mod C (learnable); train mask: seeded 66% of nodes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import build_graph, synth_features, synth_pairs


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


WORKLOADS = {
    "cora": Workload("cora", 2708, 5570, 10, 0.87, 60.0, 1433, 7, "gcn", 2, 16),
    "pubmed_gcnii": Workload("pubmed_gcnii", 19717, 44700, 8, 0.8, 60.0, 500, 3, "gcnii", 64, 64),
    "reddit": Workload("reddit", 232965, 65_300_000, 200, 0.335, 120.0, 602, 41, "gcn", 4, 256),
    # C4: ogbn-products shape (61.9M raw undirected edges -> ~123.7M stored nnz), APPNP with
    # K = 3 propagation layers over 47-wide histories, inter/intra ~1.94
    "products_appnp": Workload("products_appnp", 2449029, 61_859_140, 100, 0.34, 120.0, 100, 47, "appnp", 3, 256),
    # down-scaled shapes for fast parity runs
    "cora_appnp": Workload("cora_appnp", 2708, 5570, 10, 0.87, 60.0, 1433, 7, "appnp", 3, 64),
    "cora_gcnii": Workload("cora_gcnii", 2708, 5570, 10, 0.87, 60.0, 1433, 7, "gcnii", 8, 64),
    "reddit_mini": Workload("reddit_mini", 12000, 1_200_000, 12, 0.4, 60.0, 602, 41, "gcn", 4, 256),
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


def make_dataset(w: Workload | str, with_features: bool = True) -> Dataset:
    if isinstance(w, str):
        w = WORKLOADS[w]
    edges, comm = synth_pairs(w.num_nodes, w.num_pairs, w.parts, w.intra_fraction, gamma=2.5, min_weight=1.0,
                              max_weight=w.max_weight, seed=w.seed)
    g = build_graph(edges, w.num_nodes, symmetrize=True)
    del edges
    ro, co = g.csr()
    x = synth_features(w.num_nodes, w.in_dim, seed=w.seed + 1) if with_features else None
    rng = np.random.default_rng(w.seed + 2)
    labels = (comm % w.num_classes).astype(np.int32)
    train = (rng.random(w.num_nodes) < w.train_frac).astype(np.uint8)
    return Dataset(w, g, ro, co, x, labels, train, comm.astype(np.int32))
