"""The bench input generator: the oracle's restatement (used by bench.py's reference arm,
which must not load libgasb.so) produces the product's graph, features, labels and masks bit
for bit; features carry a learnable class signal."""
import numpy as np
import pytest

from paper_2106_05609_b200.workloads import WORKLOADS, make_dataset
from pyoracle import OracleSynth


@pytest.mark.parametrize("name", ["cora", "reddit_mini", "products_mini", "pubmed_gcnii"])
def test_oracle_generator_matches_product(name):
    a = make_dataset(name)
    b = make_dataset(name, backend=OracleSynth())
    for k in ("row_offsets", "cols", "features", "labels", "train_mask", "assignment"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_features_carry_class_signal():
    ds = make_dataset("reddit_mini")
    w = ds.workload
    assert w.signal > 0
    means = np.stack([ds.features[ds.labels == c].mean(0) for c in np.unique(ds.labels)])
    # class means differ by ~signal * N(0,1) per dimension; noise of the mean is ~1/sqrt(count)
    spread = means.std(0).mean()
    assert spread > 0.5 * w.signal


def test_down_scaled_shapes_follow_their_full_configs():
    for small, big in (("products_mini", "products_appnp"), ("papers_mini", "papers100m")):
        s, b = WORKLOADS[small], WORKLOADS[big]
        assert (s.in_dim, s.num_classes, s.kind, s.num_layers, s.hidden, s.intra_fraction) == \
               (b.in_dim, b.num_classes, b.kind, b.num_layers, b.hidden, b.intra_fraction)
        assert abs(s.num_pairs / s.num_nodes - b.num_pairs / b.num_nodes) / (b.num_pairs / b.num_nodes) < 0.01
