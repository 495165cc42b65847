"""The native propagate port (csrc/propagate.cpp) reproduces the unmodified
reference's PGC chunk assignment (partition.py:200-270) exactly: same chunk
per instance, same chunk ids, on the C1 graph and on generated graphs covering
the recurrent / LSTM / EvolveGCN / attention profiles and binding size caps
(golden arrays from tools/make_propagate_golden.py)."""
import numpy as np
import pytest

from paper_2309_03523_b200.partition import chunk_ids, propagate_labels

CASES = ["c1_recurrent", "g3k_lstm", "g3k_evolve", "g2k_attention", "g2k_cap3", "g4k_cap40"]


@pytest.fixture(scope="module")
def golden(golden_dir):
    return np.load(golden_dir / "propagate.npz")


@pytest.mark.parametrize("name", CASES)
def test_native_propagate_equals_reference(golden, name):
    n, ts, cap, rounds = (int(x) for x in golden[f"{name}/meta"])
    labels, ran, colors = propagate_labels(n, golden[f"{name}/spatial"], golden[f"{name}/temporal"],
                                           ts, golden[f"{name}/tw"], cap, rounds)
    np.testing.assert_array_equal(chunk_ids(labels), golden[f"{name}/chunk_of"])
    assert 1 <= ran <= rounds and colors >= 1
    # the size cap holds for every chunk
    assert np.bincount(labels).max() <= cap


def test_native_propagate_edge_cases():
    # no edges: every instance keeps its own label (singleton chunks)
    labels, ran, _ = propagate_labels(5, np.empty((0, 2)), np.empty((0, 2)), 128, [], 3)
    np.testing.assert_array_equal(labels, np.arange(5))
    # size cap 1: nobody may join anybody
    se = np.array([[0, 1], [1, 2], [2, 3]])
    labels, _, _ = propagate_labels(4, se, np.empty((0, 2)), 128, [], 1)
    np.testing.assert_array_equal(labels, np.arange(4))
    # a path with cap 4 collapses into one chunk labelled by one of its members
    labels, _, _ = propagate_labels(4, se, np.empty((0, 2)), 128, [], 4)
    assert len(np.unique(labels)) == 1
    with pytest.raises(ValueError):
        propagate_labels(4, se, np.empty((0, 2)), 128, [], 0)
    with pytest.raises(ValueError):
        propagate_labels(4, np.array([[0, 9]]), np.empty((0, 2)), 128, [], 2)


@pytest.mark.parametrize("name,D", [("c2", 1), ("c3d8", 8)])
def test_native_propagate_equals_frozen_reference_plans(artifacts_dir, name, D):
    """At scale: the chunks of the reference planner's frozen C2 (200k, LSTM
    profile) and C3 (1M instances, EvolveGCN profile, D = 8) plans."""
    from paper_2309_03523_b200 import load_plan_npz
    pa = load_plan_npz(artifacts_dir / name / "plan.npz")
    prof = pa.profile
    H, s, b = prof["embedding_dim"], prof["bytes_per_scalar"], prof["blocks"]
    ts = b * prof["spatial_msgs_per_block"] * H * s
    tw = np.full(len(pa.temporal_links), b * prof["temporal_msgs_per_block"] * H * s, np.int64)
    cap = -(-pa.n_instances // (4 * D))  # default_size_cap (partition.py:111-114)
    labels, _, _ = propagate_labels(pa.n_instances, pa.spatial_edges, pa.temporal_links, ts, tw,
                                    cap, 100)
    np.testing.assert_array_equal(chunk_ids(labels), pa.chunk_of)
