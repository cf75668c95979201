"""GPU parity of the device-side sample-id derivation (sampler.cu): the ids,
wedge positions and per-sample integers bfly_sample_batch draws on the GPU equal the
oracle's draws from std::mt19937_64(derive_seed(seed, q)) (sampling.cpp:101-123), for every
method, offsets, extreme seeds, and with the register engine forced onto its full-engine
fallback (BFLY_SAMPLER_FAST_DRAWS)."""
import os

import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def graph():
    l, r = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    return l, r, B.BipartiteGraph.from_edges(l, r), O.Oracle(l, r)


@pytest.mark.parametrize("seed", [4, 0, 2**64 - 1])
def test_device_ids_equal_oracle_draws(graph, seed):
    l, r, g, o = graph
    prefix, total = o.build_wedge_index()
    for method in (0, 1, 2):
        _, ids, ii, jj = B.sample_batch(g, B.Method(method), seed, 0, 3000)
        want = o.sample_draws(method, seed, 3000, prefix, total)
        np.testing.assert_array_equal(ids, want[0])
        if method == 2:
            np.testing.assert_array_equal(ii, want[1])
            np.testing.assert_array_equal(jj, want[2])


def test_device_ids_with_offset_equal_host_restatement(graph):
    _, _, g, _ = graph
    for method in (0, 1, 2):
        _, ids, ii, jj = B.sample_batch(g, B.Method(method), 77, 123456, 5000)
        h = B.sample_ids(g, B.Method(method), 77, 123456, 5000)
        np.testing.assert_array_equal(ids, h[0])
        if method == 2:
            np.testing.assert_array_equal(ii, h[1])
            np.testing.assert_array_equal(jj, h[2])


def test_counts_are_scaled_values_of_oracle(graph):
    _, _, g, o = graph
    n, m = g.vertex_count(), g.edge_count()
    _, total = o.build_wedge_index()
    for method, scale in ((0, n), (1, m), (2, total)):
        cnt, _, _, _ = B.sample_batch(g, B.Method(method), 5, 0, 400)
        want = o.run_estimator(method, 400, 5, values=True)["values"]
        got = np.array([float(c) * float(scale) / 4.0 for c in cnt])
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("fast", ["0", "1", "3"])
def test_full_engine_fallback(graph, fast):
    l, r, g, o = graph
    prefix, total = o.build_wedge_index()
    os.environ["BFLY_SAMPLER_FAST_DRAWS"] = fast
    try:
        got = [B.sample_batch(g, B.Method(m), 9, 0, 700) for m in (0, 1, 2)]
    finally:
        del os.environ["BFLY_SAMPLER_FAST_DRAWS"]
    for m in (0, 1, 2):
        want = o.sample_draws(m, 9, 700, prefix, total)
        np.testing.assert_array_equal(got[m][1], want[0])
        if m == 2:
            np.testing.assert_array_equal(got[m][2], want[1])
            np.testing.assert_array_equal(got[m][3], want[2])


def test_sampler_errors():
    l, r = np.array([0, 1], np.uint64), np.array([0, 1], np.uint64)  # perfect matching
    g = B.BipartiteGraph.from_edges(l, r)
    with pytest.raises(B.NoWedgesError):
        B.sample_batch(g, B.Method.Wedge, 1, 0, 10)
    with pytest.raises(B.ArgumentError):
        B.sample_batch(g, B.Method.FastEdge, 1, 0, 10)
    cnt, ids, _, _ = B.sample_batch(g, B.Method.Vertex, 1, 0, 0)
    assert len(cnt) == 0
