"""GPU parity of Method::FastEdge (sampling.cpp:93-147): device engines, automaton-classified
draws and batched has_edge probes equal the reference's values bit for bit (goldens from the
reference build) and the oracle's per-iteration values, hits and edge ids; run_estimator's
mean, median-of-means and validation match the reference."""
import os

import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
FAST = sorted({k.split("/")[0] for k in GOLD.files if k.endswith("/fast_iter")})


@pytest.mark.parametrize("case", FAST)
def test_fast_edge_matches_reference_goldens(case):
    e = GOLD[f"{case}/edges"]
    g = B.BipartiteGraph.from_edges(e[0], e[1])
    vals, _, _ = B.fast_edge_batch(g, 7, 0, 64, 50)
    assert vals.tolist() == GOLD[f"{case}/fast_iter"].tolist()
    est = B.run_estimator(g, B.Method.FastEdge, iterations=257, seed=99, fast_edge_repeats=100)
    assert est.value == GOLD[f"{case}/est3"][0]
    mom = B.run_estimator(g, B.Method.FastEdge, seed=7, groups=5, group_size=20,
                          fast_edge_repeats=30)
    assert [mom.value] + mom.per_group_means == GOLD[f"{case}/mom3"].tolist()


@pytest.mark.parametrize("repeats", [1, 7, 33, 1000])
def test_fast_edge_matches_oracle_power_law(repeats):
    l, r = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    n = 300
    vals, hits, eids = B.fast_edge_batch(g, 11, 1000, n, repeats)
    for i in range(n):
        v, k, h = o.fast_iteration(repeats, 11, 1000 + i)
        assert (vals[i], int(eids[i]), int(hits[i])) == (v, k, h), i


def test_fast_edge_degenerate_degrees():
    # star: every edge has a degree-1 endpoint -> value 0, no draws after the edge
    l = np.zeros(9, np.uint64)
    r = np.arange(9, dtype=np.uint64)
    g = B.BipartiteGraph.from_edges(l, r)
    vals, hits, _ = B.fast_edge_batch(g, 3, 0, 50, 10)
    assert not vals.any() and not hits.any()
    # K_{2,5}: left degree 5 draws, right degree 2 draws nothing (uniform_index(1))
    a, b = np.meshgrid(np.arange(2), np.arange(5), indexing="ij")
    l, r = a.ravel().astype(np.uint64), b.ravel().astype(np.uint64)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    vals, hits, eids = B.fast_edge_batch(g, 5, 0, 40, 17)
    for i in range(40):
        assert (vals[i], int(eids[i]), int(hits[i])) == o.fast_iteration(17, 5, i)


def test_fast_edge_validation():
    l, r = O.random_bipartite_edges(15, 15, 0.4, 9)
    g = B.BipartiteGraph.from_edges(l, r)
    with pytest.raises(B.ArgumentError):
        B.fast_edge_batch(g, 1, 0, 4, 0)
    with pytest.raises(B.ArgumentError):
        B.run_estimator(g, B.Method.FastEdge, iterations=4, fast_edge_repeats=0)
    est = B.run_estimator(g, B.Method.FastEdge, iterations=100, seed=11, record_trace=True,
                          fast_edge_repeats=20)
    assert [t[0] for t in est.trace] == [1, 2, 4, 8, 16, 32, 64, 100]
    o = O.Oracle(l, r)
    want = o.run_estimator(3, 100, 11, repeats=20)["value"]
    assert est.value == want


@pytest.mark.slow
def test_fast_edge_config2_subset():
    l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
    g = B.BipartiteGraph.from_edges(l, r)
    vals, hits, eids = B.fast_edge_batch(g, 4, 0, 1 << 16, 1000)
    o = O.Oracle(l, r)
    for i in range(0, 1 << 16, 257):
        assert (vals[i], int(eids[i]), int(hits[i])) == o.fast_iteration(1000, 4, i), i
