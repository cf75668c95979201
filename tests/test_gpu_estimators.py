"""GPU parity of the estimators (sampling.cpp / sparsify.cpp) through the C++ facade:
run_estimator values bit-equal to the reference's (goldens) and to the oracle, for every
method, median-of-means, thread counts, trace and validation (tests/test_sampling.cpp)."""
import os

import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
SAMPLED = sorted({k.split("/")[0] for k in GOLD.files if k.endswith("/est0")})


@pytest.mark.parametrize("case", SAMPLED)
def test_estimators_match_reference_goldens(case):
    e = GOLD[f"{case}/edges"]
    g = B.BipartiteGraph.from_edges(e[0], e[1])
    for method in (0, 1, 2):
        est = B.run_estimator(g, B.Method(method), iterations=257, seed=99, threads=4)
        assert est.value == GOLD[f"{case}/est{method}"][0]
        assert est.iterations_done == 257
        mom = B.run_estimator(g, B.Method(method), seed=7, groups=5, group_size=20, threads=2)
        assert [mom.value] + mom.per_group_means == GOLD[f"{case}/mom{method}"].tolist()
    run = B.sparsify_run(g, 0, p=0.4, seed=99, trials=8)
    assert [run.value] + run.per_group_means == GOLD[f"{case}/sprun_edge"].tolist()
    run = B.sparsify_run(g, 1, colors=2, seed=99, trials=8)
    assert [run.value] + run.per_group_means == GOLD[f"{case}/sprun_color"].tolist()


def test_sample_ids_match_oracle_draws():
    l, r = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    prefix, total = o.build_wedge_index()
    for method in (0, 1, 2):
        got = B.sample_ids(g, B.Method(method), 4, 0, 2000)
        want = o.sample_draws(method, 4, 2000, prefix, total)
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)


def test_thread_count_independent_and_trace():
    l, r = O.random_bipartite_edges(40, 40, 0.2, 21)
    g = B.BipartiteGraph.from_edges(l, r)
    for m in (B.Method.Vertex, B.Method.Edge, B.Method.Wedge):
        a = B.run_estimator(g, m, iterations=257, seed=99, threads=1)
        c = B.run_estimator(g, m, iterations=257, seed=99, threads=4)
        assert a.value == c.value
        assert B.run_estimator(g, m, iterations=257, seed=100).value != a.value
    l, r = O.random_bipartite_edges(15, 15, 0.4, 9)
    g = B.BipartiteGraph.from_edges(l, r)
    est = B.run_estimator(g, B.Method.Edge, iterations=100, seed=11, record_trace=True, threads=8)
    assert [t[0] for t in est.trace] == [1, 2, 4, 8, 16, 32, 64, 100]
    assert est.trace[-1][1] == est.value
    o = O.Oracle(l, r)
    vals = o.run_estimator(1, 100, 11, values=True)["values"]
    s = 0.0
    want = []
    for i, v in enumerate(vals, 1):
        s += v
        if i in (1, 2, 4, 8, 16, 32, 64, 100):
            want.append(s / i)
    assert [t[1] for t in est.trace] == want


def test_time_budget_whole_blocks():
    g = B.BipartiteGraph.from_edges(*H.k33())
    est = B.run_estimator(g, B.Method.Vertex, seed=3, time_budget_seconds=0.02)
    assert est.iterations_done >= 64 and est.iterations_done % 64 == 0
    assert est.value == 9.0  # every K33 vertex value is 6 * 6 / 4


def test_validation_and_no_wedges():
    g = B.BipartiteGraph.from_edges(*H.k22())
    with pytest.raises(B.ArgumentError):
        B.run_estimator(g, B.Method.Vertex)  # nothing set
    with pytest.raises(B.ArgumentError):
        B.run_estimator(g, B.Method.Vertex, iterations=10, time_budget_seconds=1.0)
    with pytest.raises(B.ArgumentError):
        B.run_estimator(g, B.Method.Vertex, groups=4, group_size=2)
    est = B.run_estimator(g, B.Method.Vertex, iterations=9, groups=3)
    assert est.iterations_done == 27
    single = B.BipartiteGraph.from_edges([1], [1])
    with pytest.raises(B.NoWedgesError):
        B.run_estimator(single, B.Method.Wedge, iterations=5)


def test_degenerate_estimators_constant():
    g22 = B.BipartiteGraph.from_edges(*H.k22())
    g33 = B.BipartiteGraph.from_edges(*H.k33())
    assert B.build_wedge_index(g33).total == 18
    for seed in range(10):
        assert B.run_estimator(g22, B.Method.Vertex, iterations=1, seed=seed).value == 1.0
        assert B.run_estimator(g33, B.Method.Wedge, iterations=1, seed=seed).value == 9.0


def test_pinned_outcome_values():
    g32 = B.BipartiteGraph.from_edges(*H.k32())
    assert B.vertex_sample_value(g32, B.VertexRef(B.Side.Left, 0)) == 2.5
    assert B.vertex_sample_value(g32, B.VertexRef(B.Side.Right, 1)) == 3.75
    for k in range(6):
        assert B.edge_sample_value(g32, *g32.edge_at(k)) == 3.0
    assert B.wedge_sample_value(g32, 9, B.VertexRef(B.Side.Right, 0), 0, 1) == 2.25
    assert B.wedge_sample_value(g32, 9, B.VertexRef(B.Side.Left, 0), 0, 1) == 4.5
