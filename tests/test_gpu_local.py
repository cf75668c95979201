"""GPU parity: per-vertex / per-edge counts, per-sample kernels, sparsify-then-count.

Bit-exact against the oracle (integers) and the reference goldens (tests/golden)."""
import os

import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
CASES = sorted({k.split("/")[0] for k in GOLD.files if k.endswith("/edges")})


@pytest.mark.parametrize("case", CASES)
def test_goldens_all_local(case):
    e = GOLD[f"{case}/edges"]
    g = B.BipartiteGraph.from_edges(e[0], e[1])
    assert [g.left_count(), g.right_count(), g.edge_count()] == GOLD[f"{case}/sizes"].tolist()
    loff, ladj, roff, radj, reid, lids, rids = g.export()
    for name, arr in (("loff", loff), ("ladj", ladj), ("roff", roff), ("radj", radj),
                      ("lids", lids), ("rids", rids)):
        np.testing.assert_array_equal(arr, GOLD[f"{case}/{name}"], err_msg=name)
    assert B.exact_count(g) == int(GOLD[f"{case}/exact"][0])
    st = B.compute_stats(g)
    assert [st.n, st.left, st.right, st.m, st.wedge_count, st.max_degree] == \
        GOLD[f"{case}/stats_u64"].tolist()
    c = B.choose_side(g)
    assert [int(c.chosen)] == GOLD[f"{case}/side"].tolist()
    assert [c.cost_left, c.cost_right] == GOLD[f"{case}/costs"].tolist()
    if f"{case}/vertex" in GOLD:
        np.testing.assert_array_equal(B.count_all_vertices(g), GOLD[f"{case}/vertex"])
        np.testing.assert_array_equal(B.count_all_edges(g), GOLD[f"{case}/edge"])


def test_local_sums_and_hand_values():
    g33 = B.BipartiteGraph.from_edges(*H.k33())
    assert all(B.count_per_vertex(g33, B.VertexRef(s, i)) == 6 for s in B.Side for i in range(3))
    assert all(B.count_per_edge(g33, l, r) == 4 for l in range(3) for r in range(3))
    assert B.count_per_edge(B.BipartiteGraph.from_edges(*H.k(8, 2)), 0, 0) == 7
    assert B.count_per_edge(B.BipartiteGraph.from_edges(*H.k(2, 8)), 0, 0) == 7
    assert B.count_per_edge(B.BipartiteGraph.from_edges(*H.k(1, 3)), 0, 0) == 0
    with pytest.raises(B.ArgumentError):
        B.count_per_vertex(B.BipartiteGraph.from_edges(*H.k22()), B.VertexRef(B.Side.Left, 2))
    with pytest.raises(B.ArgumentError):
        B.count_per_edge(B.BipartiteGraph.from_edges(*H.two_k22()), 0, 3)
    with pytest.raises(B.ArgumentError):
        B.count_per_edge(B.BipartiteGraph.from_edges(*H.k22()), 0, 5)
    for l, r in O.random_suite_edges(30, 13, 13, [0.25, 0.5, 0.75], 9000):
        g = B.BipartiteGraph.from_edges(l, r)
        b = B.exact_count(g)
        assert int(B.count_all_vertices(g).sum()) == 4 * b
        assert int(B.count_all_edges(g).sum()) == 4 * b


def test_config1_all_vertices():
    l, r = B.synth_uniform(10000, 5000, 100000, 1)
    g = B.BipartiteGraph.from_edges(l, r)
    assert B.exact_count(g) == int(GOLD["config1/exact"][0])
    np.testing.assert_array_equal(B.count_all_vertices(g), GOLD["config1/vertex"])
    assert int(B.count_all_edges(g).sum()) == int(GOLD["config1/edge_sum"][0])


def test_power_law_local_vs_oracle():
    l, r = B.synth_chung_lu(20000, 40000, 300000, 2.1, 2.5, 5)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    np.testing.assert_array_equal(B.count_all_vertices(g), o.count_all_vertices())
    ks = np.random.default_rng(5).integers(0, o.m, 20000).astype(np.uint64)
    e_all = B.count_all_edges(g)
    want = o.count_edges_subset(ks)
    np.testing.assert_array_equal(e_all[ks], want)
    np.testing.assert_array_equal(B.count_edges(g, ks), want)
    gids = np.random.default_rng(6).integers(0, o.n, 20000).astype(np.uint64)
    np.testing.assert_array_equal(B.count_vertices(g, gids), o.count_vertices_subset(gids))


def test_vertex_only_pass_then_edges_and_back():
    # count_all_vertices on a fresh handle runs the vertex-only LOCAL pass (no per-edge
    # accumulators, priority CSR without edge ids); count_all_edges afterwards runs the full
    # pass on rebuilt priority rows; both orders and the exact count in between must agree
    # with the oracle (local.cpp:11-44)
    l, r = B.synth_chung_lu(30000, 60000, 500000, 2.1, 2.4, 9)
    o = O.Oracle(l, r)
    want_v = o.count_all_vertices()
    ks = np.random.default_rng(9).integers(0, o.m, 30000).astype(np.uint64)
    want_e = o.count_edges_subset(ks)
    total = o.exact_count()
    g = B.BipartiteGraph.from_edges(l, r)
    v1 = B.count_all_vertices(g)
    np.testing.assert_array_equal(v1, want_v)
    assert B.exact_count(g) == total
    e1 = B.count_all_edges(g)
    np.testing.assert_array_equal(e1[ks], want_e)
    assert int(e1.sum(dtype=np.uint64)) == 4 * total
    np.testing.assert_array_equal(B.count_all_vertices(g), want_v)
    g.close()
    g = B.BipartiteGraph.from_edges(l, r)  # edges first, vertices from the same full pass
    np.testing.assert_array_equal(B.count_all_edges(g)[ks], want_e)
    np.testing.assert_array_equal(B.count_all_vertices(g), want_v)
    g.close()


def test_sample_batches_vs_oracle_draws():
    l, r = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    prefix, total = o.build_wedge_index()
    wi = B.build_wedge_index(g)
    assert wi.total == total
    np.testing.assert_array_equal(wi.prefix, prefix)
    ids, _, _ = o.sample_draws(0, 4, 3000)
    np.testing.assert_array_equal(B.count_vertices(g, ids), o.count_vertices_subset(ids))
    ids, _, _ = o.sample_draws(1, 4, 3000)
    np.testing.assert_array_equal(B.count_edges(g, ids), o.count_edges_subset(ids))
    c, i, j = o.sample_draws(2, 4, 3000, prefix, total)
    got = B.wedge_common_minus_1(g, c, i, j)
    loff, ladj, roff, radj = o.csr()[:4]
    want = []
    for q in range(len(c)):
        cg = int(c[q])
        side = 0 if cg < o.L else 1
        ci = cg if side == 0 else cg - o.L
        adj = ladj[loff[ci]:loff[ci + 1]] if side == 0 else radj[roff[ci]:roff[ci + 1]]
        want.append(o.wedge_common_minus_1(side, int(adj[i[q]]), int(adj[j[q]])))
    np.testing.assert_array_equal(got, np.array(want, np.uint64))


@pytest.mark.parametrize("case", ["rb40", "chunglu_small", "uniform_small", "named_k33",
                                  "named_k24", "rand5000_3"])
def test_sparsify_vs_goldens(case):
    e = GOLD[f"{case}/edges"]
    g = B.BipartiteGraph.from_edges(e[0], e[1])
    for seed in (0, 1, 42):
        assert [B.edge_sparsify_estimate(g, 0.5, seed), B.edge_sparsify_estimate(g, 0.3, seed)] \
            == GOLD[f"{case}/espar{seed}"].tolist()
        assert [B.color_sparsify_estimate(g, 2, seed), B.color_sparsify_estimate(g, 3, seed)] \
            == GOLD[f"{case}/cspar{seed}"].tolist()


def test_sparsify_identities_and_errors():
    for l, r in H.named_suite():
        g = B.BipartiteGraph.from_edges(l, r)
        exact = float(B.exact_count(g))
        for seed in (0, 1, 42, 987654321):
            assert B.edge_sparsify_estimate(g, 1.0, seed) == exact
            assert B.color_sparsify_estimate(g, 1, seed) == exact
    g = B.BipartiteGraph.from_edges(*H.k22())
    assert B.edge_sparsify_value(g, np.zeros(4, np.uint8), 0.5) == 0.0
    assert B.color_sparsify_value(g, np.array([0, 1, 0, 1], np.uint32), 2) == 0.0
    assert B.edge_sparsify_value(g, np.ones(4, np.uint8), 1.0) == 1.0
    for bad in (0.0, 1.5, -0.1):
        with pytest.raises(B.ArgumentError):
            B.edge_sparsify_estimate(g, bad, 0)
    with pytest.raises(B.ArgumentError):
        B.color_sparsify_estimate(g, 0, 0)


def test_sparsify_power_law_vs_oracle():
    l, r = B.synth_chung_lu(20000, 40000, 300000, 2.1, 2.5, 5)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    for p in (0.1, 0.5):
        _, c, k = o.edge_sparsify_estimate(p, 5)
        assert B.espar_count(g, p, 5) == (c, k)
    for n in (2, 10):
        _, c, k = o.color_sparsify_estimate(n, 5)
        assert B.cspar_count(g, n, 5) == (c, k)
