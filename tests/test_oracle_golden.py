"""CPU: pin the oracle (C restatement, oracle/bfly_oracle.c) before trusting it.

1. Known-answer tests the reference's own suite holds (proj/tests/*.cpp).
2. Golden vectors produced by the unmodified reference compiled here
   (tests/golden/make_golden.py -> golden.npz).
3. Direct comparison with oracle/_ref when the reference build is present.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
CASES = sorted({k.split("/")[0] for k in GOLD.files if k.endswith("/edges")})


def test_choose2_and_checked_arithmetic():
    # tests/test_exact.cpp:85-94
    assert O.choose2(4294967296 - 1) == 9223372030412324865
    assert [O.choose2(c) for c in (0, 1, 2, 5)] == [0, 0, 1, 10]
    with pytest.raises(O.OracleError):
        O.choose2(1 << 33)


def test_rng_pins():
    xs = [0, 1, 2, 3, 42, 2 ** 63, 2 ** 64 - 1]
    assert [O.mix64(x) for x in xs] == GOLD["rng/mix64"].tolist()
    assert [O.derive_seed(x, y) for x in xs for y in xs] == GOLD["rng/derive"].tolist()
    firsts = []
    for s in (0, 4, 99):
        for i in range(16):
            firsts.append(O.Rng(O.derive_seed(s, i)).next())
    assert firsts == GOLD["rng/stream_first"].tolist()


def test_biclique_grid_closed_form():
    # tests/test_exact.cpp:11-17 (full 60 x 60 grid)
    for a in range(1, 61):
        for b in range(1, 61, 7):
            o = O.Oracle(*H.k(a, b), threads=1)
            assert o.exact_count() == O.choose2(a) * O.choose2(b)


def test_k_10000_10_and_side_choice():
    o = O.Oracle(*H.k(10000, 10))
    assert o.exact_count() == 2249775000  # tests/test_exact.cpp:59-62
    chosen, cl, cr = o.choose_side()
    assert (chosen, cl, cr) == (1, 1e6, 1e9)  # tests/test_exact.cpp:37-45
    assert O.Oracle(*H.k(2, 100)).choose_side()[0] == 0
    assert O.Oracle(*H.k33()).choose_side()[0] == 0  # ties go left


def test_butterfly_free():
    for l, r in (H.cycle6(), H.star15(), H.path4()):
        assert O.Oracle(l, r).exact_count() == 0


def test_local_hand_values():
    # tests/test_local.cpp:11-44
    g33 = O.Oracle(*H.k33())
    assert all(g33.count_per_vertex(s, i) == 6 for s in (0, 1) for i in range(3))
    assert all(g33.count_per_edge(l, r) == 4 for l in range(3) for r in range(3))
    assert O.Oracle(*H.k22()).count_per_vertex(0, 0) == 1
    assert O.Oracle(*H.k22()).count_per_edge(0, 0) == 1
    assert O.Oracle(*H.k(1, 3)).count_per_edge(0, 0) == 0
    assert O.Oracle(*H.k(8, 2)).count_per_edge(0, 0) == 7
    assert O.Oracle(*H.k(2, 8)).count_per_edge(0, 0) == 7
    with pytest.raises(O.OracleError):
        O.Oracle(*H.k22()).count_per_vertex(0, 2)
    with pytest.raises(O.OracleError):
        O.Oracle(*H.two_k22()).count_per_edge(0, 3)


def test_sampling_pinned_values():
    # tests/test_sampling.cpp:45-62
    g = O.Oracle(*H.k32())
    assert g.vertex_sample_value(0, 0) == 2.5
    assert g.vertex_sample_value(1, 1) == 3.75
    for k in range(6):
        assert g.edge_sample_value(*g.edge_at(k)) == 3.0
    assert g.wedge_sample_value(9, 1, 0, 0, 1) == 2.25
    assert g.wedge_sample_value(9, 0, 0, 0, 1) == 4.5
    assert O.Oracle(*H.k33()).build_wedge_index()[1] == 18


def test_sparsify_identities():
    # tests/test_sparsify.cpp:42-53, 172-176, 224-231
    for l, r in H.named_suite():
        o = O.Oracle(l, r)
        exact = float(o.exact_count())
        for seed in (0, 1, 42, 987654321):
            assert o.edge_sparsify_estimate(1.0, seed)[0] == exact
            assert o.color_sparsify_estimate(1, seed)[0] == exact
    assert O.Oracle(*H.k(5, 5)).sparsify_run(1, colors=1, trials=3)["value"] == 100.0
    g = O.Oracle(*H.k22())
    assert g.edge_sparsify_value(np.zeros(4, np.uint8), 0.5) == 0.0
    assert g.color_sparsify_value(np.array([0, 1, 0, 1], np.uint32), 2) == 0.0


def test_local_sums_four_times_global():
    # tests/test_local.cpp:61-77
    for l, r in O.random_suite_edges(20, 13, 13, [0.25, 0.5, 0.75], 9000):
        o = O.Oracle(l, r)
        b = o.exact_count()
        assert int(o.count_all_vertices().sum()) == 4 * b
        assert int(o.count_all_edges().sum()) == 4 * b


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_goldens(case):
    e = GOLD[f"{case}/edges"]
    o = O.Oracle(e[0], e[1])
    assert [o.L, o.R, o.m] == GOLD[f"{case}/sizes"].tolist()
    loff, ladj, roff, radj, lids, rids = o.csr()
    for name, arr in (("loff", loff), ("ladj", ladj), ("roff", roff), ("radj", radj),
                      ("lids", lids), ("rids", rids)):
        np.testing.assert_array_equal(arr, GOLD[f"{case}/{name}"], err_msg=name)
    ex = GOLD[f"{case}/exact"].tolist()
    assert [o.exact_count(), o.exact_count_side(0), o.exact_count_side(1)] == ex
    side, cl, cr = o.choose_side()
    assert side == int(GOLD[f"{case}/side"][0])
    assert [cl, cr] == GOLD[f"{case}/costs"].tolist()
    st = o.compute_stats()
    assert [st["n"], st["left"], st["right"], st["m"], st["wedge_count"], st["max_degree"]] == \
        GOLD[f"{case}/stats_u64"].tolist()
    if f"{case}/vertex" in GOLD:
        np.testing.assert_array_equal(o.count_all_vertices(), GOLD[f"{case}/vertex"])
        np.testing.assert_array_equal(o.count_all_edges(), GOLD[f"{case}/edge"])
    if f"{case}/iter0" in GOLD:
        prefix, total = o.build_wedge_index()
        for method in (0, 1, 2):
            got = []
            for i in range(64):
                ids = o.sample_draws(method, 7, i + 1, prefix, total)
                got.append(_iteration_value(o, method, ids, i, total))
            assert got == GOLD[f"{case}/iter{method}"].tolist()
            assert o.run_estimator(method, 257, 99)["value"] == GOLD[f"{case}/est{method}"][0]
            mom = o.run_estimator(method, 0, 7, groups=5, group_size=20)
            assert [mom["value"]] + mom["per_group_means"] == GOLD[f"{case}/mom{method}"].tolist()
        if f"{case}/fast_iter" in GOLD:  # Method::FastEdge (sampling.cpp:125-147)
            got = [o.fast_iteration(50, 7, i)[0] for i in range(64)]
            assert got == GOLD[f"{case}/fast_iter"].tolist()
            assert o.run_estimator(3, 257, 99, repeats=100)["value"] == GOLD[f"{case}/est3"][0]
            mom = o.run_estimator(3, 0, 7, groups=5, group_size=20, repeats=30)
            assert [mom["value"]] + mom["per_group_means"] == GOLD[f"{case}/mom3"].tolist()
        for seed in (0, 1, 42):
            assert [o.edge_sparsify_estimate(0.5, seed)[0], o.edge_sparsify_estimate(0.3, seed)[0]] \
                == GOLD[f"{case}/espar{seed}"].tolist()
            assert [o.color_sparsify_estimate(2, seed)[0], o.color_sparsify_estimate(3, seed)[0]] \
                == GOLD[f"{case}/cspar{seed}"].tolist()
        run = o.sparsify_run(0, p=0.4, seed=99, trials=8)
        assert [run["value"]] + run["per_group_means"] == GOLD[f"{case}/sprun_edge"].tolist()
        run = o.sparsify_run(1, colors=2, seed=99, trials=8)
        assert [run["value"]] + run["per_group_means"] == GOLD[f"{case}/sprun_color"].tolist()


def _iteration_value(o, method, ids, i, total):
    id0, ii, jj = int(ids[0][i]), int(ids[1][i]), int(ids[2][i])
    if method == 0:
        side = 0 if id0 < o.L else 1
        return o.vertex_sample_value(side, id0 if side == 0 else id0 - o.L)
    if method == 1:
        return o.edge_sample_value(*o.edge_at(id0))
    side = 0 if id0 < o.L else 1
    ci = id0 if side == 0 else id0 - o.L
    loff, ladj, roff, radj = o.csr()[:4]
    adj = ladj[loff[ci]:loff[ci + 1]] if side == 0 else radj[roff[ci]:roff[ci + 1]]
    return o.wedge_sample_value(total, side, ci, int(adj[ii]), int(adj[jj]))


def test_config1_goldens():
    import paper_1801_00338_b200 as B
    l, r = B.synth_uniform(10000, 5000, 100000, 1)
    sha = np.frombuffer(hashlib.sha256(l.tobytes() + r.tobytes()).digest(), np.uint8)
    np.testing.assert_array_equal(sha, GOLD["config1/edges_sha"][0])
    o = O.Oracle(l, r)
    assert o.exact_count() == int(GOLD["config1/exact"][0])
    np.testing.assert_array_equal(o.count_all_vertices(), GOLD["config1/vertex"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no reference tree)")
def test_oracle_vs_reference_random_suites():
    # acceptance.cpp:95-106 style: many random graphs, all counters agree
    for l, r in O.random_suite_edges(120, 12, 12, [0.2, 0.5, 0.8], 9000):
        o, ref = O.Oracle(l, r), O.Ref(l, r)
        assert o.exact_count() == ref.exact_count() == ref.brute_force_count()
        np.testing.assert_array_equal(o.count_all_vertices(), ref.count_all_vertices())
        np.testing.assert_array_equal(o.count_all_edges(), ref.count_edges())


TEXTS = sorted({k.split("/")[0] for k in GOLD.files if k.startswith("text")},
               key=lambda s: int(s[4:]))


@pytest.mark.parametrize("case", TEXTS)
def test_oracle_text_io_matches_reference(case):
    """load_edge_list / serialize_edge_list restated (graph.cpp:75-112) vs the reference."""
    text = GOLD[f"{case}/bytes"].tobytes()
    res = O.parse_text(text)
    if f"{case}/parse" in GOLD:
        assert res[0] == "parse"
        want = GOLD[f"{case}/parse"].tobytes().decode()
        line = int(GOLD[f"{case}/line"][0])
        assert (res[1] + f" (line {line})", res[2]) == (want, line)
        return
    assert res[0] == "ok"
    if f"{case}/empty" in GOLD:
        assert len(res[1]) == 0
        return
    o = O.Oracle(res[1], res[2])
    assert o.serialize() == GOLD[f"{case}/serialized"].tobytes()
    assert o.exact_count() == int(GOLD[f"{case}/exact"][0])
