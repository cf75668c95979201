"""GPU parity: exact counts through the C-ABI vs the oracle (and reference known answers)."""
import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu


def test_device_ok():
    assert B.device_ok(), B._abi.last_error()


def test_biclique_closed_form_grid():
    # tests/test_exact.cpp:11-17 (sub-grid; the full 60x60 grid runs in the slow test)
    for a in (1, 2, 3, 5, 8, 13, 21, 34, 60):
        for b in (1, 2, 4, 7, 16, 31, 60):
            g = B.BipartiteGraph.from_edges(*H.k(a, b))
            assert B.exact_count(g) == O.choose2(a) * O.choose2(b)


def test_k_10000_10():
    # tests/test_exact.cpp:59-62
    g = B.BipartiteGraph.from_edges(*H.k(10000, 10))
    assert B.exact_count(g) == 2249775000
    c = B.choose_side(g)
    assert c.cost_left == 1e6 and c.cost_right == 1e9 and c.chosen == B.Side.Right


def test_named_and_random_suites_vs_oracle():
    suite = H.named_suite() + O.random_suite_edges(60, 12, 12, [0.2, 0.5, 0.8], 5000)
    for l, r in suite:
        o = O.Oracle(l, r)
        g = B.BipartiteGraph.from_edges(l, r)
        want = o.exact_count()
        assert B.exact_count(g) == want
        assert B.exact_count_side(g, B.Side.Left) == want
        assert B.exact_count_side(g, B.Side.Right) == want
        if o.L <= 64 and o.R <= 64:
            assert o.brute_force_count() == want


def test_config1_uniform():
    l, r = B.synth_uniform(10000, 5000, 100000, 1)
    o = O.Oracle(l, r)
    g = B.BipartiteGraph.from_edges(l, r)
    assert B.exact_count(g) == o.exact_count()


@pytest.mark.parametrize("seed", [11, 12])
def test_power_law_medium(seed):
    l, r = B.synth_chung_lu(200000, 500000, 2000000, 2.1, 2.5, seed)
    o = O.Oracle(l, r)
    g = B.BipartiteGraph.from_edges(l, r)
    assert B.exact_count(g) == o.exact_count()


def test_concurrent_handles_two_threads():
    # exact counts of different handles from two host threads at once: the bucket kernels of
    # both share the per-device side streams (fork/join events are per call)
    import threading
    graphs = [B.synth_chung_lu(60000, 150000, 600000, 2.1, 2.5, s) for s in (21, 22)]
    want = [O.Oracle(l, r).exact_count() for l, r in graphs]
    got = [[], []]

    def work(i):
        l, r = graphs[i]
        for _ in range(4):
            g = B.BipartiteGraph.from_edges(l, r)
            got[i].append(B.exact_count(g))
            g.close()

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert got[0] == [want[0]] * 4 and got[1] == [want[1]] * 4


@pytest.mark.parametrize("width", ["off", "1", "2", "8", "32"])
def test_dense_top_hub_widths(monkeypatch, width):
    # the top-hub masks (hubdense.cuh) at every width against the oracle, on a graph whose
    # largest end vertices exceed one 4096-entry chunk (tasks merged through the global rows);
    # then count -> local counts -> count on one handle (the local pass rebuilds the hub plan
    # without the dense hubs; the later count runs on that plan)
    if width == "off":
        monkeypatch.setenv("BFLY_HUB_DENSE", "0")
    else:
        monkeypatch.setenv("BFLY_HUB_DENSE_W", width)
        monkeypatch.setenv("BFLY_HUB_DENSE_MIN", "0")  # (whatever the top hubs' share)
    l, r = B.synth_chung_lu(100000, 250000, 1500000, 2.1, 2.5, 31)
    o = O.Oracle(l, r)
    want = o.exact_count()
    g = B.BipartiteGraph.from_edges(l, r)
    assert B.compute_stats(g).max_degree > 4096
    assert B.exact_count(g) == want
    ds = B.last_dense_stats(g)
    if width == "off":
        assert ds["wedges"] == 0
    else:
        # (fewer words when the graph has fewer than 32 * width hub starts)
        assert 1 <= ds["words"] <= int(width) and ds["hubs"] <= 32 * ds["words"]
        assert ds["wedges"] > 0
        assert ds["wedges"] <= B.last_exact_stats(g).wedges_processed
    assert B.exact_count_side(g, B.Side.Left) == want
    pv = B.count_all_vertices(g)
    assert int(pv.sum(dtype=np.uint64)) == 4 * want
    assert B.exact_count(g) == want
    g.close()


def test_dense_top_hubs_on_bicliques(monkeypatch):
    # every start is a top hub: K_{a,b} counts come from the masks alone
    monkeypatch.setenv("BFLY_HUB_DENSE_MIN", "0")
    for a, b in ((300, 40), (40, 300), (1000, 1000), (5000, 33)):
        g = B.BipartiteGraph.from_edges(*H.k(a, b))
        assert B.exact_count(g) == O.choose2(a) * O.choose2(b)
        g.close()
