"""GPU parity of the graph build (BipartiteGraph::from_edges, graph.cpp:31-58) across the
device build's paths: left-grouped input (group-by-left sort skipped), input with duplicate
edges (flag/scan compaction) and without (row-sorted arrays kept), and rows of every size
class of the per-row sorts (sub-warp, warp, CTA, device-wide for rows > 8192 entries).
CSR arrays, external ids and the exact count are compared with the oracle."""
import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def check(l, r):
    o = O.Oracle(l, r)
    g = B.BipartiteGraph.from_edges(l, r)
    loff, ladj, roff, radj, reid, lids, rids = g.export()
    w = o.csr()
    for name, a, b in zip(("loff", "ladj", "roff", "radj", "lids", "rids"),
                          (loff, ladj, roff, radj, lids, rids), w):
        np.testing.assert_array_equal(a, b, err_msg=name)
    # reid: canonical edge id of every right-CSR entry (its (l, r) in the left CSR)
    lrow = np.repeat(np.arange(len(loff) - 1, dtype=np.uint64), np.diff(loff).astype(np.int64))
    rrow = np.repeat(np.arange(len(roff) - 1, dtype=np.uint64), np.diff(roff).astype(np.int64))
    np.testing.assert_array_equal(lrow[reid.astype(np.int64)], radj)
    np.testing.assert_array_equal(ladj[reid.astype(np.int64)], rrow)
    assert B.exact_count(g) == o.exact_count()
    g.close()


def hub_graph(seed, dup_frac):
    """Power-law left side with rows of every size class up to > 8192 entries."""
    rng = np.random.default_rng(seed)
    L, R = 3000, 40000
    deg = np.minimum((30000 / (np.arange(L) + 1) ** 0.9).astype(np.int64) + 1, R)
    l = np.repeat(np.arange(L, dtype=np.uint32), deg)
    r = np.concatenate([rng.choice(R, size=d, replace=False) for d in deg]).astype(np.uint32)
    nd = int(len(l) * dup_frac)
    if nd:
        pick = rng.integers(0, len(l), nd)
        l = np.concatenate([l, l[pick]])
        r = np.concatenate([r, r[pick]])
    return l, r, rng


@pytest.mark.parametrize("dup_frac", [0.0, 0.05])
def test_grouped_input(dup_frac):
    l, r, rng = hub_graph(1, dup_frac)
    order = np.lexsort((rng.random(len(l)), l))  # grouped by left id, rows unsorted
    check(l[order], r[order])


@pytest.mark.parametrize("dup_frac", [0.0, 0.05])
def test_random_order_input(dup_frac):
    l, r, rng = hub_graph(2, dup_frac)
    perm = rng.permutation(len(l))
    check(l[perm], r[perm])


def test_sorted_input_and_reversed_ids():
    l, r, _ = hub_graph(3, 0.0)
    order = np.lexsort((r, l))
    check(l[order], r[order])
    check((3000 - 1 - l).astype(np.uint32), r)  # descending left ids, grouped


def test_power_law_duplicates_random_order():
    l, r = B.synth_chung_lu(50000, 120000, 400000, 2.1, 2.5, 7)
    rng = np.random.default_rng(7)
    pick = rng.integers(0, len(l), 20000)
    l2 = np.concatenate([l, l[pick]])
    r2 = np.concatenate([r, r[pick]])
    perm = rng.permutation(len(l2))
    check(l2[perm], r2[perm])


def _same_graph(a, b):
    for name, x, y in zip(("loff", "ladj", "roff", "radj", "reid", "lids", "rids"), a.export(),
                          b.export()):
        np.testing.assert_array_equal(x, y, err_msg=name)


@pytest.mark.parametrize("wide", [False, True])
def test_reference_pair_layout(wide):
    """from_edges(const vector<pair<uint64_t, uint64_t>>&) (graph.hpp:43) through the
    interleaved-pair entry (bfly_graph_build_pairs): several staging chunks, duplicates, and
    ids >= 2^32 (the u64 fallback) give the same graph as the split-array build and the
    oracle."""
    l, r, rng = hub_graph(3, 0.05)
    perm = rng.permutation(len(l))
    l, r = l[perm].astype(np.uint64), r[perm].astype(np.uint64)
    reps = 1 + (3 << 20) // len(l)  # > 3 staging chunks of 2^20 edges
    l = np.tile(l, reps)
    r = np.tile(r, reps)
    if wide:
        l = l * np.uint64(7919) + np.uint64(1 << 33)
    pairs = np.stack([l, r], axis=1)
    g = B.BipartiteGraph.from_pairs(pairs)
    h = B.BipartiteGraph.from_edges(l, r)
    _same_graph(g, h)
    o = O.Oracle(l, r)
    np.testing.assert_array_equal(g.export()[5], o.csr()[4])
    assert B.exact_count(g) == o.exact_count()
    g.close()
    h.close()


def test_reference_pair_layout_empty_and_errors():
    g = B.BipartiteGraph.from_pairs(np.zeros((0, 2), np.uint64))
    assert g.edge_count() == 0
    g.close()
