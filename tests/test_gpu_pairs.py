"""GPU: butterfly pair types at scale (pairs.cu; reference oracle.cpp:60-116).

1. == the reference's own classify_pairs / variance_bounds on every golden graph
   (tests/golden/pairs.json), through the guarded contract and the unguarded at-scale call.
2. Closed forms on complete bicliques up to K_{1000,1000}, whose C(bfly,2) exceeds 2^64.
3. == the oracle's moment checker (pinned to the reference in tests/test_pairs_oracle.py) on
   config 1 and on power-law graphs far beyond enumeration size, where hub pairs take the
   engine's heavy rows and medium tables.
"""
import json
import os
from math import comb

import numpy as np
import pytest

import paper_1801_00338_b200 as B
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pairs.json")))
CASES = GOLD["cases"]


def _graph(c):
    return B.BipartiteGraph.from_edges(np.array(c["left"], np.uint64),
                                       np.array(c["right"], np.uint64))


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_pair_types_vs_reference(c):
    g = _graph(c)
    got = B.classify_pairs_at_scale(g)
    assert list(got.as_tuple()) == c["counts"]
    if c["counts"][0] <= 2000 and g.left_count() <= 64 and g.right_count() <= 64:
        assert list(B.classify_pairs(g).as_tuple()) == c["counts"]
    st = B.compute_stats(g)
    for p in (0.5, 0.1):
        b = B.variance_bounds(st, got, p)
        assert [b.vsamp, b.esamp, b.wsamp, b.espar, b.clrspar] == c[f"bounds_p{p}"]


def test_guards_match_reference():
    with pytest.raises(B.SizeGuardError, match="side exceeds 64 vertices"):
        B.classify_pairs(B.BipartiteGraph.from_edges(*O.complete_biclique_edges(70, 3)))
    k33 = B.BipartiteGraph.from_edges(*O.complete_biclique_edges(3, 3))
    with pytest.raises(B.SizeGuardError, match="9 butterflies exceeds pair classification limit of 2"):
        B.classify_pairs(k33, B.OracleGuards(max_butterflies=2))
    with pytest.raises(B.ArgumentError):
        B.variance_bounds(B.compute_stats(k33), B.classify_pairs(k33), 0.0)


def _kab(a, b):
    """Closed forms for K_{a,b}: every left pair has c = b common neighbours, every right
    pair c = a; bfly_v = (a-1) C(b,2) on the left, (b-1) C(a,2) on the right; bfly_e =
    (a-1)(b-1)."""
    bf = comb(a, 2) * comb(b, 2)
    p1w = 3 * (comb(a, 2) * comb(b, 3) + comb(b, 2) * comb(a, 3))
    p2v = 3 * (comb(a, 2) * comb(b, 4) + comb(b, 2) * comb(a, 4))
    e2 = a * b * comb((a - 1) * (b - 1), 2)
    v2 = a * comb((a - 1) * comb(b, 2), 2) + b * comb((b - 1) * comb(a, 2), 2)
    p1e = e2 - 2 * p1w
    p1v = v2 - 2 * p2v - 2 * p1e - 3 * p1w
    return (bf, comb(bf, 2) - p1v - p2v - p1e - p1w, p1v, p2v, p1e, p1w)


@pytest.mark.parametrize("a,b", [(2, 2), (3, 2), (5, 7), (64, 3), (300, 40), (1000, 1000)])
def test_biclique_closed_forms(a, b):
    g = B.BipartiteGraph.from_edges(*O.complete_biclique_edges(a, b))
    assert B.classify_pairs_at_scale(g).as_tuple() == _kab(a, b)


@pytest.mark.parametrize("shape", [
    ("uniform", 10_000, 5_000, 100_000, None, None, 1),          # BASELINE config 1
    ("chung_lu", 3_000, 6_000, 30_000, 2.1, 2.5, 2),             # smoke-sized power law
    ("chung_lu", 8_000, 16_000, 150_000, 2.1, 2.5, 5),           # hub pairs in heavy rows
])
def test_pair_types_vs_moment_checker(shape):
    kind, U, V, m, gu, gv, seed = shape
    if kind == "uniform":
        l, r = B.synth_uniform(U, V, m, seed)
    else:
        l, r = B.synth_chung_lu(U, V, m, gu, gv, seed)
    g = B.BipartiteGraph.from_edges(l, r)
    want = O.Oracle(l, r).pair_counts_by_moments()
    assert B.classify_pairs_at_scale(g).as_tuple() == want
