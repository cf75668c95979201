"""CPU: pin the oracle's pair-type restatement (oracle/bfly_oracle.c, reference
oracle.cpp:60-116) to the reference's own classify_pairs / variance_bounds
(tests/golden/pairs.json, made by tests/golden/make_pair_goldens.py from oracle/_ref), and pin
the moment-identity checker that the GPU tests use beyond enumeration size to the same
goldens."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pairs.json")))
CASES = GOLD["cases"]


def _oracle(c):
    return O.Oracle(np.array(c["left"], np.uint64), np.array(c["right"], np.uint64), threads=2)


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_enumeration_restatement_vs_reference(c):
    if c["counts"][0] > 20000:
        pytest.skip("enumeration of > 2e8 pairs: covered by the moment checker below")
    assert list(_oracle(c).classify_pairs(1 << 30, 1 << 62)) == c["counts"]


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_moment_identities_vs_reference(c):
    """p_1w = 3 S3, p_2v = 3 S4, p_1e = E2 - 2 p_1w, p_1v = V2 - 2 p_2v - 2 p_1e - 3 p_1w,
    p_0v = C(bfly,2) - the rest (pairs.cu header) reproduce the reference's enumeration."""
    assert list(_oracle(c).pair_counts_by_moments()) == c["counts"]


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_variance_bounds_vs_reference(c):
    o = _oracle(c)
    st = o.compute_stats()
    for p in (0.5, 0.1):
        got = O.Oracle.variance_bounds(st["n"], st["m"], st["wedge_count"], c["counts"], p)
        assert list(got) == c[f"bounds_p{p}"]


def test_guards_and_arguments():
    o = O.Oracle(*O.complete_biclique_edges(70, 3))
    with pytest.raises(O.OracleError):
        o.classify_pairs()  # side 70 > 64 (oracle.cpp:13-17)
    with pytest.raises(O.OracleError):
        O.Oracle(*O.complete_biclique_edges(3, 3)).classify_pairs(64, 2)  # 9 > 2 (:62-67)
    with pytest.raises(O.OracleError):
        O.Oracle.variance_bounds(5, 6, 9, [3, 0, 0, 0, 0, 3], 0.0)  # oracle.cpp:98
