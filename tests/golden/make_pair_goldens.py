"""Golden pair-type counts and variance bounds from the UNMODIFIED reference (oracle/_ref).

classify_pairs (reference oracle.cpp:60-94) enumerates every butterfly and classifies all
C(bfly, 2) pairs, so the goldens stay at sizes it can finish: the reference tests' named
fixtures, random_bipartite suites (graph.cpp:123-134, the same generator the reference tests
use) and a few denser graphs under raised OracleGuards (up to ~60K butterflies, 1.8e9 pairs).
variance_bounds (oracle.cpp:96-116) is recorded at p = 0.5 and p = 0.1.

  python tests/golden/make_pair_goldens.py     # -> tests/golden/pairs.json (about a minute)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "pairs.json")


def named():
    k = O.complete_biclique_edges
    two_k22 = ([1, 1, 2, 2, 3, 3, 4, 4], [1, 2, 1, 2, 3, 4, 3, 4])
    cycle6 = ([1, 2, 2, 3, 3, 1], [1, 1, 2, 2, 3, 3])
    path4 = ([1, 2, 2], [1, 1, 2])
    return [("k22", k(2, 2)), ("k32", k(3, 2)), ("k24", k(2, 4)), ("k33", k(3, 3)),
            ("two_k22", two_k22), ("cycle6", cycle6), ("star15", k(1, 5)), ("path4", path4),
            ("k55", k(5, 5)), ("k64", k(6, 4))]


def randoms():
    out = []
    for i, (a, b, p) in enumerate([(10, 10, 0.3), (10, 10, 0.5), (10, 10, 0.7), (12, 9, 0.6),
                                   (15, 15, 0.4), (20, 12, 0.35), (8, 30, 0.5), (25, 25, 0.3),
                                   (30, 30, 0.35), (40, 20, 0.3), (35, 35, 0.4), (50, 50, 0.25),
                                   (60, 60, 0.4), (100, 40, 0.3)]):
        try:
            out.append((f"random_{a}x{b}_p{p}_s{7000 + i}", O.random_bipartite_edges(a, b, p, 7000 + i)))
        except O.OracleError:
            pass
    return out


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref/libbfly_ref.so missing: make -C oracle")
    cases = []
    t0 = time.perf_counter()
    for name, (l, r) in named() + randoms():
        l = np.asarray(l, np.uint64)
        r = np.asarray(r, np.uint64)
        ref = O.Ref(l, r)
        c = ref.classify_pairs(max_side=1 << 30, max_butterflies=1 << 62)
        cases.append({"name": name, "left": [int(x) for x in l], "right": [int(x) for x in r],
                      "counts": list(c),
                      "bounds_p0.5": list(ref.variance_bounds(c, 0.5)),
                      "bounds_p0.1": list(ref.variance_bounds(c, 0.1))})
        print(name, c, flush=True)
    obj = {"generated_by": "tests/golden/make_pair_goldens.py",
           "reference_build": "oracle/_ref/libbfly_ref.so (g++ -O3 -DNDEBUG)",
           "fields": ["bfly", "p_0v", "p_1v", "p_2v", "p_1e", "p_1w"],
           "seconds": time.perf_counter() - t0, "cases": cases}
    with open(OUT, "w") as f:
        json.dump(obj, f, indent=0)


if __name__ == "__main__":
    main()
