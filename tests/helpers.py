"""Shared helpers: reference fixtures (tests/support/fixtures.hpp) as edge lists."""
import numpy as np

from oracle import oracle as O


def k(a, b):
    return O.complete_biclique_edges(a, b)


def pairs(lst):
    a = np.array(lst, dtype=np.uint64).reshape(-1, 2)
    return a[:, 0].copy(), a[:, 1].copy()


# fixtures.hpp:31-65
def k22():
    return k(2, 2)


def k32():
    return k(3, 2)


def k24():
    return k(2, 4)


def k33():
    return k(3, 3)


def two_k22():
    return pairs([(1, 1), (1, 2), (2, 1), (2, 2), (3, 3), (3, 4), (4, 3), (4, 4)])


def cycle6():
    return pairs([(1, 1), (2, 1), (2, 2), (3, 2), (3, 3), (1, 3)])


def star15():
    return k(1, 5)


def path4():
    return pairs([(1, 1), (2, 1), (2, 2)])


def named_suite():
    return [k22(), k32(), k24(), k33(), two_k22(), cycle6(), star15(), path4()]
