"""TEST INFRASTRUCTURE ONLY: ctypes front for the CPU parity checker.

Two checkers live under oracle/:
  * ``Oracle``  -- liboracle.so, the plain-C restatement (bfly_oracle.c) of the reference;
  * ``Ref``     -- _ref/libbfly_ref.so, the UNMODIFIED reference sources compiled here
                   (namespace renamed to bfly_ref) behind a C shim (ref_shim.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)
F64P = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)

STATUS_NAMES = {0: "ok", 1: "ArgumentError", 2: "EmptyGraphError", 3: "OverflowError",
                4: "NoWedgesError", 5: "InternalError", 6: "SizeGuardError"}


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}")
        self.status = status


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _check(st: int, where: str):
    if st != 0:
        raise OracleError(st, where)


class _Graph(C.Structure):
    _fields_ = [("L", C.c_uint32), ("R", C.c_uint32), ("m", C.c_uint64),
                ("loff", U64P), ("ladj", U32P), ("roff", U64P), ("radj", U32P),
                ("lids", U64P), ("rids", U64P)]


class _Stats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("left", C.c_uint64), ("right", C.c_uint64), ("m", C.c_uint64),
                ("sum_deg_sq_left", C.c_double), ("sum_deg_sq_right", C.c_double),
                ("wedge_count", C.c_uint64), ("max_degree", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        G = C.POINTER(_Graph)
        sig = {
            "bo_mix64": (C.c_uint64, [C.c_uint64]),
            "bo_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "bo_unit_double": (C.c_double, [C.c_uint64]),
            "bo_bounded_from_bits": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "bo_choose2": (C.c_int, [C.c_uint64, U64P]),
            "bo_graph_from_edges": (C.c_int, [G, U64P, U64P, C.c_uint64]),
            "bo_graph_from_edges_u32": (C.c_int, [G, U32P, U32P, C.c_uint64]),
            "bo_graph_free": (None, [G]),
            "bo_has_edge": (C.c_int, [G, C.c_uint32, C.c_uint32]),
            "bo_edge_at": (C.c_int, [G, C.c_uint64, U32P, U32P]),
            "bo_complete_biclique_edges": (C.c_int, [C.c_uint32, C.c_uint32, C.POINTER(U64P),
                                                     C.POINTER(U64P), U64P]),
            "bo_random_bipartite_edges": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                                    C.POINTER(U64P), C.POINTER(U64P), U64P]),
            "bo_free": (None, [C.c_void_p]),
            "bo_compute_stats": (C.c_int, [G, C.POINTER(_Stats)]),
            "bo_choose_side": (None, [G, C.POINTER(C.c_int), F64P, F64P]),
            "bo_exact_count_side": (C.c_int, [G, C.c_int, C.c_int, U64P]),
            "bo_exact_count": (C.c_int, [G, C.c_int, U64P]),
            "bo_count_per_vertex": (C.c_int, [G, C.c_int, C.c_uint32, U64P]),
            "bo_count_per_edge": (C.c_int, [G, C.c_uint32, C.c_uint32, U64P]),
            "bo_count_all_vertices": (C.c_int, [G, C.c_int, U64P]),
            "bo_count_all_edges": (C.c_int, [G, C.c_int, U64P]),
            "bo_count_edges_subset": (C.c_int, [G, U64P, C.c_uint64, C.c_int, U64P]),
            "bo_count_vertices_subset": (C.c_int, [G, U64P, C.c_uint64, C.c_int, U64P]),
            "bo_build_wedge_index": (C.c_int, [G, U64P, U64P]),
            "bo_vertex_sample_value": (C.c_int, [G, C.c_int, C.c_uint32, F64P]),
            "bo_edge_sample_value": (C.c_int, [G, C.c_uint32, C.c_uint32, F64P]),
            "bo_wedge_sample_value": (C.c_int, [G, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                                C.c_uint32, F64P]),
            "bo_wedge_common_minus_1": (C.c_int, [G, C.c_int, C.c_uint32, C.c_uint32, U64P]),
            "bo_sample_draw": (C.c_int, [G, U64P, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                         U64P, U32P, U32P]),
            "bo_sample_iteration": (C.c_int, [G, U64P, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                              F64P]),
            "bo_run_estimator": (C.c_int, [G, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_uint64, C.c_int, F64P, U64P, F64P, F64P]),
            "bo_run_estimator_ex": (C.c_int, [G, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_uint64, C.c_uint64, C.c_int, F64P, U64P, F64P,
                                              F64P]),
            "bo_fast_esamp_iteration": (C.c_int, [G, C.c_uint64, C.c_uint64, C.c_uint64, F64P,
                                                  U64P, U64P]),
            "bo_count_retained": (C.c_int, [G, U8P, C.c_int, U64P, U64P]),
            "bo_edge_sparsify_value": (C.c_int, [G, U8P, C.c_double, C.c_int, F64P]),
            "bo_color_sparsify_value": (C.c_int, [G, U32P, C.c_uint64, C.c_int, F64P]),
            "bo_edge_sparsify_estimate": (C.c_int, [G, C.c_double, C.c_uint64, C.c_int, F64P,
                                                    U64P, U64P]),
            "bo_color_sparsify_estimate": (C.c_int, [G, C.c_uint64, C.c_uint64, C.c_int, F64P,
                                                     U64P, U64P]),
            "bo_sparsify_run": (C.c_int, [G, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                          C.c_uint64, C.c_int, F64P, F64P]),
            "bo_brute_force_count": (C.c_int, [G, U64P]),
            "bo_classify_pairs": (C.c_int, [G, C.c_uint32, C.c_uint64, U64P]),
            "bo_variance_bounds": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, U64P,
                                             C.c_double, F64P]),
            "bo_pair_counts_by_moments": (C.c_int, [G, C.c_int, U64P]),
            "bo_parse_edge_list": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(U64P),
                                             C.POINTER(U64P), U64P, U64P, C.c_char_p,
                                             C.c_uint64]),
            "bo_serialize_edge_list": (C.c_uint64, [G, C.c_char_p, C.c_uint64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# ---------------------------------------------------------------------------
def complete_biclique_edges(a: int, b: int):
    l, r, m = U64P(), U64P(), C.c_uint64()
    _check(lib().bo_complete_biclique_edges(a, b, C.byref(l), C.byref(r), C.byref(m)),
           "complete_biclique")
    return _take(l, r, m.value)


def random_bipartite_edges(a: int, b: int, p: float, seed: int):
    """graph.cpp:123-134; raises OracleError(EmptyGraphError) when nothing survives."""
    l, r, m = U64P(), U64P(), C.c_uint64()
    st = lib().bo_random_bipartite_edges(a, b, p, seed, C.byref(l), C.byref(r), C.byref(m))
    if st not in (0, 2):
        _check(st, "random_bipartite")
    out = _take(l, r, m.value)
    if st == 2:
        raise OracleError(2, "random_bipartite")
    return out


def _take(l, r, m):
    L = np.ctypeslib.as_array(l, shape=(max(m, 1),))[:m].copy()
    R = np.ctypeslib.as_array(r, shape=(max(m, 1),))[:m].copy()
    lib().bo_free(C.cast(l, C.c_void_p))
    lib().bo_free(C.cast(r, C.c_void_p))
    return L, R


def random_suite_edges(count, max_a, max_b, ps, seed_base):
    """tests/support/fixtures.hpp:68-85 random_suite, as edge lists."""
    out = []
    seed = seed_base
    while len(out) < count:
        pick = Rng(derive_seed(seed_base, seed))
        a = 1 + pick.uniform_index(max_a)
        b = 1 + pick.uniform_index(max_b)
        p = ps[pick.uniform_index(len(ps))]
        try:
            out.append(random_bipartite_edges(a, b, p, seed))
        except OracleError as e:
            if e.status != 2:
                raise
        seed += 1
    return out


def mix64(x):
    return lib().bo_mix64(x)


def derive_seed(s, i):
    return lib().bo_derive_seed(s, i)


def unit_double(bits):
    return lib().bo_unit_double(bits)


def bounded_from_bits(bits, n):
    return lib().bo_bounded_from_bits(bits, n)


def choose2(c):
    out = C.c_uint64()
    _check(lib().bo_choose2(c, C.byref(out)), "choose2")
    return out.value


class Rng:
    """Pure-Python mt19937_64 wrapper over nothing: small-scale use only (fixture picks)."""

    def __init__(self, seed):
        import random  # noqa: F401  (documentational: we implement MT19937-64 directly)
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.mti = 312

    def next(self):
        M = 0xFFFFFFFFFFFFFFFF
        if self.mti >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.mti = 0
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000 & M
        x ^= (x << 37) & 0xFFF7EEE000000000 & M
        x ^= x >> 43
        return x & M

    def uniform_index(self, n):
        if n <= 1:
            return 0
        mask = (1 << (n - 1).bit_length()) - 1
        while True:
            r = self.next() & mask
            if r < n:
                return r


# ---------------------------------------------------------------------------
def parse_text(text: bytes):
    """load_edge_list restated (graph.cpp:75-99): ("ok", l, r) with the edges in line order
    (empty arrays -> the caller's EmptyGraphError) or ("parse", what, line)."""
    lp, rp = U64P(), U64P()
    m, line = C.c_uint64(), C.c_uint64()
    msg = C.create_string_buffer(512)
    st = lib().bo_parse_edge_list(bytes(text), len(text), C.byref(lp), C.byref(rp), C.byref(m),
                                  C.byref(line), msg, 512)
    if st == 6:
        return ("parse", msg.value.decode(), line.value)
    _check(st, "parse_edge_list")
    n = m.value
    l = np.ctypeslib.as_array(lp, shape=(max(n, 1),))[:n].copy()
    r = np.ctypeslib.as_array(rp, shape=(max(n, 1),))[:n].copy()
    libc = C.CDLL(None)
    libc.free(C.cast(lp, C.c_void_p))
    libc.free(C.cast(rp, C.c_void_p))
    return ("ok", l, r)


class Oracle:
    """The C restatement on one graph (built with the reference's from_edges rules)."""

    def __init__(self, l, r, threads: int | None = None):
        self.threads = threads or default_threads()
        l = np.ascontiguousarray(l)
        r = np.ascontiguousarray(r)
        self._g = _Graph()
        if l.dtype == np.uint32 and r.dtype == np.uint32:
            st = lib().bo_graph_from_edges_u32(C.byref(self._g), _p(l, U32P), _p(r, U32P), len(l))
        else:
            l = l.astype(np.uint64)
            r = r.astype(np.uint64)
            st = lib().bo_graph_from_edges(C.byref(self._g), _p(l, U64P), _p(r, U64P), len(l))
        _check(st, "from_edges")

    def __del__(self):
        if getattr(self, "_g", None) is not None and lib() is not None:
            lib().bo_graph_free(C.byref(self._g))
            self._g = None

    # accessors -------------------------------------------------------------
    @property
    def L(self):
        return self._g.L

    @property
    def R(self):
        return self._g.R

    @property
    def m(self):
        return self._g.m

    @property
    def n(self):
        return self._g.L + self._g.R

    def serialize(self) -> bytes:
        """serialize_edge_list restated (graph.cpp:107-112)."""
        n = lib().bo_serialize_edge_list(C.byref(self._g), None, 0)
        buf = C.create_string_buffer(max(n, 1))
        lib().bo_serialize_edge_list(C.byref(self._g), buf, n)
        return buf.raw[:n]

    def csr(self):
        g = self._g
        loff = np.ctypeslib.as_array(g.loff, shape=(g.L + 1,)).copy()
        roff = np.ctypeslib.as_array(g.roff, shape=(g.R + 1,)).copy()
        ladj = np.ctypeslib.as_array(g.ladj, shape=(max(g.m, 1),))[:g.m].copy()
        radj = np.ctypeslib.as_array(g.radj, shape=(max(g.m, 1),))[:g.m].copy()
        lids = np.ctypeslib.as_array(g.lids, shape=(max(g.L, 1),))[:g.L].copy()
        rids = np.ctypeslib.as_array(g.rids, shape=(max(g.R, 1),))[:g.R].copy()
        return loff, ladj, roff, radj, lids, rids

    def degrees(self):
        loff, _, roff, _, _, _ = self.csr()
        return np.diff(loff), np.diff(roff)

    def edge_at(self, k):
        l, r = C.c_uint32(), C.c_uint32()
        _check(lib().bo_edge_at(C.byref(self._g), k, C.byref(l), C.byref(r)), "edge_at")
        return l.value, r.value

    def has_edge(self, l, r):
        return bool(lib().bo_has_edge(C.byref(self._g), l, r))

    # counts ----------------------------------------------------------------
    def compute_stats(self):
        s = _Stats()
        _check(lib().bo_compute_stats(C.byref(self._g), C.byref(s)), "compute_stats")
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    def choose_side(self):
        c, cl, cr = C.c_int(), C.c_double(), C.c_double()
        lib().bo_choose_side(C.byref(self._g), C.byref(c), C.byref(cl), C.byref(cr))
        return c.value, cl.value, cr.value

    def exact_count(self):
        out = C.c_uint64()
        _check(lib().bo_exact_count(C.byref(self._g), self.threads, C.byref(out)), "exact_count")
        return out.value

    def exact_count_side(self, side):
        out = C.c_uint64()
        _check(lib().bo_exact_count_side(C.byref(self._g), side, self.threads, C.byref(out)),
               "exact_count_side")
        return out.value

    def brute_force_count(self):
        out = C.c_uint64()
        _check(lib().bo_brute_force_count(C.byref(self._g), C.byref(out)), "brute_force")
        return out.value

    def classify_pairs(self, max_side=64, max_butterflies=2000):
        """oracle.cpp:60-94 (enumeration): (bfly, p_0v, p_1v, p_2v, p_1e, p_1w)."""
        out = (C.c_uint64 * 6)()
        _check(lib().bo_classify_pairs(C.byref(self._g), max_side, max_butterflies, out),
               "classify_pairs")
        return tuple(int(x) for x in out)

    def pair_counts_by_moments(self):
        """The same six counts from pair moments + local counts (Python ints)."""
        out = (C.c_uint64 * 11)()
        _check(lib().bo_pair_counts_by_moments(C.byref(self._g), self.threads, out),
               "pair_counts_by_moments")
        return (int(out[0]),) + tuple(int(out[1 + 2 * q]) | (int(out[2 + 2 * q]) << 64)
                                      for q in range(5))

    @staticmethod
    def variance_bounds(n, m, wedges, counts, p):
        """oracle.cpp:96-116: (vsamp, esamp, wsamp, espar, clrspar)."""
        cs = (C.c_uint64 * 6)(*counts)
        out = (C.c_double * 5)()
        _check(lib().bo_variance_bounds(n, m, wedges, cs, p, out), "variance_bounds")
        return tuple(out)

    def count_per_vertex(self, side, index):
        out = C.c_uint64()
        _check(lib().bo_count_per_vertex(C.byref(self._g), side, index, C.byref(out)),
               "count_per_vertex")
        return out.value

    def count_per_edge(self, l, r):
        out = C.c_uint64()
        _check(lib().bo_count_per_edge(C.byref(self._g), l, r, C.byref(out)), "count_per_edge")
        return out.value

    def count_all_vertices(self):
        out = np.zeros(self.n, dtype=np.uint64)
        _check(lib().bo_count_all_vertices(C.byref(self._g), self.threads, _p(out, U64P)),
               "count_all_vertices")
        return out

    def count_all_edges(self):
        out = np.zeros(self.m, dtype=np.uint64)
        _check(lib().bo_count_all_edges(C.byref(self._g), self.threads, _p(out, U64P)),
               "count_all_edges")
        return out

    def count_edges_subset(self, ks):
        ks = np.ascontiguousarray(ks, dtype=np.uint64)
        out = np.zeros(len(ks), dtype=np.uint64)
        _check(lib().bo_count_edges_subset(C.byref(self._g), _p(ks, U64P), len(ks), self.threads,
                                           _p(out, U64P)), "count_edges_subset")
        return out

    def count_vertices_subset(self, gids):
        gids = np.ascontiguousarray(gids, dtype=np.uint64)
        out = np.zeros(len(gids), dtype=np.uint64)
        _check(lib().bo_count_vertices_subset(C.byref(self._g), _p(gids, U64P), len(gids),
                                              self.threads, _p(out, U64P)),
               "count_vertices_subset")
        return out

    def build_wedge_index(self):
        prefix = np.zeros(self.n + 1, dtype=np.uint64)
        total = C.c_uint64()
        _check(lib().bo_build_wedge_index(C.byref(self._g), _p(prefix, U64P), C.byref(total)),
               "build_wedge_index")
        return prefix, total.value

    def vertex_sample_value(self, side, index):
        out = C.c_double()
        _check(lib().bo_vertex_sample_value(C.byref(self._g), side, index, C.byref(out)), "vsv")
        return out.value

    def edge_sample_value(self, l, r):
        out = C.c_double()
        _check(lib().bo_edge_sample_value(C.byref(self._g), l, r, C.byref(out)), "esv")
        return out.value

    def wedge_sample_value(self, total, centre_side, centre, v, w):
        out = C.c_double()
        _check(lib().bo_wedge_sample_value(C.byref(self._g), total, centre_side, centre, v, w,
                                           C.byref(out)), "wsv")
        return out.value

    def wedge_common_minus_1(self, centre_side, v, w):
        out = C.c_uint64()
        _check(lib().bo_wedge_common_minus_1(C.byref(self._g), centre_side, v, w, C.byref(out)),
               "wedge_common")
        return out.value

    def sample_draws(self, method, seed, count, prefix=None, total=0):
        """Sample ids of iterations 0..count-1 (sampling.cpp:101-123)."""
        if method == 2 and prefix is None:
            prefix, total = self.build_wedge_index()
        pp = _p(prefix, U64P) if prefix is not None else None
        ids = np.zeros(count, dtype=np.uint64)
        ii = np.zeros(count, dtype=np.uint32)
        jj = np.zeros(count, dtype=np.uint32)
        a, b, c = C.c_uint64(), C.c_uint32(), C.c_uint32()
        for k in range(count):
            _check(lib().bo_sample_draw(C.byref(self._g), pp, total, method, seed, k, C.byref(a),
                                        C.byref(b), C.byref(c)), "sample_draw")
            ids[k], ii[k], jj[k] = a.value, b.value, c.value
        return ids, ii, jj

    def fast_iteration(self, repeats, seed, index):
        """(value, canonical edge id, hits) of fast_esamp_iteration (sampling.cpp:125-147)."""
        v, k, h = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib().bo_fast_esamp_iteration(C.byref(self._g), repeats, seed, index, C.byref(v),
                                             C.byref(k), C.byref(h)), "fast_iteration")
        return v.value, k.value, h.value

    def run_estimator(self, method, iterations, seed, groups=1, group_size=0, values=False,
                      repeats=1000):
        total = iterations if groups == 1 else groups * (group_size or iterations)
        val, done = C.c_double(), C.c_uint64()
        per = np.zeros(max(groups, 1), dtype=np.float64)
        vals = np.zeros(max(total, 1), dtype=np.float64)
        _check(lib().bo_run_estimator_ex(C.byref(self._g), method, iterations, seed, groups,
                                         group_size, repeats, self.threads, C.byref(val),
                                         C.byref(done), _p(per, F64P), _p(vals, F64P)),
               "run_estimator")
        res = {"value": val.value, "iterations_done": done.value,
               "per_group_means": per.tolist() if groups > 1 else []}
        if values:
            res["values"] = vals[:total]
        return res

    def count_retained(self, keep):
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        c, k = C.c_uint64(), C.c_uint64()
        _check(lib().bo_count_retained(C.byref(self._g), _p(keep, U8P), self.threads, C.byref(c),
                                       C.byref(k)), "count_retained")
        return c.value, k.value

    def edge_sparsify_value(self, keep, p):
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        out = C.c_double()
        _check(lib().bo_edge_sparsify_value(C.byref(self._g), _p(keep, U8P), p, self.threads,
                                            C.byref(out)), "edge_sparsify_value")
        return out.value

    def color_sparsify_value(self, colors, n_colors):
        colors = np.ascontiguousarray(colors, dtype=np.uint32)
        out = C.c_double()
        _check(lib().bo_color_sparsify_value(C.byref(self._g), _p(colors, U32P), n_colors,
                                             self.threads, C.byref(out)), "color_sparsify_value")
        return out.value

    def edge_sparsify_estimate(self, p, seed):
        out, c, k = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib().bo_edge_sparsify_estimate(C.byref(self._g), p, seed, self.threads,
                                               C.byref(out), C.byref(c), C.byref(k)), "espar")
        return out.value, c.value, k.value

    def color_sparsify_estimate(self, n_colors, seed):
        out, c, k = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib().bo_color_sparsify_estimate(C.byref(self._g), n_colors, seed, self.threads,
                                                C.byref(out), C.byref(c), C.byref(k)), "cspar")
        return out.value, c.value, k.value

    def sparsify_run(self, sparsifier, p=0.5, colors=2, seed=0, trials=1):
        val = C.c_double()
        per = np.zeros(max(trials, 1), dtype=np.float64)
        _check(lib().bo_sparsify_run(C.byref(self._g), sparsifier, p, colors, seed, trials,
                                     self.threads, C.byref(val), _p(per, F64P)), "sparsify_run")
        return {"value": val.value, "per_group_means": per[:trials].tolist()}


# ---------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libbfly_ref.so"))


def ref_lib():
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libbfly_ref.so")
        R = C.CDLL(path)
        VP = C.c_void_p
        sig = {
            "ref_graph_build": (C.c_int, [U64P, U64P, C.c_uint64, C.POINTER(VP)]),
            "ref_graph_build_u32": (C.c_int, [U32P, U32P, C.c_uint64, C.POINTER(VP)]),
            "ref_complete_biclique": (C.c_int, [C.c_uint32, C.c_uint32, C.POINTER(VP)]),
            "ref_random_bipartite": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                               C.POINTER(VP)]),
            "ref_graph_free": (None, [VP]),
            "ref_graph_sizes": (None, [VP, U32P, U32P, U64P]),
            "ref_graph_export": (None, [VP, U64P, U32P, U64P, U32P, U64P, U64P]),
            "ref_compute_stats": (C.c_int, [VP, U64P, F64P]),
            "ref_choose_side": (C.c_int, [VP, C.POINTER(C.c_int), F64P, F64P]),
            "ref_exact_count": (C.c_int, [VP, U64P]),
            "ref_exact_count_side": (C.c_int, [VP, C.c_int, U64P]),
            "ref_brute_force_count": (C.c_int, [VP, U64P]),
            "ref_classify_pairs": (C.c_int, [VP, C.c_uint32, C.c_uint64, U64P]),
            "ref_variance_bounds": (C.c_int, [VP, U64P, C.c_double, F64P]),
            "ref_count_per_vertex": (C.c_int, [VP, C.c_int, C.c_uint32, U64P]),
            "ref_count_per_edge": (C.c_int, [VP, C.c_uint32, C.c_uint32, U64P]),
            "ref_edge_at": (C.c_int, [VP, C.c_uint64, U32P, U32P]),
            "ref_count_all_vertices": (C.c_int, [VP, C.c_int, U64P]),
            "ref_count_edges": (C.c_int, [VP, U64P, C.c_uint64, C.c_int, U64P]),
            "ref_build_wedge_index": (C.c_int, [VP, U64P, U64P]),
            "ref_vertex_sample_value": (C.c_int, [VP, C.c_int, C.c_uint32, F64P]),
            "ref_edge_sample_value": (C.c_int, [VP, C.c_uint32, C.c_uint32, F64P]),
            "ref_wedge_sample_value": (C.c_int, [VP, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                                 C.c_uint32, F64P]),
            "ref_iteration": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_uint64, F64P]),
            "ref_run_estimator": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_uint64, C.c_uint, F64P, U64P, F64P]),
            "ref_run_estimator_ex": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                               C.c_uint64, C.c_uint64, C.c_uint, F64P, U64P,
                                               F64P]),
            "ref_fast_iteration": (C.c_int, [VP, C.c_uint64, C.c_uint64, C.c_uint64, F64P]),
            "ref_load_text": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p),
                                        C.c_char_p, C.c_uint64, U64P]),
            "ref_serialize": (C.c_int, [VP, C.c_char_p, C.c_uint64, U64P]),
            "ref_edge_sparsify_estimate": (C.c_int, [VP, C.c_double, C.c_uint64, F64P]),
            "ref_color_sparsify_estimate": (C.c_int, [VP, C.c_uint64, C.c_uint64, F64P]),
            "ref_sparsify_run": (C.c_int, [VP, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                           C.c_uint64, F64P, F64P]),
            "ref_mix64": (C.c_uint64, [C.c_uint64]),
            "ref_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "ref_rng_stream_first": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(R, name)
            f.restype = res
            f.argtypes = args
        _ref = R
    return _ref


class Ref:
    """The unmodified reference library (oracle/_ref) on one graph."""

    def __init__(self, l=None, r=None, handle=None):
        self._h = C.c_void_p()
        if handle is not None:
            self._h = handle
            return
        l = np.ascontiguousarray(l)
        r = np.ascontiguousarray(r)
        if l.dtype == np.uint32 and r.dtype == np.uint32:
            st = ref_lib().ref_graph_build_u32(_p(l, U32P), _p(r, U32P), len(l), C.byref(self._h))
        else:
            l = l.astype(np.uint64)
            r = r.astype(np.uint64)
            st = ref_lib().ref_graph_build(_p(l, U64P), _p(r, U64P), len(l), C.byref(self._h))
        _check(st, "ref from_edges")

    @classmethod
    def load_text(cls, text: bytes):
        """load_edge_list on an in-memory stream: ("ok", Ref) | ("parse", what, line) |
        ("empty", what)."""
        h = C.c_void_p()
        msg = C.create_string_buffer(512)
        line = C.c_uint64()
        st = ref_lib().ref_load_text(bytes(text), len(text), C.byref(h), msg, 512, C.byref(line))
        if st == 0:
            return ("ok", cls(handle=h))
        if st == 7:
            return ("parse", msg.value.decode(), line.value)
        if st == 2:
            return ("empty", msg.value.decode())
        raise RuntimeError(f"ref load_text failed ({st}): {msg.value.decode()}")

    def serialize(self) -> bytes:
        n = C.c_uint64()
        _check(ref_lib().ref_serialize(self._h, None, 0, C.byref(n)), "ref serialize")
        buf = C.create_string_buffer(max(n.value, 1))
        _check(ref_lib().ref_serialize(self._h, buf, n.value, C.byref(n)), "ref serialize")
        return buf.raw[:n.value]

    @classmethod
    def complete_biclique(cls, a, b):
        h = C.c_void_p()
        _check(ref_lib().ref_complete_biclique(a, b, C.byref(h)), "ref complete_biclique")
        return cls(handle=h)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            ref_lib().ref_graph_free(self._h)
            self._h = C.c_void_p()

    def sizes(self):
        L, R, m = C.c_uint32(), C.c_uint32(), C.c_uint64()
        ref_lib().ref_graph_sizes(self._h, C.byref(L), C.byref(R), C.byref(m))
        return L.value, R.value, m.value

    def csr(self):
        L, R, m = self.sizes()
        loff = np.zeros(L + 1, np.uint64)
        roff = np.zeros(R + 1, np.uint64)
        ladj = np.zeros(max(m, 1), np.uint32)
        radj = np.zeros(max(m, 1), np.uint32)
        lids = np.zeros(max(L, 1), np.uint64)
        rids = np.zeros(max(R, 1), np.uint64)
        ref_lib().ref_graph_export(self._h, _p(loff, U64P), _p(ladj, U32P), _p(roff, U64P),
                                   _p(radj, U32P), _p(lids, U64P), _p(rids, U64P))
        return loff, ladj[:m], roff, radj[:m], lids[:L], rids[:R]

    def compute_stats(self):
        u = np.zeros(6, np.uint64)
        d = np.zeros(2, np.float64)
        _check(ref_lib().ref_compute_stats(self._h, _p(u, U64P), _p(d, F64P)), "ref stats")
        return {"n": int(u[0]), "left": int(u[1]), "right": int(u[2]), "m": int(u[3]),
                "wedge_count": int(u[4]), "max_degree": int(u[5]),
                "sum_deg_sq_left": float(d[0]), "sum_deg_sq_right": float(d[1])}

    def choose_side(self):
        c, cl, cr = C.c_int(), C.c_double(), C.c_double()
        _check(ref_lib().ref_choose_side(self._h, C.byref(c), C.byref(cl), C.byref(cr)), "ref cs")
        return c.value, cl.value, cr.value

    def exact_count(self):
        out = C.c_uint64()
        _check(ref_lib().ref_exact_count(self._h, C.byref(out)), "ref exact_count")
        return out.value

    def exact_count_side(self, side):
        out = C.c_uint64()
        _check(ref_lib().ref_exact_count_side(self._h, side, C.byref(out)), "ref exact side")
        return out.value

    def brute_force_count(self):
        out = C.c_uint64()
        _check(ref_lib().ref_brute_force_count(self._h, C.byref(out)), "ref brute")
        return out.value

    def classify_pairs(self, max_side=64, max_butterflies=2000):
        out = (C.c_uint64 * 6)()
        _check(ref_lib().ref_classify_pairs(self._h, max_side, max_butterflies, out),
               "ref classify_pairs")
        return tuple(int(x) for x in out)

    def variance_bounds(self, counts, p):
        cs = (C.c_uint64 * 6)(*counts)
        out = (C.c_double * 5)()
        _check(ref_lib().ref_variance_bounds(self._h, cs, p, out), "ref variance_bounds")
        return tuple(out)

    def count_per_vertex(self, side, index):
        out = C.c_uint64()
        _check(ref_lib().ref_count_per_vertex(self._h, side, index, C.byref(out)), "ref cpv")
        return out.value

    def count_per_edge(self, l, r):
        out = C.c_uint64()
        _check(ref_lib().ref_count_per_edge(self._h, l, r, C.byref(out)), "ref cpe")
        return out.value

    def count_all_vertices(self, threads=None):
        L, R, _ = self.sizes()
        out = np.zeros(L + R, np.uint64)
        _check(ref_lib().ref_count_all_vertices(self._h, threads or default_threads(),
                                                _p(out, U64P)), "ref all vertices")
        return out

    def count_edges(self, ks=None, threads=None):
        _, _, m = self.sizes()
        if ks is None:
            out = np.zeros(m, np.uint64)
            _check(ref_lib().ref_count_edges(self._h, None, m, threads or default_threads(),
                                             _p(out, U64P)), "ref edges")
            return out
        ks = np.ascontiguousarray(ks, np.uint64)
        out = np.zeros(len(ks), np.uint64)
        _check(ref_lib().ref_count_edges(self._h, _p(ks, U64P), len(ks),
                                         threads or default_threads(), _p(out, U64P)), "ref edges")
        return out

    def build_wedge_index(self):
        L, R, _ = self.sizes()
        prefix = np.zeros(L + R + 1, np.uint64)
        total = C.c_uint64()
        _check(ref_lib().ref_build_wedge_index(self._h, _p(prefix, U64P), C.byref(total)), "ref wi")
        return prefix, total.value

    def iteration(self, method, seed, index):
        out = C.c_double()
        _check(ref_lib().ref_iteration(self._h, method, seed, index, C.byref(out)), "ref iter")
        return out.value

    def fast_iteration(self, repeats, seed, index):
        """fast_esamp_iteration of Rng::stream(seed, index) (sampling.cpp:143-147)."""
        out = C.c_double()
        _check(ref_lib().ref_fast_iteration(self._h, repeats, seed, index, C.byref(out)),
               "ref fast iter")
        return out.value

    def run_estimator(self, method, iterations, seed, groups=1, group_size=0, threads=1,
                      repeats=1000):
        val, done = C.c_double(), C.c_uint64()
        per = np.zeros(max(groups, 1), np.float64)
        _check(ref_lib().ref_run_estimator_ex(self._h, method, iterations, seed, groups,
                                              group_size, repeats, threads, C.byref(val),
                                              C.byref(done), _p(per, F64P)),
               "ref run_estimator")
        return {"value": val.value, "iterations_done": done.value,
                "per_group_means": per.tolist() if groups > 1 else []}

    def edge_sparsify_estimate(self, p, seed):
        out = C.c_double()
        _check(ref_lib().ref_edge_sparsify_estimate(self._h, p, seed, C.byref(out)), "ref espar")
        return out.value

    def color_sparsify_estimate(self, n, seed):
        out = C.c_double()
        _check(ref_lib().ref_color_sparsify_estimate(self._h, n, seed, C.byref(out)), "ref cspar")
        return out.value

    def sparsify_run(self, sparsifier, p=0.5, colors=2, seed=0, trials=1):
        val = C.c_double()
        per = np.zeros(max(trials, 1), np.float64)
        _check(ref_lib().ref_sparsify_run(self._h, sparsifier, p, colors, seed, trials,
                                          C.byref(val), _p(per, F64P)), "ref sparsify_run")
        return {"value": val.value, "per_group_means": per[:trials].tolist()}
