"""Python mirror of the reference counting API (proj/include/bfly/*.hpp) over the C-ABI.

Names, argument meaning and exception types follow the reference so tests read like
proj/tests/*.cpp. Every call runs on the GPU through libbfly_b200.so; there is no CPU
fallback (a missing library or device raises).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import NamedTuple

import numpy as np

from . import _abi
from ._abi import F64P, U8P, U32P, U64P, VP


# ---- errors.hpp:10-58 -------------------------------------------------------------------
class Error(RuntimeError):
    pass


class ParseError(Error):
    def __init__(self, what: str, line: int = 0):
        super().__init__(what)
        self.line = line


class EmptyGraphError(Error):
    pass


class ArgumentError(Error):
    pass


class NoWedgesError(Error):
    pass


class OverflowError(Error):  # noqa: A001 (reference name)
    pass


class SizeGuardError(Error):
    pass


class InternalError(Error):
    pass


_STATUS = {1: ArgumentError, 2: EmptyGraphError, 3: OverflowError, 4: NoWedgesError, 5: Error,
           6: ParseError}


def _check(status: int):
    if status != 0:
        raise _STATUS.get(status, Error)(_abi.last_error())


def _p(a, t):
    return a.ctypes.data_as(t)


# ---- graph.hpp:11-35 --------------------------------------------------------------------
class Side(IntEnum):
    Left = 0
    Right = 1


def opposite(s: Side) -> Side:
    return Side.Right if s == Side.Left else Side.Left


class VertexRef(NamedTuple):
    side: Side
    index: int


@dataclass
class GraphStats:
    n: int = 0
    left: int = 0
    right: int = 0
    m: int = 0
    sum_deg_sq_left: float = 0.0
    sum_deg_sq_right: float = 0.0
    wedge_count: int = 0
    max_degree: int = 0


@dataclass
class SideChoice:
    chosen: Side = Side.Left
    cost_left: float = 0.0
    cost_right: float = 0.0


class BipartiteGraph:
    """Device-resident graph; from_edges mirrors graph.cpp:31-58 (first-seen dense ids)."""

    def __init__(self, handle):
        self._h = handle
        self._csr = None
        L, R, m = C.c_uint32(), C.c_uint32(), C.c_uint64()
        _check(_abi.lib().bfly_graph_sizes(self._h, C.byref(L), C.byref(R), C.byref(m)))
        self._L, self._R, self._m = L.value, R.value, m.value

    @classmethod
    def from_edges(cls, left, right=None):
        if right is None:  # list of (l, r) pairs
            arr = np.asarray(left, dtype=np.uint64).reshape(-1, 2)
            left, right = arr[:, 0], arr[:, 1]
        left = np.ascontiguousarray(left)
        right = np.ascontiguousarray(right)
        if len(left) != len(right):
            raise ArgumentError("left and right id arrays differ in length")
        h = VP()
        if left.dtype == np.uint32 and right.dtype == np.uint32:
            st = _abi.lib().bfly_graph_build_u32(_p(left, U32P), _p(right, U32P), len(left),
                                                 C.byref(h))
        else:
            if (np.asarray(left).size and (np.min(left) < 0 or np.min(right) < 0)):
                raise ArgumentError("vertex ids must be non-negative")
            l64 = np.ascontiguousarray(left, dtype=np.uint64)
            r64 = np.ascontiguousarray(right, dtype=np.uint64)
            st = _abi.lib().bfly_graph_build_u64(_p(l64, U64P), _p(r64, U64P), len(l64),
                                                 C.byref(h))
        _check(st)
        return cls(h)

    @classmethod
    def from_pairs(cls, pairs):
        """from_edges over the reference's own input layout: an (m, 2) array of uint64
        (left, right) pairs -- the storage of a vector<pair<uint64_t, uint64_t>>
        (bfly_graph_build_pairs)."""
        pairs = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1, 2)
        h = VP()
        _check(_abi.lib().bfly_graph_build_pairs(_p(pairs, U64P), len(pairs), C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, dptr_left: int, dptr_right: int, m: int):
        h = VP()
        _check(_abi.lib().bfly_graph_build_u32_device(VP(dptr_left), VP(dptr_right), m,
                                                      C.byref(h)))
        return cls(h)

    @classmethod
    def from_text(cls, text: bytes):
        """load_edge_list (graph.cpp:75-99), parsed on the device (bfly_graph_load_text);
        ParseError carries .line, the 1-based number of the first malformed line."""
        h = VP()
        line = C.c_uint64()
        text = bytes(text)  # c_char_p passes the bytes object's own buffer (no copy)
        st = _abi.lib().bfly_graph_load_text(text, len(text), C.byref(h), C.byref(line))
        if st == 6:
            raise ParseError(_abi.last_error(), line.value)
        _check(st)
        return cls(h)

    def serialize(self) -> bytes:
        """serialize_edge_list (graph.cpp:107-112), formatted on the device."""
        n = C.c_uint64()
        _check(_abi.lib().bfly_graph_serialize(self._h, None, 0, C.byref(n)))
        buf = np.empty(max(n.value, 1), np.uint8)
        _check(_abi.lib().bfly_graph_serialize(self._h, buf.ctypes.data_as(C.c_char_p), n.value,
                                               C.byref(n)))
        return buf[:n.value].tobytes()

    def close(self):
        if self._h:
            _abi.lib().bfly_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    @property
    def handle(self):
        return self._h

    # graph.hpp:47-51
    def left_count(self) -> int:
        return self._L

    def right_count(self) -> int:
        return self._R

    def side_count(self, s: Side) -> int:
        return self._L if s == Side.Left else self._R

    def vertex_count(self) -> int:
        return self._L + self._R

    def edge_count(self) -> int:
        return self._m

    def export(self):
        """(loff, ladj, roff, radj, reid, lids, rids) copied from the device, cached."""
        if self._csr is None:
            L, R, m = self._L, self._R, self._m
            loff = np.zeros(L + 1, np.uint64)
            roff = np.zeros(R + 1, np.uint64)
            ladj = np.zeros(max(m, 1), np.uint32)
            radj = np.zeros(max(m, 1), np.uint32)
            reid = np.zeros(max(m, 1), np.uint32)
            lids = np.zeros(max(L, 1), np.uint64)
            rids = np.zeros(max(R, 1), np.uint64)
            _check(_abi.lib().bfly_graph_export(self._h, _p(loff, U64P), _p(ladj, U32P),
                                                _p(roff, U64P), _p(radj, U32P), _p(reid, U32P),
                                                _p(lids, U64P), _p(rids, U64P)))
            self._csr = (loff, ladj[:m], roff, radj[:m], reid[:m], lids[:L], rids[:R])
        return self._csr

    def neighbors(self, s: Side, i: int) -> np.ndarray:
        loff, ladj, roff, radj = self.export()[:4]
        if s == Side.Left:
            return ladj[int(loff[i]):int(loff[i + 1])]
        return radj[int(roff[i]):int(roff[i + 1])]

    def degree(self, s, i=None) -> int:
        if i is None:  # VertexRef
            s, i = s.side, s.index
        return len(self.neighbors(s, i))

    def has_edge(self, l: int, r: int) -> bool:
        return bool(self.has_edges([l], [r])[0])

    def has_edges(self, ls, rs) -> np.ndarray:
        ls = np.ascontiguousarray(ls, dtype=np.uint32)
        rs = np.ascontiguousarray(rs, dtype=np.uint32)
        out = np.zeros(len(ls), np.uint8)
        _check(_abi.lib().bfly_has_edge_batch(self._h, _p(ls, U32P), _p(rs, U32P), len(ls),
                                              _p(out, U8P)))
        return out.astype(bool)

    def edge_at(self, k: int):
        l, r = self.edges_at([k])
        return int(l[0]), int(r[0])

    def edges_at(self, ks):
        ks = np.ascontiguousarray(ks, dtype=np.uint64)
        l = np.zeros(len(ks), np.uint32)
        r = np.zeros(len(ks), np.uint32)
        _check(_abi.lib().bfly_edge_at_batch(self._h, _p(ks, U64P), len(ks), _p(l, U32P),
                                             _p(r, U32P)))
        return l, r

    def external_id(self, s: Side, i: int) -> int:
        lids, rids = self.export()[5:7]
        return int(lids[i] if s == Side.Left else rids[i])

    def vertex_at(self, g: int) -> VertexRef:
        if g < self._L:
            return VertexRef(Side.Left, g)
        return VertexRef(Side.Right, g - self._L)

    def global_index(self, v: VertexRef) -> int:
        return v.index if v.side == Side.Left else self._L + v.index


def compute_stats(g: BipartiteGraph) -> GraphStats:
    """graph.cpp:136-155."""
    s = _abi.Stats()
    _check(_abi.lib().bfly_graph_stats(g.handle, C.byref(s)))
    return GraphStats(s.n, s.left, s.right, s.m, s.sum_deg_sq_left, s.sum_deg_sq_right,
                      s.wedge_count, s.max_degree)


# ---- exact.hpp --------------------------------------------------------------------------
def choose_side(g: BipartiteGraph) -> SideChoice:
    """exact.cpp:9-21: chosen = cost_left < cost_right ? Right : Left."""
    c, cl, cr = C.c_int(), C.c_double(), C.c_double()
    _check(_abi.lib().bfly_choose_side(g.handle, C.byref(c), C.byref(cl), C.byref(cr)))
    return SideChoice(Side(c.value), cl.value, cr.value)


def exact_count_side(g: BipartiteGraph, iterate: Side) -> int:
    out = C.c_uint64()
    _check(_abi.lib().bfly_exact_count(g.handle, int(iterate), C.byref(out)))
    return out.value


def exact_count(g: BipartiteGraph) -> int:
    out = C.c_uint64()
    _check(_abi.lib().bfly_exact_count(g.handle, -1, C.byref(out)))
    return out.value


@dataclass
class ExactStats:
    wedges_processed: int
    ref_wedges: int
    bucket_starts: list = field(default_factory=list)
    bucket_wedges: list = field(default_factory=list)
    bucket_entries: list = field(default_factory=list)


def last_exact_stats(g: BipartiteGraph) -> ExactStats:
    w, rw = C.c_uint64(), C.c_uint64()
    bs = np.zeros(13, np.uint64)
    bw = np.zeros(12, np.uint64)
    be = np.zeros(12, np.uint64)
    _check(_abi.lib().bfly_last_exact_stats(g.handle, C.byref(w), C.byref(rw), _p(bs, U64P),
                                            _p(bw, U64P), _p(be, U64P)))
    return ExactStats(w.value, rw.value, [int(x) for x in bs], [int(x) for x in bw],
                      [int(x) for x in be])


def last_dense_stats(g: BipartiteGraph) -> dict:
    """The dense top-hub part of the last exact count (csrc/hubdense.cuh)."""
    o = np.zeros(5, np.uint64)
    _check(_abi.lib().bfly_last_dense_stats(g.handle, _p(o, U64P)))
    return {"hubs": int(o[0]), "words": int(o[1]), "wedges": int(o[2]), "entries": int(o[3]),
            "big_entries": int(o[4])}


# ---- local.hpp ---------------------------------------------------------------------------
def count_per_vertex(g: BipartiteGraph, v: VertexRef) -> int:
    """local.cpp:11-21 (ArgumentError when the index is out of range)."""
    if v.index < 0 or v.index >= g.side_count(v.side):
        raise ArgumentError("vertex index out of range")
    return int(count_vertices(g, [g.global_index(v)])[0])


def count_per_edge(g: BipartiteGraph, l: int, r: int) -> int:
    """local.cpp:23-44 (ArgumentError when (l, r) is out of range or not an edge)."""
    if l < 0 or r < 0:
        raise ArgumentError("edge endpoint out of range")
    ls = np.array([l], np.uint32)
    rs = np.array([r], np.uint32)
    out = np.zeros(1, np.uint64)
    _check(_abi.lib().bfly_local_edge_pairs(g.handle, _p(ls, U32P), _p(rs, U32P), 1,
                                            _p(out, U64P)))
    return int(out[0])


def count_vertices(g: BipartiteGraph, gids) -> np.ndarray:
    """Batched count_per_vertex over global vertex ids (per-sample kernel)."""
    gids = np.ascontiguousarray(gids, dtype=np.uint64)
    out = np.zeros(len(gids), np.uint64)
    _check(_abi.lib().bfly_local_vertex_batch(g.handle, _p(gids, U64P), len(gids),
                                              _p(out, U64P)))
    return out


def count_edges(g: BipartiteGraph, ks) -> np.ndarray:
    """Batched count_per_edge(edge_at(k)) over canonical edge ids (per-sample kernel)."""
    ks = np.ascontiguousarray(ks, dtype=np.uint64)
    out = np.zeros(len(ks), np.uint64)
    _check(_abi.lib().bfly_local_edge_batch(g.handle, _p(ks, U64P), len(ks), _p(out, U64P)))
    return out


def last_sample_path(g: BipartiteGraph) -> str:
    """Which path served the last vertex/edge sample batch on g."""
    return {0: "per-sample", 1: "all-subjects+gather"}.get(
        _abi.lib().bfly_last_sample_path(g.handle), "?")


def count_all_vertices(g: BipartiteGraph) -> np.ndarray:
    out = np.zeros(max(g.vertex_count(), 1), np.uint64)
    _check(_abi.lib().bfly_local_vertex_all(g.handle, _p(out, U64P)))
    return out[:g.vertex_count()]


def count_all_edges(g: BipartiteGraph) -> np.ndarray:
    out = np.zeros(max(g.edge_count(), 1), np.uint64)
    _check(_abi.lib().bfly_local_edge_all(g.handle, _p(out, U64P)))
    return out[:g.edge_count()]


# ---- sampling.hpp (outcome values; the estimator lives in the C++ host library) -----------
@dataclass
class WedgeIndex:
    prefix: np.ndarray
    total: int


def build_wedge_index(g: BipartiteGraph) -> WedgeIndex:
    prefix = np.zeros(g.vertex_count() + 1, np.uint64)
    total = C.c_uint64()
    _check(_abi.lib().bfly_wedge_index(g.handle, _p(prefix, U64P), C.byref(total)))
    return WedgeIndex(prefix, total.value)


def wedge_common_minus_1(g: BipartiteGraph, centres, i, j) -> np.ndarray:
    c = np.ascontiguousarray(centres, dtype=np.uint64)
    i = np.ascontiguousarray(i, dtype=np.uint32)
    j = np.ascontiguousarray(j, dtype=np.uint32)
    out = np.zeros(len(c), np.uint64)
    _check(_abi.lib().bfly_wedge_batch(g.handle, _p(c, U64P), _p(i, U32P), _p(j, U32P), len(c),
                                       _p(out, U64P)))
    return out


def vertex_sample_value(g: BipartiteGraph, v: VertexRef) -> float:
    """sampling.cpp:75-78."""
    return float(count_per_vertex(g, v)) * float(g.vertex_count()) / 4.0


def edge_sample_value(g: BipartiteGraph, l: int, r: int) -> float:
    """sampling.cpp:80-83."""
    return float(count_per_edge(g, l, r)) * float(g.edge_count()) / 4.0


def wedge_sample_value(g: BipartiteGraph, total_wedges: int, center: VertexRef, v: int,
                       w: int) -> float:
    """sampling.cpp:85-91: |N(v) & N(w)| - 1 over the leaf side, scaled (no adjacency
    check, uint64 arithmetic, exactly like the reference)."""
    leaf = opposite(center.side)
    common = int(common_neighbors(g, leaf, [v], [w])[0])
    return float((common - 1) % (1 << 64)) * float(total_wedges) / 4.0


def common_neighbors(g: BipartiteGraph, side: Side, vs, ws) -> np.ndarray:
    """|N(v) & N(w)| for same-side vertex pairs (sampling.cpp:22-36), batched on the GPU."""
    vs = np.ascontiguousarray(vs, dtype=np.uint32)
    ws = np.ascontiguousarray(ws, dtype=np.uint32)
    out = np.zeros(len(vs), np.uint64)
    _check(_abi.lib().bfly_common_neighbors_batch(g.handle, int(side), _p(vs, U32P),
                                                  _p(ws, U32P), len(vs), _p(out, U64P)))
    return out


class Method(IntEnum):
    Vertex = 0
    Edge = 1
    Wedge = 2
    FastEdge = 3


@dataclass
class Estimate:
    value: float = 0.0
    iterations_done: int = 0
    per_group_means: list = field(default_factory=list)
    trace: list = field(default_factory=list)  # (iteration, estimate, elapsed_seconds)


def _host_check(status: int):
    if status != 0:
        msg = _abi.host().bfly_host_last_error()
        raise _STATUS.get(status, Error)(msg.decode() if msg else "")


def run_estimator(g: BipartiteGraph, method: Method, iterations: int = 0, seed: int = 0,
                  groups: int = 1, group_size: int = 0, threads: int = 1,
                  time_budget_seconds: float = 0.0, record_trace: bool = False,
                  fast_edge_repeats: int = 1000) -> Estimate:
    """sampling.cpp:206-278 through the C++ facade: seeded sample ids and batched per-sample
    counts on the GPU, index-ordered double reduction on the host."""
    val, done = C.c_double(), C.c_uint64()
    per = np.zeros(max(groups, 1), np.float64)
    cap = 128
    tr = np.zeros(3 * cap, np.float64)
    tl = C.c_uint64(cap)
    _host_check(_abi.host().bfly_host_run_estimator_ex(
        g.handle, int(method), iterations, time_budget_seconds, seed, groups, group_size,
        fast_edge_repeats, 1 if record_trace else 0, threads, C.byref(val), C.byref(done),
        _p(per, F64P), _p(tr, F64P), C.byref(tl)))
    trace = [(int(tr[3 * i]), float(tr[3 * i + 1]), float(tr[3 * i + 2]))
             for i in range(min(tl.value, cap))] if record_trace else []
    return Estimate(val.value, done.value, per.tolist() if groups > 1 else [], trace)


def time_from_pairs(left, right, reps: int = 3):
    """Wall ms of the reference-signature sequence through the C++ facade:
    BipartiteGraph::from_edges(const vector<pair<u64,u64>>&) + exact_count, per repetition
    (the vector is built before timing); returns (ms list, count)."""
    left = np.ascontiguousarray(left, np.uint32)
    right = np.ascontiguousarray(right, np.uint32)
    ms = np.zeros(reps, np.float64)
    cnt = C.c_uint64()
    _host_check(_abi.host().bfly_host_time_from_pairs(_p(left, U32P), _p(right, U32P), len(left),
                                                      reps, _p(ms, F64P), C.byref(cnt)))
    return ms.tolist(), cnt.value


def sample_ids(g: BipartiteGraph, method: Method, seed: int, first: int, count: int,
               threads: int = 8):
    """Outcome ids of iterations [first, first+count) from Rng::stream(seed, i)."""
    ids = np.zeros(count, np.uint64)
    ii = np.zeros(count, np.uint32)
    jj = np.zeros(count, np.uint32)
    _host_check(_abi.host().bfly_host_sample_ids(g.handle, int(method), seed, first, count,
                                                 threads, _p(ids, U64P), _p(ii, U32P),
                                                 _p(jj, U32P)))
    return ids, ii, jj


def sample_batch(g: BipartiteGraph, method: Method, seed: int, first: int, count: int):
    """Per-sample integers of iterations [first, first+count) with the sample ids drawn on the
    GPU (bfly_sample_batch); returns (counts, ids, i, j)."""
    cnt = np.zeros(count, np.uint64)
    ids = np.zeros(count, np.uint64)
    ii = np.zeros(count, np.uint32)
    jj = np.zeros(count, np.uint32)
    _check(_abi.lib().bfly_sample_batch(g.handle, int(method), seed, first, count, _p(cnt, U64P),
                                        _p(ids, U64P), _p(ii, U32P), _p(jj, U32P)))
    return cnt, ids, ii, jj


def fast_edge_batch(g: BipartiteGraph, seed: int, first: int, count: int, repeats: int = 1000):
    """Method::FastEdge iterations [first, first+count) on the GPU (bfly_fast_edge_batch):
    (values, hits, canonical edge ids)."""
    vals = np.zeros(count, np.float64)
    hits = np.zeros(count, np.uint64)
    eids = np.zeros(count, np.uint64)
    _check(_abi.lib().bfly_fast_edge_batch(g.handle, seed, first, count, repeats, _p(vals, F64P),
                                           _p(hits, U64P), _p(eids, U64P)))
    return vals, hits, eids


# ---- sparsify.hpp --------------------------------------------------------------------------
def sparsify_run(g: BipartiteGraph, sparsifier: int, p: float = 0.5, colors: int = 2,
                 seed: int = 0, trials: int = 1) -> Estimate:
    """sparsify.cpp:73-94 (sparsifier 0 = edge / ESpar, 1 = colour / CSpar)."""
    val = C.c_double()
    per = np.zeros(max(trials, 1), np.float64)
    _host_check(_abi.host().bfly_host_sparsify_run(g.handle, sparsifier, p, colors, seed, trials,
                                                   C.byref(val), _p(per, F64P)))
    return Estimate(val.value, trials, per[:trials].tolist())

def _check_p(p):
    if not (p > 0.0 and p <= 1.0):
        raise ArgumentError("retention probability must be in (0, 1]")


# ---- pair types and variance bounds (oracle.hpp:13-58, oracle.cpp:60-116) ------------------
@dataclass
class OracleGuards:
    max_side: int = 64
    max_butterflies: int = 2000


@dataclass
class PairTypeCounts:
    bfly: int = 0
    p_0v: int = 0
    p_1v: int = 0
    p_2v: int = 0
    p_1e: int = 0
    p_1w: int = 0

    def p_V(self) -> int:
        return self.p_1v + self.p_2v + self.p_1e + self.p_1w

    def p_E(self) -> int:
        return self.p_1e + self.p_1w

    def total_pairs(self) -> int:
        return self.p_0v + self.p_1v + self.p_2v + self.p_1e + self.p_1w

    def as_tuple(self):
        return (self.bfly, self.p_0v, self.p_1v, self.p_2v, self.p_1e, self.p_1w)


@dataclass
class VarianceBounds:
    vsamp: float
    esamp: float
    wsamp: float
    espar: float
    clrspar: float


def classify_pairs_at_scale(g: BipartiteGraph) -> PairTypeCounts:
    """Pair-type counts on the GPU by counting identities (bfly_pair_type_counts); no guards,
    counts are exact Python ints (they exceed 64 bits on large graphs)."""
    c = _abi.PairCounts()
    _check(_abi.lib().bfly_pair_type_counts(g.handle, C.byref(c)))
    w = lambda a: int(a[0]) | (int(a[1]) << 64)  # noqa: E731
    return PairTypeCounts(int(c.bfly), w(c.p_0v), w(c.p_1v), w(c.p_2v), w(c.p_1e), w(c.p_1w))


def classify_pairs(g: BipartiteGraph, guards: OracleGuards = None) -> PairTypeCounts:
    """oracle.cpp:60-94 contract: the same guards and SizeGuardError messages."""
    guards = guards or OracleGuards()
    if g.left_count() > guards.max_side or g.right_count() > guards.max_side:
        raise SizeGuardError(f"oracle guard: side exceeds {guards.max_side} vertices "
                             "(raise the guard to override)")
    b = exact_count(g)
    if b > guards.max_butterflies:
        raise SizeGuardError(f"oracle guard: {b} butterflies exceeds pair classification limit "
                             f"of {guards.max_butterflies} (raise the guard to override)")
    return classify_pairs_at_scale(g)


def variance_bounds(stats: GraphStats, c: PairTypeCounts, p: float) -> VarianceBounds:
    """oracle.cpp:96-116 (operation order kept; each count converted to double once)."""
    if not (p > 0.0 and p <= 1.0):
        raise ArgumentError("retention probability must be in (0, 1]")
    bfly, n, m, wedges = float(c.bfly), float(stats.n), float(stats.m), float(stats.wedge_count)
    inv = 1.0 / p
    p1w2, p1e2, p2v2 = 2.0 * float(c.p_1w), 2.0 * float(c.p_1e), 2.0 * float(c.p_2v)
    return VarianceBounds(
        n * (bfly + float(c.p_V())) / 4.0,
        m * (bfly + float(c.p_E())) / 4.0,
        wedges * (bfly + float(c.p_1w)) / 4.0,
        bfly * inv * inv * inv * inv + p1w2 * inv * inv + p1e2 * inv,
        bfly * inv * inv * inv + p1w2 * inv * inv + (p1e2 + p2v2) * inv)


def espar_count(g: BipartiteGraph, p: float, seed: int):
    """(retained butterflies, retained edges) of the ESpar subgraph (sparsify.cpp:57-63)."""
    c, k = C.c_uint64(), C.c_uint64()
    _check(_abi.lib().bfly_espar_count(g.handle, p, seed, C.byref(c), C.byref(k)))
    return c.value, k.value


def cspar_count(g: BipartiteGraph, n_colors: int, seed: int):
    c, k = C.c_uint64(), C.c_uint64()
    _check(_abi.lib().bfly_cspar_count(g.handle, n_colors, seed, C.byref(c), C.byref(k)))
    return c.value, k.value


def sparsify_stats(g: BipartiteGraph, collect: int = -1) -> dict:
    """Figures of the last sparsify call on g (bfly_sparsify_stats); collect=1/0 switches the
    retained-graph statistics (W_C', n') on/off for later calls."""
    out = np.zeros(6, np.uint64)
    _check(_abi.lib().bfly_sparsify_stats(g.handle, collect, _p(out, U64P)))
    keys = ("kept", "peeled_edges", "sub_left", "sub_right", "retained_wc", "retained_n")
    return {k: int(v) for k, v in zip(keys, out)}


def edge_sparsify_value(g: BipartiteGraph, keep, p: float) -> float:
    """sparsify.cpp:36-41: count * inv * inv * inv * inv (multiplication order kept)."""
    _check_p(p)
    keep = np.ascontiguousarray(keep, dtype=np.uint8)
    if len(keep) != g.edge_count():
        raise ArgumentError("keep mask size mismatch")
    c, k = C.c_uint64(), C.c_uint64()
    _check(_abi.lib().bfly_keep_mask_count(g.handle, _p(keep, U8P), C.byref(c), C.byref(k)))
    inv = 1.0 / p
    return float(c.value) * inv * inv * inv * inv


def color_sparsify_value(g: BipartiteGraph, colors, n_colors: int) -> float:
    """sparsify.cpp:43-55: count * n * n * n."""
    if n_colors == 0:
        raise ArgumentError("palette must have at least one color")
    colors = np.ascontiguousarray(colors, dtype=np.uint32)
    if len(colors) != g.vertex_count():
        raise ArgumentError("color vector size mismatch")
    c, k = C.c_uint64(), C.c_uint64()
    _check(_abi.lib().bfly_color_mask_count(g.handle, _p(colors, U32P), C.byref(c), C.byref(k)))
    n = float(n_colors)
    return float(c.value) * n * n * n


def edge_sparsify_estimate(g: BipartiteGraph, p: float, seed: int) -> float:
    _check_p(p)
    c, _ = espar_count(g, p, seed)
    inv = 1.0 / p
    return float(c) * inv * inv * inv * inv


def color_sparsify_estimate(g: BipartiteGraph, n_colors: int, seed: int) -> float:
    if n_colors == 0:
        raise ArgumentError("palette must have at least one color")
    c, _ = cspar_count(g, n_colors, seed)
    n = float(n_colors)
    return float(c) * n * n * n


# ---- instrumentation ---------------------------------------------------------------------
def profile_enable(on: bool = True):
    _abi.lib().bfly_profile_enable(1 if on else 0)


def profile_reset():
    _abi.lib().bfly_profile_reset()


def profile_snapshot() -> dict:
    lib = _abi.lib()
    out = {}
    for i in range(lib.bfly_profile_count()):
        name, ms, n = C.c_char_p(), C.c_double(), C.c_uint64()
        _check(lib.bfly_profile_get(i, C.byref(name), C.byref(ms), C.byref(n)))
        out[name.value.decode()] = (ms.value, n.value)
    return out


def set_stream(stream_ptr: int):
    """Run handles built later on this thread on a caller-owned cudaStream_t (0 = private)."""
    _abi.lib().bfly_set_stream(VP(stream_ptr) if stream_ptr else None)


def launch_count() -> int:
    return int(_abi.lib().bfly_launch_count())


def trim_pool(keep_bytes: int = 0):
    """Release the engine pool's unused device memory beyond keep_bytes (bfly_trim_pool)."""
    _check(_abi.lib().bfly_trim_pool(keep_bytes))


def device_ok() -> bool:
    return bool(_abi.lib().bfly_device_ok())


# ---- synthetic inputs (bench / tests) -------------------------------------------------------
def synth_uniform(U: int, V: int, m: int, seed: int):
    l = np.zeros(m, np.uint32)
    r = np.zeros(m, np.uint32)
    st = _abi.synth().bfly_synth_uniform(U, V, m, seed, _p(l, U32P), _p(r, U32P))
    if st:
        raise ArgumentError(f"synth_uniform failed ({st})")
    return l, r


def synth_chung_lu(U: int, V: int, m: int, gamma_u: float, gamma_v: float, seed: int,
                   max_degree: int = 0):
    l = np.zeros(m, np.uint32)
    r = np.zeros(m, np.uint32)
    st = _abi.synth().bfly_synth_chung_lu(U, V, m, gamma_u, gamma_v, max_degree, seed,
                                          _p(l, U32P), _p(r, U32P))
    if st:
        raise ArgumentError(f"synth_chung_lu failed ({st})")
    return l, r
