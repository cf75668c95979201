// bfly_b200_host.cpp -- implementation of the C++ facade (bfly_b200.hpp) over the C-ABI,
// plus C exports (bfly_host.h) of the host-side estimator drivers for Python callers.
//
// Division of labour: every butterfly count (exact, per-vertex, per-edge, per-sample,
// sparsified) is computed on the GPU by libbfly_b200.so. The host does what the reference
// does outside its counting loops: seeded mt19937_64 sample-id derivation
// (sampling.cpp:101-123, rng.hpp:36-62), index-ordered double reductions and median of
// group means (sampling.cpp:183-202), and the sparsifier scaling (sparsify.cpp:36-55).
#include "bfly_b200.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <mutex>
#include <thread>
#include <type_traits>

#include "../../include/bfly_b200.h"
#include "bfly_host.h"

namespace bfly {

namespace {

[[noreturn]] void raise(int status) {
  const char* msg = bfly_last_error();
  std::string m = msg ? msg : "";
  switch (status) {
    case BFLY_ARGUMENT: throw ArgumentError(m);
    case BFLY_EMPTY: throw EmptyGraphError(m);
    case BFLY_OVERFLOW: throw OverflowError(m);
    case BFLY_NO_WEDGES: throw NoWedgesError(m);
    default: throw Error(m.empty() ? "bfly_b200 internal error" : m);
  }
}

inline void ck(int status) {
  if (status != BFLY_OK) raise(status);
}

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t) {
  return std::chrono::duration<double>(Clock::now() - t).count();
}

}  // namespace

void throw_status(int status) {
  if (status != BFLY_OK) raise(status);
}

// ---- checked.hpp:9-27 ------------------------------------------------------------------------
uint64_t checked_add(uint64_t a, uint64_t b) {
  uint64_t r;
  if (__builtin_add_overflow(a, b, &r)) throw OverflowError("64-bit counter overflow in addition");
  return r;
}
uint64_t checked_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  if (__builtin_mul_overflow(a, b, &r))
    throw OverflowError("64-bit counter overflow in multiplication");
  return r;
}
uint64_t choose2(uint64_t c) {
  if (c < 2) return 0;
  return (c % 2 == 0) ? checked_mul(c / 2, c - 1) : checked_mul(c, (c - 1) / 2);
}

// ---- rng.hpp:10-58 -----------------------------------------------------------------------------
uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t seed, uint64_t index) { return mix64(mix64(seed) ^ mix64(index)); }
double unit_double(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
uint64_t bounded_from_bits(uint64_t bits, uint64_t n) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(bits) * n) >> 64);
}
uint64_t Rng::uniform_index(uint64_t n) {
  if (n <= 1) return 0;
  const uint64_t mask = ~uint64_t{0} >> __builtin_clzll(n - 1);
  uint64_t r;
  do {
    r = next() & mask;
  } while (r >= n);
  return r;
}

// ---- graph -------------------------------------------------------------------------------------
struct BipartiteGraph::Mirror {
  std::vector<uint64_t> loff, roff, lids, rids;
  std::vector<uint32_t> ladj, radj;
};

namespace {
std::shared_ptr<bfly_graph> own(bfly_graph* h, bool owning) {
  if (owning) return std::shared_ptr<bfly_graph>(h, [](bfly_graph* p) { bfly_graph_free(p); });
  return std::shared_ptr<bfly_graph>(h, [](bfly_graph*) {});
}
}  // namespace

BipartiteGraph BipartiteGraph::adopt(bfly_graph* handle, bool owning) {
  if (!handle) throw ArgumentError("null graph handle");
  BipartiteGraph g;
  g.h_ = own(handle, owning);
  ck(bfly_graph_sizes(handle, &g.L_, &g.R_, &g.m_));
  g.mirror_ = std::make_shared<Mirror>();
  return g;
}

BipartiteGraph BipartiteGraph::from_edges(
    const std::vector<std::pair<uint64_t, uint64_t>>& edges) {
  // the vector's storage is the interleaved (left, right) layout bfly_graph_build_pairs takes
  static_assert(sizeof(std::pair<uint64_t, uint64_t>) == 2 * sizeof(uint64_t) &&
                    std::is_standard_layout_v<std::pair<uint64_t, uint64_t>>,
                "pair<uint64_t, uint64_t> must be two packed uint64_t");
  bfly_graph* h = nullptr;
  ck(bfly_graph_build_pairs(reinterpret_cast<const uint64_t*>(edges.data()), edges.size(), &h));
  return adopt(h, true);
}

BipartiteGraph BipartiteGraph::from_edges_u32(const uint32_t* left, const uint32_t* right,
                                              uint64_t m) {
  bfly_graph* h = nullptr;
  ck(bfly_graph_build_u32(left, right, m, &h));
  return adopt(h, true);
}

const BipartiteGraph::Mirror& BipartiteGraph::mirror() const {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  Mirror& mr = *mirror_;
  if (mr.loff.empty()) {
    mr.loff.resize(uint64_t{L_} + 1);
    mr.roff.resize(uint64_t{R_} + 1);
    mr.ladj.resize(m_);
    mr.radj.resize(m_);
    mr.lids.resize(L_);
    mr.rids.resize(R_);
    ck(bfly_graph_export(h_.get(), mr.loff.data(), mr.ladj.data(), mr.roff.data(),
                         mr.radj.data(), nullptr, mr.lids.data(), mr.rids.data()));
  }
  return mr;
}

std::span<const uint32_t> BipartiteGraph::neighbors(Side s, uint32_t i) const {
  if (i >= side_count(s)) throw ArgumentError("vertex index out of range");
  const Mirror& mr = mirror();
  const auto& off = s == Side::Left ? mr.loff : mr.roff;
  const auto& adj = s == Side::Left ? mr.ladj : mr.radj;
  return {adj.data() + off[i], static_cast<size_t>(off[i + 1] - off[i])};
}

uint32_t BipartiteGraph::degree(Side s, uint32_t i) const {
  return static_cast<uint32_t>(neighbors(s, i).size());
}

bool BipartiteGraph::has_edge(uint32_t l, uint32_t r) const {
  auto la = neighbors(Side::Left, l);
  auto ra = neighbors(Side::Right, r);
  if (la.size() <= ra.size()) return std::binary_search(la.begin(), la.end(), r);
  return std::binary_search(ra.begin(), ra.end(), l);
}

std::pair<uint32_t, uint32_t> BipartiteGraph::edge_at(uint64_t k) const {
  if (k >= m_) throw ArgumentError("edge index out of range");
  const Mirror& mr = mirror();
  auto it = std::upper_bound(mr.loff.begin(), mr.loff.end(), k);
  const uint32_t l = static_cast<uint32_t>(it - mr.loff.begin() - 1);
  return {l, mr.ladj[k]};
}

uint64_t BipartiteGraph::external_id(Side s, uint32_t i) const {
  if (i >= side_count(s)) throw ArgumentError("vertex index out of range");
  const Mirror& mr = mirror();
  return s == Side::Left ? mr.lids[i] : mr.rids[i];
}

BipartiteGraph load_edge_list(std::istream& in) {  // graph.cpp:75-99
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  bfly_graph* h = nullptr;
  uint64_t line = 0;
  const int st = bfly_graph_load_text(text.data(), text.size(), &h, &line);
  if (st == BFLY_PARSE) {  // the C-ABI message carries the reference's " (line N)" suffix
    std::string m = bfly_last_error();
    const std::string suffix = " (line " + std::to_string(line) + ")";
    if (m.size() >= suffix.size() && m.compare(m.size() - suffix.size(), suffix.size(), suffix) == 0)
      m.resize(m.size() - suffix.size());
    throw ParseError(m, line);
  }
  ck(st);
  return BipartiteGraph::adopt(h, true);
}

BipartiteGraph load_edge_list_file(const std::string& path) {  // graph.cpp:101-105
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error("cannot open '" + path + "'");
  return load_edge_list(in);
}

void serialize_edge_list(const BipartiteGraph& g, std::ostream& out) {  // graph.cpp:107-112
  uint64_t len = 0;
  ck(bfly_graph_serialize(g.device(), nullptr, 0, &len));
  std::string buf(len, '\0');
  ck(bfly_graph_serialize(g.device(), buf.data(), len, &len));
  out.write(buf.data(), static_cast<std::streamsize>(len));
}

BipartiteGraph complete_biclique(uint32_t a, uint32_t b) {  // graph.cpp:114-121
  if (a == 0 || b == 0) throw ArgumentError("biclique sides must be at least 1");
  std::vector<std::pair<uint64_t, uint64_t>> edges;
  edges.reserve(uint64_t{a} * b);
  for (uint32_t i = 1; i <= a; ++i)
    for (uint32_t j = 1; j <= b; ++j) edges.emplace_back(i, j);
  return BipartiteGraph::from_edges(edges);
}

BipartiteGraph random_bipartite(uint32_t a, uint32_t b, double p, uint64_t seed) {  // :123-134
  if (a == 0 || b == 0) throw ArgumentError("side sizes must be at least 1");
  if (!(p >= 0.0 && p <= 1.0)) throw ArgumentError("edge probability must be in [0, 1]");
  Rng rng(seed);
  std::vector<std::pair<uint64_t, uint64_t>> edges;
  for (uint32_t i = 1; i <= a; ++i)
    for (uint32_t j = 1; j <= b; ++j)
      if (rng.uniform_unit() < p) edges.emplace_back(i, j);
  if (edges.empty())
    throw EmptyGraphError("random instance came out empty after normalization");
  return BipartiteGraph::from_edges(edges);
}

GraphStats compute_stats(const BipartiteGraph& g) {
  bfly_stats s{};
  ck(bfly_graph_stats(g.device(), &s));
  GraphStats o;
  o.n = s.n;
  o.left = s.left;
  o.right = s.right;
  o.m = s.m;
  o.sum_deg_sq_left = s.sum_deg_sq_left;
  o.sum_deg_sq_right = s.sum_deg_sq_right;
  o.wedge_count = s.wedge_count;
  o.max_degree = s.max_degree;
  return o;
}

// ---- pair types (oracle.cpp:60-116) ----------------------------------------------------------------
PairTypeCountsWide classify_pairs_at_scale(const BipartiteGraph& g) {
  bfly_pair_counts c{};
  ck(bfly_pair_type_counts(g.device(), &c));
  auto wide = [](const uint64_t* w) { return (static_cast<unsigned __int128>(w[1]) << 64) | w[0]; };
  PairTypeCountsWide o;
  o.bfly = c.bfly;
  o.p_0v = wide(c.p_0v);
  o.p_1v = wide(c.p_1v);
  o.p_2v = wide(c.p_2v);
  o.p_1e = wide(c.p_1e);
  o.p_1w = wide(c.p_1w);
  return o;
}

PairTypeCounts classify_pairs(const BipartiteGraph& g, const OracleGuards& guards) {
  // oracle.cpp:13-17 (check_side_guard), :62-67 (butterfly limit)
  if (g.left_count() > guards.max_side || g.right_count() > guards.max_side)
    throw SizeGuardError("oracle guard: side exceeds " + std::to_string(guards.max_side) +
                         " vertices (raise the guard to override)");
  const uint64_t b = exact_count(g);
  if (b > guards.max_butterflies)
    throw SizeGuardError("oracle guard: " + std::to_string(b) +
                         " butterflies exceeds pair classification limit of " +
                         std::to_string(guards.max_butterflies) +
                         " (raise the guard to override)");
  const PairTypeCountsWide w = classify_pairs_at_scale(g);
  auto narrow = [](unsigned __int128 x) {
    if (x >> 64) throw OverflowError("pair count exceeds 64 bits");
    return static_cast<uint64_t>(x);
  };
  PairTypeCounts o;
  o.bfly = w.bfly;
  o.p_0v = narrow(w.p_0v);
  o.p_1v = narrow(w.p_1v);
  o.p_2v = narrow(w.p_2v);
  o.p_1e = narrow(w.p_1e);
  o.p_1w = narrow(w.p_1w);
  return o;
}

namespace {
// oracle.cpp:96-116, operation order kept (inputs already converted to double)
VarianceBounds bounds_of(const GraphStats& stats, double bfly, double pV, double pE, double p1w,
                         double p1e, double p2v, double p) {
  if (!(p > 0.0 && p <= 1.0)) throw ArgumentError("retention probability must be in (0, 1]");
  VarianceBounds b;
  const double n = static_cast<double>(stats.n), m = static_cast<double>(stats.m),
               wedges = static_cast<double>(stats.wedge_count);
  b.vsamp = n * (bfly + pV) / 4.0;
  b.esamp = m * (bfly + pE) / 4.0;
  b.wsamp = wedges * (bfly + p1w) / 4.0;
  const double inv = 1.0 / p, p1w2 = 2.0 * p1w, p1e2 = 2.0 * p1e, p2v2 = 2.0 * p2v;
  b.espar = bfly * inv * inv * inv * inv + p1w2 * inv * inv + p1e2 * inv;
  b.clrspar = bfly * inv * inv * inv + p1w2 * inv * inv + (p1e2 + p2v2) * inv;
  return b;
}
}  // namespace

VarianceBounds variance_bounds(const GraphStats& stats, const PairTypeCounts& c, double p) {
  return bounds_of(stats, static_cast<double>(c.bfly), static_cast<double>(c.p_V()),
                   static_cast<double>(c.p_E()), static_cast<double>(c.p_1w),
                   static_cast<double>(c.p_1e), static_cast<double>(c.p_2v), p);
}

VarianceBounds variance_bounds(const GraphStats& stats, const PairTypeCountsWide& c, double p) {
  return bounds_of(stats, static_cast<double>(c.bfly),
                   static_cast<double>(c.p_1v + c.p_2v + c.p_1e + c.p_1w),
                   static_cast<double>(c.p_1e + c.p_1w), static_cast<double>(c.p_1w),
                   static_cast<double>(c.p_1e), static_cast<double>(c.p_2v), p);
}

// ---- exact ---------------------------------------------------------------------------------------
SideChoice choose_side(const BipartiteGraph& g) {
  SideChoice c;
  int chosen = 0;
  ck(bfly_choose_side(g.device(), &chosen, &c.cost_left, &c.cost_right));
  c.chosen = chosen == BFLY_SIDE_LEFT ? Side::Left : Side::Right;
  return c;
}

uint64_t exact_count_side(const BipartiteGraph& g, Side iterate) {
  uint64_t out = 0;
  ck(bfly_exact_count(g.device(), iterate == Side::Left ? BFLY_SIDE_LEFT : BFLY_SIDE_RIGHT, &out));
  return out;
}

uint64_t exact_count(const BipartiteGraph& g) {
  uint64_t out = 0;
  ck(bfly_exact_count(g.device(), BFLY_SIDE_AUTO, &out));
  return out;
}

// ---- local ---------------------------------------------------------------------------------------
uint64_t count_per_vertex(const BipartiteGraph& g, VertexRef v) {
  if (v.index >= g.side_count(v.side)) throw ArgumentError("vertex index out of range");
  const uint64_t gid = g.global_index(v);
  uint64_t out = 0;
  ck(bfly_local_vertex_batch(g.device(), &gid, 1, &out));
  return out;
}

uint64_t count_per_edge(const BipartiteGraph& g, uint32_t l, uint32_t r) {
  uint64_t out = 0;
  ck(bfly_local_edge_pairs(g.device(), &l, &r, 1, &out));
  return out;
}

std::vector<uint64_t> count_all_vertices(const BipartiteGraph& g) {
  std::vector<uint64_t> out(g.vertex_count());
  ck(bfly_local_vertex_all(g.device(), out.data()));
  return out;
}

std::vector<uint64_t> count_all_edges(const BipartiteGraph& g) {
  std::vector<uint64_t> out(g.edge_count());
  ck(bfly_local_edge_all(g.device(), out.data()));
  return out;
}

std::vector<uint64_t> count_vertices(const BipartiteGraph& g, const std::vector<uint64_t>& gids) {
  std::vector<uint64_t> out(gids.size());
  ck(bfly_local_vertex_batch(g.device(), gids.data(), gids.size(), out.data()));
  return out;
}

std::vector<uint64_t> count_edges(const BipartiteGraph& g, const std::vector<uint64_t>& ks) {
  std::vector<uint64_t> out(ks.size());
  ck(bfly_local_edge_batch(g.device(), ks.data(), ks.size(), out.data()));
  return out;
}

// ---- sampling ------------------------------------------------------------------------------------
const char* method_name(Method m) {
  switch (m) {
    case Method::Vertex: return "vertex";
    case Method::Edge: return "edge";
    case Method::Wedge: return "wedge";
    case Method::FastEdge: return "fast-edge";
  }
  return "?";
}

WedgeIndex build_wedge_index(const BipartiteGraph& g) {
  WedgeIndex w;
  w.prefix.resize(g.vertex_count() + 1);
  ck(bfly_wedge_index(g.device(), w.prefix.data(), &w.total));
  return w;
}

double vertex_sample_value(const BipartiteGraph& g, VertexRef v) {
  return static_cast<double>(count_per_vertex(g, v)) * static_cast<double>(g.vertex_count()) / 4.0;
}

double edge_sample_value(const BipartiteGraph& g, uint32_t l, uint32_t r) {
  return static_cast<double>(count_per_edge(g, l, r)) * static_cast<double>(g.edge_count()) / 4.0;
}

double wedge_sample_value(const BipartiteGraph& g, uint64_t total_wedges, VertexRef center,
                          uint32_t v, uint32_t w) {
  const Side leaf = opposite(center.side);
  uint64_t common = 0;
  ck(bfly_common_neighbors_batch(g.device(), leaf == Side::Left ? 0 : 1, &v, &w, 1, &common));
  // the centre itself is always shared for a real wedge; like the reference, no check
  return static_cast<double>(common - 1) * static_cast<double>(total_wedges) / 4.0;
}

namespace {

// One iteration's outcome (sampling.cpp:101-123); i/j only for Wedge.
inline void draw_one(const BipartiteGraph& g, Method m, const WedgeIndex* index, Rng& rng,
                     uint64_t& id, uint32_t& i, uint32_t& j) {
  i = j = 0;
  if (m == Method::Vertex) {
    id = rng.uniform_index(g.vertex_count());
  } else if (m == Method::Edge) {
    id = rng.uniform_index(g.edge_count());
  } else {
    if (index->total == 0) throw NoWedgesError("graph has no wedges to sample");
    const uint64_t r = rng.uniform_index(index->total);
    auto it = std::upper_bound(index->prefix.begin(), index->prefix.end(), r);
    id = static_cast<uint64_t>(it - index->prefix.begin()) - 1;
    const VertexRef c = g.vertex_at(id);
    const uint64_t d = g.degree(c);
    i = static_cast<uint32_t>(rng.uniform_index(d));
    j = static_cast<uint32_t>(rng.uniform_index(d - 1));
    if (j >= i) ++j;
  }
}

template <class F>
void parallel_for(uint64_t n, unsigned threads, F&& f) {
  threads = std::max(1u, threads);
  if (threads == 1 || n < 4096) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const uint64_t chunk = (n + threads - 1) / threads;
  for (unsigned t = 0; t < threads; ++t) {
    const uint64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

double vsamp_iteration(const BipartiteGraph& g, Rng& rng) {
  uint64_t id;
  uint32_t i, j;
  draw_one(g, Method::Vertex, nullptr, rng, id, i, j);
  return vertex_sample_value(g, g.vertex_at(id));
}

double esamp_iteration(const BipartiteGraph& g, Rng& rng) {
  uint64_t id;
  uint32_t i, j;
  draw_one(g, Method::Edge, nullptr, rng, id, i, j);
  auto [l, r] = g.edge_at(id);
  return edge_sample_value(g, l, r);
}

double wsamp_iteration(const BipartiteGraph& g, const WedgeIndex& index, Rng& rng) {
  uint64_t id;
  uint32_t i, j;
  draw_one(g, Method::Wedge, &index, rng, id, i, j);
  const VertexRef c = g.vertex_at(id);
  auto adj = g.neighbors(c.side, c.index);
  return wedge_sample_value(g, index.total, c, adj[i], adj[j]);
}

namespace {
// sampling.cpp:39-44 draw_excluding: uniform over adj minus `skip` (which is in adj)
uint32_t draw_excluding(std::span<const uint32_t> adj, uint32_t skip, Rng& rng) {
  const size_t pos = std::lower_bound(adj.begin(), adj.end(), skip) - adj.begin();
  uint64_t k = rng.uniform_index(adj.size() - 1);
  if (k >= pos) ++k;
  return adj[k];
}
}  // namespace

double fast_edge_pair_value(const BipartiteGraph& g, uint32_t l, uint32_t r, uint32_t other_l,
                            uint32_t other_r) {  // sampling.cpp:93-99
  uint8_t hit = 0;
  ck(bfly_has_edge_batch(g.device(), &other_l, &other_r, 1, &hit));
  if (!hit) return 0.0;
  const double dl = g.degree(Side::Left, l);
  const double dr = g.degree(Side::Right, r);
  return (dl - 1.0) * (dr - 1.0);
}

double fast_ebfc_estimate(const BipartiteGraph& g, uint32_t l, uint32_t r, uint64_t repeats,
                          Rng& rng) {  // sampling.cpp:125-141
  uint8_t is_edge = 0;
  if (l < g.left_count() && r < g.right_count())
    ck(bfly_has_edge_batch(g.device(), &l, &r, 1, &is_edge));
  if (!is_edge) throw ArgumentError("(l, r) is not an edge");
  if (repeats == 0) throw ArgumentError("repeats must be at least 1");
  const uint64_t dl = g.degree(Side::Left, l), dr = g.degree(Side::Right, r);
  if (dl == 1 || dr == 1) return 0.0;
  std::vector<uint32_t> ol(repeats), orr(repeats);
  const auto nr = g.neighbors(Side::Right, r), nl = g.neighbors(Side::Left, l);
  for (uint64_t t = 0; t < repeats; ++t) {
    ol[t] = draw_excluding(nr, l, rng);
    orr[t] = draw_excluding(nl, r, rng);
  }
  std::vector<uint8_t> hit(repeats);
  ck(bfly_has_edge_batch(g.device(), ol.data(), orr.data(), repeats, hit.data()));
  uint64_t hits = 0;
  for (uint8_t h : hit) hits += h;
  return static_cast<double>(hits) / static_cast<double>(repeats) *
         static_cast<double>(dl - 1) * static_cast<double>(dr - 1);
}

double fast_esamp_iteration(const BipartiteGraph& g, uint64_t repeats, Rng& rng) {
  auto [l, r] = g.edge_at(rng.uniform_index(g.edge_count()));  // sampling.cpp:143-147
  return fast_ebfc_estimate(g, l, r, repeats, rng) * static_cast<double>(g.edge_count()) / 4.0;
}

SampleIds sample_ids(const BipartiteGraph& g, Method m, uint64_t seed, uint64_t first,
                     uint64_t count, const WedgeIndex* index, unsigned threads) {
  if (m == Method::FastEdge) throw ArgumentError("fast-edge has no per-sample id list");  // API addition
  if (m == Method::Wedge) {
    if (!index) throw ArgumentError("wedge sampling needs a wedge index");
    if (index->total == 0) throw NoWedgesError("graph has no wedges to sample");
    (void)g.neighbors(Side::Left, 0);  // materialise the host mirror before threading
  }
  SampleIds s;
  s.id.resize(count);
  if (m == Method::Wedge) {
    s.i.resize(count);
    s.j.resize(count);
  }
  parallel_for(count, threads, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t q = lo; q < hi; ++q) {
      Rng rng = Rng::stream(seed, first + q);
      uint32_t i, j;
      draw_one(g, m, index, rng, s.id[q], i, j);
      if (m == Method::Wedge) {
        s.i[q] = i;
        s.j[q] = j;
      }
    }
  });
  return s;
}

namespace {

void validate(const BipartiteGraph& g, const EstimatorConfig& cfg) {  // sampling.cpp:168-181
  const bool has_iters = cfg.iterations > 0 || (cfg.groups > 1 && cfg.group_size > 0);
  const bool has_budget = cfg.time_budget_seconds > 0.0;
  if (has_iters == has_budget)
    throw ArgumentError("exactly one of iterations and time budget must be set");
  if (cfg.groups == 0) throw ArgumentError("groups must be at least 1");
  if (cfg.groups > 1 && cfg.groups % 2 == 0)
    throw ArgumentError("median-of-means group count must be odd");
  if (cfg.groups > 1 && has_budget)
    throw ArgumentError("median-of-means needs a fixed iteration count, not a time budget");
  if (cfg.fast_edge_repeats == 0) throw ArgumentError("fast-edge repeats must be at least 1");
  if (g.vertex_count() == 0 || g.edge_count() == 0)
    throw ArgumentError("cannot sample an empty graph");
}

// values of iterations [first, first+count) through one device batch: the sample ids are
// drawn on the GPU from the same per-iteration engines (bfly_sample_batch), so no id list
// crosses PCIe; sample_ids() above is the host restatement the tests compare against
void batch_values(const BipartiteGraph& g, const EstimatorConfig& cfg, uint64_t wedge_total,
                  uint64_t first, uint64_t count, double* out) {
  if (cfg.method == Method::FastEdge) {  // engines, draws and probes on the device
    ck(bfly_fast_edge_batch(g.device(), cfg.seed, first, count, cfg.fast_edge_repeats, out,
                            nullptr, nullptr));
    return;
  }
  std::vector<uint64_t> c(count);
  const int method = cfg.method == Method::Vertex ? 0 : cfg.method == Method::Edge ? 1 : 2;
  ck(bfly_sample_batch(g.device(), method, cfg.seed, first, count, c.data(), nullptr, nullptr,
                       nullptr));
  const double scale = cfg.method == Method::Vertex ? static_cast<double>(g.vertex_count())
                       : cfg.method == Method::Edge ? static_cast<double>(g.edge_count())
                                                    : static_cast<double>(wedge_total);
  for (uint64_t q = 0; q < count; ++q) out[q] = static_cast<double>(c[q]) * scale / 4.0;
}

double median_of(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

constexpr uint64_t kBatch = 1ull << 22;

}  // namespace

Estimate run_estimator(const BipartiteGraph& g, const EstimatorConfig& cfg, unsigned threads) {
  (void)threads;  // ids are drawn on the device; kept for API compatibility
  validate(g, cfg);
  uint64_t wedge_total = 0;  // sampling.cpp:63-73 total; the prefix itself stays on the GPU
  if (cfg.method == Method::Wedge) {
    wedge_total = compute_stats(g).wedge_count;
    if (wedge_total == 0) throw NoWedgesError("graph has no wedges to sample");
  }
  const auto start = Clock::now();
  Estimate est;
  est.seed = cfg.seed;

  if (cfg.time_budget_seconds > 0.0) {
    // sampling.cpp:217-241: whole 64-iteration blocks until the budget is spent; blocks
    // are evaluated in device batches that double in size
    std::vector<double> vals;
    uint64_t i = 0, next_cp = 1, block = 64;
    double running = 0.0;
    while (true) {
      const size_t base = vals.size();
      vals.resize(base + block);
      batch_values(g, cfg, wedge_total, i, block, vals.data() + base);
      bool out_of_time = false;
      for (uint64_t q = 0; q < block; ++q) {
        running += vals[base + q];
        ++i;
        if (cfg.record_trace && i == next_cp) {
          est.trace.push_back({seconds_since(start), i, running / static_cast<double>(i)});
          next_cp *= 2;
        }
        if (i % 64 == 0 && !out_of_time) out_of_time = seconds_since(start) >= cfg.time_budget_seconds;
        if (out_of_time && i % 64 == 0) break;
      }
      if (out_of_time) break;
      block = std::min<uint64_t>(block * 2, kBatch);
    }
    if (cfg.record_trace && (est.trace.empty() || est.trace.back().iteration != i))
      est.trace.push_back({seconds_since(start), i, running / static_cast<double>(i)});
    est.iterations_done = i;
    est.value = running / static_cast<double>(i);
    est.elapsed_seconds = seconds_since(start);
    return est;
  }

  const uint64_t alpha = cfg.group_size > 0 ? cfg.group_size : cfg.iterations;
  const uint64_t total = cfg.groups == 1 ? cfg.iterations : checked_mul(cfg.groups, alpha);
  std::vector<double> values(total);
  for (uint64_t b = 0; b < total; b += kBatch)
    batch_values(g, cfg, wedge_total, b, std::min(kBatch, total - b), values.data() + b);
  // sampling.cpp:183-202: sequential index-order sums
  double sum = 0.0;
  uint64_t next_cp = 1;
  for (uint64_t i = 1; i <= total; ++i) {
    sum += values[i - 1];
    if (cfg.record_trace && (i == next_cp || i == total)) {
      est.trace.push_back({seconds_since(start), i, sum / static_cast<double>(i)});
      while (next_cp <= i) next_cp *= 2;
    }
  }
  est.iterations_done = total;
  if (cfg.groups == 1) {
    est.value = sum / static_cast<double>(total);
  } else {
    const uint64_t a = total / cfg.groups;
    for (uint64_t t = 0; t < cfg.groups; ++t) {
      double gs = 0.0;
      for (uint64_t i = t * a; i < (t + 1) * a; ++i) gs += values[i];
      est.per_group_means.push_back(gs / static_cast<double>(a));
    }
    est.value = median_of(est.per_group_means);
  }
  est.elapsed_seconds = seconds_since(start);
  return est;
}

IterationPlan plan_iterations(double variance_bound, double pilot_bfly, double epsilon,
                              double delta) {  // sampling.cpp:280-294
  if (!(variance_bound >= 0.0)) throw ArgumentError("variance bound must be nonnegative");
  if (!(pilot_bfly > 0.0)) throw ArgumentError("pilot estimate must be positive");
  if (!(epsilon > 0.0)) throw ArgumentError("epsilon must be positive");
  if (!(delta > 0.0 && delta < 1.0)) throw ArgumentError("delta must be in (0, 1)");
  IterationPlan plan;
  uint64_t t = static_cast<uint64_t>(std::ceil(8.0 * std::log(1.0 / delta)));
  if (t < 1) t = 1;
  if (t > 1 && t % 2 == 0) ++t;
  plan.groups = t;
  const double a = std::ceil(32.0 * variance_bound / (epsilon * epsilon * pilot_bfly * pilot_bfly));
  plan.group_size = a < 1.0 ? 1 : static_cast<uint64_t>(a);
  return plan;
}

// ---- sparsify --------------------------------------------------------------------------------------
const char* sparsifier_name(Sparsifier s) { return s == Sparsifier::Edge ? "espar" : "clrspar"; }

namespace {
void check_p(double p) {
  if (!(p > 0.0 && p <= 1.0)) throw ArgumentError("retention probability must be in (0, 1]");
}
}  // namespace

double edge_sparsify_value(const BipartiteGraph& g, const std::vector<bool>& keep, double p) {
  check_p(p);
  if (keep.size() != g.edge_count()) throw ArgumentError("keep mask size mismatch");
  std::vector<uint8_t> k(keep.size());
  for (size_t i = 0; i < keep.size(); ++i) k[i] = keep[i] ? 1 : 0;
  uint64_t count = 0, kept = 0;
  ck(bfly_keep_mask_count(g.device(), k.data(), &count, &kept));
  const double inv = 1.0 / p;
  return static_cast<double>(count) * inv * inv * inv * inv;
}

double color_sparsify_value(const BipartiteGraph& g, const std::vector<uint32_t>& colors,
                            uint64_t n_colors) {
  if (n_colors == 0) throw ArgumentError("palette must have at least one color");
  if (colors.size() != g.vertex_count()) throw ArgumentError("color vector size mismatch");
  uint64_t count = 0, kept = 0;
  ck(bfly_color_mask_count(g.device(), colors.data(), &count, &kept));
  const double n = static_cast<double>(n_colors);
  return static_cast<double>(count) * n * n * n;
}

double edge_sparsify_estimate(const BipartiteGraph& g, double p, uint64_t seed) {
  check_p(p);
  uint64_t count = 0, kept = 0;
  ck(bfly_espar_count(g.device(), p, seed, &count, &kept));
  const double inv = 1.0 / p;
  return static_cast<double>(count) * inv * inv * inv * inv;
}

double color_sparsify_estimate(const BipartiteGraph& g, uint64_t n_colors, uint64_t seed) {
  if (n_colors == 0) throw ArgumentError("palette must have at least one color");
  uint64_t count = 0, kept = 0;
  ck(bfly_cspar_count(g.device(), n_colors, seed, &count, &kept));
  const double n = static_cast<double>(n_colors);
  return static_cast<double>(count) * n * n * n;
}

Estimate sparsify_run(const BipartiteGraph& g, const SparsifyConfig& cfg) {  // :73-94
  if (cfg.trials == 0) throw ArgumentError("trials must be at least 1");
  if (g.edge_count() == 0) throw ArgumentError("cannot sparsify an empty graph");
  Estimate est;
  est.seed = cfg.seed;
  est.iterations_done = cfg.trials;
  const auto start = Clock::now();
  double sum = 0.0;
  for (uint64_t t = 0; t < cfg.trials; ++t) {
    const uint64_t ts = derive_seed(cfg.seed, t);
    const double v = cfg.sparsifier == Sparsifier::Edge ? edge_sparsify_estimate(g, cfg.p, ts)
                                                        : color_sparsify_estimate(g, cfg.colors, ts);
    est.per_group_means.push_back(v);
    sum += v;
  }
  est.value = sum / static_cast<double>(cfg.trials);
  est.elapsed_seconds = seconds_since(start);
  return est;
}

SparsifyThresholds suggest_p(const GraphStats& stats, double pilot_bfly) {  // :96-105
  if (!(pilot_bfly > 0.0)) throw ArgumentError("pilot estimate must be positive");
  const double d = static_cast<double>(stats.max_degree);
  SparsifyThresholds t;
  t.espar_min_p = std::max({std::pow(24.0 / pilot_bfly, 0.25), std::sqrt(24.0 * d / pilot_bfly),
                            24.0 * d * d / pilot_bfly});
  t.clrspar_min_p = std::max({std::cbrt(32.0 / pilot_bfly), std::sqrt(32.0 * d / pilot_bfly),
                              32.0 * d * d / pilot_bfly});
  return t;
}

}  // namespace bfly

// ---- C exports for non-C++ callers (Python tests, bench.py) ------------------------------------
namespace {
thread_local std::string t_host_err;

template <class F>
int host_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const bfly::ArgumentError& e) {
    t_host_err = e.what();
    return BFLY_ARGUMENT;
  } catch (const bfly::EmptyGraphError& e) {
    t_host_err = e.what();
    return BFLY_EMPTY;
  } catch (const bfly::OverflowError& e) {
    t_host_err = e.what();
    return BFLY_OVERFLOW;
  } catch (const bfly::NoWedgesError& e) {
    t_host_err = e.what();
    return BFLY_NO_WEDGES;
  } catch (const std::exception& e) {
    t_host_err = e.what();
    return BFLY_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* bfly_host_last_error(void) { return t_host_err.c_str(); }

int bfly_host_run_estimator(bfly_graph* g, int method, uint64_t iterations, double time_budget,
                            uint64_t seed, uint64_t groups, uint64_t group_size,
                            int record_trace, unsigned threads, double* value,
                            uint64_t* iterations_done, double* per_group, double* trace_out,
                            uint64_t* trace_len) {
  return bfly_host_run_estimator_ex(g, method, iterations, time_budget, seed, groups, group_size,
                                    1000, record_trace, threads, value, iterations_done,
                                    per_group, trace_out, trace_len);
}

int bfly_host_run_estimator_ex(bfly_graph* g, int method, uint64_t iterations, double time_budget,
                               uint64_t seed, uint64_t groups, uint64_t group_size,
                               uint64_t fast_edge_repeats, int record_trace, unsigned threads,
                               double* value, uint64_t* iterations_done, double* per_group,
                               double* trace_out, uint64_t* trace_len) {
  return host_guard([&] {
    bfly::BipartiteGraph bg = bfly::BipartiteGraph::adopt(g, false);
    bfly::EstimatorConfig cfg;
    cfg.method = static_cast<bfly::Method>(method);
    cfg.iterations = iterations;
    cfg.time_budget_seconds = time_budget;
    cfg.seed = seed;
    cfg.groups = groups;
    cfg.group_size = group_size;
    cfg.fast_edge_repeats = fast_edge_repeats;
    cfg.record_trace = record_trace != 0;
    bfly::Estimate e = bfly::run_estimator(bg, cfg, threads);
    *value = e.value;
    *iterations_done = e.iterations_done;
    if (per_group)
      for (size_t i = 0; i < e.per_group_means.size(); ++i) per_group[i] = e.per_group_means[i];
    if (trace_len) {
      const uint64_t cap = *trace_len;
      *trace_len = e.trace.size();
      for (size_t i = 0; trace_out && i < e.trace.size() && i < cap; ++i) {
        trace_out[3 * i] = static_cast<double>(e.trace[i].iteration);
        trace_out[3 * i + 1] = e.trace[i].estimate;
        trace_out[3 * i + 2] = e.trace[i].elapsed_seconds;
      }
    }
  });
}

int bfly_host_time_from_pairs(const uint32_t* left, const uint32_t* right, uint64_t m, int reps,
                              double* ms, uint64_t* count) {
  return host_guard([&] {
    std::vector<std::pair<uint64_t, uint64_t>> edges(m);  // the caller's input, built untimed
    for (uint64_t i = 0; i < m; ++i) edges[i] = {left[i], right[i]};
    for (int k = 0; k < reps; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      const bfly::BipartiteGraph g = bfly::BipartiteGraph::from_edges(edges);
      *count = bfly::exact_count(g);
      ms[k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count();
    }
  });
}

int bfly_host_sample_ids(bfly_graph* g, int method, uint64_t seed, uint64_t first, uint64_t count,
                         unsigned threads, uint64_t* id, uint32_t* i, uint32_t* j) {
  return host_guard([&] {
    bfly::BipartiteGraph bg = bfly::BipartiteGraph::adopt(g, false);
    bfly::WedgeIndex wi;
    const auto m = static_cast<bfly::Method>(method);
    if (m == bfly::Method::Wedge) wi = bfly::build_wedge_index(bg);
    bfly::SampleIds s = bfly::sample_ids(bg, m, seed, first, count, &wi, threads);
    std::memcpy(id, s.id.data(), count * 8);
    if (m == bfly::Method::Wedge) {
      std::memcpy(i, s.i.data(), count * 4);
      std::memcpy(j, s.j.data(), count * 4);
    }
  });
}

int bfly_host_sparsify_run(bfly_graph* g, int sparsifier, double p, uint64_t colors, uint64_t seed,
                           uint64_t trials, double* value, double* per_trial) {
  return host_guard([&] {
    bfly::BipartiteGraph bg = bfly::BipartiteGraph::adopt(g, false);
    bfly::SparsifyConfig cfg;
    cfg.sparsifier = sparsifier == 0 ? bfly::Sparsifier::Edge : bfly::Sparsifier::Color;
    cfg.p = p;
    cfg.colors = colors;
    cfg.seed = seed;
    cfg.trials = trials;
    bfly::Estimate e = bfly::sparsify_run(bg, cfg);
    *value = e.value;
    for (size_t t = 0; per_trial && t < e.per_group_means.size(); ++t) per_trial[t] = e.per_group_means[t];
  });
}

}  // extern "C"
