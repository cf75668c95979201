// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library, compiled straight from
// /root/reference/proj/src/*.cpp with -Dbfly=bfly_ref (see oracle/Makefile) into
// oracle/_ref/libbfly_ref.so. Used to (a) validate the C restatement in
// oracle/bfly_oracle.c, (b) generate golden vectors under tests/golden/, and (c) time
// the reference CPU path in bench.py (--impl reference, cpu_baseline kind "reference").
// No reference source is copied into this repository.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <exception>
#include <thread>
#include <utility>
#include <vector>

#include "bfly/errors.hpp"
#include "bfly/exact.hpp"
#include "bfly/graph.hpp"
#include "bfly/local.hpp"
#include "bfly/oracle.hpp"
#include "bfly/rng.hpp"
#include "bfly/sampling.hpp"
#include "bfly/sparsify.hpp"

using namespace bfly;  // becomes bfly_ref under -Dbfly=bfly_ref

namespace {

int code_of(const std::exception& e) {
  if (dynamic_cast<const ArgumentError*>(&e)) return 1;
  if (dynamic_cast<const EmptyGraphError*>(&e)) return 2;
  if (dynamic_cast<const OverflowError*>(&e)) return 3;
  if (dynamic_cast<const NoWedgesError*>(&e)) return 4;
  if (dynamic_cast<const SizeGuardError*>(&e)) return 6;
  return 5;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

BipartiteGraph* G(void* h) { return static_cast<BipartiteGraph*>(h); }

}  // namespace

extern "C" {

int ref_graph_build(const uint64_t* l, const uint64_t* r, uint64_t m, void** out) {
  return guard([&] {
    std::vector<std::pair<uint64_t, uint64_t>> edges(m);
    for (uint64_t i = 0; i < m; ++i) edges[i] = {l[i], r[i]};
    *out = new BipartiteGraph(BipartiteGraph::from_edges(edges));
  });
}

// load_edge_list (graph.cpp:75-99) from an in-memory stream. Returns 0, 2 (EmptyGraphError)
// or 7 (ParseError: msg = what(), *line = line()); other failures per code_of.
int ref_load_text(const char* text, uint64_t len, void** out, char* msg, uint64_t cap,
                  uint64_t* line) {
  *line = 0;
  try {
    std::istringstream in(std::string(text, len));
    *out = new BipartiteGraph(load_edge_list(in));
    return 0;
  } catch (const ParseError& e) {
    std::snprintf(msg, cap, "%s", e.what());
    *line = e.line();
    return 7;
  } catch (const std::exception& e) {
    std::snprintf(msg, cap, "%s", e.what());
    return code_of(e);
  }
}

// serialize_edge_list (graph.cpp:107-112); *len = bytes, copied when buf holds them
int ref_serialize(void* h, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    std::ostringstream out;
    serialize_edge_list(*G(h), out);
    const std::string t = out.str();
    *len = t.size();
    if (buf && cap >= t.size()) std::memcpy(buf, t.data(), t.size());
  });
}

int ref_graph_build_u32(const uint32_t* l, const uint32_t* r, uint64_t m, void** out) {
  return guard([&] {
    std::vector<std::pair<uint64_t, uint64_t>> edges(m);
    for (uint64_t i = 0; i < m; ++i) edges[i] = {l[i], r[i]};
    *out = new BipartiteGraph(BipartiteGraph::from_edges(edges));
  });
}

int ref_complete_biclique(uint32_t a, uint32_t b, void** out) {
  return guard([&] { *out = new BipartiteGraph(complete_biclique(a, b)); });
}

int ref_random_bipartite(uint32_t a, uint32_t b, double p, uint64_t seed, void** out) {
  return guard([&] { *out = new BipartiteGraph(random_bipartite(a, b, p, seed)); });
}

void ref_graph_free(void* h) { delete G(h); }

void ref_graph_sizes(void* h, uint32_t* L, uint32_t* R, uint64_t* m) {
  *L = G(h)->left_count();
  *R = G(h)->right_count();
  *m = G(h)->edge_count();
}

// Canonical left CSR (edge_at order) + right CSR + external ids.
void ref_graph_export(void* h, uint64_t* loff, uint32_t* ladj, uint64_t* roff, uint32_t* radj,
                      uint64_t* lids, uint64_t* rids) {
  const BipartiteGraph& g = *G(h);
  uint64_t k = 0;
  for (uint32_t i = 0; i < g.left_count(); ++i) {
    loff[i] = k;
    for (uint32_t x : g.neighbors(Side::Left, i)) ladj[k++] = x;
    lids[i] = g.external_id(Side::Left, i);
  }
  loff[g.left_count()] = k;
  k = 0;
  for (uint32_t i = 0; i < g.right_count(); ++i) {
    roff[i] = k;
    for (uint32_t x : g.neighbors(Side::Right, i)) radj[k++] = x;
    rids[i] = g.external_id(Side::Right, i);
  }
  roff[g.right_count()] = k;
}

int ref_compute_stats(void* h, uint64_t* u64s /*n,left,right,m,wedges,maxdeg*/, double* sq /*2*/) {
  return guard([&] {
    GraphStats s = compute_stats(*G(h));
    u64s[0] = s.n;
    u64s[1] = s.left;
    u64s[2] = s.right;
    u64s[3] = s.m;
    u64s[4] = s.wedge_count;
    u64s[5] = s.max_degree;
    sq[0] = s.sum_deg_sq_left;
    sq[1] = s.sum_deg_sq_right;
  });
}

int ref_choose_side(void* h, int* chosen, double* cl, double* cr) {
  return guard([&] {
    SideChoice c = choose_side(*G(h));
    *chosen = c.chosen == Side::Left ? 0 : 1;
    *cl = c.cost_left;
    *cr = c.cost_right;
  });
}

int ref_exact_count(void* h, uint64_t* out) {
  return guard([&] { *out = exact_count(*G(h)); });
}

int ref_exact_count_side(void* h, int side, uint64_t* out) {
  return guard([&] { *out = exact_count_side(*G(h), side == 0 ? Side::Left : Side::Right); });
}

int ref_brute_force_count(void* h, uint64_t* out) {
  return guard([&] { *out = brute_force_count(*G(h)); });
}

// oracle.cpp:60-94 classify_pairs with OracleGuards{max_side, max_butterflies}:
// out[6] = bfly, p_0v, p_1v, p_2v, p_1e, p_1w (status 6 = SizeGuardError)
int ref_classify_pairs(void* h, uint32_t max_side, uint64_t max_bfly, uint64_t* out) {
  return guard([&] {
    OracleGuards gd;
    gd.max_side = max_side;
    gd.max_butterflies = max_bfly;
    const PairTypeCounts c = classify_pairs(*G(h), gd);
    const uint64_t v[6] = {c.bfly, c.p_0v, c.p_1v, c.p_2v, c.p_1e, c.p_1w};
    std::memcpy(out, v, sizeof(v));
  });
}

// oracle.cpp:96-116 variance_bounds on the graph's stats and the given counts
int ref_variance_bounds(void* h, const uint64_t* counts, double p, double* out) {
  return guard([&] {
    PairTypeCounts c;
    c.bfly = counts[0];
    c.p_0v = counts[1];
    c.p_1v = counts[2];
    c.p_2v = counts[3];
    c.p_1e = counts[4];
    c.p_1w = counts[5];
    const VarianceBounds b = variance_bounds(compute_stats(*G(h)), c, p);
    const double v[5] = {b.vsamp, b.esamp, b.wsamp, b.espar, b.clrspar};
    std::memcpy(out, v, sizeof(v));
  });
}

int ref_count_per_vertex(void* h, int side, uint32_t index, uint64_t* out) {
  return guard([&] {
    *out = count_per_vertex(*G(h), VertexRef{side == 0 ? Side::Left : Side::Right, index});
  });
}

int ref_count_per_edge(void* h, uint32_t l, uint32_t r, uint64_t* out) {
  return guard([&] { *out = count_per_edge(*G(h), l, r); });
}

int ref_edge_at(void* h, uint64_t k, uint32_t* l, uint32_t* r) {
  return guard([&] {
    auto e = G(h)->edge_at(k);
    *l = e.first;
    *r = e.second;
  });
}

// All-subject loops over the thread-safe local counts (local.hpp:10-11).
int ref_count_all_vertices(void* h, int threads, uint64_t* out) {
  const BipartiteGraph& g = *G(h);
  uint64_t n = g.vertex_count();
  int status = 0;
  auto work = [&](uint64_t lo, uint64_t hi) {
    int st = guard([&] {
      for (uint64_t v = lo; v < hi; ++v) out[v] = count_per_vertex(g, g.vertex_at(v));
    });
    if (st) status = st;
  };
  std::vector<std::thread> pool;
  uint64_t T = threads < 1 ? 1 : threads, chunk = (n + T - 1) / T;
  for (uint64_t t = 0; t < T; ++t) {
    uint64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  return status;
}

int ref_count_edges(void* h, const uint64_t* ks, uint64_t nk, int threads, uint64_t* out) {
  const BipartiteGraph& g = *G(h);
  int status = 0;
  auto work = [&](uint64_t lo, uint64_t hi) {
    int st = guard([&] {
      for (uint64_t i = lo; i < hi; ++i) {
        auto e = g.edge_at(ks ? ks[i] : i);
        out[i] = count_per_edge(g, e.first, e.second);
      }
    });
    if (st) status = st;
  };
  std::vector<std::thread> pool;
  uint64_t T = threads < 1 ? 1 : threads, chunk = (nk + T - 1) / T;
  for (uint64_t t = 0; t < T; ++t) {
    uint64_t lo = t * chunk, hi = std::min(nk, lo + chunk);
    if (lo < hi) pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  return status;
}

int ref_build_wedge_index(void* h, uint64_t* prefix, uint64_t* total) {
  return guard([&] {
    WedgeIndex w = build_wedge_index(*G(h));
    std::memcpy(prefix, w.prefix.data(), w.prefix.size() * sizeof(uint64_t));
    *total = w.total;
  });
}

int ref_vertex_sample_value(void* h, int side, uint32_t index, double* out) {
  return guard([&] {
    *out = vertex_sample_value(*G(h), VertexRef{side == 0 ? Side::Left : Side::Right, index});
  });
}

int ref_edge_sample_value(void* h, uint32_t l, uint32_t r, double* out) {
  return guard([&] { *out = edge_sample_value(*G(h), l, r); });
}

int ref_wedge_sample_value(void* h, uint64_t total, int cside, uint32_t centre, uint32_t v,
                           uint32_t w, double* out) {
  return guard([&] {
    *out = wedge_sample_value(*G(h), total, VertexRef{cside == 0 ? Side::Left : Side::Right, centre},
                              v, w);
  });
}

// One iteration value from Rng::stream(seed, index) (sampling.cpp:157-166).
int ref_iteration(void* h, int method, uint64_t seed, uint64_t index, double* out) {
  return guard([&] {
    const BipartiteGraph& g = *G(h);
    Rng rng = Rng::stream(seed, index);
    if (method == 0) *out = vsamp_iteration(g, rng);
    else if (method == 1) *out = esamp_iteration(g, rng);
    else {
      WedgeIndex w = build_wedge_index(g);
      *out = wsamp_iteration(g, w, rng);
    }
  });
}

int ref_run_estimator(void* h, int method, uint64_t iterations, uint64_t seed, uint64_t groups,
                      uint64_t group_size, unsigned threads, double* value, uint64_t* done,
                      double* per_group) {
  return guard([&] {
    EstimatorConfig cfg;
    cfg.method = method == 0 ? Method::Vertex : method == 1 ? Method::Edge : Method::Wedge;
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.groups = groups;
    cfg.group_size = group_size;
    Estimate e = run_estimator(*G(h), cfg, threads);
    *value = e.value;
    *done = e.iterations_done;
    if (per_group)
      for (size_t i = 0; i < e.per_group_means.size(); ++i) per_group[i] = e.per_group_means[i];
  });
}

// Method::FastEdge: one iteration of Rng::stream(seed, index) (sampling.cpp:143-147) and
// run_estimator with fast_edge_repeats (sampling.hpp:22).
int ref_fast_iteration(void* h, uint64_t repeats, uint64_t seed, uint64_t index, double* out) {
  return guard([&] {
    Rng rng = Rng::stream(seed, index);
    *out = fast_esamp_iteration(*G(h), repeats, rng);
  });
}

int ref_run_estimator_ex(void* h, int method, uint64_t iterations, uint64_t seed,
                         uint64_t groups, uint64_t group_size, uint64_t repeats, unsigned threads,
                         double* value, uint64_t* done, double* per_group) {
  return guard([&] {
    EstimatorConfig cfg;
    cfg.method = method == 0 ? Method::Vertex
                 : method == 1 ? Method::Edge
                 : method == 2 ? Method::Wedge
                               : Method::FastEdge;
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.groups = groups;
    cfg.group_size = group_size;
    cfg.fast_edge_repeats = repeats;
    Estimate e = run_estimator(*G(h), cfg, threads);
    *value = e.value;
    *done = e.iterations_done;
    if (per_group)
      for (size_t i = 0; i < e.per_group_means.size(); ++i) per_group[i] = e.per_group_means[i];
  });
}

int ref_edge_sparsify_estimate(void* h, double p, uint64_t seed, double* out) {
  return guard([&] { *out = edge_sparsify_estimate(*G(h), p, seed); });
}

int ref_color_sparsify_estimate(void* h, uint64_t n, uint64_t seed, double* out) {
  return guard([&] { *out = color_sparsify_estimate(*G(h), n, seed); });
}

int ref_sparsify_run(void* h, int sparsifier, double p, uint64_t colors, uint64_t seed,
                     uint64_t trials, double* value, double* per_trial) {
  return guard([&] {
    SparsifyConfig cfg;
    cfg.sparsifier = sparsifier == 0 ? Sparsifier::Edge : Sparsifier::Color;
    cfg.p = p;
    cfg.colors = colors;
    cfg.seed = seed;
    cfg.trials = trials;
    Estimate e = sparsify_run(*G(h), cfg);
    *value = e.value;
    if (per_trial)
      for (size_t i = 0; i < e.per_group_means.size(); ++i) per_trial[i] = e.per_group_means[i];
  });
}

uint64_t ref_mix64(uint64_t x) { return mix64(x); }
uint64_t ref_derive_seed(uint64_t s, uint64_t i) { return derive_seed(s, i); }
uint64_t ref_rng_stream_first(uint64_t seed, uint64_t index) { return Rng::stream(seed, index).next(); }

}  // extern "C"
