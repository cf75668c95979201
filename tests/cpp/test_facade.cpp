// test_facade.cpp -- the reference's own test cases (proj/tests/test_exact.cpp,
// test_local.cpp, test_sampling.cpp, test_sparsify.cpp), restated against the B200 facade
// (bfly_b200.hpp). Built with g++ against the facade header only and linked to
// libbfly_host.so + libbfly_b200.so: this is the switch-over a maintainer performs.
#include <sstream>
#include <algorithm>
#include <cmath>
#include <vector>

#include "bfly_b200.hpp"
#include "mini_test.hpp"

using namespace bfly;

namespace {

// Test inputs built like the reference's generators (graph.cpp:114-134).
BipartiteGraph biclique(uint32_t a, uint32_t b) {
  std::vector<std::pair<uint64_t, uint64_t>> e;
  for (uint32_t i = 1; i <= a; ++i)
    for (uint32_t j = 1; j <= b; ++j) e.emplace_back(i, j);
  return BipartiteGraph::from_edges(e);
}

std::vector<std::pair<uint64_t, uint64_t>> coin_edges(uint32_t a, uint32_t b, double p,
                                                      uint64_t seed) {
  Rng rng(seed);
  std::vector<std::pair<uint64_t, uint64_t>> e;
  for (uint32_t i = 1; i <= a; ++i)
    for (uint32_t j = 1; j <= b; ++j)
      if (rng.uniform_unit() < p) e.emplace_back(i, j);
  return e;
}

// tests/support/fixtures.hpp random_suite: seeded sizes/probabilities, skipping empties
std::vector<BipartiteGraph> suite(size_t count, uint32_t ma, uint32_t mb, std::vector<double> ps,
                                  uint64_t base) {
  std::vector<BipartiteGraph> out;
  for (uint64_t seed = base; out.size() < count; ++seed) {
    Rng pick(derive_seed(base, seed));
    uint32_t a = 1 + static_cast<uint32_t>(pick.uniform_index(ma));
    uint32_t b = 1 + static_cast<uint32_t>(pick.uniform_index(mb));
    double p = ps[pick.uniform_index(ps.size())];
    auto e = coin_edges(a, b, p, seed);
    if (!e.empty()) out.push_back(BipartiteGraph::from_edges(e));
  }
  return out;
}

// independent ground truth: sum over left pairs of C(|common|, 2) (oracle.cpp:50-57)
uint64_t pair_count(const BipartiteGraph& g) {
  uint64_t t = 0;
  for (uint32_t a = 0; a < g.left_count(); ++a)
    for (uint32_t b = a + 1; b < g.left_count(); ++b) {
      auto na = g.neighbors(Side::Left, a), nb = g.neighbors(Side::Left, b);
      std::vector<uint32_t> c;
      std::set_intersection(na.begin(), na.end(), nb.begin(), nb.end(), std::back_inserter(c));
      t += choose2(c.size());
    }
  return t;
}

BipartiteGraph edges(std::vector<std::pair<uint64_t, uint64_t>> e) {
  return BipartiteGraph::from_edges(e);
}

}  // namespace

TEST_CASE("graph: edge-list text in and out (graph.cpp:75-112)") {
  std::istringstream in("% bip\n10 20\n\n# c\n 11\t20 extra\r\n10 21\n10 20\n");
  auto g = load_edge_list(in);
  CHECK(g.left_count() == 2);
  CHECK(g.right_count() == 2);
  CHECK(g.edge_count() == 3);
  std::ostringstream out;
  serialize_edge_list(g, out);
  CHECK(out.str() == "% bip\n10 20\n10 21\n11 20\n");
  std::istringstream bad("1 2\n3\n");
  try {
    load_edge_list(bad);
    CHECK(false);
  } catch (const ParseError& e) {
    CHECK(e.line() == 2);
    CHECK(std::string(e.what()) == "expected two vertex ids, got 1 (line 2)");
  }
  std::istringstream empty("% nothing\n");
  CHECK_THROWS_AS(load_edge_list(empty), EmptyGraphError);
  CHECK_THROWS_AS(load_edge_list_file("/nonexistent/file.txt"), Error);
}

TEST_CASE("graph: fixture generators (graph.cpp:114-134)") {
  auto k = complete_biclique(4, 3);
  CHECK(k.edge_count() == 12);
  CHECK(exact_count(k) == 18);  // C(4,2) * C(3,2)
  CHECK(k.external_id(Side::Left, 0) == 1);
  CHECK_THROWS_AS(complete_biclique(0, 3), ArgumentError);
  auto r = random_bipartite(40, 40, 0.2, 21);
  CHECK(r.edge_count() == coin_edges(40, 40, 0.2, 21).size());
  CHECK_THROWS_AS(random_bipartite(3, 3, 1.5, 1), ArgumentError);
  CHECK_THROWS_AS(random_bipartite(3, 3, 0.0, 1), EmptyGraphError);
}

TEST_CASE("exact: closed form over a biclique grid") {
  for (uint32_t a = 1; a <= 60; a += 3)
    for (uint32_t b = 1; b <= 60; b += 7) CHECK(exact_count(biclique(a, b)) == choose2(a) * choose2(b));
}

TEST_CASE("exact: (10^4, 10) biclique and side choice") {
  auto g = biclique(10000, 10);
  CHECK(exact_count(g) == 2249775000ULL);
  SideChoice c = choose_side(g);
  CHECK(c.cost_left == 1e6);
  CHECK(c.cost_right == 1e9);
  CHECK(c.chosen == Side::Right);
  CHECK(choose_side(biclique(2, 100)).chosen == Side::Left);
  CHECK(choose_side(biclique(3, 3)).chosen == Side::Left);
}

TEST_CASE("exact: agrees with pair enumeration for either side") {
  for (const auto& g : suite(60, 12, 12, {0.2, 0.5, 0.8}, 5000)) {
    uint64_t truth = pair_count(g);
    CHECK(exact_count(g) == truth);
    CHECK(exact_count_side(g, Side::Left) == truth);
    CHECK(exact_count_side(g, Side::Right) == truth);
  }
}

TEST_CASE("exact: butterfly-free graphs") {
  CHECK(exact_count(edges({{1, 1}, {2, 1}, {2, 2}, {3, 2}, {3, 3}, {1, 3}})) == 0);
  CHECK(exact_count(biclique(1, 5)) == 0);
  CHECK(exact_count(edges({{1, 1}, {2, 1}, {2, 2}})) == 0);
}

TEST_CASE("checked arithmetic") {
  CHECK_THROWS_AS(checked_add(~uint64_t{0}, 1), OverflowError);
  CHECK_THROWS_AS(checked_mul(uint64_t{1} << 33, uint64_t{1} << 33), OverflowError);
  CHECK_THROWS_AS(choose2(uint64_t{1} << 33), OverflowError);
  CHECK(choose2(4294967296ULL - 1) == 9223372030412324865ULL);
}

TEST_CASE("local: hand values and errors") {
  auto g33 = biclique(3, 3);
  for (uint32_t i = 0; i < 3; ++i) {
    CHECK(count_per_vertex(g33, {Side::Left, i}) == 6);
    CHECK(count_per_vertex(g33, {Side::Right, i}) == 6);
  }
  for (uint32_t l = 0; l < 3; ++l)
    for (uint32_t r = 0; r < 3; ++r) CHECK(count_per_edge(g33, l, r) == 4);
  CHECK(count_per_edge(biclique(1, 3), 0, 0) == 0);
  CHECK(count_per_edge(biclique(8, 2), 0, 0) == 7);
  CHECK(count_per_edge(biclique(2, 8), 0, 0) == 7);
  CHECK_THROWS_AS(count_per_vertex(biclique(2, 2), {Side::Left, 2}), ArgumentError);
  auto two = edges({{1, 1}, {1, 2}, {2, 1}, {2, 2}, {3, 3}, {3, 4}, {4, 3}, {4, 4}});
  CHECK_THROWS_AS(count_per_edge(two, 0, 3), ArgumentError);
  CHECK_THROWS_AS(count_per_edge(biclique(2, 2), 0, 5), ArgumentError);
}

TEST_CASE("local: sums recover four times the global count") {
  for (const auto& g : suite(30, 13, 13, {0.25, 0.5, 0.75}, 9000)) {
    uint64_t total = exact_count(g), by_v = 0, by_e = 0;
    for (uint64_t v = 0; v < g.vertex_count(); ++v) by_v += count_per_vertex(g, g.vertex_at(v));
    for (uint64_t k = 0; k < g.edge_count(); ++k) {
      auto [l, r] = g.edge_at(k);
      by_e += count_per_edge(g, l, r);
    }
    CHECK(by_v == 4 * total);
    CHECK(by_e == 4 * total);
    auto av = count_all_vertices(g);
    auto ae = count_all_edges(g);
    for (uint64_t v = 0; v < g.vertex_count(); ++v) CHECK(av[v] == count_per_vertex(g, g.vertex_at(v)));
    uint64_t se = 0;
    for (uint64_t x : ae) se += x;
    CHECK(se == 4 * total);
  }
}

TEST_CASE("sampling: pinned per-outcome values") {
  auto g32 = biclique(3, 2);
  CHECK(vertex_sample_value(g32, {Side::Left, 0}) == 2.5);
  CHECK(vertex_sample_value(g32, {Side::Right, 1}) == 3.75);
  for (uint64_t k = 0; k < 6; ++k) {
    auto [l, r] = g32.edge_at(k);
    CHECK(edge_sample_value(g32, l, r) == 3.0);
  }
  CHECK(wedge_sample_value(g32, 9, {Side::Right, 0}, 0, 1) == 2.25);
  CHECK(wedge_sample_value(g32, 9, {Side::Left, 0}, 0, 1) == 4.5);
  CHECK(build_wedge_index(biclique(3, 3)).total == 18);
}

TEST_CASE("sampling: degenerate estimators are constant") {
  auto g22 = biclique(2, 2), g33 = biclique(3, 3);
  WedgeIndex w33 = build_wedge_index(g33);
  for (uint64_t seed = 0; seed < 20; ++seed) {
    Rng r1(seed), r2(seed);
    CHECK(vsamp_iteration(g22, r1) == 1.0);
    CHECK(wsamp_iteration(g33, w33, r2) == 9.0);
    Rng r3(seed);
    CHECK(fast_esamp_iteration(g22, 3, r3) == 1.0);
  }
}

TEST_CASE("sampling: fast edge skips degree-one endpoints without sampling") {
  auto star = biclique(1, 3);
  Rng rng(1);
  CHECK(fast_ebfc_estimate(star, 0, 1, 1000, rng) == 0.0);
  Rng fresh(1);  // an untouched engine proves no draws happened
  CHECK(rng.next() == fresh.next());
  CHECK_THROWS_AS(fast_ebfc_estimate(star, 0, 5, 10, rng), ArgumentError);
  CHECK_THROWS_AS(fast_ebfc_estimate(biclique(2, 2), 0, 0, 0, rng), ArgumentError);
  CHECK(fast_edge_pair_value(biclique(3, 3), 0, 0, 1, 1) == 4.0);
}

TEST_CASE("sampling: fast edge run_estimator replays the per-iteration API") {
  auto g = BipartiteGraph::from_edges(coin_edges(40, 40, 0.2, 21));
  EstimatorConfig cfg;
  cfg.method = Method::FastEdge;
  cfg.iterations = 257;
  cfg.seed = 99;
  cfg.fast_edge_repeats = 16;
  Estimate a = run_estimator(g, cfg, 1), c = run_estimator(g, cfg, 4);
  CHECK(a.value == c.value);
  double sum = 0.0;  // device engines vs the host engine + device probes, per iteration
  for (uint64_t i = 0; i < 257; ++i) {
    Rng rng = Rng::stream(99, i);
    sum += fast_esamp_iteration(g, 16, rng);
  }
  CHECK(a.value == sum / 257.0);
  cfg.seed = 100;
  CHECK(run_estimator(g, cfg, 1).value != a.value);
}

TEST_CASE("sampling: reproducible, thread independent, replays from streams") {
  auto g = BipartiteGraph::from_edges(coin_edges(40, 40, 0.2, 21));
  for (Method m : {Method::Vertex, Method::Edge, Method::Wedge}) {
    EstimatorConfig cfg;
    cfg.method = m;
    cfg.iterations = 257;
    cfg.seed = 99;
    Estimate a = run_estimator(g, cfg, 1), c = run_estimator(g, cfg, 4);
    CHECK(a.value == c.value);
    CHECK(a.iterations_done == 257);
    cfg.seed = 100;
    CHECK(run_estimator(g, cfg, 1).value != a.value);
  }
  auto h = BipartiteGraph::from_edges(coin_edges(20, 20, 0.3, 33));
  EstimatorConfig cfg;
  cfg.method = Method::Edge;
  cfg.iterations = 100;
  cfg.seed = 5;
  Estimate est = run_estimator(h, cfg, 4);
  double sum = 0.0;
  for (uint64_t i = 0; i < 100; ++i) {
    Rng rng = Rng::stream(5, i);
    sum += esamp_iteration(h, rng);
  }
  CHECK(est.value == sum / 100.0);
}

TEST_CASE("sampling: median of contiguous group means") {
  auto g = biclique(3, 2);
  EstimatorConfig cfg;
  cfg.method = Method::Wedge;
  cfg.seed = 7;
  cfg.groups = 5;
  cfg.group_size = 20;
  Estimate est = run_estimator(g, cfg, 2);
  CHECK(est.iterations_done == 100);
  WedgeIndex index = build_wedge_index(g);
  std::vector<double> means;
  for (uint64_t t = 0; t < 5; ++t) {
    double s = 0.0;
    for (uint64_t i = t * 20; i < (t + 1) * 20; ++i) {
      Rng rng = Rng::stream(7, i);
      s += wsamp_iteration(g, index, rng);
    }
    CHECK(est.per_group_means[t] == s / 20.0);
    means.push_back(s / 20.0);
  }
  std::sort(means.begin(), means.end());
  CHECK(est.value == means[2]);
}

TEST_CASE("sampling: config validation") {
  auto g = biclique(2, 2);
  EstimatorConfig cfg;
  cfg.method = Method::Vertex;
  CHECK_THROWS_AS(run_estimator(g, cfg, 1), ArgumentError);
  cfg.iterations = 10;
  cfg.time_budget_seconds = 1.0;
  CHECK_THROWS_AS(run_estimator(g, cfg, 1), ArgumentError);
  cfg.time_budget_seconds = 0.0;
  cfg.groups = 4;
  cfg.group_size = 2;
  CHECK_THROWS_AS(run_estimator(g, cfg, 1), ArgumentError);
  cfg.groups = 3;
  cfg.group_size = 0;
  cfg.iterations = 9;
  CHECK(run_estimator(g, cfg, 1).iterations_done == 27);
  auto single = edges({{1, 1}});
  EstimatorConfig w;
  w.method = Method::Wedge;
  w.iterations = 5;
  CHECK_THROWS_AS(run_estimator(single, w, 1), NoWedgesError);
}

TEST_CASE("sparsify: full retention, derived-seed trials, empties") {
  for (const auto& g : suite(10, 8, 8, {0.3, 0.6}, 4100)) {
    double exact = static_cast<double>(exact_count(g));
    for (uint64_t seed : {uint64_t{0}, uint64_t{1}, uint64_t{42}}) {
      CHECK(edge_sparsify_estimate(g, 1.0, seed) == exact);
      CHECK(color_sparsify_estimate(g, 1, seed) == exact);
    }
  }
  auto g = biclique(2, 4);
  SparsifyConfig cfg;
  cfg.p = 0.4;
  cfg.seed = 99;
  cfg.trials = 8;
  Estimate est = sparsify_run(g, cfg);
  REQUIRE(est.per_group_means.size() == 8);
  for (uint64_t t = 0; t < 8; ++t)
    CHECK(est.per_group_means[t] == edge_sparsify_estimate(g, 0.4, derive_seed(99, t)));
  SparsifyConfig clr;
  clr.sparsifier = Sparsifier::Color;
  clr.colors = 1;
  clr.trials = 3;
  CHECK(sparsify_run(biclique(5, 5), clr).value == 100.0);
  auto k22 = biclique(2, 2);
  CHECK(edge_sparsify_value(k22, std::vector<bool>(4, false), 0.5) == 0.0);
  CHECK(color_sparsify_value(k22, {0, 1, 0, 1}, 2) == 0.0);
  CHECK_THROWS_AS(edge_sparsify_value(k22, std::vector<bool>(4, true), 0.0), ArgumentError);
  CHECK_THROWS_AS(color_sparsify_estimate(k22, 0, 0), ArgumentError);
  SparsifyConfig none;
  none.trials = 0;
  CHECK_THROWS_AS(sparsify_run(k22, none), ArgumentError);
}

int main() { return mini_main(); }
