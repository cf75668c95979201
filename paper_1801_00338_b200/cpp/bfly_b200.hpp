// bfly_b200.hpp -- C++ facade of the B200 engine with the reference's counting API.
//
// Drop-in for the reference headers proj/include/bfly/{graph,exact,local,sampling,
// sparsify,rng,checked,errors}.hpp: same namespace (bfly), same names, argument meaning and
// exception types. Every counting call runs on the GPU through the C-ABI of
// libbfly_b200.so (include/bfly_b200.h); this layer owns the handle, host-side RNG streams
// (std::mt19937_64, rng.hpp:36-62), index-ordered double reductions and error mapping.
// See INTEGRATION.md for the switch-over recipe.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

struct bfly_graph;

namespace bfly {

// ---- errors (errors.hpp:10-58) ---------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ParseError : public Error {
 public:
  ParseError(const std::string& what, uint64_t line)
      : Error(what + " (line " + std::to_string(line) + ")"), line_(line) {}
  uint64_t line() const { return line_; }

 private:
  uint64_t line_;
};
#define BFLY_B200_ERROR(Name) \
  class Name : public Error { \
   public:                    \
    using Error::Error;       \
  };
BFLY_B200_ERROR(EmptyGraphError)
BFLY_B200_ERROR(ArgumentError)
BFLY_B200_ERROR(NoWedgesError)
BFLY_B200_ERROR(OverflowError)
BFLY_B200_ERROR(SizeGuardError)
BFLY_B200_ERROR(InternalError)
#undef BFLY_B200_ERROR

// Throws the reference exception type matching a C-ABI status (no-op on 0).
void throw_status(int status);

// ---- checked arithmetic (checked.hpp:9-27) ------------------------------------------------
uint64_t checked_add(uint64_t a, uint64_t b);
uint64_t checked_mul(uint64_t a, uint64_t b);
uint64_t choose2(uint64_t c);

// ---- rng (rng.hpp:10-62) -------------------------------------------------------------------
uint64_t mix64(uint64_t x);
uint64_t derive_seed(uint64_t seed, uint64_t index);
double unit_double(uint64_t bits);
uint64_t bounded_from_bits(uint64_t bits, uint64_t n);

class Rng {
 public:
  explicit Rng(uint64_t seed) : engine_(seed) {}
  static Rng stream(uint64_t seed, uint64_t index) { return Rng(derive_seed(seed, index)); }
  uint64_t next() { return engine_(); }
  double uniform_unit() { return unit_double(next()); }
  uint64_t uniform_index(uint64_t n);  // mask rejection, n <= 1 draws nothing

 private:
  std::mt19937_64 engine_;
};

// ---- graph (graph.hpp:11-112) ----------------------------------------------------------------
enum class Side : uint8_t { Left, Right };
inline Side opposite(Side s) { return s == Side::Left ? Side::Right : Side::Left; }
inline const char* side_name(Side s) { return s == Side::Left ? "left" : "right"; }

struct VertexRef {
  Side side;
  uint32_t index;
};
inline bool operator==(VertexRef a, VertexRef b) { return a.side == b.side && a.index == b.index; }

struct GraphStats {
  uint64_t n = 0;
  uint64_t left = 0;
  uint64_t right = 0;
  uint64_t m = 0;
  double sum_deg_sq_left = 0.0;
  double sum_deg_sq_right = 0.0;
  uint64_t wedge_count = 0;
  uint32_t max_degree = 0;
};

// Device-resident, immutable. Copies share the device handle. neighbors() reads a host
// mirror of the canonical CSR that is downloaded on first use.
class BipartiteGraph {
 public:
  static BipartiteGraph from_edges(const std::vector<std::pair<uint64_t, uint64_t>>& edges);
  // API addition: contiguous 32-bit id arrays (what the synthetic configs use)
  static BipartiteGraph from_edges_u32(const uint32_t* left, const uint32_t* right, uint64_t m);
  // Wrap a handle built through the C-ABI (owning: freed with the last copy).
  static BipartiteGraph adopt(bfly_graph* handle, bool owning);

  uint32_t left_count() const { return L_; }
  uint32_t right_count() const { return R_; }
  uint32_t side_count(Side s) const { return s == Side::Left ? L_ : R_; }
  uint64_t vertex_count() const { return uint64_t{L_} + R_; }
  uint64_t edge_count() const { return m_; }

  std::span<const uint32_t> neighbors(Side s, uint32_t i) const;
  uint32_t degree(Side s, uint32_t i) const;
  uint32_t degree(VertexRef v) const { return degree(v.side, v.index); }
  bool has_edge(uint32_t l, uint32_t r) const;
  std::pair<uint32_t, uint32_t> edge_at(uint64_t k) const;
  uint64_t external_id(Side s, uint32_t i) const;
  VertexRef vertex_at(uint64_t g) const {
    if (g < L_) return {Side::Left, static_cast<uint32_t>(g)};
    return {Side::Right, static_cast<uint32_t>(g - L_)};
  }
  uint64_t global_index(VertexRef v) const {
    return v.side == Side::Left ? v.index : uint64_t{L_} + v.index;
  }

  bfly_graph* device() const { return h_.get(); }

 private:
  struct Mirror;
  BipartiteGraph() = default;
  const Mirror& mirror() const;
  std::shared_ptr<bfly_graph> h_;
  std::shared_ptr<Mirror> mirror_;
  uint32_t L_ = 0, R_ = 0;
  uint64_t m_ = 0;
};

GraphStats compute_stats(const BipartiteGraph& g);

// graph.cpp:75-112: edge-list text in and out, parsed / formatted on the device
BipartiteGraph load_edge_list(std::istream& in);
BipartiteGraph load_edge_list_file(const std::string& path);
void serialize_edge_list(const BipartiteGraph& g, std::ostream& out);
// graph.cpp:114-134 fixture generators (edge list drawn on the host, built on the device)
BipartiteGraph complete_biclique(uint32_t a, uint32_t b);
BipartiteGraph random_bipartite(uint32_t a, uint32_t b, double p, uint64_t seed);

// ---- exact (exact.hpp:9-27) -------------------------------------------------------------------
struct SideChoice {
  Side chosen = Side::Left;
  double cost_left = 0.0;
  double cost_right = 0.0;
};
SideChoice choose_side(const BipartiteGraph& g);
uint64_t exact_count_side(const BipartiteGraph& g, Side iterate);
uint64_t exact_count(const BipartiteGraph& g);

// ---- local (local.hpp:12-19) + all-subject additions ------------------------------------------
uint64_t count_per_vertex(const BipartiteGraph& g, VertexRef v);
uint64_t count_per_edge(const BipartiteGraph& g, uint32_t l, uint32_t r);
std::vector<uint64_t> count_all_vertices(const BipartiteGraph& g);  // global order
std::vector<uint64_t> count_all_edges(const BipartiteGraph& g);     // canonical order
std::vector<uint64_t> count_vertices(const BipartiteGraph& g, const std::vector<uint64_t>& gids);
std::vector<uint64_t> count_edges(const BipartiteGraph& g, const std::vector<uint64_t>& ks);

// ---- sampling (sampling.hpp:11-91) --------------------------------------------------------------
enum class Method : uint8_t { Vertex, Edge, Wedge, FastEdge };
const char* method_name(Method m);

struct EstimatorConfig {
  Method method = Method::Edge;
  uint64_t iterations = 0;
  double time_budget_seconds = 0.0;
  uint64_t seed = 0;
  uint64_t groups = 1;
  uint64_t group_size = 0;
  uint64_t fast_edge_repeats = 1000;
  bool record_trace = false;
};

struct TracePoint {
  double elapsed_seconds = 0.0;
  uint64_t iteration = 0;
  double estimate = 0.0;
};

struct Estimate {
  double value = 0.0;
  uint64_t iterations_done = 0;
  double elapsed_seconds = 0.0;
  uint64_t seed = 0;
  std::vector<double> per_group_means;
  std::vector<TracePoint> trace;
};

struct WedgeIndex {
  std::vector<uint64_t> prefix;
  uint64_t total = 0;
};

WedgeIndex build_wedge_index(const BipartiteGraph& g);
double vertex_sample_value(const BipartiteGraph& g, VertexRef v);
double edge_sample_value(const BipartiteGraph& g, uint32_t l, uint32_t r);
double wedge_sample_value(const BipartiteGraph& g, uint64_t total_wedges, VertexRef center,
                          uint32_t v, uint32_t w);
double vsamp_iteration(const BipartiteGraph& g, Rng& rng);
double esamp_iteration(const BipartiteGraph& g, Rng& rng);
double wsamp_iteration(const BipartiteGraph& g, const WedgeIndex& index, Rng& rng);
// Method::FastEdge (sampling.cpp:93-99, 125-147). The caller's Rng advances exactly as in the
// reference (draws on the host engine); the probes run as one device has_edge batch.
double fast_edge_pair_value(const BipartiteGraph& g, uint32_t l, uint32_t r, uint32_t other_l,
                            uint32_t other_r);
double fast_ebfc_estimate(const BipartiteGraph& g, uint32_t l, uint32_t r, uint64_t repeats,
                          Rng& rng);
double fast_esamp_iteration(const BipartiteGraph& g, uint64_t repeats, Rng& rng);

// Batched B200 estimator: sample ids drawn on the GPU from Rng::stream(seed, i)-identical
// engines (bfly_sample_batch), per-sample counts in the same device batch, index-ordered
// double reduction on the host. Equal to the reference's run_estimator; `threads` is
// accepted for compatibility and unused.
Estimate run_estimator(const BipartiteGraph& g, const EstimatorConfig& cfg, unsigned threads = 1);

struct IterationPlan {
  uint64_t groups = 1;
  uint64_t group_size = 1;
};
IterationPlan plan_iterations(double variance_bound, double pilot_bfly, double epsilon,
                              double delta);

// Host restatement of the sample ids of iterations [first, first+count) on `threads` host
// threads (the device sampler must reproduce these exactly):
// Vertex -> global vertex id; Edge -> canonical edge id; Wedge -> centre global id + the
// two leaf positions in its adjacency (sampling.cpp:101-123).
struct SampleIds {
  std::vector<uint64_t> id;
  std::vector<uint32_t> i, j;
};
SampleIds sample_ids(const BipartiteGraph& g, Method m, uint64_t seed, uint64_t first,
                     uint64_t count, const WedgeIndex* index, unsigned threads);

// ---- sparsify (sparsify.hpp:11-52) -----------------------------------------------------------
enum class Sparsifier : uint8_t { Edge, Color };
const char* sparsifier_name(Sparsifier s);

struct SparsifyConfig {
  Sparsifier sparsifier = Sparsifier::Edge;
  double p = 0.5;
  uint64_t colors = 2;
  uint64_t seed = 0;
  uint64_t trials = 1;
};

double edge_sparsify_value(const BipartiteGraph& g, const std::vector<bool>& keep, double p);
double color_sparsify_value(const BipartiteGraph& g, const std::vector<uint32_t>& colors,
                            uint64_t n_colors);
double edge_sparsify_estimate(const BipartiteGraph& g, double p, uint64_t seed);
double color_sparsify_estimate(const BipartiteGraph& g, uint64_t n_colors, uint64_t seed);
Estimate sparsify_run(const BipartiteGraph& g, const SparsifyConfig& cfg);

// ---- butterfly pair types and variance bounds (oracle.hpp:13-58) ----------
struct OracleGuards {
  uint32_t max_side = 64;           // per side
  uint64_t max_butterflies = 2000;  // pair classification limit
};

struct PairTypeCounts {
  uint64_t bfly = 0;
  uint64_t p_0v = 0;  // disjoint
  uint64_t p_1v = 0;  // one shared vertex
  uint64_t p_2v = 0;  // two shared vertices, same side, no shared edge
  uint64_t p_1e = 0;  // one shared edge
  uint64_t p_1w = 0;  // one shared wedge

  uint64_t p_V() const { return p_1v + p_2v + p_1e + p_1w; }
  uint64_t p_E() const { return p_1e + p_1w; }
  uint64_t total_pairs() const { return p_0v + p_1v + p_2v + p_1e + p_1w; }
};

struct VarianceBounds {
  double vsamp = 0.0;    // n (bfly + p_V) / 4
  double esamp = 0.0;    // m (bfly + p_E) / 4
  double wsamp = 0.0;    // wedges (bfly + p_1w) / 4
  double espar = 0.0;    // bfly p^-4 + 2 p_1w p^-2 + 2 p_1e p^-1
  double clrspar = 0.0;  // bfly p^-3 + 2 p_1w p^-2 + 2 (p_1e + p_2v) p^-1
};

// The reference's classify_pairs contract (same guards, same SizeGuardError messages, counts
// equal to its enumeration), computed on the GPU from counting identities instead of by
// enumerating the C(bfly,2) pairs (bfly_pair_type_counts).
PairTypeCounts classify_pairs(const BipartiteGraph& g, const OracleGuards& guards = {});
VarianceBounds variance_bounds(const GraphStats& stats, const PairTypeCounts& counts, double p);

// At scale (API addition): no guards; the pair counts of large graphs exceed 64 bits.
struct PairTypeCountsWide {
  uint64_t bfly = 0;
  unsigned __int128 p_0v = 0, p_1v = 0, p_2v = 0, p_1e = 0, p_1w = 0;
};
PairTypeCountsWide classify_pairs_at_scale(const BipartiteGraph& g);
// oracle.cpp:96-116 with the wide counts (each converted to double once, as the reference
// converts its uint64 fields; equal to variance_bounds whenever the counts fit 64 bits)
VarianceBounds variance_bounds(const GraphStats& stats, const PairTypeCountsWide& counts,
                               double p);

struct SparsifyThresholds {
  double espar_min_p = 0.0;
  double clrspar_min_p = 0.0;
};
SparsifyThresholds suggest_p(const GraphStats& stats, double pilot_bfly);

}  // namespace bfly
