/*
 * bfly_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference butterfly-counting library
 * (/root/reference/proj, namespace bfly). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * Every function cites the reference file:line whose behaviour it restates.
 *
 * Parity pins: tests/test_oracle_golden.py checks this restatement against the
 * reference's own known-answer tests (proj/tests/) and against golden vectors
 * produced by the reference compiled here (oracle/_ref, tests/golden/).
 *
 * Status codes mirror the C-ABI in include/bfly_b200.h:
 *   0 ok, 1 ArgumentError, 2 EmptyGraphError, 3 OverflowError, 4 NoWedgesError,
 *   5 internal / allocation failure.
 */
#ifndef BFLY_ORACLE_H
#define BFLY_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:10-31 -------------------------------------------------------- */
uint64_t bo_mix64(uint64_t x);
uint64_t bo_derive_seed(uint64_t seed, uint64_t index);
double bo_unit_double(uint64_t bits);
uint64_t bo_bounded_from_bits(uint64_t bits, uint64_t n);

/* ---- rng.hpp:36-62: std::mt19937_64 + mask-rejection bounded draws ---------- */
typedef struct {
  uint64_t mt[312];
  int mti;
} bo_rng;
void bo_rng_seed(bo_rng* r, uint64_t seed);
void bo_rng_stream(bo_rng* r, uint64_t seed, uint64_t index);
uint64_t bo_rng_next(bo_rng* r);
double bo_rng_uniform_unit(bo_rng* r);
uint64_t bo_rng_uniform_index(bo_rng* r, uint64_t n);

/* ---- checked.hpp:9-27 ------------------------------------------------------ */
/* returns 0 ok / 3 overflow */
int bo_choose2(uint64_t c, uint64_t* out);

/* ---- graph.hpp:40-89, graph.cpp:31-73 -------------------------------------- */
typedef struct {
  uint32_t L, R;
  uint64_t m;
  uint64_t* loff; /* L+1 */
  uint32_t* ladj; /* m, sorted per list */
  uint64_t* roff; /* R+1 */
  uint32_t* radj; /* m, sorted per list */
  uint64_t* lids; /* external ids, first-seen order */
  uint64_t* rids;
} bo_graph;

int bo_graph_from_edges(bo_graph* g, const uint64_t* l, const uint64_t* r, uint64_t m_in);
int bo_graph_from_edges_u32(bo_graph* g, const uint32_t* l, const uint32_t* r, uint64_t m_in);
void bo_graph_free(bo_graph* g);
int bo_parse_edge_list(const char* t, uint64_t len, uint64_t** l, uint64_t** r, uint64_t* m,
                       uint64_t* err_line, char* msg, uint64_t cap);
uint64_t bo_serialize_edge_list(const bo_graph* g, char* buf, uint64_t cap);
int bo_has_edge(const bo_graph* g, uint32_t l, uint32_t r);
int bo_edge_at(const bo_graph* g, uint64_t k, uint32_t* l, uint32_t* r);

/* graph.cpp:114-134 test generators (fixtures) -> edge lists (caller frees) */
int bo_complete_biclique_edges(uint32_t a, uint32_t b, uint64_t** l, uint64_t** r, uint64_t* m);
int bo_random_bipartite_edges(uint32_t a, uint32_t b, double p, uint64_t seed, uint64_t** l,
                              uint64_t** r, uint64_t* m);
void bo_free(void* p);

/* graph.cpp:136-155 */
typedef struct {
  uint64_t n, left, right, m;
  double sum_deg_sq_left, sum_deg_sq_right;
  uint64_t wedge_count;
  uint32_t max_degree;
} bo_stats;
int bo_compute_stats(const bo_graph* g, bo_stats* s);

/* ---- exact.cpp:9-47 -------------------------------------------------------- */
/* side: 0 = Left, 1 = Right */
void bo_choose_side(const bo_graph* g, int* chosen, double* cost_left, double* cost_right);
int bo_exact_count_side(const bo_graph* g, int side, int threads, uint64_t* out);
int bo_exact_count(const bo_graph* g, int threads, uint64_t* out);

/* ---- local.cpp:11-44 ------------------------------------------------------- */
int bo_count_per_vertex(const bo_graph* g, int side, uint32_t index, uint64_t* out);
int bo_count_per_edge(const bo_graph* g, uint32_t l, uint32_t r, uint64_t* out);
/* all subjects (loops the tests use, local.cpp thread-safety note local.hpp:10-11) */
int bo_count_all_vertices(const bo_graph* g, int threads, uint64_t* out /* n, global order */);
int bo_count_all_edges(const bo_graph* g, int threads, uint64_t* out /* m, canonical order */);
int bo_count_edges_subset(const bo_graph* g, const uint64_t* ks, uint64_t nk, int threads,
                          uint64_t* out);
int bo_count_vertices_subset(const bo_graph* g, const uint64_t* gids, uint64_t nk, int threads,
                             uint64_t* out);

/* ---- sampling.cpp:22-123 --------------------------------------------------- */
int bo_build_wedge_index(const bo_graph* g, uint64_t* prefix /* n+1 */, uint64_t* total);
uint64_t bo_intersection_size(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb);
int bo_vertex_sample_value(const bo_graph* g, int side, uint32_t index, double* out);
int bo_edge_sample_value(const bo_graph* g, uint32_t l, uint32_t r, double* out);
int bo_wedge_sample_value(const bo_graph* g, uint64_t total_wedges, int centre_side,
                          uint32_t centre, uint32_t v, uint32_t w, double* out);
/* per-outcome integer counts (what the device returns) */
int bo_wedge_common_minus_1(const bo_graph* g, int centre_side, uint32_t v, uint32_t w,
                            uint64_t* out);

/* Sample-id draws of {v,e,w}samp_iteration (sampling.cpp:101-123) from
 * Rng::stream(seed, index). method: 0 vertex, 1 edge, 2 wedge.
 * id0: vertex -> global vertex index; edge -> canonical edge index;
 *      wedge -> centre global index.  id1,id2: wedge leaf positions i, j in adj. */
int bo_sample_draw(const bo_graph* g, const uint64_t* prefix, uint64_t total_wedges, int method,
                   uint64_t seed, uint64_t index, uint64_t* id0, uint32_t* id1, uint32_t* id2);
int bo_sample_iteration(const bo_graph* g, const uint64_t* prefix, uint64_t total_wedges,
                        int method, uint64_t seed, uint64_t index, double* value);

/* run_estimator fixed-iteration mode (sampling.cpp:157-202, 243-278).
 * per_group (groups entries) may be NULL when groups == 1. */
int bo_run_estimator(const bo_graph* g, int method, uint64_t iterations, uint64_t seed,
                     uint64_t groups, uint64_t group_size, int threads, double* value,
                     uint64_t* iterations_done, double* per_group, double* values_out);
int bo_run_estimator_ex(const bo_graph* g, int method, uint64_t iterations, uint64_t seed,
                        uint64_t groups, uint64_t group_size, uint64_t repeats, int threads,
                        double* value, uint64_t* iterations_done, double* per_group,
                        double* values_out);
/* Method::FastEdge (sampling.cpp:125-147) */
int bo_fast_ebfc_estimate(const bo_graph* g, uint32_t l, uint32_t r, uint64_t repeats,
                          bo_rng* rng, double* out, uint64_t* hits);
int bo_fast_esamp_iteration(const bo_graph* g, uint64_t repeats, uint64_t seed, uint64_t index,
                            double* value, uint64_t* edge_id, uint64_t* hits);

/* ---- sparsify.cpp:15-94 ---------------------------------------------------- */
int bo_count_retained(const bo_graph* g, const uint8_t* keep, int threads, uint64_t* count,
                      uint64_t* kept_edges);
int bo_edge_sparsify_value(const bo_graph* g, const uint8_t* keep, double p, int threads,
                           double* out);
int bo_color_sparsify_value(const bo_graph* g, const uint32_t* colors, uint64_t n_colors,
                            int threads, double* out);
int bo_edge_sparsify_estimate(const bo_graph* g, double p, uint64_t seed, int threads,
                              double* out, uint64_t* count, uint64_t* kept_edges);
int bo_color_sparsify_estimate(const bo_graph* g, uint64_t n_colors, uint64_t seed, int threads,
                               double* out, uint64_t* count, uint64_t* kept_edges);
int bo_sparsify_run(const bo_graph* g, int sparsifier /*0 edge, 1 color*/, double p,
                    uint64_t colors, uint64_t seed, uint64_t trials, int threads, double* value,
                    double* per_trial);

/* ---- oracle.cpp:37-58 (brute force, desk scale) ----------------------------- */
int bo_brute_force_count(const bo_graph* g, uint64_t* out);
/* oracle.cpp:60-94 classify_pairs (enumeration; guards as OracleGuards): out[6] = bfly,
 * p_0v, p_1v, p_2v, p_1e, p_1w */
int bo_classify_pairs(const bo_graph* g, uint32_t max_side, uint64_t max_bfly, uint64_t* out);
/* oracle.cpp:96-116 variance_bounds: out[5] = vsamp, esamp, wsamp, espar, clrspar */
int bo_variance_bounds(uint64_t n, uint64_t m, uint64_t wedges, const uint64_t* counts, double p,
                       double* out);
/* the same pair counts from pair moments + local counts (checker beyond enumeration size):
 * out[11] = bfly, (lo, hi) of p_0v, p_1v, p_2v, p_1e, p_1w */
int bo_pair_counts_by_moments(const bo_graph* g, int threads, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
