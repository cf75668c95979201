/*
 * bfly_b200.h -- C-ABI of the B200-native butterfly-counting engine (sm_100a).
 *
 * This is the drop-in boundary under the reference's C++ counting API
 * (/root/reference/proj/include/bfly/ headers). The reference is a plain static C++ library
 * with no FFI of its own; a maintainer switches to this engine by linking
 * libbfly_b200.so and either calling these functions directly or using the C++ facade
 * in paper_1801_00338_b200/cpp/bfly_b200.hpp, which keeps the reference's names,
 * argument meaning and exception types.
 *
 * Conventions
 *   - Plain pointers and sizes only. Every pointer argument is a HOST pointer unless the
 *     function name ends in _device (then it is a device pointer on the handle's GPU).
 *   - Every function returns a status: 0 ok; nonzero maps to the reference's exception
 *     hierarchy (errors.hpp:10-58):
 *       BFLY_ARGUMENT 1 -> ArgumentError      BFLY_EMPTY 2    -> EmptyGraphError
 *       BFLY_OVERFLOW 3 -> OverflowError      BFLY_NO_WEDGES 4 -> NoWedgesError
 *       BFLY_INTERNAL 5 -> Error (CUDA failure, out of memory, missing device)
 *       BFLY_PARSE 6    -> ParseError (malformed edge-list line)
 *     bfly_last_error() returns the calling thread's last message.
 *   - Vertex numbering is the reference's: dense ids per side in first-seen order of the
 *     input edge list (graph.cpp:19-27); global index = left block first (graph.hpp:72-78);
 *     canonical edge k = k-th edge in (left, right) lexicographic order (graph.hpp:63-65).
 *   - A handle is immutable after build. Calls on one handle serialise on the handle's
 *     CUDA stream (a per-handle mutex); distinct handles run concurrently.
 *   - There is no CPU fallback: without a usable sm_100 device every call that needs the
 *     GPU fails with BFLY_INTERNAL.
 */
#ifndef BFLY_B200_H
#define BFLY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFLY_OK 0
#define BFLY_ARGUMENT 1
#define BFLY_EMPTY 2
#define BFLY_OVERFLOW 3
#define BFLY_NO_WEDGES 4
#define BFLY_INTERNAL 5
#define BFLY_PARSE 6

#define BFLY_SIDE_AUTO (-1)
#define BFLY_SIDE_LEFT 0
#define BFLY_SIDE_RIGHT 1

typedef struct bfly_graph bfly_graph; /* opaque device-resident graph */

/* graph.hpp:26-35 GraphStats */
typedef struct {
  uint64_t n, left, right, m;
  double sum_deg_sq_left, sum_deg_sq_right;
  uint64_t wedge_count; /* sum over all vertices of C(d,2) */
  uint32_t max_degree;
} bfly_stats;

/* ---- library ----------------------------------------------------------------------- */
const char* bfly_last_error(void);
const char* bfly_version(void);
/* 1 when an sm_100 device is usable, 0 otherwise (sets last_error). */
int bfly_device_ok(void);

/* ---- graph build: replaces BipartiteGraph::from_edges (graph.hpp:43, graph.cpp:31-58) --
 * Raw (left_id, right_id) multiset -> dense first-seen ids per side, duplicates dropped,
 * sorted adjacency both directions, left prefix offsets, right CSR with canonical edge ids.
 * m_in == 0 yields an empty graph (like the reference; its loaders reject that case).
 * At most m_in <= 2^31-1 input edges (checked -> ARGUMENT; the device sorts and the hub
 * plan index entries with 32-bit positions). */
int bfly_graph_build_u32(const uint32_t* left_ext, const uint32_t* right_ext, uint64_t m_in,
                         bfly_graph** out);
/* The reference's own input layout: `pairs` holds m_in interleaved (left, right) ids, i.e.
 * the storage of a std::vector<std::pair<uint64_t, uint64_t>> (graph.hpp:43). Pageable host
 * memory is narrowed to u32 by host threads into a page-locked stage and copied chunk by
 * chunk while the rest is packed (ids >= 2^32 take the u64 build). */
int bfly_graph_build_pairs(const uint64_t* pairs, uint64_t m_in, bfly_graph** out);
int bfly_graph_build_u64(const uint64_t* left_ext, const uint64_t* right_ext, uint64_t m_in,
                         bfly_graph** out);
/* Same, with the edge list already resident in device memory (bench 'value' path). The
 * arrays are read on the handle's stream: they must be complete before the call (the
 * producer synchronised), or be produced on the stream given to bfly_set_stream(). */
int bfly_graph_build_u32_device(const uint32_t* d_left_ext, const uint32_t* d_right_ext,
                                uint64_t m_in, bfly_graph** out);
void bfly_graph_free(bfly_graph* g);

/* ---- text ingestion / serialisation ------------------------------
 * load_edge_list (graph.cpp:75-99): `text` holds the whole stream (len bytes). Lines whose
 * first byte outside " \t\r" is missing, '%' or '#' are skipped; otherwise the first two
 * whitespace-separated tokens must be decimal uint64 ids (further tokens ignored). The
 * edges go through from_edges on the device. PARSE on the first malformed line
 * (*err_line = its 1-based number, message as the reference's ParseError); EMPTY when no
 * edge remains. */
int bfly_graph_load_text(const char* text, uint64_t len, bfly_graph** out, uint64_t* err_line);
/* serialize_edge_list (graph.cpp:107-112): "% bip\n" then "lid rid\n" per canonical edge
 * with external ids. *len = bytes needed; the text is written when buf != NULL (ARGUMENT
 * when cap < *len). */
int bfly_graph_serialize(bfly_graph* g, char* buf, uint64_t cap, uint64_t* len);

/* graph.hpp:47-51 left_count / right_count / edge_count */
int bfly_graph_sizes(const bfly_graph* g, uint32_t* left, uint32_t* right, uint64_t* m);
/* D2H copy of the canonical representation (any pointer may be NULL to skip):
 * loff[L+1], ladj[m] (left CSR, canonical order), roff[R+1], radj[m] (right CSR),
 * reid[m] (canonical edge id of each right-CSR entry), lids[L], rids[R] (external ids). */
int bfly_graph_export(const bfly_graph* g, uint64_t* loff, uint32_t* ladj, uint64_t* roff,
                      uint32_t* radj, uint32_t* reid, uint64_t* lids, uint64_t* rids);
/* graph.cpp:60-66 has_edge, graph.cpp:68-73 edge_at -- batched */
int bfly_has_edge_batch(bfly_graph* g, const uint32_t* l, const uint32_t* r, uint64_t k,
                        uint8_t* out);
int bfly_edge_at_batch(bfly_graph* g, const uint64_t* edge_idx, uint64_t k, uint32_t* l,
                       uint32_t* r);

/* graph.cpp:136-155 compute_stats (OVERFLOW when the wedge count exceeds 2^64-1) */
int bfly_graph_stats(bfly_graph* g, bfly_stats* out);
/* exact.cpp:9-21 choose_side: chosen = cost_left < cost_right ? RIGHT : LEFT */
int bfly_choose_side(bfly_graph* g, int* chosen, double* cost_left, double* cost_right);

/* ---- exact count: replaces exact_count / exact_count_side (exact.hpp:18-27) -----------
 * side: BFLY_SIDE_AUTO | LEFT | RIGHT. The count is the same for either side
 * (exact.hpp:20-24); the side is validated and reported, the device kernel is the
 * degree-priority wedge aggregation described in DESIGN.md. OVERFLOW iff bfly >= 2^64. */
int bfly_exact_count(bfly_graph* g, int side, uint64_t* out);

/* ---- local counts: replaces count_per_vertex / count_per_edge (local.hpp:12-19) -------
 * All-subject forms (API addition): out[g] = count_per_vertex(vertex_at(g)),
 * out[k] = count_per_edge(edge_at(k)). */
int bfly_local_vertex_all(bfly_graph* g, uint64_t* out /* n */);
int bfly_local_edge_all(bfly_graph* g, uint64_t* out /* m */);
/* Batched per-subject forms (per-sample kernels). ARGUMENT on an out-of-range id. */
int bfly_local_vertex_batch(bfly_graph* g, const uint64_t* gids, uint64_t k, uint64_t* out);
int bfly_local_edge_batch(bfly_graph* g, const uint64_t* edge_idx, uint64_t k, uint64_t* out);
/* count_per_edge(l, r) with explicit endpoints; ARGUMENT when (l, r) is not an edge. */
int bfly_local_edge_pairs(bfly_graph* g, const uint32_t* l, const uint32_t* r, uint64_t k,
                          uint64_t* out);
/* Wedge samples (sampling.cpp:85-91): centre global id, positions i != j in its adjacency;
 * out = |N(adj[i]) & N(adj[j])| - 1. */
int bfly_wedge_batch(bfly_graph* g, const uint64_t* centre_gid, const uint32_t* i,
                     const uint32_t* j, uint64_t k, uint64_t* out);
/* |N(v) & N(w)| for same-side pairs (side 0: left ids, 1: right ids) -- the sorted-merge
 * intersection_size of sampling.cpp:22-36, batched. ARGUMENT on an out-of-range id. */
int bfly_common_neighbors_batch(bfly_graph* g, int side, const uint32_t* v, const uint32_t* w,
                                uint64_t k, uint64_t* out);
/* sampling.cpp:63-73 build_wedge_index: prefix[n+1] of C(d,2) over global order. */
int bfly_wedge_index(bfly_graph* g, uint64_t* prefix /* n+1 */, uint64_t* total);

/* Batched estimator iterations with DEVICE-side sample ids: iteration q in
 * [first, first+count) draws from std::mt19937_64(derive_seed(seed, q)) exactly as
 * sampling.cpp:101-123 does (method 0 vertex: uniform_index(n); 1 edge: uniform_index(m);
 * 2 wedge: uniform_index(total) -> upper_bound over the C(d,2) prefix -> positions i, j).
 * counts[q] = the per-sample integer before scaling (count_per_vertex, count_per_edge,
 * or common - 1). ids / wi / wj (host, may be NULL) receive the drawn sample ids.
 * ARGUMENT on an empty graph, NO_WEDGES for method 2 on a wedge-free graph. */
int bfly_sample_batch(bfly_graph* g, int method, uint64_t seed, uint64_t first, uint64_t count,
                      uint64_t* counts, uint64_t* ids, uint32_t* wi, uint32_t* wj);

/* Method::FastEdge iterations (sampling.cpp:125-147) [first, first+count) with device-side
 * engines: iteration q draws (l, r) = edge_at(uniform_index(m)) from
 * std::mt19937_64(derive_seed(seed, q)), then `repeats` Bernoulli probes
 * has_edge(draw_excluding(N(r), l), draw_excluding(N(l), r)).
 * values[q] = fast_esamp_iteration's value (hits / repeats * (d_l-1) * (d_r-1) * m / 4, the
 * reference's operation order, bit-exact). hits / edge_ids (may be NULL) receive the probe
 * successes and the canonical edge id. ARGUMENT on repeats == 0 or an empty graph. */
int bfly_fast_edge_batch(bfly_graph* g, uint64_t seed, uint64_t first, uint64_t count,
                         uint64_t repeats, double* values, uint64_t* hits, uint64_t* edge_ids);

/* ---- sparsify-then-count: replaces count_retained + exact_count (sparsify.cpp:15-71) ---
 * ESpar keeps canonical edge k iff unit_double(derive_seed(seed,k)) < p (p in (0,1]);
 * CSpar keeps edges whose endpoints share colour bounded_from_bits(derive_seed(seed,g),N).
 * count = exact butterfly count of the retained subgraph; kept = retained edge count. */
int bfly_espar_count(bfly_graph* g, double p, uint64_t seed, uint64_t* count, uint64_t* kept);
int bfly_cspar_count(bfly_graph* g, uint64_t n_colors, uint64_t seed, uint64_t* count,
                     uint64_t* kept);
/* Explicit masks (edge_sparsify_value / color_sparsify_value, sparsify.hpp:26-29). */
int bfly_keep_mask_count(bfly_graph* g, const uint8_t* keep /* m */, uint64_t* count,
                         uint64_t* kept);
int bfly_color_mask_count(bfly_graph* g, const uint32_t* colors /* n */, uint64_t* count,
                          uint64_t* kept);

/* ---- butterfly pair types at scale: replaces classify_pairs (oracle.hpp:34-44, -------
 * oracle.cpp:60-94). The reference enumerates every butterfly and
 * classifies all C(bfly,2) pairs (guarded to desk-size graphs); this computes the same
 * five counts from counting identities: per-subject local counts,
 * and the moments sum C(c,3), sum C(c,4) of the common-neighbour counts c of all same-side
 * vertex pairs (one device pass with work = the wedge count). Counts can exceed 64 bits
 * on large graphs (C(bfly,2) alone does on config 2), so each is a (low, high) pair of
 * 64-bit words. No size guard: the facade's classify_pairs applies the reference's
 * OracleGuards itself. OVERFLOW iff bfly >= 2^64. */
typedef struct {
  uint64_t bfly;
  uint64_t p_0v[2], p_1v[2], p_2v[2], p_1e[2], p_1w[2]; /* (low, high) words */
} bfly_pair_counts;
int bfly_pair_type_counts(bfly_graph* g, bfly_pair_counts* out);

/* ---- instrumentation (bench / profiling; not part of the reference API) -------------- */
/* Opaque cudaStream_t of the handle (for callers that time with their own events). */
void* bfly_graph_stream(bfly_graph* g);
/* Handles built later by the calling thread run on `stream` (a cudaStream_t the caller
 * owns and keeps alive) instead of a private stream; NULL restores private streams. */
void bfly_set_stream(void* stream);
/* Path of the last vertex/edge sample batch on g: 0 per-sample kernels, 1 all-subject LOCAL
 * pass (cached on the handle) + gather. Both give identical counts; the cheaper is chosen
 * from the batch's walk length (environment BFLY_SAMPLE_PATH=direct|all forces one). */
int bfly_last_sample_path(bfly_graph* g);
/* When enabled, every library kernel launch is bracketed by CUDA events on the handle's
 * stream; per-kernel-name totals are kept until reset. */
void bfly_profile_enable(int on);
void bfly_profile_reset(void);
/* Number of distinct kernel names recorded; fill name/ms/launches for index i. */
int bfly_profile_count(void);
int bfly_profile_get(int i, const char** name, double* total_ms, uint64_t* launches);
/* Launch counter (always on): total kernels launched by the library since reset. */
uint64_t bfly_launch_count(void);
/* Sparsify diagnostics (bench roofline). collect >= 0 switches collection on g on (1) or
 * off (0; the default: it costs an extra pass); out (6 values, may be NULL) receives the last
 * ESpar / CSpar / mask call's figures: retained edges m', edges left after peeling the
 * retained-degree-1 endpoints, left / right vertices of the counted sub-graph, W_C of the
 * retained graph under the reference's side rule (collected only), vertices of the
 * retained graph (collected only). */
int bfly_sparsify_stats(bfly_graph* g, int collect, uint64_t* out);
/* Device memory: every engine allocation comes from a private stream-ordered pool per
 * device (the default pool and its release threshold are left alone). The pool keeps freed
 * memory for reuse and grows once to about 160 B per input edge on the first build of a
 * size; bfly_trim_pool releases all but keep_bytes of the unused part to the driver
 * (cudaMemPoolTrimTo) on the current device. */
int bfly_trim_pool(uint64_t keep_bytes);
/* Work statistics of the last exact count on g: wedges processed by the priority kernels,
 * the reference's anchor-side wedge count W_C for the chosen side, and per bucket the
 * tasks, wedges and adjacency segments processed: [0,6) start path, [6,12) hub path, each
 * (tiny, small-A, small-B, medium, medium-wide, heavy/split); bucket_starts[12] = number of
 * hub starts k. */
int bfly_last_exact_stats(bfly_graph* g, uint64_t* wedges_processed, uint64_t* ref_wedges,
                          uint64_t* bucket_starts /* 13 */, uint64_t* bucket_wedges /* 12 */,
                          uint64_t* bucket_entries /* 12 */);
/* The dense top-hub part of the last exact count on g (csrc/hubdense.cuh; no counterpart in
 * the reference, whose exact.cpp:29-41 walks every wedge): out[0] = hubs H counted from
 * per-vertex masks, out[1] = mask words per vertex, out[2] = wedges taken by that path (they
 * are part of wedges_processed above), out[3] = adjacency entries (mask rows) it read,
 * out[4] = those of them that belong to end vertices of more than 255 entries. */
int bfly_last_dense_stats(bfly_graph* g, uint64_t* out /* 5 */);

#ifdef __cplusplus
}
#endif
#endif
