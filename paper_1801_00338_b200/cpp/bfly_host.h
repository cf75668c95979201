/* bfly_host.h -- C exports of the C++ facade's host-side drivers (libbfly_host.so), for
 * callers that are not C++ (the Python tests and bench.py). They wrap bfly::run_estimator,
 * bfly::sample_ids and bfly::sparsify_run over a handle built through include/bfly_b200.h.
 * Status codes are those of bfly_b200.h; message via bfly_host_last_error(). */
#ifndef BFLY_HOST_H
#define BFLY_HOST_H
#include <stdint.h>

#include "../../include/bfly_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* bfly_host_last_error(void);

/* method: 0 vertex, 1 edge, 2 wedge. per_group: `groups` doubles (groups > 1).
 * trace_out: 3 doubles per point (iteration, estimate, elapsed); *trace_len in = capacity,
 * out = number of points. */
int bfly_host_run_estimator(bfly_graph* g, int method, uint64_t iterations, double time_budget,
                            uint64_t seed, uint64_t groups, uint64_t group_size,
                            int record_trace, unsigned threads, double* value,
                            uint64_t* iterations_done, double* per_group, double* trace_out,
                            uint64_t* trace_len);

/* same with EstimatorConfig::fast_edge_repeats (sampling.hpp:22) */
int bfly_host_run_estimator_ex(bfly_graph* g, int method, uint64_t iterations, double time_budget,
                               uint64_t seed, uint64_t groups, uint64_t group_size,
                               uint64_t fast_edge_repeats, int record_trace, unsigned threads,
                               double* value, uint64_t* iterations_done, double* per_group,
                               double* trace_out, uint64_t* trace_len);

/* Wall time of the reference-signature call sequence: BipartiteGraph::from_edges(
 * const std::vector<std::pair<uint64_t, uint64_t>>&) + exact_count, reps times, on an edge
 * vector built (untimed) from left/right; ms[reps] per call, *count = the last count. */
int bfly_host_time_from_pairs(const uint32_t* left, const uint32_t* right, uint64_t m, int reps,
                              double* ms, uint64_t* count);

int bfly_host_sample_ids(bfly_graph* g, int method, uint64_t seed, uint64_t first, uint64_t count,
                         unsigned threads, uint64_t* id, uint32_t* i, uint32_t* j);

int bfly_host_sparsify_run(bfly_graph* g, int sparsifier, double p, uint64_t colors, uint64_t seed,
                           uint64_t trials, double* value, double* per_trial);

#ifdef __cplusplus
}
#endif
#endif
