// local.cuh -- host entry points of the local-count, sample and sparsify translation units.
#pragma once

#include "graph.cuh"

namespace bflyd {

namespace agg {
struct LocalOut;
struct RunStats;
}  // namespace agg

// exact.cu: hub path + start path over every start; LOCAL scatters per-vertex/per-edge
template <bool LOCAL>
uint64_t count_all_starts(bfly_graph* g, agg::LocalOut lo, agg::RunStats* rs_hub,
                          agg::RunStats* rs_start);

// local.cu
void ensure_two_hop(bfly_graph* g);
void local_all(bfly_graph* g, bool edges, DBuf<unsigned long long>& vcnt,
               DBuf<unsigned long long>& ecnt);
void local_vertex_all(bfly_graph* g, uint64_t* out);
void local_edge_all(bfly_graph* g, uint64_t* out);
void local_vertex_batch_device(bfly_graph* g, const uint64_t* d_gids, uint64_t k,
                               unsigned long long* d_out);
void ensure_local(bfly_graph* g, bool edges);
uint64_t device_sum(bfly_graph* g, const unsigned long long* a, uint64_t k);
bool prefer_all_subjects(bfly_graph* g, uint64_t direct_cost, bool edges);
void gather_all_subjects(bfly_graph* g, bool edges, const uint64_t* d_idx, uint64_t k,
                         unsigned long long* d_out);

// samples.cu
// d_k (canonical ids of the pairs) may be null; computed when the gather path is chosen
void local_edge_batch_device(bfly_graph* g, const uint32_t* d_l, const uint32_t* d_r,
                             const uint64_t* d_k, uint64_t k, unsigned long long* d_out);
void edge_at_device(bfly_graph* g, const uint64_t* d_k, uint64_t k, uint32_t* d_l, uint32_t* d_r);
void has_edge_device(bfly_graph* g, const uint32_t* d_l, const uint32_t* d_r, uint64_t k,
                     uint8_t* d_out);
void wedge_batch_device(bfly_graph* g, const uint64_t* d_c, const uint32_t* d_i,
                        const uint32_t* d_j, uint64_t k, unsigned long long* d_out);
void wedge_index(bfly_graph* g, uint64_t* prefix, uint64_t* total);
void wedge_prefix_device(bfly_graph* g, unsigned long long* d_pre, uint64_t* total);

// sampler.cu: device-side mt19937_64 sample ids (method 0 vertex, 1 edge, 2 wedge)
void ensure_wedge_prefix(bfly_graph* g);
void draw_samples_device(bfly_graph* g, int method, uint64_t seed, uint64_t first,
                         uint64_t count, uint64_t* d_ids, uint32_t* d_i, uint32_t* d_j);
void sample_counts_device(bfly_graph* g, int method, uint64_t seed, uint64_t first,
                          uint64_t count, unsigned long long* d_out, uint64_t* d_ids,
                          uint32_t* d_i, uint32_t* d_j);
void common_pairs_device(bfly_graph* g, int side, const uint32_t* d_v, const uint32_t* d_w,
                         uint64_t k, unsigned long long* d_out);

// fastedge.cu: Method::FastEdge iterations [first, first+count) (values, hits, edge ids)
void fast_edge_device(bfly_graph* g, uint64_t seed, uint64_t first, uint64_t count,
                      uint64_t repeats, double* d_values, uint64_t* d_hits, uint64_t* d_edges);

// textio.cu: load_edge_list / serialize_edge_list on the device
uint64_t parse_text_device(cudaStream_t s, const char* text, uint64_t len, DBuf<uint64_t>& dl,
                           DBuf<uint64_t>& dr, uint64_t* err_line);
uint64_t serialize_device(bfly_graph* g, char* out);

// pairs.cu: pair-type counts (oracle.cpp:60-94 by counting identities)
void pair_moments(bfly_graph* g, uint64_t* c2_total, unsigned __int128* s3, unsigned __int128* s4);
void local_choose2_sums(bfly_graph* g, unsigned __int128* v2, unsigned __int128* e2);

// sparsify.cu
void sparsify_count(bfly_graph* g, int mode, double p, uint64_t n_colors, uint64_t seed,
                    const uint8_t* h_keep, const uint32_t* h_colors, uint64_t* count,
                    uint64_t* kept);

}  // namespace bflyd
