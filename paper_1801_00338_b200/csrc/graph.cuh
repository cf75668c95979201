// graph.cuh -- the device-resident bipartite graph behind the opaque bfly_graph handle.
//
// HBM layout (all arrays device-resident for the handle's lifetime):
//   canonical (reference numbering, graph.hpp:40-89)
//     loff[L+1] u64, ladj[m] u32      left CSR, canonical edge order (edge_at(k) = row of k)
//     roff[R+1] u64, radj[m] u32      right CSR, lists sorted by dense left id
//     reid[m]   u32                   canonical edge id of each right-CSR entry
//     lids[L], rids[R] u64            external ids in first-seen order
//   priority (built lazily for exact / all-local counts)
//     rank[n], inv[n] u32             global id <-> priority id (degree desc, gid asc)
//     poff[n+1] u64, padj[2m] u32     merged-side CSR in priority ids, lists ascending
//     psrc[2m] u32                    row (priority id) of every entry
//     peid[2m] u32                    canonical edge id of every entry (local-edge only)
//     sfx[2m]  u32                    forward entries (u -> v, v > u): position of u in N(v)+1
//     work[n]  u64                    wedges of start u = sum over forward entries of the
//                                     suffix N(v) after u
#pragma once

#include <cstdint>
#include <mutex>

#include "../../include/bfly_b200.h"
#include "common.cuh"

// Declared first in bfly_graph so it is destroyed LAST: every DBuf member frees its memory
// on the stream (cudaFreeAsync) before the stream itself is synchronised and destroyed.
struct StreamOwner {
  cudaStream_t s = nullptr;
  bool owns = false;
  ~StreamOwner() {
    if (s) {
      cudaStreamSynchronize(s);
      if (owns) cudaStreamDestroy(s);
    }
  }
};

struct bfly_graph {
  StreamOwner owner;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  std::mutex mu;

  uint32_t L = 0, R = 0;
  uint64_t m = 0;

  bflyd::DBuf<uint64_t> loff, roff;
  bflyd::DBuf<uint32_t> ladj, radj, reid;
  // reid is derived on first use for handles made by build_graph (ensure_reid)
  bool reid_ready = true;
  bflyd::DBuf<uint64_t> lids, rids;
  // row of every CSR entry, kept from the build (left id of canonical edge k; right id of
  // right-CSR entry j); empty on handles not made by build_graph (sparsify sub-graphs)
  bflyd::DBuf<uint32_t> lrow, rrow;

  // degree statistics (computed once)
  bool stats_ready = false;
  int stats_status = 0;
  bfly_stats stats{};
  double cost_left = 0.0, cost_right = 0.0;
  unsigned __int128 wedges_side[2] = {0, 0};  // sum C(d,2) per side (exact)

  // priority structure
  bool prio_ready = false;
  bool prio_has_eid = false;
  bflyd::DBuf<uint32_t> rank, inv;
  bflyd::DBuf<uint64_t> poff;
  bflyd::DBuf<uint32_t> padj, psrc, peid;
  bflyd::DBuf<uint2> fseg;  // forward entry u -> v: (start, length) of N(v) after u
  bflyd::DBuf<uint64_t> work;
  bflyd::DBuf<uint64_t> fwd;  // first forward entry of each start
  uint64_t total_work = 0;
  uint64_t prio_nz = 0;  // priority ids with edges (degree order: ids >= prio_nz are isolated)

  // two-hop walk length per global vertex (vertex-sample work), built lazily
  bool two_hop_ready = false;
  bflyd::DBuf<uint64_t> two_hop;

  // all-subject local counts (local.cu), cached: lv per global vertex, le per canonical edge
  bool local_ready = false;  // lv and le hold the all-subject counts
  bool lv_ready = false;     // lv does (vertex-only pass or the full one)
  bflyd::DBuf<unsigned long long> lv, le;
  int last_sample_path = 0;  // 0 per-sample kernels, 1 all-subject pass + gather

  // wedge-sampling prefix of C(d,2) over global order (sampling.cpp:63-73), built lazily
  bool wpre_ready = false;
  bflyd::DBuf<unsigned long long> wpre;
  uint64_t wtotal = 0;

  // hub plan (exact.cu): starts u < hub_k are enumerated from their end vertex w
  bool hub_ready = false;
  uint32_t hub_k = 0;
  uint32_t hub_k1 = 0;  // hubs below k1 need 32-bit counters (degree >= 65536)
  uint32_t start_deg_max = 0xFFFFFFFFu;  // degree of priority id hub_k: bounds every start task's counts
  bflyd::DBuf<uint16_t> hlen;     // per priority-CSR entry (w -> v): hub prefix length of N(v)
  bflyd::DBuf<uint32_t> hpst;     // per entry with hlen > 0: poff[v] (m < 2^31 -> fits)
  bflyd::DBuf<uint64_t> hub_work; // per end vertex w: keys of its hub task
  // dense top-hub path (hubdense.cuh): the plan's segments skip the hubs below hub_h, whose
  // wedges are counted from the per-vertex masks hmask[v * hub_w + j] (hub_h = 0: no dense
  // path; such a plan serves the local-count pass too, a plan with hub_h > 0 only the count)
  uint32_t hub_h = 0, hub_w = 0;
  bflyd::DBuf<uint32_t> hmask;
  uint64_t hub_dense_keys = 0, hub_dense_entries = 0, hub_dense_big_entries = 0;
  uint64_t hub_bucket_tasks[6] = {}, hub_bucket_keys[6] = {};
  uint64_t hub_bucket_entries[6] = {};

  // exact-count bookkeeping
  uint64_t last_wedges = 0;
  int last_side = -1;  // side argument of the last exact count (W_C is derived lazily)
  // per bucket: tiny, small-A, small-B, medium, medium-wide, heavy/split (aggregate.cuh)
  uint64_t bucket_starts[6] = {}, bucket_wedges[6] = {};
  uint64_t bucket_entries[6] = {};


  // sparsify statistics of the last ESpar/CSpar/mask call (collected when spar_stats_on):
  // [0] retained edges m', [1] edges left after peeling, [2] / [3] left / right vertices of
  // the counted sub-graph, [4] W_C of the retained graph G' under the reference's side rule
  // (exact.cpp:9-21 on G'), [5] vertices of G' (endpoints of retained edges)
  bool spar_stats_on = false;
  uint64_t spar_stats[6] = {};

  uint64_t n() const { return uint64_t{L} + R; }
};

namespace bflyd {

// hub path: at most kHubMax hub starts; a start becomes a hub when its work exceeds
// kHubMinWork (it would otherwise leave the shared-memory buckets)
constexpr uint64_t kHubMax = 32767;  // < 2^15: hub prefix lengths fit 15 bits
constexpr uint64_t kHubMinWork = 8192;

// graph_build.cu
// canonical edge id of every right-CSR entry (reid), derived on first use (graph_build.cu)
void ensure_reid(bfly_graph* g);

// in-place ascending sort of keys[rs[r] .. rs[r+1]) for every row r (segsort.cu); adds the
// number of adjacent equal keys inside the sorted rows to *dups (device counter)
void seg_sort_rows(uint32_t* keys, const uint32_t* rs, uint32_t rows, int kbits, cudaStream_t s,
                   unsigned long long* dups);

template <typename K>
void build_graph(bfly_graph* g, const K* d_l, const K* d_r, uint64_t m_in,
                 cudaEvent_t right_ready = nullptr);
void ensure_stats(bfly_graph* g);

// priority.cu
void ensure_priority(bfly_graph* g, bool with_eid);

// exact.cu
uint64_t exact_count_device(bfly_graph* g, const uint32_t* d_poff_override = nullptr);

// Generic sub-graph counter used by exact and sparsify: counts butterflies of the graph
// given by a canonical left CSR over the same dense ids (rows L, cols R).
struct CsrView {
  uint32_t L, R;
  uint64_t m;
  const uint64_t* loff;
  const uint32_t* ladj;
  const uint64_t* roff;
  const uint32_t* radj;
  const uint32_t* reid;
};

}  // namespace bflyd
