// local.cu -- per-vertex / per-edge butterfly counts (replaces count_per_vertex and
// count_per_edge, local.cpp:11-44) for all subjects and for batches of vertex samples.
//
// All subjects: one LOCAL pass of the priority wedge aggregation (aggregate.cuh) scatters
// every butterfly to its 4 vertices and 4 edges; sum_v = sum_e = 4 * bfly
// (tests/test_local.cpp:61-77). Vertex samples: a task per sample walks the unfiltered
// distance-2 neighbourhood N(N(v)) \ {v} exactly as local.cpp:14-18 does.
#include <cstdlib>
#include <cstring>

#include "aggregate.cuh"
#include "local.cuh"

namespace bflyd {
namespace {

__global__ void k_gather_vertex(const unsigned long long* __restrict__ vcnt,
                                const uint32_t* __restrict__ rank, uint64_t n,
                                unsigned long long* __restrict__ out) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n;
       g += (uint64_t)gridDim.x * blockDim.x)
    out[g] = vcnt[rank[g]];
}

// W2[x] = sum over y in N(x) of (d_y - 1), per global vertex (left block first):
// the element count of the distance-2 walk of count_per_vertex(x).
__global__ void k_two_hop(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                          const uint64_t* __restrict__ ooff, uint32_t rows, uint64_t nnz,
                          const uint32_t* __restrict__ rowof, uint64_t gbase,
                          unsigned long long* __restrict__ w2) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) & ~31ull;
  for (uint64_t base = warp * 32; base < nnz; base += stride) {
    const uint64_t e = base + lane;
    const bool valid = e < nnz;
    const uint32_t r = valid ? rowof[e] : 0xFFFFFFFFu;
    unsigned long long x = 0;
    if (valid) {
      const uint32_t y = adj[e];
      x = ooff[y + 1] - ooff[y] - 1;
    }
    const unsigned full = 0xffffffffu;
    const uint32_t up = __shfl_up_sync(full, r, 1);
    const bool head = lane == 0 || up != r;
    const unsigned heads = __ballot_sync(full, head);
    const int my_head = 31 - __clz(heads & ((2u << lane) - 1u));
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(full, x, o);
      if ((int)lane - o >= my_head) x += y;
    }
    const uint32_t dn = __shfl_down_sync(full, r, 1);
    const bool tail = lane == 31 || dn != r;
    if (valid && tail && x) atomicAdd(&w2[gbase + r], x);
  }
  (void)off;
  (void)rows;
}

// per-entry accumulators -> canonical edge counts (each edge has two priority entries)
__global__ void k_fold_edges(const unsigned long long* __restrict__ pacc,
                             const uint32_t* __restrict__ peid, uint64_t nnz,
                             unsigned long long* __restrict__ ecnt) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = pacc[e];
    if (x) atomicAdd(&ecnt[peid[e]], x);
  }
}

__global__ void k_mark_rows2(const uint64_t* __restrict__ off, uint32_t rows,
                             uint32_t* __restrict__ mark) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    if (off[r + 1] > off[r]) mark[off[r]] = static_cast<uint32_t>(r);
}

__global__ void k_sample_work(const uint64_t* __restrict__ gids, uint64_t k,
                              const unsigned long long* __restrict__ w2,
                              unsigned long long* __restrict__ work) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x)
    work[i] = w2[gids[i]];
}

}  // namespace

void ensure_two_hop(bfly_graph* g) {
  if (g->two_hop_ready) return;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n();
  g->two_hop.alloc(n ? n : 1, s);
  g->two_hop.zero();
  if (g->m) {
    for (int side = 0; side < 2; ++side) {
      const uint64_t* off = side == 0 ? g->loff.p : g->roff.p;
      const uint32_t* adj = side == 0 ? g->ladj.p : g->radj.p;
      const uint64_t* ooff = side == 0 ? g->roff.p : g->loff.p;
      const uint32_t rows = side == 0 ? g->L : g->R;
      DBuf<uint32_t> mark(g->m, s), rowof(g->m, s);
      mark.zero();
      launch("local_mark_rows", k_mark_rows2, grid_for(rows, 256), 256, 0, s, off, rows, mark.p);
      inclusive_max(mark.p, rowof.p, g->m, s);
      launch("local_two_hop", k_two_hop, grid_for(g->m, 256, 148u * 64u), 256, 0, s, off, adj,
             ooff, rows, g->m, rowof.p, side == 0 ? uint64_t{0} : uint64_t{g->L},
             reinterpret_cast<unsigned long long*>(g->two_hop.p));
    }
  }
  g->two_hop_ready = true;
}

// LOCAL pass over all starts; vcnt is indexed by priority id, ecnt by canonical edge id.
// edges = false: per-vertex counts only -- no per-entry accumulators, no canonical edge ids in
// the priority CSR, and no global atomic per wedge in the walks (the per-key scatter exists
// only for the wedge's second edge).
void local_all(bfly_graph* g, bool edges, DBuf<unsigned long long>& vcnt,
               DBuf<unsigned long long>& ecnt) {
  cudaStream_t s = g->stream;
  ensure_priority(g, edges);
  const uint64_t n = g->n();
  vcnt.alloc(n ? n : 1, s);
  vcnt.zero();
  if (edges) {
    ecnt.alloc(g->m ? g->m : 1, s);
    ecnt.zero();
  }
  if (n == 0 || g->m == 0) return;
  const uint64_t nnz = 2 * g->m;
  DBuf<unsigned long long> pacc;
  if (edges) {
    pacc.alloc(nnz, s);
    pacc.zero();
  }
  agg::LocalOut lo{vcnt.p, pacc.p, edges ? g->peid.p : nullptr, g->padj.p};
  count_all_starts<true>(g, lo, nullptr, nullptr);
  if (edges)
    launch("local_fold_edges", k_fold_edges, grid_for(nnz, 256), 256, 0, s, pacc.p, g->peid.p, nnz,
           ecnt.p);
}

// All-subject counts, computed once per graph by one LOCAL pass and cached (the graph is
// immutable): lv[g] in global vertex order, le[k] in canonical edge order. A caller that only
// needs vertices (count_all_vertices, vertex sample gathers) gets the cheaper vertex-only pass;
// a later request for edges runs the full pass (which refreshes lv with the same values).
void ensure_local(bfly_graph* g, bool edges) {
  if (g->local_ready || (!edges && g->lv_ready)) return;
  cudaStream_t s = g->stream;
  DBuf<unsigned long long> vcnt, ecnt;
  local_all(g, edges, vcnt, ecnt);
  const uint64_t n = g->n();
  g->lv.alloc(n ? n : 1, s);
  if (n)
    launch("local_gather_vertex", k_gather_vertex, grid_for(n, 256), 256, 0, s, vcnt.p,
           g->rank.p, n, reinterpret_cast<unsigned long long*>(g->lv.p));
  if (edges) g->le = std::move(ecnt);
  BFLY_CUDA(cudaStreamSynchronize(s));
  g->lv_ready = true;
  if (edges) g->local_ready = true;
}

void local_vertex_all(bfly_graph* g, uint64_t* out) {
  cudaStream_t s = g->stream;
  ensure_local(g, false);
  if (g->n() == 0) return;
  BFLY_CUDA(cudaMemcpyAsync(out, g->lv.p, g->n() * 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
}

void local_edge_all(bfly_graph* g, uint64_t* out) {
  cudaStream_t s = g->stream;
  ensure_local(g, true);
  if (g->m == 0) return;
  BFLY_CUDA(cudaMemcpyAsync(out, g->le.p, g->m * 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
}

namespace {

__global__ void k_gather_u64(const unsigned long long* __restrict__ src,
                             const uint64_t* __restrict__ idx, uint64_t k,
                             unsigned long long* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

__global__ void k_sum_u64(const unsigned long long* __restrict__ a, uint64_t k,
                          unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x)
    s += a[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

}  // namespace

uint64_t device_sum(bfly_graph* g, const unsigned long long* a, uint64_t k) {
  cudaStream_t s = g->stream;
  DBuf<unsigned long long> acc(1, s);
  acc.zero();
  if (k) launch("sum_u64", k_sum_u64, grid_for(k, 256, 592), 256, 0, s, a, k, acc.p);
  unsigned long long h = 0;
  BFLY_CUDA(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Per-sample kernels or all-subject pass + gather: both give identical integers; choose
// the cheaper one (BFLY_SAMPLE_PATH=direct|all overrides). direct_cost = elements the
// per-sample walks would touch.
bool prefer_all_subjects(bfly_graph* g, uint64_t direct_cost, bool edges) {
  const char* env = std::getenv("BFLY_SAMPLE_PATH");
  if (env && std::strcmp(env, "direct") == 0) return false;
  if (env && std::strcmp(env, "all") == 0) return true;
  if (g->local_ready || (!edges && g->lv_ready)) return true;
  if (direct_cost < (200ull << 20)) return false;
  ensure_priority(g, edges);
  const uint64_t all_cost =
      2 * (device_sum(g, reinterpret_cast<const unsigned long long*>(g->work.p), g->n()) + 2 * g->m);
  return direct_cost > 2 * all_cost;
}

void gather_all_subjects(bfly_graph* g, bool edges, const uint64_t* d_idx, uint64_t k,
                         unsigned long long* d_out) {
  ensure_local(g, edges);
  launch("local_gather_samples", k_gather_u64, grid_for(k, 256), 256, 0, g->stream,
         reinterpret_cast<const unsigned long long*>(edges ? g->le.p : g->lv.p), d_idx, k, d_out);
}

void local_vertex_batch_device(bfly_graph* g, const uint64_t* d_gids, uint64_t k,
                               unsigned long long* d_out) {
  cudaStream_t s = g->stream;
  BFLY_CUDA(cudaMemsetAsync(d_out, 0, k * 8, s));
  if (k == 0 || g->m == 0) return;
  ensure_two_hop(g);
  DBuf<unsigned long long> work(k, s);
  launch("vsamp_work", k_sample_work, grid_for(k, 256), 256, 0, s, d_gids, k,
         reinterpret_cast<const unsigned long long*>(g->two_hop.p), work.p);
  if (prefer_all_subjects(g, device_sum(g, work.p, k), false)) {
    g->last_sample_path = 1;
    gather_all_subjects(g, false, d_gids, k, d_out);
    return;
  }
  g->last_sample_path = 0;
  agg::VertexSrc src{d_gids, g->L, g->loff.p, g->ladj.p, g->roff.p, g->radj.p};
  static const char* const names[8] = {"vsamp_bucket", "vsamp_tiny",   "vsamp_small",
                                       "vsamp_medium", "vsamp_medium", "vsamp_heavy", "vsamp_phase", "vsamp_small_b"};
  const uint64_t n_row = std::max<uint64_t>(std::max<uint64_t>(g->L, g->R), 1);
  const agg::Plan<agg::Hash<9>, agg::Hash<10>, agg::Hash<14>> plan{
      0, {32, 256, 512, 8192}, 0};
  agg::run<agg::VertexSrc, false>(g, src, plan, work.p, nullptr, k, n_row, d_out,
                                  agg::LocalOut{nullptr, nullptr, nullptr, nullptr}, nullptr,
                                  names);
}

}  // namespace bflyd
