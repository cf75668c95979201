// sampler.cu -- device-side sample-id derivation for the batched estimators.
//
// Iteration q of run_estimator draws from its own engine std::mt19937_64(derive_seed(seed, q))
// (rng.hpp:36-62, sampling.cpp:101-123): vertex / edge ids by mask-rejection
// uniform_index, wedges by uniform_index(total) -> upper_bound over the C(d,2) prefix ->
// two distinct neighbour positions. The host facade used to derive these ids on its cores
// (~0.4 us per engine seed + twist); here one thread per sample produces the identical
// draws on the GPU and feeds them straight into the per-sample count kernels.
//
// LazyMT: the first 156 outputs of mt19937_64 only read ORIGINAL state words (the twist of
// word j < n-m = 156 reads x[j], x[j+1], x[j+156]), so two running cursors of the seeding
// recurrence x[i] = f*(x[i-1] ^ x[i-1] >> 62) + i produce them in registers: 156 seeding
// steps up front, then 2 per draw. A sample that needs a 157th draw (mask rejection makes
// that astronomically rare, but it must still be exact) is listed and redrawn by
// k_slow_samples with the full 312-word engine in global scratch.
#include <cstdlib>

#include "common.cuh"
#include "graph.cuh"
#include "local.cuh"
#include "mt.cuh"

namespace bflyd {
namespace {

using namespace mt;

struct SampleArgs {
  int method;  // 0 vertex, 1 edge, 2 wedge
  uint64_t seed, first, count;
  uint64_t n, m, total;
  uint32_t L;
  const uint64_t* loff;
  const uint64_t* roff;
  const unsigned long long* wpre;  // n+1 prefix of C(d,2) (wedge only)
  uint64_t* ids;
  uint32_t* wi;
  uint32_t* wj;
};

// one iteration of sampling.cpp:101-123 (draw part); false when the engine bailed out
template <class Gen>
__device__ bool draw_sample(const SampleArgs& a, Gen& gen, uint64_t q) {
  uint64_t id;
  if (a.method == 0) {
    if (!uniform_index(gen, a.n, id)) return false;
    a.ids[q] = id;
    return true;
  }
  if (a.method == 1) {
    if (!uniform_index(gen, a.m, id)) return false;
    a.ids[q] = id;
    return true;
  }
  uint64_t r;
  if (!uniform_index(gen, a.total, r)) return false;
  uint64_t lo = 0, hi = a.n + 1;  // upper_bound(prefix, r) - 1
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a.wpre[mid] <= r) lo = mid + 1;
    else hi = mid;
  }
  id = lo - 1;
  const uint64_t d =
      id < a.L ? a.loff[id + 1] - a.loff[id] : a.roff[id - a.L + 1] - a.roff[id - a.L];
  uint64_t i, j;
  if (!uniform_index(gen, d, i)) return false;
  if (!uniform_index(gen, d - 1, j)) return false;
  if (j >= i) ++j;
  a.ids[q] = id;
  a.wi[q] = static_cast<uint32_t>(i);
  a.wj[q] = static_cast<uint32_t>(j);
  return true;
}

__global__ void __launch_bounds__(256) k_draw_samples(SampleArgs a, uint32_t max_draws,
                                                      uint64_t* __restrict__ slow,
                                                      unsigned long long* __restrict__ n_slow) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < a.count;
       q += (uint64_t)gridDim.x * blockDim.x) {
    LazyMT gen;
    gen.seed(derive_seed(a.seed, a.first + q), max_draws);
    if (!draw_sample(a, gen, q)) slow[atomicAdd(n_slow, 1ull)] = q;
  }
}

__global__ void k_slow_samples(SampleArgs a, const uint64_t* __restrict__ slow,
                               const unsigned long long* __restrict__ n_slow,
                               uint64_t* __restrict__ scratch) {
  const uint64_t ns = *n_slow;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  FullMT gen{scratch + t * kMtN, 0};
  for (uint64_t s = t; s < ns; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = slow[s];
    gen.seed(derive_seed(a.seed, a.first + q));
    draw_sample(a, gen, q);
  }
}

}  // namespace

void ensure_wedge_prefix(bfly_graph* g) {
  if (g->wpre_ready) return;
  g->wpre.alloc(g->n() + 1, g->stream);
  wedge_prefix_device(g, g->wpre.p, &g->wtotal);
  g->wpre_ready = true;
}

// ids (+ wedge positions) of iterations [first, first+count) into device arrays
void draw_samples_device(bfly_graph* g, int method, uint64_t seed, uint64_t first,
                         uint64_t count, uint64_t* d_ids, uint32_t* d_i, uint32_t* d_j) {
  if (!count) return;
  cudaStream_t s = g->stream;
  SampleArgs a{};
  a.method = method;
  a.seed = seed;
  a.first = first;
  a.count = count;
  a.n = g->n();
  a.m = g->m;
  a.L = g->L;
  a.loff = g->loff.p;
  a.roff = g->roff.p;
  a.ids = d_ids;
  a.wi = d_i;
  a.wj = d_j;
  if (method == 2) {
    ensure_wedge_prefix(g);
    if (g->wtotal == 0) fail(kNoWedges, "graph has no wedges to sample");
    a.total = g->wtotal;
    a.wpre = g->wpre.p;
  }
  // BFLY_SAMPLER_FAST_DRAWS lowers the register engine's draw limit (tests drive the
  // full-engine path with it); the default is the whole first twist block
  uint32_t max_draws = kMtM;
  if (const char* env = std::getenv("BFLY_SAMPLER_FAST_DRAWS")) max_draws = (uint32_t)std::atoi(env);
  DBuf<uint64_t> slow(count, s);
  DBuf<unsigned long long> n_slow(1, s);
  n_slow.zero();
  launch("sampler_draw", k_draw_samples, grid_for(count, 256), 256, 0, s, a, max_draws, slow.p,
         n_slow.p);
  const uint32_t slow_threads = (uint32_t)std::min<uint64_t>(count, 1024);
  DBuf<uint64_t> scratch(uint64_t{slow_threads} * kMtN, s);
  launch("sampler_slow", k_slow_samples, (slow_threads + 127) / 128, 128, 0, s, a, slow.p,
         n_slow.p, scratch.p);
}

// counts of iterations [first, first+count): the per-sample integers of vsamp / esamp /
// wsamp (sampling.cpp:75-99) before scaling
void sample_counts_device(bfly_graph* g, int method, uint64_t seed, uint64_t first,
                          uint64_t count, unsigned long long* d_out, uint64_t* d_ids,
                          uint32_t* d_i, uint32_t* d_j) {
  draw_samples_device(g, method, seed, first, count, d_ids, d_i, d_j);
  if (!count) return;
  if (method == 0) {
    local_vertex_batch_device(g, d_ids, count, d_out);
  } else if (method == 1) {
    DBuf<uint32_t> dl(count, g->stream), dr(count, g->stream);
    edge_at_device(g, d_ids, count, dl.p, dr.p);
    local_edge_batch_device(g, dl.p, dr.p, d_ids, count, d_out);
  } else {
    wedge_batch_device(g, d_ids, d_i, d_j, count, d_out);
  }
}

}  // namespace bflyd
