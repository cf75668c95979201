// exact.cu -- exact butterfly count on B200 (replaces exact_count_side, exact.cpp:23-43),
// plus the shared bucketing kernel and heavy-row scratch of the aggregation engine.
//
// Each butterfly is counted once at its highest-priority vertex u (priority.cu). The
// reference anchors at every vertex of the chosen side and walks w < v in dense-id order;
// both enumerate each butterfly exactly once, so the uint64 results are identical for
// either reference side (exact.hpp:20-24). See aggregate.cuh for the kernels.
#include "aggregate.cuh"

namespace bflyd {
namespace agg {

__global__ void k_bucket(const unsigned long long* __restrict__ work, uint64_t n,
                         uint32_t* __restrict__ lists, unsigned long long* __restrict__ counts,
                         unsigned long long* __restrict__ wsum,
                         unsigned long long* __restrict__ heavy_work) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) & ~31ull;
  for (uint64_t base = warp * 32; base < n; base += stride) {
    const uint64_t u = base + lane;
    const unsigned long long wk = u < n ? work[u] : 0ull;
    const int b = wk == 0 ? -1 : wk <= kTinyMax ? 0 : wk <= kSmallMax ? 1 : wk <= kMedMax ? 2 : 3;
    for (int q = 0; q < 4; ++q) {
      const unsigned mask = __ballot_sync(0xffffffffu, b == q);
      if (!mask) continue;
      const int leader = __ffs(mask) - 1;
      unsigned long long s = (b == q) ? wk : 0ull;
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      unsigned long long basei = 0;
      if ((int)lane == leader) {
        basei = atomicAdd(&counts[q], (unsigned long long)__popc(mask));
        atomicAdd(&wsum[q], s);
      }
      basei = __shfl_sync(0xffffffffu, basei, leader);
      if (b == q) {
        const uint64_t idx = basei + __popc(mask & ((1u << lane) - 1u));
        lists[q * n + idx] = static_cast<uint32_t>(u);
        if (q == 3) heavy_work[idx] = wk;
      }
    }
  }
}

void ensure_rows(bfly_graph* g, uint64_t n_row) {
  cudaStream_t s = g->stream;
  const uint64_t budget = 4ull << 30;  // rows + touched lists
  const uint32_t want =
      static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(64, budget / (n_row * 8))));
  if (g->rows.n >= uint64_t{want} * n_row) {
    g->row_slots = static_cast<uint32_t>(std::min<uint64_t>(64, g->rows.n / n_row));
    return;
  }
  g->rows.alloc(uint64_t{want} * n_row, s);
  g->rows.zero();
  g->row_touched.alloc(uint64_t{want} * n_row, s);
  g->row_ntouched.alloc(want, s);
  g->row_ntouched.zero();
  g->row_slots = want;
}

}  // namespace agg

uint64_t exact_count_device(bfly_graph* g, const uint32_t*) {
  ensure_priority(g, false);
  g->last_wedges = 0;
  for (int q = 0; q < 4; ++q) g->bucket_starts[q] = g->bucket_wedges[q] = 0;
  const uint64_t n = g->n();
  if (n == 0 || g->m == 0) return 0;
  agg::ExactSrc src{g->poff.p, g->padj.p, g->sfx.p, g->fwd.p};
  agg::RunStats rs;
  static const char* const names[4] = {"exact_bucket", "exact_tiny", "exact_small",
                                       "exact_medium"};
  const uint64_t total = agg::run<agg::ExactSrc, false>(
      g, src, reinterpret_cast<const unsigned long long*>(g->work.p), n, n, nullptr,
      agg::LocalOut{nullptr, nullptr, nullptr, nullptr}, &rs, names);
  for (int q = 0; q < 4; ++q) {
    g->bucket_starts[q] = rs.starts[q];
    g->bucket_wedges[q] = rs.wedges[q];
    g->last_wedges += rs.wedges[q];
  }
  return total;
}

}  // namespace bflyd
