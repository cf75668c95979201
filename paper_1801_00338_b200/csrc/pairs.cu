// pairs.cu -- butterfly pair-type counts at scale, the input of the
// variance tables. Replaces the enumeration in classify_pairs (reference oracle.cpp:60-94),
// which lists every butterfly and classifies all C(bfly, 2) pairs, by counting identities
// that need only per-subject counts and per-pair moments:
//
//   c_xy = |N(x) & N(y)| for a same-side pair {x, y} (both sides);
//   S3 = sum over same-side pairs of C(c,3),  S4 = sum of C(c,4)
//   V2 = sum over vertices of C(bfly_v, 2),   E2 = sum over edges of C(bfly_e, 2)
//
//   p_1w = 3 S3        two butterflies share a wedge {x, y | a} + a 4th vertex each:
//                      per pair {x, y}, c (c-1 choose 2) = 3 C(c,3)
//   p_2v = 3 S4        share {x, y} only: disjoint 2-subsets of the c common neighbours
//   p_1e = E2 - 2 p_1w every pair sharing k edges appears k times in E2 (p_1w pairs share 2)
//   p_1v = V2 - 2 p_2v - 2 p_1e - 3 p_1w   (pairs sharing k vertices appear k times in V2)
//   p_0v = C(bfly, 2) - p_1v - p_2v - p_1e - p_1w
//
// S3 and S4 come from one pass of the aggregation engine (aggregate.cuh, PairSrc): task = u,
// entries = all of N(u), segment = N(v) after u (priority order), so every same-side pair is
// aggregated once with its FULL multiplicity; the final multiplicities are drained into
// 128-bit sums. The pass's own C(c,2) total must equal 2 * bfly (each butterfly has one pair
// per side), which is checked. Work = sum over all vertices of C(d,2) (the wedge count).
#include "aggregate.cuh"
#include "local.cuh"

namespace bflyd {
namespace {

// aseg[q] for every directed priority entry q = (u -> v): the suffix of N(v) after u (u is in
// N(v); rows ascend). work[u] = sum of the suffix lengths (warp-segmented, one atomic per run).
__global__ void k_pair_plan(const uint64_t* __restrict__ poff, const uint32_t* __restrict__ padj,
                            const uint32_t* __restrict__ psrc, uint64_t nnz,
                            uint2* __restrict__ aseg, unsigned long long* __restrict__ work) {
  const unsigned lane = threadIdx.x & 31, full = 0xffffffffu;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) & ~31ull;
  for (uint64_t base = warp * 32; base < nnz; base += stride) {
    const uint64_t q = base + lane;
    const bool valid = q < nnz;
    const uint32_t u = valid ? psrc[q] : 0xFFFFFFFFu;
    unsigned long long wk = 0;
    if (valid) {
      const uint32_t v = padj[q];
      uint64_t lo = poff[v], hi = poff[v + 1];
      const uint64_t e = hi;
      while (lo < hi) {  // lower_bound(u) in N(v)
        const uint64_t mid = (lo + hi) >> 1;
        if (padj[mid] < u) lo = mid + 1;
        else hi = mid;
      }
      aseg[q] = make_uint2(static_cast<uint32_t>(lo + 1), static_cast<uint32_t>(e - lo - 1));
      wk = e - lo - 1;
    }
    const uint32_t up = __shfl_up_sync(full, u, 1);
    const unsigned heads = __ballot_sync(full, lane == 0 || up != u);
    const int my_head = 31 - __clz(heads & ((2u << lane) - 1u));
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long y = __shfl_up_sync(full, wk, off);
      if ((int)lane - off >= my_head) wk += y;
    }
    const uint32_t dn = __shfl_down_sync(full, u, 1);
    if (valid && (lane == 31 || dn != u) && wk) atomicAdd(&work[u], wk);
  }
}

// out[0..1] += sum over i of C(a[i], 2) as a 128-bit (lo, hi) pair
__global__ void k_sum_choose2(const unsigned long long* __restrict__ a, uint64_t k,
                              unsigned long long* __restrict__ out) {
  unsigned __int128 s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = a[i];
    if (x >= 2) {
      const unsigned long long p = x & 1 ? x : x >> 1, q = x & 1 ? (x - 1) >> 1 : x - 1;
      s += (unsigned __int128)p * q;  // C(x,2) < 2^127 for any 64-bit x
    }
  }
  for (int off = 16; off > 0; off >>= 1) s += agg::shfl_xor_u128(s, off);
  if ((threadIdx.x & 31) == 0 && s) agg::atomic_add_u128(out, s);
}

}  // namespace

// (Sigma C(c,2), S3, S4) over all same-side pairs
void pair_moments(bfly_graph* g, uint64_t* c2_total, unsigned __int128* s3, unsigned __int128* s4) {
  cudaStream_t s = g->stream;
  *c2_total = 0;
  *s3 = *s4 = 0;
  const uint64_t n = g->n(), nnz = 2 * g->m;
  if (n == 0 || g->m == 0) return;
  ensure_priority(g, false);
  DBuf<uint2> aseg(nnz, s);
  DBuf<unsigned long long> work(n, s), mom(4, s);
  work.zero();
  mom.zero();
  launch("pair_plan", k_pair_plan, grid_for(nnz, 256, 148u * 64u), 256, 0, s, g->poff.p,
         g->padj.p, g->psrc.p, nnz, aseg.p, work.p);
  agg::PairSrc src{g->poff.p, g->padj.p, aseg.p};
  agg::LocalOut lo{nullptr, nullptr, nullptr, nullptr};
  lo.mom = mom.p;
  static const char* const names[8] = {"pair_bucket", "pair_tiny",   "pair_small",
                                       "pair_medium", "pair_medium", "pair_heavy",
                                       "pair_phase",  "pair_small_b"};
  const agg::Plan<agg::Hash<9>, agg::Hash<10>, agg::Hash<14>> plan{0, {32, 256, 512, 8192}, 0};
  *c2_total = agg::run<agg::PairSrc, false>(g, src, plan, work.p, nullptr, n, n, nullptr, lo,
                                            nullptr, names);
  unsigned long long h[4] = {0, 0, 0, 0};
  read_back(s, {{h, mom.p, sizeof(h)}});
  *s3 = ((unsigned __int128)h[1] << 64) | h[0];
  *s4 = ((unsigned __int128)h[3] << 64) | h[2];
}

// V2 and E2 from the all-subject counts (computed once per handle, local.cu)
void local_choose2_sums(bfly_graph* g, unsigned __int128* v2, unsigned __int128* e2) {
  cudaStream_t s = g->stream;
  *v2 = *e2 = 0;
  if (g->m == 0) return;
  ensure_local(g, true);
  DBuf<unsigned long long> acc(4, s);
  acc.zero();
  const uint64_t n = g->n(), m = g->m;
  launch("pair_sum_v2", k_sum_choose2, grid_for(n, 256, 592), 256, 0, s,
         reinterpret_cast<const unsigned long long*>(g->lv.p), n, acc.p);
  launch("pair_sum_e2", k_sum_choose2, grid_for(m, 256, 592), 256, 0, s,
         reinterpret_cast<const unsigned long long*>(g->le.p), m, acc.p + 2);
  unsigned long long h[4];
  read_back(s, {{h, acc.p, sizeof(h)}});
  *v2 = ((unsigned __int128)h[1] << 64) | h[0];
  *e2 = ((unsigned __int128)h[3] << 64) | h[2];
}

}  // namespace bflyd
