// graph_build.cu -- device-side BipartiteGraph::from_edges (graph.cpp:31-58) and
// compute_stats / choose_side (graph.cpp:136-155, exact.cpp:9-21).
//
// Reference semantics reproduced exactly:
//   * dense ids per side in FIRST-SEEN order of the input list (graph.cpp:19-27):
//     stable radix sort of (external id, position); the head of each equal-key run holds
//     the first position; flags at first positions + exclusive scan rank the distinct ids
//     by first appearance.
//   * duplicate edges dropped, left lists sorted (graph.cpp:46-49): radix sort of packed
//     (dense_l << rb | dense_r) keys + unique -> canonical edge order = left CSR.
//   * right lists sorted (graph.cpp:50-53): stable sort of canonical edges by right id;
//     the payload is the canonical edge id (reid), needed by per-edge and ESpar paths.
#include <algorithm>
#include <mutex>
#include <vector>

#include <thrust/iterator/transform_iterator.h>

#include "cubwrap.cuh"
#include "graph.cuh"

namespace bflyd {
namespace {

__global__ void k_iota(uint32_t* v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

template <typename K>
__global__ void k_heads(const K* __restrict__ ks, const uint32_t* __restrict__ pos, uint64_t n,
                        uint32_t* __restrict__ headidx, uint32_t* __restrict__ firstflag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    bool h = (i == 0) || ks[i] != ks[i - 1];
    headidx[i] = h ? static_cast<uint32_t>(i) : 0u;
    if (h) firstflag[pos[i]] = 1u;
  }
}

template <typename K>
__global__ void k_assign(const K* __restrict__ ks, const uint32_t* __restrict__ pos,
                         const uint32_t* __restrict__ segstart,
                         const uint32_t* __restrict__ dense_of_pos, uint64_t n,
                         uint32_t* __restrict__ dense, uint64_t* __restrict__ ids) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = segstart[i];
    uint32_t d = dense_of_pos[pos[s]];
    dense[pos[i]] = d;
    if (s == i) ids[d] = static_cast<uint64_t>(ks[i]);
  }
}

// direct-address first-seen ids: first[id] = min position of id. An element skips the update
// when an earlier occurrence is already known: the previous element has the same id (runs),
// a per-block direct-mapped cache holds (id, a position of it below this one), or first[id]
// already is smaller (one cached read; most elements stop there). The cache keeps hub ids (up to
// ~10^6 occurrences in any input order) from serialising one L2 address.
template <typename K>
__global__ void __launch_bounds__(256) k_first_pos(const K* __restrict__ ks, uint64_t n,
                                                   uint32_t* __restrict__ first) {
  constexpr int kC = 2048;
  __shared__ unsigned long long cache[kC];
  for (int t = threadIdx.x; t < kC; t += blockDim.x) cache[t] = ~0ull;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = ks[i];
    if (i > 0 && ks[i - 1] == k) continue;
    const uint32_t pi = static_cast<uint32_t>(i);
    const uint32_t h = (static_cast<uint32_t>(k) * 0x9E3779B1u) >> 21;
    const unsigned long long c = cache[h];
    if (static_cast<uint32_t>(c >> 32) == static_cast<uint32_t>(k) &&
        static_cast<uint32_t>(c) <= pi)
      continue;
    // a stale (cached) value is never below the true minimum, so a cached read can only
    // cause a redundant atomicMin, never a wrong skip
    const uint32_t cur = __ldg(first + k);
    if (pi < cur) atomicMin(&first[k], pi);
    cache[h] = (static_cast<unsigned long long>(k) << 32) | (cur < pi ? cur : pi);
  }
}

// First-seen numbering without sorting: the first positions of the distinct ids are
// distinct, so one bit per input position marks them; dense id of an id = the number of
// marked positions below its first position (word prefix + popcount).
__global__ void k_mark_first(const uint32_t* __restrict__ first, uint64_t span,
                             uint32_t* __restrict__ bits) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < span;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = first[k];
    if (f != 0xFFFFFFFFu) atomicOr(&bits[f >> 5], 1u << (f & 31));
  }
}

__global__ void k_store_count(const uint32_t* __restrict__ wpre_last,
                              const uint32_t* __restrict__ bits_last, uint32_t* __restrict__ out) {
  *out = *wpre_last + __popc(*bits_last);
}

struct Popc {
  __host__ __device__ uint32_t operator()(uint32_t x) const {
#ifdef __CUDA_ARCH__
    return __popc(x);
#else
    return static_cast<uint32_t>(__builtin_popcount(x));
#endif
  }
};

// ids[d] = id and first[id] := d (the dense-id map, in place: one thread per id)
__global__ void k_number_ids(uint32_t* __restrict__ first, uint64_t span,
                             const uint32_t* __restrict__ bits, const uint32_t* __restrict__ wpre,
                             uint64_t* __restrict__ ids) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < span;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = first[k];
    if (f == 0xFFFFFFFFu) continue;
    const uint32_t d = wpre[f >> 5] + __popc(bits[f >> 5] & ((1u << (f & 31)) - 1u));
    first[k] = d;
    ids[d] = k;
  }
}

template <typename K>
__global__ void k_dense_direct(const K* __restrict__ ks, uint64_t n,
                               const uint32_t* __restrict__ idmap, uint32_t* __restrict__ dense) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dense[i] = idmap[ks[i]];
}

// 1 in *flag if some v[i] < v[i-1]
__global__ void k_descent(const uint32_t* __restrict__ v, uint64_t n, unsigned* __restrict__ flag) {
  bool bad = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    bad |= v[i] < v[i - 1];
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}


// rs[l] = first position of left id l in the grouped (non-decreasing) id array; rs[L] = n
__global__ void k_row_starts(const uint32_t* __restrict__ l, uint64_t n, uint32_t L,
                             uint32_t* __restrict__ rs) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i == 0 || l[i] != l[i - 1]) rs[l[i]] = static_cast<uint32_t>(i);
    if (i == n - 1) rs[L] = static_cast<uint32_t>(n);
  }
}

// first occurrence of each (l, r) in canonical order
__global__ void k_dedup_flags(const uint32_t* __restrict__ l, const uint32_t* __restrict__ r,
                              uint64_t n, uint32_t* __restrict__ flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x)
    flag[k] = (k == 0 || l[k] != l[k - 1] || r[k] != r[k - 1]) ? 1u : 0u;
}

__global__ void k_widen_offsets(const uint32_t* __restrict__ in, uint64_t n,
                                uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// compact the unique pairs: lcan (left id of each canonical edge), ladj, loff
__global__ void k_left_csr(const uint32_t* __restrict__ l, const uint32_t* __restrict__ r,
                           const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                           uint64_t n, uint64_t m, uint32_t L, uint32_t* __restrict__ lcan,
                           uint32_t* __restrict__ ladj, uint64_t* __restrict__ loff) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    if (!flag[k]) continue;
    const uint64_t j = pos[k];
    lcan[j] = l[k];
    ladj[j] = r[k];
    if (k == 0 || l[k - 1] != l[k]) loff[l[k]] = j;
    if (j == m - 1) loff[L] = m;
  }
}

__global__ void k_right_offsets(const uint32_t* __restrict__ rks, uint64_t m, uint32_t R,
                                uint64_t* __restrict__ roff) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rks[j];
    if (j == 0 || rks[j - 1] != r) roff[r] = j;
    if (j == m - 1) roff[R] = m;
  }
}

// ---- statistics: per-block partial sums in 128 bits ---------------------------------
// q = 0: sum d^2 left, 1: sum d^2 right, 2: sum C(d,2) left, 3: sum C(d,2) right
struct StatPart {
  unsigned long long lo[4], hi[4];
  unsigned long long maxdeg, pad;
};

__global__ void k_stats(const uint64_t* __restrict__ loff, const uint64_t* __restrict__ roff,
                        uint32_t L, uint32_t R, StatPart* __restrict__ parts) {
  unsigned long long lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0}, mx = 0;
  uint64_t n = uint64_t{L} + R;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n;
       g += (uint64_t)gridDim.x * blockDim.x) {
    int side = g < L ? 0 : 1;
    uint64_t d = side == 0 ? loff[g + 1] - loff[g] : roff[g - L + 1] - roff[g - L];
    unsigned __int128 d2 = (unsigned __int128)d * d;
    unsigned long long x = (unsigned long long)d2, xh = (unsigned long long)(d2 >> 64);
    unsigned long long t = lo[side] + x;
    hi[side] += xh + (t < lo[side]);
    lo[side] = t;
    unsigned long long c2 = d < 2 ? 0ull : (d % 2 == 0 ? (d / 2) * (d - 1) : d * ((d - 1) / 2));
    t = lo[2 + side] + c2;
    hi[2 + side] += (t < lo[2 + side]);
    lo[2 + side] = t;
    if (d > mx) mx = d;
  }
  for (int off = 16; off > 0; off >>= 1) {
    for (int q = 0; q < 4; ++q) {
      unsigned long long olo = __shfl_down_sync(0xffffffffu, lo[q], off);
      unsigned long long ohi = __shfl_down_sync(0xffffffffu, hi[q], off);
      unsigned long long t = lo[q] + olo;
      hi[q] += ohi + (t < lo[q]);
      lo[q] = t;
    }
    unsigned long long om = __shfl_down_sync(0xffffffffu, mx, off);
    if (om > mx) mx = om;
  }
  __shared__ unsigned long long s[9][32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    for (int q = 0; q < 4; ++q) {
      s[q][wid] = lo[q];
      s[4 + q][wid] = hi[q];
    }
    s[8][wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    StatPart o{};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      for (int q = 0; q < 4; ++q) {
        unsigned long long t = o.lo[q] + s[q][w];
        o.hi[q] += s[4 + q][w] + (t < o.lo[q]);
        o.lo[q] = t;
      }
      if (s[8][w] > o.maxdeg) o.maxdeg = s[8][w];
    }
    parts[blockIdx.x] = o;
  }
}

// (known_max: the largest id when the caller already read it back, else null)
// The number of distinct ids goes to *d_count (device): callers read it together with their
// next read-back; ids is sized by a bound until then.
template <typename K>
void dense_ids(const K* d_keys, uint64_t n, cudaStream_t s, DBuf<uint32_t>& dense,
               DBuf<uint64_t>& ids, uint32_t* d_count, const K* known_max = nullptr) {
  K hmax = 0;
  if (known_max) {
    hmax = *known_max;
  } else {
    DBuf<K> dmax(1, s);
    reduce_max(d_keys, dmax.p, n, s);
    read_back(s, {{&hmax, dmax.p, sizeof(K)}});
  }
  const uint64_t span = static_cast<uint64_t>(hmax) + 1;
  if (span <= std::max<uint64_t>(uint64_t{1} << 26, 4 * n) && span < (uint64_t{1} << 32)) {
    // Direct-address path (ids are small integers): first position of each id by atomicMin
    // into an L2-resident table, then rank first positions with one scan.
    // first position per id, then the distinct ids sorted by it (a sort over the distinct
    // ids, not the n elements), then one gather per element
    DBuf<uint32_t> first(span, s);
    BFLY_CUDA(cudaMemsetAsync(first.p, 0xFF, span * 4, s));
    launch("build_first_pos", k_first_pos<K>, grid_for(n, 256), 256, 0, s, d_keys, n, first.p);
    const uint64_t nw = (n + 31) / 32;
    DBuf<uint32_t> bits(nw, s), wpre(nw + 1, s);
    bits.zero();
    launch("build_mark_first", k_mark_first, grid_for(span, 256), 256, 0, s, first.p, span, bits.p);
    {
      ProfScope ps("build_first_scan", s);
      thrust::transform_iterator<Popc, const uint32_t*, uint32_t> pc(bits.p, Popc{});
      size_t bytes = 0;
      BFLY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, pc, wpre.p, nw, s));
      DBuf<unsigned char> tmp(bytes ? bytes : 1, s);
      BFLY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, pc, wpre.p, nw, s));
    }
    launch("build_count_ids", k_store_count, 1, 1, 0, s, wpre.p + nw - 1, bits.p + nw - 1,
           d_count);
    dense.alloc(n, s);
    ids.alloc(std::max<uint64_t>(1, std::min<uint64_t>(span, n)), s);  // >= the distinct ids
    launch("build_number_ids", k_number_ids, grid_for(span, 256), 256, 0, s, first.p, span, bits.p,
           wpre.p, ids.p);
    launch("build_dense_direct", k_dense_direct<K>, grid_for(n, 256), 256, 0, s, d_keys, n,
           first.p, dense.p);
    return;
  }
  int kb = bits_for(static_cast<uint64_t>(hmax));
  DBuf<K> ks(n, s);
  DBuf<uint32_t> pos0(n, s), pos(n, s);
  launch("build_iota", k_iota, grid_for(n, 256), 256, 0, s, pos0.p, n);
  sort_pairs(d_keys, ks.p, pos0.p, pos.p, n, 0, kb, s, "sort_dense_ids");
  pos0.release();
  DBuf<uint32_t> headidx(n, s), firstflag(n, s), segstart(n, s), dense_of_pos(n, s);
  firstflag.zero();
  launch("build_heads", k_heads<K>, grid_for(n, 256), 256, 0, s, ks.p, pos.p, n, headidx.p,
         firstflag.p);
  inclusive_max(headidx.p, segstart.p, n, s);
  headidx.release();
  exclusive_sum(firstflag.p, dense_of_pos.p, n, s);
  uint32_t last[2] = {0, 0};
  read_back(s, {{&last[0], dense_of_pos.p + n - 1, 4}, {&last[1], firstflag.p + n - 1, 4}});
  const uint32_t count = last[0] + last[1];
  // (pageable source: the copy is staged before cudaMemcpyAsync returns)
  BFLY_CUDA(cudaMemcpyAsync(d_count, &count, 4, cudaMemcpyHostToDevice, s));
  dense.alloc(n, s);
  ids.alloc(count ? count : 1, s);
  launch("build_assign", k_assign<K>, grid_for(n, 256), 256, 0, s, ks.p, pos.p, segstart.p,
         dense_of_pos.p, n, dense.p, ids.p);
}

}  // namespace

// Grow the device's stream-ordered pool once to cover a whole build + count of this input
// size (about 96 B per input edge at peak; the all-subject LOCAL pass about 160 B), so later
// calls never map new physical memory
// in the middle of a step (that cost showed up as 0.5-1.2 s stalls); the pool keeps freed
// memory (release threshold = max; the engine's private pool, abi.cu: engine_pool).
static void reserve_pool(uint64_t m_in, cudaStream_t s) {
  static std::mutex mu;
  static uint64_t reserved[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t want = std::max<uint64_t>(1ull << 30, 160ull * m_in);
  std::lock_guard<std::mutex> lk(mu);
  if (reserved[dev & 63] >= want) return;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const uint64_t bytes = std::min<uint64_t>(want, free_b * 3 / 4);
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, bytes, engine_pool(), s) == cudaSuccess) {
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    reserved[dev & 63] = bytes;
  }
  cudaGetLastError();
}

template <typename K>
void build_graph(bfly_graph* g, const K* d_l, const K* d_r, uint64_t m_in,
                 cudaEvent_t right_ready) {
  cudaStream_t s = g->stream;
  if (m_in >= (1ull << 31))
    fail(kArgument, "edge list too long: at most 2^31-1 input edges per graph");
  reserve_pool(m_in, s);
  if (m_in == 0) {
    g->L = g->R = 0;
    g->m = 0;
    g->loff.alloc(1, s);
    g->roff.alloc(1, s);
    g->loff.zero();
    g->roff.zero();
    g->ladj.alloc(1, s);
    g->radj.alloc(1, s);
    g->reid.alloc(1, s);
    g->lids.alloc(1, s);
    g->rids.alloc(1, s);
    BFLY_CUDA(cudaStreamSynchronize(s));
    return;
  }
  DBuf<uint32_t> dl, dr;
  DBuf<uint32_t> dcount(2, s);  // distinct left / right ids, read with the order check below
  if (right_ready) {
    dense_ids<K>(d_l, m_in, s, dl, g->lids, dcount.p);
    // (host input: the right ids may still be in flight on the copy stream)
    BFLY_CUDA(cudaStreamWaitEvent(s, right_ready, 0));
    dense_ids<K>(d_r, m_in, s, dr, g->rids, dcount.p + 1);
  } else {  // both sides resident: one read-back for both id spans
    DBuf<K> dmax(2, s);
    reduce_max(d_l, dmax.p, m_in, s);
    reduce_max(d_r, dmax.p + 1, m_in, s);
    K hmax[2] = {0, 0};
    read_back(s, {{hmax, dmax.p, sizeof(hmax)}});
    dense_ids<K>(d_l, m_in, s, dl, g->lids, dcount.p, &hmax[0]);
    dense_ids<K>(d_r, m_in, s, dr, g->rids, dcount.p + 1, &hmax[1]);
  }
  // left ids already grouped (each left id's edges contiguous: first-seen ids non-decreasing)?
  // read together with the id counts
  uint32_t LR[2] = {0, 0};
  bool grouped;
  {
    DBuf<unsigned> f(1, s);
    f.zero();
    if (m_in > 1)
      launch("build_order_check", k_descent, grid_for(m_in, 256, 148u * 8u), 256, 0, s, dl.p, m_in,
             f.p);
    unsigned hf = 0;
    read_back(s, {{LR, dcount.p, sizeof(LR)}, {&hf, f.p, 4}});
    grouped = hf == 0;
  }
  const uint32_t L = LR[0], R = LR[1];
  g->L = L;
  g->R = R;
  int rb = bits_for(R > 0 ? R - 1 : 0), lb = bits_for(L > 0 ? L - 1 : 0);
  if (rb == 0) rb = 1;
  if (lb == 0) lb = 1;
  // canonical (l, r) order: edges grouped by left id (a stable sort by l, skipped when the
  // input already lists each left id's edges contiguously), then every left row sorted by
  // right id on its own (seg_sort_rows); duplicates end up adjacent
  DBuf<uint32_t> l2, r2;
  if (grouped) {
    l2 = std::move(dl);
    r2 = std::move(dr);
  } else {
    l2.alloc(m_in, s);
    r2.alloc(m_in, s);
    if (!sort_pairs_db(dl.p, l2.p, dr.p, r2.p, m_in, 0, lb, s, "sort_canonical_l")) {
      std::swap(l2, dl);
      std::swap(r2, dr);
    }
    dl.release();
    dr.release();
  }
  DBuf<uint32_t> rs(uint64_t{L} + 1, s);
  uint64_t m = 0;
  {
    DBuf<unsigned long long> dups(1, s);
    dups.zero();
    launch("build_row_starts", k_row_starts, grid_for(m_in, 256), 256, 0, s, l2.p, m_in, L, rs.p);
    seg_sort_rows(r2.p, rs.p, L, std::max(1, bits_for(R)), s, dups.p);  // 2^bits > every right id
    unsigned long long hd = 0;
    read_back(s, {{&hd, dups.p, 8}});
    m = m_in - hd;
  }
  trace_mark("build: ids+canonical sort");
  g->m = m;
  g->loff.alloc(uint64_t{L} + 1, s);
  if (m == m_in) {
    // no duplicate edges (the rows' sort counted none): the grouped, row-sorted arrays already
    // are the left CSR
    g->ladj = std::move(r2);
    g->lrow = std::move(l2);
    launch("build_left_offsets", k_widen_offsets, grid_for(uint64_t{L} + 1, 256), 256, 0, s,
           rs.p, uint64_t{L} + 1, g->loff.p);
  } else {
    DBuf<uint32_t> flag(m_in, s), pos(m_in, s);
    launch("build_dedup_flags", k_dedup_flags, grid_for(m_in, 256), 256, 0, s, l2.p, r2.p, m_in,
           flag.p);
    exclusive_sum(flag.p, pos.p, m_in, s);
    g->ladj.alloc(m, s);
    g->lrow.alloc(m, s);
    launch("build_left_csr", k_left_csr, grid_for(m_in, 256), 256, 0, s, l2.p, r2.p, flag.p,
           pos.p, m_in, m, L, g->lrow.p, g->ladj.p, g->loff.p);
  }
  rs.release();
  l2.release();
  r2.release();
  uint32_t* lcan = g->lrow.p;
  // right CSR: stable sort of the canonical edges by right id carrying their left id, so the
  // sorted payload is radj itself (right lists ascend in left id); the canonical edge ids of
  // the right entries (reid: per-edge counts, sparsification, export) come on first use
  g->rrow.alloc(m, s);
  uint32_t* rks = g->rrow.p;
  g->radj.alloc(m, s);
  sort_pairs(g->ladj.p, rks, lcan, g->radj.p, m, 0, rb, s, "sort_right_csr");  // ladj stays
  g->roff.alloc(uint64_t{R} + 1, s);
  launch("build_right_offsets", k_right_offsets, grid_for(m, 256), 256, 0, s, rks, m, R,
         g->roff.p);
  g->reid.release();
  g->reid_ready = false;
  trace_mark("build: right csr (queued)");  // stream-ordered: no host sync needed here
}

template void build_graph<uint32_t>(bfly_graph*, const uint32_t*, const uint32_t*, uint64_t,
                                    cudaEvent_t);
template void build_graph<uint64_t>(bfly_graph*, const uint64_t*, const uint64_t*, uint64_t,
                                    cudaEvent_t);

// reid: the same stable sort by right id, carrying the canonical edge id (the left CSR
// position) instead of the left id
void ensure_reid(bfly_graph* g) {
  if (g->reid_ready) return;
  cudaStream_t s = g->stream;
  const uint64_t m = g->m;
  g->reid.alloc(m ? m : 1, s);
  if (m) {
    const int rb = std::max(1, bits_for(g->R > 0 ? g->R - 1 : 0));
    DBuf<uint32_t> iota(m, s), kout(m, s);
    launch("build_iota", k_iota, grid_for(m, 256), 256, 0, s, iota.p, m);
    sort_pairs(g->ladj.p, kout.p, iota.p, g->reid.p, m, 0, rb, s, "sort_right_eid");
  }
  g->reid_ready = true;
}

void ensure_stats(bfly_graph* g) {
  if (g->stats_ready) return;
  cudaStream_t s = g->stream;
  bfly_stats st{};
  st.left = g->L;
  st.right = g->R;
  st.n = g->n();
  st.m = g->m;
  unsigned __int128 sq[2] = {0, 0}, wsd[2] = {0, 0};
  uint64_t mx = 0;
  if (g->n() > 0) {
    unsigned blocks = grid_for(g->n(), 256, 592);
    DBuf<StatPart> parts(blocks, s);
    launch("graph_stats", k_stats, blocks, 256, 0, s, g->loff.p, g->roff.p, g->L, g->R, parts.p);
    std::vector<StatPart> h(blocks);
    read_back(s, {{h.data(), parts.p, blocks * sizeof(StatPart)}});
    for (auto& p : h) {
      for (int q = 0; q < 2; ++q) {
        sq[q] += ((unsigned __int128)p.hi[q] << 64) | p.lo[q];
        wsd[q] += ((unsigned __int128)p.hi[2 + q] << 64) | p.lo[2 + q];
      }
      if (p.maxdeg > mx) mx = p.maxdeg;
    }
  }
  unsigned __int128 wed = wsd[0] + wsd[1];
  g->wedges_side[0] = wsd[0];
  g->wedges_side[1] = wsd[1];
  // The reference sums d*d in double, sequentially (graph.cpp:142-152, exact.cpp:11-18).
  // While the exact integer total is below 2^53 every partial sum is exact, so the double
  // equals the integer. Above that, replay the sequential double sum on the host.
  double cost[2];
  for (int q = 0; q < 2; ++q) {
    if (sq[q] < ((unsigned __int128)1 << 53)) {
      cost[q] = static_cast<double>(static_cast<uint64_t>(sq[q]));
    } else {
      uint32_t cnt = q == 0 ? g->L : g->R;
      std::vector<uint64_t> off(uint64_t{cnt} + 1);
      read_back(s, {{off.data(), q == 0 ? g->loff.p : g->roff.p, off.size() * 8}});
      double acc = 0.0;
      for (uint32_t i = 0; i < cnt; ++i) {
        double d = static_cast<double>(off[i + 1] - off[i]);
        acc += d * d;
      }
      cost[q] = acc;
    }
  }
  st.sum_deg_sq_left = cost[0];
  st.sum_deg_sq_right = cost[1];
  st.max_degree = static_cast<uint32_t>(mx);
  g->stats_status = (wed >> 64) ? kOverflow : kOk;
  st.wedge_count = static_cast<uint64_t>(wed);
  g->stats = st;
  g->cost_left = cost[0];
  g->cost_right = cost[1];
  g->stats_ready = true;
}

}  // namespace bflyd
