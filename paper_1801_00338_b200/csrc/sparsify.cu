// sparsify.cu -- sparsify-then-count (replaces count_retained + exact_count,
// sparsify.cpp:15-71).
//
// The keep predicate is evaluated per canonical edge inside the compaction kernels:
//   ESpar  keep k  iff  unit_double(derive_seed(seed, k)) < p           (sparsify.cpp:60-61)
//   CSpar  keep (l,r) iff colour(l) == colour(L + r),
//          colour(g) = bounded_from_bits(derive_seed(seed, g), N)       (sparsify.cpp:65-70)
//
// The reference rebuilds the retained sub-graph through from_edges, which renumbers the
// vertices that keep an edge (sparsify.cpp:15-24), and counts it. Butterfly counts are
// invariant under relabelling, and a vertex with one retained edge lies on no butterfly, so
// its edge can be dropped without changing the count. The pipeline:
//
//   1. keep bits over the left CSR (canonical order): a warp evaluates 1024 consecutive
//      edges, 32 per ballot, and writes the bitmap with coalesced 32-bit stores (ESpar reads
//      nothing: the key is the edge index; CSpar reads the row and column of each edge and
//      two entries of a per-vertex colour table computed once per call) + tile popcounts.
//   2. one-CTA scan of the tile counts; every tile emits its kept edges (left, right) at its
//      offset -- the retained list in canonical order, m' = its length (the `kept` result).
//   3. peeling rounds: drop edges with an endpoint of retained degree 1 (left degrees are run
//      lengths of the sorted list; right degrees ">= 2" by two atomicOr bitmaps), until a
//      round removes under 2% -- the count is unchanged, the graph shrinks by 10-100x at the
//      BASELINE keep rates.
//   4. live vertices = endpoints of the remaining edges, as bitmaps over L and R; a popcount
//      prefix per bitmap word gives each its new dense id with two cached reads.
//   5. left CSR straight from the sorted list; right CSR by a counting-scatter transpose
//      (rows unsorted: the priority build sorts every row itself); the exact kernels count it.
//
// Traffic per input edge: ESpar 1 bit written (hashing is ALU work), CSpar 8 B read + 1 bit;
// everything after step 1 is O(m') -- no pass over the right CSR, no reid.
#include <cmath>

#include "local.cuh"
#include "scan.cuh"

namespace bflyd {
namespace {

constexpr int kTileThreads = 256;                // 8 warps
constexpr int kTileEntries = kTileThreads * 32;  // 8192 edges = 256 bitmap words per tile

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ bool bit(const uint32_t* __restrict__ bm, uint32_t x) {
  return (__ldg(bm + (x >> 5)) >> (x & 31)) & 1u;
}

// ---- keep predicates over canonical edge index e ------------------------------------------
struct HashKeep {  // ESpar (sparsify.cpp:60-61)
  uint64_t ms, thr;
  __device__ __forceinline__ bool operator()(uint64_t e) const {
    return (mix64(ms ^ mix64(e)) >> 11) < thr;
  }
};
struct MaskKeep {  // caller's keep byte per canonical edge (edge_sparsify_value)
  const uint8_t* keep;
  __device__ __forceinline__ bool operator()(uint64_t e) const { return keep[e] != 0; }
};
template <typename C>
struct ColourKeep {  // CSpar / caller colours: colour(l) == colour(L + r)
  const C* col;
  const uint32_t* lrow;
  const uint32_t* ladj;
  uint32_t L;
  __device__ __forceinline__ bool operator()(uint64_t e) const {
    return col[__ldcs(lrow + e)] == col[uint64_t{L} + __ldcs(ladj + e)];
  }
};

// colour(g) = bounded_from_bits(derive_seed(seed, g), N), once per vertex and call
template <typename C>
__global__ void k_colours(uint64_t ms, uint64_t n_colors, uint64_t n, C* __restrict__ col) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n;
       g += (uint64_t)gridDim.x * blockDim.x)
    col[g] = static_cast<C>(__umul64hi(mix64(ms ^ mix64(g)), n_colors));
}

// Keep bitmap + per-tile kept count. Word q of tile t covers edges t*8192 + q*32 + [0, 32).
template <typename P>
__global__ void __launch_bounds__(kTileThreads)
    k_keep_bits(P pred, uint64_t m, uint32_t* __restrict__ bits, uint32_t* __restrict__ tile_cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = uint64_t{blockIdx.x} * kTileEntries + static_cast<uint64_t>(warp) * 1024;
  uint32_t mine = 0;
#pragma unroll 4
  for (int i = 0; i < 32; ++i) {
    const uint64_t e = base + i * 32 + lane;
    const uint32_t w = __ballot_sync(0xffffffffu, e < m && pred(e));
    if (lane == i) mine = w;
  }
  const uint64_t wi = uint64_t{blockIdx.x} * kTileThreads + threadIdx.x;
  if (wi * 32 < m) bits[wi] = mine;
  uint32_t c = __popc(mine);
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ uint32_t s[kTileThreads / 32];
  if (lane == 0) s[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int q = 0; q < kTileThreads / 32; ++q) t += s[q];
    tile_cnt[blockIdx.x] = t;
  }
}

// Emit the kept edges of every tile in canonical order: kl[pos] = left, kr[pos] = right.
__global__ void __launch_bounds__(kTileThreads)
    k_emit(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ tile_off,
           const uint32_t* __restrict__ lrow, const uint32_t* __restrict__ ladj, uint64_t m,
           uint32_t* __restrict__ kl, uint32_t* __restrict__ kr) {
  using BS = cub::BlockScan<uint32_t, kTileThreads>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t wi = uint64_t{blockIdx.x} * kTileThreads + threadIdx.x;
  uint32_t w = wi * 32 < m ? bits[wi] : 0u;
  uint32_t pre;
  BS(tmp).ExclusiveSum(static_cast<uint32_t>(__popc(w)), pre);
  uint32_t pos = tile_off[blockIdx.x] + pre;
  while (w) {
    const int b = __ffs(w) - 1;
    w &= w - 1;
    const uint64_t e = wi * 32 + b;
    kl[pos] = lrow[e];
    kr[pos] = ladj[e];
    ++pos;
  }
}

// Degree >= 2 bitmaps of the retained list (sorted by left): a left vertex repeats in the
// previous entry; a right vertex is seen twice when its `once` bit was already set.
__global__ void k_degree2(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ kr,
                          uint32_t c, uint32_t* __restrict__ twice_l, uint32_t* __restrict__ once_r,
                          uint32_t* __restrict__ twice_r) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const uint32_t l = kl[i], r = kr[i];
    // second entry of a left run: one atomic per row
    if (i > 0 && kl[i - 1] == l && (i == 1 || kl[i - 2] != l))
      atomicOr(twice_l + (l >> 5), 1u << (l & 31));
    // right hubs recur across the whole list: read before the atomics, so a vertex already
    // seen twice costs one cached load instead of two serialised atomics on one word
    const uint32_t b = 1u << (r & 31);
    if (__ldcg(twice_r + (r >> 5)) & b) continue;
    if (__ldcg(once_r + (r >> 5)) & b) atomicOr(twice_r + (r >> 5), b);
    else if (atomicOr(once_r + (r >> 5), b) & b) atomicOr(twice_r + (r >> 5), b);
  }
}

struct Deg2Pred {
  const uint32_t* twice_l;
  const uint32_t* twice_r;
  __device__ __forceinline__ bool operator()(uint64_t, uint32_t l, uint32_t r) const {
    return bit(twice_l, l) && bit(twice_r, r);
  }
};

// Live bitmaps: every endpoint of the remaining edges.
__global__ void k_mark_live(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ kr,
                            uint32_t c, uint32_t* __restrict__ live_l, uint32_t* __restrict__ live_r) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const uint32_t l = kl[i], r = kr[i];
    if (i == 0 || kl[i - 1] != l) atomicOr(live_l + (l >> 5), 1u << (l & 31));
    const uint32_t b = 1u << (r & 31);
    if (!(__ldcg(live_r + (r >> 5)) & b)) atomicOr(live_r + (r >> 5), b);
  }
}

// Rank support over a bitmap of nw words: tiles of 256 words; pass 1 tile popcounts.
__global__ void __launch_bounds__(256) k_bm_tiles(const uint32_t* __restrict__ bm, uint64_t nw,
                                                  uint32_t* __restrict__ tcnt) {
  const uint64_t wi = uint64_t{blockIdx.x} * 256 + threadIdx.x;
  uint32_t c = wi < nw ? __popc(bm[wi]) : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ uint32_t s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int q = 0; q < 8; ++q) t += s[q];
    tcnt[blockIdx.x] = t;
  }
}

// pass 3: wpre[w] = number of set bits before word w
__global__ void __launch_bounds__(256) k_bm_prefix(const uint32_t* __restrict__ bm, uint64_t nw,
                                                   const uint32_t* __restrict__ toff,
                                                   uint32_t* __restrict__ wpre) {
  using BS = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t wi = uint64_t{blockIdx.x} * 256 + threadIdx.x;
  const uint32_t c = wi < nw ? __popc(bm[wi]) : 0u;
  uint32_t pre;
  BS(tmp).ExclusiveSum(c, pre);
  if (wi < nw) wpre[wi] = toff[blockIdx.x] + pre;
}

__device__ __forceinline__ uint32_t rank_of(const uint32_t* __restrict__ bm,
                                            const uint32_t* __restrict__ wpre, uint32_t x) {
  return __ldg(wpre + (x >> 5)) + __popc(__ldg(bm + (x >> 5)) & ((1u << (x & 31)) - 1u));
}

// Left CSR in new ids (list sorted by left): off'[rank(l)] = i at run heads, adj'[i] =
// rank(r); right degrees counted for the transpose.
__global__ void k_fill_left(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ kr,
                            uint32_t c, const uint32_t* __restrict__ lbm,
                            const uint32_t* __restrict__ lpre, const uint32_t* __restrict__ rbm,
                            const uint32_t* __restrict__ rpre, uint32_t rows,
                            uint64_t* __restrict__ off, uint32_t* __restrict__ adj,
                            uint32_t* __restrict__ rdeg) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const uint32_t l = kl[i];
    if (i == 0 || kl[i - 1] != l) off[rank_of(lbm, lpre, l)] = i;
    const uint32_t r = rank_of(rbm, rpre, kr[i]);
    adj[i] = r;
    // right hubs recur within a warp's rows: one atomic per distinct vertex per warp
    const unsigned act = __activemask();
    const unsigned same = __match_any_sync(act, r);
    if ((__ffs(same) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(rdeg + r, __popc(same));
    if (i == 0) off[rows] = c;
  }
}

// Right CSR by counting scatter: entry of edge i at roff[r'] + (arrival order in row r').
__global__ void k_scatter_right(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ ladj2,
                                uint32_t c, const uint32_t* __restrict__ lbm,
                                const uint32_t* __restrict__ lpre,
                                const uint64_t* __restrict__ roff, uint32_t* __restrict__ cur,
                                uint32_t* __restrict__ radj) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const uint32_t r = ladj2[i];
    const unsigned act = __activemask();
    const unsigned same = __match_any_sync(act, r);
    const int lead = __ffs(same) - 1, lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lead == lane) base = atomicAdd(cur + r, __popc(same));
    base = __shfl_sync(same, base, lead);
    radj[roff[r] + base + __popc(same & ((1u << lane) - 1u))] = rank_of(lbm, lpre, kl[i]);
  }
}

// row of every CSR entry (fallback for handles without the build's lrow): warp per row
__global__ void k_row_of(const uint64_t* __restrict__ off, uint32_t rows, uint32_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5)
    for (uint64_t e = off[r] + lane; e < off[r + 1]; e += 32) out[e] = static_cast<uint32_t>(r);
}

// ---- statistics of the retained graph G' (bench roofline; off by default) -----------------
__global__ void k_spar_degrees(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ kr,
                               uint32_t c, uint32_t L, uint32_t* __restrict__ deg) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const unsigned act = __activemask();
    const uint32_t l = kl[i];
    const unsigned sl = __match_any_sync(act, l);
    if ((__ffs(sl) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(deg + l, __popc(sl));
    const uint32_t r = L + kr[i];
    const unsigned sr = __match_any_sync(act, r);
    if ((__ffs(sr) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(deg + r, __popc(sr));
  }
}

// out: [0/1] sum d^2 left / right, [2/3] sum C(d,2) left / right, [4] vertices with d > 0
__global__ void k_spar_degsums(const uint32_t* __restrict__ deg, uint64_t n, uint32_t L,
                               unsigned long long* __restrict__ out) {
  unsigned long long a[5] = {0, 0, 0, 0, 0};
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = deg[g];
    const int sd = g < L ? 0 : 1;
    a[sd] += d * d;
    a[2 + sd] += d * (d - (d > 0)) / 2;
    a[4] += d > 0;
  }
  for (int q = 0; q < 5; ++q) {
    unsigned long long v = a[q];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + q, v);
  }
}

void retained_stats(bfly_graph* g, const uint32_t* kl, const uint32_t* kr, uint32_t mk,
                    cudaStream_t s) {
  const uint64_t n = g->n();
  DBuf<uint32_t> deg(n, s);
  deg.zero();
  DBuf<unsigned long long> sums(5, s);
  sums.zero();
  launch("spar_stats", k_spar_degrees, grid_for(mk, 256), 256, 0, s, kl, kr, mk, g->L, deg.p);
  launch("spar_stats", k_spar_degsums, grid_for(n, 256, 592), 256, 0, s, deg.p, n, g->L, sums.p);
  unsigned long long h[5] = {0, 0, 0, 0, 0};
  read_back(s, {{h, sums.p, sizeof(h)}});
  // exact.cpp:9-21 on G': anchors Right iff cost_left < cost_right; W_C = centre-side wedges
  // (the sums of squares are exact integers here, so the double comparison is the same)
  const bool anchor_right = h[0] < h[1];
  g->spar_stats[4] = anchor_right ? h[2] : h[3];
  g->spar_stats[5] = h[4];
}

// rank support of a bitmap of `nbits` bits; toff[tiles] = total
void bitmap_rank(const uint32_t* bm, uint64_t nbits, DBuf<uint32_t>& wpre, DBuf<uint32_t>& toff,
                 cudaStream_t s) {
  const uint64_t nw = (nbits + 31) / 32;
  const unsigned tiles = static_cast<unsigned>((nw + 255) / 256);
  wpre.alloc(nw ? nw : 1, s);
  toff.alloc(uint64_t{tiles} + 1, s);
  if (!tiles) {
    BFLY_CUDA(cudaMemsetAsync(toff.p, 0, 4, s));
    return;
  }
  DBuf<uint32_t> tcnt(tiles, s);
  launch("spar_rank", k_bm_tiles, tiles, 256, 0, s, bm, nw, tcnt.p);
  launch("spar_rank", scan::k_scan_tiles<uint32_t>, 1, 1024, 0, s, tcnt.p, tiles, toff.p);
  launch("spar_rank", k_bm_prefix, tiles, 256, 0, s, bm, nw, toff.p, wpre.p);
}

template <typename P>
void keep_bits(P pred, uint64_t m, uint32_t* bits, uint32_t* tcnt, unsigned tiles, cudaStream_t s) {
  launch("spar_keep", k_keep_bits<P>, tiles, kTileThreads, 0, s, pred, m, bits, tcnt);
}

template <typename C>
void colour_bits(uint64_t ms, uint64_t n_colors, const uint32_t* hcol, const bfly_graph* g,
                 const uint32_t* lrow, uint32_t* bits, uint32_t* tcnt, unsigned tiles,
                 cudaStream_t s) {
  DBuf<C> col;
  const C* table = reinterpret_cast<const C*>(hcol);
  if (!hcol) {
    col.alloc(g->n(), s);
    launch("spar_colours", k_colours<C>, grid_for(g->n(), 256), 256, 0, s, ms, n_colors, g->n(),
           col.p);
    table = col.p;
  }
  keep_bits(ColourKeep<C>{table, lrow, g->ladj.p, g->L}, g->m, bits, tcnt, tiles, s);
}

}  // namespace

void sparsify_count(bfly_graph* g, int mode, double p, uint64_t n_colors, uint64_t seed,
                    const uint8_t* h_keep, const uint32_t* h_colors, uint64_t* count,
                    uint64_t* kept) {
  cudaStream_t s = g->stream;
  const uint64_t m = g->m, n = g->n();
  *count = 0;
  *kept = 0;
  g->last_wedges = 0;
  for (int q = 0; q < 6; ++q) g->bucket_starts[q] = g->bucket_wedges[q] = g->bucket_entries[q] = 0;
  for (int q = 0; q < 6; ++q) g->spar_stats[q] = 0;
  if (m == 0) return;
  uint64_t ms;
  {  // mix64(seed) is hoisted: derive_seed(seed, i) = mix64(mix64(seed) ^ mix64(i))
    uint64_t x = seed + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    ms = x ^ (x >> 31);
  }
  // left row of every canonical edge (kept from the build)
  DBuf<uint32_t> lrow_tmp;
  const uint32_t* lrow = g->lrow.p;
  if (!lrow) {
    lrow_tmp.alloc(m, s);
    launch("spar_row_of", k_row_of, grid_for(uint64_t{g->L} * 32, 256), 256, 0, s, g->loff.p,
           g->L, lrow_tmp.p);
    lrow = lrow_tmp.p;
  }
  const unsigned tiles = static_cast<unsigned>((m + kTileEntries - 1) / kTileEntries);
  DBuf<uint32_t> bits((m + 31) / 32, s), tcnt(tiles, s), toff(uint64_t{tiles} + 1, s);
  if (mode == 0) {
    // unit_double(h) = (h >> 11) * 2^-53 is exact, so unit_double(h) < p <=> (h >> 11) < p*2^53
    // (exact: a power-of-two scaling) <=> (h >> 11) < ceil(p * 2^53) for the integer h >> 11
    keep_bits(HashKeep{ms, static_cast<uint64_t>(std::ceil(p * 0x1.0p53))}, m, bits.p, tcnt.p,
              tiles, s);
  } else if (mode == 2) {
    DBuf<uint8_t> dkeep(m, s);
    BFLY_CUDA(cudaMemcpyAsync(dkeep.p, h_keep, m, cudaMemcpyHostToDevice, s));
    keep_bits(MaskKeep{dkeep.p}, m, bits.p, tcnt.p, tiles, s);
  } else if (mode == 3) {
    DBuf<uint32_t> dcol(n, s);
    BFLY_CUDA(cudaMemcpyAsync(dcol.p, h_colors, n * 4, cudaMemcpyHostToDevice, s));
    colour_bits<uint32_t>(ms, 0, dcol.p, g, lrow, bits.p, tcnt.p, tiles, s);
  } else if (n_colors <= 256) {
    colour_bits<uint8_t>(ms, n_colors, nullptr, g, lrow, bits.p, tcnt.p, tiles, s);
  } else if (n_colors <= 65536) {
    colour_bits<uint16_t>(ms, n_colors, nullptr, g, lrow, bits.p, tcnt.p, tiles, s);
  } else {
    colour_bits<uint32_t>(ms, n_colors, nullptr, g, lrow, bits.p, tcnt.p, tiles, s);
  }
  launch("spar_scan", scan::k_scan_tiles<uint32_t>, 1, 1024, 0, s, tcnt.p, tiles, toff.p);
  uint32_t mk = 0;
  read_back(s, {{&mk, toff.p + tiles, 4}});
  *kept = mk;
  g->spar_stats[0] = mk;
  if (mk == 0) return;  // sparsify.cpp:22: nothing retained -> 0

  // the retained edges (left, right) in canonical order, old dense ids
  DBuf<uint32_t> kl(mk, s), kr(mk, s);
  launch("spar_emit", k_emit, tiles, kTileThreads, 0, s, bits.p, toff.p, lrow, g->ladj.p, m,
         kl.p, kr.p);
  bits.release();
  lrow_tmp.release();
  if (g->spar_stats_on) retained_stats(g, kl.p, kr.p, mk, s);

  const uint64_t lw = (uint64_t{g->L} + 31) / 32, rw = (uint64_t{g->R} + 31) / 32;
  // peel retained-degree-1 endpoints (their edges lie on no butterfly)
  uint32_t c = mk;
  {
    DBuf<uint32_t> bm(lw + 2 * rw, s), kl2(mk, s), kr2(mk, s);
    for (int round = 0; round < 8 && c; ++round) {
      bm.zero();
      launch("spar_peel", k_degree2, grid_for(c, 256), 256, 0, s, kl.p, kr.p, c, bm.p,
             bm.p + lw, bm.p + lw + rw);
      const uint32_t c2 = scan::compact_pairs(kl.p, kr.p, c, Deg2Pred{bm.p, bm.p + lw + rw},
                                              kl2.p, kr2.p, s, "spar_peel");
      std::swap(kl.p, kl2.p);
      std::swap(kr.p, kr2.p);
      const bool small_step = uint64_t{c - c2} * 50 < c;  // < 2% removed: stop
      c = c2;
      if (small_step) break;
    }
  }
  g->spar_stats[1] = c;
  if (c == 0) return;  // no vertex pair with two common neighbours: no butterfly

  // live vertices of each side and their new ids
  DBuf<uint32_t> live(lw + rw, s);
  live.zero();
  uint32_t* livel = live.p;
  uint32_t* liver = live.p + lw;
  launch("spar_live", k_mark_live, grid_for(c, 256), 256, 0, s, kl.p, kr.p, c, livel, liver);
  DBuf<uint32_t> lpre, lto, rpre, rto;
  bitmap_rank(livel, g->L, lpre, lto, s);
  bitmap_rank(liver, g->R, rpre, rto, s);
  uint32_t sizes[2] = {0, 0};
  read_back(s, {{&sizes[0], lto.p + (lto.n - 1), 4}, {&sizes[1], rto.p + (rto.n - 1), 4}});

  g->spar_stats[2] = sizes[0];
  g->spar_stats[3] = sizes[1];
  bfly_graph sub;
  sub.device = g->device;
  sub.stream = s;
  sub.L = sizes[0];
  sub.R = sizes[1];
  sub.m = c;
  sub.reid_ready = false;
  sub.loff.alloc(uint64_t{sub.L} + 1, s);
  sub.roff.alloc(uint64_t{sub.R} + 1, s);
  sub.ladj.alloc(c, s);
  sub.radj.alloc(c, s);
  DBuf<uint32_t> rdeg(uint64_t{sub.R} + 1, s);
  rdeg.zero();
  launch("spar_fill", k_fill_left, grid_for(c, 256), 256, 0, s, kl.p, kr.p, c, livel, lpre.p,
         liver, rpre.p, sub.L, sub.loff.p, sub.ladj.p, rdeg.p);
  scan::exclusive_sum<uint64_t>(rdeg.p, sub.R, sub.roff.p, s, "spar_fill");
  rdeg.zero();
  launch("spar_fill", k_scatter_right, grid_for(c, 256), 256, 0, s, kl.p, sub.ladj.p, c, livel,
         lpre.p, sub.roff.p, rdeg.p, sub.radj.p);
  kl.release();
  kr.release();
  *count = exact_count_device(&sub);
  g->last_wedges = sub.last_wedges;
  for (int q = 0; q < 6; ++q) {
    g->bucket_starts[q] = sub.bucket_starts[q];
    g->bucket_wedges[q] = sub.bucket_wedges[q];
    g->bucket_entries[q] = sub.bucket_entries[q];
  }
  BFLY_CUDA(cudaStreamSynchronize(s));
}

}  // namespace bflyd
