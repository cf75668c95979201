// sparsify.cu -- sparsify-then-count (replaces count_retained + exact_count,
// sparsify.cpp:15-71).
//
// The keep predicate is evaluated per canonical edge inside the compaction kernels:
//   ESpar  keep k  iff  unit_double(derive_seed(seed, k)) < p           (sparsify.cpp:60-61)
//   CSpar  keep (l,r) iff colour(l) == colour(L + r),
//          colour(g) = bounded_from_bits(derive_seed(seed, g), N)       (sparsify.cpp:65-70)
//
// The reference rebuilds the retained sub-graph through from_edges, which renumbers the
// vertices that keep an edge (sparsify.cpp:15-24). Here the sub-graph is compacted straight
// out of the two resident CSR directions, with the same renumbering (butterfly counts are
// invariant under it; only the order of the ids differs from first-seen order):
//
//   1. keep bits, one bit per entry, for the left CSR (canonical order) and the right CSR:
//      a warp evaluates 1024 consecutive entries, 32 per ballot, so the bitmaps are written
//      with coalesced 32-bit stores and never exist as byte or word flags. ESpar's left pass
//      reads nothing (the key is the entry index); its right pass reads reid and tests the
//      left bitmap (37.5 MB at 300M edges: L2-resident). CSpar evaluates the colours of both
//      endpoints from the entry and its row.
//   2. per-tile popcounts -> one-CTA scan -> every tile emits its kept entries (row, column)
//      at its offset: the kept lists come out in CSR order of each direction.
//   3. live vertices = rows with a kept entry (run heads of the sorted kept lists) as
//      bitmaps over L and R; a popcount prefix per bitmap word gives every live vertex its
//      new dense id (rank) with two cached reads.
//   4. the sub-graph's CSRs are written with the new ids; the exact pipeline counts it.
//
// Traffic per input edge: ESpar 4 B (reid) + 2 bits, CSpar 16 B (rows + columns of both
// directions) + 2 bits; plus O(m') for the kept entries -- instead of the u32 flags, u64
// scans and full-width compactions over all L + R ids of a plain compaction.
#include <cmath>

#include <cub/block/block_scan.cuh>

#include "local.cuh"

namespace bflyd {
namespace {

constexpr int kTileThreads = 256;                // 8 warps
constexpr int kTileEntries = kTileThreads * 32;  // 8192 entries = 256 bitmap words per tile

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint32_t colour(uint64_t ms, uint64_t g, uint64_t n_colors) {
  return static_cast<uint32_t>(__umul64hi(mix64(ms ^ mix64(g)), n_colors));
}

struct KeepArgs {
  uint64_t ms;         // mix64(seed), hoisted out of derive_seed(seed, i)
  uint64_t thr;        // ESpar: keep iff (h >> 11) < thr  (== unit_double(h) < p)
  uint64_t n_colors;   // CSpar
  uint32_t L;
  const uint8_t* hkeep;   // mode 2: caller's keep byte per canonical edge
  const uint32_t* hcol;   // mode 3: caller's colour per global vertex
  const uint32_t* lbits;  // right pass of modes 0/2: the left keep bitmap
};

// MODE 0 ESpar, 1 CSpar, 2 keep mask, 3 colour mask. RIGHT: entry j of the right CSR
// (row = right id, col = left id, key = reid[j]); else entry k of the left CSR (row = left
// id, col = right id, key = k).
template <int MODE, bool RIGHT>
__device__ __forceinline__ bool keep_entry(const KeepArgs& a, uint64_t idx, uint32_t row,
                                           uint32_t col, uint32_t key) {
  if (MODE == 0 || MODE == 2) {
    if (RIGHT) return (a.lbits[key >> 5] >> (key & 31)) & 1u;
    if (MODE == 2) return a.hkeep[idx] != 0;
    return (mix64(a.ms ^ mix64(idx)) >> 11) < a.thr;
  }
  const uint64_t gl = RIGHT ? col : row;
  const uint64_t gr = uint64_t{a.L} + (RIGHT ? row : col);
  if (MODE == 1) return colour(a.ms, gl, a.n_colors) == colour(a.ms, gr, a.n_colors);
  return a.hcol[gl] == a.hcol[gr];
}

// Keep bitmap + per-tile kept count. Word q of tile t covers entries t*8192 + q*32 + [0, 32).
template <int MODE, bool RIGHT>
__global__ void __launch_bounds__(kTileThreads)
    k_keep_bits(KeepArgs a, const uint32_t* __restrict__ rowof, const uint32_t* __restrict__ adj,
                const uint32_t* __restrict__ key, uint64_t m, uint32_t* __restrict__ bits,
                uint32_t* __restrict__ tile_cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = uint64_t{blockIdx.x} * kTileEntries + static_cast<uint64_t>(warp) * 1024;
  uint32_t mine = 0;
#pragma unroll 4
  for (int i = 0; i < 32; ++i) {
    const uint64_t e = base + i * 32 + lane;
    bool keep = false;
    if (e < m) {
      const bool need_rc = MODE == 1 || MODE == 3;
      const uint32_t row = need_rc ? __ldcs(rowof + e) : 0u;
      const uint32_t col = need_rc ? __ldcs(adj + e) : 0u;
      const uint32_t k = (RIGHT && !need_rc) ? __ldcs(key + e) : 0u;
      keep = keep_entry<MODE, RIGHT>(a, e, row, col, k);
    }
    const uint32_t w = __ballot_sync(0xffffffffu, keep);
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

// Exclusive scan of n u32 counts in one CTA (n <= 2^18: tiles of 8192 entries, m < 2^31);
// out[n] = total.
__global__ void __launch_bounds__(1024) k_scan_one_cta(const uint32_t* __restrict__ in, uint32_t n,
                                                       uint32_t* __restrict__ out) {
  using BS = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(n, b + per);
  uint32_t s = 0;
  for (uint32_t i = b; i < e; ++i) s += in[i];
  uint32_t pre, total;
  BS(tmp).ExclusiveSum(s, pre, total);
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t v = in[i];
    out[i] = pre;
    pre += v;
  }
  if (threadIdx.x == 0) out[n] = total;
}

// Emit the kept entries of every tile in CSR order: kr[pos] = row, kc[pos] = column.
__global__ void __launch_bounds__(kTileThreads)
    k_emit(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ tile_off,
           const uint32_t* __restrict__ rowof, const uint32_t* __restrict__ adj, uint64_t m,
           uint32_t* __restrict__ kr, uint32_t* __restrict__ kc) {
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
    kr[pos] = rowof[e];
    kc[pos] = adj[e];
    ++pos;
  }
}

// Live-row bitmap: one bit per row that heads a run of the sorted kept rows.
__global__ void k_mark_live(const uint32_t* __restrict__ kr, uint32_t mk, uint32_t* __restrict__ live) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mk; i += gridDim.x * blockDim.x) {
    const uint32_t r = kr[i];
    if (i == 0 || kr[i - 1] != r) atomicOr(live + (r >> 5), 1u << (r & 31));
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

// Sub-graph CSR in new ids: off'[rank(row)] = i at run heads, adj'[i] = rank(column).
__global__ void k_fill(const uint32_t* __restrict__ kr, const uint32_t* __restrict__ kc, uint32_t mk,
                       const uint32_t* __restrict__ rbm, const uint32_t* __restrict__ rpre,
                       const uint32_t* __restrict__ cbm, const uint32_t* __restrict__ cpre,
                       uint32_t rows, uint64_t* __restrict__ off, uint32_t* __restrict__ adj) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mk; i += gridDim.x * blockDim.x) {
    const uint32_t r = kr[i];
    if (i == 0 || kr[i - 1] != r) off[rank_of(rbm, rpre, r)] = i;
    adj[i] = rank_of(cbm, cpre, kc[i]);
    if (i == 0) off[rows] = mk;
  }
}

// row of every CSR entry (fallback for handles without the build's lrow / rrow): warp per row
__global__ void k_row_of(const uint64_t* __restrict__ off, uint32_t rows, uint32_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5)
    for (uint64_t e = off[r] + lane; e < off[r + 1]; e += 32) out[e] = static_cast<uint32_t>(r);
}

template <bool RIGHT>
void launch_keep(int mode, const KeepArgs& a, const uint32_t* rowof, const uint32_t* adj,
                 const uint32_t* key, uint64_t m, uint32_t* bits, uint32_t* tcnt, unsigned tiles,
                 cudaStream_t s) {
  const char* nm = RIGHT ? "spar_keep_right" : "spar_keep_left";
  switch (mode) {
    case 0: launch(nm, k_keep_bits<0, RIGHT>, tiles, kTileThreads, 0, s, a, rowof, adj, key, m, bits, tcnt); break;
    case 1: launch(nm, k_keep_bits<1, RIGHT>, tiles, kTileThreads, 0, s, a, rowof, adj, key, m, bits, tcnt); break;
    case 2: launch(nm, k_keep_bits<2, RIGHT>, tiles, kTileThreads, 0, s, a, rowof, adj, key, m, bits, tcnt); break;
    default: launch(nm, k_keep_bits<3, RIGHT>, tiles, kTileThreads, 0, s, a, rowof, adj, key, m, bits, tcnt); break;
  }
}

// rank support of a bitmap of `bitsn` bits; returns the device total in *d_total (u32)
void bitmap_rank(const uint32_t* bm, uint64_t bitsn, DBuf<uint32_t>& wpre, DBuf<uint32_t>& tcnt,
                 DBuf<uint32_t>& toff, cudaStream_t s) {
  const uint64_t nw = (bitsn + 31) / 32;
  const unsigned tiles = static_cast<unsigned>((nw + 255) / 256);
  wpre.alloc(nw ? nw : 1, s);
  tcnt.alloc(tiles ? tiles : 1, s);
  toff.alloc(uint64_t{tiles} + 1, s);
  if (!tiles) {
    BFLY_CUDA(cudaMemsetAsync(toff.p, 0, 4, s));
    return;
  }
  launch("spar_rank_tiles", k_bm_tiles, tiles, 256, 0, s, bm, nw, tcnt.p);
  launch("spar_rank_scan", k_scan_one_cta, 1, 1024, 0, s, tcnt.p, tiles, toff.p);
  launch("spar_rank_words", k_bm_prefix, tiles, 256, 0, s, bm, nw, toff.p, wpre.p);
}

}  // namespace

void sparsify_count(bfly_graph* g, int mode, double p, uint64_t n_colors, uint64_t seed,
                    const uint8_t* h_keep, const uint32_t* h_colors, uint64_t* count,
                    uint64_t* kept) {
  cudaStream_t s = g->stream;
  const uint64_t m = g->m, n = g->n();
  *count = 0;
  *kept = 0;
  if (m == 0) return;
  KeepArgs a{};
  {  // mix64(seed) is hoisted: derive_seed(seed, i) = mix64(mix64(seed) ^ mix64(i))
    uint64_t x = seed + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    a.ms = x ^ (x >> 31);
  }
  // unit_double(h) = (h >> 11) * 2^-53 is exact, so unit_double(h) < p <=> (h >> 11) < p*2^53
  // (exact: scaling by a power of two) <=> (h >> 11) < ceil(p * 2^53) for the integer h >> 11
  if (mode == 0) a.thr = static_cast<uint64_t>(std::ceil(p * 0x1.0p53));
  a.n_colors = n_colors;
  a.L = g->L;
  DBuf<uint8_t> dkeep;
  DBuf<uint32_t> dcol;
  if (mode == 2) {
    dkeep.alloc(m, s);
    BFLY_CUDA(cudaMemcpyAsync(dkeep.p, h_keep, m, cudaMemcpyHostToDevice, s));
    a.hkeep = dkeep.p;
  } else if (mode == 3) {
    dcol.alloc(n, s);
    BFLY_CUDA(cudaMemcpyAsync(dcol.p, h_colors, n * 4, cudaMemcpyHostToDevice, s));
    a.hcol = dcol.p;
  }
  // row of every entry of both directions (kept from the build)
  DBuf<uint32_t> lrow_tmp, rrow_tmp;
  const uint32_t* lrow = g->lrow.p;
  const uint32_t* rrow = g->rrow.p;
  if (!lrow) {
    lrow_tmp.alloc(m, s);
    launch("spar_row_of", k_row_of, grid_for(uint64_t{g->L} * 32, 256), 256, 0, s, g->loff.p, g->L,
           lrow_tmp.p);
    lrow = lrow_tmp.p;
  }
  if (!rrow) {
    rrow_tmp.alloc(m, s);
    launch("spar_row_of", k_row_of, grid_for(uint64_t{g->R} * 32, 256), 256, 0, s, g->roff.p, g->R,
           rrow_tmp.p);
    rrow = rrow_tmp.p;
  }
  if (mode == 0 || mode == 2) ensure_reid(g);  // right entries test their canonical edge's bit

  const uint64_t words = (m + 31) / 32;
  const unsigned tiles = static_cast<unsigned>((m + kTileEntries - 1) / kTileEntries);
  DBuf<uint32_t> lbits(words, s), rbits(words, s);
  DBuf<uint32_t> cnt(2 * uint64_t{tiles}, s), off(2 * (uint64_t{tiles} + 1), s);
  uint32_t* lcnt = cnt.p;
  uint32_t* rcnt = cnt.p + tiles;
  uint32_t* loffs = off.p;
  uint32_t* roffs = off.p + tiles + 1;
  launch_keep<false>(mode, a, lrow, g->ladj.p, nullptr, m, lbits.p, lcnt, tiles, s);
  a.lbits = lbits.p;
  launch_keep<true>(mode, a, rrow, g->radj.p, g->reid.p, m, rbits.p, rcnt, tiles, s);
  launch("spar_scan", k_scan_one_cta, 1, 1024, 0, s, lcnt, tiles, loffs);
  launch("spar_scan", k_scan_one_cta, 1, 1024, 0, s, rcnt, tiles, roffs);
  uint32_t tot[2] = {0, 0};
  BFLY_CUDA(cudaMemcpyAsync(&tot[0], loffs + tiles, 4, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaMemcpyAsync(&tot[1], roffs + tiles, 4, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  const uint32_t mk = tot[0];
  if (tot[1] != mk)
    fail(kInternal, "sparsify: left and right CSR retained different edge counts");
  *kept = mk;
  if (mk == 0) return;  // sparsify.cpp:22: nothing retained -> 0

  // kept entries of both directions in CSR order (row, column), old dense ids
  DBuf<uint32_t> klr(mk, s), klc(mk, s), krr(mk, s), krc(mk, s);
  launch("spar_emit_left", k_emit, tiles, kTileThreads, 0, s, lbits.p, loffs, lrow, g->ladj.p, m,
         klr.p, klc.p);
  launch("spar_emit_right", k_emit, tiles, kTileThreads, 0, s, rbits.p, roffs, rrow, g->radj.p, m,
         krr.p, krc.p);
  lbits.release();
  rbits.release();
  // live vertices of each side and their new ids
  const uint64_t lw = (uint64_t{g->L} + 31) / 32, rw = (uint64_t{g->R} + 31) / 32;
  DBuf<uint32_t> live(lw + rw, s);
  live.zero();
  uint32_t* livel = live.p;
  uint32_t* liver = live.p + lw;
  launch("spar_live", k_mark_live, grid_for(mk, 256), 256, 0, s, klr.p, mk, livel);
  launch("spar_live", k_mark_live, grid_for(mk, 256), 256, 0, s, krr.p, mk, liver);
  DBuf<uint32_t> lpre, ltc, lto, rpre, rtc, rto;
  bitmap_rank(livel, g->L, lpre, ltc, lto, s);
  bitmap_rank(liver, g->R, rpre, rtc, rto, s);
  uint32_t sizes[2] = {0, 0};
  BFLY_CUDA(cudaMemcpyAsync(&sizes[0], lto.p + (lto.n - 1), 4, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaMemcpyAsync(&sizes[1], rto.p + (rto.n - 1), 4, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));

  bfly_graph sub;
  sub.device = g->device;
  sub.stream = s;
  sub.L = sizes[0];
  sub.R = sizes[1];
  sub.m = mk;
  sub.reid_ready = false;
  sub.loff.alloc(uint64_t{sub.L} + 1, s);
  sub.roff.alloc(uint64_t{sub.R} + 1, s);
  sub.ladj.alloc(mk, s);
  sub.radj.alloc(mk, s);
  launch("spar_fill_left", k_fill, grid_for(mk, 256), 256, 0, s, klr.p, klc.p, mk, livel, lpre.p,
         liver, rpre.p, sub.L, sub.loff.p, sub.ladj.p);
  launch("spar_fill_right", k_fill, grid_for(mk, 256), 256, 0, s, krr.p, krc.p, mk, liver, rpre.p,
         livel, lpre.p, sub.R, sub.roff.p, sub.radj.p);
  klr.release();
  klc.release();
  krr.release();
  krc.release();
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
