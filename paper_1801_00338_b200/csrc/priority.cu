// priority.cu -- degree-priority relabelling and the wedge plan of the exact kernels.
//
// Every vertex of both sides gets a priority id p: degree descending, ties by global index
// ascending (a strict total order). The merged-side CSR lists neighbours in ascending p.
// A butterfly is counted once, at its highest-priority vertex u ("start"): wedges
// (u, v, w) with v > u and w > u in priority order. The reference anchors at every vertex
// of one side and walks w < v in dense-id order (exact.cpp:29-41); both enumerate every
// butterfly exactly once, so the uint64 totals are identical.
//
// Build: row p of the priority CSR is the canonical row of inv[p] mapped through rank[] and
// sorted; every row is sorted independently where it fits (RowIn / RowOut below). The wedge
// plan then locates each forward entry's start vertex inside the list it points to.
#include <cub/block/block_radix_sort.cuh>
#include <utility>
#include <cub/warp/warp_merge_sort.cuh>

#include "cubwrap.cuh"
#include "graph.cuh"

#include <cstdlib>

namespace bflyd {
namespace {

__global__ void k_degkeys(const uint64_t* __restrict__ loff, const uint64_t* __restrict__ roff,
                          uint32_t L, uint32_t R, uint32_t* __restrict__ key,
                          uint32_t* __restrict__ gid) {
  uint64_t n = uint64_t{L} + R;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = g < L ? loff[g + 1] - loff[g] : roff[g - L + 1] - roff[g - L];
    key[g] = 0xFFFFFFFFu - static_cast<uint32_t>(d);
    gid[g] = static_cast<uint32_t>(g);
  }
}

__global__ void k_rank(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ inv,
                       uint64_t n, uint32_t* __restrict__ rank, uint64_t* __restrict__ pdeg) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p <= n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    if (p == n) {
      pdeg[n] = 0;
    } else {
      rank[inv[p]] = static_cast<uint32_t>(p);
      pdeg[p] = 0xFFFFFFFFu - skey[p];
    }
  }
}

// ---- priority CSR by per-row sorts ---------------------------------------------------------
// Row p of the priority CSR is the canonical row of x = inv[p] with every neighbour y mapped
// to rank[y] and sorted ascending. Rows are independent, so each is sorted where it fits:
// sub-warp bitonic networks (<= 32 entries), one warp (<= 256, merge sort in registers), one
// CTA (<= 8192, radix sort in shared memory), and one device-wide radix sort of
// (p, rank) keys for the few longer rows. Priority ids are degree-descending, so every size
// class is a contiguous range of p and needs no classification pass.
// (Recording each entry's position under its canonical edge id, so that the plan could
// read the reverse entry instead of searching for it, was measured slower: those writes are
// scattered 8-byte partial-sector stores, 2.2 ms on config 2 against 1.2 ms of search.)
struct RowIn {
  const uint32_t* inv;
  uint32_t L;
  const uint64_t* loff;
  const uint32_t* ladj;
  const uint64_t* roff;
  const uint32_t* radj;
  const uint32_t* reid;
  const uint32_t* rank;
  bool want_e;  // canonical edge ids wanted (with_eid): right rows then also read reid
  __device__ __forceinline__ void row(uint32_t p, uint64_t& off, bool& left) const {
    const uint32_t x = inv[p];
    left = x < L;
    off = left ? loff[x] : roff[x - L];
  }
  // j-th canonical entry of the row, key only (builds that keep no canonical edge ids)
  __device__ __forceinline__ uint32_t key_of(bool left, uint64_t off, uint32_t j) const {
    return left ? rank[L + ladj[off + j]] : rank[radj[off + j]];
  }
  // j-th canonical entry of the row: (rank of the neighbour, canonical edge id)
  __device__ __forceinline__ void entry(bool left, uint64_t off, uint32_t j, uint32_t& key,
                                        uint32_t& e) const {
    if (left) {
      key = rank[L + ladj[off + j]];
      e = static_cast<uint32_t>(off + j);
    } else {
      key = rank[radj[off + j]];
      e = want_e ? reid[off + j] : 0u;
    }
  }
};

// Per-vertex head record for the wedge plan: (row start, degree, first kHead entries) in one
// 64-byte line, so a lookup of u in N(v) usually costs one sector pair instead of the offsets
// plus the start of the list.
constexpr uint32_t kHead = 14;

struct RowOut {
  const uint64_t* poff;
  uint32_t* padj;
  uint32_t* psrc;
  uint32_t* peid;  // null: canonical edge ids not kept
  uint64_t* fwd;
  uint32_t* head;  // 16 words per priority id
  // entry j of row p (degree d) at position q
  __device__ __forceinline__ void put(uint32_t p, uint64_t q, uint32_t j, uint32_t d,
                                      uint32_t key, uint32_t e) const {
    padj[q] = key;
    psrc[q] = p;
    if (peid) peid[q] = e;
    uint32_t* h = head + 16ull * p;
    if (j < kHead) h[2 + j] = key;
    if (j == 0) {
      h[0] = static_cast<uint32_t>(q);
      h[1] = d;
    }
  }
};

// ascending bitonic sort of (key, e) over aligned groups of G lanes (lane index j in group)
// (WE = false: keys only -- the counting-only build keeps no edge ids, and the payload would
// double the shuffles of every compare-exchange step)
template <int G, bool WE>
__device__ __forceinline__ void group_bitonic(uint32_t& key, uint32_t& e, unsigned j) {
#pragma unroll
  for (int k = 2; k <= G; k <<= 1)
#pragma unroll
    for (int s = k >> 1; s > 0; s >>= 1) {
      const uint32_t ok = __shfl_xor_sync(0xffffffffu, key, s);
      uint32_t oe = 0;
      if constexpr (WE) oe = __shfl_xor_sync(0xffffffffu, e, s);
      const bool up = (j & k) == 0;
      const bool lower = (j & s) == 0;
      if constexpr (WE) {
        const bool take = (lower == up) ? (ok < key) : (ok > key);
        if (take) {
          key = ok;
          e = oe;
        }
      } else {
        key = (lower == up) ? min(key, ok) : max(key, ok);
      }
    }
}

// rows of degree <= G (G a power of two <= 32): 32/G rows per warp. Rows of degree 0 (G = 1
// class) only get fwd.
template <int G, bool WE>
__global__ void __launch_bounds__(256) k_prow_small(RowIn in, RowOut out, uint32_t pa,
                                                    uint32_t pb) {
  constexpr unsigned R = 32 / G;
  const unsigned lane = threadIdx.x & 31, j = lane % G;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = pa + gw * R; base < pb; base += nw * R) {
    const uint64_t pp = base + lane / G;
    const bool vrow = pp < pb;
    const uint32_t p = static_cast<uint32_t>(pp);
    uint32_t d = 0;
    uint64_t off = 0, q0 = 0;
    bool left = true;
    if (vrow) {
      q0 = out.poff[p];
      d = static_cast<uint32_t>(out.poff[p + 1] - q0);
      if (d) in.row(p, off, left);
    }
    uint32_t key = 0xFFFFFFFFu, e = 0;
    if (j < d) {
      if constexpr (WE) in.entry(left, off, j, key, e);
      else key = in.key_of(left, off, j);
    }
    if constexpr (G > 1) group_bitonic<G, WE>(key, e, j);
    if (j < d) out.put(p, q0 + j, j, d, key, e);
    const unsigned below = __ballot_sync(0xffffffffu, j < d && key < p);
    if (vrow && j == 0) {
      const unsigned gm = G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u);
      out.fwd[p] = q0 + __popc((below >> (lane & ~(G - 1u))) & gm);
    }
  }
}

struct LessU32 {
  __device__ __forceinline__ bool operator()(uint32_t a, uint32_t b) const { return a < b; }
};

// rows of degree <= 32 * ITEMS: one warp per row, merge sort in registers
template <int ITEMS, bool WE>
__global__ void __launch_bounds__(256) k_prow_warp(RowIn in, RowOut out, uint32_t pa,
                                                   uint32_t pb) {
  using WS = std::conditional_t<WE, cub::WarpMergeSort<uint32_t, ITEMS, 32, uint32_t>,
                                cub::WarpMergeSort<uint32_t, ITEMS, 32>>;
  __shared__ typename WS::TempStorage ts[8];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t pp = pa + gw; pp < pb; pp += nw) {
    const uint32_t p = static_cast<uint32_t>(pp);
    const uint64_t q0 = out.poff[p];
    const uint32_t d = static_cast<uint32_t>(out.poff[p + 1] - q0);
    uint64_t off;
    bool left;
    in.row(p, off, left);
    uint32_t k[ITEMS], v[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = i * 32 + lane;
      k[i] = 0xFFFFFFFFu;
      v[i] = 0;
      if (idx < d) {
        if constexpr (WE) in.entry(left, off, idx, k[i], v[i]);
        else k[i] = in.key_of(left, off, idx);
      }
    }
    if constexpr (WE) WS(ts[wl]).Sort(k, v, LessU32());
    else WS(ts[wl]).Sort(k, LessU32());
    unsigned nb = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t pos = lane * ITEMS + i;
      if (pos < d) {
        out.put(p, q0 + pos, pos, d, k[i], v[i]);
        nb += k[i] < p;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0) out.fwd[p] = q0 + nb;
    __syncwarp();
  }
}

// rows of degree <= BLOCK * ITEMS: one CTA per row, radix sort in shared memory on the low
// kbits bits (2^kbits > n: the padding key sorts after every rank)
template <int BLOCK, int ITEMS, bool WE>
__global__ void __launch_bounds__(BLOCK) k_prow_block(RowIn in, RowOut out, uint32_t pa,
                                                      uint32_t pb, int kbits) {
  using BRS = std::conditional_t<WE, cub::BlockRadixSort<uint32_t, BLOCK, ITEMS, uint32_t>,
                                 cub::BlockRadixSort<uint32_t, BLOCK, ITEMS>>;
  __shared__ typename BRS::TempStorage ts;
  for (uint32_t p = pa + blockIdx.x; p < pb; p += gridDim.x) {
    const uint64_t q0 = out.poff[p];
    const uint32_t d = static_cast<uint32_t>(out.poff[p + 1] - q0);
    uint64_t off;
    bool left;
    in.row(p, off, left);
    uint32_t k[ITEMS], v[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = i * BLOCK + threadIdx.x;
      k[i] = 0xFFFFFFFFu;
      v[i] = 0;
      if (idx < d) {
        if constexpr (WE) in.entry(left, off, idx, k[i], v[i]);
        else k[i] = in.key_of(left, off, idx);
      }
    }
    if constexpr (WE) BRS(ts).SortBlockedToStriped(k, v, 0, kbits);
    else BRS(ts).SortBlockedToStriped(k, 0, kbits);
    int nb = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t pos = i * BLOCK + threadIdx.x;
      const bool ok = pos < d;
      if (ok) out.put(p, q0 + pos, pos, d, k[i], v[i]);
      nb += __syncthreads_count(ok && k[i] < p);
    }
    if (threadIdx.x == 0) out.fwd[p] = q0 + nb;
    __syncthreads();
  }
}

// rows [0, pb) (the longest): key = p << kbits | rank, value = canonical edge id
template <typename K>
__global__ void k_prow_big_fill(RowIn in, const uint64_t* __restrict__ poff, uint32_t pb,
                                uint64_t nq, int kbits, K* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = pb;  // last p with poff[p] <= q
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(poff + mid) <= q) lo = mid;
      else hi = mid;
    }
    uint64_t off;
    bool left;
    in.row(lo, off, left);
    uint32_t key, e;
    in.entry(left, off, static_cast<uint32_t>(q - poff[lo]), key, e);
    keys[q] = (static_cast<K>(lo) << kbits) | key;
    if (vals) vals[q] = e;
  }
}

template <typename K>
__global__ void k_prow_big_post(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                uint64_t nq, int kbits, RowOut out) {
  const K mask = (K(1) << kbits) - 1;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const K kq = keys[q];
    const uint32_t p = static_cast<uint32_t>(kq >> kbits), r = static_cast<uint32_t>(kq & mask);
    const uint64_t q0 = out.poff[p], q1 = out.poff[p + 1];
    const uint32_t j = static_cast<uint32_t>(q - q0), d = static_cast<uint32_t>(q1 - q0);
    out.put(p, q, j, d, r, vals ? vals[q] : 0u);  // vals: canonical edge ids (with_eid only)
    const uint32_t prev = j ? static_cast<uint32_t>(keys[q - 1] & mask) : 0u;
    if (r > p && (j == 0 || prev < p)) out.fwd[p] = q;
    if (r < p && j == d - 1) out.fwd[p] = q1;
  }
}

// number of priority ids of degree > thr[t] (degrees are non-increasing in p)
__global__ void k_prow_bounds(const uint64_t* __restrict__ poff, uint64_t n,
                              const uint32_t* __restrict__ thr, int nt,
                              unsigned long long* __restrict__ cnt) {
  const int t = threadIdx.x;
  if (t < nt) {
    uint64_t lo = 0, hi = n;  // first p with deg(p) <= thr
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (poff[mid + 1] - poff[mid] > thr[t]) lo = mid + 1;
      else hi = mid;
    }
    cnt[t] = lo;
    cnt[nt + t] = poff[lo];
  }
}

// Wedge plan, one thread per directed entry q = (u -> v). A forward entry (v > u) needs the
// position of u inside the ascending list N(v): the wedge suffix is N(v) after u. u has the
// higher priority, so it usually sits near the front of N(v): v's 64-byte head record (row
// start, degree, first kHead entries, written by the row sorts) is read whole and counted, and
// only longer prefixes fall back to a binary search. fseg is written for every entry (whole
// sectors; backward entries get (0, 0)). work[u] = sum of the suffix lengths (warp-segmented,
// one atomic per run of equal u).
__global__ void k_plan(const uint32_t* __restrict__ head, const uint32_t* __restrict__ padj,
                       const uint32_t* __restrict__ psrc, uint64_t nnz, uint2* __restrict__ fseg,
                       unsigned long long* __restrict__ work) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) & ~31ull;
  for (uint64_t base = warp * 32; base < nnz; base += stride) {
    const uint64_t q = base + lane;
    const bool valid = q < nnz;
    const uint32_t u = valid ? __ldcs(psrc + q) : 0xFFFFFFFFu;  // streamed: keep L2 for heads
    unsigned long long wk = 0;
    if (valid) {
      const uint32_t v = __ldcs(padj + q);
      uint2 f = make_uint2(0u, 0u);
      if (v > u) {
        const uint4* hp = reinterpret_cast<const uint4*>(head + 16ull * v);
        const uint4 h0 = __ldg(hp), h1 = __ldg(hp + 1), h2 = __ldg(hp + 2), h3 = __ldg(hp + 3);
        const uint32_t b = h0.x, dv = h0.y, e = b + dv;
        const uint32_t xs[kHead] = {h0.z, h0.w, h1.x, h1.y, h1.z, h1.w, h2.x,
                                    h2.y, h2.z, h2.w, h3.x, h3.y, h3.z, h3.w};
        const uint32_t nh = dv < kHead ? dv : kHead;
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < (int)kHead; ++i) c += ((uint32_t)i < nh && xs[i] < u);
        uint32_t lo = b + c;
        if (c == nh && nh < dv) {  // u lies beyond the head entries
          uint32_t hi = e;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (padj[mid] < u) lo = mid + 1;
            else hi = mid;
          }
        }
        f = make_uint2(lo + 1, e - lo - 1);
        wk = e - lo - 1;
      }
      __stcs(fseg + q, f);
    }
    const unsigned full = 0xffffffffu;
    const uint32_t up = __shfl_up_sync(full, u, 1);
    const bool head = lane == 0 || up != u;
    const unsigned heads = __ballot_sync(full, head);
    const int my_head = 31 - __clz(heads & ((2u << lane) - 1u));
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long y = __shfl_up_sync(full, wk, off);
      if ((int)lane - off >= my_head) wk += y;
    }
    const uint32_t dn = __shfl_down_sync(full, u, 1);
    const bool tail = lane == 31 || dn != u;
    if (valid && tail && wk) atomicAdd(&work[u], wk);
  }
}

}  // namespace

// Sort the rows of the priority CSR (RowIn / RowOut above), then derive the wedge plan.
static void build_priority_rows(bfly_graph* g, bool with_eid) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n(), nnz = 2 * g->m;
  const int kbits = std::max(1, bits_for(n));  // 2^kbits > n > every rank
  g->psrc.alloc(nnz, s);
  // (+4 words: the vectorised walks read whole aligned 16-byte chunks, aggregate.cuh)
  g->padj.alloc(nnz + 4, s);
  if (reinterpret_cast<uintptr_t>(g->padj.p) & 15u) fail(kInternal, "priority adjacency not 16-byte aligned");
  uint32_t* peid = nullptr;
  if (with_eid) {
    g->peid.alloc(nnz, s);
    peid = g->peid.p;
  }
  g->fwd.alloc(n, s);
  const RowIn in{g->inv.p,  g->L,    g->loff.p, g->ladj.p, g->roff.p,
                 g->radj.p, g->reid.p, g->rank.p, with_eid};
  // size classes: P[c] = number of priority ids of degree > thr[c] (P[14]: of any degree;
  // isolated vertices -- sparsified sub-graphs keep every id -- come last and need no head)
  constexpr int kNT = 15;
  static const uint32_t thr_h[kNT] = {8192, 4096, 2048, 1024, 512, 256, 128, 64,
                                      32,   16,   8,    4,   2,   1,   0};
  DBuf<uint32_t> thr(kNT, s);
  DBuf<unsigned long long> cnt(2 * kNT, s);
  BFLY_CUDA(cudaMemcpyAsync(thr.p, thr_h, sizeof(thr_h), cudaMemcpyHostToDevice, s));
  launch("prio_rows_bounds", k_prow_bounds, 1, 32, 0, s, g->poff.p, n, thr.p, kNT, cnt.p);
  unsigned long long P[2 * kNT];
  read_back(s, {{P, cnt.p, sizeof(P)}});
  g->prio_nz = P[14];
  DBuf<uint32_t> head(16 * std::max<uint64_t>(1, P[14]), s);  // (lives until the plan below)
  const RowOut out{g->poff.p, g->padj.p, g->psrc.p, peid, g->fwd.p, head.p};
  // rows [0, P[0]) (degree > 8192): one device-wide sort of (p << kbits | rank) keys
  const uint32_t pbig = static_cast<uint32_t>(P[0]);
  const uint64_t nbig = P[kNT];
  if (nbig) {
    auto big = [&](auto zero_key) {
      using K = decltype(zero_key);
      const int bits = kbits + std::max(1, bits_for(pbig - 1));
      DBuf<K> k0(nbig, s), k1(nbig, s);
      DBuf<uint32_t> v0, v1;
      if (with_eid) {
        v0.alloc(nbig, s);
        v1.alloc(nbig, s);
      }
      launch("prio_rows_big_fill", k_prow_big_fill<K>, grid_for(nbig, 256, 148u * 16u), 256, 0, s,
             in, g->poff.p, pbig, nbig, kbits, k0.p, v0.p);
      const bool alt = with_eid
                           ? sort_pairs_db(k0.p, k1.p, v0.p, v1.p, nbig, 0, bits, s, "sort_prio_rows_big")
                           : sort_keys_db(k0.p, k1.p, nbig, 0, bits, s, "sort_prio_rows_big");
      if (!alt) {
        std::swap(k0, k1);
        std::swap(v0, v1);
      }
      launch("prio_rows_big_post", k_prow_big_post<K>, grid_for(nbig, 256, 148u * 16u), 256, 0, s,
             k1.p, v1.p, nbig, kbits, out);
    };
    if (kbits + bits_for(pbig - 1) <= 32) big(uint32_t{0});
    else big(uint64_t{0});
  }
  auto range = [&](int c) {  // priority ids of class c: [P[c-1], P[c])
    return std::make_pair(static_cast<uint32_t>(P[c - 1]), static_cast<uint32_t>(P[c]));
  };
  auto block = [&](auto kern, int blk, int c) {
    const auto r = range(c);
    if (r.second > r.first)
      launch("prio_rows_block", kern, std::min<uint32_t>(r.second - r.first, 148u * 8u), blk, 0, s,
             in, out, r.first, r.second, kbits);
  };
  auto warp = [&](auto kern, int c) {
    const auto r = range(c);
    if (r.second > r.first)
      launch("prio_rows_warp", kern, grid_for(uint64_t{r.second - r.first} * 32, 256, 148u * 16u),
             256, 0, s, in, out, r.first, r.second);
  };
  auto small = [&](auto kern, int G, uint32_t a, uint32_t b) {
    if (b > a)
      launch("prio_rows_small", kern, grid_for(uint64_t{b - a} * G, 256, 148u * 16u), 256, 0, s,
             in, out, a, b);
  };
  auto rows = [&](auto we) {
    constexpr bool WE = decltype(we)::value;
    block(k_prow_block<512, 16, WE>, 512, 1);  // (4096, 8192]
    block(k_prow_block<256, 16, WE>, 256, 2);  // (2048, 4096]
    block(k_prow_block<256, 8, WE>, 256, 3);   // (1024, 2048]
    block(k_prow_block<256, 4, WE>, 256, 4);   // (512, 1024]
    block(k_prow_block<256, 2, WE>, 256, 5);   // (256, 512]
    warp(k_prow_warp<8, WE>, 6);  // (128, 256]
    warp(k_prow_warp<4, WE>, 7);  // (64, 128]
    warp(k_prow_warp<2, WE>, 8);  // (32, 64]
    small(k_prow_small<32, WE>, 32, range(9).first, range(9).second);     // (16, 32]
    small(k_prow_small<16, WE>, 16, range(10).first, range(10).second);   // (8, 16]
    small(k_prow_small<8, WE>, 8, range(11).first, range(11).second);     // (4, 8]
    small(k_prow_small<4, WE>, 4, range(12).first, range(12).second);     // (2, 4]
    small(k_prow_small<2, WE>, 2, range(13).first, range(13).second);     // (1, 2]
    small(k_prow_small<1, WE>, 1, static_cast<uint32_t>(P[13]), static_cast<uint32_t>(n));  // <= 1
  };
  // (keys only when the build keeps no canonical edge ids: the exact count's build)
  if (with_eid) rows(std::true_type{});
  else rows(std::false_type{});
  // wedge plan
  g->fseg.alloc(nnz, s);
  g->work.alloc(n, s);
  g->work.zero();
  launch("prio_plan", k_plan, grid_for(nnz, 256, 148u * 64u), 256, 0, s, head.p, g->padj.p,
         g->psrc.p, nnz, g->fseg.p, reinterpret_cast<unsigned long long*>(g->work.p));
}

void ensure_priority(bfly_graph* g, bool with_eid) {
  if (g->prio_ready && (!with_eid || g->prio_has_eid)) return;
  if (with_eid) ensure_reid(g);  // right rows carry canonical edge ids
  cudaStream_t s = g->stream;
  const uint64_t n = g->n();
  g->prio_ready = false;
  g->hub_ready = false;  // the hub plan indexes priority-CSR entries
  if (n == 0) {
    g->poff.alloc(1, s);
    g->poff.zero();
    g->rank.alloc(1, s);
    g->inv.alloc(1, s);
    g->padj.alloc(1, s);
    g->psrc.alloc(1, s);
    g->fseg.alloc(1, s);
    g->work.alloc(1, s);
    g->fwd.alloc(1, s);
    g->total_work = 0;
    g->prio_ready = true;
    g->prio_has_eid = with_eid;
    return;
  }
  // 1. priority order: degree descending, ties by global id (stable sort of ~degree)
  {
    DBuf<uint32_t> key(n, s), gid(n, s), skey(n, s);
    launch("prio_degkeys", k_degkeys, grid_for(n, 256), 256, 0, s, g->loff.p, g->roff.p, g->L,
           g->R, key.p, gid.p);
    g->inv.alloc(n, s);
    if (!sort_pairs_db(key.p, skey.p, gid.p, g->inv.p, n, 0, 32, s, "sort_priority_order")) {
      std::swap(key, skey);
      std::swap(gid, g->inv);
    }
    g->rank.alloc(n, s);
    DBuf<uint64_t> pdeg(n + 1, s);
    launch("prio_rank", k_rank, grid_for(n + 1, 256), 256, 0, s, skey.p, g->inv.p, n, g->rank.p,
           pdeg.p);
    g->poff.alloc(n + 1, s);
    exclusive_sum(pdeg.p, g->poff.p, n + 1, s);
  }
  // 2. sorted rows, 3. wedge plan
  build_priority_rows(g, with_eid);
  trace_mark("priority csr + plan (queued)");
  g->prio_ready = true;
  g->prio_has_eid = with_eid;
}

}  // namespace bflyd
