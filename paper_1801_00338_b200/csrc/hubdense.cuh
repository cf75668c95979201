// hubdense.cuh -- the dense top-hub path of the exact count: bit-sliced multiplicities.
//
// The H highest-priority hubs (H = 32 W, W words) carry a large share of all wedges (the top
// 256 of config 2's 22,417 hubs: 38%). For these the hub path's "one key per wedge" form is
// wasteful: every vertex v gets a W-word MASK of its hub neighbours u < min(H, v) (k_hub_mask),
// and a hub task w adds the masks of its entries v in N(w) instead of walking their key
// segments. The multiplicities c(u, w) = |{v in N(w) : u in N(v)}| of 32 hubs at a time are kept
// BIT-SLICED: plane P_j holds bit j of all 32 counters, and adding a mask is a carry-save
// ripple that stops at the first empty carry (one AND + XOR per plane reached). The task's
// value follows from the planes without ever materialising a counter:
//     sum_u C(c_u, 2) = sum_j (4^j - 2^j)/2 popc(P_j) + sum_{j<l} 2^(j+l) popc(P_j & P_l)
// (from c_u = sum_j 2^j P_j[u], c^2 = sum_{j,l} 2^(j+l) P_j P_l). One mask word costs about
// the instructions of ONE key of the segment walks, whatever number of hubs it holds.
// The segment walks keep the hubs [H, k): the hub plan starts every segment behind the
// entries below H (k_hub_plan). Same wedges, same integer total (exact.cpp:29-41 restated
// over the priority order).
//
//   k_hub_mask     W lanes per vertex: mask[v][j] from the first tH(v) entries of N(v)
//   k_dense_small  W lanes per task of <= 255 entries (8 planes), 32 / W tasks per warp
//   k_dense_big    tasks of > 255 entries (a prefix of the priority order: degrees descend):
//                  CTAs take fixed chunks of their contiguous entry range, see below
#pragma once

#include <cuda/barrier>

#include "aggregate.cuh"

namespace bflyd {
namespace agg {

constexpr uint32_t kDenseSmallMax = 255;  // entries of a k_dense_small task: 8 planes

// P += M (every set bit of M increments its counter); NP planes
template <int NP>
__device__ __forceinline__ void csa_add(uint32_t (&P)[NP], uint32_t M) {
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const uint32_t c = P[j] & M;
    P[j] ^= M;
    M = c;
    if (M == 0) break;
  }
}

// A += B for two bit-sliced counter sets (ripple-carry over the planes)
template <int NP>
__device__ __forceinline__ void planes_add(uint32_t (&A)[NP], const uint32_t (&B)[NP]) {
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const uint32_t x = A[j] ^ B[j];
    const uint32_t nc = (A[j] & B[j]) | (c & x);
    A[j] = x ^ c;
    c = nc;
  }
}

// sum over the 32 counters of C(c, 2); every term is non-negative and the sum is at most the
// graph's butterfly count (< 2^61), so 64 bits never overflow
template <int NP>
__device__ __forceinline__ unsigned long long planes_c2(const uint32_t (&P)[NP]) {
  uint32_t hi = 0;
#pragma unroll
  for (int j = 1; j < NP; ++j) hi |= P[j];
  if (hi == 0) return 0ull;  // every counter is 0 or 1
  unsigned long long s = 0;
#pragma unroll
  for (int l = 1; l < NP; ++l) {
    if (P[l] == 0) continue;
    s += (((1ull << (2 * l)) - (1ull << l)) >> 1) * __popc(P[l]);
#pragma unroll
    for (int j = 0; j < l; ++j) s += static_cast<unsigned long long>(__popc(P[j] & P[l])) << (j + l);
  }
  return s;
}

// bits of word j a task w may count: hubs u < w (u < H already holds for every mask bit)
__device__ __forceinline__ uint32_t dense_cut(uint32_t w, uint32_t j) {
  const uint32_t wj = w >> 5;
  return wj > j ? 0xFFFFFFFFu : wj == j ? (1u << (w & 31u)) - 1u : 0u;
}

// mask[v * W + j]: bit b set iff hub u = 32 j + b is a neighbour of v with u < min(H, v);
// th[v] = the number of such hubs (they are the first th[v] entries of the ascending N(v)).
// One thread per vertex: the row is built in registers from its th[v] entries (1.7 on average
// on config 2, at most H) and written whole (W lanes per vertex, each re-reading the entries
// for its own word, took 0.21 ms there).
template <int W>
__global__ void k_hub_mask(const uint64_t* __restrict__ poff, const uint32_t* __restrict__ padj,
                           const uint2* __restrict__ vinfo, uint64_t n,
                           uint32_t* __restrict__ mask) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = t; v < n; v += stride) {
    const uint2 vi = vinfo[v];
    const uint32_t th = vi.x >> 16;
    const uint32_t* p = padj + vi.y;
    uint32_t m[W];
#pragma unroll
    for (int j = 0; j < W; ++j) m[j] = 0;
    for (uint32_t q = 0; q < th; ++q) {
      const uint32_t u = __ldg(p + q);
      const uint32_t bit = 1u << (u & 31u);
#pragma unroll
      for (int j = 0; j < W; ++j) m[j] |= (u >> 5) == (uint32_t)j ? bit : 0u;
    }
    if constexpr (W % 4 == 0) {
      uint4* row = reinterpret_cast<uint4*>(mask + v * W);
#pragma unroll
      for (int j = 0; j < W / 4; ++j) row[j] = make_uint4(m[4 * j], m[4 * j + 1], m[4 * j + 2], m[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) mask[v * W + j] = m[j];
    }
  }
}

// out[0] total, out[1] overflow flag, out[2] keys (wedges) taken by the dense path, out[3] the
// entries (mask rows) it read, out[4] those of them read by k_dense_big
__device__ __forceinline__ void dense_flush(unsigned long long t, unsigned long long keys,
                                            unsigned long long ents, unsigned long long* out) {
  Acc a;
  a.v = t;
  flush_acc(a, out, reinterpret_cast<unsigned*>(out + 1));
  for (int off = 16; off > 0; off >>= 1) {
    keys += __shfl_xor_sync(0xffffffffu, keys, off);
    ents += __shfl_xor_sync(0xffffffffu, ents, off);
  }
  if ((threadIdx.x & 31) == 0 && keys) atomicAdd(out + 2, keys);
  if ((threadIdx.x & 31) == 0 && ents) atomicAdd(out + 3, ents);
}

// W lanes per task, 32 / W tasks per warp; four mask loads in flight per lane. (Measured on
// config 2, W = 8, kernel alone: 0.84 ms; two tasks in flight per group 1.10 ms and a software-
// pipelined entry stream 1.29 ms -- both need more registers and lose resident warps. The kernel
// is bound by random 32-byte sector reads of the 221 MB mask array, not by its load chains.)
template <int W>
__global__ void __launch_bounds__(256) k_dense_small(const uint64_t* __restrict__ poff,
                                                     const uint32_t* __restrict__ padj,
                                                     const uint32_t* __restrict__ mask,
                                                     uint64_t nt, uint32_t H,
                                                     unsigned long long* __restrict__ out) {
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t ngroups = ((uint64_t)gridDim.x * blockDim.x) / W;
  const uint32_t j = static_cast<uint32_t>(gt % W);
  unsigned long long total = 0, keys = 0, ents = 0;
  for (uint64_t w = gt / W; w < nt; w += ngroups) {
    const uint64_t e0 = poff[w], e1 = poff[w + 1];
    // (one entry: no pair of wedges; more than kDenseSmallMax: k_dense_big)
    if (e1 - e0 > kDenseSmallMax || e1 - e0 < 2) continue;
    const uint32_t cut = w < H ? dense_cut(static_cast<uint32_t>(w), j) : 0xFFFFFFFFu;
    uint32_t P[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t nk = 0;
    uint64_t e = e0;
    for (; e + 4 <= e1; e += 4) {
      uint32_t v[4], M[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldg(padj + e + q);
#pragma unroll
      for (int q = 0; q < 4; ++q) M[q] = __ldg(mask + (uint64_t)v[q] * W + j) & cut;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (M[q]) {
          nk += __popc(M[q]);
          csa_add(P, M[q]);
        }
      }
    }
    for (; e < e1; ++e) {
      const uint32_t M = __ldg(mask + (uint64_t)__ldg(padj + e) * W + j) & cut;
      if (M) {
        nk += __popc(M);
        csa_add(P, M);
      }
    }
    keys += nk;
    if (j == 0) ents += e1 - e0;
    total += planes_c2(P);
  }
  dense_flush(total, keys, ents, out);
}

// dinfo[0] = the number of tasks with more than kDenseSmallMax entries (a prefix of the
// priority order: degrees descend), dinfo[1] = their entries = poff[dinfo[0]]
__global__ void k_dense_bounds(const uint64_t* __restrict__ poff, uint64_t nt,
                               unsigned long long* __restrict__ dinfo) {
  if (threadIdx.x || blockIdx.x) return;
  uint64_t lo = 0, hi = nt;  // first w with degree <= kDenseSmallMax
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (poff[mid + 1] - poff[mid] > kDenseSmallMax) lo = mid + 1;
    else hi = mid;
  }
  dinfo[0] = lo;
  dinfo[1] = poff[lo];
}

// The entries of the big tasks are one contiguous range [0, E) of the priority CSR: CTAs take
// chunks of kDensePart entries, and inside a chunk one task segment after the other (psrc
// names the task of an entry). 256 / W sub-lanes stride a segment's entries with W lanes each
// (one per mask word); their planes are merged by bit-sliced ripple additions through shuffles
// and shared memory. A segment that is a whole task is finalised from the planes; a task cut
// by chunk boundaries merges its parts' counts m(u) in a global row of H counters with the
// old-value identity (a part that finds o adds o m + C(m, 2): the parts sum to C(c, 2)).
constexpr uint32_t kDensePart = 4096;  // <= 2^13 - 1 entries per segment: 13 planes
constexpr int kDensePlanes = 13;
inline uint64_t dense_rows(uint64_t nnz) { return nnz / kDensePart + 2; }

// The neighbour ids of a chunk are one aligned run of the priority adjacency: a bulk
// asynchronous copy (cp.async.bulk, one issuing thread, completion on an mbarrier) stages them
// in shared memory, double-buffered, so the next chunk's ids arrive while this chunk's mask
// rows are read and the id -> mask row load chain is one global load shorter.
#ifndef BFLY_DENSE_BULK
#define BFLY_DENSE_BULK 1
#endif
template <int W>
__global__ void __launch_bounds__(256) k_dense_big(const uint64_t* __restrict__ poff,
                                                   const uint32_t* __restrict__ padj,
                                                   const uint32_t* __restrict__ psrc,
                                                   const uint32_t* __restrict__ mask,
                                                   const unsigned long long* __restrict__ dinfo,
                                                   uint32_t H, uint32_t* __restrict__ rows,
                                                   unsigned long long* __restrict__ out) {
  static_assert(W >= 1 && W <= 32 && (W & (W - 1)) == 0, "W: a power of two up to 32");
  constexpr int NP = kDensePlanes;
  constexpr int S = 256 / W;  // sub-lanes: entries a + s, a + s + S, ...
  __shared__ uint32_t sm[8 * NP * W];
  __shared__ uint32_t fin[NP * W];
#if BFLY_DENSE_BULK
  using barrier_t = cuda::barrier<cuda::thread_scope_block>;
  __shared__ alignas(16) uint32_t ids[2][kDensePart];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier_t bar[2];
  if (threadIdx.x == 0) {
    init(&bar[0], blockDim.x);
    init(&bar[1], blockDim.x);
    cuda::device::experimental::fence_proxy_async_shared_cta();
  }
  __syncthreads();
#endif
  const uint32_t j = threadIdx.x % W, sl = threadIdx.x / W;
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint64_t E = dinfo[1];
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4] = E;  // (statistics: entries of the big tasks)
  unsigned long long total = 0, keys = 0, ents = 0;
  const uint64_t step = gridDim.x * (uint64_t)kDensePart;
#if BFLY_DENSE_BULK
  // every thread arrives once per chunk on the chunk's barrier; thread 0 also issues the copy
  // and adds its bytes to the barrier's transaction count
  auto stage = [&](uint64_t c0, int b) -> barrier_t::arrival_token {
    if (threadIdx.x == 0) {
      const uint64_t c1 = c0 + kDensePart < E ? c0 + kDensePart : E;
      const uint32_t bytes = (static_cast<uint32_t>(c1 - c0) * 4u + 15u) & ~15u;  // (padj is padded)
      cuda::device::memcpy_async_tx(ids[b], padj + c0, cuda::aligned_size_t<16>(bytes), bar[b]);
      return cuda::device::barrier_arrive_tx(bar[b], 1, bytes);
    }
    return bar[b].arrive();
  };
  barrier_t::arrival_token tok[2];
  if (blockIdx.x * (uint64_t)kDensePart < E) tok[0] = stage(blockIdx.x * (uint64_t)kDensePart, 0);
  int buf = 0;
#endif
  for (uint64_t c0 = blockIdx.x * (uint64_t)kDensePart; c0 < E; c0 += step) {
    const uint64_t c1 = c0 + kDensePart < E ? c0 + kDensePart : E;
#if BFLY_DENSE_BULK
    // (the other buffer was last read in the previous chunk, which ended with a barrier)
    if (c0 + step < E) tok[buf ^ 1] = stage(c0 + step, buf ^ 1);
    bar[buf].wait(std::move(tok[buf]));
    const uint32_t* cid = ids[buf] - c0;  // entry e of the chunk at cid[e]
#else
    const uint32_t* cid = padj;
#endif
    uint64_t a = c0;
    while (a < c1) {  // (CTA-uniform)
      const uint32_t w = __ldg(psrc + a);
      const uint64_t r0 = poff[w], r1 = poff[w + 1];
      const uint64_t b = r1 < c1 ? r1 : c1;
      const bool whole = a == r0 && b == r1;
      const uint32_t cut = w < H ? dense_cut(w, j) : 0xFFFFFFFFu;
      uint32_t P[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) P[q] = 0;
      uint32_t nk = 0;
      // four mask loads in flight per lane
      for (uint64_t e = a + sl; e < b; e += 4 * S) {
        uint32_t M[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          M[q] = e + q * S < b ? __ldg(mask + (uint64_t)cid[e + q * S] * W + j) & cut : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (M[q]) {
            nk += __popc(M[q]);
            csa_add(P, M[q]);
          }
        }
      }
      keys += nk;
      if (threadIdx.x == 0) ents += b - a;
      // merge the sub-lanes of a warp (lanes with equal j), then the warps
#pragma unroll
      for (int off = W; off < 32; off <<= 1) {
        uint32_t Q[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) Q[q] = __shfl_xor_sync(0xffffffffu, P[q], off);
        planes_add(P, Q);
      }
      if (lane < W) {
#pragma unroll
        for (int q = 0; q < NP; ++q) sm[(wl * NP + q) * W + lane] = P[q];
      }
      __syncthreads();
      if (threadIdx.x < W) {
        for (int w8 = 1; w8 < 8; ++w8) {
          uint32_t Q[NP];
#pragma unroll
          for (int q = 0; q < NP; ++q) Q[q] = sm[(w8 * NP + q) * W + threadIdx.x];
          planes_add(P, Q);
        }
        if (whole) {
          total += planes_c2(P);
        } else {
#pragma unroll
          for (int q = 0; q < NP; ++q) fin[q * W + threadIdx.x] = P[q];
        }
      }
      if (!whole) {
        __syncthreads();
        uint32_t* row = rows + (r0 / kDensePart + 1) * (uint64_t)(32 * W);
        for (uint32_t h = threadIdx.x; h < 32u * W; h += 256) {
          uint32_t m = 0;
#pragma unroll
          for (int q = 0; q < NP; ++q) m |= ((fin[q * W + (h >> 5)] >> (h & 31u)) & 1u) << q;
          if (m) {
            const unsigned long long o = atomicAdd(row + h, m);
            total += o * m + static_cast<unsigned long long>(m) * (m - 1u) / 2u;
          }
        }
      }
      __syncthreads();
      a = b;
    }
#if BFLY_DENSE_BULK
    buf ^= 1;
#endif
  }
  dense_flush(total, keys, ents, out);
}

}  // namespace agg
}  // namespace bflyd
