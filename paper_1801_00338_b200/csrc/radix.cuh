// radix.cuh -- hand-written LSD radix sort for sm_100a, used by the graph build in place of a
// library device sort (the reference's per-list std::sort + unique in from_edges,
// graph.cpp:40-47, becomes stable device-wide sorts of (key, payload) pairs).
//
// Structure: per 8-bit digit, reduce-then-scan (no serial chain between tiles):
//   k_upsweep    per tile of 4096 keys: the digit histogram (shared-memory counters),
//                written digit-major so that
//   scan         one exclusive scan of the (256 x tiles) table (scan.cuh) gives every
//                (digit, tile) its global start;
//   k_downsweep  per tile: (1) coalesced warp-striped load of keys + payload; (2) stable rank
//                of every key inside its warp and digit -- __match_any_sync over the digits
//                gives a key's peers, the lowest peer bumps the warp's private counter; (3)
//                per-digit offsets of the warps and tile-local digit starts; (4) the tile is
//                re-ordered by digit in shared memory and written out in runs, so consecutive
//                threads store consecutive addresses of a digit's run.
// Traffic per pass: keys read twice, payload once, both written once (20 B per u32 pair)
// plus 1 KB of histogram per tile; no look-back chain across tiles (an earlier decoupled
// look-back single-sweep variant moved 16 B per pair but measured slower: DESIGN.md).
#pragma once

#include <utility>

#include "common.cuh"
#include "scan.cuh"

namespace bflyd {
namespace radix {

constexpr int kDigitBits = 8;
constexpr int kRadix = 1 << kDigitBits;
constexpr int kSweep = 512;  // CTA of both per-pass kernels: 16 warps
constexpr int kSweepWarps = kSweep / 32;
constexpr int kItems = 8;    // keys per thread (register budget: 2 CTAs of 16 warps per SM)
constexpr int kTile = kSweep * kItems;  // 4096 keys
constexpr int kMaxPasses = 8;  // 64-bit keys

struct NoVal {};

struct PassDesc {
  int shift[kMaxPasses];
  uint32_t mask[kMaxPasses];
  int passes;
};

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift, uint32_t mask) {
  return static_cast<uint32_t>(k >> shift) & mask;
}

// upsweep: the tile's digit histogram, written digit-major (hist[d * ntiles + tile]) so one
// exclusive scan of the whole table gives every (digit, tile) its global start
template <typename K>
__global__ void __launch_bounds__(kSweep) k_upsweep(const K* __restrict__ keys, uint64_t n,
                                                    int shift, uint32_t mask, uint32_t ntiles,
                                                    uint32_t* __restrict__ hist) {
  __shared__ unsigned wc[kSweepWarps][kRadix];  // one copy per warp
  const unsigned t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < kSweepWarps * kRadix; i += kSweep) (&wc[0][0])[i] = 0;
  __syncthreads();
  const uint64_t wbase = static_cast<uint64_t>(blockIdx.x) * kTile + uint64_t{w} * (kItems * 32);
  uint32_t d[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {  // all loads first
    const uint64_t idx = wbase + 32 * i + lane;
    d[i] = idx < n ? digit_of(__ldg(keys + idx), shift, mask) : 0xFFFFFFFFu;
  }
  // (plain shared atomics: pre-combining equal digits with __match_any_sync measured 2.3x
  // slower for this kernel)
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (d[i] != 0xFFFFFFFFu) atomicAdd(&wc[w][d[i]], 1u);
  __syncthreads();
  if (t < kRadix) {
    unsigned c = 0;
#pragma unroll
    for (int q = 0; q < kSweepWarps; ++q) c += wc[q][t];
    hist[uint64_t{t} * ntiles + blockIdx.x] = c;
  }
}

// downsweep: stable rank inside the tile, then the tile's keys re-ordered by digit in shared
// memory and written as runs at the scanned offsets
template <typename K, typename V, bool HAS_V>
__global__ void __launch_bounds__(kSweep, 2) k_downsweep(const K* __restrict__ kin,
                                                         K* __restrict__ kout,
                                                         const V* __restrict__ vin,
                                                         V* __restrict__ vout, uint64_t n,
                                                         int shift, uint32_t mask, uint32_t ntiles,
                                                         const uint32_t* __restrict__ offs) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);
  V* sv = reinterpret_cast<V*>(smem + sizeof(K) * kTile);
  __shared__ unsigned wcnt[kSweepWarps][kRadix];  // per-warp digit counts -> offsets in digit
  __shared__ unsigned dstart[kRadix];              // tile-local start of each digit
  __shared__ unsigned gdst[kRadix];                // global start of the digit's run here
  __shared__ unsigned wt[kRadix / 32];
  const unsigned t = threadIdx.x, lane = t & 31, w = t >> 5, full = 0xffffffffu;
  for (int i = t; i < kSweepWarps * kRadix; i += kSweep) (&wcnt[0][0])[i] = 0;
  if (t < kRadix) gdst[t] = offs[uint64_t{t} * ntiles + blockIdx.x];
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  const uint64_t wbase = base + static_cast<uint64_t>(w) * (kItems * 32);

  // (1) warp-striped load: item i of lane l is key wbase + 32 i + l
  K k[kItems];
  V v[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t idx = wbase + 32 * i + lane;
    if (idx < n) {
      k[i] = kin[idx];
      if constexpr (HAS_V) v[i] = vin[idx];
    }
  }
  // (2) stable rank inside (warp, digit). The peer sets of all items first (independent
  // match instructions in flight together), then one pass in index order: the lowest peer
  // reserves the group's slots in the warp's own counter and broadcasts the old count
  // (warp-private counters: the warp's program order is the items' index order).
  unsigned peers[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool valid = wbase + 32 * i + lane < n;
    peers[i] = __match_any_sync(full, valid ? digit_of(k[i], shift, mask) : 0xFFFFFFFFu);
  }
  uint32_t rk[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool valid = wbase + 32 * i + lane < n;
    const int leader = __ffs(peers[i]) - 1;
    uint32_t c = 0;
    if (valid && (int)lane == leader)
      c = atomicAdd(&wcnt[w][digit_of(k[i], shift, mask)], __popc(peers[i]));
    c = __shfl_sync(full, c, leader);
    rk[i] = c + __popc(peers[i] & ((1u << lane) - 1u));
  }
  __syncthreads();
  // (3) threads t < 256 own digit t: per-warp offsets inside the digit, tile-local digit starts
  if (t < kRadix) {
    unsigned cw[kSweepWarps];
#pragma unroll
    for (int q = 0; q < kSweepWarps; ++q) cw[q] = wcnt[q][t];
    unsigned run = 0;
#pragma unroll
    for (int q = 0; q < kSweepWarps; ++q) {
      wcnt[q][t] = run;
      run += cw[q];
    }
    unsigned incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(full, incl, o);
      if ((int)lane >= o) incl += y;
    }
    if (lane == 31) wt[w] = incl;
    dstart[t] = incl - run;  // (warp-local part; the other warps' totals added below)
  }
  __syncthreads();
  if (t < kRadix) {
    unsigned pre = 0;
    for (unsigned q = 0; q < w; ++q) pre += wt[q];
    dstart[t] += pre;
  }
  __syncthreads();
  // (4) re-order the tile by digit in shared memory, then write runs out
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (wbase + 32 * i + lane < n) {
      const uint32_t d = digit_of(k[i], shift, mask);
      const unsigned pos = dstart[d] + wcnt[w][d] + rk[i];
      sk[pos] = k[i];
      if constexpr (HAS_V) sv[pos] = v[i];
    }
  }
  __syncthreads();
  const unsigned tn = static_cast<unsigned>(n - base < kTile ? n - base : kTile);
  for (unsigned j = t; j < tn; j += kSweep) {
    const K key = sk[j];
    const uint32_t d = digit_of(key, shift, mask);
    const uint64_t o = static_cast<uint64_t>(gdst[d]) + (j - dstart[d]);
    kout[o] = key;
    if constexpr (HAS_V) vout[o] = sv[j];
  }
}

inline PassDesc passes_for(int begin_bit, int end_bit) {
  PassDesc pd{};
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  pd.passes = (end_bit - begin_bit + kDigitBits - 1) / kDigitBits;
  for (int p = 0; p < pd.passes; ++p) {
    pd.shift[p] = begin_bit + kDigitBits * p;
    const int w = std::min(kDigitBits, end_bit - pd.shift[p]);
    pd.mask[p] = (1u << w) - 1u;
  }
  return pd;
}

// Sorts n (key, payload) pairs by bits [begin_bit, end_bit) of the key, stably. buf(p) gives
// the (keys, payload) source of pass p (p = 0: the input) and buf(p + 1) its destination.
template <typename K, typename V, bool HAS_V, class Buf>
void sort_passes(uint64_t n, int begin_bit, int end_bit, cudaStream_t s, const char* name,
                 Buf&& buf) {
  ProfScope ps(name, s);
  if (n >= (1ull << 31)) fail(kArgument, "sort larger than 2^31-1 items");
  const PassDesc pd = passes_for(begin_bit, end_bit);
  const uint32_t ntiles = static_cast<uint32_t>((n + kTile - 1) / kTile);
  const uint64_t nh = uint64_t{kRadix} * ntiles;
  DBuf<uint32_t> hist(nh, s), offs(nh + 1, s);
  constexpr size_t smem = (sizeof(K) + (HAS_V ? sizeof(V) : 0)) * kTile;
  auto down = k_downsweep<K, V, HAS_V>;
  BFLY_CUDA(cudaFuncSetAttribute(down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int p = 0; p < pd.passes; ++p) {
    auto src = buf(p);
    auto dst = buf(p + 1);
    launch("radix_upsweep", k_upsweep<K>, ntiles, kSweep, 0, s, (const K*)src.first, n,
           pd.shift[p], pd.mask[p], ntiles, hist.p);
    scan::exclusive_sum<uint32_t>(hist.p, nh, offs.p, s, "radix_scan");
    launch("radix_downsweep", down, ntiles, kSweep, smem, s, (const K*)src.first, dst.first,
           (const V*)src.second, dst.second, n, pd.shift[p], pd.mask[p], ntiles,
           (const uint32_t*)offs.p);
  }
}

// ---- the cubwrap.cuh call shapes ---------------------------------------------------------
// (k, v) -> (kalt, valt) ping-pong; true when the result ended in the alternate buffers
template <typename K, typename V>
bool sort_pairs_db(K* k, K* kalt, V* v, V* valt, uint64_t n, int begin_bit, int end_bit,
                   cudaStream_t s, const char* name) {
  if (n == 0) return false;
  const int P = passes_for(begin_bit, end_bit).passes;
  sort_passes<K, V, true>(n, begin_bit, end_bit, s, name, [&](int p) {
    return (p & 1) ? std::make_pair(kalt, valt) : std::make_pair(k, v);
  });
  return (P & 1) != 0;
}

template <typename K>
bool sort_keys_db(K* k, K* kalt, uint64_t n, int begin_bit, int end_bit, cudaStream_t s,
                  const char* name) {
  if (n == 0) return false;
  const int P = passes_for(begin_bit, end_bit).passes;
  sort_passes<K, NoVal, false>(n, begin_bit, end_bit, s, name, [&](int p) {
    return std::make_pair((p & 1) ? kalt : k, static_cast<NoVal*>(nullptr));
  });
  return (P & 1) != 0;
}

// const input -> (kout, vout); a scratch pair only when the pass count needs it
template <typename K, typename V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit,
                int end_bit, cudaStream_t s, const char* name) {
  if (n == 0) return;
  const int P = passes_for(begin_bit, end_bit).passes;
  DBuf<K> kt;
  DBuf<V> vt;
  if (P > 1) {
    kt.alloc(n, s);
    vt.alloc(n, s);
  }
  // destinations alternate so that the last pass lands in (kout, vout)
  sort_passes<K, V, true>(n, begin_bit, end_bit, s, name, [&](int p) {
    if (p == 0) return std::make_pair(const_cast<K*>(kin), const_cast<V*>(vin));
    return ((P - p) & 1) == 0 ? std::make_pair(kout, vout) : std::make_pair(kt.p, vt.p);
  });
}

}  // namespace radix
}  // namespace bflyd
