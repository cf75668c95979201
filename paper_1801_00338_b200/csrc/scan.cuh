// scan.cuh -- hand-written device-wide exclusive scans and stable compactions (sm_100a).
//
// Reduce-then-scan over tiles of kTile elements (256 threads x 8 consecutive items):
//   pass 1  per-tile sums (or predicate counts)
//   pass 2  one CTA scans the tile sums (<= 2^20 tiles: inputs < 2^31 elements)
//   pass 3  every tile rescans its items from its offset and writes the result
// Each thread's 8 items are one 32-byte run, so a warp touches 1 KB per pass with full
// sectors. Used where a pass runs over O(m) items once or twice per call; the inputs are
// read twice, which beats a decoupled look-back's serial chain at these sizes.
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace bflyd {
namespace scan {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr uint64_t kTile = uint64_t{kThreads} * kItems;  // 2048

inline unsigned tiles_for(uint64_t n) { return static_cast<unsigned>((n + kTile - 1) / kTile); }

// Exclusive scan of n <= 2^20 u32 tile sums in one CTA; out[n] = total (u64 when the sum of
// all items may pass 2^32).
template <typename T>
__global__ void __launch_bounds__(1024) k_scan_tiles(const uint32_t* __restrict__ in, uint32_t n,
                                                     T* __restrict__ out) {
  using BS = cub::BlockScan<T, 1024>;
  __shared__ typename BS::TempStorage tmp;
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t b = min(n, threadIdx.x * per), e = min(n, b + per);
  T s = 0;
  for (uint32_t i = b; i < e; ++i) s += in[i];
  T pre, total;
  BS(tmp).ExclusiveSum(s, pre, total);
  for (uint32_t i = b; i < e; ++i) {
    const T v = in[i];
    out[i] = pre;
    pre += v;
  }
  if (threadIdx.x == 0) out[n] = total;
}

// ---- exclusive sum of u32 values -> T offsets (out[n] = total) ----------------------------
static __global__ void __launch_bounds__(kThreads) k_sum_tiles(const uint32_t* __restrict__ in, uint64_t n,
                                                        uint32_t* __restrict__ tsum) {
  const uint64_t b = blockIdx.x * kTile + threadIdx.x * uint64_t{kItems};
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (b + i < n) s += in[b + i];
  using BR = cub::BlockReduce<uint32_t, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  s = BR(tmp).Sum(s);
  if (threadIdx.x == 0) tsum[blockIdx.x] = s;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_scan_write(const uint32_t* __restrict__ in, uint64_t n,
                                                         const T* __restrict__ toff,
                                                         T* __restrict__ out) {
  const uint64_t b = blockIdx.x * kTile + threadIdx.x * uint64_t{kItems};
  uint32_t v[kItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    v[i] = b + i < n ? in[b + i] : 0u;
    s += v[i];
  }
  using BS = cub::BlockScan<T, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  T pre;
  BS(tmp).ExclusiveSum(s, pre);
  pre += toff[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (b + i < n) {
      out[b + i] = pre;
      pre += v[i];
    }
}

// out[0..n] = exclusive prefix of in[0..n), out[n] = total. Scratch from the engine pool.
template <typename T>
void exclusive_sum(const uint32_t* in, uint64_t n, T* out, cudaStream_t s, const char* name) {
  if (n == 0) {
    BFLY_CUDA(cudaMemsetAsync(out, 0, sizeof(T), s));
    return;
  }
  const unsigned tiles = tiles_for(n);
  DBuf<uint32_t> tsum(tiles, s);
  DBuf<T> toff(uint64_t{tiles} + 1, s);
  launch(name, k_sum_tiles, tiles, kThreads, 0, s, in, n, tsum.p);
  launch(name, k_scan_tiles<T>, 1, 1024, 0, s, tsum.p, tiles, toff.p);
  launch(name, k_scan_write<T>, tiles, kThreads, 0, s, in, n, toff.p, out);
  BFLY_CUDA(cudaMemcpyAsync(out + n, toff.p + tiles, sizeof(T), cudaMemcpyDeviceToDevice, s));
}

// ---- stable compaction of index-aligned u32 pairs by a predicate --------------------------
// pred(i, a[i], b[i]) -> bool; keeps the order of the kept items.
template <typename P>
__global__ void __launch_bounds__(kThreads) k_count_if(const uint32_t* __restrict__ a,
                                                       const uint32_t* __restrict__ b, uint64_t n,
                                                       P pred, uint32_t* __restrict__ tcnt) {
  const uint64_t base = blockIdx.x * kTile + threadIdx.x * uint64_t{kItems};
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (base + i < n && pred(base + i, a[base + i], b[base + i])) ++c;
  using BR = cub::BlockReduce<uint32_t, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  c = BR(tmp).Sum(c);
  if (threadIdx.x == 0) tcnt[blockIdx.x] = c;
}

template <typename P>
__global__ void __launch_bounds__(kThreads) k_compact_if(const uint32_t* __restrict__ a,
                                                         const uint32_t* __restrict__ b, uint64_t n,
                                                         P pred, const uint32_t* __restrict__ toff,
                                                         uint32_t* __restrict__ oa,
                                                         uint32_t* __restrict__ ob) {
  const uint64_t base = blockIdx.x * kTile + threadIdx.x * uint64_t{kItems};
  uint32_t va[kItems], vb[kItems];
  uint32_t keep = 0, c = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool in = base + i < n;
    va[i] = in ? a[base + i] : 0u;
    vb[i] = in ? b[base + i] : 0u;
    if (in && pred(base + i, va[i], vb[i])) {
      keep |= 1u << i;
      ++c;
    }
  }
  using BS = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  uint32_t pos;
  BS(tmp).ExclusiveSum(c, pos);
  pos += toff[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (keep >> i & 1u) {
      oa[pos] = va[i];
      ob[pos] = vb[i];
      ++pos;
    }
}

// Compacts (a, b)[0..n) into (oa, ob) and returns the kept count (one host read-back).
template <typename P>
uint32_t compact_pairs(const uint32_t* a, const uint32_t* b, uint64_t n, P pred, uint32_t* oa,
                       uint32_t* ob, cudaStream_t s, const char* name) {
  if (n == 0) return 0;
  const unsigned tiles = tiles_for(n);
  DBuf<uint32_t> tcnt(tiles, s), toff(uint64_t{tiles} + 1, s);
  launch(name, k_count_if<P>, tiles, kThreads, 0, s, a, b, n, pred, tcnt.p);
  launch(name, k_scan_tiles<uint32_t>, 1, 1024, 0, s, tcnt.p, tiles, toff.p);
  launch(name, k_compact_if<P>, tiles, kThreads, 0, s, a, b, n, pred, toff.p, oa, ob);
  uint32_t kept = 0;
  read_back(s, {{&kept, toff.p + tiles, 4}});
  return kept;
}

}  // namespace scan
}  // namespace bflyd
