// aggregate.cuh -- the degree-bucketed multiset-aggregation engine shared by the exact
// count, the all-subject local counts and the per-vertex sample kernels.
//
// A TASK is a multiset of vertex ids ("keys") given as a list of ENTRIES, each entry naming
// one contiguous SEGMENT of an adjacency array. The task's value is
//     sum over distinct keys x of C(c(x), 2)
// where c(x) is the multiplicity of x. It is accumulated with the identity
// C(c,2) = 0 + 1 + ... + (c-1): every increment contributes the counter value it found,
// so the tables never need a separate flush pass.
//
//   start tasks      task = start u (priority id), entries = forward entries u -> v,
//   (ExactSrc)       segment = N(v) after u, keys = end vertices w      (exact.cpp:29-41)
//   hub tasks        task = end vertex w, entries = all of N(w), segment = the prefix of
//   (HubSrc)         N(v) below min(k, v, w), keys = hub starts u < k. The same wedges as
//                    the start tasks of the k highest-priority starts, enumerated from the
//                    other end so the counter table is a dense k-entry array.
//   vertex samples   task = sample i, entries = N(v), segment = N(x), x in N(v), key v itself
//   (VertexSrc)      excluded                                           (local.cpp:11-21)
//
// Tables: Hash<BITS> (open addressing, insert-or-increment) for start/sample tasks,
// BitHash<BITS> (first-occurrence bitmap + repeat hash) and DirectByte / DirectSplit (dense
// 8-bit or 32/16-bit counters indexed by the key) for hub tasks.
// Buckets by task work (number of keys): tiny -> warp, keys in registers (__match_any_sync);
// small -> warp with a private shared-memory table; medium -> CTA with a shared-memory table
// (persistent CTAs, atomic queue); heavy (start tasks only) -> task split over many CTAs,
// dense per-task rows in global memory (L2 atomics), processed in waves without host syncs.
// LOCAL mode re-walks every task once its counts are final and scatters the per-vertex /
// per-edge contributions (generalised to the priority order): both
// same-side endpoints get C(c,2) per pair, the middle vertex and both wedge edges get c-1.
#pragma once
#include <string>

#include <algorithm>
#include <cstdlib>
#include <cub/block/block_scan.cuh>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "cubwrap.cuh"
#include "graph.cuh"

namespace bflyd {
namespace agg {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
#ifndef BFLY_SMALL_WARPS
#define BFLY_SMALL_WARPS 8
#endif
constexpr int kSmallWarps = BFLY_SMALL_WARPS;  // warps (one table each) per warp-table CTA
constexpr int kMedBlock = 512;
constexpr uint64_t kHeavyChunk = 32768;
constexpr uint64_t kMaxRows = 4096;  // global rows in flight per heavy wave

// Per-thread partial sums need no carry check: every partial is at most the graph's
// butterfly count, and bfly <= C(m, 2) < 2^61 for the m < 2^31 the build accepts. Carries
// are checked where partials of different threads meet (warp_sum, flush_acc).
struct Acc {
  unsigned long long v = 0;
  unsigned ovf = 0;
  __device__ __forceinline__ void add(unsigned long long x) { v += x; }
};

__device__ __forceinline__ Acc warp_sum(Acc a) {
  for (int off = 16; off > 0; off >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, a.v, off);
    unsigned o = __shfl_xor_sync(0xffffffffu, a.ovf, off);
    unsigned long long t = a.v + y;
    a.ovf |= o | (t < a.v);
    a.v = t;
  }
  return a;
}

// lane 0 of every warp adds the warp's total into *total
__device__ __forceinline__ void flush_acc(Acc a, unsigned long long* total, unsigned* ovf) {
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) {
    if (a.v) {
      unsigned long long old = atomicAdd(total, a.v);
      if (old + a.v < old) a.ovf = 1;
    }
    if (a.ovf) atomicOr(ovf, 1u);
  }
}

__device__ __forceinline__ unsigned long long c2(unsigned long long c) {
  return c < 2 ? 0ull : c * (c - 1) / 2;
}

// ---- tables -------------------------------------------------------------------------------
// Open-addressing hash of 2^BITS (key, count) slots.
template <int BITS>
struct Hash {
  static constexpr uint32_t kSlots = 1u << BITS;
  uint32_t* keys;
  uint32_t* cnt;
  __host__ __device__ static constexpr uint32_t words(uint32_t) { return 2u * kSlots; }
  __device__ __forceinline__ void bind(uint32_t* mem, uint32_t) {
    keys = mem;
    cnt = mem + kSlots;
  }
  __device__ __forceinline__ void init(uint32_t t, uint32_t stride) {
    for (uint32_t i = t; i < kSlots; i += stride) {
      keys[i] = kEmpty;
      cnt[i] = 0;
    }
  }
  // insert-or-increment; returns the count before the increment
  __device__ __forceinline__ uint32_t inc(uint32_t w) {
    uint32_t h = (w * 0x9E3779B1u) >> (32 - BITS);
    volatile uint32_t* vk = keys;
    while (true) {
      const uint32_t k = vk[h];
      if (k == w) break;
      if (k == kEmpty) {
        const uint32_t prev = atomicCAS(&keys[h], kEmpty, w);
        if (prev == kEmpty || prev == w) break;
      }
      h = (h + 1u) & (kSlots - 1u);
    }
    return atomicAdd(&cnt[h], 1u);
  }
  __device__ __forceinline__ uint32_t get(uint32_t w) const {
    uint32_t h = (w * 0x9E3779B1u) >> (32 - BITS);
    while (keys[h] != w) h = (h + 1u) & (kSlots - 1u);
    return cnt[h];
  }
  __device__ __forceinline__ void reset_all(uint32_t t, uint32_t stride) {
    uint4* k4 = reinterpret_cast<uint4*>(keys);
    uint4* c4 = reinterpret_cast<uint4*>(cnt);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u), e = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    for (uint32_t i = t; i < kSlots / 4; i += stride) {
      k4[i] = e;
      c4[i] = z;
    }
  }
  // visit f(key, count) for every occupied slot and empty the table (thread t of stride)
  template <class F>
  __device__ __forceinline__ void drain(uint32_t t, uint32_t stride, F&& f) {
    for (uint32_t s = t; s < kSlots; s += stride) {
      if (keys[s] != kEmpty) f(keys[s], cnt[s]);
      keys[s] = kEmpty;
      cnt[s] = 0;
    }
  }
};

// Open-addressing hash of 2^BITS one-word slots (key << CBITS | count): half the footprint of
// Hash<BITS>. Valid while every key is below 2^(32 - CBITS) - 1 and every count below
// 2^CBITS (a task of fewer than 2^CBITS keys); the caller checks both.
template <int BITS, int CBITS>
struct PackedHash {
  static constexpr uint32_t kSlots = 1u << BITS;
  static constexpr uint32_t kMask = (1u << CBITS) - 1u;
  uint32_t* slot;
  __host__ __device__ static constexpr uint32_t words(uint32_t) { return kSlots; }
  __device__ __forceinline__ void bind(uint32_t* mem, uint32_t) { slot = mem; }
  __device__ __forceinline__ void init(uint32_t t, uint32_t stride) {
    for (uint32_t i = t; i < kSlots; i += stride) slot[i] = kEmpty;
  }
  __device__ __forceinline__ uint32_t find_or_insert(uint32_t w) {
    uint32_t h = (w * 0x9E3779B1u) >> (32 - BITS);
    volatile uint32_t* vs = slot;
    while (true) {
      const uint32_t v = vs[h];
      if ((v >> CBITS) == w && v != kEmpty) break;
      if (v == kEmpty) {
        const uint32_t prev = atomicCAS(&slot[h], kEmpty, w << CBITS);
        if (prev == kEmpty || (prev >> CBITS) == w) break;
      }
      h = (h + 1u) & (kSlots - 1u);
    }
    return h;
  }
  // insert-or-increment; returns the count before the increment
  __device__ __forceinline__ uint32_t inc(uint32_t w) {
    const uint32_t h = find_or_insert(w);
    return atomicAdd(&slot[h], 1u) & kMask;
  }
  __device__ __forceinline__ uint32_t get(uint32_t w) const {
    uint32_t h = (w * 0x9E3779B1u) >> (32 - BITS);
    while (true) {
      const uint32_t v = slot[h];
      if (v != kEmpty && (v >> CBITS) == w) return v & kMask;
      h = (h + 1u) & (kSlots - 1u);
    }
  }
  __device__ __forceinline__ void reset_all(uint32_t t, uint32_t stride) {
    uint4* s4 = reinterpret_cast<uint4*>(slot);
    const uint4 e = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    for (uint32_t i = t; i < kSlots / 4; i += stride) s4[i] = e;
  }
  template <class F>
  __device__ __forceinline__ void drain(uint32_t t, uint32_t stride, F&& f) {
    for (uint32_t i = t; i < kSlots; i += stride) {
      const uint32_t v = slot[i];
      if (v != kEmpty) f(v >> CBITS, v & kMask);
      slot[i] = kEmpty;
    }
  }
};

// Striped placement of small hub keys in packed tables (BFLY_HUB_STRIPE=1; measured slower, off): key u of a table
// of W words goes to word u mod W, sub-field u div W, so consecutive hub ids -- the ascending
// runs a hub-prefix segment holds -- land in consecutive words (different banks, different
// addresses) instead of sharing one word. u div W by a multiply-high with ceil(2^32 / W):
// exact for u, W < 2^16 (the error u (m W - 2^32) / 2^32 stays below u / 2^32 < 1 / W).
#ifndef BFLY_HUB_STRIPE
#define BFLY_HUB_STRIPE 0
#endif
struct Stripe {
  uint32_t W, magic;
  __device__ __forceinline__ void set(uint32_t w) {
    W = w;
    magic = w ? 0xFFFFFFFFu / w + 1u : 0u;
  }
  __device__ __forceinline__ uint32_t sub(uint32_t u) const { return __umulhi(u, magic); }
  __device__ __forceinline__ uint32_t word(uint32_t u, uint32_t q) const { return u - q * W; }
};

// Keys in [0, K), K < 2^16 (hub ids): a bitmap absorbs first occurrences (count 0 -> 1,
// contribution 0) and an open-addressing hash holds only keys seen twice or more. A hash slot
// packs the key and its repeat count in one word (key << 16 | c - 1; tasks have < 2^16 keys),
// so the table is K/32 + 2^BITS words.
template <int BITS>
struct BitHash {
  static constexpr uint32_t kSlots = 1u << BITS;
  uint32_t* bits;
  uint32_t* slot;
  uint32_t K;
  Stripe st;  // BFLY_HUB_STRIPE: key u -> bit u div Wb of word u mod Wb
  // bitmap words, padded to whole uint4s (mem is 16-byte aligned)
  __host__ __device__ static constexpr uint32_t bwords(uint32_t k) { return ((k + 31) / 32 + 3) & ~3u; }
  __host__ __device__ static constexpr uint32_t words(uint32_t kk) {
    return bwords(kk & 0xFFFFu) + kSlots;
  }
  __device__ __forceinline__ void bind(uint32_t* mem, uint32_t kk) {
    const uint32_t k = kk & 0xFFFFu;
    K = k;
    bits = mem;
    slot = mem + bwords(k);
    st.set(bwords(k));
  }
  __device__ __forceinline__ void init(uint32_t t, uint32_t stride) {
    for (uint32_t i = t; i < bwords(K); i += stride) bits[i] = 0;
    for (uint32_t i = t; i < kSlots; i += stride) slot[i] = kEmpty;
  }
  // slot of a repeated key u (inserted with count 0 if new)
  __device__ __forceinline__ uint32_t find_or_insert(uint32_t u) {
    uint32_t h = (u * 0x9E3779B1u) >> (32 - BITS);
    volatile uint32_t* vs = slot;
    while (true) {
      const uint32_t v = vs[h];
      if ((v >> 16) == u) break;
      if (v == kEmpty) {
        const uint32_t prev = atomicCAS(&slot[h], kEmpty, u << 16);
        if (prev == kEmpty || (prev >> 16) == u) break;
      }
      h = (h + 1u) & (kSlots - 1u);
    }
    return h;
  }
  __device__ __forceinline__ uint32_t inc(uint32_t u) {
#if BFLY_HUB_STRIPE
    const uint32_t q = st.sub(u), bit = 1u << q;
    if (!(atomicOr(&bits[st.word(u, q)], bit) & bit)) return 0;  // first occurrence
#else
    const uint32_t bit = 1u << (u & 31);
    if (!(atomicOr(&bits[u >> 5], bit) & bit)) return 0;  // first occurrence
#endif
    const uint32_t h = find_or_insert(u);
    return (atomicAdd(&slot[h], 1u) & 0xFFFFu) + 1u;
  }
  // n occurrences at once; returns the sum of the n old counts. A first occurrence is
  // linearised at the bitmap update, the other n-1 at the slot update (which may interleave
  // with another warp's: its returned field is the count they found).
  __device__ __forceinline__ uint32_t add(uint32_t u, uint32_t n) {
#if BFLY_HUB_STRIPE
    const uint32_t q = st.sub(u), bit = 1u << q;
    const bool seen = atomicOr(&bits[st.word(u, q)], bit) & bit;
#else
    const uint32_t bit = 1u << (u & 31);
    const bool seen = atomicOr(&bits[u >> 5], bit) & bit;
#endif
    const uint32_t m = seen ? n : n - 1u;  // increments that go to the slot
    if (m == 0) return 0;
    const uint32_t h = find_or_insert(u);
    const uint32_t f = (atomicAdd(&slot[h], m) & 0xFFFFu) + 1u;  // count before them
    return m * f + m * (m - 1u) / 2u;
  }
  __device__ __forceinline__ uint32_t get(uint32_t u) const {
    uint32_t h = (u * 0x9E3779B1u) >> (32 - BITS);
    while (true) {
      const uint32_t v = slot[h];
      if ((v >> 16) == u) return (v & 0xFFFFu) + 1u;
      if (v == kEmpty) return 1u;
      h = (h + 1u) & (kSlots - 1u);
    }
  }
  // whole-table reset, 16 bytes per store: bitmap to 0, slots to empty
  __device__ __forceinline__ void reset_all(uint32_t t, uint32_t stride) {
    uint4* b4 = reinterpret_cast<uint4*>(bits);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u), e = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    for (uint32_t i = t; i < bwords(K) / 4; i += stride) b4[i] = z;
    uint4* s4 = reinterpret_cast<uint4*>(slot);
    for (uint32_t i = t; i < kSlots / 4; i += stride) s4[i] = e;
  }
  template <class F>
  __device__ __forceinline__ void drain(uint32_t t, uint32_t stride, F&& f) {
    for (uint32_t i = t; i < kSlots; i += stride) {
      const uint32_t v = slot[i];
      if (v != kEmpty) f(v >> 16, (v & 0xFFFFu) + 1u);
      slot[i] = kEmpty;
    }
    uint4* b4 = reinterpret_cast<uint4*>(bits);  // first occurrences: clear the bitmap whole
    for (uint32_t i = t; i < bwords(K) / 4; i += stride) b4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
};

// Dense counters for hub keys u in [0, K): 32-bit for u < K1, 16-bit pairs packed in 32-bit
// words for u >= K1, plus a bitmap of touched keys. A key's multiplicity c(u, w) is at most
// deg(u), and K1 is chosen (exact.cu) so that every u >= K1 has deg(u) < 65536: a 16-bit
// counter never carries into its neighbour. K1 is a multiple of 32.
struct DirectSplit {
  uint32_t* c32;
  uint32_t* c16;  // word j holds keys K1 + 2j (low half) and K1 + 2j + 1 (high half)
                  // (BFLY_HUB_STRIPE: keys K1 + j and K1 + j + W16 instead)
  uint32_t K, K1;
  Stripe st;
  // geometry kk = K | K1 << 16 (K <= 65535, K1 a multiple of 32); the 16-bit region is padded
  // to whole uint4s. No touched bitmap: the drain scans the counters 4 words at a time.
  __host__ __device__ static constexpr uint32_t w16(uint32_t kk) {
    return ((((kk & 0xFFFFu) - (kk >> 16) + 1) / 2) + 3) & ~3u;
  }
  __host__ __device__ static constexpr uint32_t words(uint32_t kk) { return (kk >> 16) + w16(kk); }
  __device__ __forceinline__ void bind(uint32_t* mem, uint32_t kk) {
    K = kk & 0xFFFFu;
    K1 = kk >> 16;
    c32 = mem;
    c16 = mem + K1;
    st.set(w16(kk));
  }
  // (word, shift) of 16-bit key j = u - K1
  __device__ __forceinline__ void at16(uint32_t j, uint32_t& w, uint32_t& sh) const {
#if BFLY_HUB_STRIPE
    const uint32_t q = st.sub(j);
    w = st.word(j, q);
    sh = q << 4;
#else
    w = j >> 1;
    sh = (j & 1u) << 4;
#endif
  }
  __device__ __forceinline__ void init(uint32_t t, uint32_t stride) {
    const uint32_t nw = K1 + w16(K | (K1 << 16));
    for (uint32_t i = t; i < nw; i += stride) c32[i] = 0;
  }
  __device__ __forceinline__ uint32_t inc(uint32_t u) {
    uint32_t old;
    if (u < K1) {
      old = atomicAdd(&c32[u], 1u);
    } else {
      uint32_t w, sh;
      at16(u - K1, w, sh);
      old = (atomicAdd(&c16[w], 1u << sh) >> sh) & 0xFFFFu;
    }
    return old;
  }
  // n increments at once: sum of the n old values (a 32-bit counter's sum is bounded by the
  // task's C(keys, 2): callers accumulate it in 64 bits)
  __device__ __forceinline__ unsigned long long add(uint32_t u, uint32_t n) {
    uint32_t old;
    if (u < K1) {
      old = atomicAdd(&c32[u], n);
    } else {
      uint32_t w, sh;
      at16(u - K1, w, sh);
      old = (atomicAdd(&c16[w], n << sh) >> sh) & 0xFFFFu;
    }
    return static_cast<unsigned long long>(n) * old + n * (n - 1u) / 2u;
  }
  __device__ __forceinline__ uint32_t get(uint32_t u) const {
    if (u < K1) return c32[u];
    uint32_t w, sh;
    at16(u - K1, w, sh);
    return (c16[w] >> sh) & 0xFFFFu;
  }
  // (measured: the conditional zeroing of drain beats whole-table stores for these tasks)
  __device__ __forceinline__ void reset_all(uint32_t t, uint32_t stride) {
    drain(t, stride, [](uint32_t, uint32_t) {});
  }
  // visit f(key, count) for every nonzero counter and zero the table
  template <class F>
  __device__ __forceinline__ void drain(uint32_t t, uint32_t stride, F&& f) {
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    uint4* a4 = reinterpret_cast<uint4*>(c32);
    for (uint32_t i = t; i < K1 / 4; i += stride) {
      const uint4 v = a4[i];
      if ((v.x | v.y | v.z | v.w) == 0) continue;
      const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (q[j]) f(i * 4 + j, q[j]);
      a4[i] = z;
    }
    uint4* b4 = reinterpret_cast<uint4*>(c16);
    const uint32_t n4 = w16(K | (K1 << 16)) / 4;
    for (uint32_t i = t; i < n4; i += stride) {
      const uint4 v = b4[i];
      if ((v.x | v.y | v.z | v.w) == 0) continue;
      const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t c = (q[j] >> (16 * h)) & 0xFFFFu;
#if BFLY_HUB_STRIPE
          if (c) f(K1 + h * st.W + (i * 4 + j), c);
#else
          if (c) f(K1 + 2 * (i * 4 + j) + h, c);
#endif
        }
      b4[i] = z;
    }
  }
};

// Dense 8-bit counters for hub keys u in [0, K), four per 32-bit word, for tasks with fewer
// than 256 entries (c(u, w) <= entries of w < 256, so a byte never carries into its
// neighbour). A quarter of a 32-bit table's footprint -> more resident CTAs.
struct DirectByte {
  uint32_t* c8;  // word j holds keys 4j .. 4j+3 (byte u & 3)
                 // (BFLY_HUB_STRIPE: keys j + b W, byte b, W = words(K))
  uint32_t K;
  Stripe st;
  // no touched bitmap: the drain scans the K bytes 16 at a time (K/16 uint4 loads per task,
  // cheaper than a bitmap update on every first occurrence)
  __host__ __device__ static constexpr uint32_t groups(uint32_t k) { return (k + 127) / 128; }
  __host__ __device__ static constexpr uint32_t words(uint32_t kk) {
    return groups(kk & 0xFFFFu) * 32;
  }
  __device__ __forceinline__ void bind(uint32_t* mem, uint32_t kk) {
    K = kk & 0xFFFFu;
    c8 = mem;
    st.set(words(K));
  }
  __device__ __forceinline__ void init(uint32_t t, uint32_t stride) {
    for (uint32_t i = t; i < words(K); i += stride) c8[i] = 0;
  }
  __device__ __forceinline__ void at(uint32_t u, uint32_t& w, uint32_t& sh) const {
#if BFLY_HUB_STRIPE
    const uint32_t q = st.sub(u);
    w = st.word(u, q);
    sh = q << 3;
#else
    w = u >> 2;
    sh = (u & 3u) << 3;
#endif
  }
  __device__ __forceinline__ uint32_t inc(uint32_t u) {
    uint32_t w, sh;
    at(u, w, sh);
    const uint32_t old = (atomicAdd(&c8[w], 1u << sh) >> sh) & 0xFFu;
    return old;
  }
  __device__ __forceinline__ uint32_t add(uint32_t u, uint32_t n) {
    uint32_t w, sh;
    at(u, w, sh);
    const uint32_t old = (atomicAdd(&c8[w], n << sh) >> sh) & 0xFFu;
    return n * old + n * (n - 1u) / 2u;
  }
  __device__ __forceinline__ uint32_t get(uint32_t u) const {
    uint32_t w, sh;
    at(u, w, sh);
    return (c8[w] >> sh) & 0xFFu;
  }
  // zero the whole table (counting runs: nothing to read back)
  __device__ __forceinline__ void reset_all(uint32_t t, uint32_t stride) {
    uint4* c4 = reinterpret_cast<uint4*>(c8);
    for (uint32_t i = t; i < groups(K) * 8; i += stride) c4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // visit f(key, count) for every nonzero counter (16 per uint4) and zero the table
  template <class F>
  __device__ __forceinline__ void drain(uint32_t t, uint32_t stride, F&& f) {
    uint4* c4 = reinterpret_cast<uint4*>(c8);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t i = t; i < groups(K) * 8; i += stride) {
      const uint4 v = c4[i];
      if ((v.x | v.y | v.z | v.w) == 0) continue;
      const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t c = (q[j] >> (8 * b)) & 0xFFu;
#if BFLY_HUB_STRIPE
          if (c) f(b * st.W + i * 4 + j, c);
#else
          if (c) f(i * 16 + j * 4 + b, c);
#endif
        }
      c4[i] = z;
    }
  }
};

// ---- task sources ---------------------------------------------------------------------
// kVec4: the counting runs walk this source's segments with 16-byte loads (the vectorised
// walks below); its padj must be the 16-byte aligned, padded priority adjacency.
#ifndef BFLY_VEC4_HUB
#define BFLY_VEC4_HUB 1
#endif
#ifndef BFLY_VEC4_EXACT
#define BFLY_VEC4_EXACT 0
#endif
// Start tasks on the priority CSR; task = start u.
struct ExactSrc {
  const uint64_t* poff;
  const uint32_t* padj;
  const uint2* fseg;  // per forward entry: (start, length) of the wedge suffix (prio_plan)
  const uint64_t* fwd;
  __device__ __forceinline__ void entries(uint32_t u, uint64_t& e0, uint64_t& e1) const {
    e0 = fwd[u];
    e1 = poff[u + 1];
  }
  __device__ __forceinline__ uint32_t seg(uint32_t, uint64_t e, const uint32_t*& p) const {
    const uint2 sg = __ldg(fseg + e);
    p = padj + sg.x;
    return sg.y;
  }
  static constexpr bool kExcl = false;
  static constexpr bool kNarrowScan = false;
  static constexpr bool kVec4 = BFLY_VEC4_EXACT;  // segments of 1-3 keys in the small buckets
  __device__ __forceinline__ uint32_t excl(uint32_t) const { return kEmpty; }
};

// Hub tasks on the priority CSR; task = end vertex w, keys = hub starts u < k.
struct HubSrc {
  const uint64_t* poff;
  const uint32_t* padj;
  const uint16_t* hlen;  // per entry (w -> v): |{u in N(v) : u < min(k, v, w)}|
  const uint32_t* hpst;  // per entry with hlen > 0: poff[v] (no dependent padj[e] load)
  __device__ __forceinline__ void entries(uint32_t w, uint64_t& e0, uint64_t& e1) const {
    e0 = poff[w];
    e1 = poff[w + 1];
  }
  __device__ __forceinline__ uint32_t seg(uint32_t, uint64_t e, const uint32_t*& p) const {
    p = padj + __ldg(hpst + e);  // garbage (never dereferenced) where hlen is 0
    return __ldg(hlen + e);
  }
  static constexpr bool kExcl = false;
  static constexpr bool kNarrowScan = true;  // hlen < 2^15 (k <= kHubMax < 2^15)
  static constexpr bool kVec4 = BFLY_VEC4_HUB;  // prefixes of 13-23 keys on average: uint4 loads
  __device__ __forceinline__ uint32_t excl(uint32_t) const { return kEmpty; }
};

// Vertex samples on the canonical CSRs; task = sample index, gids[i] = global vertex id.
struct VertexSrc {
  const uint64_t* gids;
  uint32_t L;
  const uint64_t* loff;
  const uint32_t* ladj;
  const uint64_t* roff;
  const uint32_t* radj;
  __device__ __forceinline__ void entries(uint32_t i, uint64_t& e0, uint64_t& e1) const {
    const uint64_t v = gids[i];
    if (v < L) {
      e0 = loff[v];
      e1 = loff[v + 1];
    } else {
      e0 = roff[v - L];
      e1 = roff[v - L + 1];
    }
  }
  __device__ __forceinline__ uint32_t seg(uint32_t i, uint64_t e, const uint32_t*& p) const {
    const uint64_t v = gids[i];
    if (v < L) {
      const uint32_t x = ladj[e];  // right vertex; its list holds left ids
      p = radj + roff[x];
      return static_cast<uint32_t>(roff[x + 1] - roff[x]);
    }
    const uint32_t x = radj[e];
    p = ladj + loff[x];
    return static_cast<uint32_t>(loff[x + 1] - loff[x]);
  }
  static constexpr bool kExcl = true;
  static constexpr bool kNarrowScan = false;
  static constexpr bool kVec4 = false;
  __device__ __forceinline__ uint32_t excl(uint32_t i) const {
    const uint64_t v = gids[i];
    return static_cast<uint32_t>(v < L ? v : v - L);
  }
};

// Same-side vertex pairs on the priority CSR; task = start u, entries = ALL of N(u),
// segment = N(v) after u (apair per entry, pairs.cu), keys = w > u on u's side. c(w) is the
// full |N(u) & N(w)|, and every unordered same-side pair is the task of its higher-priority
// end exactly once: the pair-moment pass of the variance tables (reference oracle.cpp:60-94).
struct PairSrc {
  const uint64_t* poff;
  const uint32_t* padj;
  const uint2* aseg;  // per entry u -> v: (start, length) of N(v) after u
  __device__ __forceinline__ void entries(uint32_t u, uint64_t& e0, uint64_t& e1) const {
    e0 = poff[u];
    e1 = poff[u + 1];
  }
  __device__ __forceinline__ uint32_t seg(uint32_t, uint64_t e, const uint32_t*& p) const {
    const uint2 sg = __ldg(aseg + e);
    p = padj + sg.x;
    return sg.y;
  }
  static constexpr bool kExcl = false;
  static constexpr bool kNarrowScan = false;
  static constexpr bool kVec4 = false;
  __device__ __forceinline__ uint32_t excl(uint32_t) const { return kEmpty; }
};

// Sources whose final key multiplicities feed the pair moments (drained, not just reset)
template <class S>
constexpr bool kMoments = false;
template <>
constexpr bool kMoments<PairSrc> = true;

// Per-thread 128-bit sums of C(c,3) and C(c,4) over distinct keys with final multiplicity c
// (c < 2^32: C(c,3) < 2^94, C(c,4) < 2^126).
struct Mom {
  unsigned __int128 s3 = 0, s4 = 0;
  __device__ __forceinline__ void add(uint32_t c) {
    if (c < 3) return;
    unsigned long long x = c, y = c - 1u, z = c - 2u;
    if (x % 3 == 0) x /= 3;  // one of three consecutive integers is a multiple of 3
    else if (y % 3 == 0) y /= 3;
    else z /= 3;
    if ((x & 1) == 0) x >>= 1;  // dividing by 3 keeps parity: one of x, y is even
    else y >>= 1;
    const unsigned __int128 c3 = (unsigned __int128)(x * y) * z;  // x*y < 2^63
    s3 += c3;
    s4 += (c3 * (c - 3u)) >> 2;  // C(c,4) = C(c,3) (c-3) / 4, exact
  }
};

__device__ __forceinline__ unsigned __int128 shfl_xor_u128(unsigned __int128 v, int off) {
  const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, off);
  const unsigned long long hi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(v >> 64), off);
  return ((unsigned __int128)hi << 64) | lo;
}

// 128-bit add into (lo, hi) words: the low word's carry-out of each add goes to the high word
__device__ __forceinline__ void atomic_add_u128(unsigned long long* p, unsigned __int128 v) {
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  unsigned long long carry = 0;
  if (lo) {
    const unsigned long long old = atomicAdd(p, lo);
    carry = old + lo < old;
  }
  if (hi + carry) atomicAdd(p + 1, hi + carry);
}

// whole warp: lane 0 adds the warp's sums into mom[0..1] (s3) and mom[2..3] (s4)
__device__ __forceinline__ void flush_mom(Mom m, unsigned long long* mom) {
  for (int off = 16; off > 0; off >>= 1) {
    m.s3 += shfl_xor_u128(m.s3, off);
    m.s4 += shfl_xor_u128(m.s4, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (m.s3) atomic_add_u128(mom, m.s3);
    if (m.s4) atomic_add_u128(mom + 2, m.s4);
  }
}

// per-vertex / per-edge outputs of LOCAL mode (priority ids / canonical edge ids)
// vcnt per priority id; pacc per priority-CSR entry (both directions of an edge are folded
// into the canonical edge counts after the pass, local.cu): keys of one segment are
// consecutive entries of N(v), so their per-edge atomics hit consecutive addresses
struct LocalOut {
  unsigned long long* vcnt;
  unsigned long long* pacc;
  const uint32_t* peid;
  const uint32_t* padj;
  // hub runs: per-block private rows for the C(c,2) of keys < kstride (every hub task adds
  // to the same few thousand hub counters; private rows avoid the L2 hot spots), summed
  // into vcnt after the run
  unsigned long long* krow = nullptr;
  uint32_t kstride = 0;
  // pair-moment runs (kMoments sources): 128-bit sums of C(c,3) at [0,2), C(c,4) at [2,4)
  unsigned long long* mom = nullptr;
};
constexpr uint32_t kKeyRows = 148 * 8;  // >= the grid of every k_small / k_medium launch

__device__ __forceinline__ void add_key(const LocalOut& lo, uint32_t key, unsigned long long v) {
  if (lo.krow && key < lo.kstride) atomicAdd(&lo.krow[(uint64_t)blockIdx.x * lo.kstride + key], v);
  else atomicAdd(&lo.vcnt[key], v);
}

// one wedge (task -> entry e -> element at pe) with final key multiplicity c
__device__ __forceinline__ void emit_wedge(const LocalOut& lo, uint64_t e, const uint32_t* pe,
                                           uint32_t c) {
  if (c >= 2) {
    const unsigned long long x = c - 1;
    atomicAdd(&lo.vcnt[lo.padj[e]], x);
    if (lo.pacc) {  // (null: per-vertex counts only)
      atomicAdd(&lo.pacc[e], x);
      atomicAdd(&lo.pacc[pe - lo.padj], x);
    }
  }
}

// Segment-aggregated form for the walkers: the per-element part (the wedge's second edge)
// is emitted per key; the middle vertex and the first edge are the same for every key of an
// entry, so their c-1 contributions are summed over each run of equal entries in a warp
// round (segmented shuffle scan) and emitted once per run.
__device__ __forceinline__ unsigned long long emit_key(const LocalOut& lo, const uint32_t* pe,
                                                       uint32_t c) {
  if (c < 2) return 0ull;
  const unsigned long long x = c - 1;
  // per-vertex counts only (pacc null): the wedge's second edge needs nothing, and a walk
  // then issues no global atomic per key -- only one per run of equal entries (EmitEntry)
  if (lo.pacc) atomicAdd(&lo.pacc[pe - lo.padj], x);
  return x;
}
struct EmitEntry {
  LocalOut lo;
  __device__ __forceinline__ void operator()(uint64_t e, unsigned long long x) const {
    atomicAdd(&lo.vcnt[lo.padj[e]], x);
    if (lo.pacc) atomicAdd(&lo.pacc[e], x);
  }
};
// all 32 lanes of a walk round: B = the round's segment-start mask (bit b set: a new entry
// starts at lane b + 1), valid lanes a prefix. One call of g(entry, run sum) per run of
// equal entries with a nonzero sum: a plain warp prefix sum, and each run's tail subtracts
// the prefix at the previous run's tail.
template <class G>
__device__ __forceinline__ void seg_emit(bool valid, unsigned B, uint64_t entry,
                                         unsigned long long x, const G& g) {
  const unsigned full = 0xffffffffu, lane = threadIdx.x & 31;
  if (!valid) x = 0;
  if (!__any_sync(full, x != 0)) return;
  unsigned long long incl = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long y = __shfl_up_sync(full, incl, off);
    if ((int)lane >= off) incl += y;
  }
  const unsigned vm = __ballot_sync(full, valid);
  const unsigned lastv = 31u - __clz(vm);
  const unsigned lt = B & ((1u << lane) - 1u);
  const int p = lt ? 31 - __clz(lt) : -1;  // previous run's tail lane
  const unsigned long long before = __shfl_sync(full, incl, p < 0 ? 0 : p);
  const unsigned long long sum = incl - (p < 0 ? 0ull : before);
  if (valid && (((B >> lane) & 1u) || lane == lastv) && sum) g(entry, sum);
}

// position of the k-th (0-based) set bit of m (k < popc(m)): five branch-free halving steps
// (__fns lowers to a much longer sequence)
__device__ __forceinline__ unsigned nth_set_bit(unsigned m, unsigned k) {
  unsigned pos = 0;
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    const unsigned c = __popc(m & ((1u << sh) - 1u));
    const bool up = k >= c;
    k -= up ? c : 0u;
    m = up ? (m >> sh) : m;
    pos += up ? sh : 0u;
  }
  return pos;
}

// Warp-combined updates (BFLY_HUB_MATCH=1, hub counting runs): the lanes of a walk round that
// hold the same key are found with one __match_any_sync, and only the lowest of them calls
// f(key, n) with the multiplicity n -- one table update per distinct key per round instead of
// n serialised same-address atomics.
#ifndef BFLY_HUB_MATCH
#define BFLY_HUB_MATCH 0
#endif
template <class F>
struct Combine {
  F f;
};
template <class F>
struct IsCombine : std::false_type {};
template <class F>
struct IsCombine<Combine<F>> : std::true_type {};

template <class F>
__device__ __forceinline__ void combined_call(F& f, bool ok, uint32_t key) {
  const unsigned act = __ballot_sync(0xffffffffu, ok);
  if (ok) {
    const unsigned mm = __match_any_sync(act, key);
    if ((int)(threadIdx.x & 31) == __ffs(mm) - 1) f.f(key, static_cast<uint32_t>(__popc(mm)));
  }
}

// ---- flattened walk of one task's entry range by one warp --------------------------------
// f(key, p_elem, e): key = element, p_elem = its address, e = entry index.
struct NoSeg {
  static constexpr bool kActive = false;
  __device__ __forceinline__ void operator()(uint64_t, unsigned long long) const {}
};
template <class G>
struct Seg {
  static constexpr bool kActive = true;
  G g;
  __device__ __forceinline__ void operator()(uint64_t e, unsigned long long x) const { g(e, x); }
};

// f(key, p_elem, e) per element; with an active Seg functor f returns a value that is summed
// per run of equal entries in each round and passed to seg(e, sum)
// (NEED_E = false: f ignores its entry argument and the walk skips computing it)
template <bool NEED_E = true, int kU = 4, class Src, class F, class SG = NoSeg>
__device__ __forceinline__ void warp_walk_range(const Src& src, uint32_t task, uint64_t e0,
                                                uint64_t e1, F&& f, const SG& seg = SG{}) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const uint32_t ex = src.excl(task);
  for (uint64_t eb = e0; eb < e1; eb += 32) {
    const uint64_t e = eb + lane;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    // compact the non-empty segments into the low lanes (once per 32 entries)
    const unsigned nz = __ballot_sync(full, len > 0);
    if (!nz) continue;
    const unsigned ne = __popc(nz);
    // (no empty segment below the last non-empty one: the compaction is the identity)
    const unsigned srcl = (nz & (nz + 1u)) == 0u ? lane : (lane < ne ? nth_set_bit(nz, lane) : 0u);
    uint32_t clen = __shfl_sync(full, len, srcl);
    const unsigned long long cp =
        __shfl_sync(full, reinterpret_cast<unsigned long long>(p), srcl);
    if (lane >= ne) clen = 0;
    uint32_t incl = clen;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(full, incl, off);
      if ((int)lane >= off) incl += y;
    }
    const uint32_t tot = __shfl_sync(full, incl, 31);
    const uint32_t excl = incl - clen;
    const unsigned long long basep = cp - 4ull * excl;  // element idx -> basep + 4*idx
    // owner of element r + lane = first compacted segment + number of segment starts in
    // (r, r + lane]: one OR-reduction of start bits per 32 elements, no search. Each
    // compacted segment's start bit is fixed for the batch: its round and bit, once.
    const uint32_t srd = (lane < ne && excl > 0) ? (excl - 1) >> 5 : 0xFFFFFFFFu;
    const unsigned sbit = 1u << ((excl - 1) & 31);
    uint32_t own0 = 0;  // (kU rounds per iteration: independent key loads in flight)
    for (uint32_t r = 0; r < tot; r += 32 * kU) {
      const uint32_t* pes[kU];
      unsigned olane[kU], Bs[kU];
      bool ok[kU];
      const uint32_t nr = (tot - r + 31) / 32;  // rounds left (warp-uniform)
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        ok[j] = false;
        pes[j] = nullptr;
        olane[j] = 0;
        Bs[j] = 0;
        if ((uint32_t)j >= nr) continue;
        const uint32_t rr = r + 32 * j;
        const unsigned B = __reduce_or_sync(full, srd == (rr >> 5) ? sbit : 0u);
        Bs[j] = B;
        const uint32_t own = own0 + __popc(B & ((1u << lane) - 1u));
        const unsigned long long bp = __shfl_sync(full, basep, own);
        if constexpr (NEED_E || SG::kActive) olane[j] = __shfl_sync(full, srcl, own);
        ok[j] = rr + lane < tot;
        pes[j] = reinterpret_cast<const uint32_t*>(bp) + (rr + lane);
        own0 += __popc(B);
      }
      uint32_t ws[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) ws[j] = ok[j] ? __ldg(pes[j]) : 0u;
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        if constexpr (SG::kActive) {
          unsigned long long x = 0;
          if (ok[j] && (!Src::kExcl || ws[j] != ex)) x = f(ws[j], pes[j], eb + olane[j]);
          if ((uint32_t)j < nr) seg_emit(ok[j], Bs[j], eb + olane[j], x, seg);
        } else {
          if constexpr (IsCombine<std::decay_t<F>>::value) combined_call(f, ok[j], ws[j]);
          else if (ok[j] && (!Src::kExcl || ws[j] != ex)) f(ws[j], pes[j], eb + olane[j]);
        }
      }
    }
  }
}

// ---- vectorised walks (counting runs): 16-byte adjacency loads ---------------------------------
// The walks above place ONE 4-byte key per lane and round, so the owner mapping (start-bit
// reduction, popcounts, shuffles of the segment base) is paid per key. Here a segment is cut
// into the aligned 16-byte chunks that cover it and the flattened space is chunks: a lane
// loads a uint4 (ld.global.nc.v4) and feeds up to four keys to the table, the words of the
// first and last chunk that lie outside the segment are masked by the segment's [lo, hi)
// range in the word space of the batch. One owner mapping serves up to 128 keys of a warp.
// padj is 16-byte aligned and padded by 4 words (priority.cu), so the rounded-out chunks stay
// inside the allocation. f(key) per element; sources with kVec4 only.
#ifndef BFLY_VEC4
#define BFLY_VEC4 1
#endif
#ifndef BFLY_VEC4_KU
#define BFLY_VEC4_KU 2
#endif
// Measured on config 2 (kernels alone, profiles/r2_ab_vec4.txt): the CTA walks gain (hub
// medium 0.78 -> 0.64 ms with one chunk round per iteration -- two spill at its 32-register
// budget --, medium-wide 0.88 -> 0.73, split 0.14 -> 0.13); the warp tables do not (small-A
// 2.27 -> 2.23 / 2.44 ms with one / two rounds, small-B 1.48 -> 1.52 / 1.49: their cost is the
// per-task steps and the table updates, not the owner mapping), nor the start path, whose
// segments hold 1-3 keys in the small buckets (exact kernels 1.96 -> 2.25 ms).
#ifndef BFLY_VEC4_SMALL
#define BFLY_VEC4_SMALL 0
#endif
__device__ __forceinline__ uint32_t u4_word(const uint4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}

template <int kU = BFLY_VEC4_KU, class Src, class F>
__device__ __forceinline__ void warp_walk_range_v4(const Src& src, uint32_t task, uint64_t e0,
                                                   uint64_t e1, F&& f) {
  static_assert(Src::kVec4 && !Src::kExcl, "aligned, padded adjacency without an excluded key");
  const unsigned lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  for (uint64_t eb = e0; eb < e1; eb += 32) {
    const uint64_t e = eb + lane;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    const unsigned nz = __ballot_sync(full, len > 0);
    if (!nz) continue;
    const unsigned ne = __popc(nz);
    const unsigned srcl = (nz & (nz + 1u)) == 0u ? lane : (lane < ne ? nth_set_bit(nz, lane) : 0u);
    uint32_t clen = __shfl_sync(full, len, srcl);
    const uint32_t po = __shfl_sync(full, static_cast<uint32_t>(p - src.padj), srcl);  // word offset
    if (lane >= ne) clen = 0;
    const uint32_t lead = po & 3u;
    const uint32_t nch = clen ? (lead + clen + 3u) >> 2 : 0u;  // aligned chunks of the segment
    uint32_t incl = nch;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(full, incl, off);
      if ((int)lane >= off) incl += y;
    }
    const uint32_t tot = __shfl_sync(full, incl, 31);
    const uint32_t excl = incl - nch;
    // chunk c of the batch starts at word A + 4 c of padj and holds words [4 c, 4 c + 4) of the
    // batch's word space; the segment's keys are the words [lo, hi) of that space
    const uint32_t lo = 4u * excl + lead, hi = lo + clen;
    const uint32_t A = (po - lead) - 4u * excl;
    const uint32_t srd = (lane < ne && excl > 0) ? (excl - 1) >> 5 : 0xFFFFFFFFu;
    const unsigned sbit = 1u << ((excl - 1) & 31);
    uint32_t own0 = 0;
    for (uint32_t r = 0; r < tot; r += 32 * kU) {
      uint32_t wi[kU], los[kU], his[kU];
      bool ok[kU];
      const uint32_t nr = (tot - r + 31) / 32;  // rounds left (warp-uniform)
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        ok[j] = false;
        wi[j] = los[j] = his[j] = 0;
        if ((uint32_t)j >= nr) continue;
        const uint32_t rr = r + 32 * j;
        const unsigned B = __reduce_or_sync(full, srd == (rr >> 5) ? sbit : 0u);
        const uint32_t own = own0 + __popc(B & ((1u << lane) - 1u));
        wi[j] = __shfl_sync(full, A, own) + 4u * (rr + lane);
        los[j] = __shfl_sync(full, lo, own);
        his[j] = __shfl_sync(full, hi, own);
        ok[j] = rr + lane < tot;
        own0 += __popc(B);
      }
      uint4 ks[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j)
        ks[j] = ok[j] ? __ldg(reinterpret_cast<const uint4*>(src.padj + wi[j]))
                      : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t x0 = 4u * (r + 32 * j + lane);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (ok[j] && x0 + q >= los[j] && x0 + q < his[j]) f(u4_word(ks[j], q));
      }
    }
  }
}

template <class Src, class F>
__device__ __forceinline__ void warp_walk(const Src& src, uint32_t task, F&& f) {
  uint64_t e0, e1;
  src.entries(task, e0, e1);
  warp_walk_range(src, task, e0, e1, f);
}

// ---- grouped walks (BFLY_GROUP_WALK=1): segments handed to groups of kGroup lanes ----------
// The flattened walks above map every element of a round to its segment (an OR-reduction of
// segment starts + two popcounts + a shuffle of the segment base per element round): about
// half of the hub kernels' instructions. Here a group of kGroup lanes owns one segment at a
// time and reads it kGroup keys per step (consecutive lanes, consecutive keys); a group that
// exhausts its segment claims the next one (ballot + popcount inside the warp, a shared
// counter across a CTA). No per-element owner search; segments are compacted first, so empty
// ones cost nothing. Counting runs only (no entry index is passed to f).
#ifndef BFLY_GROUP_WALK
#define BFLY_GROUP_WALK 0
#endif
constexpr int kGroup = 8;

// one warp, entries [e0, e1) of one task: f(key) per element
template <class Src, class F>
__device__ __forceinline__ void warp_group_walk(const Src& src, uint32_t task, uint64_t e0,
                                                uint64_t e1, F&& f) {
  constexpr int G = kGroup, NG = 32 / G;
  const unsigned lane = threadIdx.x & 31, full = 0xffffffffu;
  const unsigned gl = lane & (G - 1);
  const unsigned lead_bit = 1u << (lane & ~unsigned(G - 1));
  for (uint64_t eb = e0; eb < e1; eb += 32) {
    const uint64_t e = eb + lane;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    const unsigned nz = __ballot_sync(full, len > 0);
    if (!nz) continue;
    const unsigned ne = __popc(nz);
    const unsigned srcl = (nz & (nz + 1u)) == 0u ? lane : (lane < ne ? nth_set_bit(nz, lane) : 0u);
    uint32_t clen = __shfl_sync(full, len, srcl);
    const unsigned long long cp = __shfl_sync(full, reinterpret_cast<unsigned long long>(p), srcl);
    if (lane >= ne) clen = 0;
    // group g starts on compacted segment g; `next` (warp-uniform) is the first unclaimed one
    uint32_t sg = lane / G, next = NG, off = 0;
    uint32_t sl = __shfl_sync(full, clen, sg);
    const uint32_t* sp = reinterpret_cast<const uint32_t*>(__shfl_sync(full, cp, sg));
    if (sg >= ne) sl = 0;
    while (true) {
      const bool act = sg < ne;
      if (!__any_sync(full, act)) break;
      const uint32_t x0 = off + gl, x1 = off + G + gl;
      const uint32_t k0 = act && x0 < sl ? __ldg(sp + x0) : 0u;
      const uint32_t k1 = act && x1 < sl ? __ldg(sp + x1) : 0u;
      if (act && x0 < sl) f(k0);
      if (act && x1 < sl) f(k1);
      off += 2 * G;
      const bool need = act && off >= sl;  // group-uniform
      const unsigned dm = __ballot_sync(full, need && gl == 0);
      if (dm) {  // warp-uniform
        const uint32_t ns = need ? next + __popc(dm & (lead_bit - 1u)) : sg;
        next += __popc(dm);
        const uint32_t nl = __shfl_sync(full, clen, ns & 31u);
        const unsigned long long np = __shfl_sync(full, cp, ns & 31u);
        if (need) {
          sg = ns;
          off = 0;
          sl = ns < ne ? nl : 0u;
          sp = reinterpret_cast<const uint32_t*>(np);
        }
      }
    }
  }
}

// ---- tiny: warp per task, keys in registers --------------------------------------------------
// A tiny task has at most 32 keys, so lane L can own element L of the task outright: one
// scan of the segment lengths of a batch of 32 entries places every element, and all key
// loads of the task are issued at once. kTinyTasks tasks are interleaved per warp so their
// dependent load chains (list -> entries -> segments -> keys) overlap.
#ifndef BFLY_TINY_TASKS
#define BFLY_TINY_TASKS 4
#endif
constexpr int kTinyTasks = BFLY_TINY_TASKS;

// Place the elements of one batch of entries (this lane's entry e, segment len at p) at lanes
// filled, filled + 1, ...: lane L < 32 in that range gets pe = its element's address and
// ent = its entry index.
template <bool NEED_E>
__device__ __forceinline__ void tiny_place(uint32_t len, const uint32_t* p, uint64_t eb,
                                           uint32_t& filled, const uint32_t*& pe, uint64_t& ent) {
  const unsigned full = 0xffffffffu, lane = threadIdx.x & 31;
  const unsigned nz = __ballot_sync(full, len > 0);
  if (!nz) return;
  const unsigned ne = __popc(nz);
  const unsigned srcl = (nz & (nz + 1u)) == 0u ? lane : (lane < ne ? nth_set_bit(nz, lane) : 0u);
  uint32_t clen = __shfl_sync(full, len, srcl);
  const unsigned long long cp = __shfl_sync(full, reinterpret_cast<unsigned long long>(p), srcl);
  if (lane >= ne) clen = 0;
  uint32_t incl = clen;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(full, incl, off);
    if ((int)lane >= off) incl += y;
  }
  const uint32_t tot = __shfl_sync(full, incl, 31);
  const uint32_t st = filled + incl - clen;  // first lane of compacted segment `lane`
  const unsigned B = __reduce_or_sync(full, (lane < ne && st < 32u) ? (1u << st) : 0u);
  const unsigned own = __popc(B & (0xFFFFFFFFu >> (31u - lane))) - 1u;  // starts <= lane
  const unsigned long long bp = __shfl_sync(full, cp - 4ull * st, own & 31u);
  const bool mine = lane >= filled && lane < filled + tot;
  if (mine) pe = reinterpret_cast<const uint32_t*>(bp) + lane;
  if constexpr (NEED_E) {
    const unsigned ol = __shfl_sync(full, srcl, own & 31u);
    if (mine) ent = eb + ol;
  }
  filled += tot;
}

template <class Src, bool LOCAL>
__device__ __forceinline__ void tiny_flat(const Src& src, const uint32_t* __restrict__ list,
                                          uint64_t count, unsigned long long* task_out,
                                          Acc& acc, const LocalOut& lo, Mom& mom) {
  constexpr int T = kTinyTasks;
  const unsigned lane = threadIdx.x & 31, full = 0xffffffffu;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = gw; i < count; i += T * nw) {
    uint32_t task[T];
    uint64_t e0[T], e1[T];
#pragma unroll
    for (int j = 0; j < T; ++j) task[j] = i + j * nw < count ? list[i + j * nw] : kEmpty;
#pragma unroll
    for (int j = 0; j < T; ++j) {
      e0[j] = e1[j] = 0;
      if (task[j] != kEmpty) src.entries(task[j], e0[j], e1[j]);
    }
    uint32_t len[T];
    const uint32_t* p[T];
#pragma unroll
    for (int j = 0; j < T; ++j) {
      len[j] = 0;
      p[j] = nullptr;
      if (e0[j] + lane < e1[j]) len[j] = src.seg(task[j], e0[j] + lane, p[j]);
    }
    uint32_t filled[T];
    const uint32_t* pe[T];
    uint64_t ent[T];
#pragma unroll
    for (int j = 0; j < T; ++j) {
      filled[j] = 0;
      pe[j] = nullptr;
      ent[j] = 0;
      tiny_place<LOCAL>(len[j], p[j], e0[j], filled[j], pe[j], ent[j]);
      for (uint64_t eb = e0[j] + 32; eb < e1[j]; eb += 32) {  // tasks with > 32 entries
        uint32_t l2 = 0;
        const uint32_t* p2 = nullptr;
        if (eb + lane < e1[j]) l2 = src.seg(task[j], eb + lane, p2);
        tiny_place<LOCAL>(l2, p2, eb, filled[j], pe[j], ent[j]);
      }
    }
    uint32_t x[T];
#pragma unroll
    for (int j = 0; j < T; ++j) x[j] = lane < filled[j] ? __ldg(pe[j]) : 0u;
#pragma unroll
    for (int j = 0; j < T; ++j) {
      if (task[j] == kEmpty) continue;  // warp-uniform
      Acc ta;
      const unsigned act = __ballot_sync(full, lane < filled[j]);
      if (lane < filled[j]) {
        const unsigned mm = __match_any_sync(act, x[j]);
        const unsigned long long c = __popc(mm);
        if ((int)lane == __ffs(mm) - 1) {
          ta.add(c2(c));
          if (LOCAL && c >= 2) atomicAdd(&lo.vcnt[x[j]], c2(c));
          if constexpr (kMoments<Src>) mom.add(static_cast<uint32_t>(c));
        }
        if (LOCAL) emit_wedge(lo, ent[j], pe[j], static_cast<uint32_t>(c));
      }
      if (LOCAL || task_out) {
        ta = warp_sum(ta);
        if (lane == 0) {
          if (task_out) task_out[task[j]] = ta.v;
          if (LOCAL && ta.v) atomicAdd(&lo.vcnt[task[j]], ta.v);
        }
        acc.add(lane == 0 ? ta.v : 0ull);
        acc.ovf |= ta.ovf;
      } else {
        acc.add(ta.v);
      }
    }
  }
}

// Lane per task (counting only): each lane gathers its task's <= 32 keys into a private
// shared-memory column and counts, for every key, the equal keys gathered before it
// (sum = sum of C(c,2)). No warp-wide scans or matches per task: a warp finishes 32 tasks in
// about the instructions the warp-per-task path spends on one.
#ifndef BFLY_TINY_LANE
#define BFLY_TINY_LANE 1
#endif
// key bound of the counting-only tiny bucket (lane per task); the local-count pass keeps 32
// (one element per lane of a warp)
#ifndef BFLY_TINY_LANE_MAX
#define BFLY_TINY_LANE_MAX 32
#endif
constexpr uint32_t kTinyLaneMax = BFLY_TINY_LANE_MAX;
template <class Src>
__device__ __forceinline__ void tiny_lane(const Src& src, const uint32_t* __restrict__ list,
                                          uint64_t count, unsigned long long* task_out,
                                          Acc& acc) {
  __shared__ uint32_t kbuf[8][kTinyLaneMax * 32];  // per warp, slot-major: key j of lane l at j*32 + l
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* kb = kbuf[wl];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = gw * 32; base < count; base += nw * 32) {
    const uint64_t i = base + lane;
    if (i >= count) continue;
    const uint32_t task = list[i];
    uint64_t e0, e1;
    src.entries(task, e0, e1);
    uint32_t nk = 0;
    for (uint64_t e = e0; e < e1; ++e) {
      const uint32_t* p = nullptr;
      uint32_t len = src.seg(task, e, p);
      if (len > kTinyLaneMax - nk) len = kTinyLaneMax - nk;  // (tiny: <= kTinyLaneMax keys)
#pragma unroll 4
      for (uint32_t j = 0; j < len; ++j) kb[(nk + j) * 32 + lane] = __ldg(p + j);
      nk += len;
    }
    unsigned long long t = 0;
    for (uint32_t j = 1; j < nk; ++j) {
      const uint32_t x = kb[j * 32 + lane];
      uint32_t c = 0;
      for (uint32_t q = 0; q < j; ++q) c += kb[q * 32 + lane] == x;
      t += c;
    }
    if (task_out) task_out[task] = t;
    acc.add(t);
  }
}

template <class Src, bool LOCAL>
__global__ void __launch_bounds__(256) k_tiny(Src src, const uint32_t* __restrict__ list,
                                              uint64_t count, unsigned long long* task_out,
                                              unsigned long long* total, unsigned* ovf,
                                              LocalOut lo) {
  Acc acc;
  if constexpr (!Src::kExcl) {
    Mom mom;
    if (!LOCAL && !kMoments<Src> && BFLY_TINY_LANE) tiny_lane<Src>(src, list, count, task_out, acc);
    else tiny_flat<Src, LOCAL>(src, list, count, task_out, acc, lo, mom);
    flush_acc(acc, total, ovf);
    if constexpr (kMoments<Src>) flush_mom(mom, lo.mom);
    return;
  } else {
  __shared__ uint32_t bw[8][32];
  __shared__ const uint32_t* bq[LOCAL ? 8 : 1][32];
  __shared__ uint64_t be[LOCAL ? 8 : 1][32];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = gw; i < count; i += nw) {
    const uint32_t task = list[i];
    uint32_t filled = 0;
    const uint32_t ex = src.excl(task);
    uint64_t e0, e1;
    src.entries(task, e0, e1);
    for (uint64_t eb = e0; eb < e1; eb += 32) {
      const uint64_t e = eb + lane;
      uint32_t len = 0;
      const uint32_t* p = nullptr;
      if (e < e1) len = src.seg(task, e, p);
      uint32_t keep = 0;  // the excluded element occurs at most once per segment
      for (uint32_t t = 0; t < len; ++t) keep += (p[t] != ex);
      uint32_t kin = keep;
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, kin, off);
        if ((int)lane >= off) kin += y;
      }
      const uint32_t ktot = __shfl_sync(0xffffffffu, kin, 31);
      uint32_t pos = filled + kin - keep;
      for (uint32_t t = 0; t < len; ++t) {
        const uint32_t w = p[t];
        if (w == ex) continue;
        if (pos < 32) {
          bw[wl][pos] = w;
          if (LOCAL) {
            bq[wl][pos] = p + t;
            be[wl][pos] = e;
          }
        }
        ++pos;
      }
      filled += ktot;
    }
    __syncwarp();
    Acc ta;
    const unsigned act = __ballot_sync(0xffffffffu, lane < filled);
    if (lane < filled) {
      const uint32_t x = bw[wl][lane];
      const unsigned mm = __match_any_sync(act, x);
      const unsigned long long c = __popc(mm);
      if ((int)lane == __ffs(mm) - 1) {
        ta.add(c2(c));
        if (LOCAL && c >= 2) atomicAdd(&lo.vcnt[x], c2(c));
      }
      if (LOCAL) emit_wedge(lo, be[wl][lane], bq[wl][lane], static_cast<uint32_t>(c));
    }
    if (LOCAL || task_out) {
      ta = warp_sum(ta);
      if (lane == 0) {
        if (task_out) task_out[task] = ta.v;
        if (LOCAL && ta.v) atomicAdd(&lo.vcnt[task], ta.v);
      }
      acc.add(lane == 0 ? ta.v : 0ull);
      acc.ovf |= ta.ovf;
    } else {
      acc.add(ta.v);
    }
    __syncwarp();
  }
  flush_acc(acc, total, ovf);
  }
}

// Tables whose increments return small old values, so one thread's sum over one task fits
// 32 bits: byte counters (< 256, tasks < 2^23 keys), BitHash (<= 512 keys), Hash (<= 8192
// keys per task). DirectSplit's 32-bit hub counters do not qualify.
template <class T>
constexpr bool kNarrowOld = false;
template <>
constexpr bool kNarrowOld<DirectByte> = true;
template <int B>
constexpr bool kNarrowOld<BitHash<B>> = true;
template <int B>
constexpr bool kNarrowOld<Hash<B>> = true;
template <int B, int C>
constexpr bool kNarrowOld<PackedHash<B, C>> = true;

// rounds of 32 keys per walk iteration in the warp-table kernels (tasks of <= 512 keys)
#ifndef BFLY_SMALL_KU
#define BFLY_SMALL_KU 4
#endif
constexpr int kSmallU = BFLY_SMALL_KU;
#ifndef BFLY_SMALL_PREFETCH
#define BFLY_SMALL_PREFETCH 0  // measured: phase 10.06 -> 10.20 ms with it on
#endif

// ---- small: warp per task, private shared-memory table ---------------------------------------
// per-warp memory: Tab::words(K) rounded to 16 bytes; the table is reset whole after each task
// (uint4 stores: cheaper than tracking touched slots at these sizes)
template <class Src, bool LOCAL, class Tab>
__global__ void __launch_bounds__(kSmallWarps * 32) k_small(
    Src src, const uint32_t* __restrict__ list, uint64_t count, uint32_t K,
    unsigned long long* task_out, unsigned long long* total, unsigned* ovf, LocalOut lo) {
  extern __shared__ uint32_t smem[];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* base = smem + wl * ((Tab::words(K) + 3) & ~3u);  // 16-byte aligned
  Tab tab;
  tab.bind(base, K);
  tab.init(lane, 32);
  __syncwarp();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  Acc acc;
  Mom mom;
  // the next task's id and entry range are fetched while this one is walked: the dependent
  // load chain list -> offsets of a task overlaps the previous task's work
  // (BFLY_SMALL_PREFETCH=0: only the id is fetched ahead, for A/B)
  uint32_t ntask = 0;
  uint64_t ne0 = 0, ne1 = 0;
  if (gw < count) {
    ntask = list[gw];
    src.entries(ntask, ne0, ne1);
  }
  for (uint64_t i = gw; i < count; i += nw) {
    const uint32_t task = ntask;
    uint64_t ce0_ = ne0, ce1_ = ne1;
    const uint64_t& ce0 = ce0_;
    const uint64_t& ce1 = ce1_;
    if (i + nw < count) {
      ntask = __ldg(list + i + nw);
      if (BFLY_SMALL_PREFETCH) src.entries(ntask, ne0, ne1);
    }
    if (!BFLY_SMALL_PREFETCH) src.entries(task, ce0_, ce1_);
    Acc ta;
    {
      const uint64_t e0 = ce0, e1 = ce1;
      uint32_t t32 = 0;  // per-lane sum of one task: < 2^32 (kNarrowOld)
      if constexpr (BFLY_HUB_MATCH && !LOCAL && std::is_same_v<Src, HubSrc>) {
        auto cf = [&](uint32_t w, uint32_t n) { t32 += tab.add(w, n); };
        warp_walk_range<false, kSmallU>(src, task, e0, e1, Combine<decltype(cf)>{cf});
      } else if constexpr (BFLY_GROUP_WALK && !LOCAL && !Src::kExcl && !kMoments<Src>) {
        warp_group_walk(src, task, e0, e1, [&](uint32_t w) {
          if constexpr (kNarrowOld<Tab>) t32 += tab.inc(w);
          else ta.add(tab.inc(w));
        });
      } else if constexpr (BFLY_VEC4 && BFLY_VEC4_SMALL && !LOCAL && Src::kVec4 && !kMoments<Src>) {
        warp_walk_range_v4(src, task, e0, e1, [&](uint32_t w) {
          if constexpr (kNarrowOld<Tab>) t32 += tab.inc(w);
          else ta.add(tab.inc(w));
        });
      } else {
        warp_walk_range<false, kSmallU>(src, task, e0, e1, [&](uint32_t w, const uint32_t*, uint64_t) {
          if constexpr (kNarrowOld<Tab>) t32 += tab.inc(w);
          else ta.add(tab.inc(w));
        });
      }
      ta.add(t32);
    }
    __syncwarp();
    if (LOCAL) {
      warp_walk_range(
          src, task, ce0, ce1,
          [&](uint32_t w, const uint32_t* pe, uint64_t) { return emit_key(lo, pe, tab.get(w)); },
          Seg<EmitEntry>{EmitEntry{lo}});
      __syncwarp();
    }
    if (LOCAL) {
      tab.drain(lane, 32, [&](uint32_t key, uint32_t c) {
        if (c >= 2) add_key(lo, key, c2(c));
      });
    } else if constexpr (kMoments<Src>) {
      tab.drain(lane, 32, [&](uint32_t, uint32_t c) { mom.add(c); });
    } else {
      tab.reset_all(lane, 32);
    }
    if (LOCAL || task_out) {  // per-task totals only when someone needs them
      ta = warp_sum(ta);
      if (lane == 0) {
        if (task_out) task_out[task] = ta.v;
        if (LOCAL && ta.v) atomicAdd(&lo.vcnt[task], ta.v);
      }
      acc.add(lane == 0 ? ta.v : 0ull);
      acc.ovf |= ta.ovf;
    } else {
      acc.add(ta.v);  // per-lane partial, < 2^61 like every partial
    }
    __syncwarp();
  }
  flush_acc(acc, total, ovf);
  if constexpr (kMoments<Src>) flush_mom(mom, lo.mom);
}

// ---- block-level flattened walk -----------------------------------------------------------
// Chunk scan word: (segment length << SH) | non-empty flag. Sources whose segments are
// short (hub prefixes: < 2^15 keys, at most 256 entries per chunk) use a 32-bit word with
// SH = 9; the others 64-bit words with SH = 32.
template <class Src, int BLOCK>
struct ScanWord {
  static constexpr bool kNarrow = Src::kNarrowScan && BLOCK <= 256;
  using T = std::conditional_t<kNarrow, uint32_t, unsigned long long>;
  static constexpr int SH = kNarrow ? 9 : 32;
};

#ifndef BFLY_CUB_SCAN
#define BFLY_CUB_SCAN 0
#endif
template <int BLOCK, class ST = unsigned long long>
struct BlockWalkSmem {
  ST warp_tot[BLOCK / 32];       // per-warp totals of the chunk scan
  uint32_t incl[BLOCK];          // compacted segment start offsets (strictly increasing)
  const uint32_t* base[BLOCK];   // element idx -> base[seg] + idx
  uint32_t entry[BLOCK];         // entry index within the chunk
};

template <int BLOCK, bool NEED_E = true, class Src, class F, class SG = NoSeg, int kU = 4>
__device__ __forceinline__ void block_walk_range(const Src& src, uint32_t task, uint64_t e0,
                                                 uint64_t e1, BlockWalkSmem<BLOCK, typename ScanWord<Src, BLOCK>::T>& sm,
                                                 F&& f, bool last_sync = true, const SG& seg = SG{}) {
  // One scan of (segment length << 32 | non-empty flag) compacts the non-empty segments of
  // BLOCK entries into smem with strictly increasing start offsets. Each warp then walks a
  // contiguous slice of the chunk's elements; the owner segment of every element comes from
  // one OR-reduction of segment-start bits per 32 elements (no per-element search).
  // (last_sync = false: the caller's next barrier protects the chunk state of the last chunk)
  using SW = ScanWord<Src, BLOCK>;
  using ST = typename SW::T;

  constexpr ST kNzMask = (ST(1) << SW::SH) - 1;
  const uint32_t ex = src.excl(task);
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  constexpr unsigned W = BLOCK / 32;
  for (uint64_t eb = e0; eb < e1; eb += BLOCK) {
    const uint64_t e = eb + threadIdx.x;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    const ST mine = (static_cast<ST>(len) << SW::SH) | static_cast<ST>(len > 0);
    ST incl, totv;
    // inclusive block scan; only the warps holding entries of this chunk scan (hub tasks
    // have a few dozen entries: most warps of a chunk are empty)
#if BFLY_CUB_SCAN
    {
      using Scan = cub::BlockScan<ST, BLOCK, cub::BLOCK_SCAN_WARP_SCANS>;
      __shared__ typename Scan::TempStorage cub_ts;
      Scan(cub_ts).InclusiveSum(mine, incl, totv);
    }
#else
    {
      const uint64_t left = e1 - eb;
      const unsigned nwa = left >= BLOCK ? W : static_cast<unsigned>((left + 31) / 32);
      ST x = mine;
      if (wl < nwa) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const ST y = __shfl_up_sync(0xffffffffu, x, off);
          if ((int)lane >= off) x += y;
        }
        if (lane == 31) sm.warp_tot[wl] = x;
      }
      __syncthreads();
      ST pre = 0, tv = 0;
      for (unsigned w = 0; w < nwa; ++w) {
        const ST t = sm.warp_tot[w];
        pre += w < wl ? t : ST(0);
        tv += t;
      }
      incl = x + pre;
      totv = tv;
    }
#endif
    const uint32_t tot = static_cast<uint32_t>(totv >> SW::SH);
    const uint32_t nnz = static_cast<uint32_t>(totv & kNzMask);
    if (len) {
      const uint32_t slot = static_cast<uint32_t>(incl & kNzMask) - 1u;
      const uint32_t ex_off = static_cast<uint32_t>(incl >> SW::SH) - len;
      sm.incl[slot] = ex_off;  // segment start offset
      sm.base[slot] = p - ex_off;
      if constexpr (NEED_E || SG::kActive) sm.entry[slot] = static_cast<uint32_t>(threadIdx.x);
    }
    __syncthreads();
    if (tot) {
      const uint32_t a = static_cast<uint32_t>((static_cast<uint64_t>(tot) * wl) / W);
      const uint32_t b = static_cast<uint32_t>((static_cast<uint64_t>(tot) * (wl + 1)) / W);
      // owner of element a: last compacted segment with start <= a (the starts ascend: count
      // them 32 at a time with a ballot)
      uint32_t cnt = 0;
      for (uint32_t base = 0; base < nnz; base += 32) {
        const unsigned le =
            __ballot_sync(0xffffffffu, base + lane < nnz && sm.incl[base + lane] <= a);
        cnt += __popc(le);
        if (le != 0xffffffffu) break;
      }
      uint32_t own = cnt - 1;
      // kU rounds of 32 elements per iteration: owners first, then kU independent key loads
      // in flight, then the table updates
      for (uint32_t r = a; r < b; r += 32 * kU) {
        const uint32_t* pes[kU];
        uint32_t ents[kU];
        unsigned Bs[kU];
        bool ok[kU];
        const uint32_t nr = (b - r + 31) / 32;  // rounds left (warp-uniform)
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          ok[j] = false;
          pes[j] = nullptr;
          ents[j] = 0;
          Bs[j] = 0;
          if ((uint32_t)j >= nr) continue;
          const uint32_t rr = r + 32 * j;
          const uint32_t t = own + 1 + lane;
          const uint32_t st = t < nnz ? sm.incl[t] : 0u;
          const uint32_t d = st - rr - 1;  // start inside (rr, rr + 32] <=> d < 32 (unsigned)
          const unsigned bit = d < 32u ? (1u << d) : 0u;
          const unsigned B = __reduce_or_sync(0xffffffffu, bit);
          Bs[j] = B;
          const uint32_t mo = own + __popc(B & ((1u << lane) - 1u));
          ok[j] = rr + lane < b;
          pes[j] = sm.base[mo] + (rr + lane);
          if constexpr (NEED_E || SG::kActive) ents[j] = sm.entry[mo];
          own += __popc(B);
        }
        uint32_t ws[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) ws[j] = ok[j] ? __ldg(pes[j]) : 0u;
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          if constexpr (SG::kActive) {
            unsigned long long x = 0;
            if (ok[j] && (!Src::kExcl || ws[j] != ex)) x = f(ws[j], pes[j], eb + ents[j]);
            if ((uint32_t)j < nr) seg_emit(ok[j], Bs[j], eb + ents[j], x, seg);
          } else if constexpr (IsCombine<std::decay_t<F>>::value) {
            combined_call(f, ok[j], ws[j]);
          } else {
            if (ok[j] && (!Src::kExcl || ws[j] != ex)) f(ws[j], pes[j], eb + ents[j]);
          }
        }
      }
    }
    if (last_sync || eb + BLOCK < e1) __syncthreads();
  }
}

// The block walk over 16-byte chunks (see warp_walk_range_v4): the compacted segments keep
// (A, hi) in the base slot and lo in the entry slot of the walk state.
template <int BLOCK, class Src, class F, int kU = BFLY_VEC4_KU>
__device__ __forceinline__ void block_walk_range_v4(
    const Src& src, uint32_t task, uint64_t e0, uint64_t e1,
    BlockWalkSmem<BLOCK, typename ScanWord<Src, BLOCK>::T>& sm, F&& f, bool last_sync = true) {
  static_assert(Src::kVec4 && !Src::kExcl, "aligned, padded adjacency without an excluded key");
  using SW = ScanWord<Src, BLOCK>;
  using ST = typename SW::T;
  static_assert(sizeof(sm.base[0]) == sizeof(uint2), "(A, hi) share a pointer slot");
  uint2* meta = reinterpret_cast<uint2*>(sm.base);
  constexpr ST kNzMask = (ST(1) << SW::SH) - 1;
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  constexpr unsigned W = BLOCK / 32;
  for (uint64_t eb = e0; eb < e1; eb += BLOCK) {
    const uint64_t e = eb + threadIdx.x;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    const uint32_t po = static_cast<uint32_t>(p - src.padj);  // (unused where len is 0)
    const uint32_t lead = po & 3u;
    const uint32_t nch = len ? (lead + len + 3u) >> 2 : 0u;
    const ST mine = (static_cast<ST>(nch) << SW::SH) | static_cast<ST>(len > 0);
    ST incl, totv;
    {
      const uint64_t left = e1 - eb;
      const unsigned nwa = left >= BLOCK ? W : static_cast<unsigned>((left + 31) / 32);
      ST x = mine;
      if (wl < nwa) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const ST y = __shfl_up_sync(0xffffffffu, x, off);
          if ((int)lane >= off) x += y;
        }
        if (lane == 31) sm.warp_tot[wl] = x;
      }
      __syncthreads();
      ST pre = 0, tv = 0;
      for (unsigned w = 0; w < nwa; ++w) {
        const ST t = sm.warp_tot[w];
        pre += w < wl ? t : ST(0);
        tv += t;
      }
      incl = x + pre;
      totv = tv;
    }
    const uint32_t tot = static_cast<uint32_t>(totv >> SW::SH);  // chunks of the batch
    const uint32_t nnz = static_cast<uint32_t>(totv & kNzMask);
    if (len) {
      const uint32_t slot = static_cast<uint32_t>(incl & kNzMask) - 1u;
      const uint32_t ex_off = static_cast<uint32_t>(incl >> SW::SH) - nch;  // first chunk
      const uint32_t lo = 4u * ex_off + lead;
      sm.incl[slot] = ex_off;
      meta[slot] = make_uint2((po - lead) - 4u * ex_off, lo + len);
      sm.entry[slot] = lo;
    }
    __syncthreads();
    if (tot) {
      const uint32_t a = static_cast<uint32_t>((static_cast<uint64_t>(tot) * wl) / W);
      const uint32_t b = static_cast<uint32_t>((static_cast<uint64_t>(tot) * (wl + 1)) / W);
      uint32_t cnt = 0;
      for (uint32_t base = 0; base < nnz; base += 32) {
        const unsigned le =
            __ballot_sync(0xffffffffu, base + lane < nnz && sm.incl[base + lane] <= a);
        cnt += __popc(le);
        if (le != 0xffffffffu) break;
      }
      uint32_t own = cnt - 1;
      for (uint32_t r = a; r < b; r += 32 * kU) {
        uint32_t wi[kU], los[kU], his[kU];
        bool ok[kU];
        const uint32_t nr = (b - r + 31) / 32;  // rounds left (warp-uniform)
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          ok[j] = false;
          wi[j] = los[j] = his[j] = 0;
          if ((uint32_t)j >= nr) continue;
          const uint32_t rr = r + 32 * j;
          const uint32_t t = own + 1 + lane;
          const uint32_t st = t < nnz ? sm.incl[t] : 0u;
          const uint32_t d = st - rr - 1;  // start inside (rr, rr + 32] <=> d < 32 (unsigned)
          const unsigned bit = d < 32u ? (1u << d) : 0u;
          const unsigned B = __reduce_or_sync(0xffffffffu, bit);
          const uint32_t mo = own + __popc(B & ((1u << lane) - 1u));
          ok[j] = rr + lane < b;
          const uint2 m = meta[mo];
          wi[j] = m.x + 4u * (rr + lane);
          his[j] = m.y;
          los[j] = sm.entry[mo];
          own += __popc(B);
        }
        uint4 ks[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j)
          ks[j] = ok[j] ? __ldg(reinterpret_cast<const uint4*>(src.padj + wi[j]))
                        : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          const uint32_t x0 = 4u * (r + 32 * j + lane);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (ok[j] && x0 + q >= los[j] && x0 + q < his[j]) f(u4_word(ks[j], q));
        }
      }
    }
    if (last_sync || eb + BLOCK < e1) __syncthreads();
  }
}

template <int BLOCK, bool NEED_E = true, class Src, class F, class SG = NoSeg>
__device__ __forceinline__ void block_walk(const Src& src, uint32_t task,
                                           BlockWalkSmem<BLOCK, typename ScanWord<Src, BLOCK>::T>& sm,
                                           F&& f, bool last_sync = true, const SG& seg = SG{}) {
  uint64_t e0, e1;
  src.entries(task, e0, e1);
  block_walk_range<BLOCK, NEED_E>(src, task, e0, e1, sm, f, last_sync, seg);
}

// one CTA, entries [e0, e1) of one task: f(key) per element. Per chunk of BLOCK entries the
// non-empty segments are compacted into shared memory (one block scan of the non-empty
// flags), then the BLOCK / kGroup groups consume them with a shared claim counter.
template <int BLOCK, class Src, class F>
__device__ __forceinline__ void block_group_walk(const Src& src, uint32_t task, uint64_t e0,
                                                 uint64_t e1,
                                                 BlockWalkSmem<BLOCK, typename ScanWord<Src, BLOCK>::T>& sm,
                                                 unsigned* s_next, F&& f) {
  constexpr int G = kGroup, NG = BLOCK / G;
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5, full = 0xffffffffu;
  const unsigned gl = threadIdx.x & (G - 1);
  const unsigned gmask = ((1u << G) - 1u) << (lane & ~unsigned(G - 1));
  for (uint64_t eb = e0; eb < e1; eb += BLOCK) {
    const uint64_t e = eb + threadIdx.x;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    const unsigned nzw = __ballot_sync(full, len > 0);
    if (lane == 0) sm.warp_tot[wl] = __popc(nzw);
    if (threadIdx.x == 0) *s_next = NG;
    __syncthreads();
    uint32_t pre = 0, nnz = 0;
    for (unsigned w = 0; w < BLOCK / 32; ++w) {
      const uint32_t c = static_cast<uint32_t>(sm.warp_tot[w]);
      pre += w < wl ? c : 0u;
      nnz += c;
    }
    if (len) {
      const uint32_t slot = pre + __popc(nzw & ((1u << lane) - 1u));
      sm.incl[slot] = len;  // (the flattened walk's arrays: segment length and start)
      sm.base[slot] = p;
    }
    __syncthreads();
    uint32_t sg = threadIdx.x / G, off = 0, sl = 0;
    const uint32_t* sp = nullptr;
    if (sg < nnz) {
      sl = sm.incl[sg];
      sp = sm.base[sg];
    }
    while (sg < nnz) {  // group-uniform
      const uint32_t x0 = off + gl, x1 = off + G + gl;
      const uint32_t k0 = x0 < sl ? __ldg(sp + x0) : 0u;
      const uint32_t k1 = x1 < sl ? __ldg(sp + x1) : 0u;
      if (x0 < sl) f(k0);
      if (x1 < sl) f(k1);
      off += 2 * G;
      if (off >= sl) {  // claim the next segment (group leader), broadcast inside the group
        uint32_t ns = 0;
        if (gl == 0) ns = atomicAdd(s_next, 1u);
        ns = __shfl_sync(gmask, ns, 0, G);
        sg = ns;
        off = 0;
        if (sg < nnz) {
          sl = sm.incl[sg];
          sp = sm.base[sg];
        }
      }
    }
    __syncthreads();  // the chunk's arrays and counter are reused by the next chunk
  }
}

template <int BLOCK>
__device__ __forceinline__ Acc block_sum(Acc a, unsigned long long* red, unsigned* redo) {
  a = warp_sum(a);
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  if (lane == 0) {
    red[wl] = a.v;
    redo[wl] = a.ovf;
  }
  __syncthreads();
  Acc r;
  if (threadIdx.x == 0) {
    for (int q = 0; q < BLOCK / 32; ++q) {
      r.add(red[q]);
      r.ovf |= redo[q];
    }
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// resident 256-thread CTAs per SM to size registers for: the 22 KB byte table fits 7
template <class Tab>
struct MediumMinBlocks {
  static constexpr int v = 6;
};
template <>
struct MediumMinBlocks<DirectByte> {
  static constexpr int v = 7;
};

// ---- medium: CTA per task, shared-memory table, persistent queue -----------------------------
template <class Src, bool LOCAL, class Tab, int BLOCK>
__global__ void __launch_bounds__(BLOCK, BLOCK == 256   ? (LOCAL ? 4 : MediumMinBlocks<Tab>::v)
                                         : BLOCK == 128 ? (LOCAL ? 8 : 2 * MediumMinBlocks<Tab>::v)
                                                        : 1)
    k_medium(Src src, const uint32_t* __restrict__ list,
                                                  uint64_t count, uint32_t K,
                                                  unsigned long long* next,
                                                  unsigned long long* task_out,
                                                  unsigned long long* total, unsigned* ovf,
                                                  LocalOut lo) {
  extern __shared__ uint32_t smem[];
  Tab tab;
  tab.bind(smem, K);
  __shared__ BlockWalkSmem<BLOCK, typename ScanWord<Src, BLOCK>::T> wsm;
  __shared__ unsigned long long s_item[2];
  __shared__ unsigned long long red[BLOCK / 32];
  __shared__ unsigned redo[BLOCK / 32];
  __shared__ unsigned s_claim;  // (grouped walk: next unclaimed segment of the chunk)
  tab.init(threadIdx.x, BLOCK);
  Acc acc;
  Mom mom;
  if (threadIdx.x == 0) s_item[0] = atomicAdd(next, 1ull);
  __syncthreads();
  // Barriers per task: the walk's scan + post-compaction barrier, and one after the inserts.
  // The next task id is fetched at the start of a task into the other s_item slot (read only
  // after this task's barriers); the drain of task i is ordered before the inserts of task
  // i+1 by the walk barrier of task i+1.
  for (uint32_t it = 0;; ++it) {
    const unsigned long long item = s_item[it & 1];
    if (item >= count) break;
    if (threadIdx.x == 0) s_item[(it + 1) & 1] = atomicAdd(next, 1ull);
    const uint32_t task = list[item];
    Acc ta;
    uint32_t t32 = 0;  // per-thread sum of one task: < 2^32 (kNarrowOld)
    if constexpr (BFLY_HUB_MATCH && !LOCAL && std::is_same_v<Src, HubSrc>) {
      auto cf = [&](uint32_t w, uint32_t n) {
        if constexpr (kNarrowOld<Tab>) t32 += tab.add(w, n);
        else ta.add(tab.add(w, n));
      };
      block_walk<BLOCK, false>(src, task, wsm, Combine<decltype(cf)>{cf}, LOCAL);
    } else if constexpr (BFLY_GROUP_WALK && !LOCAL && !Src::kExcl && !kMoments<Src>) {
      uint64_t ge0, ge1;
      src.entries(task, ge0, ge1);
      block_group_walk<BLOCK>(src, task, ge0, ge1, wsm, &s_claim, [&](uint32_t w) {
        if constexpr (kNarrowOld<Tab>) t32 += tab.inc(w);
        else ta.add(tab.inc(w));
      });
    } else if constexpr (BFLY_VEC4 && !LOCAL && Src::kVec4 && !kMoments<Src>) {
      uint64_t ve0, ve1;
      src.entries(task, ve0, ve1);
      auto vf = [&](uint32_t w) {
        if constexpr (kNarrowOld<Tab>) t32 += tab.inc(w);
        else ta.add(tab.inc(w));
      };
      constexpr int kVU = std::is_same_v<Tab, DirectByte> ? 1 : BFLY_VEC4_KU;
      block_walk_range_v4<BLOCK, Src, decltype(vf)&, kVU>(src, task, ve0, ve1, wsm, vf, false);
    } else {
      block_walk<BLOCK, false>(
          src, task, wsm,
          [&](uint32_t w, const uint32_t*, uint64_t) {
            if constexpr (kNarrowOld<Tab>) t32 += tab.inc(w);
            else ta.add(tab.inc(w));
          },
          LOCAL);
    }
    ta.add(t32);
    if (LOCAL) {
      block_walk<BLOCK>(
          src, task, wsm,
          [&](uint32_t w, const uint32_t* pe, uint64_t) { return emit_key(lo, pe, tab.get(w)); },
          false, Seg<EmitEntry>{EmitEntry{lo}});
    }
    __syncthreads();  // inserts done; walk state free
    if constexpr (LOCAL) {
      tab.drain(threadIdx.x, BLOCK, [&](uint32_t key, uint32_t c) {
        if (c >= 2) atomicAdd(&lo.vcnt[key], c2(c));  // rows: L2-resident here
      });
    } else if constexpr (kMoments<Src>) {
      tab.drain(threadIdx.x, BLOCK, [&](uint32_t, uint32_t c) { mom.add(c); });
    } else {
      tab.reset_all(threadIdx.x, BLOCK);  // counts were summed at insert: just zero
    }
    if (task_out) {  // exact per-task totals: one block reduction
      Acc r = block_sum<BLOCK>(ta, red, redo);
      if (threadIdx.x == 0) {
        task_out[task] = r.v;
        if (LOCAL && r.v) atomicAdd(&lo.vcnt[task], r.v);
        acc.add(r.v);
        acc.ovf |= r.ovf;
      }
    } else if (LOCAL) {  // the task's own count: one atomic per warp, no block barrier
      const Acc w = warp_sum(ta);
      if ((threadIdx.x & 31) == 0 && w.v) atomicAdd(&lo.vcnt[task], w.v);
      acc.add((threadIdx.x & 31) == 0 ? w.v : 0ull);
      acc.ovf |= w.ovf;
    } else {
      acc.add(ta.v);
    }
  }
  flush_acc(acc, total, ovf);
  if constexpr (kMoments<Src>) flush_mom(mom, lo.mom);
}

// ---- heavy (start tasks): split over CTAs, dense rows in global memory -----------------------
struct HeavyTask {
  uint32_t task, row;
  uint64_t e0, e1;  // entry range of this CTA
};

template <class Src, bool LOCAL, bool PASS2>
__global__ void __launch_bounds__(256) k_heavy(Src src, const HeavyTask* __restrict__ tasks,
                                               uint32_t* __restrict__ rows, uint64_t n_row,
                                               uint32_t* __restrict__ touched,
                                               unsigned long long* __restrict__ ntouched,
                                               unsigned long long* task_out,
                                               unsigned long long* total, unsigned* ovf,
                                               LocalOut lo,
                                               const unsigned long long* ntasks = nullptr) {
  if (ntasks && blockIdx.x >= *ntasks) return;  // device-built task list, grid = a bound
  const HeavyTask t = tasks[blockIdx.x];
  uint32_t* row = rows + (uint64_t)t.row * n_row;
  uint32_t* tl = touched + (uint64_t)t.row * n_row;
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5, W = blockDim.x >> 5;
  // contiguous sub-range of entries per warp, flattened across lanes
  const uint64_t n = t.e1 - t.e0;
  const uint64_t a = t.e0 + n * wl / W, b = t.e0 + n * (wl + 1) / W;
  Acc acc;
  if (!PASS2) {
    warp_walk_range(src, t.task, a, b, [&](uint32_t x, const uint32_t*, uint64_t) {
      const uint32_t old = atomicAdd(&row[x], 1u);
      acc.add(old);
      if (old == 0) tl[atomicAdd(&ntouched[t.row], 1ull)] = x;
    });
  } else {
    warp_walk_range(
        src, t.task, a, b,
        [&](uint32_t x, const uint32_t* pe, uint64_t) { return emit_key(lo, pe, row[x]); },
        Seg<EmitEntry>{EmitEntry{lo}});
  }
  (void)lane;
  if (!PASS2) {
    Acc w = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && w.v) {
      if (task_out) atomicAdd(&task_out[t.task], w.v);
      if (LOCAL) atomicAdd(&lo.vcnt[t.task], w.v);
    }
    flush_acc(acc, total, ovf);
  }
}

// ---- split (dense-key tasks): entry range per CTA, shared-memory table, merged in L2 -------
// A part's local counts m(x) are merged into the task's global row: atomicAdd returns the
// count o already merged by earlier parts, and o*m + C(m, 2) is exactly what the m increments
// would have contributed one by one (C(m, 2) is already in the part's running sum), so the
// task total is sum_x C(c(x), 2) however the entries are split. Only the distinct keys of a
// part touch L2 (k_heavy pays one L2 atomic per element).
template <class Src, bool LOCAL, class Tab, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_split(Src src, const HeavyTask* __restrict__ tasks,
                                                 uint32_t K, uint32_t* __restrict__ rows,
                                                 uint64_t n_row, uint32_t* __restrict__ touched,
                                                 unsigned long long* __restrict__ ntouched,
                                                 unsigned long long* task_out,
                                                 unsigned long long* total, unsigned* ovf,
                                                 LocalOut lo,
                                                 const unsigned long long* ntasks = nullptr) {
  if (ntasks && blockIdx.x >= *ntasks) return;  // device-built task list, grid = a bound
  extern __shared__ uint32_t smem[];
  Tab tab;
  tab.bind(smem, K);
  __shared__ BlockWalkSmem<BLOCK, typename ScanWord<Src, BLOCK>::T> wsm;
  __shared__ unsigned long long red[BLOCK / 32];
  __shared__ unsigned redo[BLOCK / 32];
  tab.init(threadIdx.x, BLOCK);
  __syncthreads();
  const HeavyTask t = tasks[blockIdx.x];
  uint32_t* row = rows + (uint64_t)t.row * n_row;
  uint32_t* tl = touched + (uint64_t)t.row * n_row;
  Acc ta;
  if constexpr (BFLY_VEC4 && Src::kVec4)
    block_walk_range_v4<BLOCK>(src, t.task, t.e0, t.e1, wsm, [&](uint32_t w) { ta.add(tab.inc(w)); },
                               false);
  else
    block_walk_range<BLOCK, false>(src, t.task, t.e0, t.e1, wsm,
                                   [&](uint32_t w, const uint32_t*, uint64_t) {
                                     ta.add(tab.inc(w));
                                   },
                                   false);
  __syncthreads();
  tab.drain(threadIdx.x, BLOCK, [&](uint32_t key, uint32_t c) {
    const uint32_t o = atomicAdd(&row[key], c);
    if (o == 0) tl[atomicAdd(&ntouched[t.row], 1ull)] = key;
    ta.add(static_cast<unsigned long long>(o) * c);
  });
  const Acc r = block_sum<BLOCK>(ta, red, redo);
  if (threadIdx.x == 0 && r.v) {
    if (task_out) atomicAdd(&task_out[t.task], r.v);
    if (LOCAL) atomicAdd(&lo.vcnt[t.task], r.v);
  }
  flush_acc(threadIdx.x == 0 ? r : Acc{}, total, ovf);
}

// per row r of the wave: optional LOCAL scatter of C(c,2) to the key vertex, then zero the
// touched entries and the touched counter
template <bool LOCAL>
__global__ void k_reset_rows(uint32_t* __restrict__ rows, uint64_t n_row,
                             const uint32_t* __restrict__ touched,
                             unsigned long long* __restrict__ ntouched, uint32_t row0,
                             LocalOut lo) {
  const uint32_t r = row0 + blockIdx.y;
  const unsigned long long nt = ntouched[r];
  Mom mom;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = touched[(uint64_t)r * n_row + i];
    uint32_t* cell = rows + (uint64_t)r * n_row + w;
    if (LOCAL && *cell >= 2) atomicAdd(&lo.vcnt[w], c2(*cell));
    if (lo.mom) mom.add(*cell);  // pair-moment runs: the final multiplicity of key w
    *cell = 0;
  }
  if (lo.mom) flush_mom(mom, lo.mom);  // (block-uniform branch; whole warps)
}

__global__ void k_zero_counters(unsigned long long* p, uint32_t n);

// (e0, e1) = (j, P) on input -> the j-th of P equal entry-count chunks of the task
template <class Src>
__global__ void k_heavy_ranges(Src src, HeavyTask* __restrict__ t, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = t[i].e0, P = t[i].e1;
    uint64_t E0, E1;
    src.entries(t[i].task, E0, E1);
    const uint64_t len = E1 - E0;
    t[i].e0 = E0 + len * j / P;
    t[i].e1 = E0 + len * (j + 1) / P;
  }
}

// parts of heavy task i: enough kHeavyChunk-key (and, with split > 0, split-entry) ranges
__device__ __forceinline__ uint32_t heavy_parts(unsigned long long keys, unsigned long long units,
                                                uint64_t split) {
  uint64_t parts = (keys + kHeavyChunk - 1) / kHeavyChunk;
  if (split) {
    const uint64_t by_units = (units + split - 1) / split;
    if (by_units > parts) parts = by_units;
  }
  if (parts < 1) parts = 1;
  if (parts > 4096) parts = 4096;
  return static_cast<uint32_t>(parts);
}

static __global__ void k_heavy_parts(const unsigned long long* __restrict__ hw,
                              const unsigned long long* __restrict__ hu, uint64_t nh,
                              uint64_t split, unsigned long long* __restrict__ parts) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nh;
       i += (uint64_t)gridDim.x * blockDim.x)
    parts[i] = i < nh ? heavy_parts(hw[i], hu[i], split) : 0ull;
}

// heavy task i (row i) -> its parts at pstart[i] .. with their entry ranges; warp per task
template <class Src>
__global__ void k_heavy_build(Src src, const uint32_t* __restrict__ hl,
                              const unsigned long long* __restrict__ hw,
                              const unsigned long long* __restrict__ hu, uint64_t nh,
                              uint64_t split, const unsigned long long* __restrict__ pstart,
                              HeavyTask* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nh; i += nw) {
    const uint32_t P = heavy_parts(hw[i], hu[i], split);
    uint64_t E0, E1;
    src.entries(hl[i], E0, E1);
    const uint64_t len = E1 - E0, base = pstart[i];
    for (uint32_t j = lane; j < P; j += 32)
      out[base + j] = {hl[i], static_cast<uint32_t>(i), E0 + len * j / P, E0 + len * (j + 1) / P};
  }
}

// ---- element-balanced heavy parts (start / sample / pair tasks) -------------------------------
// A heavy task can hold few entries with huge segments (a vertex sample next to a hub walks
// the hub's whole list through ONE entry), so its parts are cut in the flattened element
// space, not by entries: part j of task i covers elements [X j / P, X (j+1) / P) of the
// concatenated segments, X = the task's element count, P = ceil(X / kHeavyChunk). A part
// boundary is an (entry, offset in its segment) pair; a CTA walks its part with the block walk
// over a source whose first and last segments are clipped to the part.
struct HeavyBound {
  uint64_t e;    // entry holding the boundary element
  uint32_t off;  // offset of the boundary element in that entry's segment
  uint32_t pad;
};
struct HeavyPart {
  uint32_t task, row;
  uint64_t b;  // index of the part's first boundary (its end is b + 1)
};

template <class S>
struct PartSrc {
  S s;
  uint64_t e_first, e_last;
  uint32_t off_first, off_last;  // elements [off_first, ...) of e_first, [0, off_last) of e_last
  __device__ __forceinline__ uint32_t seg(uint32_t task, uint64_t e, const uint32_t*& p) const {
    const uint32_t len = s.seg(task, e, p);
    const uint32_t lo = e == e_first ? off_first : 0u;
    uint32_t hi = e == e_last ? off_last : len;
    if (hi > len) hi = len;
    if (lo >= hi) return 0u;
    p += lo;
    return hi - lo;
  }
  static constexpr bool kExcl = S::kExcl;
  static constexpr bool kNarrowScan = S::kNarrowScan;
  static constexpr bool kVec4 = false;  // (clipped segments)
  __device__ __forceinline__ uint32_t excl(uint32_t task) const { return s.excl(task); }
};

// warp per heavy task: X = element count, P = parts
template <class Src>
__global__ void k_heavy_sizes(Src src, const uint32_t* __restrict__ hl, uint64_t nh,
                              unsigned long long* __restrict__ X,
                              unsigned long long* __restrict__ P) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i <= nh; i += nw) {
    if (i == nh) {
      if (lane == 0) P[nh] = 0;  // (exclusive-scan sentinel)
      continue;
    }
    uint64_t E0, E1;
    src.entries(hl[i], E0, E1);
    unsigned long long x = 0;
    for (uint64_t e = E0 + lane; e < E1; e += 32) {
      const uint32_t* p;
      x += src.seg(hl[i], e, p);
    }
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) {
      X[i] = x;
      const unsigned long long parts = (x + kHeavyChunk - 1) / kHeavyChunk;
      P[i] = parts ? parts : 1ull;
    }
  }
}

// warp per heavy task: its P + 1 part boundaries at bnd[pstart[i] + i ...]
template <class Src>
__global__ void k_heavy_bounds(Src src, const uint32_t* __restrict__ hl, uint64_t nh,
                               const unsigned long long* __restrict__ X,
                               const unsigned long long* __restrict__ pstart,
                               HeavyBound* __restrict__ bnd) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nh; i += nw) {
    uint64_t E0, E1;
    src.entries(hl[i], E0, E1);
    const unsigned long long x = X[i], P = pstart[i + 1] - pstart[i];
    HeavyBound* out = bnd + pstart[i] + i;
    if (x == 0) {  // nothing to walk: one empty part
      if (lane == 0) {
        out[0] = {E0, 0u, 0u};
        out[1] = {E1, 0u, 0u};
      }
      continue;
    }
    unsigned long long s = 0;  // elements before this batch of entries
    for (uint64_t eb = E0; eb < E1; eb += 32) {
      const uint64_t e = eb + lane;
      uint32_t len = 0;
      if (e < E1) {
        const uint32_t* p;
        len = src.seg(hl[i], e, p);
      }
      unsigned long long incl = len;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      const unsigned long long se = s + incl - len;  // this entry's elements: [se, se + len)
      if (len) {
        // boundaries k < P with x_k = floor(x k / P) in [se, se + len)
        unsigned long long k = (se * P + x - 1) / x;  // smallest k with x k / P >= se
        for (; k < P; ++k) {
          const unsigned long long xk = x * k / P;
          if (xk >= se + len) break;
          out[k] = {e, static_cast<uint32_t>(xk - se), 0u};
        }
      }
      s += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) out[P] = {E1, 0u, 0u};
  }
}

// one CTA per part: the block walk over the part's clipped entries; dense rows in L2
template <class Src, bool LOCAL, bool PASS2>
__global__ void __launch_bounds__(256) k_heavy_el(Src src, const HeavyPart* __restrict__ parts,
                                                  const HeavyBound* __restrict__ bnd,
                                                  uint32_t* __restrict__ rows, uint64_t n_row,
                                                  uint32_t* __restrict__ touched,
                                                  unsigned long long* __restrict__ ntouched,
                                                  unsigned long long* task_out,
                                                  unsigned long long* total, unsigned* ovf,
                                                  LocalOut lo) {
  using PS = PartSrc<Src>;
  __shared__ BlockWalkSmem<256, typename ScanWord<PS, 256>::T> wsm;
  const HeavyPart t = parts[blockIdx.x];
  const HeavyBound b0 = bnd[t.b], b1 = bnd[t.b + 1];
  const PS ps{src, b0.e, b1.e, b0.off, b1.off};
  const uint64_t e_end = b1.e + (b1.off > 0 ? 1 : 0);
  uint32_t* row = rows + (uint64_t)t.row * n_row;
  uint32_t* tl = touched + (uint64_t)t.row * n_row;
  Acc acc;
  (void)tl;
  (void)ntouched;
  if (!PASS2) {
    // branch-free: the old value only feeds the sum, so a warp keeps several L2 atomics in
    // flight (the touched keys are found again by k_heavy_el_drain's walk, not listed here)
    auto f = [&](uint32_t x, const uint32_t*, uint64_t) { acc.add(atomicAdd(&row[x], 1u)); };
    block_walk_range<256, false, PS, decltype(f)&, NoSeg, 8>(ps, t.task, b0.e, e_end, wsm, f);
    const Acc w = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && w.v) {
      if (task_out) atomicAdd(&task_out[t.task], w.v);
      if (LOCAL) atomicAdd(&lo.vcnt[t.task], w.v);
    }
    flush_acc(acc, total, ovf);
  } else {
    block_walk_range<256>(
        ps, t.task, b0.e, e_end, wsm,
        [&](uint32_t x, const uint32_t* pe, uint64_t) { return emit_key(lo, pe, row[x]); }, true,
        Seg<EmitEntry>{EmitEntry{lo}});
  }
}

// after a wave: every part walks its elements again and takes its keys' final counts out of
// the row with atomicExch (the first walker of a key gets c, later ones 0): LOCAL scatters
// C(c,2) to the key vertex, pair-moment runs add C(c,3) / C(c,4); the row is zero again
template <class Src, bool LOCAL>
__global__ void __launch_bounds__(256) k_heavy_el_drain(Src src, const HeavyPart* __restrict__ parts,
                                                        const HeavyBound* __restrict__ bnd,
                                                        uint32_t* __restrict__ rows, uint64_t n_row,
                                                        LocalOut lo) {
  using PS = PartSrc<Src>;
  __shared__ BlockWalkSmem<256, typename ScanWord<PS, 256>::T> wsm;
  const HeavyPart t = parts[blockIdx.x];
  const HeavyBound b0 = bnd[t.b], b1 = bnd[t.b + 1];
  const PS ps{src, b0.e, b1.e, b0.off, b1.off};
  const uint64_t e_end = b1.e + (b1.off > 0 ? 1 : 0);
  uint32_t* row = rows + (uint64_t)t.row * n_row;
  Mom mom;
  auto f = [&](uint32_t x, const uint32_t*, uint64_t) {
    const uint32_t c = atomicExch(&row[x], 0u);
    if (LOCAL && c >= 2) atomicAdd(&lo.vcnt[x], c2(c));
    if (lo.mom) mom.add(c);
  };
  block_walk_range<256, false, PS, decltype(f)&, NoSeg, 8>(ps, t.task, b0.e, e_end, wsm, f);
  if (lo.mom) flush_mom(mom, lo.mom);
}

// drain of whole rows (rows listed in row_ids, blockIdx.y picks one): every nonzero counter
// is a touched key with its final count; LOCAL / pair-moment contributions, then zero
template <bool LOCAL>
__global__ void __launch_bounds__(256) k_row_drain(uint32_t* __restrict__ rows, uint64_t n_row,
                                                   const uint32_t* __restrict__ row_ids,
                                                   LocalOut lo) {
  uint32_t* row = rows + (uint64_t)row_ids[blockIdx.y] * n_row;
  Mom mom;
  const uint64_t n4 = n_row / 4;  // aligned part (n_row of a row start: row * n_row words)
  const bool aligned = ((reinterpret_cast<uintptr_t>(row) & 15u) == 0);
  const uint64_t vec = aligned ? n4 : 0;
  uint4* r4 = reinterpret_cast<uint4*>(row);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < vec;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = r4[i];
    if ((v.x | v.y | v.z | v.w) == 0) continue;
    const uint32_t c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (LOCAL && c[j] >= 2) atomicAdd(&lo.vcnt[i * 4 + j], c2(c[j]));
      if (lo.mom) mom.add(c[j]);
    }
    r4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (uint64_t i = vec * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_row;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = row[i];
    if (!c) continue;
    if (LOCAL && c >= 2) atomicAdd(&lo.vcnt[i], c2(c));
    if (lo.mom) mom.add(c);
    row[i] = 0u;
  }
  if (lo.mom) flush_mom(mom, lo.mom);
}

// ---- bucketing ---------------------------------------------------------------------------
// Buckets: 0 tiny, 1 small-A, 2 small-B, 3 medium, 4 medium-wide, 5 heavy.
// counts[6] tasks, wsum[6] keys, esum[6] entries (units may be null) per bucket;
// bucket q = first q with work <= lim[q] (heavy otherwise); a medium task with
// units >= wide_units (when nonzero) is medium-wide; tasks below skip_below are skipped
constexpr int kBuckets = 6;
__global__ void k_bucket(const unsigned long long* __restrict__ work,
                         const unsigned long long* __restrict__ units, uint64_t n,
                         uint64_t lim0, uint64_t lim1, uint64_t lim2, uint64_t lim3,
                         uint64_t wide_units, uint64_t wide_work, uint64_t split_units,
                         uint64_t skip_below, uint32_t* __restrict__ lists,
                         unsigned long long* __restrict__ counts,
                         unsigned long long* __restrict__ wsum,
                         unsigned long long* __restrict__ esum,
                         unsigned long long* __restrict__ heavy_work,
                         unsigned long long* __restrict__ heavy_units);

// ---- host orchestration ------------------------------------------------------------------
// reported per bucket (kBuckets order): tiny, small-A, small-B, medium, medium-wide, heavy
struct RunStats {
  uint64_t starts[6] = {};
  uint64_t wedges[6] = {};
  uint64_t entries[6] = {};
};

// warp-table policies (small-A, small-B), CTA-table policy and bucket limits of one run
// With wide_units != 0, medium tasks with >= wide_units entries run as a second medium launch
// with WideTab (wider counters); the rest keep MedTab (narrow counters, valid while a key's
// multiplicity stays below wide_units).
template <class SmallTab, class SmallTabB, class MedTab, class WideTab = MedTab>
struct Plan {
  uint32_t K;             // table geometry (K | K1 << 16) for Direct*/BitHash; Hash ignores it
  uint64_t lim[4];        // tiny / small-A / small-B / medium work limits; above -> heavy
  uint64_t skip_below;    // tasks with id < skip_below are not processed
  int med_block = kMedBlock;  // CTA size of the medium bucket (256 or 512)
  uint64_t wide_units = 0;    // see above
  // split_units != 0: medium tasks with >= split_units entries join the heavy bucket, and the
  // heavy bucket runs k_split with MedTab/WideTab-free SplitTab = WideTab (entry-range parts
  // of about split_units entries, merged in global rows of n_row counters)
  uint64_t split_units = 0;
  uint64_t wide_work = 0;  // != 0: medium tasks with more keys than this are medium-wide
  int wide_block = 0;      // CTA size of the medium-wide launch (0: med_block)
};

// Process-wide heavy-row scratch per device (zero-invariant between calls; exact.cu).
struct RowScratch {
  std::recursive_mutex mu;  // a thread may hold it for two runs (count_all_starts)
  uint32_t* rows = nullptr;
  uint32_t* touched = nullptr;
  unsigned long long* ntouched = nullptr;
  uint64_t cap_words = 0;
};
RowScratch& row_scratch(int device);
uint32_t ensure_rows(RowScratch& rs, uint64_t n_row, uint64_t need, cudaStream_t s);

// per-device side streams of the aggregation runs (created once, never destroyed); the fork
// and join events are per call, so concurrent calls from several host threads stay ordered
// resident CTAs per SM a bucket kernel's grid is sized for: its occupancy, capped by
// BFLY_CAP_<kernel name> (e.g. BFLY_CAP_hub_small=3) -- the bucket kernels of a counting phase
// share the SMs, and a kernel sized to fill them alone keeps the later ones out until its
// CTAs retire
inline int ctas_per_sm(const char* name, int occupancy) {
  const std::string key = std::string("BFLY_CAP_") + name;
  const char* e = std::getenv(key.c_str());
  const int cap = e ? std::atoi(e) : 0;
  return std::max(1, cap > 0 ? std::min(cap, occupancy) : occupancy);
}

struct SideStreams {
  static constexpr int kN = 12;  // two runs of five bucket streams + the dense hub kernels
  cudaStream_t s[kN];
};
struct ForkJoin {
  cudaEvent_t fork = nullptr, join[5] = {};
  ForkJoin() {
    BFLY_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (auto& e : join) BFLY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~ForkJoin() {
    cudaEventDestroy(fork);
    for (auto& e : join) cudaEventDestroy(e);
  }
  ForkJoin(const ForkJoin&) = delete;
  ForkJoin& operator=(const ForkJoin&) = delete;
};
inline SideStreams& side_streams(int device) {
  static std::mutex mu;
  static SideStreams* per[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  SideStreams*& p = per[device & 63];
  if (!p) {
    p = new SideStreams;
    for (int q = 0; q < SideStreams::kN; ++q)
      BFLY_CUDA(cudaStreamCreateWithFlags(&p->s[q], cudaStreamNonBlocking));
  }
  return *p;
}
inline bool agg_concurrent() {
  static const bool v = [] {
    const char* e = std::getenv("BFLY_AGG_CONCURRENT");
    return !(e && e[0] == '0');
  }();
  return v;
}

// One aggregation run over the tasks of a source, in three steps so that several runs can
// share their host synchronisations and overlap on the device (count_all_starts):
//   constructor   launches the bucketing kernel (no sync)
//   counts_item   -> read_back the per-bucket task / key / entry counts
//   start(base)   launches every bucket's kernel: buckets 0-4 on side streams base..base+4
//                 (forked from the graph stream), the heavy bucket on the graph stream
//   join()        makes the graph stream wait for the side streams
//   total_item    -> read_back (total, overflow flag); result() checks and returns it
template <class Src, bool LOCAL, class SmallTab, class SmallTabB, class MedTab, class WideTab>
struct Agg {
  bfly_graph* g;
  cudaStream_t s;
  Src src;
  Plan<SmallTab, SmallTabB, MedTab, WideTab> plan;
  const unsigned long long* d_work;
  const unsigned long long* d_units;
  uint64_t ntask, n_row;
  unsigned long long* d_task_out;
  LocalOut lo;
  RunStats* rs;
  const char* const* names;
  // [0,6) tasks, [6,12) keys, [12,18) entries, [18] total, [19] ovf, [20] medium queue,
  // [21] medium-wide queue
  DBuf<unsigned long long> ctl;
  DBuf<uint32_t> lists;
  DBuf<unsigned long long> heavy_work, heavy_units;
  DBuf<HeavyTask> dtasks;
  std::unique_lock<std::recursive_mutex> rows_lock;  // held until the final synchronisation
  unsigned long long hh[18] = {};
  unsigned long long h[6] = {};
  unsigned long long res[2] = {};
  ForkJoin fj;
  bool conc = false;
  int base = 0;

  Agg(bfly_graph* g_, const Src& src_, const Plan<SmallTab, SmallTabB, MedTab, WideTab>& plan_,
      const unsigned long long* d_work_, const unsigned long long* d_units_, uint64_t ntask_,
      uint64_t n_row_, unsigned long long* d_task_out_, LocalOut lo_, RunStats* rs_,
      const char* const names_[8])
      : g(g_), s(g_->stream), src(src_), plan(plan_), d_work(d_work_), d_units(d_units_),
        ntask(ntask_), n_row((n_row_ + 3) & ~uint64_t{3}),  // row stride: whole uint4s
        d_task_out(d_task_out_), lo(lo_), rs(rs_), names(names_) {
    if (ntask == 0) return;
    // [0,6) tasks, [6,12) keys, [12,18) entries, [18] total, [19] ovf, [20] medium queue,
    // [21] medium-wide queue
    ctl.alloc(22, s);
    ctl.zero();
    unsigned long long* counts = ctl.p;
    unsigned long long* wsum = ctl.p + 6;
    unsigned long long* esum = ctl.p + 12;
    lists.alloc(kBuckets * ntask, s);
    heavy_work.alloc(ntask, s);
    heavy_units.alloc(ntask, s);
    launch(names[0], k_bucket, grid_for(ntask, 256), 256, 0, s, d_work, d_units, ntask, plan.lim[0],
           plan.lim[1], plan.lim[2], plan.lim[3], plan.wide_units, plan.wide_work, plan.split_units,
           plan.skip_below,
           lists.p, counts, wsum, esum,
           heavy_work.p, heavy_units.p);
  }
  ReadBack::Item counts_item() { return {hh, ctl.p, sizeof(hh)}; }
  ReadBack::Item total_item() { return {res, ctl.p + 18, sizeof(res)}; }

  void start(SideStreams& ss, int base_) {
    if (ntask == 0) return;
    base = base_;
    unsigned long long* total = ctl.p + 18;
    unsigned* ovf = reinterpret_cast<unsigned*>(ctl.p + 19);
    unsigned long long* next = ctl.p + 20;
    // The buckets' kernels are independent (own task lists and queues, atomic shared totals):
    // each runs on its own side stream, so one bucket's tail overlaps the next one's start and
    // kernels with different bottlenecks share the SMs. join() makes the graph stream wait.
    conc = agg_concurrent();
    if (conc) {
      BFLY_CUDA(cudaEventRecord(fj.fork, s));
      for (int q = 0; q < 5; ++q) BFLY_CUDA(cudaStreamWaitEvent(ss.s[base + q], fj.fork, 0));
    }
    auto on = [&](int q) { return conc ? ss.s[base + q] : s; };
    trace_mark(names[0]);
    if (rs) {
      for (int q = 0; q < kBuckets; ++q) {
        rs->starts[q] += hh[q];
        rs->wedges[q] += hh[6 + q];
        rs->entries[q] += hh[12 + q];
      }
    }
    // h[]: tiny, small-A, small-B, medium, medium-wide, heavy task counts
    for (int q = 0; q < 6; ++q) h[q] = hh[q];
    cudaStream_t ls = on(0);
    if (h[0])
      launch(names[1], k_tiny<Src, LOCAL>, grid_for(h[0] * 32, 256, 148u * 64u), 256, 0, ls, src,
             lists.p, (uint64_t)h[0], d_task_out, total, ovf, lo);
    auto small = [&](auto kern, uint64_t cnt, const uint32_t* lst, size_t words, const char* nm) {
      const size_t sm = kSmallWarps * ((words + 3) & ~size_t{3}) * 4;
      BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSmallWarps * 32, sm);
      launch(nm, kern, grid_for(cnt * 32, kSmallWarps * 32, 148u * ctas_per_sm(nm, per_sm)),
             kSmallWarps * 32, sm, ls, src, lst, cnt, plan.K, d_task_out, total, ovf, lo);
    };
    ls = on(1);
    if (h[1])
      small(k_small<Src, LOCAL, SmallTab>, h[1], lists.p + ntask, SmallTab::words(plan.K), names[2]);
    ls = on(2);
    if (h[2])
      small(k_small<Src, LOCAL, SmallTabB>, h[2], lists.p + 2 * ntask, SmallTabB::words(plan.K),
            names[7]);
    auto medium = [&](auto tab, unsigned long long cnt, const uint32_t* lst,
                      unsigned long long* queue, const char* name, int blk) {
      using Tab = decltype(tab);
      const size_t sm = Tab::words(plan.K) * 4;
      auto go = [&](auto kern, int block) {
        BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, sm);
        const unsigned grid = static_cast<unsigned>(
            std::min<unsigned long long>(cnt, 148ull * ctas_per_sm(name, per_sm)));
        launch(name, kern, grid, block, sm, ls, src, lst, (uint64_t)cnt, plan.K, queue, d_task_out,
               total, ovf, lo);
      };
      if (blk == 256) go(k_medium<Src, LOCAL, Tab, 256>, 256);
      else if (blk == 128) go(k_medium<Src, LOCAL, Tab, 128>, 128);
      else if (blk == 1024) go(k_medium<Src, LOCAL, Tab, 1024>, 1024);
      else go(k_medium<Src, LOCAL, Tab, kMedBlock>, kMedBlock);
    };
    ls = on(3);
    if (h[3]) medium(MedTab{}, h[3], lists.p + 3 * ntask, next, names[3], plan.med_block);
    ls = on(4);
    if (h[4])
      medium(WideTab{}, h[4], lists.p + 4 * ntask, ctl.p + 21, names[4],
             plan.wide_block ? plan.wide_block : plan.med_block);
    bool heavy_on_device = false;
    if (h[5] && plan.split_units) {
      // split tasks: one row per task, the part list built on the device (no host round trip);
      // the grid is a bound from the bucket sums, surplus CTAs exit at once
      RowScratch& scr = row_scratch(g->device);
      rows_lock = std::unique_lock<std::recursive_mutex>(scr.mu);
      const uint32_t slots = ensure_rows(scr, n_row, h[5], s);
      if (h[5] <= slots) {
        heavy_on_device = true;
        const uint64_t nh = h[5];
        DBuf<unsigned long long> parts(nh + 1, s), pstart(nh + 1, s);
        launch("agg_heavy_parts", k_heavy_parts, grid_for(nh + 1, 256), 256, 0, s, heavy_work.p,
               heavy_units.p, nh, plan.split_units, parts.p);
        exclusive_sum(parts.p, pstart.p, nh + 1, s);
        const uint64_t bound = hh[6 + 5] / kHeavyChunk + hh[12 + 5] / plan.split_units + 2 * nh + 1;
        dtasks.alloc(bound, s);
        launch("agg_heavy_build", k_heavy_build<Src>, grid_for(nh * 32, 256), 256, 0, s, src,
               lists.p + 5 * ntask, heavy_work.p, heavy_units.p, nh, plan.split_units, pstart.p,
               dtasks.p);
        const unsigned long long* ntasks = pstart.p + nh;
        auto kern = k_split<Src, LOCAL, WideTab, 256>;
        const size_t sm = WideTab::words(plan.K) * 4;
        BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        launch(names[5], kern, static_cast<unsigned>(bound), 256, sm, s, src, dtasks.p, plan.K,
               scr.rows, n_row, scr.touched, scr.ntouched, d_task_out, total, ovf, lo, ntasks);
        if (LOCAL)
          launch("agg_heavy_local", k_heavy<Src, LOCAL, true>, static_cast<unsigned>(bound), 256, 0,
                 s, src, dtasks.p, scr.rows, n_row, scr.touched, scr.ntouched, d_task_out, total,
                 ovf, lo, ntasks);
        launch("agg_reset_rows", k_reset_rows<LOCAL>, dim3(148, static_cast<unsigned>(nh)), 256, 0, s,
               scr.rows, n_row, scr.touched, scr.ntouched, 0u, lo);
        launch("agg_zero_counters", k_zero_counters, 1, 64, 0, s, scr.ntouched,
               static_cast<uint32_t>(nh));
        // (pstart / parts are released in stream order; dtasks lives until the final sync)
      } else {
        rows_lock.unlock();
      }
    }
    if (h[5] && !heavy_on_device && !plan.split_units) {
      // element-balanced parts built on the device; tasks grouped into waves of rows on the host
      const uint64_t nh = h[5];
      const uint32_t* hl = lists.p + 5 * ntask;
      DBuf<unsigned long long> X(nh + 1, s), pc(nh + 1, s), ps(nh + 1, s);
      launch("agg_heavy_sizes", k_heavy_sizes<Src>, grid_for((nh + 1) * 32, 256), 256, 0, s, src,
             hl, nh, X.p, pc.p);
      exclusive_sum(pc.p, ps.p, nh + 1, s);
      std::vector<unsigned long long> hx(nh), hps(nh + 1);
      std::vector<uint32_t> htask(nh);
      read_back(s, {{hx.data(), X.p, nh * 8}, {hps.data(), ps.p, (nh + 1) * 8},
                    {htask.data(), hl, nh * 4}});
      const uint64_t nparts = hps[nh];
      DBuf<HeavyBound> bnd(nparts + nh, s);
      launch("agg_heavy_bounds", k_heavy_bounds<Src>, grid_for(nh * 32, 256), 256, 0, s, src, hl,
             nh, (const unsigned long long*)X.p, (const unsigned long long*)ps.p, bnd.p);
      RowScratch& scr = row_scratch(g->device);
      if (!rows_lock.owns_lock()) rows_lock = std::unique_lock<std::recursive_mutex>(scr.mu);
      const uint32_t slots = ensure_rows(scr, n_row, nh, s);
      std::vector<uint32_t> order(nh);
      for (uint32_t i = 0; i < nh; ++i) order[i] = i;
      std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return hx[a] > hx[b]; });
      // waves: at most `slots` rows and about 32M touched keys (row sectors kept in L2)
      const uint64_t wave_keys = 32ull << 20;
      // Every part goes to `parts` (the counting walk); a task's keys are then drained either
      // by scanning its whole row (tasks with at least n_row / 10 elements: a coalesced read of
      // the row is cheaper than re-walking them) or by a second walk of its parts (`dparts2`).
      std::vector<HeavyPart> parts, parts2;
      std::vector<uint32_t> scan_rows;
      parts.reserve(nparts);
      struct Wave {
        size_t p0, p1, q0, q1, r0, r1;
        uint32_t rows;
      };
      std::vector<Wave> waves;
      size_t q = 0;
      while (q < order.size()) {
        Wave wv{parts.size(), 0, parts2.size(), 0, scan_rows.size(), 0, 0};
        uint64_t budget = 0;
        while (q < order.size() && wv.rows < slots &&
               (wv.rows == 0 || budget + std::min<uint64_t>(hx[order[q]], n_row) <= wave_keys)) {
          const uint32_t i = order[q];
          budget += std::min<uint64_t>(hx[i], n_row);
          const uint64_t b0 = hps[i] + i, P = hps[i + 1] - hps[i];
          const bool by_scan = hx[i] >= n_row / 10;
          for (uint64_t j = 0; j < P; ++j) {
            parts.push_back({htask[i], wv.rows, b0 + j});
            if (!by_scan) parts2.push_back({htask[i], wv.rows, b0 + j});
          }
          if (by_scan) scan_rows.push_back(wv.rows);
          ++wv.rows;
          ++q;
        }
        wv.p1 = parts.size();
        wv.q1 = parts2.size();
        wv.r1 = scan_rows.size();
        waves.push_back(wv);
      }
      DBuf<HeavyPart> dparts(parts.size() ? parts.size() : 1, s);
      DBuf<HeavyPart> dparts2(parts2.size() ? parts2.size() : 1, s);
      DBuf<uint32_t> drows(scan_rows.size() ? scan_rows.size() : 1, s);
      BFLY_CUDA(cudaMemcpyAsync(dparts.p, parts.data(), parts.size() * sizeof(HeavyPart),
                                cudaMemcpyHostToDevice, s));
      if (!parts2.empty())
        BFLY_CUDA(cudaMemcpyAsync(dparts2.p, parts2.data(), parts2.size() * sizeof(HeavyPart),
                                  cudaMemcpyHostToDevice, s));
      if (!scan_rows.empty())
        BFLY_CUDA(cudaMemcpyAsync(drows.p, scan_rows.data(), scan_rows.size() * 4,
                                  cudaMemcpyHostToDevice, s));
      for (const Wave& wv : waves) {
        const unsigned np = static_cast<unsigned>(wv.p1 - wv.p0);
        launch(names[5], k_heavy_el<Src, LOCAL, false>, np, 256, 0, s, src, dparts.p + wv.p0,
               (const HeavyBound*)bnd.p, scr.rows, n_row, scr.touched, scr.ntouched, d_task_out,
               total, ovf, lo);
        if (LOCAL)
          launch("agg_heavy_local", k_heavy_el<Src, LOCAL, true>, np, 256, 0, s, src,
                 dparts.p + wv.p0, (const HeavyBound*)bnd.p, scr.rows, n_row, scr.touched,
                 scr.ntouched, d_task_out, total, ovf, lo);
        if (wv.q1 > wv.q0)
          launch("agg_heavy_drain", k_heavy_el_drain<Src, LOCAL>, static_cast<unsigned>(wv.q1 - wv.q0),
                 256, 0, s, src, dparts2.p + wv.q0, (const HeavyBound*)bnd.p, scr.rows, n_row, lo);
        if (wv.r1 > wv.r0)
          launch("agg_heavy_drain", k_row_drain<LOCAL>,
                 dim3(static_cast<unsigned>(std::min<uint64_t>(1024, (n_row + 4095) / 4096)),
                      static_cast<unsigned>(wv.r1 - wv.r0)),
                 256, 0, s, scr.rows, n_row, (const uint32_t*)drows.p + wv.r0, lo);
      }
      // (the part list, bounds and sizes are released in stream order; the pageable part
      // vector was staged by cudaMemcpyAsync before it returned)
    }
    if (h[5] && !heavy_on_device && plan.split_units) {
      std::vector<uint32_t> hl(h[5]);
      std::vector<unsigned long long> hw(h[5]), hu(h[5]);
      read_back(s, {{hl.data(), lists.p + 5 * ntask, h[5] * 4}, {hw.data(), heavy_work.p, h[5] * 8}, {hu.data(), heavy_units.p, h[5] * 8}});
      RowScratch& scr = row_scratch(g->device);
      if (!rows_lock.owns_lock()) rows_lock = std::unique_lock<std::recursive_mutex>(scr.mu);
      const uint32_t slots = ensure_rows(scr, n_row, h[5], s);
      std::vector<uint32_t> order(h[5]);
      for (uint32_t i = 0; i < h[5]; ++i) order[i] = i;
      std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return hw[a] > hw[b]; });
      // waves: at most `slots` rows and about 2M distinct keys (touched sectors) in flight for
      // the per-element L2 atomics of k_heavy; k_split touches L2 once per distinct key of a part
      const uint64_t wave_keys = plan.split_units ? (256ull << 20) : (2ull << 20);
      struct Wave {
        size_t t0, t1;
        uint32_t rows;
      };
      std::vector<Wave> waves;
      std::vector<HeavyTask> tasks;  // (e0, e1) hold (j, P) until k_heavy_ranges resolves them
      size_t q = 0;
      while (q < order.size()) {
        Wave wv{tasks.size(), 0, 0};
        uint64_t budget = 0;
        while (q < order.size() && wv.rows < slots &&
               (wv.rows == 0 || budget + std::min<uint64_t>(hw[order[q]], n_row) <= wave_keys)) {
          budget += std::min<uint64_t>(hw[order[q]], n_row);
          uint64_t parts = (hw[order[q]] + kHeavyChunk - 1) / kHeavyChunk;
          if (plan.split_units)
            parts = std::max<uint64_t>(parts, (hu[order[q]] + plan.split_units - 1) / plan.split_units);
          const uint32_t P = static_cast<uint32_t>(std::min<uint64_t>(4096, parts));
          for (uint32_t j = 0; j < P; ++j)
            tasks.push_back({hl[order[q]], wv.rows, j, P});  // e0/e1 filled on device
          ++wv.rows;
          ++q;
        }
        wv.t1 = tasks.size();
        waves.push_back(wv);
      }
      dtasks.alloc(tasks.size(), s);
      BFLY_CUDA(cudaMemcpyAsync(dtasks.p, tasks.data(), tasks.size() * sizeof(HeavyTask),
                                cudaMemcpyHostToDevice, s));
      launch("agg_heavy_ranges", k_heavy_ranges<Src>, grid_for(tasks.size(), 256), 256, 0, s, src,
             dtasks.p, (uint64_t)tasks.size());
      for (const Wave& wv : waves) {
        const unsigned nt = static_cast<unsigned>(wv.t1 - wv.t0);
        if (plan.split_units) {
          auto kern = k_split<Src, LOCAL, WideTab, 256>;
          const size_t sm = WideTab::words(plan.K) * 4;
          BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          launch(names[5], kern, nt, 256, sm, s, src, dtasks.p + wv.t0, plan.K, scr.rows, n_row,
                 scr.touched, scr.ntouched, d_task_out, total, ovf, lo,
                 (const unsigned long long*)nullptr);
        } else {
          launch(names[5], k_heavy<Src, LOCAL, false>, nt, 256, 0, s, src, dtasks.p + wv.t0,
                 scr.rows, n_row, scr.touched, scr.ntouched, d_task_out, total, ovf, lo,
                 (const unsigned long long*)nullptr);
        }
        if (LOCAL)
          launch("agg_heavy_local", k_heavy<Src, LOCAL, true>, nt, 256, 0, s, src, dtasks.p + wv.t0,
                 scr.rows, n_row, scr.touched, scr.ntouched, d_task_out, total, ovf, lo,
                 (const unsigned long long*)nullptr);
        const dim3 rg(148, wv.rows);
        launch("agg_reset_rows", k_reset_rows<LOCAL>, rg, 256, 0, s, scr.rows, n_row, scr.touched,
               scr.ntouched, 0u, lo);
        launch("agg_zero_counters", k_zero_counters, 1, 64, 0, s, scr.ntouched, wv.rows);
      }
    }
  }

  void join(SideStreams& ss) {
    if (ntask == 0 || !conc) return;
    for (int q = 0; q < 5; ++q) {
      BFLY_CUDA(cudaEventRecord(fj.join[q], ss.s[base + q]));
      BFLY_CUDA(cudaStreamWaitEvent(s, fj.join[q], 0));
    }
  }

  uint64_t result() {
    if (ntask == 0) return 0;
    trace_mark(names[5]);
    if (static_cast<unsigned>(res[1]) != 0) fail(kOverflow, "64-bit counter overflow in addition");
    return res[0];
  }
};

// one run on its own (bucket, counts, kernels, total), names[6] timing its counting phase
template <class Src, bool LOCAL, class SmallTab, class SmallTabB, class MedTab, class WideTab>
uint64_t run(bfly_graph* g, const Src& src,
             const Plan<SmallTab, SmallTabB, MedTab, WideTab>& plan,
             const unsigned long long* d_work, const unsigned long long* d_units, uint64_t ntask,
             uint64_t n_row, unsigned long long* d_task_out, LocalOut lo, RunStats* rs,
             const char* const names[8]) {
  if (ntask == 0) return 0;
  Agg<Src, LOCAL, SmallTab, SmallTabB, MedTab, WideTab> a(g, src, plan, d_work, d_units, ntask,
                                                          n_row, d_task_out, lo, rs, names);
  read_back(g->stream, {a.counts_item()});
  SideStreams& ss = side_streams(g->device);
  {
    ProfScope phase(names[6], g->stream);
    a.start(ss, 0);
    a.join(ss);
  }
  read_back(g->stream, {a.total_item()});
  return a.result();
}

}  // namespace agg
}  // namespace bflyd
