// radix.cuh -- hand-written LSD radix sort for sm_100a, used by the graph build in place of a
// library device sort (the reference's per-list std::sort + unique in from_edges,
// graph.cpp:40-47, becomes stable device-wide sorts of (key, payload) pairs).
//
// Structure (one histogram pass + one single-sweep pass per 8-bit digit):
//   k_hist   one read of the keys: the digit histogram of EVERY pass at once (per-warp
//            shared-memory counters, one global atomic per nonzero counter per CTA)
//   k_base   exclusive scan of each pass's 256 counts -> global start of every digit
//   k_sweep  per pass, one CTA per tile of 4096 keys, tiles taken in ticket order:
//            (1) coalesced warp-striped load of the tile (keys + payload);
//            (2) stable rank of every key inside its warp and digit: __match_any_sync over
//                the digit gives the peers of a key in one instruction, the lowest peer bumps
//                the warp's counter for that digit;
//            (3) per-digit tile totals published for the successors, then a decoupled
//                look-back over the predecessors' published totals / inclusive prefixes gives
//                each digit's global start for this tile (no second pass over the keys);
//            (4) the tile is re-ordered by digit in shared memory and written out in runs,
//                so consecutive threads store consecutive addresses of a digit's run.
// Traffic per pass: key + payload read once and written once (16 B per u32 pair); the
// look-back words are tagged with the pass number, so one zeroed status array serves every
// pass of a sort.
#pragma once

#include <cuda/atomic>
#include <utility>

#include "common.cuh"

namespace bflyd {
namespace radix {

constexpr int kDigitBits = 8;
constexpr int kRadix = 1 << kDigitBits;
constexpr int kBlock = 256;       // histogram kernels: thread d owns digit d
constexpr int kWarps = kBlock / 32;
constexpr int kSweep = 512;       // sweep CTA: 16 warps, threads < kRadix own a digit each
constexpr int kSweepWarps = kSweep / 32;
constexpr int kItems = 8;         // keys per thread (register budget: 2 CTAs of 16 warps per SM)
constexpr int kTile = kSweep * kItems;
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

template <typename K>
__global__ void __launch_bounds__(kBlock) k_hist(const K* __restrict__ keys, uint64_t n,
                                                 PassDesc pd, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[kWarps][kRadix];  // one pass at a time, per-warp copies
  const unsigned w = threadIdx.x >> 5;
  for (int p = 0; p < pd.passes; ++p) {
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kBlock) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int shf = pd.shift[p];
    const uint32_t msk = pd.mask[p];
    for (uint64_t i = blockIdx.x * (uint64_t)kBlock + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * kBlock)
      atomicAdd(&sh[w][digit_of(__ldg(keys + i), shf, msk)], 1u);
    __syncthreads();
    unsigned c = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) c += sh[q][threadIdx.x];
    if (c) atomicAdd(&hist[p * kRadix + threadIdx.x], c);
    __syncthreads();
  }
}

// one CTA per pass: exclusive scan of the 256 digit counts (a template: header-defined)
template <int = 0>
__global__ void __launch_bounds__(kBlock) k_base(const unsigned* __restrict__ hist,
                                                 unsigned* __restrict__ base) {
  __shared__ unsigned wt[kWarps];
  const unsigned t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned x = hist[blockIdx.x * kRadix + t];
  unsigned incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += y;
  }
  if (lane == 31) wt[w] = incl;
  __syncthreads();
  unsigned pre = 0;
  for (unsigned q = 0; q < w; ++q) pre += wt[q];
  base[blockIdx.x * kRadix + t] = pre + incl - x;
}

// look-back word: [63:62] flag (1 tile total, 2 inclusive prefix), [61:56] pass tag, [39:0] value
constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62;
__device__ __forceinline__ unsigned long long lb_word(unsigned long long flag, int tag,
                                                      unsigned long long v) {
  return flag | (static_cast<unsigned long long>(tag) << 56) | v;
}

template <typename K, typename V, bool HAS_V>
__global__ void __launch_bounds__(kSweep, 2) k_sweep(const K* __restrict__ kin, K* __restrict__ kout,
                                                     const V* __restrict__ vin, V* __restrict__ vout,
                                                     uint64_t n, int shift, uint32_t mask, int tag,
                                                     const unsigned* __restrict__ gbase,
                                                     unsigned long long* __restrict__ status,
                                                     unsigned* __restrict__ ticket) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);
  V* sv = reinterpret_cast<V*>(smem + sizeof(K) * kTile);
  __shared__ unsigned wcnt[kSweepWarps][kRadix];  // per-warp digit counts -> offsets in digit
  __shared__ unsigned dstart[kRadix];              // tile-local start of each digit
  __shared__ unsigned gdst[kRadix];                // global start of the digit's run here
  __shared__ unsigned wt[kRadix / 32];
  __shared__ unsigned s_tile;
  const unsigned t = threadIdx.x, lane = t & 31, w = t >> 5, full = 0xffffffffu;
  if (t == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = t; i < kSweepWarps * kRadix; i += kSweep) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const unsigned tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * kTile;
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
  // (3) threads t < 256 own digit t: per-warp offsets inside the digit, the tile total, the
  // look-back, the tile-local digit starts
  unsigned tot = 0;
  if (t < kRadix) {
    unsigned run = 0;
#pragma unroll
    for (int q = 0; q < kSweepWarps; ++q) {
      const unsigned c = wcnt[q][t];
      wcnt[q][t] = run;
      run += c;
    }
    tot = run;
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(
        status[static_cast<uint64_t>(tile) * kRadix + t]);
    unsigned long long excl = 0;
    if (tile == 0) {
      me.store(lb_word(kPre, tag, tot), cuda::memory_order_relaxed);
    } else {
      me.store(lb_word(kAgg, tag, tot), cuda::memory_order_relaxed);
      // windowed look-back: the statuses of up to kWin predecessors are loaded at once and
      // consumed nearest first (tile totals add up until an inclusive prefix closes the sum);
      // a predecessor that has not published yet restarts the window at itself
      constexpr int kWin = 8;
      int64_t p = static_cast<int64_t>(tile) - 1;
      unsigned spins = 0;
      while (true) {
        unsigned long long x[kWin];
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
          if (p - j >= 0) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> prv(
                status[static_cast<uint64_t>(p - j) * kRadix + t]);
            x[j] = prv.load(cuda::memory_order_relaxed);
          } else {
            x[j] = lb_word(kPre, tag, 0);  // before tile 0: an empty prefix
          }
        }
        int j = 0;
        bool done = false;
#pragma unroll
        for (; j < kWin; ++j) {
          if ((x[j] >> 62) == 0 || static_cast<int>((x[j] >> 56) & 63u) != tag) break;
          excl += x[j] & ((1ull << 40) - 1);
          if ((x[j] >> 62) == 2) {
            done = true;
            break;
          }
        }
        if (done) break;
        p -= j;
        // a predecessor that never publishes is a bug: fail loudly instead of hanging
        if (j == 0 && ++spins > (1u << 26)) __trap();
      }
      me.store(lb_word(kPre, tag, excl + tot), cuda::memory_order_relaxed);
    }
    gdst[t] = gbase[t] + static_cast<unsigned>(excl);
    unsigned incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(full, incl, o);
      if ((int)lane >= o) incl += y;
    }
    if (lane == 31) wt[w] = incl;
    dstart[t] = incl - tot;  // (warp-local part; the other warps' totals added below)
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
  if (n >= (1ull << 32) - kTile) fail(kArgument, "sort larger than 2^32 items");
  const PassDesc pd = passes_for(begin_bit, end_bit);
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  DBuf<unsigned> hist(pd.passes * kRadix, s), gbase(pd.passes * kRadix, s), ticket(pd.passes, s);
  DBuf<unsigned long long> status(ntiles * kRadix, s);
  hist.zero();
  ticket.zero();
  status.zero();
  const K* k0 = buf(0).first;
  launch("radix_hist", k_hist<K>, grid_for(n, kBlock, 148u * 8u), kBlock, 0, s, k0, n, pd,
         hist.p);
  launch("radix_base", k_base<>, pd.passes, kBlock, 0, s, (const unsigned*)hist.p, gbase.p);
  constexpr size_t smem = (sizeof(K) + (HAS_V ? sizeof(V) : 0)) * kTile;
  auto kern = k_sweep<K, V, HAS_V>;
  BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int p = 0; p < pd.passes; ++p) {
    auto src = buf(p);
    auto dst = buf(p + 1);
    launch("radix_sweep", kern, static_cast<unsigned>(ntiles), kSweep, smem, s, src.first,
           dst.first, src.second, dst.second, n, pd.shift[p], pd.mask[p], p + 1,
           (const unsigned*)(gbase.p + p * kRadix), status.p, ticket.p + p);
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
