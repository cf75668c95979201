// aggregate.cuh -- the degree-bucketed multiset-aggregation engine shared by the exact
// count, the all-subject local counts and the per-vertex sample kernels.
//
// A TASK is a multiset of vertex ids ("wedge endpoints") given as a list of ENTRIES, each
// entry naming one contiguous SEGMENT of an adjacency array. The task's value is
//     sum over distinct w of C(c(w), 2)
// where c(w) is the multiplicity of w. It is accumulated with the identity
// C(c,2) = 0 + 1 + ... + (c-1): every increment contributes the counter value it found,
// so the tables never need a separate flush pass.
//
//   exact count        task = start u (priority id), entries = forward entries u -> v,
//                      segment = N(v) after u                     (exact.cpp:29-41)
//   vertex sample      task = sample i, entries = N(v), segment = N(x), x in N(v),
//                      element v itself excluded                    (local.cpp:11-21)
//
// Buckets by task work (number of elements):
//   0: <= 32     warp per task, multiset in registers (__match_any_sync)
//   1: <= 512    warp per task, private 1024-slot shared-memory hash table
//   2: <= 8192   CTA per task, 16K-slot shared-memory hash table (persistent CTAs)
//   3: > 8192    task split over many CTAs; dense per-task rows in global memory
//                (L2 atomics) with touched-list reset, processed in waves
// LOCAL mode (exact source only) re-walks every task after its counts are final and
// scatters the per-vertex / per-edge contributions (generalised to the
// priority order): w gets C(c,2), u gets the task total, the middle vertex v and the edges
// (u,v), (v,w) get c(w)-1 per wedge.
#pragma once

#include <algorithm>
#include <cub/block/block_scan.cuh>
#include <vector>

#include "cubwrap.cuh"
#include "graph.cuh"

namespace bflyd {
namespace agg {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint64_t kTinyMax = 32, kSmallMax = 512, kMedMax = 8192;
constexpr int kSmallBits = 10;
constexpr int kSmallWarps = 8;
constexpr int kMedBits = 14;
constexpr int kMedBlock = 512;
constexpr uint64_t kHeavyChunk = 16384;

struct Acc {
  unsigned long long v = 0;
  unsigned ovf = 0;
  __device__ __forceinline__ void add(unsigned long long x) {
    unsigned long long t = v + x;
    ovf |= (t < v);
    v = t;
  }
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

__device__ __forceinline__ uint32_t slot_of(uint32_t w, int bits) {
  return (w * 0x9E3779B1u) >> (32 - bits);
}

// insert-or-increment; returns the count before the increment
__device__ __forceinline__ uint32_t table_inc(uint32_t* keys, uint32_t* cnt, int bits, uint32_t w,
                                              uint32_t* touched, uint32_t* ntouched) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t h = slot_of(w, bits);
  volatile uint32_t* vk = keys;
  while (true) {
    uint32_t k = vk[h];
    if (k == w) return atomicAdd(&cnt[h], 1u);
    if (k == kEmpty) {
      uint32_t prev = atomicCAS(&keys[h], kEmpty, w);
      if (prev == kEmpty) {
        if (touched) touched[atomicAdd(ntouched, 1u)] = h;
        return atomicAdd(&cnt[h], 1u);
      }
      if (prev == w) return atomicAdd(&cnt[h], 1u);
    }
    h = (h + 1u) & mask;
  }
}

// lookup of a key known to be present
__device__ __forceinline__ uint32_t table_get(const uint32_t* keys, const uint32_t* cnt, int bits,
                                              uint32_t w) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t h = slot_of(w, bits);
  while (keys[h] != w) h = (h + 1u) & mask;
  return cnt[h];
}

__device__ __forceinline__ unsigned long long c2(unsigned long long c) {
  return c < 2 ? 0ull : c * (c - 1) / 2;
}

// ---- task sources ---------------------------------------------------------------------
// Exact / all-local: priority CSR; task = start u.
struct ExactSrc {
  const uint64_t* poff;
  const uint32_t* padj;
  const uint32_t* sfx;
  const uint64_t* fwd;
  __device__ __forceinline__ uint32_t task_of(const uint32_t* list, uint64_t i) const {
    return list[i];
  }
  __device__ __forceinline__ void entries(uint32_t u, uint64_t& e0, uint64_t& e1) const {
    e0 = fwd[u];
    e1 = poff[u + 1];
  }
  __device__ __forceinline__ uint32_t seg(uint32_t, uint64_t e, const uint32_t*& p) const {
    const uint32_t v = padj[e];
    const uint64_t st = poff[v] + sfx[e];
    p = padj + st;
    return static_cast<uint32_t>(poff[v + 1] - st);
  }
  __device__ __forceinline__ uint32_t excl(uint32_t) const { return kEmpty; }
};

// Vertex samples: canonical CSRs; task = sample index, gids[i] = global vertex id.
struct VertexSrc {
  const uint64_t* gids;
  uint32_t L;
  const uint64_t* loff;
  const uint32_t* ladj;
  const uint64_t* roff;
  const uint32_t* radj;
  __device__ __forceinline__ uint32_t task_of(const uint32_t* list, uint64_t i) const {
    return list[i];
  }
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
  __device__ __forceinline__ uint32_t excl(uint32_t i) const {
    const uint64_t v = gids[i];
    return static_cast<uint32_t>(v < L ? v : v - L);
  }
};

// per-vertex / per-edge outputs of LOCAL mode (priority ids / canonical edge ids)
struct LocalOut {
  unsigned long long* vcnt;
  unsigned long long* ecnt;
  const uint32_t* peid;
  const uint32_t* padj;
};

// ---- flattened walk of one task by one warp -------------------------------------------
// f(w, p_elem, e): w = element, p_elem = its address, e = entry index.
template <class Src, class F>
__device__ __forceinline__ void warp_walk(const Src& src, uint32_t task, F&& f) {
  const unsigned lane = threadIdx.x & 31;
  const uint32_t ex = src.excl(task);
  uint64_t e0, e1;
  src.entries(task, e0, e1);
  for (uint64_t eb = e0; eb < e1; eb += 32) {
    const uint64_t e = eb + lane;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    uint32_t incl = len;
    for (int off = 1; off < 32; off <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t* basep = p - (incl - len);
    for (uint32_t r = 0; r < tot; r += 32) {
      const uint32_t idx = r + lane;
      uint32_t k = 0;
      for (int step = 16; step > 0; step >>= 1) {
        uint32_t c = __shfl_sync(0xffffffffu, incl, k + step - 1);
        if (c <= idx) k += step;
      }
      const uint32_t* bp = reinterpret_cast<const uint32_t*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(basep), k));
      if (idx < tot) {
        const uint32_t* pe = bp + idx;
        const uint32_t w = *pe;
        if (w != ex) f(w, pe, eb + k);
      }
    }
  }
}

// ---- bucket 0 ----------------------------------------------------------------------------
template <class Src, bool LOCAL>
__global__ void __launch_bounds__(256) k_tiny(Src src, const uint32_t* __restrict__ list,
                                              uint64_t count, unsigned long long* task_out,
                                              unsigned long long* total, unsigned* ovf,
                                              LocalOut lo) {
  __shared__ uint32_t bw[8][32];
  __shared__ const uint32_t* bq[LOCAL ? 8 : 1][32];
  __shared__ uint64_t be[LOCAL ? 8 : 1][32];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  Acc acc;
  for (uint64_t i = gw; i < count; i += nw) {
    const uint32_t task = src.task_of(list, i);
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
        uint32_t y = __shfl_up_sync(0xffffffffu, kin, off);
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
      if (LOCAL && c >= 2) {
        const unsigned long long xm = c - 1;
        const uint64_t e = be[wl][lane];
        atomicAdd(&lo.vcnt[lo.padj[e]], xm);
        atomicAdd(&lo.ecnt[lo.peid[e]], xm);
        atomicAdd(&lo.ecnt[lo.peid[bq[wl][lane] - lo.padj]], xm);
      }
    }
    ta = warp_sum(ta);
    if (lane == 0) {
      if (task_out) task_out[task] = ta.v;
      if (LOCAL && ta.v) atomicAdd(&lo.vcnt[task], ta.v);
    }
    acc.add(lane == 0 ? ta.v : 0ull);
    acc.ovf |= ta.ovf;
    __syncwarp();
  }
  flush_acc(acc, total, ovf);
}

// ---- bucket 1 ----------------------------------------------------------------------------
template <class Src, bool LOCAL>
__global__ void __launch_bounds__(kSmallWarps * 32) k_small(
    Src src, const uint32_t* __restrict__ list, uint64_t count, unsigned long long* task_out,
    unsigned long long* total, unsigned* ovf, LocalOut lo) {
  extern __shared__ uint32_t smem[];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  constexpr uint32_t S = 1u << kSmallBits;
  uint32_t* keys = smem + wl * (2 * S + S / 2 + 1);
  uint32_t* cnt = keys + S;
  uint32_t* touched = cnt + S;
  uint32_t* ntouched = touched + S / 2;
  for (uint32_t t = lane; t < S; t += 32) {
    keys[t] = kEmpty;
    cnt[t] = 0;
  }
  if (lane == 0) *ntouched = 0;
  __syncwarp();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  Acc acc;
  for (uint64_t i = gw; i < count; i += nw) {
    const uint32_t task = src.task_of(list, i);
    Acc ta;
    warp_walk(src, task, [&](uint32_t w, const uint32_t*, uint64_t) {
      ta.add(table_inc(keys, cnt, kSmallBits, w, touched, ntouched));
    });
    __syncwarp();
    if (LOCAL) {
      warp_walk(src, task, [&](uint32_t w, const uint32_t* pe, uint64_t e) {
        const uint32_t c = table_get(keys, cnt, kSmallBits, w);
        if (c >= 2) {
          atomicAdd(&lo.vcnt[lo.padj[e]], (unsigned long long)(c - 1));
          atomicAdd(&lo.ecnt[lo.peid[e]], (unsigned long long)(c - 1));
          atomicAdd(&lo.ecnt[lo.peid[pe - lo.padj]], (unsigned long long)(c - 1));
        }
      });
      __syncwarp();
    }
    const uint32_t nt = *ntouched;
    for (uint32_t t = lane; t < nt; t += 32) {
      const uint32_t sl = touched[t];
      if (LOCAL && cnt[sl] >= 2) atomicAdd(&lo.vcnt[keys[sl]], c2(cnt[sl]));
      keys[sl] = kEmpty;
      cnt[sl] = 0;
    }
    ta = warp_sum(ta);
    if (lane == 0) {
      if (task_out) task_out[task] = ta.v;
      if (LOCAL && ta.v) atomicAdd(&lo.vcnt[task], ta.v);
    }
    acc.add(lane == 0 ? ta.v : 0ull);
    acc.ovf |= ta.ovf;
    __syncwarp();
    if (lane == 0) *ntouched = 0;
    __syncwarp();
  }
  flush_acc(acc, total, ovf);
}

// ---- block-level flattened walk -----------------------------------------------------------
template <int BLOCK>
struct BlockWalkSmem {
  typename cub::BlockScan<uint32_t, BLOCK>::TempStorage scan;
  uint32_t incl[BLOCK];
  const uint32_t* base[BLOCK];
};

template <int BLOCK, class Src, class F>
__device__ __forceinline__ void block_walk(const Src& src, uint32_t task, BlockWalkSmem<BLOCK>& sm,
                                           F&& f) {
  using Scan = cub::BlockScan<uint32_t, BLOCK>;
  const uint32_t ex = src.excl(task);
  uint64_t e0, e1;
  src.entries(task, e0, e1);
  for (uint64_t eb = e0; eb < e1; eb += BLOCK) {
    const uint64_t e = eb + threadIdx.x;
    uint32_t len = 0;
    const uint32_t* p = nullptr;
    if (e < e1) len = src.seg(task, e, p);
    uint32_t incl, tot;
    Scan(sm.scan).InclusiveSum(len, incl, tot);
    sm.incl[threadIdx.x] = incl;
    sm.base[threadIdx.x] = p - (incl - len);
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < tot; idx += BLOCK) {
      uint32_t lo = 0, hi = BLOCK - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sm.incl[mid] > idx) hi = mid;
        else lo = mid + 1;
      }
      const uint32_t* pe = sm.base[lo] + idx;
      const uint32_t w = *pe;
      if (w != ex) f(w, pe, eb + lo);
    }
    __syncthreads();
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

// ---- bucket 2 ----------------------------------------------------------------------------
template <class Src, bool LOCAL>
__global__ void __launch_bounds__(kMedBlock) k_medium(Src src, const uint32_t* __restrict__ list,
                                                      uint64_t count, unsigned long long* next,
                                                      unsigned long long* task_out,
                                                      unsigned long long* total, unsigned* ovf,
                                                      LocalOut lo) {
  extern __shared__ uint32_t smem[];
  constexpr uint32_t S = 1u << kMedBits;
  uint32_t* keys = smem;
  uint32_t* cnt = smem + S;
  __shared__ BlockWalkSmem<kMedBlock> wsm;
  __shared__ unsigned long long s_item;
  __shared__ unsigned long long red[kMedBlock / 32];
  __shared__ unsigned redo[kMedBlock / 32];
  for (uint32_t t = threadIdx.x; t < S; t += kMedBlock) {
    keys[t] = kEmpty;
    cnt[t] = 0;
  }
  Acc acc;
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1ull);
    __syncthreads();
    const unsigned long long item = s_item;
    if (item >= count) break;
    const uint32_t task = src.task_of(list, item);
    Acc ta;
    block_walk<kMedBlock>(src, task, wsm, [&](uint32_t w, const uint32_t*, uint64_t) {
      ta.add(table_inc(keys, cnt, kMedBits, w, nullptr, nullptr));
    });
    if (LOCAL) {
      block_walk<kMedBlock>(src, task, wsm, [&](uint32_t w, const uint32_t* pe, uint64_t e) {
        const uint32_t c = table_get(keys, cnt, kMedBits, w);
        if (c >= 2) {
          atomicAdd(&lo.vcnt[lo.padj[e]], (unsigned long long)(c - 1));
          atomicAdd(&lo.ecnt[lo.peid[e]], (unsigned long long)(c - 1));
          atomicAdd(&lo.ecnt[lo.peid[pe - lo.padj]], (unsigned long long)(c - 1));
        }
      });
    }
    for (uint32_t t = threadIdx.x; t < S; t += kMedBlock) {
      if (LOCAL && keys[t] != kEmpty && cnt[t] >= 2) atomicAdd(&lo.vcnt[keys[t]], c2(cnt[t]));
      keys[t] = kEmpty;
      cnt[t] = 0;
    }
    Acc r = block_sum<kMedBlock>(ta, red, redo);
    if (threadIdx.x == 0) {
      if (task_out) task_out[task] = r.v;
      if (LOCAL && r.v) atomicAdd(&lo.vcnt[task], r.v);
      acc.add(r.v);
      acc.ovf |= r.ovf;
    }
  }
  flush_acc(acc, total, ovf);
}

// ---- bucket 3 ----------------------------------------------------------------------------
struct HeavyTask {
  uint32_t task, j, P, row;
};

template <class Src, bool LOCAL, bool PASS2>
__global__ void __launch_bounds__(256) k_heavy(Src src, const HeavyTask* __restrict__ tasks,
                                               uint32_t* __restrict__ rows, uint64_t n_row,
                                               uint32_t* __restrict__ touched,
                                               unsigned long long* __restrict__ ntouched,
                                               unsigned long long* task_out,
                                               unsigned long long* total, unsigned* ovf,
                                               LocalOut lo) {
  const HeavyTask t = tasks[blockIdx.x];
  uint32_t* row = rows + (uint64_t)t.row * n_row;
  uint32_t* tl = touched + (uint64_t)t.row * n_row;
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5, W = blockDim.x >> 5;
  const uint32_t ex = src.excl(t.task);
  uint64_t e0, e1;
  src.entries(t.task, e0, e1);
  Acc acc;
  for (uint64_t e = e0 + t.j + (uint64_t)t.P * wl; e < e1; e += (uint64_t)t.P * W) {
    const uint32_t* p;
    const uint32_t len = src.seg(t.task, e, p);
    for (uint32_t q = lane; q < len; q += 32) {
      const uint32_t x = p[q];
      if (x == ex) continue;
      if (!PASS2) {
        const uint32_t old = atomicAdd(&row[x], 1u);
        acc.add(old);
        if (old == 0) tl[atomicAdd(&ntouched[t.row], 1ull)] = x;
      } else {
        const uint32_t c = row[x];
        if (c >= 2) {
          atomicAdd(&lo.vcnt[lo.padj[e]], (unsigned long long)(c - 1));
          atomicAdd(&lo.ecnt[lo.peid[e]], (unsigned long long)(c - 1));
          atomicAdd(&lo.ecnt[lo.peid[p + q - lo.padj]], (unsigned long long)(c - 1));
        }
      }
    }
  }
  if (!PASS2) {
    Acc w = warp_sum(acc);
    if (lane == 0 && w.v) {
      if (task_out) atomicAdd(&task_out[t.task], w.v);
      if (LOCAL) atomicAdd(&lo.vcnt[t.task], w.v);
    }
    flush_acc(acc, total, ovf);
  }
}

// per row r of the wave: optional LOCAL scatter of C(c,2) to w and the task total to u,
// then zero the touched entries
template <bool LOCAL>
__global__ void k_reset_rows(uint32_t* __restrict__ rows, uint64_t n_row,
                             const uint32_t* __restrict__ touched,
                             const unsigned long long* __restrict__ ntouched,
                             LocalOut lo) {
  const uint32_t r = blockIdx.y;
  const unsigned long long nt = ntouched[r];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = touched[(uint64_t)r * n_row + i];
    uint32_t* cell = rows + (uint64_t)r * n_row + w;
    if (LOCAL && *cell >= 2) atomicAdd(&lo.vcnt[w], c2(*cell));
    *cell = 0;
  }
}

// ---- bucketing ---------------------------------------------------------------------------
__global__ void k_bucket(const unsigned long long* __restrict__ work, uint64_t n,
                         uint32_t* __restrict__ lists, unsigned long long* __restrict__ counts,
                         unsigned long long* __restrict__ wsum,
                         unsigned long long* __restrict__ heavy_work);

// ---- host orchestration ------------------------------------------------------------------
struct RunStats {
  uint64_t starts[4] = {0, 0, 0, 0};
  uint64_t wedges[4] = {0, 0, 0, 0};
};

// Scratch for heavy rows lives in the graph handle (zero-invariant between calls).
void ensure_rows(bfly_graph* g, uint64_t n_row);

template <class Src, bool LOCAL>
uint64_t run(bfly_graph* g, const Src& src, const unsigned long long* d_work, uint64_t ntask,
             uint64_t n_row, unsigned long long* d_task_out, LocalOut lo, RunStats* rs,
             const char* const names[4]) {
  cudaStream_t s = g->stream;
  if (ntask == 0) return 0;
  DBuf<unsigned long long> ctl(12, s);
  ctl.zero();
  unsigned long long* counts = ctl.p;
  unsigned long long* wsum = ctl.p + 4;
  unsigned long long* total = ctl.p + 8;
  unsigned long long* next = ctl.p + 9;
  unsigned* ovf = reinterpret_cast<unsigned*>(ctl.p + 10);
  DBuf<uint32_t> lists(4 * ntask, s);
  DBuf<unsigned long long> heavy_work(ntask, s);
  launch(names[0], k_bucket, grid_for(ntask, 256), 256, 0, s, d_work, ntask, lists.p, counts, wsum,
         heavy_work.p);
  unsigned long long h[8];
  BFLY_CUDA(cudaMemcpyAsync(h, ctl.p, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  if (rs)
    for (int q = 0; q < 4; ++q) {
      rs->starts[q] = h[q];
      rs->wedges[q] = h[4 + q];
    }
  if (h[0])
    launch(names[1], k_tiny<Src, LOCAL>, grid_for(h[0] * 32, 256, 148u * 64u), 256, 0, s, src,
           lists.p, (uint64_t)h[0], d_task_out, total, ovf, lo);
  if (h[1]) {
    const size_t sm = kSmallWarps * ((2u << kSmallBits) + (1u << kSmallBits) / 2 + 1) * 4;
    BFLY_CUDA(cudaFuncSetAttribute(k_small<Src, LOCAL>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    launch(names[2], k_small<Src, LOCAL>, grid_for(h[1] * 32, kSmallWarps * 32, 148u * 2u),
           kSmallWarps * 32, sm, s, src, lists.p + ntask, (uint64_t)h[1], d_task_out, total, ovf,
           lo);
  }
  if (h[2]) {
    const size_t sm = (2u << kMedBits) * 4;
    BFLY_CUDA(cudaFuncSetAttribute(k_medium<Src, LOCAL>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const unsigned grid = static_cast<unsigned>(std::min<unsigned long long>(h[2], 148ull));
    launch(names[3], k_medium<Src, LOCAL>, grid, kMedBlock, sm, s, src, lists.p + 2 * ntask,
           (uint64_t)h[2], next, d_task_out, total, ovf, lo);
  }
  if (h[3]) {
    std::vector<uint32_t> hl(h[3]);
    std::vector<unsigned long long> hw(h[3]);
    BFLY_CUDA(cudaMemcpyAsync(hl.data(), lists.p + 3 * ntask, h[3] * 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaMemcpyAsync(hw.data(), heavy_work.p, h[3] * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
    ensure_rows(g, n_row);
    const uint32_t slots = g->row_slots;
    std::vector<uint32_t> order(h[3]);
    for (uint32_t i = 0; i < h[3]; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return hw[a] > hw[b]; });
    DBuf<HeavyTask> dtasks;
    for (size_t w0 = 0; w0 < order.size(); w0 += slots) {
      std::vector<HeavyTask> tasks;
      const size_t w1 = std::min(order.size(), w0 + slots);
      for (size_t q = w0; q < w1; ++q) {
        const uint64_t wk = hw[order[q]];
        const uint32_t P = static_cast<uint32_t>(
            std::min<uint64_t>(8192, (wk + kHeavyChunk - 1) / kHeavyChunk));
        for (uint32_t j = 0; j < P; ++j)
          tasks.push_back({hl[order[q]], j, P, static_cast<uint32_t>(q - w0)});
      }
      dtasks.ensure(tasks.size(), s);
      BFLY_CUDA(cudaMemcpyAsync(dtasks.p, tasks.data(), tasks.size() * sizeof(HeavyTask),
                                cudaMemcpyHostToDevice, s));
      launch("agg_heavy", k_heavy<Src, LOCAL, false>, static_cast<unsigned>(tasks.size()), 256, 0, s,
             src, dtasks.p, g->rows.p, n_row, g->row_touched.p, g->row_ntouched.p, d_task_out,
             total, ovf, lo);
      if (LOCAL) {
        launch("agg_heavy_local", k_heavy<Src, LOCAL, true>, static_cast<unsigned>(tasks.size()), 256, 0,
               s, src, dtasks.p, g->rows.p, n_row, g->row_touched.p, g->row_ntouched.p,
               d_task_out, total, ovf, lo);
      }
      const dim3 rg(296, static_cast<unsigned>(w1 - w0));
      launch("agg_reset_rows", k_reset_rows<LOCAL>, rg, 256, 0, s, g->rows.p, n_row,
             g->row_touched.p, g->row_ntouched.p, lo);
      BFLY_CUDA(cudaMemsetAsync(g->row_ntouched.p, 0, (w1 - w0) * sizeof(unsigned long long), s));
      BFLY_CUDA(cudaStreamSynchronize(s));  // host-side task vector is rebuilt per wave
    }
  }
  unsigned long long res[3];
  BFLY_CUDA(cudaMemcpyAsync(res, ctl.p + 8, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  if (static_cast<unsigned>(res[2]) != 0) fail(kOverflow, "64-bit counter overflow in addition");
  return res[0];
}

}  // namespace agg
}  // namespace bflyd
