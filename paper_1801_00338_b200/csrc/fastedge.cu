// fastedge.cu -- Method::FastEdge ("fast-eBFC", sampling.cpp:125-147) for batches of
// estimator iterations, with the iteration's mt19937_64 stream on the device (SURVEY 8(f)
// ranks 1 and 3).
//
// Iteration q: engine std::mt19937_64(derive_seed(seed, q)); (l, r) = edge_at(uniform_index(m));
// if deg(l) == 1 or deg(r) == 1 the value is 0 (no further draws); otherwise `repeats` times
//   other_l = draw_excluding(N(r), l)   -> uniform_index(deg(r) - 1)   ("A" draws)
//   other_r = draw_excluding(N(l), r)   -> uniform_index(deg(l) - 1)   ("B" draws)
//   hits += has_edge(other_l, other_r)
// value = hits / repeats * (deg(l)-1) * (deg(r)-1) * m / 4 (the reference's operation order).
//
// One warp per iteration. The engine state lives in shared memory and is twisted by the
// whole warp (three read-then-write phases of the standard generation step). Mask-rejection
// draws are data dependent, but which draw an output feeds is a 2-state automaton (next
// draw is A or B; an accepted output flips the state), so 32 outputs are classified at once
// by a warp scan over composed state maps. Accepted draws queue in shared memory in stream
// order (A, B, A, B, ...) and are resolved 32 repeats at a time: each lane maps its pair to
// (other_l, other_r) and binary-searches the shorter adjacency (graph.cpp:60-66).
#include <cstdlib>

#include "common.cuh"
#include "graph.cuh"
#include "local.cuh"
#include "mt.cuh"

namespace bflyd {
namespace {

using namespace mt;

constexpr int kFeWarps = 8;
constexpr uint32_t kQ = 128;  // accepted-draw ring per warp (power of two)

struct FeWarp {
  uint64_t st[kMtN];
  uint32_t q[kQ];
};

// the std::mt19937_64 generation step on st[0..311], cooperatively and in place
__device__ __forceinline__ void warp_twist(uint64_t* x, unsigned lane) {
  uint64_t v[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {  // k < 156: reads original words only
    const unsigned k = lane + 32 * j;
    if (k < kMtM) v[j] = twist(x[k], x[k + 1], x[k + kMtM]);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const unsigned k = lane + 32 * j;
    if (k < kMtM) x[k] = v[j];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 5; ++j) {  // 156 <= k < 311: new x[k - 156], original x[k], x[k + 1]
    const unsigned k = kMtM + lane + 32 * j;
    if (k < kMtN - 1) v[j] = twist(x[k], x[k + 1], x[k - kMtM]);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const unsigned k = kMtM + lane + 32 * j;
    if (k < kMtN - 1) x[k] = v[j];
  }
  __syncwarp();
  if (lane == 0) x[kMtN - 1] = twist(x[kMtN - 1], x[0], x[kMtM - 1]);
  __syncwarp();
}

__device__ __forceinline__ uint64_t mask_for(uint64_t n) { return ~0ull >> __clzll(n - 1); }

// first index i in [lo, hi) with a[i] > x (upper_bound), warp-cooperative 32-ary search
template <class T>
__device__ __forceinline__ uint64_t warp_upper_bound(const T* a, uint64_t lo, uint64_t hi, T x,
                                                     unsigned lane) {
  while (hi - lo > 32) {
    const uint64_t span = hi - lo;
    const uint64_t p = lo + span * (lane + 1) / 33;  // 32 probes, strictly inside
    const unsigned le = __ballot_sync(0xffffffffu, a[p] <= x);
    const int c = __popc(le);  // probes <= x form a prefix (a is sorted)
    const uint64_t nlo = c ? lo + span * c / 33 + 1 : lo;
    const uint64_t nhi = c < 32 ? lo + span * (c + 1) / 33 : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint64_t p = lo + lane;
  const unsigned le = __ballot_sync(0xffffffffu, p < hi && a[p] <= x);
  return lo + __popc(le);
}

__device__ __forceinline__ bool bsearch_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && __ldg(a + lo) == x;
}

struct FeArgs {
  uint64_t seed, first, count, repeats, m;
  uint32_t L;
  const uint64_t* loff;
  const uint32_t* ladj;
  const uint64_t* roff;
  const uint32_t* radj;
  double* values;
  uint64_t* hits_out;
  uint64_t* edge_out;
};

__global__ void __launch_bounds__(kFeWarps * 32) k_fast_edge(FeArgs a) {
  __shared__ FeWarp smem[kFeWarps];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  FeWarp& W = smem[wl];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t it = gw; it < a.count; it += nw) {
    // ---- engine: seed (sequential recurrence) + first generation step
    if (lane == 0) {
      uint64_t x = derive_seed(a.seed, a.first + it);
      W.st[0] = x;
      for (int i = 1; i < kMtN; ++i) {
        x = seed_step(x, (uint64_t)i);
        W.st[i] = x;
      }
    }
    __syncwarp();
    warp_twist(W.st, lane);
    uint32_t pos = 0;  // next unread output of the current block
    // 32 consecutive outputs (lanes past the block end are invalid)
    auto chunk = [&](uint64_t& o) -> bool {
      if (pos >= (uint32_t)kMtN) {
        warp_twist(W.st, lane);
        pos = 0;
      }
      const uint32_t idx = pos + lane;
      const bool valid = idx < (uint32_t)kMtN;
      o = valid ? temper(W.st[idx]) : 0ull;
      return valid;
    };
    // ---- edge draw: uniform_index(m)
    uint64_t k = 0;
    if (a.m > 1) {
      const uint64_t mk = mask_for(a.m);
      while (true) {
        uint64_t o;
        const bool valid = chunk(o);
        const unsigned acc = __ballot_sync(full, valid && (o & mk) < a.m);
        if (acc) {
          const int f = __ffs(acc) - 1;
          k = __shfl_sync(full, o & mk, f);
          pos += f + 1;
          break;
        }
        pos += 32;
      }
    }
    const uint32_t l = (uint32_t)(warp_upper_bound(a.loff, 0, (uint64_t)a.L + 1, k, lane) - 1);
    const uint64_t lb = a.loff[l];
    const uint32_t r = a.ladj[k];
    const uint64_t rb = a.roff[r];
    const uint64_t dl = a.loff[l + 1] - lb, dr = a.roff[r + 1] - rb;
    uint64_t hits = 0;
    if (dl > 1 && dr > 1) {
      // draw_excluding positions: r sits at k - lb in N(l); l's position in N(r) by search
      const uint64_t posr = k - lb;
      const uint64_t posl = warp_upper_bound(a.radj, rb, rb + dr, l, lane) - 1 - rb;
      const uint64_t MA = dr - 1, MB = dl - 1;  // A: other_l from N(r); B: other_r from N(l)
      const bool cA = MA > 1, cB = MB > 1;     // uniform_index(1) draws nothing
      const uint64_t mA = cA ? mask_for(MA) : 0, mB = cB ? mask_for(MB) : 0;
      const uint32_t per = (cA && cB) ? 2u : 1u;
      // resolve repeats [t0, t0 + n) from queue records starting at qh
      auto resolve = [&](uint32_t qh, uint32_t n) {
        bool hit = false;
        if (lane < n) {
          uint64_t k1 = 0, k2 = 0;
          if (per == 2) {
            k1 = W.q[(qh + 2 * lane) & (kQ - 1)];
            k2 = W.q[(qh + 2 * lane + 1) & (kQ - 1)];
          } else if (cA) {
            k1 = W.q[(qh + lane) & (kQ - 1)];
          } else if (cB) {
            k2 = W.q[(qh + lane) & (kQ - 1)];
          }  // neither draws: both positions are 0
          if (k1 >= posl) ++k1;
          if (k2 >= posr) ++k2;
          const uint32_t ol = __ldg(a.radj + rb + k1), orr = __ldg(a.ladj + lb + k2);
          const uint64_t ob = a.loff[ol], od = a.loff[ol + 1] - ob;
          const uint64_t pb = a.roff[orr], pd = a.roff[orr + 1] - pb;
          hit = od <= pd ? bsearch_u32(a.ladj + ob, od, orr) : bsearch_u32(a.radj + pb, pd, ol);
        }
        return (uint64_t)__popc(__ballot_sync(full, hit));
      };
      if (!cA && !cB) {
        hits = resolve(0, 1) ? a.repeats : 0;  // every repeat draws the same pair, no draws
      } else {
        const uint64_t need = a.repeats * per;
        uint64_t got = 0;
        uint32_t qh = 0, qt = 0;
        unsigned state = 0;  // 0: next draw is A, 1: next draw is B (only when both draw)
        while (got < need) {
          uint64_t o;
          const bool valid = chunk(o);
          const bool accA = valid && cA && (o & mA) < MA;
          const bool accB = valid && cB && (o & mB) < MB;
          bool acc;
          unsigned role;
          if (per == 2) {
            // state map of this output: bit s = next state after input state s
            unsigned code = valid ? ((accA ? 1u : 0u) | (accB ? 0u : 2u)) : 2u;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const unsigned y = __shfl_up_sync(full, code, off);
              if ((int)lane >= off) {  // code := code o y (y first)
                code = (((code >> ((y >> 0) & 1u)) & 1u)) | (((code >> ((y >> 1) & 1u)) & 1u) << 1);
              }
            }
            unsigned ex = __shfl_up_sync(full, code, 1);
            if (lane == 0) ex = 2u;  // identity
            const unsigned last = __shfl_sync(full, code, 31);
            role = (ex >> state) & 1u;
            acc = role == 0 ? accA : accB;
            state = (last >> state) & 1u;
          } else {
            role = cA ? 0u : 1u;
            acc = cA ? accA : accB;
          }
          const unsigned b = __ballot_sync(full, acc);
          const uint32_t rank = __popc(b & ((1u << lane) - 1u));
          const bool keep = acc && got + rank < need;
          if (keep) W.q[(qt + rank) & (kQ - 1)] = (uint32_t)(o & (role == 0 ? mA : mB));
          const uint32_t nk = __popc(__ballot_sync(full, keep));
          qt += nk;
          got += nk;
          pos += 32;
          __syncwarp();
          while (qt - qh >= 32 * per) {
            hits += resolve(qh, 32);
            qh += 32 * per;
          }
        }
        if (qt != qh) hits += resolve(qh, (qt - qh) / per);
      }
    }
    if (lane == 0) {
      double v = 0.0;
      if (dl > 1 && dr > 1) {
        v = __ddiv_rn((double)hits, (double)a.repeats);
        v = __dmul_rn(v, (double)(dl - 1));
        v = __dmul_rn(v, (double)(dr - 1));
      }
      v = __ddiv_rn(__dmul_rn(v, (double)a.m), 4.0);
      a.values[it] = v;
      if (a.hits_out) a.hits_out[it] = hits;
      if (a.edge_out) a.edge_out[it] = k;
    }
    __syncwarp();
  }
}

}  // namespace

void fast_edge_device(bfly_graph* g, uint64_t seed, uint64_t first, uint64_t count,
                      uint64_t repeats, double* d_values, uint64_t* d_hits, uint64_t* d_edges) {
  if (!count) return;
  FeArgs a{seed, first, count, repeats, g->m, g->L, g->loff.p, g->ladj.p, g->roff.p, g->radj.p,
           d_values, d_hits, d_edges};
  launch("fastedge_samples", k_fast_edge, grid_for(count * 32, kFeWarps * 32, 148u * 8u),
         kFeWarps * 32, 0, g->stream, a);
}

}  // namespace bflyd
