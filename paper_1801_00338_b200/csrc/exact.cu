// exact.cu -- exact butterfly count on B200 (replaces exact_count_side, exact.cpp:23-43),
// the hub plan, and the shared bucketing kernel of the aggregation engine.
//
// Each butterfly is counted once at its highest-priority vertex u (priority.cu). The
// reference anchors at every vertex of the chosen side and walks w < v in dense-id order;
// both enumerate each butterfly exactly once, so the uint64 results are identical for
// either reference side (exact.hpp:20-24).
//
// Two enumerations share the work (aggregate.cuh):
//   hub path    starts u < k (the k highest-priority vertices, where the heavy work is):
//               one task per END vertex w; keys u < k in a dense k-entry table
//   start path  starts u >= k: one task per start u; keys w in a hash table
#include <cstdio>
#include <cstdlib>

#include "aggregate.cuh"
#include "hubdense.cuh"
#include "local.cuh"

namespace bflyd {
namespace agg {

__global__ void k_bucket(const unsigned long long* __restrict__ work,
                         const unsigned long long* __restrict__ units, uint64_t n,
                         uint64_t lim0, uint64_t lim1, uint64_t lim2, uint64_t lim3,
                         uint64_t wide_units, uint64_t wide_work, uint64_t split_units,
                         uint64_t skip_below, uint32_t* __restrict__ lists,
                         unsigned long long* __restrict__ counts,
                         unsigned long long* __restrict__ wsum,
                         unsigned long long* __restrict__ esum,
                         unsigned long long* __restrict__ heavy_work,
                         unsigned long long* __restrict__ heavy_units) {
  // Per 256-task chunk: warp ballots -> block counts in shared memory -> one global atomic
  // per bucket per chunk for the list offsets; key/entry sums are accumulated per block and
  // flushed once (same-address global atomics were the bottleneck at 3 per warp per bucket).
  __shared__ unsigned s_cnt[kBuckets];
  __shared__ unsigned long long s_base[kBuckets];
  __shared__ unsigned long long s_w[kBuckets], s_e[kBuckets];
  const unsigned lane = threadIdx.x & 31;
  if (threadIdx.x < kBuckets) {
    s_w[threadIdx.x] = 0;
    s_e[threadIdx.x] = 0;
  }
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < kBuckets) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t u = base + threadIdx.x;
    const unsigned long long wk = (u < n && u >= skip_below) ? work[u] : 0ull;
    int b = wk == 0 ? -1
            : wk <= lim0 ? 0
            : wk <= lim1 ? 1
            : wk <= lim2 ? 2
            : wk <= lim3 ? 3
                         : 5;
    if (b == 3 && split_units && units[u] >= split_units) b = 5;
    if (b == 3 && ((wide_units && units[u] >= wide_units) || (wide_work && wk > wide_work))) b = 4;
    unsigned my_off = 0;
    for (int q = 0; q < kBuckets; ++q) {
      const unsigned mask = __ballot_sync(0xffffffffu, b == q);
      if (!mask) continue;
      const int leader = __ffs(mask) - 1;
      unsigned long long s = (b == q) ? wk : 0ull;
      unsigned long long es = (b == q && units) ? units[u] : 0ull;
      for (int off = 16; off > 0; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        es += __shfl_xor_sync(0xffffffffu, es, off);
      }
      unsigned wbase = 0;
      if ((int)lane == leader) {
        wbase = atomicAdd(&s_cnt[q], static_cast<unsigned>(__popc(mask)));
        atomicAdd(&s_w[q], s);
        if (es) atomicAdd(&s_e[q], es);
      }
      wbase = __shfl_sync(0xffffffffu, wbase, leader);
      if (b == q) my_off = wbase + __popc(mask & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (threadIdx.x < kBuckets && s_cnt[threadIdx.x])
      s_base[threadIdx.x] = atomicAdd(&counts[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
    __syncthreads();
    if (b >= 0) {
      const uint64_t idx = s_base[b] + my_off;
      lists[b * n + idx] = static_cast<uint32_t>(u);
      if (b == kBuckets - 1) {
        heavy_work[idx] = wk;
        heavy_units[idx] = units ? units[u] : 0ull;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < kBuckets) {
    if (s_w[threadIdx.x]) atomicAdd(&wsum[threadIdx.x], s_w[threadIdx.x]);
    if (s_e[threadIdx.x]) atomicAdd(&esum[threadIdx.x], s_e[threadIdx.x]);
  }
}

__global__ void k_zero_counters(unsigned long long* p, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

RowScratch& row_scratch(int device) {
  static RowScratch per_device[64];
  return per_device[device & 63];
}

// Size the process-wide heavy-row scratch (caller holds rs.mu). Rows stay allocated for the
// process lifetime so per-graph calls never pay a multi-GB allocation + memset; the
// zero-invariant (every touched cell is reset after use) makes reuse free.
uint32_t ensure_rows(RowScratch& rs, uint64_t n_row, uint64_t need, cudaStream_t s) {
  const uint64_t budget = 4ull << 30;  // rows + touched lists, bytes
  const uint64_t want = std::max<uint64_t>(
      1, std::min<uint64_t>(std::min<uint64_t>(kMaxRows, need), budget / (n_row * 8)));
  if (rs.cap_words < want * n_row) {
    BFLY_CUDA(cudaStreamSynchronize(s));
    // drop the old scratch first (capacity 0 until the new one is complete), then commit
    // the new rows only once every allocation and zero-fill succeeded: a failure leaves an
    // empty scratch, never a stale capacity over null or non-zeroed rows
    rs.cap_words = 0;
    if (rs.rows) cudaFree(rs.rows);
    if (rs.touched) cudaFree(rs.touched);
    if (rs.ntouched) cudaFree(rs.ntouched);
    rs.rows = rs.touched = nullptr;
    rs.ntouched = nullptr;
    uint32_t* rows = nullptr;
    uint32_t* touched = nullptr;
    unsigned long long* ntouched = nullptr;
    cudaError_t e = cudaMalloc(&rows, want * n_row * 4);
    if (e == cudaSuccess) e = cudaMalloc(&touched, want * n_row * 4);
    if (e == cudaSuccess) e = cudaMalloc(&ntouched, kMaxRows * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(rows, 0, want * n_row * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(ntouched, 0, kMaxRows * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      if (rows) cudaFree(rows);
      if (touched) cudaFree(touched);
      if (ntouched) cudaFree(ntouched);
      cudaGetLastError();
      fail(kInternal, std::string("heavy-row scratch allocation: ") + cudaGetErrorString(e));
    }
    rs.rows = rows;
    rs.touched = touched;
    rs.ntouched = ntouched;
    rs.cap_words = want * n_row;
  }
  return static_cast<uint32_t>(std::min<uint64_t>(kMaxRows, rs.cap_words / n_row));
}

__global__ void k_degree_units(const uint64_t* __restrict__ poff, uint64_t n,
                               unsigned long long* __restrict__ units) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x)
    units[u] = poff[u + 1] - poff[u];
}

__global__ void k_fwd_count(const uint64_t* __restrict__ poff, const uint64_t* __restrict__ fwd,
                            uint64_t n, unsigned long long* __restrict__ units) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x)
    units[u] = poff[u + 1] - fwd[u];
}

// vcnt[u] += sum over the private rows of krow[row * k + u]
__global__ void k_sum_key_rows(const unsigned long long* __restrict__ krow, uint32_t rows,
                               uint32_t k, unsigned long long* __restrict__ vcnt) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < k; u += gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (uint32_t r = 0; r < rows; ++r) s += krow[(uint64_t)r * k + u];
    if (s) vcnt[u] += s;
  }
}

// out[0] = 1 + the last u < scan with work[u] > min_work (0 if none); out[1] = the number of
// leading priority ids of degree >= 2^16 among those (degrees are non-increasing in u);
// out[2..3] = the start work (wedges) of the first dense_h priority ids, low and high word:
// exactly the keys the dense top-hub path would take over from the segment walks;
// out[4] = the degree of priority id k = the largest degree of a start-path task (saturated)
__global__ void k_hub_choose(const unsigned long long* __restrict__ work,
                             const uint64_t* __restrict__ poff, uint64_t scan, uint64_t n,
                             uint64_t min_work, uint32_t dense_h, uint32_t* __restrict__ out) {
  __shared__ uint32_t s_k;
  __shared__ unsigned long long s_dense;
  if (threadIdx.x == 0) {
    s_k = 0;
    s_dense = 0;
  }
  __syncthreads();
  uint32_t best = 0;
  unsigned long long dsum = 0;
  for (uint64_t u = threadIdx.x; u < scan; u += blockDim.x) {
    const unsigned long long wu = work[u];
    if (wu > min_work) best = static_cast<uint32_t>(u + 1);
    if (u < dense_h) dsum += wu;
  }
  atomicMax(&s_k, best);
  if (dsum) atomicAdd(&s_dense, dsum);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t k = s_k;
    uint32_t lo = 0, hi = k;  // first u < k with degree < 65536
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (poff[mid + 1] - poff[mid] >= 65536) lo = mid + 1;
      else hi = mid;
    }
    out[0] = k;
    out[1] = lo;
    out[2] = static_cast<uint32_t>(s_dense);
    out[3] = static_cast<uint32_t>(s_dense >> 32);
    const uint64_t dk = k < n ? poff[k + 1] - poff[k] : 0;
    out[4] = dk > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(dk);
  }
}

// per vertex v: vinfo = (t(v) | tH(v) << 16, poff[v] as u32 (m < 2^31)) with
// t(v) = |N(v) & [0, min(k, v))| and tH(v) = |N(v) & [0, min(H, v))| (H <= k: the hubs of the
// dense path, hubdense.cuh; both are prefixes of the ascending N(v), t(v) <= k < 2^15)
__global__ void k_hub_vprep(const uint64_t* __restrict__ poff, const uint32_t* __restrict__ padj,
                            uint64_t n, uint32_t k, uint32_t H, uint2* __restrict__ vinfo) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t lim = v < k ? static_cast<uint32_t>(v) : k;
    const uint64_t b = poff[v], d = poff[v + 1] - b;
    uint64_t lo = 0, hi = d < lim ? d : lim;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (padj[b + mid] < lim) lo = mid + 1;
      else hi = mid;
    }
    uint32_t th = 0;
    if (H) {
      const uint32_t limh = v < H ? static_cast<uint32_t>(v) : H;
      uint64_t l2 = 0, h2 = lo < limh ? lo : limh;
      while (l2 < h2) {
        const uint64_t mid = (l2 + h2) >> 1;
        if (padj[b + mid] < limh) l2 = mid + 1;
        else h2 = mid;
      }
      th = static_cast<uint32_t>(l2);
    }
    vinfo[v] = make_uint2(static_cast<uint32_t>(lo) | (th << 16), static_cast<uint32_t>(b));
  }
}

// hub plan: one thread per directed entry e = (w -> v): the hub keys {u in N(v) : u < min(k,v,w)}
// are a prefix of the ascending list N(v), of length t(v) when w > v, else min(t(v), rank of w
// in N(v)); hlen / hpst describe the part of it at or above H (all of it when H = 0);
// that rank is already known from prio_plan's suffix start (fseg.x = rank + poff[v] + 1), so
// the plan streams the entries with one random 8-byte load (vinfo[v]) each.
// hub_work[w] = sum of hlen over w's entries.
__global__ void k_hub_plan(const uint32_t* __restrict__ padj, const uint32_t* __restrict__ psrc,
                           const uint2* __restrict__ fseg, uint64_t nnz, uint32_t k,
                           const uint2* __restrict__ vinfo, uint16_t* __restrict__ hlen,
                           uint32_t* __restrict__ hpst, unsigned long long* __restrict__ hwork) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) & ~31ull;
  for (uint64_t base = warp * 32; base < nnz; base += stride) {
    const uint64_t e = base + lane;
    const bool valid = e < nnz;
    const uint32_t w = valid ? __ldcs(psrc + e) : 0xFFFFFFFFu;  // streamed: L2 keeps vinfo
    unsigned long long x = 0;
    if (valid) {
      const uint32_t v = __ldcs(padj + e);
      const uint2 vi = vinfo[v];
      x = vi.x & 0xFFFFu;
      // forward entry of a hub w: its rank in N(v) bounds the prefix (an end vertex w >= k
      // lies behind every hub of N(v): no fseg read for the entries of those tasks)
      if (x && v > w && w < k) {
        const uint32_t rank = __ldcs(&fseg[e].x) - 1 - vi.y;
        if (rank < x) x = rank;
      }
      // the first min(x, tH(v)) keys are hubs below H: the dense path counts them from masks
      const uint32_t th = vi.x >> 16;
      const uint32_t dx = th < x ? th : static_cast<uint32_t>(x);
      x -= dx;
      __stcs(reinterpret_cast<unsigned short*>(hlen) + e, static_cast<unsigned short>(x));
      if (x) __stcs(hpst + e, vi.y + dx);  // segment start, so walks skip padj[e]
    }
    const unsigned full = 0xffffffffu;
    const uint32_t up = __shfl_up_sync(full, w, 1);
    const bool head = lane == 0 || up != w;
    const unsigned heads = __ballot_sync(full, head);
    const int my_head = 31 - __clz(heads & ((2u << lane) - 1u));
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(full, x, o);
      if ((int)lane - o >= my_head) x += y;
    }
    const uint32_t dn = __shfl_down_sync(full, w, 1);
    const bool tail = lane == 31 || dn != w;
    if (valid && tail && x) atomicAdd(&hwork[w], x);
  }
}

}  // namespace agg

// words per vertex of the dense top-hub masks (hubdense.cuh): H = 32 W hubs. Read on every
// plan build, so tests can vary BFLY_HUB_DENSE_W / BFLY_HUB_DENSE (0: no dense path).
static uint32_t hub_dense_words() {
  const char* off = std::getenv("BFLY_HUB_DENSE");
  if (off && off[0] == '0') return 0;
  const char* e = std::getenv("BFLY_HUB_DENSE_W");
  uint32_t w = e ? static_cast<uint32_t>(std::atoi(e)) : 8u;
  if (w > 32) w = 32;
  while (w & (w - 1)) w &= w - 1;  // a power of two
  return w;
}

// wedges of the top hubs per adjacency entry from which the dense path is used
// (BFLY_HUB_DENSE_MIN; 0 forces it)
static double hub_dense_min_keys_per_entry() {
  const char* e = std::getenv("BFLY_HUB_DENSE_MIN");
  return e ? std::atof(e) : 4.0;
}

template <int W>
static void launch_hub_mask(bfly_graph* g, const uint2* vinfo) {
  const uint64_t n = g->prio_nz;  // (entries name only vertices with edges)
  launch("hub_mask", agg::k_hub_mask<W>, grid_for(n, 256, 148u * 64u), 256, 0, g->stream,
         g->poff.p, g->padj.p, vinfo, n, g->hmask.p);
}

// Choose k and build the hub plan (cached on the graph; the graph is immutable). dense: the
// caller can use the dense top-hub path (counting runs); a plan built without it serves both.
static void ensure_hub_plan(bfly_graph* g, bool dense) {
  if (g->hub_ready && (g->hub_h == 0 || dense)) return;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n(), nnz = 2 * g->m;
  // k = 1 + the last of the first kHubMax priority ids whose start work exceeds the
  // medium-table limit (those starts would otherwise need global rows); chosen on the device
  const uint64_t scan = std::min<uint64_t>(n, kHubMax);
  static const uint64_t min_work = [] {
    const char* e = std::getenv("BFLY_HUB_MIN_WORK");
    return e ? std::strtoull(e, nullptr, 10) : kHubMinWork;
  }();
  uint32_t W = dense ? hub_dense_words() : 0;
  uint32_t kk2[5] = {0, 0, 0, 0, 0};
  if (scan) {
    DBuf<uint32_t> d(5, s);
    launch("hub_choose_k", agg::k_hub_choose, 1, 1024, 0, s,
           reinterpret_cast<const unsigned long long*>(g->work.p), g->poff.p, scan, n, min_work,
           32u * W, d.p);
    read_back(s, {{kk2, d.p, sizeof(kk2)}});
  }
  trace_mark("hub: choose k");
  const uint32_t k = kk2[0];
  // 32-bit counters for hubs of degree >= 2^16 (priority order is degree descending), 16-bit
  // above: c(u, w) <= deg(u) < 65536 there (DirectSplit)
  const uint32_t k1 = std::min<uint32_t>(k, (kk2[1] + 31) & ~31u);
  g->hub_k = k;
  g->hub_k1 = k1;
  g->start_deg_max = kk2[4];
  // dense path: the H = min(32 W, k) top hubs, W the smallest power of two covering them --
  // when they carry enough wedges per adjacency entry to pay for reading every entry's mask
  // row (config 2: 8.8 wedges per entry; its walks cost about a quarter of a row read per key)
  const uint64_t dense_keys = kk2[2] | static_cast<uint64_t>(kk2[3]) << 32;
  if (dense_keys < hub_dense_min_keys_per_entry() * static_cast<double>(nnz)) W = 0;
  while (W > 1 && 32u * (W / 2) >= k) W /= 2;
  const uint32_t H = std::min<uint32_t>(32u * W, k);
  if (H == 0) W = 0;
  g->hub_h = H;
  g->hub_w = W;
  g->hlen.release();
  g->hpst.release();
  g->hub_work.release();
  g->hmask.release();
  if (k) {
    g->hlen.alloc(nnz, s);
    g->hpst.alloc(nnz, s);
    g->hub_work.alloc(n, s);
    g->hub_work.zero();
    DBuf<uint2> vinfo(n, s);
    launch("hub_vprep", agg::k_hub_vprep, grid_for(n, 256), 256, 0, s, g->poff.p, g->padj.p, n, k,
           H, vinfo.p);
    if (H) {
      g->hmask.alloc(g->prio_nz * W, s);
      if (reinterpret_cast<uintptr_t>(g->hmask.p) & 15u) fail(kInternal, "hub masks not 16-byte aligned");
      switch (W) {
        case 1: launch_hub_mask<1>(g, vinfo.p); break;
        case 2: launch_hub_mask<2>(g, vinfo.p); break;
        case 4: launch_hub_mask<4>(g, vinfo.p); break;
        case 8: launch_hub_mask<8>(g, vinfo.p); break;
        case 16: launch_hub_mask<16>(g, vinfo.p); break;
        default: launch_hub_mask<32>(g, vinfo.p); break;
      }
    }
    launch("hub_plan", agg::k_hub_plan, grid_for(nnz, 256, 148u * 64u), 256, 0, s, g->padj.p,
           g->psrc.p, g->fseg.p, nnz, k, vinfo.p, g->hlen.p, g->hpst.p,
           reinterpret_cast<unsigned long long*>(g->hub_work.p));
  }
  g->hub_ready = true;
  if (k && std::getenv("BFLY_HUB_STATS")) {  // diagnostics: hub task work histogram
    std::vector<uint64_t> hw(n), dg(n + 1);
    read_back(s, {{hw.data(), g->hub_work.p, n * 8}, {dg.data(), g->poff.p, (n + 1) * 8}});
    uint64_t cnt[64] = {}, sum[64] = {}, ent[64] = {};
    std::vector<std::pair<uint64_t, uint64_t>> top;
    for (uint64_t i = 0; i < n; ++i) {
      if (!hw[i]) continue;
      const int b = 63 - __builtin_clzll(hw[i]);
      ++cnt[b];
      sum[b] += hw[i];
      ent[b] += dg[i + 1] - dg[i];
      top.push_back({hw[i], i});
    }
    std::sort(top.rbegin(), top.rend());
    fprintf(stderr, "[hub] k=%u k1=%u dense H=%u W=%u top-hub wedges per entry %.3f\n", k, k1, H, W,
            static_cast<double>(dense_keys) / static_cast<double>(nnz ? nnz : 1));
    for (int b = 0; b < 64; ++b)
      if (cnt[b])
        fprintf(stderr, "[hub] work 2^%d: tasks %llu keys %llu entries %llu\n", b,
                (unsigned long long)cnt[b], (unsigned long long)sum[b], (unsigned long long)ent[b]);
    for (size_t i = 0; i < std::min<size_t>(10, top.size()); ++i)
      fprintf(stderr, "[hub] top task w=%llu keys=%llu deg=%llu\n", (unsigned long long)top[i].second,
              (unsigned long long)top[i].first,
              (unsigned long long)(dg[top[i].second + 1] - dg[top[i].second]));
  }
}

// Hub tasks above this many keys are split over CTAs (heavy path, global rows of k counters)
// so one large end vertex cannot serialise the tail of the medium launch.
uint64_t hub_heavy_keys() {
  static const uint64_t v = [] {
    const char* e = std::getenv("BFLY_HUB_HEAVY_KEYS");
    return e ? std::strtoull(e, nullptr, 10) : ~0ull;
  }();
  return v;
}

// Hub tasks with at least this many entries are split into entry ranges of about this size
// (k_split): the top end vertices have ~10^5 entries each and would otherwise serialise the
// tail of the medium launch (one CTA walking 1000+ chunks).
uint64_t hub_split_units() {
  static const uint64_t v = [] {
    const char* e = std::getenv("BFLY_HUB_SPLIT_UNITS");
    return e ? std::strtoull(e, nullptr, 10) : 4096ull;
  }();
  return v;
}

static unsigned env_u(const char* name, unsigned dflt) {
  const char* e = std::getenv(name);
  return e ? static_cast<unsigned>(std::atoi(e)) : dflt;
}

// The dense top-hub kernels of one counting run, on two side streams of their own (they wait
// on random mask loads and share the SMs with the issue-bound segment walks).
struct DenseRun {
  bfly_graph* g;
  DBuf<unsigned long long> out;  // total, overflow flag, keys, entries, big entries
  DBuf<unsigned long long> dinfo;  // big tasks, their entries (k_dense_bounds)
  DBuf<uint32_t> rows;  // merge rows of the big tasks cut by chunk boundaries (zeroed per run)
  unsigned long long res[5] = {};
  cudaEvent_t fork = nullptr, join[2] = {};
  bool on = false, forked = false;
  explicit DenseRun(bfly_graph* g_) : g(g_) {
    if (!g->hub_h) return;
    on = true;
    out.alloc(5, g->stream);
    out.zero();
    dinfo.alloc(2, g->stream);
    rows.alloc(agg::dense_rows(2 * g->m) * 32 * g->hub_w, g->stream);
    rows.zero();
    launch("hub_dense_bounds", agg::k_dense_bounds, 1, 32, 0, g->stream, g->poff.p, g->prio_nz,
           dinfo.p);
    BFLY_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (auto& e : join) BFLY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~DenseRun() {
    if (fork) cudaEventDestroy(fork);
    for (auto& e : join)
      if (e) cudaEventDestroy(e);
  }
  DenseRun(const DenseRun&) = delete;
  DenseRun& operator=(const DenseRun&) = delete;
  template <int W>
  void go(cudaStream_t s_small, cudaStream_t s_big, uint64_t nt) {
    const uint32_t H = g->hub_h;
    // CTAs per SM of the two kernels: they wait on random mask loads, and a few resident
    // warps of them overlap the issue-bound segment walks launched behind them
    static const unsigned per_big = env_u("BFLY_DENSE_GRID_B", 5), per_small = env_u("BFLY_DENSE_GRID_S", 8);
    launch("hub_dense_big", agg::k_dense_big<W>, 148u * per_big, 256, 0, s_big, g->poff.p, g->padj.p,
           g->psrc.p, g->hmask.p, dinfo.p, H, rows.p, out.p);
    launch("hub_dense_small", agg::k_dense_small<W>, grid_for(nt * W, 256, 148u * per_small), 256, 0,
           s_small, g->poff.p, g->padj.p, g->hmask.p, nt, H, out.p);
  }
  void start(agg::SideStreams& ss, uint64_t nt) {
    if (!on) return;
    cudaStream_t s = g->stream;
    const bool conc = agg::agg_concurrent();
    cudaStream_t a = conc ? ss.s[10] : s, b = conc ? ss.s[11] : s;
    if (conc) {
      BFLY_CUDA(cudaEventRecord(fork, s));
      BFLY_CUDA(cudaStreamWaitEvent(a, fork, 0));
      BFLY_CUDA(cudaStreamWaitEvent(b, fork, 0));
    }
    switch (g->hub_w) {
      case 1: go<1>(a, b, nt); break;
      case 2: go<2>(a, b, nt); break;
      case 4: go<4>(a, b, nt); break;
      case 8: go<8>(a, b, nt); break;
      case 16: go<16>(a, b, nt); break;
      default: go<32>(a, b, nt); break;
    }
    if (conc) {
      BFLY_CUDA(cudaEventRecord(join[0], a));
      BFLY_CUDA(cudaEventRecord(join[1], b));
      forked = true;
    }
  }
  // The graph stream waits for the mask kernels only here, after every bucket kernel of the
  // phase has been forked: a wait placed right behind the launches would hold back the fork
  // events of the runs started after it, i.e. serialise the walks behind the mask kernels.
  void join_streams() {
    if (!forked) return;
    BFLY_CUDA(cudaStreamWaitEvent(g->stream, join[0], 0));
    BFLY_CUDA(cudaStreamWaitEvent(g->stream, join[1], 0));
    forked = false;
  }
  ReadBack::Item item() { return {res, out.p, sizeof(res)}; }
  uint64_t result() {
    if (!on) return 0;
    if (static_cast<unsigned>(res[1]) != 0) fail(kOverflow, "64-bit counter overflow in addition");
    g->hub_dense_keys = res[2];
    g->hub_dense_entries = res[3];
    g->hub_dense_big_entries = res[4];
    return res[0];
  }
};

template <bool LOCAL>
uint64_t count_all_starts(bfly_graph* g, agg::LocalOut lo, agg::RunStats* rs_hub,
                          agg::RunStats* rs_start) {
  const uint64_t n = g->n();
  // tasks: priority ids with edges (the rest have no work; sparsified sub-graphs keep every id)
  const uint64_t nt = g->prio_nz;
  cudaStream_t s = g->stream;
  ensure_hub_plan(g, !LOCAL);
  const uint32_t k = g->hub_k;
  g->hub_dense_keys = g->hub_dense_entries = 0;
  // hub path (starts u < k, task = end vertex w)
  agg::HubSrc hsrc{g->poff.p, g->padj.p, g->hlen.p, g->hpst.p};
  // small hub tasks: per-warp bitmap of first occurrences + hash of repeats (<= 256
  // repeated keys for <= 512 keys); larger ones: per-CTA dense k-entry table with 32-bit
  // counters below k1 and packed 16-bit counters above (geometry k | k1 << 16)
  const uint32_t kk = k | (g->hub_k1 << 16);
  const char* mb = std::getenv("BFLY_HUB_MED_BLOCK");
  const int med_block = mb ? std::atoi(mb) : 256;
  static const char* const hnames[8] = {"hub_bucket", "hub_tiny",        "hub_small",
                                        "hub_medium", "hub_medium_wide", "hub_heavy", "hub_phase", "hub_small_b"};
  DBuf<unsigned long long> deg;  // entries of a hub task = degree of w
  if (k) {
    deg.alloc(n, s);
    launch("hub_units", agg::k_degree_units, grid_for(n, 256), 256, 0, s, g->poff.p, n, deg.p);
  }
  const auto* hw = reinterpret_cast<const unsigned long long*>(g->hub_work.p);
  // warp tables sized to the task: <= 256 keys in BitHash<8> (<= 128 repeated keys),
  // <= 512 keys in BitHash<9>; the smaller table roughly doubles resident warps. BitHash
  // tables are reset whole after each task
  // medium tasks with < 256 entries count in bytes (c(u, w) <= entries of w), the rest in
  // the 32/16-bit split table
#ifndef BFLY_HUB_SA_BITS
#define BFLY_HUB_SA_BITS 7
#endif
#ifndef BFLY_HUB_SB_BITS
#define BFLY_HUB_SB_BITS 9
#endif
  // repeat hashes of 2^BITS slots for tasks of <= 2^(BITS+1) keys: at most 2^BITS distinct
  // keys repeat, so an insert always finds a slot and a lookup of a key seen once always
  // meets an empty one (a full table leaves no key seen once)
  using SmallA = agg::BitHash<BFLY_HUB_SA_BITS>;
  using SmallB = agg::BitHash<BFLY_HUB_SB_BITS>;
#ifndef BFLY_HUB_LIM2
#define BFLY_HUB_LIM2 1024
#endif
  agg::Plan<SmallA, SmallB, agg::DirectByte, agg::DirectSplit> hplan{
      kk, {LOCAL ? 32u : agg::kTinyLaneMax, 256, BFLY_HUB_LIM2, hub_heavy_keys()}, 0, med_block,
      256, hub_split_units()};
  hplan.wide_block = [] {
    const char* e = std::getenv("BFLY_HUB_WIDE_BLOCK");
    return e ? std::atoi(e) : 0;
  }();
  agg::LocalOut hlo = lo;
  DBuf<unsigned long long> krow;
  if (LOCAL && k) {
    krow.alloc(uint64_t{agg::kKeyRows} * k, s);
    krow.zero();
    hlo.krow = krow.p;
    hlo.kstride = k;
  }
  agg::Agg<agg::HubSrc, LOCAL, SmallA, SmallB, agg::DirectByte,
           agg::DirectSplit>
      hub(g, hsrc, hplan, hw, deg.p, k ? nt : 0, k, nullptr, hlo, rs_hub, hnames);
  DenseRun dense(g);  // (off when the plan has no dense hubs: local-count runs, k = 0)
  // start path (starts u >= k, task = start u)
  agg::ExactSrc src{g->poff.p, g->padj.p, g->fseg.p, g->fwd.p};
  DBuf<unsigned long long> units(n, s);
  launch("exact_fwd_count", agg::k_fwd_count, grid_for(n, 256), 256, 0, s, g->poff.p, g->fwd.p, n,
         units.p);
  // medium start tasks: <= 2048 keys in a 4096-slot table (load <= 1/2, 32 KB -> 6 CTAs per
  // SM), up to 8192 keys in the 16384-slot table
#ifndef BFLY_EXACT_MED_BITS
#define BFLY_EXACT_MED_BITS 12
#endif
  using ExMedU = agg::Hash<BFLY_EXACT_MED_BITS>;
  // warp tables of the start path: one-word (key, count) slots when every priority id fits 23
  // bits (counts < 512: the small-B tier then stops at 511 keys), else two-word slots
  auto start_path = [&](auto small_a, auto small_b, uint32_t lim_b, auto med_tab,
                        auto wide_tab) -> uint64_t {
    using SA = decltype(small_a);
    using SB = decltype(small_b);
    using ExMed = decltype(med_tab);
    using ExWide = decltype(wide_tab);
    agg::Plan<SA, SB, ExMed, ExWide> plan{
        0, {LOCAL ? 32u : agg::kTinyLaneMax, 256, lim_b, 8192}, k};
    plan.med_block = [] {
      const char* e = std::getenv("BFLY_EXACT_MED_BLOCK");
      return (e && std::atoi(e) == 128) ? 128 : 256;
    }();
    plan.wide_work = 1u << (BFLY_EXACT_MED_BITS - 1);  // medium table load <= 1/2
    // medium-wide CTAs: 512 threads on the 64 KB one-word table (alone the kernel is slower
    // than with 1024, 0.86 against 0.67 ms, but the smaller CTAs leave room for the other
    // buckets' kernels: counting phase 8.77 -> 8.59 ms); 1024 threads on the 128 KB two-word
    // table, one per SM (BFLY_EXACT_WIDE_BLOCK overrides)
    plan.wide_block = [] {
      const char* e = std::getenv("BFLY_EXACT_WIDE_BLOCK");
      const int dflt = std::is_same_v<ExWide, agg::Hash<14>> ? 1024 : 512;
      const int v = e ? std::atoi(e) : dflt;
      return (v == 128 || v == 256 || v == 512 || v == 1024) ? v : dflt;
    }();
    static const char* const names[8] = {"exact_bucket", "exact_tiny",  "exact_small",
                                         "exact_medium", "exact_medium_wide", "exact_heavy",
                                         "exact_phase", "exact_small_b"};
    agg::Agg<agg::ExactSrc, LOCAL, SA, SB, ExMed, ExWide> ex(
        g, src, plan, reinterpret_cast<const unsigned long long*>(g->work.p), units.p, nt, n,
        nullptr, lo, rs_start, names);
    // both runs' bucket counts in one sync, then every bucket kernel of both paths in flight
    // together (hub buckets on side streams 0-4, start buckets on 5-9, heavy buckets on the
    // graph stream), one join, one sync for both totals
    if (k) read_back(s, {hub.counts_item(), ex.counts_item()});
    else read_back(s, {ex.counts_item()});
    agg::SideStreams& ss = agg::side_streams(g->device);
    {
      ProfScope phase("count_phase", s);
      static const bool dense_first = env_u("BFLY_DENSE_FIRST", 1) != 0;
      if (dense_first) dense.start(ss, nt);
      ex.start(ss, 5);  // (start path first: measured 0.04 ms better than hub first)
      if (!dense_first) dense.start(ss, nt);
      hub.start(ss, 0);
      dense.join_streams();
      hub.join(ss);
      ex.join(ss);
    }
    if (LOCAL && k)
      launch("hub_key_rows", agg::k_sum_key_rows, grid_for(k, 256), 256, 0, s, krow.p,
             agg::kKeyRows, k, lo.vcnt);
    if (k && dense.on) read_back(s, {hub.total_item(), ex.total_item(), dense.item()});
    else if (k) read_back(s, {hub.total_item(), ex.total_item()});
    else read_back(s, {ex.total_item()});
    const uint64_t total = hub.result(), t2 = ex.result(), t3 = dense.result();
    const uint64_t sum = total + t2;
    if (sum < total) fail(kOverflow, "64-bit counter overflow in addition");
    if (sum + t3 < sum) fail(kOverflow, "64-bit counter overflow in addition");
    return sum + t3;
  };
  // CTA tables of the start path: one-word slots too when, besides the 23-bit ids, no start
  // task can reach a count of 512 -- a count is at most the task's entries, and every start
  // task's degree is at most that of priority id k (degrees descend; config 2: 260)
  static const bool packed_med = env_u("BFLY_PACKED_MED", 1) != 0;
  if (n < (1u << 23) - 1) {
    if (packed_med && g->start_deg_max < 512)
      return start_path(agg::PackedHash<9, 9>{}, agg::PackedHash<10, 9>{}, 511u,
                        agg::PackedHash<BFLY_EXACT_MED_BITS, 9>{}, agg::PackedHash<14, 9>{});
    return start_path(agg::PackedHash<9, 9>{}, agg::PackedHash<10, 9>{}, 511u, ExMedU{},
                      agg::Hash<14>{});
  }
  return start_path(agg::Hash<9>{}, agg::Hash<10>{}, 512u, ExMedU{}, agg::Hash<14>{});
}

template uint64_t count_all_starts<true>(bfly_graph*, agg::LocalOut, agg::RunStats*,
                                         agg::RunStats*);

uint64_t exact_count_device(bfly_graph* g, const uint32_t*) {
  ensure_priority(g, false);
  g->last_wedges = 0;
  for (int q = 0; q < 6; ++q) {
    g->bucket_starts[q] = g->bucket_wedges[q] = g->bucket_entries[q] = 0;
    g->hub_bucket_tasks[q] = g->hub_bucket_keys[q] = g->hub_bucket_entries[q] = 0;
  }
  if (g->n() == 0 || g->m == 0) return 0;
  agg::RunStats rh, rs;
  const uint64_t total = count_all_starts<false>(
      g, agg::LocalOut{nullptr, nullptr, nullptr, nullptr}, &rh, &rs);
  for (int q = 0; q < 6; ++q) {
    g->bucket_starts[q] = rs.starts[q];
    g->bucket_wedges[q] = rs.wedges[q];
    g->bucket_entries[q] = rs.entries[q];
    g->hub_bucket_tasks[q] = rh.starts[q];
    g->hub_bucket_keys[q] = rh.wedges[q];
    g->hub_bucket_entries[q] = rh.entries[q];
    g->last_wedges += rs.wedges[q] + rh.wedges[q];
  }
  g->last_wedges += g->hub_dense_keys;  // wedges counted from the top-hub masks
  return total;
}

}  // namespace bflyd
