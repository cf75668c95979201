// samples.cu -- batched per-sample kernels and small graph queries.
//
//   edge samples   count_per_edge(l, r) (local.cpp:23-44). With a the lower-degree endpoint
//                  and b the other, the reference counts x in N(b)\{a} reached from N(a) and
//                  sums (mult - 1). Every x in N(b)\{a} is reached through w = b, so the sum
//                  equals  sum over w in N(a)\{b} of (|N(w) & N(b)| - 1)  -- an exact integer
//                  identity; the kernel evaluates it with sorted-list intersections.
//   wedge samples  |N(v) & N(w)| - 1 for two leaves of a centre (sampling.cpp:85-91).
//   has_edge       binary search in the shorter list (graph.cpp:60-66).
//   edge_at        upper_bound over the left offsets (graph.cpp:68-73).
//   wedge index    prefix of C(d,2) over the global order (sampling.cpp:63-73).
#include "cubwrap.cuh"
#include "scan.cuh"
#include "local.cuh"

namespace bflyd {
namespace {

__device__ __forceinline__ bool bsearch_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && a[lo] == x;
}

// |A & B| for two ascending lists, cooperatively by one warp (all lanes return the sum)
__device__ __forceinline__ uint64_t warp_intersect(const uint32_t* a, uint64_t na,
                                                   const uint32_t* b, uint64_t nb) {
  if (na > nb) {
    const uint32_t* t = a;
    a = b;
    b = t;
    const uint64_t tn = na;
    na = nb;
    nb = tn;
  }
  uint64_t c = 0;
  for (uint64_t i = threadIdx.x & 31; i < na; i += 32) c += bsearch_u32(b, nb, a[i]);
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  return c;
}

__global__ void k_edge_at(const uint64_t* __restrict__ loff, uint32_t L,
                          const uint32_t* __restrict__ ladj, const uint64_t* __restrict__ ks,
                          uint64_t k, uint32_t* __restrict__ lo_out, uint32_t* __restrict__ r_out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = ks[i];
    uint64_t lo = 0, hi = uint64_t{L} + 1;  // first index with loff > e
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (loff[mid] <= e) lo = mid + 1;
      else hi = mid;
    }
    lo_out[i] = static_cast<uint32_t>(lo - 1);
    r_out[i] = ladj[e];
  }
}

__global__ void k_has_edge(const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
                           const uint64_t* __restrict__ roff, const uint32_t* __restrict__ radj,
                           const uint32_t* __restrict__ l, const uint32_t* __restrict__ r,
                           uint64_t k, uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = l[i], b = r[i];
    const uint64_t dl = loff[a + 1] - loff[a], dr = roff[b + 1] - roff[b];
    out[i] = dl <= dr ? bsearch_u32(ladj + loff[a], dl, b) : bsearch_u32(radj + roff[b], dr, a);
  }
}

// ---- edge samples as balanced intersection jobs ---------------------------------------------
// count_per_edge(l, r) = sum over w in N(a) \ {b} of (|N(w) & N(b)| - 1): one JOB per (sample,
// w), cut into sub-jobs of kEdgeChunk elements of the shorter of the two lists, so a sample
// whose endpoints touch hubs no longer runs as one warp's serial loop. Sub-job (i, t, c): the
// t-th neighbour w of sample i's a, chunk c; chunk 0 also carries the -1.
constexpr uint32_t kEdgeChunk = 1024;
struct EdgeSide {
  const uint32_t* na;  // N(a) (ids on b's side)
  const uint32_t* nb;  // N(b) (ids on a's side)
  uint64_t da, db;
  uint32_t b;
  const uint64_t* woff;
  const uint32_t* wadj;
};
__device__ __forceinline__ EdgeSide edge_side(const uint64_t* loff, const uint32_t* ladj,
                                              const uint64_t* roff, const uint32_t* radj,
                                              uint32_t l, uint32_t r) {
  const uint64_t dl = loff[l + 1] - loff[l], dr = roff[r + 1] - roff[r];
  const bool swap = dl > dr;  // a = lower-degree endpoint, ties keep the left (local.cpp:29)
  EdgeSide e;
  e.na = swap ? radj + roff[r] : ladj + loff[l];
  e.da = swap ? dr : dl;
  e.nb = swap ? ladj + loff[l] : radj + roff[r];
  e.db = swap ? dl : dr;
  e.b = swap ? l : r;
  e.woff = swap ? loff : roff;
  e.wadj = swap ? ladj : radj;
  return e;
}
__device__ __forceinline__ uint32_t edge_chunks(const EdgeSide& e, uint32_t w) {
  if (w == e.b) return 0;
  const uint64_t dw = e.woff[w + 1] - e.woff[w];
  const uint64_t sm = dw < e.db ? dw : e.db;
  return static_cast<uint32_t>((sm + kEdgeChunk - 1) / kEdgeChunk);
}

// warp per sample: number of sub-jobs
__global__ void __launch_bounds__(256) k_edge_job_count(
    const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
    const uint64_t* __restrict__ roff, const uint32_t* __restrict__ radj,
    const uint32_t* __restrict__ ls, const uint32_t* __restrict__ rs, uint64_t k,
    uint32_t* __restrict__ njobs) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < k; i += nw) {
    const EdgeSide e = edge_side(loff, ladj, roff, radj, ls[i], rs[i]);
    uint32_t c = 0;
    for (uint64_t t = lane; t < e.da; t += 32) c += edge_chunks(e, e.na[t]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) njobs[i] = c;
  }
}

// warp per sample: write its sub-jobs (i, t, c) at joff[i]
__global__ void __launch_bounds__(256) k_edge_job_fill(
    const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
    const uint64_t* __restrict__ roff, const uint32_t* __restrict__ radj,
    const uint32_t* __restrict__ ls, const uint32_t* __restrict__ rs, uint64_t k,
    const uint64_t* __restrict__ joff, uint4* __restrict__ jobs) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < k; i += nw) {
    const EdgeSide e = edge_side(loff, ladj, roff, radj, ls[i], rs[i]);
    uint64_t pos = joff[i];
    for (uint64_t tb = 0; tb < e.da; tb += 32) {
      const uint64_t t = tb + lane;
      const uint32_t c = t < e.da ? edge_chunks(e, e.na[t]) : 0u;
      uint32_t incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      for (uint32_t q = 0; q < c; ++q)
        jobs[pos + incl - c + q] = make_uint4(static_cast<uint32_t>(i), static_cast<uint32_t>(t), q, 0u);
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// warp per sub-job: binary searches of one chunk of the shorter list in the longer one
__global__ void __launch_bounds__(256) k_edge_job_run(
    const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
    const uint64_t* __restrict__ roff, const uint32_t* __restrict__ radj,
    const uint32_t* __restrict__ ls, const uint32_t* __restrict__ rs,
    const uint4* __restrict__ jobs, uint64_t nj, unsigned long long* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t j = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; j < nj; j += nw) {
    const uint4 jb = jobs[j];
    const EdgeSide e = edge_side(loff, ladj, roff, radj, ls[jb.x], rs[jb.x]);
    const uint32_t w = e.na[jb.y];
    const uint32_t* nw_ = e.wadj + e.woff[w];
    const uint64_t dw = e.woff[w + 1] - e.woff[w];
    const uint32_t* sa = nw_;  // shorter list
    const uint32_t* lb = e.nb;
    uint64_t ns = dw, nl = e.db;
    if (ns > nl) {
      sa = e.nb;
      lb = nw_;
      ns = e.db;
      nl = dw;
    }
    const uint64_t c0 = uint64_t{jb.z} * kEdgeChunk;
    const uint64_t c1 = c0 + kEdgeChunk < ns ? c0 + kEdgeChunk : ns;
    unsigned long long c = 0;
    for (uint64_t q = c0 + lane; q < c1; q += 32) c += bsearch_u32(lb, nl, sa[q]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    // a is in both lists: its -1 rides on chunk 0 (modular adds; the final sum is >= 0)
    if (lane == 0) atomicAdd(&out[jb.x], jb.z == 0 ? c - 1ull : c);
  }
}

// Wedge samples: |N(v) & N(w)| - 1 for the two leaves (sampling.cpp:85-91). A warp per
// sample handles intersections whose shorter list has <= kEdgeChunk elements directly; the
// rare larger ones (two hub leaves) are cut into chunk jobs run by other warps (njobs[q] > 0;
// out[q] starts at -1 mod 2^64 and the chunks add their counts).
__device__ __forceinline__ bool wedge_leaves(const uint64_t* loff, const uint32_t* ladj,
                                             const uint64_t* roff, const uint32_t* radj,
                                             uint32_t L, uint64_t c, uint32_t i, uint32_t j,
                                             const uint32_t*& a, uint64_t& na,
                                             const uint32_t*& b, uint64_t& nb) {
  const bool left = c < L;
  const uint64_t d = left ? loff[c + 1] - loff[c] : roff[c - L + 1] - roff[c - L];
  if (i >= d || j >= d || i == j) return false;  // not two distinct neighbours
  const uint32_t* cadj = left ? ladj + loff[c] : radj + roff[c - L];
  const uint32_t v = cadj[i], w = cadj[j];
  // leaves live on the opposite side; intersect their lists (sampling.cpp:88-89)
  const uint64_t* lo = left ? roff : loff;
  const uint32_t* la = left ? radj : ladj;
  a = la + lo[v];
  na = lo[v + 1] - lo[v];
  b = la + lo[w];
  nb = lo[w + 1] - lo[w];
  if (na > nb) {  // a = the shorter list
    const uint32_t* t = a;
    a = b;
    b = t;
    const uint64_t tn = na;
    na = nb;
    nb = tn;
  }
  return true;
}

__global__ void __launch_bounds__(256) k_wedge_samples(
    const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
    const uint64_t* __restrict__ roff, const uint32_t* __restrict__ radj, uint32_t L,
    const uint64_t* __restrict__ cs, const uint32_t* __restrict__ is,
    const uint32_t* __restrict__ js, uint64_t k, unsigned long long* __restrict__ out,
    uint32_t* __restrict__ njobs, unsigned* __restrict__ err) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t q = gw; q < k; q += nw) {
    const uint32_t* a;
    const uint32_t* b;
    uint64_t na, nb;
    if (!wedge_leaves(loff, ladj, roff, radj, L, cs[q], is[q], js[q], a, na, b, nb)) {
      if (lane == 0) {
        out[q] = 0;
        njobs[q] = 0;
        atomicOr(err, 1u);
      }
      continue;
    }
    if (na > kEdgeChunk) {  // chunk jobs
      if (lane == 0) {
        out[q] = ~0ull;
        njobs[q] = static_cast<uint32_t>((na + kEdgeChunk - 1) / kEdgeChunk);
      }
      continue;
    }
    uint64_t cnt = 0;
    for (uint64_t t = lane; t < na; t += 32) cnt += bsearch_u32(b, nb, a[t]);
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (lane == 0) {
      out[q] = cnt - 1;
      njobs[q] = 0;
    }
  }
}

// thread per sample with jobs: (sample, chunk) records at joff[q]
__global__ void k_wedge_job_fill(const uint32_t* __restrict__ njobs, const uint64_t* __restrict__ joff,
                                 uint64_t k, uint2* __restrict__ jobs) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < k;
       q += (uint64_t)gridDim.x * blockDim.x)
    for (uint32_t c = 0; c < njobs[q]; ++c) jobs[joff[q] + c] = make_uint2(static_cast<uint32_t>(q), c);
}

__global__ void __launch_bounds__(256) k_wedge_job_run(
    const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
    const uint64_t* __restrict__ roff, const uint32_t* __restrict__ radj, uint32_t L,
    const uint64_t* __restrict__ cs, const uint32_t* __restrict__ is,
    const uint32_t* __restrict__ js, const uint2* __restrict__ jobs, uint64_t nj,
    unsigned long long* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t j = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; j < nj; j += nw) {
    const uint2 jb = jobs[j];
    const uint32_t* a;
    const uint32_t* b;
    uint64_t na, nb;
    wedge_leaves(loff, ladj, roff, radj, L, cs[jb.x], is[jb.x], js[jb.x], a, na, b, nb);
    const uint64_t c0 = uint64_t{jb.y} * kEdgeChunk;
    const uint64_t c1 = c0 + kEdgeChunk < na ? c0 + kEdgeChunk : na;
    unsigned long long c = 0;
    for (uint64_t t = c0 + lane; t < c1; t += 32) c += bsearch_u32(b, nb, a[t]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0 && c) atomicAdd(&out[jb.x], c);
  }
}

__global__ void __launch_bounds__(256) k_common_pairs(
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
    const uint32_t* __restrict__ vs, const uint32_t* __restrict__ ws, uint64_t k,
    unsigned long long* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t q = gw; q < k; q += nw) {
    const uint32_t v = vs[q], w = ws[q];
    const uint64_t c =
        warp_intersect(adj + off[v], off[v + 1] - off[v], adj + off[w], off[w + 1] - off[w]);
    if (lane == 0) out[q] = c;
  }
}

// elements the per-sample walk of count_per_edge(l, r) touches: sum over N(a) of degrees
__global__ void k_edge_cost(const uint64_t* __restrict__ loff, const uint64_t* __restrict__ roff,
                            uint32_t L, const unsigned long long* __restrict__ two_hop,
                            const uint32_t* __restrict__ ls, const uint32_t* __restrict__ rs,
                            uint64_t k, unsigned long long* __restrict__ cost) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t l = ls[i], r = rs[i];
    const uint64_t dl = loff[l + 1] - loff[l], dr = roff[r + 1] - roff[r];
    cost[i] = dl > dr ? two_hop[uint64_t{L} + r] + dr : two_hop[l] + dl;
  }
}

// canonical edge id of (l, r) (the pair is known to be an edge)
__global__ void k_edge_index(const uint64_t* __restrict__ loff, const uint32_t* __restrict__ ladj,
                             const uint32_t* __restrict__ ls, const uint32_t* __restrict__ rs,
                             uint64_t k, uint64_t* __restrict__ ks) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = loff[ls[i]], hi = loff[ls[i] + 1];
    const uint32_t r = rs[i];
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (ladj[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    ks[i] = lo;
  }
}

__global__ void k_choose2_global(const uint64_t* __restrict__ loff, const uint64_t* __restrict__ roff,
                                 uint32_t L, uint32_t R, unsigned long long* __restrict__ c2) {
  const uint64_t n = uint64_t{L} + R;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g <= n;
       g += (uint64_t)gridDim.x * blockDim.x) {
    if (g == n) {
      c2[g] = 0;
      continue;
    }
    const uint64_t d = g < L ? loff[g + 1] - loff[g] : roff[g - L + 1] - roff[g - L];
    c2[g] = d < 2 ? 0ull : (d % 2 == 0 ? (d / 2) * (d - 1) : d * ((d - 1) / 2));
  }
}

}  // namespace

void edge_at_device(bfly_graph* g, const uint64_t* d_k, uint64_t k, uint32_t* d_l, uint32_t* d_r) {
  if (!k) return;
  launch("edge_at", k_edge_at, grid_for(k, 256), 256, 0, g->stream, g->loff.p, g->L, g->ladj.p,
         d_k, k, d_l, d_r);
}

void has_edge_device(bfly_graph* g, const uint32_t* d_l, const uint32_t* d_r, uint64_t k,
                     uint8_t* d_out) {
  if (!k) return;
  launch("has_edge", k_has_edge, grid_for(k, 256), 256, 0, g->stream, g->loff.p, g->ladj.p,
         g->roff.p, g->radj.p, d_l, d_r, k, d_out);
}

void local_edge_batch_device(bfly_graph* g, const uint32_t* d_l, const uint32_t* d_r,
                             const uint64_t* d_k, uint64_t k, unsigned long long* d_out) {
  if (!k) return;
  cudaStream_t s = g->stream;
  ensure_two_hop(g);
  DBuf<unsigned long long> cost(k, s);
  launch("esamp_cost", k_edge_cost, grid_for(k, 256), 256, 0, s, g->loff.p, g->roff.p, g->L,
         reinterpret_cast<const unsigned long long*>(g->two_hop.p), d_l, d_r, k, cost.p);
  if (prefer_all_subjects(g, device_sum(g, cost.p, k), true)) {
    g->last_sample_path = 1;
    DBuf<uint64_t> ks;
    if (!d_k) {
      ks.alloc(k, s);
      launch("edge_index", k_edge_index, grid_for(k, 256), 256, 0, s, g->loff.p, g->ladj.p, d_l,
             d_r, k, ks.p);
      d_k = ks.p;
    }
    gather_all_subjects(g, true, d_k, k, d_out);
    BFLY_CUDA(cudaStreamSynchronize(s));
    return;
  }
  g->last_sample_path = 0;
  DBuf<uint32_t> nj(k, s);
  DBuf<uint64_t> joff(k + 1, s);
  launch("esamp_jobs", k_edge_job_count, grid_for(k * 32, 256, 148u * 64u), 256, 0, s, g->loff.p,
         g->ladj.p, g->roff.p, g->radj.p, d_l, d_r, k, nj.p);
  scan::exclusive_sum<uint64_t>(nj.p, k, joff.p, s, "esamp_jobs");
  uint64_t njobs = 0;
  read_back(s, {{&njobs, joff.p + k, 8}});
  BFLY_CUDA(cudaMemsetAsync(d_out, 0, k * 8, s));
  if (njobs == 0) return;
  DBuf<uint4> jobs(njobs, s);
  launch("esamp_jobs", k_edge_job_fill, grid_for(k * 32, 256, 148u * 64u), 256, 0, s, g->loff.p,
         g->ladj.p, g->roff.p, g->radj.p, d_l, d_r, k, (const uint64_t*)joff.p, jobs.p);
  launch("esamp_intersect", k_edge_job_run, grid_for(njobs * 32, 256, 148u * 64u), 256, 0, s,
         g->loff.p, g->ladj.p, g->roff.p, g->radj.p, d_l, d_r, (const uint4*)jobs.p, njobs,
         d_out);
}

void wedge_batch_device(bfly_graph* g, const uint64_t* d_c, const uint32_t* d_i,
                        const uint32_t* d_j, uint64_t k, unsigned long long* d_out) {
  if (!k) return;
  cudaStream_t s = g->stream;
  DBuf<unsigned> err(1, s);
  err.zero();
  DBuf<uint32_t> nj(k, s);
  DBuf<uint64_t> joff(k + 1, s);
  launch("wsamp_intersect", k_wedge_samples, grid_for(k * 32, 256, 148u * 64u), 256, 0, s,
         g->loff.p, g->ladj.p, g->roff.p, g->radj.p, g->L, d_c, d_i, d_j, k, d_out, nj.p, err.p);
  scan::exclusive_sum<uint64_t>(nj.p, k, joff.p, s, "wsamp_jobs");
  unsigned h = 0;
  uint64_t njobs = 0;
  read_back(s, {{&h, err.p, 4}, {&njobs, joff.p + k, 8}});
  if (h) fail(kArgument, "wedge sample needs two distinct neighbour positions of the centre");
  if (njobs) {  // the large intersections, in chunks
    DBuf<uint2> jobs(njobs, s);
    launch("wsamp_jobs", k_wedge_job_fill, grid_for(k, 256), 256, 0, s, (const uint32_t*)nj.p,
           (const uint64_t*)joff.p, k, jobs.p);
    launch("wsamp_intersect", k_wedge_job_run, grid_for(njobs * 32, 256, 148u * 64u), 256, 0, s,
           g->loff.p, g->ladj.p, g->roff.p, g->radj.p, g->L, d_c, d_i, d_j,
           (const uint2*)jobs.p, njobs, d_out);
    BFLY_CUDA(cudaStreamSynchronize(s));
  }
}

void common_pairs_device(bfly_graph* g, int side, const uint32_t* d_v, const uint32_t* d_w,
                         uint64_t k, unsigned long long* d_out) {
  if (!k) return;
  launch("common_pairs", k_common_pairs, grid_for(k * 32, 256, 148u * 64u), 256, 0, g->stream,
         side == 0 ? g->loff.p : g->roff.p, side == 0 ? g->ladj.p : g->radj.p, d_v, d_w, k, d_out);
}

// prefix[n+1] of C(d,2) over global order into a device buffer; *total = prefix[n]
void wedge_prefix_device(bfly_graph* g, unsigned long long* d_pre, uint64_t* total) {
  cudaStream_t s = g->stream;
  ensure_stats(g);
  if (g->stats_status) fail(g->stats_status, "64-bit counter overflow in addition");
  const uint64_t n = g->n();
  DBuf<unsigned long long> c2(n + 1, s);
  launch("wedge_index_c2", k_choose2_global, grid_for(n + 1, 256), 256, 0, s, g->loff.p, g->roff.p,
         g->L, g->R, c2.p);
  exclusive_sum(c2.p, d_pre, n + 1, s);
  unsigned long long t = 0;
  BFLY_CUDA(cudaMemcpyAsync(&t, d_pre + n, 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  *total = t;
}

void wedge_index(bfly_graph* g, uint64_t* prefix, uint64_t* total) {
  ensure_wedge_prefix(g);
  BFLY_CUDA(cudaMemcpyAsync(prefix, g->wpre.p, (g->n() + 1) * 8, cudaMemcpyDeviceToHost, g->stream));
  BFLY_CUDA(cudaStreamSynchronize(g->stream));
  *total = g->wtotal;
}

}  // namespace bflyd
