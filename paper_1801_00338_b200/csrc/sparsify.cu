// sparsify.cu -- sparsify-then-count (replaces count_retained + exact_count,
// sparsify.cpp:15-71).
//
// The keep predicate is evaluated per canonical edge inside the compaction kernels:
//   ESpar  keep k  iff  unit_double(derive_seed(seed, k)) < p           (sparsify.cpp:60-61)
//   CSpar  keep (l,r) iff colour(l) == colour(L + r),
//          colour(g) = bounded_from_bits(derive_seed(seed, g), N)       (sparsify.cpp:65-70)
// The retained edges are compacted into both CSR directions over the SAME dense ids (the
// reference renumbers through from_edges, sparsify.cpp:15-24; butterfly counts are
// invariant under relabelling and isolated vertices contribute nothing), and the exact
// kernel counts the compacted graph.
#include "cubwrap.cuh"
#include "local.cuh"

namespace bflyd {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint32_t colour(uint64_t ms, uint64_t g, uint64_t n_colors) {
  return static_cast<uint32_t>(__umul64hi(mix64(ms ^ mix64(g)), n_colors));
}

__global__ void k_mark(const uint64_t* __restrict__ off, uint32_t rows, uint32_t* __restrict__ mark) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    if (off[r + 1] > off[r]) mark[off[r]] = static_cast<uint32_t>(r);
}

// keep flag per canonical edge (left CSR order)
__global__ void k_keep(int mode, double p, uint64_t n_colors, uint64_t ms, uint32_t L,
                       const uint32_t* __restrict__ lrow, const uint32_t* __restrict__ ladj,
                       const uint8_t* __restrict__ hkeep, const uint32_t* __restrict__ hcol,
                       uint64_t m, uint32_t* __restrict__ flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x) {
    bool keep;
    if (mode == 0) {
      const uint64_t h = mix64(ms ^ mix64(k));
      keep = static_cast<double>(h >> 11) * 0x1.0p-53 < p;
    } else if (mode == 1) {
      keep = colour(ms, lrow[k], n_colors) == colour(ms, uint64_t{L} + ladj[k], n_colors);
    } else if (mode == 2) {
      keep = hkeep[k] != 0;
    } else {
      keep = hcol[lrow[k]] == hcol[uint64_t{L} + ladj[k]];
    }
    flag[k] = keep ? 1u : 0u;
  }
}

__global__ void k_right_flags(const uint32_t* __restrict__ reid, const uint32_t* __restrict__ flag,
                              uint64_t m, uint32_t* __restrict__ rflag) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m;
       j += (uint64_t)gridDim.x * blockDim.x)
    rflag[j] = flag[reid[j]];
}

// new offsets: off'[r] = pos[off[r]] (pos = exclusive scan of flags, pos[m] = m')
__global__ void k_new_off(const uint64_t* __restrict__ off, uint32_t rows,
                          const unsigned long long* __restrict__ pos, uint64_t* __restrict__ noff) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    noff[r] = pos[off[r]];
}

__global__ void k_compact_left(const uint32_t* __restrict__ ladj, const uint32_t* __restrict__ flag,
                               const unsigned long long* __restrict__ pos, uint64_t m,
                               uint32_t* __restrict__ nladj) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x)
    if (flag[k]) nladj[pos[k]] = ladj[k];
}

__global__ void k_compact_right(const uint32_t* __restrict__ radj, const uint32_t* __restrict__ reid,
                                const uint32_t* __restrict__ rflag,
                                const unsigned long long* __restrict__ rpos,
                                const unsigned long long* __restrict__ lpos, uint64_t m,
                                uint32_t* __restrict__ nradj, uint32_t* __restrict__ nreid) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m;
       j += (uint64_t)gridDim.x * blockDim.x)
    if (rflag[j]) {
      nradj[rpos[j]] = radj[j];
      nreid[rpos[j]] = static_cast<uint32_t>(lpos[reid[j]]);
    }
}

}  // namespace

void sparsify_count(bfly_graph* g, int mode, double p, uint64_t n_colors, uint64_t seed,
                    const uint8_t* h_keep, const uint32_t* h_colors, uint64_t* count,
                    uint64_t* kept) {
  cudaStream_t s = g->stream;
  const uint64_t m = g->m, n = g->n();
  *count = 0;
  *kept = 0;
  if (m == 0) return;
  // mix64(seed) is hoisted: derive_seed(seed, i) = mix64(mix64(seed) ^ mix64(i))
  uint64_t ms = seed;
  {
    uint64_t x = seed + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    ms = x ^ (x >> 31);
  }
  DBuf<uint8_t> dkeep;
  DBuf<uint32_t> dcol;
  if (mode == 2) {
    dkeep.alloc(m, s);
    BFLY_CUDA(cudaMemcpyAsync(dkeep.p, h_keep, m, cudaMemcpyHostToDevice, s));
  } else if (mode == 3) {
    dcol.alloc(n, s);
    BFLY_CUDA(cudaMemcpyAsync(dcol.p, h_colors, n * 4, cudaMemcpyHostToDevice, s));
  }
  DBuf<uint32_t> lrow_tmp;
  const uint32_t* lrow = g->lrow.p;  // left row of each canonical edge, from the build
  if ((mode == 1 || mode == 3) && !lrow) {
    DBuf<uint32_t> mark(m, s);
    mark.zero();
    lrow_tmp.alloc(m, s);
    launch("spar_mark_rows", k_mark, grid_for(g->L, 256), 256, 0, s, g->loff.p, g->L, mark.p);
    inclusive_max(mark.p, lrow_tmp.p, m, s);
    lrow = lrow_tmp.p;
  }
  ensure_reid(g);  // right entries are kept by their canonical edge's flag
  DBuf<uint32_t> flag(m + 1, s), rflag(m + 1, s);
  launch("spar_keep", k_keep, grid_for(m, 256), 256, 0, s, mode, p, n_colors, ms, g->L, lrow,
         g->ladj.p, dkeep.p, dcol.p, m, flag.p);
  launch("spar_right_flags", k_right_flags, grid_for(m, 256), 256, 0, s, g->reid.p, flag.p, m,
         rflag.p);
  BFLY_CUDA(cudaMemsetAsync(flag.p + m, 0, 4, s));
  BFLY_CUDA(cudaMemsetAsync(rflag.p + m, 0, 4, s));
  DBuf<unsigned long long> lpos(m + 1, s), rpos(m + 1, s);
  exclusive_sum(flag.p, lpos.p, m + 1, s);
  exclusive_sum(rflag.p, rpos.p, m + 1, s);
  uint64_t mk = 0;
  BFLY_CUDA(cudaMemcpyAsync(&mk, lpos.p + m, 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  *kept = mk;
  if (mk == 0) return;  // sparsify.cpp:22: nothing retained -> 0
  bfly_graph sub;
  sub.device = g->device;
  sub.stream = s;
  sub.L = g->L;
  sub.R = g->R;
  sub.m = mk;
  sub.loff.alloc(uint64_t{g->L} + 1, s);
  sub.roff.alloc(uint64_t{g->R} + 1, s);
  sub.ladj.alloc(mk, s);
  sub.radj.alloc(mk, s);
  sub.reid.alloc(mk, s);
  launch("spar_new_off", k_new_off, grid_for(uint64_t{g->L} + 1, 256), 256, 0, s, g->loff.p, g->L,
         lpos.p, sub.loff.p);
  launch("spar_new_off", k_new_off, grid_for(uint64_t{g->R} + 1, 256), 256, 0, s, g->roff.p, g->R,
         rpos.p, sub.roff.p);
  launch("spar_compact_left", k_compact_left, grid_for(m, 256), 256, 0, s, g->ladj.p, flag.p,
         lpos.p, m, sub.ladj.p);
  launch("spar_compact_right", k_compact_right, grid_for(m, 256), 256, 0, s, g->radj.p, g->reid.p,
         rflag.p, rpos.p, lpos.p, m, sub.radj.p, sub.reid.p);
  flag.release();
  rflag.release();
  lpos.release();
  rpos.release();
  *count = exact_count_device(&sub);
  g->last_wedges = sub.last_wedges;
  for (int q = 0; q < 4; ++q) {
    g->bucket_starts[q] = sub.bucket_starts[q];
    g->bucket_wedges[q] = sub.bucket_wedges[q];
    g->bucket_entries[q] = sub.bucket_entries[q];
  }
  BFLY_CUDA(cudaStreamSynchronize(s));
}

}  // namespace bflyd
