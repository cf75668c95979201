// segsort.cu -- in-place ascending sort of every row of a row-partitioned u32 array.
//
// Used by the graph build (graph_build.cu) to put each left row of the edge list in right-id
// order once the edges are grouped by left id: rows are independent, so instead of a
// device-wide radix pass over all edges each row is sorted where it fits -- sub-warp bitonic
// networks (<= 32 keys), one warp (<= 256, merge sort in registers), one CTA (<= 8192, radix
// sort in shared memory), and one device-wide sort of (row slot, key) for the few longer rows.
// Rows are classified into per-size lists first (one pass over the row offsets).
#include <algorithm>
#include <cub/block/block_radix_sort.cuh>
#include <cub/warp/warp_merge_sort.cuh>

#include "cubwrap.cuh"
#include "graph.cuh"

namespace bflyd {
namespace {

// size classes: 0 (> 8192), 1 (4096, 8192], 2 (2048, 4096], ..., 13 (1, 2]; rows of <= 1 key
// need no sort
constexpr int kSegClasses = 14;

__device__ __forceinline__ int seg_class(uint32_t len) {
  if (len <= 1) return -1;
  if (len > 8192) return 0;
  // (2^(13-c), 2^(14-c)] -> c
  const int lg = 32 - __clz(len - 1);  // ceil(log2(len)) for len >= 2
  return 14 - lg;
}

// per-class row lists; per 256-row chunk: shared-memory slot counters, one global atomic per
// class present in the chunk
__global__ void __launch_bounds__(256) k_seg_classify(const uint32_t* __restrict__ rs,
                                                      uint32_t rows, uint32_t* __restrict__ lists,
                                                      unsigned long long* __restrict__ cnt) {
  __shared__ unsigned s_cnt[kSegClasses];
  __shared__ unsigned long long s_base[kSegClasses];
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < rows;
       base += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < kSegClasses) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t r = base + threadIdx.x;
    const int c = r < rows ? seg_class(rs[r + 1] - rs[r]) : -1;
    const unsigned my = c >= 0 ? atomicAdd(&s_cnt[c], 1u) : 0u;
    __syncthreads();
    if (threadIdx.x < kSegClasses && s_cnt[threadIdx.x])
      s_base[threadIdx.x] = atomicAdd(&cnt[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
    __syncthreads();
    if (c >= 0) lists[(uint64_t)c * rows + s_base[c] + my] = static_cast<uint32_t>(r);
    __syncthreads();
  }
}

template <int G>
__device__ __forceinline__ void group_bitonic_keys(uint32_t& key, unsigned j) {
#pragma unroll
  for (int k = 2; k <= G; k <<= 1)
#pragma unroll
    for (int s = k >> 1; s > 0; s >>= 1) {
      const uint32_t ok = __shfl_xor_sync(0xffffffffu, key, s);
      const bool up = (j & k) == 0;
      const bool lower = (j & s) == 0;
      key = (lower == up) ? min(key, ok) : max(key, ok);
    }
}

// rows of <= G keys, 32/G rows per warp
// Every kernel also counts adjacent equal keys inside the sorted rows into *dups (duplicate
// edges of the caller), one atomic per warp or CTA that found any.
__device__ __forceinline__ void count_dups_warp(unsigned mine, unsigned long long* dups) {
  const unsigned d = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && d) atomicAdd(dups, (unsigned long long)d);
}

template <int G>
__global__ void __launch_bounds__(256) k_seg_small(const uint32_t* __restrict__ list, uint64_t n,
                                                   const uint32_t* __restrict__ rs,
                                                   uint32_t* __restrict__ keys,
                                                   unsigned long long* __restrict__ dups) {
  constexpr unsigned R = 32 / G;
  const unsigned lane = threadIdx.x & 31, j = lane % G;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = gw * R; base < n; base += nw * R) {
    const uint64_t t = base + lane / G;
    uint32_t a = 0, len = 0;
    if (t < n) {
      const uint32_t r = list[t];
      a = rs[r];
      len = rs[r + 1] - a;
    }
    uint32_t key = j < len ? keys[a + j] : 0xFFFFFFFFu;
    group_bitonic_keys<G>(key, j);
    if (j < len) keys[a + j] = key;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
    count_dups_warp(j > 0 && j < len && prev == key ? 1u : 0u, dups);
  }
}

struct LessKey {
  __device__ __forceinline__ bool operator()(uint32_t a, uint32_t b) const { return a < b; }
};

template <int ITEMS>
__global__ void __launch_bounds__(256) k_seg_warp(const uint32_t* __restrict__ list, uint64_t n,
                                                  const uint32_t* __restrict__ rs,
                                                  uint32_t* __restrict__ keys,
                                                  unsigned long long* __restrict__ dups) {
  using WS = cub::WarpMergeSort<uint32_t, ITEMS, 32>;
  __shared__ typename WS::TempStorage ts[8];
  const unsigned lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = gw; t < n; t += nw) {
    const uint32_t r = list[t];
    const uint32_t a = rs[r], len = rs[r + 1] - a;
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = i * 32 + lane;
      k[i] = idx < len ? keys[a + idx] : 0xFFFFFFFFu;
    }
    WS(ts[wl]).Sort(k, LessKey());
    uint32_t prev = __shfl_up_sync(0xffffffffu, k[ITEMS - 1], 1);  // blocked: lane t, items t*ITEMS..
    unsigned nd = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t pos = lane * ITEMS + i;
      if (pos < len) keys[a + pos] = k[i];
      nd += (pos > 0 && pos < len && prev == k[i]);
      prev = k[i];
    }
    count_dups_warp(nd, dups);
    __syncwarp();
  }
}

// 2^kbits > every key: the padding key sorts last on the low kbits bits
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_seg_block(const uint32_t* __restrict__ list, uint64_t n,
                                                     const uint32_t* __restrict__ rs,
                                                     uint32_t* __restrict__ keys, int kbits,
                                                     unsigned long long* __restrict__ dups) {
  using BRS = cub::BlockRadixSort<uint32_t, BLOCK, ITEMS>;
  __shared__ typename BRS::TempStorage ts;
  for (uint64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const uint32_t r = list[t];
    const uint32_t a = rs[r], len = rs[r + 1] - a;
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = i * BLOCK + threadIdx.x;
      k[i] = idx < len ? keys[a + idx] : 0xFFFFFFFFu;
    }
    BRS(ts).SortBlockedToStriped(k, 0, kbits);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t pos = i * BLOCK + threadIdx.x;
      if (pos < len) keys[a + pos] = k[i];
    }
    __syncthreads();  // the row is written: compare each key with its predecessor
    unsigned nd = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t pos = i * BLOCK + threadIdx.x;
      nd += (pos > 0 && pos < len && keys[a + pos - 1] == k[i]);
    }
    count_dups_warp(nd, dups);
  }
}

// lengths of the big rows (entry nb: 0, so the exclusive sum's last element is the total)
__global__ void k_seg_big_len(const uint32_t* __restrict__ big, uint32_t nb,
                              const uint32_t* __restrict__ rs, uint32_t* __restrict__ len) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x)
    len[b] = b < nb ? rs[big[b] + 1] - rs[big[b]] : 0u;
}

// long rows: buffer position q of big row b (its keys at [bst[b], bst[b+1])) gets
// (b << kbits) | key; after one device sort the buffer is every big row, sorted, in b order
template <typename K>
__global__ void k_seg_big_fill(const uint32_t* __restrict__ big, const uint32_t* __restrict__ bst,
                               uint32_t nb, const uint32_t* __restrict__ rs,
                               const uint32_t* __restrict__ keys, int kbits, K* __restrict__ out) {
  const uint64_t nq = bst[nb];
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nb;  // last b with bst[b] <= q
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(bst + mid) <= q) lo = mid;
      else hi = mid;
    }
    out[q] = (static_cast<K>(lo) << kbits) | keys[rs[big[lo]] + (q - bst[lo])];
  }
}

template <typename K>
__global__ void k_seg_big_back(const K* __restrict__ sorted, const uint32_t* __restrict__ big,
                               const uint32_t* __restrict__ bst, uint32_t nb,
                               const uint32_t* __restrict__ rs, int kbits,
                               uint32_t* __restrict__ keys, unsigned long long* __restrict__ dups) {
  const uint64_t nq = bst[nb];
  const K mask = (K(1) << kbits) - 1;
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; base < nq;
       base += (uint64_t)gridDim.x * blockDim.x) {  // warp-uniform trip count
    const uint64_t q = base + lane;
    bool dup = false;
    if (q < nq) {
      const K v = sorted[q];
      const uint32_t b = static_cast<uint32_t>(v >> kbits);
      keys[rs[big[b]] + (q - bst[b])] = static_cast<uint32_t>(v & mask);
      dup = q > 0 && sorted[q - 1] == v;  // (b, key): equal values are equal keys of one row
    }
    count_dups_warp(dup ? 1u : 0u, dups);
  }
}

}  // namespace

// keys[rs[r] .. rs[r+1]) sorted ascending for every row r < rows; every key < 2^kbits
void seg_sort_rows(uint32_t* keys, const uint32_t* rs, uint32_t rows, int kbits, cudaStream_t s,
                   unsigned long long* dups) {
  if (rows == 0) return;
  kbits = std::max(1, std::min(kbits, 32));
  DBuf<uint32_t> lists(uint64_t{kSegClasses} * rows, s);
  DBuf<unsigned long long> cnt(kSegClasses, s);
  cnt.zero();
  launch("seg_classify", k_seg_classify, grid_for(rows, 256), 256, 0, s, rs, rows, lists.p, cnt.p);
  unsigned long long c[kSegClasses];
  read_back(s, {{c, cnt.p, sizeof(c)}});
  auto lst = [&](int cls) { return lists.p + uint64_t{static_cast<uint32_t>(cls)} * rows; };
  if (c[0]) {  // rows of > 8192 keys
    const uint32_t nb = static_cast<uint32_t>(c[0]);
    DBuf<uint32_t> blen(nb + 1, s), dbst(nb + 1, s);
    launch("seg_big_len", k_seg_big_len, grid_for(nb + 1, 256), 256, 0, s, lst(0), nb, rs, blen.p);
    exclusive_sum(blen.p, dbst.p, nb + 1, s);
    uint32_t nq32 = 0;
    read_back(s, {{&nq32, dbst.p + nb, 4}});
    const uint64_t nq = nq32;
    const int bits = kbits + std::max(1, bits_for(nb - 1));
    auto go = [&](auto zero) {
      using K = decltype(zero);
      DBuf<K> k0(nq, s), k1(nq, s);
      launch("seg_big_fill", k_seg_big_fill<K>, grid_for(nq, 256, 148u * 16u), 256, 0, s, lst(0),
             dbst.p, nb, rs, keys, kbits, k0.p);
      if (!sort_keys_db(k0.p, k1.p, nq, 0, bits, s, "sort_seg_big")) std::swap(k0, k1);
      launch("seg_big_back", k_seg_big_back<K>, grid_for(nq, 256, 148u * 16u), 256, 0, s, k1.p,
             lst(0), dbst.p, nb, rs, kbits, keys, dups);
    };
    if (bits <= 32) go(uint32_t{0});
    else go(uint64_t{0});
  }
  auto block = [&](auto kern, int blk, int cls) {
    if (c[cls])
      launch("seg_block", kern, static_cast<unsigned>(std::min<unsigned long long>(c[cls], 148u * 8u)),
             blk, 0, s, lst(cls), (uint64_t)c[cls], rs, keys, kbits, dups);
  };
  block(k_seg_block<512, 16>, 512, 1);  // (4096, 8192]
  block(k_seg_block<256, 16>, 256, 2);  // (2048, 4096]
  block(k_seg_block<256, 8>, 256, 3);   // (1024, 2048]
  block(k_seg_block<256, 4>, 256, 4);   // (512, 1024]
  block(k_seg_block<256, 2>, 256, 5);   // (256, 512]
  auto warp = [&](auto kern, int cls) {
    if (c[cls])
      launch("seg_warp", kern, grid_for(c[cls] * 32, 256, 148u * 16u), 256, 0, s, lst(cls),
             (uint64_t)c[cls], rs, keys, dups);
  };
  warp(k_seg_warp<8>, 6);  // (128, 256]
  warp(k_seg_warp<4>, 7);  // (64, 128]
  warp(k_seg_warp<2>, 8);  // (32, 64]
  auto small = [&](auto kern, int G, int cls) {
    if (c[cls])
      launch("seg_small", kern, grid_for(c[cls] * G, 256, 148u * 16u), 256, 0, s, lst(cls),
             (uint64_t)c[cls], rs, keys, dups);
  };
  small(k_seg_small<32>, 32, 9);   // (16, 32]
  small(k_seg_small<16>, 16, 10);  // (8, 16]
  small(k_seg_small<8>, 8, 11);    // (4, 8]
  small(k_seg_small<4>, 4, 12);    // (2, 4]
  small(k_seg_small<2>, 2, 13);    // (1, 2]
}

}  // namespace bflyd
