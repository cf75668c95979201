// CUB onesweep policy sweep for the build's 50M-pair (u32 key, u32 value) sorts on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sortbench sortbench.cu
#include <cstdio>
#include <cub/device/device_radix_sort.cuh>
#include <vector>

using K = uint32_t;
using V = uint32_t;

template <int THREADS, int ITEMS, int BITS>
struct Hub {
  using B = cub::detail::radix::policy_hub<K, V, int>::Policy1000;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = BITS;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, K, BITS>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, BITS>;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, K, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT,
                                          BITS>;
    using ScanPolicy = typename B::ScanPolicy;
    using DownsweepPolicy = typename B::DownsweepPolicy;
    using AltDownsweepPolicy = typename B::AltDownsweepPolicy;
    using UpsweepPolicy = typename B::UpsweepPolicy;
    using AltUpsweepPolicy = typename B::AltUpsweepPolicy;
    using SingleTilePolicy = typename B::SingleTilePolicy;
    using SegmentedPolicy = typename B::SegmentedPolicy;
    using AltSegmentedPolicy = typename B::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy1000;
};

__global__ void fill(K* k, V* v, int n, int bits, unsigned seed);

template <class H>
float run(K* k0, K* k1, V* v0, V* v1, int n, int bits, const char* name) {
  cub::DoubleBuffer<K> dk(k0, k1);
  cub::DoubleBuffer<V> dv(v0, v1);
  size_t bytes = 0;
  using D = cub::DispatchRadixSort<false, K, V, int, H>;
  D::Dispatch(nullptr, bytes, dk, dv, n, 0, bits, true, 0);
  void* tmp;
  cudaMalloc(&tmp, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    fill<<<148 * 8, 256>>>(k0, v0, n, bits, 12345 + it);  // unsorted input every time
    cub::DoubleBuffer<K> k(k0, k1);
    cub::DoubleBuffer<V> v(v0, v1);
    cudaEventRecord(a);
    D::Dispatch(tmp, bytes, k, v, n, 0, bits, true, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  printf("%-28s bits=%d  %.3f ms\n", name, bits, best);
  cudaFree(tmp);
  return best;
}

__global__ void fill(K* k, V* v, int n, int bits, unsigned seed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned x = i * 2654435761u ^ seed;
    x ^= x >> 15; x *= 0x2c1b3c6d; x ^= x >> 12; x *= 0x297a2d39; x ^= x >> 15;
    k[i] = x & ((1u << bits) - 1);
    v[i] = i;
  }
}

float run_api(K* k0, K* k1, V* v0, V* v1, int n, int bits, const char* name) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, v0, v1, n, 0, bits);
  void* tmp;
  cudaMalloc(&tmp, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    fill<<<148 * 8, 256>>>(k0, v0, n, bits, 12345 + it);
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, v1, n, 0, bits);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  printf("%-28s bits=%d  %.3f ms (temp %zu MB)\n", name, bits, best, bytes >> 20);
  cudaFree(tmp);
  return best;
}

// power-law keys: key = floor(N * u^3) style skew (many repeats of small keys)
__global__ void fill_skew(K* k, V* v, int n, int bits, unsigned seed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned x = i * 2654435761u ^ seed;
    x ^= x >> 15; x *= 0x2c1b3c6d; x ^= x >> 12; x *= 0x297a2d39; x ^= x >> 15;
    const double u = (x & 0xFFFFFF) / 16777216.0;
    k[i] = static_cast<K>(((1u << bits) - 1) * u * u * u * u);
    v[i] = i;
  }
}

// the library's pattern: every buffer and the temp storage come from the stream-ordered pool
// per call (pool keeps its memory: release threshold = max)
float run_pool(int n, int bits, const char* name, bool pool_data = true, bool pool_tmp = true) {
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    K *k0, *k1;
    V *v0, *v1;
    if (pool_data) {
      cudaMallocAsync(&k0, n * 4ull, s); cudaMallocAsync(&k1, n * 4ull, s);
      cudaMallocAsync(&v0, n * 4ull, s); cudaMallocAsync(&v1, n * 4ull, s);
    } else {
      cudaMalloc(&k0, n * 4ull); cudaMalloc(&k1, n * 4ull);
      cudaMalloc(&v0, n * 4ull); cudaMalloc(&v1, n * 4ull);
    }
    fill<<<148 * 8, 256, 0, s>>>(k0, v0, n, bits, 777 + it);
    cudaEventRecord(a, s);
    size_t bytes = 0;
    cub::DoubleBuffer<K> dk(k0, k1);
    cub::DoubleBuffer<V> dv(v0, v1);
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, n, 0, bits, s);
    void* tmp;
    if (pool_tmp) cudaMallocAsync(&tmp, bytes, s);
    else cudaMalloc(&tmp, bytes);
    cub::DeviceRadixSort::SortPairs(tmp, bytes, dk, dv, n, 0, bits, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    if (pool_tmp) cudaFreeAsync(tmp, s);
    else cudaFree(tmp);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
    if (pool_data) {
      cudaFreeAsync(k0, s); cudaFreeAsync(k1, s); cudaFreeAsync(v0, s); cudaFreeAsync(v1, s);
    } else {
      cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1);
    }
  }
  printf("%-28s bits=%d  %.3f ms\n", name, bits, best);
  return best;
}

int main() {
  run_pool(50000000, 21, "pool data + pool tmp", true, true);
  run_pool(50000000, 21, "pool data + malloc tmp", true, false);
  run_pool(50000000, 21, "malloc data + pool tmp", false, true);
  run_pool(50000000, 21, "malloc data + malloc tmp", false, false);
  return 0;
  const int n = 50000000;
  K *k0, *k1;
  V *v0, *v1;
  cudaMalloc(&k0, n * 4ull); cudaMalloc(&k1, n * 4ull);
  cudaMalloc(&v0, n * 4ull); cudaMalloc(&v1, n * 4ull);
  {
    const int bits = 21;
    fill<<<148 * 8, 256>>>(k0, v0, n, bits, 12345);
    run_api(k0, k1, v0, v1, n, bits, "SortPairs API uniform");


  }
  for (int bits : {21, 23}) {
    auto refill = [&] { fill<<<148 * 8, 256>>>(k0, v0, n, bits, 12345); };
    refill(); run<cub::detail::radix::policy_hub<K, V, int>>(k0, k1, v0, v1, n, bits, "default");
    refill(); run<Hub<384, 23, 8>>(k0, k1, v0, v1, n, bits, "384x23 b8");
    refill(); run<Hub<256, 23, 8>>(k0, k1, v0, v1, n, bits, "256x23 b8");
    refill(); run<Hub<512, 16, 8>>(k0, k1, v0, v1, n, bits, "512x16 b8");
    refill(); run<Hub<384, 30, 8>>(k0, k1, v0, v1, n, bits, "384x30 b8");
    refill(); run<Hub<384, 23, 7>>(k0, k1, v0, v1, n, bits, "384x23 b7");
    refill(); run<Hub<256, 16, 6>>(k0, k1, v0, v1, n, bits, "256x16 b6");
    refill(); run<Hub<512, 23, 8>>(k0, k1, v0, v1, n, bits, "512x23 b8");
    refill(); run<Hub<384, 16, 8>>(k0, k1, v0, v1, n, bits, "384x16 b8");
    refill(); run<Hub<256, 30, 8>>(k0, k1, v0, v1, n, bits, "256x30 b8");
    refill(); run<Hub<384, 23, 6>>(k0, k1, v0, v1, n, bits, "384x23 b6");
    refill(); run<Hub<256, 40, 8>>(k0, k1, v0, v1, n, bits, "256x40 b8");
  }
  return 0;
}
