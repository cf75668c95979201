// Microbenchmark: throughput of shared-memory and L2 (global) atomics on B200.
// Decides the counting-table design of the wedge-aggregation kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void smem_kernel(int iters, uint32_t mask, unsigned long long* out) {
  extern __shared__ uint32_t tab[];
  for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t a = (s >> 8) & mask;
    if (MODE == 0) acc += atomicAdd(&tab[a], 1u);
    else if (MODE == 1) atomicAdd(&tab[a], 1u);
    else if (MODE == 2) acc += atomicCAS(&tab[a], 0u, s);
    else if (MODE == 3) { uint32_t v = tab[a]; tab[a] = v + 1; acc += v; }
  }
  if (acc == 0xdeadbeef) out[0] = acc;
  __syncthreads();
  if (MODE == 1 && threadIdx.x == 0) out[1] = tab[0];
}

template <int MODE>
__global__ void gmem_kernel(uint32_t* tab, int iters, uint32_t mask, unsigned long long* out) {
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t a = hsh(s) & mask;
    if (MODE == 0) acc += atomicAdd(&tab[a], 1u);
    else if (MODE == 1) atomicAdd(&tab[a], 1u);
    else if (MODE == 2) { tab[a] = 0; }
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

__global__ void read_kernel(const int4* __restrict__ p, size_t n, unsigned long long* out) {
  int4 acc = make_int4(0,0,0,0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(p + i); acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345) out[0] = 1;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s SMs=%d smemPerBlockOptin=%zu L2=%d clock=%d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.l2CacheSize, p.clockRate);
  unsigned long long* out; cudaMalloc(&out, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  for (int tbits : {10, 12, 14, 15}) {
    uint32_t mask = (1u << tbits) - 1; size_t sm = (mask + 1) * 4;
    auto run = [&](auto kern, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      for (int threads : {256, 1024}) {
        int blocks = p.multiProcessorCount * (2048 / threads);
        kern<<<blocks, threads, sm>>>(iters, mask, out);
        cudaEventRecord(a);
        kern<<<blocks, threads, sm>>>(iters, mask, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters;
        printf("smem %-10s table=%6zuB thr=%4d : %.3f Gop/s  (%.2f op/clk/SM)  err=%s\n", name, sm, threads,
               ops / ms / 1e6, ops / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3),
               cudaGetErrorString(cudaGetLastError()));
      }
    };
    run(smem_kernel<0>, "add_ret");
    run(smem_kernel<1>, "red");
    run(smem_kernel<2>, "cas");
    run(smem_kernel<3>, "ld_st");
  }
  uint32_t* g; size_t gbytes = 1ull << 30; cudaMalloc(&g, gbytes); cudaMemset(g, 0, gbytes);
  for (int tbits : {18, 21, 23, 25, 28}) {
    uint32_t mask = (1u << tbits) - 1;
    auto run = [&](auto kern, const char* name) {
      for (int occ : {4, 16, 32}) {
        int threads = 256; int blocks = p.multiProcessorCount * occ;
        int it = 1024;
        kern<<<blocks, threads>>>(g, it, mask, out);
        cudaEventRecord(a);
        kern<<<blocks, threads>>>(g, it, mask, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * it;
        printf("gmem %-8s table=%9zuB blocks=%5d : %.3f Gop/s err=%s\n", name, (size_t)(mask + 1) * 4, blocks,
               ops / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    };
    run(gmem_kernel<0>, "add_ret");
    run(gmem_kernel<1>, "red");
    run(gmem_kernel<2>, "store");
  }
  size_t n = gbytes / 16;
  read_kernel<<<p.multiProcessorCount * 8, 512>>>((const int4*)g, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) read_kernel<<<p.multiProcessorCount * 8, 512>>>((const int4*)g, n, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("HBM read: %.1f GB/s\n", 5.0 * gbytes / ms / 1e6);
  return 0;
}
