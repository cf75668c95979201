// Microbenchmark: distributed-shared-memory (cluster) atomics and smem hash
// insert-or-increment throughput on B200.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void dsmem_kernel(int iters, uint32_t mask, unsigned long long* out) {
  extern __shared__ uint32_t tab[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) tab[i] = 0;
  cl.sync();
  unsigned nr = cl.num_blocks();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t a = (s >> 8) & mask;
    unsigned r = (s >> 2) % nr;
    uint32_t* t = cl.map_shared_rank(tab, r);
    if (MODE == 0) acc += atomicAdd(t + a, 1u);
    else atomicAdd(t + a, 1u);
  }
  if (acc == 0xdeadbeef) out[0] = acc;
  cl.sync();
}

// insert-or-increment into an open-addressing smem table of (key,count)
__global__ void hash_kernel(int iters, uint32_t mask, uint32_t keyspace, unsigned long long* out) {
  extern __shared__ uint32_t sm[];
  uint32_t* keys = sm;
  uint32_t* cnt = sm + mask + 1;
  for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) { keys[i] = 0xffffffffu; cnt[i] = 0; }
  __syncthreads();
  uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t w = (s >> 4) % keyspace;
    uint32_t h = (w * 0x9E3779B1u) & mask;
    while (true) {
      uint32_t k = keys[h];
      if (k == w) { acc += atomicAdd(&cnt[h], 1u); break; }
      if (k == 0xffffffffu) {
        uint32_t prev = atomicCAS(&keys[h], 0xffffffffu, w);
        if (prev == 0xffffffffu || prev == w) { acc += atomicAdd(&cnt[h], 1u); break; }
      }
      h = (h + 1) & mask;
    }
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  unsigned long long* out; cudaMalloc(&out, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint32_t mask = (1u << 15) - 1; size_t sm = (mask + 1) * 4;
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int mode = 0; mode < 2; ++mode) {
      auto kern = mode == 0 ? dsmem_kernel<0> : dsmem_kernel<1>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      int threads = 1024;
      cfg.gridDim = dim3(p.multiProcessorCount / cs * cs); cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      int iters = 2048;
      cudaLaunchKernelEx(&cfg, kern, iters, mask, out);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, kern, iters, mask, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = (double)cfg.gridDim.x * threads * iters;
      printf("dsmem cluster=%2d %s grid=%d : %.1f Gop/s (%.2f op/clk/SM) err=%s\n", cs, mode ? "red    " : "add_ret",
             cfg.gridDim.x, ops / ms / 1e6, ops / (ms * 1e-3) / cfg.gridDim.x / 1.965e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int tb : {10, 13, 14}) {
    uint32_t m2 = (1u << tb) - 1; size_t sm2 = (m2 + 1) * 8;
    cudaFuncSetAttribute(hash_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    for (uint32_t ks : {m2 / 8, m2 / 2, (m2 * 3) / 4}) {
      int threads = 512, blocks = p.multiProcessorCount * (sm2 > 100000 ? 1 : 2), iters = 2048;
      hash_kernel<<<blocks, threads, sm2>>>(iters, m2, ks, out);
      cudaEventRecord(a);
      hash_kernel<<<blocks, threads, sm2>>>(iters, m2, ks, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = (double)blocks * threads * iters;
      printf("hash slots=%6u keys=%6u : %.1f Gop/s (%.2f op/clk/SM) err=%s\n", m2 + 1, ks, ops / ms / 1e6,
             ops / (ms * 1e-3) / p.multiProcessorCount / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
