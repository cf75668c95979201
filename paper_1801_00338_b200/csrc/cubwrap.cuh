// cubwrap.cuh -- thin stream-ordered wrappers over the CUB device primitives used for
// graph build (radix sort / scan / select). CUB is header-only and compiled into this
// library for sm_100a; every call is bracketed by the profiling scope.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"
#include "radix.cuh"

// BFLY_HAND_SORT=1: every device-wide sort of the build is the hand-written radix.cuh. The
// default (0) keeps CUB's onesweep, which measured faster on config 2 (step 21.1-21.4 ms
// against 23.1 ms with the hand-written sort: DESIGN.md section 4).
#ifndef BFLY_HAND_SORT
#define BFLY_HAND_SORT 0
#endif

namespace bflyd {

template <typename F>
inline void cub_call(const char* name, cudaStream_t s, F&& f) {
  ProfScope p(name, s);
  size_t bytes = 0;
  BFLY_CUDA(f(static_cast<void*>(nullptr), bytes));
  DBuf<unsigned char> tmp(bytes ? bytes : 1, s);
  BFLY_CUDA(f(static_cast<void*>(tmp.p), bytes));
}

template <typename K, typename V>
inline void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit,
                       int end_bit, cudaStream_t s, const char* name = "cub_sort_pairs") {
  if (n == 0) return;
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  if (n >= (1ull << 31)) fail(kArgument, "sort larger than 2^31-1 items");
#if BFLY_HAND_SORT
  radix::sort_pairs(kin, kout, vin, vout, n, begin_bit, end_bit, s, name);
  return;
#endif
  const int ni = static_cast<int>(n);  // 32-bit offsets: CUB's fastest onesweep path
  cub_call(name, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, vin, vout, ni, begin_bit, end_bit, s);
  });
}

template <typename K>
inline void sort_keys(const K* kin, K* kout, uint64_t n, int begin_bit, int end_bit,
                      cudaStream_t s, const char* name = "cub_sort_keys") {
  if (n == 0) return;
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  if (n >= (1ull << 31)) fail(kArgument, "sort larger than 2^31-1 items");
  const int ni = static_cast<int>(n);
  cub_call(name, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, kin, kout, ni, begin_bit, end_bit, s);
  });
}

// Ping-pong sorts over two caller-owned buffers (CUB may overwrite the input): no temp copy
// of the data (the const-input API allocates ~8 B per pair of scratch). Returns true when
// the sorted data ended up in the alternate buffers (kalt / valt), false when it is back in
// k / v.
template <typename K, typename V>
inline bool sort_pairs_db(K* k, K* kalt, V* v, V* valt, uint64_t n, int begin_bit, int end_bit,
                          cudaStream_t s, const char* name = "cub_sort_pairs") {
  if (n == 0) return false;
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  if (n >= (1ull << 31)) fail(kArgument, "sort larger than 2^31-1 items");
#if BFLY_HAND_SORT
  return radix::sort_pairs_db(k, kalt, v, valt, n, begin_bit, end_bit, s, name);
#endif
  const int ni = static_cast<int>(n);
  bool alt = false;
  cub_call(name, s, [&](void* t, size_t& b) {
    cub::DoubleBuffer<K> dk(k, kalt);
    cub::DoubleBuffer<V> dv(v, valt);
    const cudaError_t e = cub::DeviceRadixSort::SortPairs(t, b, dk, dv, ni, begin_bit, end_bit, s);
    if (t) alt = dk.Current() == kalt;
    return e;
  });
  return alt;
}

template <typename K>
inline bool sort_keys_db(K* k, K* kalt, uint64_t n, int begin_bit, int end_bit, cudaStream_t s,
                         const char* name = "cub_sort_keys") {
  if (n == 0) return false;
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  if (n >= (1ull << 31)) fail(kArgument, "sort larger than 2^31-1 items");
#if BFLY_HAND_SORT
  return radix::sort_keys_db(k, kalt, n, begin_bit, end_bit, s, name);
#endif
  const int ni = static_cast<int>(n);
  bool alt = false;
  cub_call(name, s, [&](void* t, size_t& b) {
    cub::DoubleBuffer<K> dk(k, kalt);
    const cudaError_t e = cub::DeviceRadixSort::SortKeys(t, b, dk, ni, begin_bit, end_bit, s);
    if (t) alt = dk.Current() == kalt;
    return e;
  });
  return alt;
}

template <typename T, typename O>
inline void exclusive_sum(const T* in, O* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  cub_call("cub_exclusive_sum", s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, in, out, n, s);
  });
}

template <typename T>
inline void inclusive_max(const T* in, T* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  cub_call("cub_inclusive_max", s, [&](void* t, size_t& b) {
    return cub::DeviceScan::InclusiveScan(t, b, in, out, cub::Max(), n, s);
  });
}

template <typename T>
inline void reduce_max(const T* in, T* out, uint64_t n, cudaStream_t s) {
  cub_call("cub_reduce_max", s, [&](void* t, size_t& b) {
    return cub::DeviceReduce::Max(t, b, in, out, n, s);
  });
}

}  // namespace bflyd
