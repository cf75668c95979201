// common.cuh -- runtime plumbing shared by every translation unit of libbfly_b200.so:
// status/exception mapping for the C-ABI, stream-ordered device buffers, the launch
// wrapper that counts launches and (optionally) times each kernel with CUDA events.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

namespace bflyd {

// Status codes of include/bfly_b200.h (map 1:1 onto the reference's exception types).
enum : int {
  kOk = 0, kArgument = 1, kEmpty = 2, kOverflow = 3, kNoWedges = 4, kInternal = 5, kParse = 6
};

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }

#define BFLY_CUDA(x)                                                                     \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      ::bflyd::fail(::bflyd::kInternal, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---- profiling / launch accounting (profile.cu) ------------------------------------
// BFLY_TRACE=1: host-side phase timestamps on stderr (diagnosing host gaps between kernels)
void trace_mark(const char* what);
void prof_record(const char* name, cudaEvent_t a, cudaEvent_t b);
bool prof_enabled();
void count_launch();
cudaEvent_t prof_event();

struct ProfScope {
  const char* name;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(const char* n, cudaStream_t st) : name(n), s(st) {
    if (prof_enabled()) {
      a = prof_event();
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, s);
      prof_record(name, a, b);
    }
  }
};

// Launch a hand-written kernel: counted, optionally timed, error-checked.
template <typename K, typename... Args>
inline void launch(const char* name, K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  ProfScope p(name, s);
  kernel<<<grid, block, smem, s>>>(args...);
  BFLY_CUDA(cudaGetLastError());
  count_launch();
}

// ---- stream-ordered device buffer ---------------------------------------------------
// Every engine allocation comes from a PRIVATE per-device pool (abi.cu: engine_pool), never
// the device's default pool, so the host application's cudaMallocAsync users keep their own
// pool settings; bfly_trim_pool() hands cached memory back to the driver.
cudaMemPool_t engine_pool();

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count)
      BFLY_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), count * sizeof(T),
                                        engine_pool(), s));
  }
  // grow-only reallocation (contents not preserved)
  void ensure(size_t count, cudaStream_t st) {
    if (count > n || p == nullptr) alloc(count ? count : 1, st);
  }
  void zero() {
    if (n) BFLY_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// Small device->host reads on the step path (counts, sizes, totals): staged through a
// thread-local pinned buffer so the copy is a plain DMA (pageable destinations cost a staging
// pass on every read), all issued before one stream synchronisation.
struct ReadBack {
  struct Item {
    void* dst;
    const void* src;
    size_t bytes;
  };
  static constexpr size_t kCap = 1 << 20;
  static unsigned char* buf() {
    static thread_local unsigned char* b = [] {
      void* p = nullptr;
      if (cudaMallocHost(&p, kCap) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
      }
      return static_cast<unsigned char*>(p);
    }();
    return b;
  }
  // copies every item (total <= kCap bytes) and synchronises the stream once
  static void run(cudaStream_t s, std::initializer_list<Item> items) {
    unsigned char* b = buf();
    size_t off = 0;
    for (const Item& it : items) {
      if (b && off + it.bytes <= kCap) {
        BFLY_CUDA(cudaMemcpyAsync(b + off, it.src, it.bytes, cudaMemcpyDeviceToHost, s));
        off += (it.bytes + 15) & ~size_t{15};
      } else {
        BFLY_CUDA(cudaMemcpyAsync(it.dst, it.src, it.bytes, cudaMemcpyDeviceToHost, s));
      }
    }
    BFLY_CUDA(cudaStreamSynchronize(s));
    off = 0;
    for (const Item& it : items) {
      if (b && off + it.bytes <= kCap) {
        std::memcpy(it.dst, b + off, it.bytes);
        off += (it.bytes + 15) & ~size_t{15};
      }
    }
  }
};
inline void read_back(cudaStream_t s, std::initializer_list<ReadBack::Item> items) {
  ReadBack::run(s, items);
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
  uint64_t g = (n + block - 1) / block;
  if (g > cap) g = cap;
  return g ? static_cast<unsigned>(g) : 1u;
}

inline int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

}  // namespace bflyd
