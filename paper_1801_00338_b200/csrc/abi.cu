// abi.cu -- extern "C" entry points of libbfly_b200.so (include/bfly_b200.h).
// Each entry point converts internal Failure exceptions into the status codes that the
// C++ facade maps back onto the reference's exception hierarchy (errors.hpp:10-58).
#include <atomic>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "graph.cuh"
#include "local.cuh"

namespace bflyd {

// The engine's private stream-ordered pool on the current device (created on first use).
// Builds allocate and free GBs per call; returning that memory to the driver at every
// synchronisation costs milliseconds, so this pool keeps what it has (release threshold =
// max) until bfly_trim_pool(). The device's default pool is left untouched.
cudaMemPool_t engine_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  static thread_local int last_dev = -1;
  static thread_local cudaMemPool_t last_pool = nullptr;
  int dev = 0;
  BFLY_CUDA(cudaGetDevice(&dev));
  if (dev == last_dev && last_pool) return last_pool;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev & 63]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    BFLY_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t thr = ~0ull;
    BFLY_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    pools[dev & 63] = pool;
  }
  last_dev = dev;
  last_pool = pools[dev & 63];
  return last_pool;
}

thread_local std::string t_err;

void set_err(const std::string& s) { t_err = s; }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Failure& e) {
    set_err(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_err("host allocation failed");
    return kInternal;
  } catch (const std::exception& e) {
    set_err(e.what());
    return kInternal;
  }
}

namespace {

void require_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  static thread_local int checked_dev = -1;
  if (e == cudaSuccess && checked_dev == dev) return;  // validated once per thread/device
  int n = 0;
  e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    fail(kInternal, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                        "); this engine has no CPU fallback");
  BFLY_CUDA(cudaGetDevice(&dev));
  int major = 0;
  BFLY_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) fail(kInternal, "device is not sm_100 (Blackwell): compute capability " +
                                      std::to_string(major) + ".x");
  checked_dev = dev;
}

thread_local cudaStream_t t_user_stream = nullptr;

bfly_graph* new_graph() {
  require_device();
  auto* g = new bfly_graph();
  BFLY_CUDA(cudaGetDevice(&g->device));
  if (t_user_stream) {
    g->stream = t_user_stream;
    g->owns_stream = false;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete g;
      fail(kInternal, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    g->owns_stream = true;
  }
  g->owner.s = g->stream;
  g->owner.owns = g->owns_stream;
  return g;
}

struct Event {
  cudaEvent_t e = nullptr;
  Event() { BFLY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Event() { cudaEventDestroy(e); }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
};

// process-wide host-to-device copy stream per device
cudaStream_t copy_stream(int device) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  cudaStream_t& cs = streams[device & 63];
  if (!cs) BFLY_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  return cs;
}

template <typename K>
int build_from_host(const K* l, const K* r, uint64_t m_in, bfly_graph** out) {
  return guarded([&] {
    if (!out) fail(kArgument, "null output handle");
    if (m_in && (!l || !r)) fail(kArgument, "null edge arrays");
    trace_mark("build(host): enter");
    bfly_graph* g = new_graph();
    trace_mark("build(host): handle");
    try {
      cudaStream_t s = g->stream;
      DBuf<K> dl(m_in ? m_in : 1, s), dr(m_in ? m_in : 1, s);
      cudaPointerAttributes al{}, ar{};
      const bool pinned = m_in && cudaPointerGetAttributes(&al, l) == cudaSuccess &&
                          cudaPointerGetAttributes(&ar, r) == cudaSuccess &&
                          al.type == cudaMemoryTypeHost && ar.type == cudaMemoryTypeHost;
      cudaGetLastError();
      if (pinned) {
        // page-locked input: copy on a side stream so the left ids are processed while the
        // right ids are still crossing PCIe
        Event ready, left, right;
        cudaStream_t cs = copy_stream(g->device);
        BFLY_CUDA(cudaEventRecord(ready.e, s));  // buffers allocated (stream-ordered)
        BFLY_CUDA(cudaStreamWaitEvent(cs, ready.e, 0));
        BFLY_CUDA(cudaMemcpyAsync(dl.p, l, m_in * sizeof(K), cudaMemcpyHostToDevice, cs));
        BFLY_CUDA(cudaEventRecord(left.e, cs));
        BFLY_CUDA(cudaMemcpyAsync(dr.p, r, m_in * sizeof(K), cudaMemcpyHostToDevice, cs));
        BFLY_CUDA(cudaEventRecord(right.e, cs));
        BFLY_CUDA(cudaStreamWaitEvent(s, left.e, 0));
        build_graph<K>(g, dl.p, dr.p, m_in, right.e);
      } else {
        if (m_in) {
          BFLY_CUDA(cudaMemcpyAsync(dl.p, l, m_in * sizeof(K), cudaMemcpyHostToDevice, s));
          BFLY_CUDA(cudaMemcpyAsync(dr.p, r, m_in * sizeof(K), cudaMemcpyHostToDevice, s));
        }
        build_graph<K>(g, dl.p, dr.p, m_in);
      }
    } catch (...) {
      bfly_graph_free(g);
      throw;
    }
    *out = g;
  });
}

// Process-wide page-locked staging buffer for pair input (grow-only; one build at a time
// uses it, guarded by mu until its copies completed).
struct PinnedStage {
  std::mutex mu;
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      BFLY_CUDA(cudaHostAlloc(&p, need, cudaHostAllocDefault));
      bytes = need;
    }
    return p;
  }
};
PinnedStage& pinned_stage() {
  static PinnedStage st;
  return st;
}

// from_edges(const vector<pair<uint64_t, uint64_t>>&) (graph.hpp:43): interleaved (left,
// right) pairs in pageable host memory. Host threads narrow them to two u32 arrays in a
// page-locked stage, chunk by chunk, and every finished chunk crosses PCIe on the copy
// stream while the threads pack the next ones; ids of 2^32 or more fall back to the u64
// build. The device then runs the u32 build.
int build_from_pairs(const uint64_t* pairs, uint64_t m_in, bfly_graph** out) {
  if (!out) return guarded([] { fail(kArgument, "null output handle"); });
  if (m_in && !pairs) return guarded([] { fail(kArgument, "null edge array"); });
  if (m_in >= (1ull << 31))
    return guarded([] { fail(kArgument, "edge list too long: at most 2^31-1 input edges per graph"); });
  bool wide = false;
  const int st = guarded([&] {
    bfly_graph* g = new_graph();
    try {
      cudaStream_t s = g->stream;
      DBuf<uint32_t> dl(m_in ? m_in : 1, s), dr(m_in ? m_in : 1, s);
      PinnedStage& ps = pinned_stage();
      std::lock_guard<std::mutex> lk(ps.mu);
      uint32_t* hl = static_cast<uint32_t*>(ps.get(std::max<uint64_t>(1, m_in) * 8));
      uint32_t* hr = hl + std::max<uint64_t>(1, m_in);
      cudaStream_t cs = copy_stream(g->device);
      Event ready, done;
      BFLY_CUDA(cudaEventRecord(ready.e, s));  // device buffers allocated (stream-ordered)
      BFLY_CUDA(cudaStreamWaitEvent(cs, ready.e, 0));
      const uint64_t chunk = 1ull << 20;
      const uint64_t nchunks = (m_in + chunk - 1) / chunk;
      const unsigned nt = static_cast<unsigned>(std::min<uint64_t>(
          std::max(1u, std::min(16u, std::thread::hardware_concurrency())), std::max<uint64_t>(1, nchunks)));
      std::atomic<uint64_t> next{0};
      std::atomic<bool> overflow{false};
      std::atomic<int> err{0};
      auto worker = [&] {
        for (uint64_t c; (c = next.fetch_add(1)) < nchunks && !overflow.load();) {
          const uint64_t b = c * chunk, e = std::min(m_in, b + chunk);
          uint64_t hi = 0;
          for (uint64_t i = b; i < e; ++i) {
            const uint64_t a = pairs[2 * i], z = pairs[2 * i + 1];
            hi |= (a | z) >> 32;
            hl[i] = static_cast<uint32_t>(a);
            hr[i] = static_cast<uint32_t>(z);
          }
          if (hi) {
            overflow.store(true);
            break;
          }
          if (cudaMemcpyAsync(dl.p + b, hl + b, (e - b) * 4, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
              cudaMemcpyAsync(dr.p + b, hr + b, (e - b) * 4, cudaMemcpyHostToDevice, cs) != cudaSuccess)
            err.store(1);
        }
      };
      std::vector<std::thread> pool;
      for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
      worker();
      for (auto& t : pool) t.join();
      BFLY_CUDA(cudaEventRecord(done.e, cs));
      BFLY_CUDA(cudaEventSynchronize(done.e));  // the stage is reusable once this returns
      if (err.load()) fail(kInternal, "host-to-device copy of the edge list failed");
      wide = overflow.load();
      if (!wide) {
        BFLY_CUDA(cudaStreamWaitEvent(s, done.e, 0));
        build_graph<uint32_t>(g, dl.p, dr.p, m_in);
      }
      // (dl / dr are released on g's stream here, before g itself may go)
    } catch (...) {
      bfly_graph_free(g);
      throw;
    }
    if (wide) bfly_graph_free(g);
    else *out = g;
  });
  if (st != kOk || !wide) return st;
  // some id needs 64 bits: split into two u64 arrays and run the u64 build
  std::vector<uint64_t> l(m_in), r(m_in);
  for (uint64_t i = 0; i < m_in; ++i) {
    l[i] = pairs[2 * i];
    r[i] = pairs[2 * i + 1];
  }
  return build_from_host<uint64_t>(l.data(), r.data(), m_in, out);
}

}  // namespace
}  // namespace bflyd

using namespace bflyd;

extern "C" {

const char* bfly_last_error(void) { return t_err.c_str(); }
const char* bfly_version(void) { return "bfly_b200 0.1 (sm_100a)"; }

int bfly_device_ok(void) {
  int st = guarded([] { require_device(); });
  return st == kOk ? 1 : 0;
}

int bfly_graph_build_pairs(const uint64_t* pairs, uint64_t m_in, bfly_graph** out) {
  return build_from_pairs(pairs, m_in, out);
}

int bfly_graph_build_u32(const uint32_t* l, const uint32_t* r, uint64_t m_in, bfly_graph** out) {
  return build_from_host<uint32_t>(l, r, m_in, out);
}

int bfly_graph_build_u64(const uint64_t* l, const uint64_t* r, uint64_t m_in, bfly_graph** out) {
  return build_from_host<uint64_t>(l, r, m_in, out);
}

int bfly_graph_build_u32_device(const uint32_t* dl, const uint32_t* dr, uint64_t m_in,
                                bfly_graph** out) {
  return guarded([&] {
    if (!out) fail(kArgument, "null output handle");
    bfly_graph* g = new_graph();
    try {
      build_graph<uint32_t>(g, dl, dr, m_in);
    } catch (...) {
      bfly_graph_free(g);
      throw;
    }
    *out = g;
  });
}

int bfly_graph_load_text(const char* text, uint64_t len, bfly_graph** out, uint64_t* err_line) {
  if (err_line) *err_line = 0;
  return guarded([&] {
    if (!out || (len && !text)) fail(kArgument, "null argument");
    bfly_graph* g = new_graph();
    try {
      DBuf<uint64_t> dl, dr;
      uint64_t line = 0;
      uint64_t m_in = 0;
      try {
        m_in = parse_text_device(g->stream, text, len, dl, dr, &line);
      } catch (...) {
        if (err_line) *err_line = line;
        throw;
      }
      if (m_in == 0) fail(kEmpty, "edge list contains no edges");  // graph.cpp:97
      build_graph<uint64_t>(g, dl.p, dr.p, m_in);
    } catch (...) {
      bfly_graph_free(g);
      throw;
    }
    *out = g;
  });
}

int bfly_graph_serialize(bfly_graph* g, char* buf, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    if (!g || !len) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    const uint64_t need = serialize_device(g, nullptr);
    *len = need;
    if (!buf) return;
    if (cap < need) fail(kArgument, "serialisation buffer too small");
    serialize_device(g, buf);
  });
}

void bfly_graph_free(bfly_graph* g) {
  if (!g) return;
  { std::lock_guard<std::mutex> lk(g->mu); }  // wait for a call in flight on another thread
  delete g;  // buffers are freed on the stream, then the stream (StreamOwner, destroyed last)
  cudaGetLastError();  // a failed async free must not poison the next launch's error check
}

int bfly_graph_sizes(const bfly_graph* g, uint32_t* left, uint32_t* right, uint64_t* m) {
  return guarded([&] {
    if (!g) fail(kArgument, "null graph");
    if (left) *left = g->L;
    if (right) *right = g->R;
    if (m) *m = g->m;
  });
}

int bfly_graph_export(const bfly_graph* gc, uint64_t* loff, uint32_t* ladj, uint64_t* roff,
                      uint32_t* radj, uint32_t* reid, uint64_t* lids, uint64_t* rids) {
  bfly_graph* g = const_cast<bfly_graph*>(gc);
  return guarded([&] {
    if (!g) fail(kArgument, "null graph");
    std::lock_guard<std::mutex> lk(g->mu);
    cudaStream_t s = g->stream;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) BFLY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    cp(loff, g->loff.p, (uint64_t{g->L} + 1) * 8);
    cp(roff, g->roff.p, (uint64_t{g->R} + 1) * 8);
    cp(ladj, g->ladj.p, g->m * 4);
    cp(radj, g->radj.p, g->m * 4);
    if (reid) ensure_reid(g);
    cp(reid, g->reid.p, g->m * 4);
    cp(lids, g->lids.p, uint64_t{g->L} * 8);
    cp(rids, g->rids.p, uint64_t{g->R} * 8);
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_graph_stats(bfly_graph* g, bfly_stats* out) {
  return guarded([&] {
    if (!g || !out) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    ensure_stats(g);
    *out = g->stats;
    if (g->stats_status) fail(g->stats_status, "64-bit counter overflow in addition");
  });
}

int bfly_choose_side(bfly_graph* g, int* chosen, double* cl, double* cr) {
  return guarded([&] {
    if (!g) fail(kArgument, "null graph");
    std::lock_guard<std::mutex> lk(g->mu);
    ensure_stats(g);
    if (chosen) *chosen = g->cost_left < g->cost_right ? BFLY_SIDE_RIGHT : BFLY_SIDE_LEFT;
    if (cl) *cl = g->cost_left;
    if (cr) *cr = g->cost_right;
  });
}

int bfly_exact_count(bfly_graph* g, int side, uint64_t* out) {
  return guarded([&] {
    if (!g || !out) fail(kArgument, "null argument");
    if (side != BFLY_SIDE_AUTO && side != BFLY_SIDE_LEFT && side != BFLY_SIDE_RIGHT)
      fail(kArgument, "side must be -1 (auto), 0 (left) or 1 (right)");
    std::lock_guard<std::mutex> lk(g->mu);
    trace_mark("exact: enter");
    // the count is the same for either side (exact.hpp:20-24); the side only feeds the
    // reference work figure W_C, computed lazily by bfly_last_exact_stats (no host sync here)
    g->last_side = side;
    *out = exact_count_device(g);
  });
}

int bfly_last_exact_stats(bfly_graph* g, uint64_t* wedges, uint64_t* ref_wedges,
                          uint64_t* bucket_starts, uint64_t* bucket_wedges,
                          uint64_t* bucket_entries) {
  return guarded([&] {
    if (!g) fail(kArgument, "null graph");
    std::lock_guard<std::mutex> lk(g->mu);
    if (wedges) *wedges = g->last_wedges;
    if (ref_wedges) {
      ensure_stats(g);
      int chosen = g->last_side;
      if (chosen == BFLY_SIDE_AUTO)
        chosen = g->cost_left < g->cost_right ? BFLY_SIDE_RIGHT : BFLY_SIDE_LEFT;
      // the reference walks sum over the centre side (opposite of the anchor) of C(d,2)
      const unsigned __int128 wc = g->wedges_side[1 - chosen];
      *ref_wedges = (wc >> 64) ? ~0ull : static_cast<uint64_t>(wc);
    }
    for (int q = 0; q < 6; ++q) {
      if (bucket_starts) {
        bucket_starts[q] = g->bucket_starts[q];
        bucket_starts[6 + q] = g->hub_bucket_tasks[q];
      }
      if (bucket_wedges) {
        bucket_wedges[q] = g->bucket_wedges[q];
        bucket_wedges[6 + q] = g->hub_bucket_keys[q];
      }
      if (bucket_entries) {
        bucket_entries[q] = g->bucket_entries[q];
        bucket_entries[6 + q] = g->hub_bucket_entries[q];
      }
    }
    if (bucket_starts) bucket_starts[12] = g->hub_k;
  });
}

int bfly_last_dense_stats(bfly_graph* g, uint64_t* out) {
  return guarded([&] {
    if (!g || !out) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    out[0] = g->hub_dense_keys ? g->hub_h : 0;
    out[1] = g->hub_dense_keys ? g->hub_w : 0;
    out[2] = g->hub_dense_keys;
    out[3] = g->hub_dense_entries;
    out[4] = g->hub_dense_big_entries;
  });
}

void* bfly_graph_stream(bfly_graph* g) { return g ? static_cast<void*>(g->stream) : nullptr; }

void bfly_set_stream(void* stream) { t_user_stream = static_cast<cudaStream_t>(stream); }

int bfly_sparsify_stats(bfly_graph* g, int collect, uint64_t* out) {
  return guarded([&] {
    if (!g) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    if (collect >= 0) g->spar_stats_on = collect != 0;
    if (out)
      for (int q = 0; q < 6; ++q) out[q] = g->spar_stats[q];
  });
}

int bfly_trim_pool(uint64_t keep_bytes) {
  return guarded([&] {
    require_device();
    BFLY_CUDA(cudaDeviceSynchronize());
    BFLY_CUDA(cudaMemPoolTrimTo(engine_pool(), keep_bytes));
  });
}

int bfly_last_sample_path(bfly_graph* g) { return g ? g->last_sample_path : -1; }

int bfly_has_edge_batch(bfly_graph* g, const uint32_t* l, const uint32_t* r, uint64_t k,
                        uint8_t* out) {
  return guarded([&] {
    if (!g || (k && (!l || !r || !out))) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    for (uint64_t i = 0; i < k; ++i)
      if (l[i] >= g->L || r[i] >= g->R) fail(kArgument, "edge endpoint out of range");
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint32_t> dl(k, s), dr(k, s);
    DBuf<uint8_t> dout(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dl.p, l, k * 4, cudaMemcpyHostToDevice, s));
    BFLY_CUDA(cudaMemcpyAsync(dr.p, r, k * 4, cudaMemcpyHostToDevice, s));
    has_edge_device(g, dl.p, dr.p, k, dout.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dout.p, k, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_edge_at_batch(bfly_graph* g, const uint64_t* ks, uint64_t k, uint32_t* l, uint32_t* r) {
  return guarded([&] {
    if (!g || (k && (!ks || !l || !r))) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    for (uint64_t i = 0; i < k; ++i)
      if (ks[i] >= g->m) fail(kArgument, "edge index out of range");  // graph.cpp:69
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint64_t> dk(k, s);
    DBuf<uint32_t> dl(k, s), dr(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dk.p, ks, k * 8, cudaMemcpyHostToDevice, s));
    edge_at_device(g, dk.p, k, dl.p, dr.p);
    BFLY_CUDA(cudaMemcpyAsync(l, dl.p, k * 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaMemcpyAsync(r, dr.p, k * 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_local_vertex_all(bfly_graph* g, uint64_t* out) {
  return guarded([&] {
    if (!g || (g->n() && !out)) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    local_vertex_all(g, out);
  });
}

int bfly_local_edge_all(bfly_graph* g, uint64_t* out) {
  return guarded([&] {
    if (!g || (g->m && !out)) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    local_edge_all(g, out);
  });
}

int bfly_local_vertex_batch(bfly_graph* g, const uint64_t* gids, uint64_t k, uint64_t* out) {
  return guarded([&] {
    if (!g || (k && (!gids || !out))) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    for (uint64_t i = 0; i < k; ++i)
      if (gids[i] >= g->n()) fail(kArgument, "vertex index out of range");  // local.cpp:12
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint64_t> dg(k, s);
    DBuf<unsigned long long> dout(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dg.p, gids, k * 8, cudaMemcpyHostToDevice, s));
    local_vertex_batch_device(g, dg.p, k, dout.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dout.p, k * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_local_edge_batch(bfly_graph* g, const uint64_t* ks, uint64_t k, uint64_t* out) {
  return guarded([&] {
    if (!g || (k && (!ks || !out))) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    for (uint64_t i = 0; i < k; ++i)
      if (ks[i] >= g->m) fail(kArgument, "edge index out of range");  // graph.cpp:69
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint64_t> dk(k, s);
    DBuf<uint32_t> dl(k, s), dr(k, s);
    DBuf<unsigned long long> dout(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dk.p, ks, k * 8, cudaMemcpyHostToDevice, s));
    edge_at_device(g, dk.p, k, dl.p, dr.p);
    local_edge_batch_device(g, dl.p, dr.p, dk.p, k, dout.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dout.p, k * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_local_edge_pairs(bfly_graph* g, const uint32_t* l, const uint32_t* r, uint64_t k,
                          uint64_t* out) {
  return guarded([&] {
    if (!g || (k && (!l || !r || !out))) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    for (uint64_t i = 0; i < k; ++i)  // local.cpp:24-25
      if (l[i] >= g->L || r[i] >= g->R) fail(kArgument, "edge endpoint out of range");
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint32_t> dl(k, s), dr(k, s);
    DBuf<uint8_t> dh(k, s);
    DBuf<unsigned long long> dout(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dl.p, l, k * 4, cudaMemcpyHostToDevice, s));
    BFLY_CUDA(cudaMemcpyAsync(dr.p, r, k * 4, cudaMemcpyHostToDevice, s));
    has_edge_device(g, dl.p, dr.p, k, dh.p);
    std::vector<uint8_t> hh(k);
    BFLY_CUDA(cudaMemcpyAsync(hh.data(), dh.p, k, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < k; ++i)
      if (!hh[i]) fail(kArgument, "(l, r) is not an edge");  // local.cpp:26
    local_edge_batch_device(g, dl.p, dr.p, nullptr, k, dout.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dout.p, k * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_wedge_batch(bfly_graph* g, const uint64_t* c, const uint32_t* i, const uint32_t* j,
                     uint64_t k, uint64_t* out) {
  return guarded([&] {
    if (!g || (k && (!c || !i || !j || !out))) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    for (uint64_t q = 0; q < k; ++q)
      if (c[q] >= g->n()) fail(kArgument, "vertex index out of range");
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint64_t> dc(k, s);
    DBuf<uint32_t> di(k, s), dj(k, s);
    DBuf<unsigned long long> dout(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dc.p, c, k * 8, cudaMemcpyHostToDevice, s));
    BFLY_CUDA(cudaMemcpyAsync(di.p, i, k * 4, cudaMemcpyHostToDevice, s));
    BFLY_CUDA(cudaMemcpyAsync(dj.p, j, k * 4, cudaMemcpyHostToDevice, s));
    wedge_batch_device(g, dc.p, di.p, dj.p, k, dout.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dout.p, k * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_common_neighbors_batch(bfly_graph* g, int side, const uint32_t* v, const uint32_t* w,
                                uint64_t k, uint64_t* out) {
  return guarded([&] {
    if (!g || (k && (!v || !w || !out))) fail(kArgument, "null argument");
    if (side != 0 && side != 1) fail(kArgument, "side must be 0 (left) or 1 (right)");
    std::lock_guard<std::mutex> lk(g->mu);
    const uint32_t cnt = side == 0 ? g->L : g->R;
    for (uint64_t q = 0; q < k; ++q)
      if (v[q] >= cnt || w[q] >= cnt) fail(kArgument, "vertex index out of range");
    if (!k) return;
    cudaStream_t s = g->stream;
    DBuf<uint32_t> dv(k, s), dw(k, s);
    DBuf<unsigned long long> dout(k, s);
    BFLY_CUDA(cudaMemcpyAsync(dv.p, v, k * 4, cudaMemcpyHostToDevice, s));
    BFLY_CUDA(cudaMemcpyAsync(dw.p, w, k * 4, cudaMemcpyHostToDevice, s));
    common_pairs_device(g, side, dv.p, dw.p, k, dout.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dout.p, k * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_wedge_index(bfly_graph* g, uint64_t* prefix, uint64_t* total) {
  return guarded([&] {
    if (!g || !prefix || !total) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    wedge_index(g, prefix, total);
  });
}

int bfly_sample_batch(bfly_graph* g, int method, uint64_t seed, uint64_t first, uint64_t count,
                      uint64_t* counts, uint64_t* ids, uint32_t* wi, uint32_t* wj) {
  return guarded([&] {
    if (!g || (count && !counts)) fail(kArgument, "null argument");
    if (method < 0 || method > 2) fail(kArgument, "method must be 0 (vertex), 1 (edge) or 2 (wedge)");
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->n() == 0 || g->m == 0) fail(kArgument, "cannot sample an empty graph");
    if (!count) return;
    cudaStream_t s = g->stream;
    DBuf<uint64_t> did(count, s);
    DBuf<uint32_t> di(method == 2 ? count : 1, s), dj(method == 2 ? count : 1, s);
    DBuf<unsigned long long> dout(count, s);
    sample_counts_device(g, method, seed, first, count, dout.p, did.p, di.p, dj.p);
    BFLY_CUDA(cudaMemcpyAsync(counts, dout.p, count * 8, cudaMemcpyDeviceToHost, s));
    if (ids) BFLY_CUDA(cudaMemcpyAsync(ids, did.p, count * 8, cudaMemcpyDeviceToHost, s));
    if (method == 2 && wi) BFLY_CUDA(cudaMemcpyAsync(wi, di.p, count * 4, cudaMemcpyDeviceToHost, s));
    if (method == 2 && wj) BFLY_CUDA(cudaMemcpyAsync(wj, dj.p, count * 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_fast_edge_batch(bfly_graph* g, uint64_t seed, uint64_t first, uint64_t count,
                         uint64_t repeats, double* values, uint64_t* hits, uint64_t* edge_ids) {
  return guarded([&] {
    if (!g || (count && !values)) fail(kArgument, "null argument");
    if (repeats == 0) fail(kArgument, "fast-edge repeats must be at least 1");  // sampling.cpp:178
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->n() == 0 || g->m == 0) fail(kArgument, "cannot sample an empty graph");
    if (!count) return;
    cudaStream_t s = g->stream;
    DBuf<double> dv(count, s);
    DBuf<uint64_t> dh(count, s), de(count, s);
    fast_edge_device(g, seed, first, count, repeats, dv.p, dh.p, de.p);
    BFLY_CUDA(cudaMemcpyAsync(values, dv.p, count * 8, cudaMemcpyDeviceToHost, s));
    if (hits) BFLY_CUDA(cudaMemcpyAsync(hits, dh.p, count * 8, cudaMemcpyDeviceToHost, s));
    if (edge_ids) BFLY_CUDA(cudaMemcpyAsync(edge_ids, de.p, count * 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  });
}

int bfly_espar_count(bfly_graph* g, double p, uint64_t seed, uint64_t* count, uint64_t* kept) {
  return guarded([&] {
    if (!g || !count || !kept) fail(kArgument, "null argument");
    if (!(p > 0.0 && p <= 1.0))  // sparsify.cpp:26-28
      fail(kArgument, "retention probability must be in (0, 1]");
    std::lock_guard<std::mutex> lk(g->mu);
    sparsify_count(g, 0, p, 0, seed, nullptr, nullptr, count, kept);
  });
}

int bfly_cspar_count(bfly_graph* g, uint64_t n_colors, uint64_t seed, uint64_t* count,
                     uint64_t* kept) {
  return guarded([&] {
    if (!g || !count || !kept) fail(kArgument, "null argument");
    if (n_colors == 0) fail(kArgument, "palette must have at least one color");  // :45-46
    std::lock_guard<std::mutex> lk(g->mu);
    sparsify_count(g, 1, 0.0, n_colors, seed, nullptr, nullptr, count, kept);
  });
}

int bfly_keep_mask_count(bfly_graph* g, const uint8_t* keep, uint64_t* count, uint64_t* kept) {
  return guarded([&] {
    if (!g || !count || !kept || (g->m && !keep)) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    sparsify_count(g, 2, 0.0, 0, 0, keep, nullptr, count, kept);
  });
}

int bfly_color_mask_count(bfly_graph* g, const uint32_t* colors, uint64_t* count, uint64_t* kept) {
  return guarded([&] {
    if (!g || !count || !kept || (g->n() && !colors)) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    sparsify_count(g, 3, 0.0, 0, 0, nullptr, colors, count, kept);
  });
}

int bfly_pair_type_counts(bfly_graph* g, bfly_pair_counts* out) {
  return guarded([&] {
    if (!g || !out) fail(kArgument, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    using u128 = unsigned __int128;
    const uint64_t b = exact_count_device(g);
    uint64_t c2 = 0;
    u128 s3 = 0, s4 = 0, v2 = 0, e2 = 0;
    pair_moments(g, &c2, &s3, &s4);
    // each butterfly is C(c,2)-counted once through its left pair and once through its right
    if (c2 != 2 * b) fail(kInternal, "pair pass total " + std::to_string(c2) + " != 2 * bfly");
    local_choose2_sums(g, &v2, &e2);
    const u128 p1w = 3 * s3, p2v = 3 * s4;
    if (e2 < 2 * p1w) fail(kInternal, "impossible butterfly pair: shared-edge count below 2 p_1w");
    const u128 p1e = e2 - 2 * p1w;
    const u128 shared = 2 * p2v + 2 * p1e + 3 * p1w;
    if (v2 < shared) fail(kInternal, "impossible butterfly pair: shared-vertex count");
    const u128 p1v = v2 - shared;
    const u128 bb = b, all = bb * (bb - (b ? 1 : 0)) / 2;
    const u128 touching = p1v + p2v + p1e + p1w;
    if (all < touching) fail(kInternal, "impossible butterfly pair: more touching pairs than pairs");
    const u128 p0v = all - touching;
    auto put = [](uint64_t* w, u128 x) {
      w[0] = static_cast<uint64_t>(x);
      w[1] = static_cast<uint64_t>(x >> 64);
    };
    out->bfly = b;
    put(out->p_0v, p0v);
    put(out->p_1v, p1v);
    put(out->p_2v, p2v);
    put(out->p_1e, p1e);
    put(out->p_1w, p1w);
  });
}

}  // extern "C"
