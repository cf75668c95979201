// profile.cu -- launch counter and per-kernel CUDA-event timing registry.
// bench.py reads per-kernel device time from here (events recorded on the stream the
// kernel was launched on), so the roofline figure is measured live, not inferred.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace bflyd {
namespace {

struct Pending {
  const char* name;
  cudaEvent_t a, b;
};
struct Totals {
  double ms = 0.0;
  uint64_t launches = 0;
};

std::mutex g_mu;
std::atomic<bool> g_on{false};
std::atomic<uint64_t> g_launches{0};
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_free;
std::map<std::string, Totals> g_totals;
std::vector<std::pair<std::string, Totals>> g_snapshot;

// BFLY_PROF_GAPS=1: device idle time between consecutive timed scopes, keyed by the scope
// that follows the gap (where the host was late: syncs, host-side setup), printed on stderr
// by bfly_profile_count
std::map<std::string, Totals> g_gaps;
const bool g_gaps_on = [] {
  const char* e = std::getenv("BFLY_PROF_GAPS");
  return e && e[0] == '1';
}();

void resolve_locked() {
  for (size_t i = 0; i < g_pending.size(); ++i) {
    auto& p = g_pending[i];
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    auto& t = g_totals[p.name];
    t.ms += ms;
    t.launches += 1;
    if (g_gaps_on && i > 0) {
      float gap = 0.f;
      cudaEventElapsedTime(&gap, g_pending[i - 1].b, p.a);
      if (gap > 0.f && gap < 5.f) {  // (larger: the caller's own pause between steps)
        auto& gt = g_gaps[p.name];
        gt.ms += gap;
        gt.launches += 1;
      }
    }
  }
  for (auto& p : g_pending) {
    g_free.push_back(p.a);
    g_free.push_back(p.b);
  }
  g_pending.clear();
}

}  // namespace

bool prof_enabled() { return g_on.load(std::memory_order_relaxed); }

void trace_mark(const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("BFLY_TRACE");
    return e && e[0] == '1';
  }();
  if (!on) return;
  using C = std::chrono::steady_clock;
  static thread_local C::time_point last = C::now();
  const C::time_point now = C::now();
  std::fprintf(stderr, "[bfly] %-28s +%8.3f ms\n", what,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaEvent_t prof_event() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_free.empty()) {
    cudaEvent_t e = g_free.back();
    g_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_record(const char* name, cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_pending.push_back({name, a, b});
  if (g_pending.size() > 4096) resolve_locked();
}

}  // namespace bflyd

extern "C" {

void bfly_profile_enable(int on) { bflyd::g_on.store(on != 0); }

void bfly_profile_reset(void) {
  std::lock_guard<std::mutex> lk(bflyd::g_mu);
  bflyd::resolve_locked();
  bflyd::g_totals.clear();
  bflyd::g_gaps.clear();
  bflyd::g_snapshot.clear();
  bflyd::g_launches.store(0);
}

int bfly_profile_count(void) {
  std::lock_guard<std::mutex> lk(bflyd::g_mu);
  bflyd::resolve_locked();
  if (bflyd::g_gaps_on && !bflyd::g_gaps.empty()) {
    std::vector<std::pair<double, std::string>> v;
    double tot = 0.0;
    for (auto& kv : bflyd::g_gaps) {
      v.push_back({kv.second.ms, kv.first});
      tot += kv.second.ms;
    }
    std::sort(v.rbegin(), v.rend());
    std::fprintf(stderr, "[bfly gaps] total %.3f ms\n", tot);
    for (size_t i = 0; i < v.size() && i < 20; ++i)
      std::fprintf(stderr, "[bfly gaps] before %-28s %.3f ms\n", v[i].second.c_str(), v[i].first);
  }
  bflyd::g_snapshot.assign(bflyd::g_totals.begin(), bflyd::g_totals.end());
  return static_cast<int>(bflyd::g_snapshot.size());
}

int bfly_profile_get(int i, const char** name, double* total_ms, uint64_t* launches) {
  std::lock_guard<std::mutex> lk(bflyd::g_mu);
  if (i < 0 || i >= static_cast<int>(bflyd::g_snapshot.size())) return bflyd::kArgument;
  *name = bflyd::g_snapshot[i].first.c_str();
  *total_ms = bflyd::g_snapshot[i].second.ms;
  *launches = bflyd::g_snapshot[i].second.launches;
  return 0;
}

uint64_t bfly_launch_count(void) { return bflyd::g_launches.load(); }

}  // extern "C"
