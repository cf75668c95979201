// synth.cpp -- see synth.h. Part of the bench/test harness, not of the counting path.
#include "synth.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
inline uint64_t derive(uint64_t seed, uint64_t i) { return mix64(mix64(seed) ^ mix64(i)); }
inline double unit(uint64_t b) { return static_cast<double>(b >> 11) * 0x1.0p-53; }
inline uint64_t bounded(uint64_t b, uint64_t n) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(b) * n) >> 64);
}

struct PairSet {
  std::vector<uint64_t> keys;
  uint64_t mask;
  explicit PairSet(uint64_t m) {
    uint64_t cap = 1024;
    while (cap < 2 * m + 1024) cap <<= 1;
    keys.assign(cap, ~0ull);
    mask = cap - 1;
  }
  bool insert(uint64_t k) {
    uint64_t h = mix64(k) & mask;
    while (true) {
      uint64_t v = keys[h];
      if (v == k) return false;
      if (v == ~0ull) {
        keys[h] = k;
        return true;
      }
      h = (h + 1) & mask;
    }
  }
};

template <typename Gen>
int run(uint64_t m, uint32_t cap, uint32_t U, uint32_t V, Gen&& gen, uint32_t* l, uint32_t* r) {
  if (m == 0) return 0;
  if (U == 0 || V == 0) return 1;
  if (cap == 0 && static_cast<double>(U) * V < static_cast<double>(m)) return 1;
  PairSet set(m);
  std::vector<uint32_t> dl, dr;
  if (cap) {
    dl.assign(U, 0);
    dr.assign(V, 0);
  }
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const uint64_t B = 1ull << 22;
  std::vector<uint32_t> cl(B), cr(B);
  uint64_t got = 0, t0 = 0;
  uint64_t guard = 0;
  while (got < m) {
    std::vector<std::thread> th;
    for (unsigned k = 0; k < nt; ++k)
      th.emplace_back([&, k] {
        uint64_t lo = B * k / nt, hi = B * (k + 1) / nt;
        for (uint64_t i = lo; i < hi; ++i) gen(t0 + i, cl[i], cr[i]);
      });
    for (auto& x : th) x.join();
    for (uint64_t i = 0; i < B && got < m; ++i) {
      uint32_t a = cl[i], b = cr[i];
      if (cap && (dl[a] >= cap || dr[b] >= cap)) continue;
      if (!set.insert((static_cast<uint64_t>(a) << 32) | b)) continue;
      if (cap) {
        ++dl[a];
        ++dr[b];
      }
      l[got] = a;
      r[got] = b;
      ++got;
    }
    t0 += B;
    if (++guard > 4096 && got < m / 2) return 2;  // cannot reach m distinct edges
  }
  return 0;
}

std::vector<double> prefix_weights(uint32_t n, double gamma) {
  std::vector<double> p(n);
  double acc = 0.0, ex = -1.0 / (gamma - 1.0);
  for (uint32_t i = 0; i < n; ++i) {
    acc += std::pow(static_cast<double>(i) + 1.0, ex);
    p[i] = acc;
  }
  return p;
}

inline uint32_t draw(const std::vector<double>& p, uint64_t bits) {
  double x = unit(bits) * p.back();
  auto it = std::upper_bound(p.begin(), p.end(), x);
  size_t i = static_cast<size_t>(it - p.begin());
  return static_cast<uint32_t>(i < p.size() ? i : p.size() - 1);
}

}  // namespace

extern "C" int bfly_synth_uniform(uint32_t U, uint32_t V, uint64_t m, uint64_t seed, uint32_t* l,
                                  uint32_t* r) {
  uint64_t sl = derive(seed, 1), sr = derive(seed, 2);
  return run(m, 0, U, V,
             [&](uint64_t t, uint32_t& a, uint32_t& b) {
               a = static_cast<uint32_t>(bounded(derive(sl, t), U));
               b = static_cast<uint32_t>(bounded(derive(sr, t), V));
             },
             l, r);
}

extern "C" int bfly_synth_chung_lu(uint32_t U, uint32_t V, uint64_t m, double gu, double gv,
                                   uint32_t max_degree, uint64_t seed, uint32_t* l, uint32_t* r) {
  if (!(gu > 1.0) || !(gv > 1.0)) return 1;
  std::vector<double> pu = prefix_weights(U, gu), pv = prefix_weights(V, gv);
  uint64_t sl = derive(seed, 1), sr = derive(seed, 2);
  return run(m, max_degree, U, V,
             [&](uint64_t t, uint32_t& a, uint32_t& b) {
               a = draw(pu, derive(sl, t));
               b = draw(pv, derive(sr, t));
             },
             l, r);
}
