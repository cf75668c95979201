/*
 * bfly_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU parity checker.
 *
 * A plain-C restatement of the reference library's algorithms
 * (/root/reference/proj/src/ and include/bfly/). It is loaded only by
 * tests/, __graft_entry__.smoke() and the cpu_baseline / --impl reference legs of
 * bench.py. The product path (paper_1801_00338_b200) never links or calls it.
 *
 * Differences from the reference are representation only and do not change any
 * result: hash maps become dense scratch arrays plus touched lists, per-list
 * std::sort becomes one radix sort of packed (row, col) keys, and the
 * single-threaded loops may be split over anchor / subject ranges with per-thread
 * scratch (integer sums are order independent; the overflow contract is kept by
 * summing in 128 bits and failing when the total reaches 2^64, which is exactly
 * when the reference's running checked_add would throw).
 */
#define _GNU_SOURCE
#include "bfly_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum {
  BO_OK = 0, BO_ARG = 1, BO_EMPTY = 2, BO_OVERFLOW = 3, BO_NOWEDGE = 4, BO_INTERNAL = 5, BO_PARSE = 6
};

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* rng.hpp:10-15 mix64 (splitmix64 finaliser)                                */
uint64_t bo_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
/* rng.hpp:18-20 */
uint64_t bo_derive_seed(uint64_t seed, uint64_t index) {
  return bo_mix64(bo_mix64(seed) ^ bo_mix64(index));
}
/* rng.hpp:23-25 */
double bo_unit_double(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }
/* rng.hpp:29-31 */
uint64_t bo_bounded_from_bits(uint64_t bits, uint64_t n) {
  return (uint64_t)(((u128)bits * n) >> 64);
}

/* rng.hpp:36-62. std::mt19937_64 (parameters fixed by [rand.predef]). */
#define MT_N 312
#define MT_M 156
void bo_rng_seed(bo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
}
void bo_rng_stream(bo_rng* r, uint64_t seed, uint64_t index) {  /* rng.hpp:41-43 */
  bo_rng_seed(r, bo_derive_seed(seed, index));
}
uint64_t bo_rng_next(bo_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (r->mti >= MT_N) {
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    for (; i < MT_N - 1; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    uint64_t x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}
double bo_rng_uniform_unit(bo_rng* r) { return bo_unit_double(bo_rng_next(r)); }
/* rng.hpp:50-58: mask rejection; n <= 1 draws nothing */
uint64_t bo_rng_uniform_index(bo_rng* r, uint64_t n) {
  if (n <= 1) return 0;
  uint64_t mask = ~(uint64_t)0 >> __builtin_clzll(n - 1);
  uint64_t x;
  do {
    x = bo_rng_next(r) & mask;
  } while (x >= n);
  return x;
}

/* checked.hpp:24-27 */
int bo_choose2(uint64_t c, uint64_t* out) {
  if (c < 2) {
    *out = 0;
    return BO_OK;
  }
  uint64_t a = (c % 2 == 0) ? c / 2 : c, b = (c % 2 == 0) ? c - 1 : (c - 1) / 2;
  if (__builtin_mul_overflow(a, b, out)) return BO_OVERFLOW;
  return BO_OK;
}

void bo_free(void* p) { free(p); }

/* ------------------------------------------------------------------------ */
/* first-seen dense ids (graph.cpp:19-27): open-addressing map ext -> dense    */
typedef struct {
  uint64_t* keys;
  uint32_t* vals;
  uint8_t* used;
  uint64_t mask;
} idmap;

static int idmap_init(idmap* h, uint64_t n) {
  uint64_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  h->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
  h->vals = (uint32_t*)malloc(cap * sizeof(uint32_t));
  h->used = (uint8_t*)calloc(cap, 1);
  h->mask = cap - 1;
  return (h->keys && h->vals && h->used) ? BO_OK : BO_INTERNAL;
}
static void idmap_free(idmap* h) {
  free(h->keys);
  free(h->vals);
  free(h->used);
}
static uint32_t idmap_dense(idmap* h, uint64_t** ids, uint64_t* nids, uint64_t ext) {
  uint64_t s = bo_mix64(ext) & h->mask;
  while (h->used[s]) {
    if (h->keys[s] == ext) return h->vals[s];
    s = (s + 1) & h->mask;
  }
  uint32_t id = (uint32_t)*nids;
  h->used[s] = 1;
  h->keys[s] = ext;
  h->vals[s] = id;
  (*ids)[(*nids)++] = ext;
  return id;
}

/* LSD radix sort of 64-bit keys over bits [0, bits) */
static int radix_sort_u64(uint64_t* a, uint64_t n, int bits) {
  if (n < 2 || bits <= 0) return BO_OK;
  uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!tmp) return BO_INTERNAL;
  const int D = 11;
  uint64_t* src = a;
  uint64_t* dst = tmp;
  for (int shift = 0; shift < bits; shift += D) {
    uint64_t cnt[1 << D];
    memset(cnt, 0, sizeof cnt);
    for (uint64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & ((1 << D) - 1)]++;
    uint64_t s = 0;
    for (int b = 0; b < (1 << D); ++b) {
      uint64_t c = cnt[b];
      cnt[b] = s;
      s += c;
    }
    for (uint64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & ((1 << D) - 1)]++] = src[i];
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != a) memcpy(a, src, n * sizeof(uint64_t));
  free(tmp);
  return BO_OK;
}

static int bits_for(uint64_t n) {
  int b = 0;
  while (b < 64 && (n >> b) != 0) ++b;
  return b;
}

/* Build one CSR direction from packed (row << cb | col) keys: sort, unique. */
static int build_csr(uint64_t* keys, uint64_t n, int cb, uint32_t rows, uint64_t** off,
                     uint32_t** adj, uint64_t* m_out) {
  int st = radix_sort_u64(keys, n, cb + bits_for(rows));
  if (st) return st;
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];
  *off = (uint64_t*)calloc((uint64_t)rows + 1, sizeof(uint64_t));
  *adj = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
  if (!*off || !*adj) return BO_INTERNAL;
  uint64_t cmask = (cb == 64) ? ~0ULL : ((1ULL << cb) - 1);
  for (uint64_t i = 0; i < m; ++i) {
    (*off)[(keys[i] >> cb) + 1]++;
    (*adj)[i] = (uint32_t)(keys[i] & cmask);
  }
  for (uint32_t v = 0; v < rows; ++v) (*off)[v + 1] += (*off)[v];
  *m_out = m;
  return BO_OK;
}

/* graph.cpp:31-58 BipartiteGraph::from_edges */
int bo_graph_from_edges(bo_graph* g, const uint64_t* l, const uint64_t* r, uint64_t m_in) {
  memset(g, 0, sizeof *g);
  idmap lm, rm;
  int st = idmap_init(&lm, m_in);
  if (!st) st = idmap_init(&rm, m_in);
  if (st) return st;
  g->lids = (uint64_t*)malloc((m_in ? m_in : 1) * sizeof(uint64_t));
  g->rids = (uint64_t*)malloc((m_in ? m_in : 1) * sizeof(uint64_t));
  uint32_t* dl = (uint32_t*)malloc((m_in ? m_in : 1) * sizeof(uint32_t));
  uint32_t* dr = (uint32_t*)malloc((m_in ? m_in : 1) * sizeof(uint32_t));
  if (!g->lids || !g->rids || !dl || !dr) return BO_INTERNAL;
  uint64_t nl = 0, nr = 0;
  for (uint64_t i = 0; i < m_in; ++i) {
    dl[i] = idmap_dense(&lm, &g->lids, &nl, l[i]);
    dr[i] = idmap_dense(&rm, &g->rids, &nr, r[i]);
  }
  idmap_free(&lm);
  idmap_free(&rm);
  g->L = (uint32_t)nl;
  g->R = (uint32_t)nr;
  uint64_t* keys = (uint64_t*)malloc((m_in ? m_in : 1) * sizeof(uint64_t));
  if (!keys) return BO_INTERNAL;
  int rb = bits_for(g->R), lb = bits_for(g->L);
  for (uint64_t i = 0; i < m_in; ++i) keys[i] = ((uint64_t)dl[i] << rb) | dr[i];
  uint64_t m1 = 0, m2 = 0;
  st = build_csr(keys, m_in, rb, g->L, &g->loff, &g->ladj, &m1);
  if (!st) {
    for (uint64_t i = 0; i < m_in; ++i) keys[i] = ((uint64_t)dr[i] << lb) | dl[i];
    st = build_csr(keys, m_in, lb, g->R, &g->roff, &g->radj, &m2);
  }
  free(keys);
  free(dl);
  free(dr);
  if (st) return st;
  if (m1 != m2) return BO_INTERNAL;
  g->m = m1;
  return BO_OK;
}

int bo_graph_from_edges_u32(bo_graph* g, const uint32_t* l, const uint32_t* r, uint64_t m_in) {
  uint64_t* a = (uint64_t*)malloc((m_in ? m_in : 1) * 8);
  uint64_t* b = (uint64_t*)malloc((m_in ? m_in : 1) * 8);
  if (!a || !b) return BO_INTERNAL;
  for (uint64_t i = 0; i < m_in; ++i) {
    a[i] = l[i];
    b[i] = r[i];
  }
  int st = bo_graph_from_edges(g, a, b, m_in);
  free(a);
  free(b);
  return st;
}

void bo_graph_free(bo_graph* g) {
  free(g->loff);
  free(g->ladj);
  free(g->roff);
  free(g->radj);
  free(g->lids);
  free(g->rids);
  memset(g, 0, sizeof *g);
}

static inline const uint32_t* nbr(const bo_graph* g, int side, uint32_t i, uint64_t* deg) {
  const uint64_t* off = side == 0 ? g->loff : g->roff;
  *deg = off[i + 1] - off[i];
  return (side == 0 ? g->ladj : g->radj) + off[i];
}
static inline uint64_t degree(const bo_graph* g, int side, uint32_t i) {
  const uint64_t* off = side == 0 ? g->loff : g->roff;
  return off[i + 1] - off[i];
}
static inline uint32_t side_count(const bo_graph* g, int side) { return side == 0 ? g->L : g->R; }

static int bsearch_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && a[lo] == x;
}

/* graph.cpp:75-99 load_edge_list over an in-memory stream. On success *l, *r (malloc'd,
 * caller frees) hold the edges in line order and *m their count (0 -> the caller raises
 * EmptyGraphError). On a malformed line returns BO_PARSE with *err_line (1-based) and the
 * reference's message (without the " (line N)" suffix) in msg. */
static int ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}
int bo_parse_edge_list(const char* t, uint64_t len, uint64_t** l, uint64_t** r, uint64_t* m,
                       uint64_t* err_line, char* msg, uint64_t cap) {
  uint64_t n = 0, capn = 1024, line_no = 0;
  uint64_t* L = (uint64_t*)malloc(capn * 8);
  uint64_t* R = (uint64_t*)malloc(capn * 8);
  *err_line = 0;
  for (uint64_t a = 0; a < len;) {
    uint64_t b = a;
    while (b < len && t[b] != '\n') ++b; /* std::getline */
    ++line_no;
    uint64_t p = a;
    while (p < b && (t[p] == ' ' || t[p] == '\t' || t[p] == '\r')) ++p;
    if (p < b && t[p] != '%' && t[p] != '#') {
      uint64_t ids[2], q = a;
      for (int k = 0; k < 2; ++k) {
        while (q < b && ws(t[q])) ++q;
        if (q == b) {
          snprintf(msg, cap, "expected two vertex ids, got %d", k);
          *err_line = line_no;
          free(L);
          free(R);
          return BO_PARSE;
        }
        uint64_t s0 = q, v = 0;
        int ok = 1;
        while (q < b && !ws(t[q])) ++q;
        for (uint64_t i = s0; i < q && ok; ++i) { /* std::from_chars, whole token */
          int d = t[i] - '0';
          if (d < 0 || d > 9 || v > (UINT64_MAX - (uint64_t)d) / 10) ok = 0;
          else v = v * 10 + (uint64_t)d;
        }
        if (!ok) {
          snprintf(msg, cap, "bad vertex id '%.*s'", (int)(q - s0), t + s0);
          *err_line = line_no;
          free(L);
          free(R);
          return BO_PARSE;
        }
        ids[k] = v;
      }
      if (n == capn) {
        capn *= 2;
        L = (uint64_t*)realloc(L, capn * 8);
        R = (uint64_t*)realloc(R, capn * 8);
      }
      L[n] = ids[0];
      R[n] = ids[1];
      ++n;
    }
    a = b + 1;
  }
  *l = L;
  *r = R;
  *m = n;
  return BO_OK;
}

/* graph.cpp:107-112 serialize_edge_list: bytes into buf (when cap allows); returns length */
uint64_t bo_serialize_edge_list(const bo_graph* g, char* buf, uint64_t cap) {
  uint64_t n = 0;
  char tmp[48];
  const char* head = "% bip\n";
  for (const char* c = head; *c; ++c, ++n)
    if (buf && n < cap) buf[n] = *c;
  for (uint32_t lv = 0; lv < g->L; ++lv)
    for (uint64_t k = g->loff[lv]; k < g->loff[lv + 1]; ++k) {
      int w = snprintf(tmp, sizeof tmp, "%llu %llu\n", (unsigned long long)g->lids[lv],
                       (unsigned long long)g->rids[g->ladj[k]]);
      for (int i = 0; i < w; ++i, ++n)
        if (buf && n < cap) buf[n] = tmp[i];
    }
  return n;
}

/* graph.cpp:60-66 */
int bo_has_edge(const bo_graph* g, uint32_t l, uint32_t r) {
  uint64_t dl, dr;
  const uint32_t* la = nbr(g, 0, l, &dl);
  const uint32_t* ra = nbr(g, 1, r, &dr);
  if (dl <= dr) return bsearch_u32(la, dl, r);
  return bsearch_u32(ra, dr, l);
}

/* graph.cpp:68-73 (upper_bound on left_offsets_) */
int bo_edge_at(const bo_graph* g, uint64_t k, uint32_t* l, uint32_t* r) {
  if (k >= g->m) return BO_ARG;
  uint64_t lo = 0, hi = (uint64_t)g->L + 1; /* first index with off > k */
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (g->loff[mid] <= k) lo = mid + 1;
    else hi = mid;
  }
  *l = (uint32_t)(lo - 1);
  *r = g->ladj[k];
  return BO_OK;
}

/* graph.cpp:114-121 */
int bo_complete_biclique_edges(uint32_t a, uint32_t b, uint64_t** l, uint64_t** r, uint64_t* m) {
  if (a == 0 || b == 0) return BO_ARG;
  uint64_t n = (uint64_t)a * b;
  *l = (uint64_t*)malloc(n * 8);
  *r = (uint64_t*)malloc(n * 8);
  if (!*l || !*r) return BO_INTERNAL;
  uint64_t k = 0;
  for (uint32_t i = 1; i <= a; ++i)
    for (uint32_t j = 1; j <= b; ++j) {
      (*l)[k] = i;
      (*r)[k] = j;
      ++k;
    }
  *m = n;
  return BO_OK;
}

/* graph.cpp:123-134 */
int bo_random_bipartite_edges(uint32_t a, uint32_t b, double p, uint64_t seed, uint64_t** l,
                              uint64_t** r, uint64_t* m) {
  if (a == 0 || b == 0) return BO_ARG;
  if (!(p >= 0.0 && p <= 1.0)) return BO_ARG;
  bo_rng rng;
  bo_rng_seed(&rng, seed);
  uint64_t n = (uint64_t)a * b;
  *l = (uint64_t*)malloc(n * 8);
  *r = (uint64_t*)malloc(n * 8);
  if (!*l || !*r) return BO_INTERNAL;
  uint64_t k = 0;
  for (uint32_t i = 1; i <= a; ++i)
    for (uint32_t j = 1; j <= b; ++j)
      if (bo_rng_uniform_unit(&rng) < p) {
        (*l)[k] = i;
        (*r)[k] = j;
        ++k;
      }
  *m = k;
  if (k == 0) return BO_EMPTY;
  return BO_OK;
}

/* graph.cpp:136-155 */
int bo_compute_stats(const bo_graph* g, bo_stats* s) {
  memset(s, 0, sizeof *s);
  s->left = g->L;
  s->right = g->R;
  s->n = s->left + s->right;
  s->m = g->m;
  for (int side = 0; side < 2; ++side)
    for (uint32_t i = 0; i < side_count(g, side); ++i) {
      uint64_t d = degree(g, side, i);
      double dd = (double)d;
      if (side == 0) s->sum_deg_sq_left += dd * dd;
      else s->sum_deg_sq_right += dd * dd;
      uint64_t c;
      if (bo_choose2(d, &c)) return BO_OVERFLOW;
      if (__builtin_add_overflow(s->wedge_count, c, &s->wedge_count)) return BO_OVERFLOW;
      if (d > s->max_degree) s->max_degree = (uint32_t)d;
    }
  return BO_OK;
}

/* exact.cpp:9-21 */
void bo_choose_side(const bo_graph* g, int* chosen, double* cost_left, double* cost_right) {
  double cl = 0.0, cr = 0.0;
  for (uint32_t i = 0; i < g->L; ++i) {
    double d = (double)degree(g, 0, i);
    cl += d * d;
  }
  for (uint32_t i = 0; i < g->R; ++i) {
    double d = (double)degree(g, 1, i);
    cr += d * d;
  }
  *chosen = cl < cr ? 1 : 0;
  if (cost_left) *cost_left = cl;
  if (cost_right) *cost_right = cr;
}

/* ------------------------------------------------------------------------ */
/* A tiny parallel-for over [0, n) in dynamic chunks.                         */
typedef struct par_ctx par_ctx;
typedef int (*par_body)(par_ctx* c, int tid, uint64_t lo, uint64_t hi);
struct par_ctx {
  uint64_t n, chunk;
  uint64_t next; /* atomic */
  par_body body;
  int status;   /* first nonzero wins */
  void* user;
  int tid_counter;
};

static void* par_worker(void* arg) {
  par_ctx* c = (par_ctx*)arg;
  int tid = __atomic_fetch_add(&c->tid_counter, 1, __ATOMIC_RELAXED);
  for (;;) {
    if (__atomic_load_n(&c->status, __ATOMIC_RELAXED)) break;
    uint64_t lo = __atomic_fetch_add(&c->next, c->chunk, __ATOMIC_RELAXED);
    if (lo >= c->n) break;
    uint64_t hi = lo + c->chunk < c->n ? lo + c->chunk : c->n;
    int st = c->body(c, tid, lo, hi);
    if (st) {
      int zero = 0;
      __atomic_compare_exchange_n(&c->status, &zero, st, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED);
      break;
    }
  }
  return NULL;
}

static int par_for(uint64_t n, uint64_t chunk, int threads, par_body body, void* user) {
  par_ctx c;
  memset(&c, 0, sizeof c);
  c.n = n;
  c.chunk = chunk ? chunk : 1;
  c.body = body;
  c.user = user;
  if (threads < 1) threads = 1;
  if (threads == 1 || n <= c.chunk) {
    par_worker(&c);
    return c.status;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  int started = 0;
  for (int t = 0; t < threads; ++t)
    if (pthread_create(&th[t], NULL, par_worker, &c) == 0) ++started;
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
  free(th);
  if (started == 0) par_worker(&c);
  return c.status;
}

/* ------------------------------------------------------------------------ */
/* exact.cpp:23-43 exact_count_side                                           */
#define MAX_THREADS 512
typedef struct {
  const bo_graph* g;
  int side;
  uint32_t* mult[MAX_THREADS];
  uint32_t* touched[MAX_THREADS];
  u128 total[MAX_THREADS];
} exact_ctx;

static int exact_body(par_ctx* c, int tid, uint64_t lo, uint64_t hi) {
  exact_ctx* x = (exact_ctx*)c->user;
  const bo_graph* g = x->g;
  int it = x->side, opp = 1 - it;
  uint32_t side_n = side_count(g, it);
  if (!x->mult[tid]) {
    x->mult[tid] = (uint32_t*)calloc(side_n ? side_n : 1, 4);
    x->touched[tid] = (uint32_t*)malloc((side_n ? side_n : 1) * 4);
    if (!x->mult[tid] || !x->touched[tid]) return BO_INTERNAL;
  }
  uint32_t* mult = x->mult[tid];
  uint32_t* touched = x->touched[tid];
  u128 total = 0;
  for (uint64_t v = lo; v < hi; ++v) {
    uint64_t dv, nt = 0;
    const uint32_t* nv = nbr(g, it, (uint32_t)v, &dv);
    for (uint64_t a = 0; a < dv; ++a) {
      uint64_t du;
      const uint32_t* nu = nbr(g, opp, nv[a], &du);
      for (uint64_t b = 0; b < du; ++b) {
        uint32_t w = nu[b];
        if (w >= v) break; /* exact.cpp:33 adjacency sorted: anchors below v only */
        if (mult[w]++ == 0) touched[nt++] = w;
      }
    }
    for (uint64_t t = 0; t < nt; ++t) {
      uint64_t c2;
      bo_choose2(mult[touched[t]], &c2); /* mult < 2^32: cannot overflow */
      total += c2;
      mult[touched[t]] = 0;
    }
  }
  x->total[tid] += total;
  return BO_OK;
}

int bo_exact_count_side(const bo_graph* g, int side, int threads, uint64_t* out) {
  if (side != 0 && side != 1) return BO_ARG;
  if (threads > MAX_THREADS) threads = MAX_THREADS;
  exact_ctx* x = (exact_ctx*)calloc(1, sizeof(exact_ctx));
  if (!x) return BO_INTERNAL;
  x->g = g;
  x->side = side;
  int st = par_for(side_count(g, side), 64, threads, exact_body, x);
  u128 total = 0;
  for (int t = 0; t < MAX_THREADS; ++t) {
    total += x->total[t];
    free(x->mult[t]);
    free(x->touched[t]);
  }
  free(x);
  if (st) return st;
  if (total >> 64) return BO_OVERFLOW; /* checked_add (exact.cpp:37) would have thrown */
  *out = (uint64_t)total;
  return BO_OK;
}

/* exact.cpp:45-47 */
int bo_exact_count(const bo_graph* g, int threads, uint64_t* out) {
  int chosen;
  bo_choose_side(g, &chosen, NULL, NULL);
  return bo_exact_count_side(g, chosen, threads, out);
}

/* ------------------------------------------------------------------------ */
/* local.cpp:11-21 count_per_vertex, with caller scratch                     */
typedef struct {
  uint32_t* mult;    /* sized max(L, R) */
  uint32_t* touched; /* sized max(L, R) */
  uint8_t* in_b;     /* sized max(L, R) */
} scratch;

static int scratch_init(scratch* s, const bo_graph* g) {
  uint64_t n = g->L > g->R ? g->L : g->R;
  if (n == 0) n = 1;
  s->mult = (uint32_t*)calloc(n, 4);
  s->touched = (uint32_t*)malloc(n * 4);
  s->in_b = (uint8_t*)calloc(n, 1);
  return (s->mult && s->touched && s->in_b) ? BO_OK : BO_INTERNAL;
}
static void scratch_free(scratch* s) {
  free(s->mult);
  free(s->touched);
  free(s->in_b);
}

static int per_vertex(const bo_graph* g, int side, uint32_t index, scratch* s, uint64_t* out) {
  if (index >= side_count(g, side)) return BO_ARG; /* local.cpp:12 */
  int other = 1 - side;
  uint64_t dv, nt = 0;
  const uint32_t* nv = nbr(g, side, index, &dv);
  for (uint64_t a = 0; a < dv; ++a) {
    uint64_t du;
    const uint32_t* nu = nbr(g, other, nv[a], &du);
    for (uint64_t b = 0; b < du; ++b) {
      uint32_t w = nu[b];
      if (w != index && s->mult[w]++ == 0) s->touched[nt++] = w;
    }
  }
  uint64_t total = 0;
  int st = BO_OK;
  for (uint64_t t = 0; t < nt; ++t) {
    uint64_t c2;
    if (!st && bo_choose2(s->mult[s->touched[t]], &c2)) st = BO_OVERFLOW;
    if (!st && __builtin_add_overflow(total, c2, &total)) st = BO_OVERFLOW; /* local.cpp:19 */
    s->mult[s->touched[t]] = 0;
  }
  if (st) return st;
  *out = total;
  return BO_OK;
}

/* local.cpp:23-44 count_per_edge */
static int per_edge(const bo_graph* g, uint32_t l, uint32_t r, scratch* s, uint64_t* out) {
  if (l >= g->L || r >= g->R) return BO_ARG;
  if (!bo_has_edge(g, l, r)) return BO_ARG;
  int a_side = 0, b_side = 1;
  uint32_t a = l, b = r;
  if (degree(g, 0, l) > degree(g, 1, r)) { /* local.cpp:29 swap */
    a_side = 1;
    b_side = 0;
    a = r;
    b = l;
  }
  uint64_t db, da;
  const uint32_t* bn = nbr(g, b_side, b, &db);
  for (uint64_t i = 0; i < db; ++i) s->in_b[bn[i]] = 1;
  const uint32_t* an = nbr(g, a_side, a, &da);
  uint64_t nt = 0;
  for (uint64_t i = 0; i < da; ++i) {
    uint64_t dw;
    const uint32_t* wn = nbr(g, b_side, an[i], &dw);
    for (uint64_t j = 0; j < dw; ++j) {
      uint32_t x = wn[j];
      if (x != a && s->in_b[x] && s->mult[x]++ == 0) s->touched[nt++] = x;
    }
  }
  uint64_t total = 0;
  for (uint64_t t = 0; t < nt; ++t) {
    total += s->mult[s->touched[t]] - 1; /* local.cpp:42 unchecked */
    s->mult[s->touched[t]] = 0;
  }
  for (uint64_t i = 0; i < db; ++i) s->in_b[bn[i]] = 0;
  *out = total;
  return BO_OK;
}

int bo_count_per_vertex(const bo_graph* g, int side, uint32_t index, uint64_t* out) {
  if (side != 0 && side != 1) return BO_ARG;
  if (index >= side_count(g, side)) return BO_ARG;
  scratch s;
  if (scratch_init(&s, g)) return BO_INTERNAL;
  int st = per_vertex(g, side, index, &s, out);
  scratch_free(&s);
  return st;
}

int bo_count_per_edge(const bo_graph* g, uint32_t l, uint32_t r, uint64_t* out) {
  if (l >= g->L || r >= g->R) return BO_ARG;
  scratch s;
  if (scratch_init(&s, g)) return BO_INTERNAL;
  int st = per_edge(g, l, r, &s, out);
  scratch_free(&s);
  return st;
}

typedef struct {
  const bo_graph* g;
  const uint64_t* ids; /* NULL = identity */
  uint64_t* out;
  scratch sc[MAX_THREADS];
} all_ctx;

static int all_vertex_body(par_ctx* c, int tid, uint64_t lo, uint64_t hi) {
  all_ctx* x = (all_ctx*)c->user;
  if (!x->sc[tid].mult && scratch_init(&x->sc[tid], x->g)) return BO_INTERNAL;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t gid = x->ids ? x->ids[i] : i;
    if (gid >= (uint64_t)x->g->L + x->g->R) return BO_ARG;
    int side = gid < x->g->L ? 0 : 1;
    uint32_t idx = (uint32_t)(side == 0 ? gid : gid - x->g->L);
    int st = per_vertex(x->g, side, idx, &x->sc[tid], &x->out[i]);
    if (st) return st;
  }
  return BO_OK;
}

static int all_edge_body(par_ctx* c, int tid, uint64_t lo, uint64_t hi) {
  all_ctx* x = (all_ctx*)c->user;
  if (!x->sc[tid].mult && scratch_init(&x->sc[tid], x->g)) return BO_INTERNAL;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t k = x->ids ? x->ids[i] : i;
    uint32_t l, r;
    int st = bo_edge_at(x->g, k, &l, &r);
    if (!st) st = per_edge(x->g, l, r, &x->sc[tid], &x->out[i]);
    if (st) return st;
  }
  return BO_OK;
}

static int run_all(const bo_graph* g, const uint64_t* ids, uint64_t n, int threads, uint64_t* out,
                   par_body body) {
  if (threads > MAX_THREADS) threads = MAX_THREADS;
  all_ctx* x = (all_ctx*)calloc(1, sizeof(all_ctx));
  if (!x) return BO_INTERNAL;
  x->g = g;
  x->ids = ids;
  x->out = out;
  int st = par_for(n, 16, threads, body, x);
  for (int t = 0; t < MAX_THREADS; ++t)
    if (x->sc[t].mult) scratch_free(&x->sc[t]);
  free(x);
  return st;
}

int bo_count_all_vertices(const bo_graph* g, int threads, uint64_t* out) {
  return run_all(g, NULL, (uint64_t)g->L + g->R, threads, out, all_vertex_body);
}
int bo_count_all_edges(const bo_graph* g, int threads, uint64_t* out) {
  return run_all(g, NULL, g->m, threads, out, all_edge_body);
}
int bo_count_edges_subset(const bo_graph* g, const uint64_t* ks, uint64_t nk, int threads,
                          uint64_t* out) {
  return run_all(g, ks, nk, threads, out, all_edge_body);
}
int bo_count_vertices_subset(const bo_graph* g, const uint64_t* gids, uint64_t nk, int threads,
                             uint64_t* out) {
  return run_all(g, gids, nk, threads, out, all_vertex_body);
}

/* ------------------------------------------------------------------------ */
/* sampling.cpp:63-73 */
int bo_build_wedge_index(const bo_graph* g, uint64_t* prefix, uint64_t* total) {
  uint64_t n = (uint64_t)g->L + g->R;
  prefix[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t d = v < g->L ? degree(g, 0, (uint32_t)v) : degree(g, 1, (uint32_t)(v - g->L));
    uint64_t c;
    if (bo_choose2(d, &c)) return BO_OVERFLOW;
    if (__builtin_add_overflow(prefix[v], c, &prefix[v + 1])) return BO_OVERFLOW;
  }
  *total = prefix[n];
  return BO_OK;
}

/* sampling.cpp:22-36 */
uint64_t bo_intersection_size(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb) {
  uint64_t count = 0, i = 0, j = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else {
      ++count;
      ++i;
      ++j;
    }
  }
  return count;
}

/* sampling.cpp:75-78 */
int bo_vertex_sample_value(const bo_graph* g, int side, uint32_t index, double* out) {
  uint64_t c;
  int st = bo_count_per_vertex(g, side, index, &c);
  if (st) return st;
  *out = (double)c * (double)((uint64_t)g->L + g->R) / 4.0;
  return BO_OK;
}
/* sampling.cpp:80-83 */
int bo_edge_sample_value(const bo_graph* g, uint32_t l, uint32_t r, double* out) {
  uint64_t c;
  int st = bo_count_per_edge(g, l, r, &c);
  if (st) return st;
  *out = (double)c * (double)g->m / 4.0;
  return BO_OK;
}
int bo_wedge_common_minus_1(const bo_graph* g, int centre_side, uint32_t v, uint32_t w,
                            uint64_t* out) {
  int leaf = 1 - centre_side;
  if (v >= side_count(g, leaf) || w >= side_count(g, leaf)) return BO_ARG;
  uint64_t dv, dw;
  const uint32_t* nv = nbr(g, leaf, v, &dv);
  const uint32_t* nw = nbr(g, leaf, w, &dw);
  *out = bo_intersection_size(nv, dv, nw, dw) - 1; /* sampling.cpp:89-90 */
  return BO_OK;
}
/* sampling.cpp:85-91 */
int bo_wedge_sample_value(const bo_graph* g, uint64_t total_wedges, int centre_side,
                          uint32_t centre, uint32_t v, uint32_t w, double* out) {
  (void)centre;
  uint64_t c;
  int st = bo_wedge_common_minus_1(g, centre_side, v, w, &c);
  if (st) return st;
  *out = (double)c * (double)total_wedges / 4.0;
  return BO_OK;
}

/* sampling.cpp:101-123: which outcome an iteration picks */
int bo_sample_draw(const bo_graph* g, const uint64_t* prefix, uint64_t total_wedges, int method,
                   uint64_t seed, uint64_t index, uint64_t* id0, uint32_t* id1, uint32_t* id2) {
  bo_rng rng;
  bo_rng_stream(&rng, seed, index);
  uint64_t n = (uint64_t)g->L + g->R;
  *id1 = *id2 = 0;
  if (method == 0) {
    *id0 = bo_rng_uniform_index(&rng, n);
    return BO_OK;
  }
  if (method == 1) {
    *id0 = bo_rng_uniform_index(&rng, g->m);
    return BO_OK;
  }
  if (method == 2) {
    if (total_wedges == 0) return BO_NOWEDGE;
    uint64_t r = bo_rng_uniform_index(&rng, total_wedges);
    uint64_t lo = 0, hi = n + 1; /* upper_bound(prefix, r) */
    while (lo < hi) {
      uint64_t mid = (lo + hi) / 2;
      if (prefix[mid] <= r) lo = mid + 1;
      else hi = mid;
    }
    uint64_t c = lo - 1;
    uint64_t d = c < g->L ? degree(g, 0, (uint32_t)c) : degree(g, 1, (uint32_t)(c - g->L));
    uint64_t i = bo_rng_uniform_index(&rng, d);
    uint64_t j = bo_rng_uniform_index(&rng, d - 1);
    if (j >= i) ++j;
    *id0 = c;
    *id1 = (uint32_t)i;
    *id2 = (uint32_t)j;
    return BO_OK;
  }
  return BO_ARG;
}

int bo_sample_iteration(const bo_graph* g, const uint64_t* prefix, uint64_t total_wedges,
                        int method, uint64_t seed, uint64_t index, double* value) {
  uint64_t id0;
  uint32_t i, j;
  int st = bo_sample_draw(g, prefix, total_wedges, method, seed, index, &id0, &i, &j);
  if (st) return st;
  if (method == 0) {
    int side = id0 < g->L ? 0 : 1;
    return bo_vertex_sample_value(g, side, (uint32_t)(side ? id0 - g->L : id0), value);
  }
  if (method == 1) {
    uint32_t l, r;
    st = bo_edge_at(g, id0, &l, &r);
    if (st) return st;
    return bo_edge_sample_value(g, l, r, value);
  }
  int cs = id0 < g->L ? 0 : 1;
  uint32_t ci = (uint32_t)(cs ? id0 - g->L : id0);
  uint64_t d;
  const uint32_t* adj = nbr(g, cs, ci, &d);
  return bo_wedge_sample_value(g, total_wedges, cs, ci, adj[i], adj[j], value);
}

/* sampling.cpp:39-44 draw_excluding: uniform over adj minus `skip` (skip is in adj) */
static uint32_t draw_excluding(const uint32_t* adj, uint64_t d, uint32_t skip, bo_rng* rng) {
  uint64_t lo = 0, hi = d; /* lower_bound(adj, skip) */
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (adj[mid] < skip) lo = mid + 1;
    else hi = mid;
  }
  uint64_t k = bo_rng_uniform_index(rng, d - 1);
  if (k >= lo) ++k;
  return adj[k];
}

/* sampling.cpp:125-141 fast_ebfc_estimate; *hits = Bernoulli successes (0 when a degree is 1) */
int bo_fast_ebfc_estimate(const bo_graph* g, uint32_t l, uint32_t r, uint64_t repeats,
                          bo_rng* rng, double* out, uint64_t* hits_out) {
  if (l >= g->L || r >= g->R || !bo_has_edge(g, l, r)) return BO_ARG;
  if (repeats == 0) return BO_ARG;
  uint64_t dl, dr;
  const uint32_t* la = nbr(g, 0, l, &dl);
  const uint32_t* ra = nbr(g, 1, r, &dr);
  uint64_t hits = 0;
  if (dl == 1 || dr == 1) {
    *out = 0.0;
    if (hits_out) *hits_out = 0;
    return BO_OK;
  }
  for (uint64_t t = 0; t < repeats; ++t) {
    uint32_t other_l = draw_excluding(ra, dr, l, rng);
    uint32_t other_r = draw_excluding(la, dl, r, rng);
    if (bo_has_edge(g, other_l, other_r)) ++hits;
  }
  if (hits_out) *hits_out = hits;
  *out = (double)hits / (double)repeats * (double)(dl - 1) * (double)(dr - 1);
  return BO_OK;
}

/* sampling.cpp:143-147 fast_esamp_iteration of Rng::stream(seed, index) */
int bo_fast_esamp_iteration(const bo_graph* g, uint64_t repeats, uint64_t seed, uint64_t index,
                            double* value, uint64_t* edge_id, uint64_t* hits) {
  bo_rng rng;
  bo_rng_stream(&rng, seed, index);
  uint64_t k = bo_rng_uniform_index(&rng, g->m);
  uint32_t l, r;
  int st = bo_edge_at(g, k, &l, &r);
  if (st) return st;
  double est;
  st = bo_fast_ebfc_estimate(g, l, r, repeats, &rng, &est, hits);
  if (st) return st;
  if (edge_id) *edge_id = k;
  *value = est * (double)g->m / 4.0;
  return BO_OK;
}

typedef struct {
  const bo_graph* g;
  const uint64_t* prefix;
  uint64_t total_wedges;
  int method;
  uint64_t seed;
  uint64_t repeats;
  double* values;
  scratch sc[MAX_THREADS];
} est_ctx;

static int est_body(par_ctx* c, int tid, uint64_t lo, uint64_t hi) {
  est_ctx* x = (est_ctx*)c->user;
  const bo_graph* g = x->g;
  if (!x->sc[tid].mult && scratch_init(&x->sc[tid], g)) return BO_INTERNAL;
  for (uint64_t i = lo; i < hi; ++i) {
    if (x->method == 3) {
      int st = bo_fast_esamp_iteration(g, x->repeats, x->seed, i, &x->values[i], NULL, NULL);
      if (st) return st;
      continue;
    }
    uint64_t id0;
    uint32_t a, b;
    int st = bo_sample_draw(g, x->prefix, x->total_wedges, x->method, x->seed, i, &id0, &a, &b);
    if (st) return st;
    uint64_t cnt;
    double scale;
    if (x->method == 0) {
      int side = id0 < g->L ? 0 : 1;
      st = per_vertex(g, side, (uint32_t)(side ? id0 - g->L : id0), &x->sc[tid], &cnt);
      scale = (double)((uint64_t)g->L + g->R);
    } else if (x->method == 1) {
      uint32_t l, r;
      st = bo_edge_at(g, id0, &l, &r);
      if (!st) st = per_edge(g, l, r, &x->sc[tid], &cnt);
      scale = (double)g->m;
    } else {
      int cs = id0 < g->L ? 0 : 1;
      uint64_t d;
      const uint32_t* adj = nbr(g, cs, (uint32_t)(cs ? id0 - g->L : id0), &d);
      st = bo_wedge_common_minus_1(g, cs, adj[a], adj[b], &cnt);
      scale = (double)x->total_wedges;
    }
    if (st) return st;
    x->values[i] = (double)cnt * scale / 4.0;
  }
  return BO_OK;
}

/* sampling.cpp:168-181 validate (fixed-iteration subset), 183-202 aggregate,
 * 243-278 fixed-count branch. */
int bo_run_estimator(const bo_graph* g, int method, uint64_t iterations, uint64_t seed,
                     uint64_t groups, uint64_t group_size, int threads, double* value,
                     uint64_t* iterations_done, double* per_group, double* values_out) {
  return bo_run_estimator_ex(g, method, iterations, seed, groups, group_size, 1000, threads,
                             value, iterations_done, per_group, values_out);
}

/* same, with EstimatorConfig::fast_edge_repeats (sampling.hpp:22) for method 3 = FastEdge */
int bo_run_estimator_ex(const bo_graph* g, int method, uint64_t iterations, uint64_t seed,
                        uint64_t groups, uint64_t group_size, uint64_t repeats, int threads,
                        double* value, uint64_t* iterations_done, double* per_group,
                        double* values_out) {
  if (method < 0 || method > 3) return BO_ARG;
  if (repeats == 0) return BO_ARG; /* sampling.cpp:178 (checked for every method) */
  int has_iters = iterations > 0 || (groups > 1 && group_size > 0);
  if (!has_iters) return BO_ARG;
  if (groups == 0) return BO_ARG;
  if (groups > 1 && groups % 2 == 0) return BO_ARG;
  if ((uint64_t)g->L + g->R == 0 || g->m == 0) return BO_ARG;
  uint64_t* prefix = NULL;
  uint64_t total_w = 0;
  if (method == 2) {
    prefix = (uint64_t*)malloc(((uint64_t)g->L + g->R + 1) * 8);
    if (!prefix) return BO_INTERNAL;
    int st = bo_build_wedge_index(g, prefix, &total_w);
    if (st) {
      free(prefix);
      return st;
    }
    if (total_w == 0) {
      free(prefix);
      return BO_NOWEDGE;
    }
  }
  uint64_t alpha = group_size > 0 ? group_size : iterations;
  uint64_t total;
  if (groups == 1) total = iterations;
  else if (__builtin_mul_overflow(groups, alpha, &total)) {
    free(prefix);
    return BO_OVERFLOW;
  }
  double* values = values_out ? values_out : (double*)malloc((total ? total : 1) * 8);
  if (threads > MAX_THREADS) threads = MAX_THREADS;
  est_ctx* x = (est_ctx*)calloc(1, sizeof(est_ctx));
  if (!values || !x) return BO_INTERNAL;
  x->g = g;
  x->prefix = prefix;
  x->total_wedges = total_w;
  x->method = method;
  x->seed = seed;
  x->repeats = repeats;
  x->values = values;
  int st = par_for(total, 64, threads, est_body, x);
  for (int t = 0; t < MAX_THREADS; ++t)
    if (x->sc[t].mult) scratch_free(&x->sc[t]);
  free(x);
  free(prefix);
  if (!st) {
    double sum = 0.0;
    for (uint64_t i = 0; i < total; ++i) sum += values[i]; /* sequential, index order */
    if (groups == 1) {
      *value = sum / (double)total;
    } else {
      uint64_t a = total / groups;
      double* means = (double*)malloc(groups * 8);
      for (uint64_t t = 0; t < groups; ++t) {
        double gs = 0.0;
        for (uint64_t i = t * a; i < (t + 1) * a; ++i) gs += values[i];
        means[t] = gs / (double)a;
        if (per_group) per_group[t] = means[t];
      }
      /* median_of: sort copy, take middle (sampling.cpp:45-48) */
      for (uint64_t i = 1; i < groups; ++i) {
        double v = means[i];
        uint64_t j = i;
        while (j > 0 && means[j - 1] > v) {
          means[j] = means[j - 1];
          --j;
        }
        means[j] = v;
      }
      *value = means[groups / 2];
      free(means);
    }
    *iterations_done = total;
  }
  if (!values_out) free(values);
  return st;
}

/* ------------------------------------------------------------------------ */
/* sparsify.cpp:15-24 count_retained: rebuild from external ids, exact count  */
int bo_count_retained(const bo_graph* g, const uint8_t* keep, int threads, uint64_t* count,
                      uint64_t* kept_edges) {
  uint64_t n = 0;
  for (uint64_t k = 0; k < g->m; ++k) n += keep[k] ? 1 : 0;
  if (kept_edges) *kept_edges = n;
  if (n == 0) {
    *count = 0;
    return BO_OK;
  }
  uint64_t* l = (uint64_t*)malloc(n * 8);
  uint64_t* r = (uint64_t*)malloc(n * 8);
  if (!l || !r) return BO_INTERNAL;
  uint64_t j = 0;
  for (uint32_t lv = 0; lv < g->L; ++lv)
    for (uint64_t k = g->loff[lv]; k < g->loff[lv + 1]; ++k)
      if (keep[k]) {
        l[j] = g->lids[lv];
        r[j] = g->rids[g->ladj[k]];
        ++j;
      }
  bo_graph h;
  int st = bo_graph_from_edges(&h, l, r, n);
  free(l);
  free(r);
  if (!st) st = bo_exact_count(&h, threads, count);
  bo_graph_free(&h);
  return st;
}

static int check_p(double p) { return (p > 0.0 && p <= 1.0) ? BO_OK : BO_ARG; }

/* sparsify.cpp:36-41 */
int bo_edge_sparsify_value(const bo_graph* g, const uint8_t* keep, double p, int threads,
                           double* out) {
  if (check_p(p)) return BO_ARG;
  double inv = 1.0 / p;
  uint64_t c;
  int st = bo_count_retained(g, keep, threads, &c, NULL);
  if (st) return st;
  *out = (double)c * inv * inv * inv * inv;
  return BO_OK;
}

/* sparsify.cpp:43-55 */
int bo_color_sparsify_value(const bo_graph* g, const uint32_t* colors, uint64_t n_colors,
                            int threads, double* out) {
  if (n_colors == 0) return BO_ARG;
  uint8_t* keep = (uint8_t*)malloc(g->m ? g->m : 1);
  if (!keep) return BO_INTERNAL;
  for (uint32_t lv = 0; lv < g->L; ++lv)
    for (uint64_t k = g->loff[lv]; k < g->loff[lv + 1]; ++k)
      keep[k] = colors[lv] == colors[(uint64_t)g->L + g->ladj[k]];
  uint64_t c;
  int st = bo_count_retained(g, keep, threads, &c, NULL);
  free(keep);
  if (st) return st;
  double n = (double)n_colors;
  *out = (double)c * n * n * n;
  return BO_OK;
}

/* sparsify.cpp:57-63 */
int bo_edge_sparsify_estimate(const bo_graph* g, double p, uint64_t seed, int threads,
                              double* out, uint64_t* count, uint64_t* kept_edges) {
  if (check_p(p)) return BO_ARG;
  uint8_t* keep = (uint8_t*)malloc(g->m ? g->m : 1);
  if (!keep) return BO_INTERNAL;
  for (uint64_t k = 0; k < g->m; ++k) keep[k] = bo_unit_double(bo_derive_seed(seed, k)) < p;
  uint64_t c;
  int st = bo_count_retained(g, keep, threads, &c, kept_edges);
  free(keep);
  if (st) return st;
  double inv = 1.0 / p;
  if (count) *count = c;
  *out = (double)c * inv * inv * inv * inv;
  return BO_OK;
}

/* sparsify.cpp:65-71 */
int bo_color_sparsify_estimate(const bo_graph* g, uint64_t n_colors, uint64_t seed, int threads,
                               double* out, uint64_t* count, uint64_t* kept_edges) {
  if (n_colors == 0) return BO_ARG;
  uint64_t n = (uint64_t)g->L + g->R;
  uint32_t* colors = (uint32_t*)malloc((n ? n : 1) * 4);
  uint8_t* keep = (uint8_t*)malloc(g->m ? g->m : 1);
  if (!colors || !keep) return BO_INTERNAL;
  for (uint64_t v = 0; v < n; ++v)
    colors[v] = (uint32_t)bo_bounded_from_bits(bo_derive_seed(seed, v), n_colors);
  for (uint32_t lv = 0; lv < g->L; ++lv)
    for (uint64_t k = g->loff[lv]; k < g->loff[lv + 1]; ++k)
      keep[k] = colors[lv] == colors[(uint64_t)g->L + g->ladj[k]];
  uint64_t c;
  int st = bo_count_retained(g, keep, threads, &c, kept_edges);
  free(colors);
  free(keep);
  if (st) return st;
  if (count) *count = c;
  double nn = (double)n_colors;
  *out = (double)c * nn * nn * nn;
  return BO_OK;
}

/* sparsify.cpp:73-94 */
int bo_sparsify_run(const bo_graph* g, int sparsifier, double p, uint64_t colors, uint64_t seed,
                    uint64_t trials, int threads, double* value, double* per_trial) {
  if (trials == 0) return BO_ARG;
  if (g->m == 0) return BO_ARG;
  double sum = 0.0;
  for (uint64_t t = 0; t < trials; ++t) {
    uint64_t ts = bo_derive_seed(seed, t);
    double v;
    int st = sparsifier == 0 ? bo_edge_sparsify_estimate(g, p, ts, threads, &v, NULL, NULL)
                             : bo_color_sparsify_estimate(g, colors, ts, threads, &v, NULL, NULL);
    if (st) return st;
    if (per_trial) per_trial[t] = v;
    sum += v;
  }
  *value = sum / (double)trials;
  return BO_OK;
}

/* oracle.cpp:37-58 brute force over left pairs (guard 64 per side) */
int bo_brute_force_count(const bo_graph* g, uint64_t* out) {
  if (g->L > 64 || g->R > 64) return BO_ARG; /* SizeGuardError */
  uint64_t total = 0;
  for (uint32_t a = 0; a < g->L; ++a)
    for (uint32_t b = a + 1; b < g->L; ++b) {
      uint64_t da, db;
      const uint32_t* na = nbr(g, 0, a, &da);
      const uint32_t* nb = nbr(g, 0, b, &db);
      uint64_t c2;
      if (bo_choose2(bo_intersection_size(na, da, nb, db), &c2)) return BO_OVERFLOW;
      if (__builtin_add_overflow(total, c2, &total)) return BO_OVERFLOW;
    }
  *out = total;
  return BO_OK;
}

/* ---- oracle.cpp:60-94 classify_pairs, oracle.cpp:96-116 variance_bounds -------------------
 * Pair types of two distinct butterflies by (shared vertices, shared edges): the reference
 * enumerates every butterfly {a<b | i<j} over left pairs (oracle.cpp:41-50) and classifies
 * all unordered pairs; shared edges = shared-left * shared-right (both are bicliques).
 * Guards as OracleGuards (oracle.hpp:15-18): BO_ARG when a side exceeds max_side or the
 * list exceeds max_butterflies (SizeGuardError in the reference). out[6] = bfly, p_0v, p_1v,
 * p_2v, p_1e, p_1w. */
typedef struct {
  uint32_t l[2], r[2];
} bo_bfly;

static uint32_t shared2(const uint32_t* a, const uint32_t* b) {
  return (uint32_t)(a[0] == b[0] || a[0] == b[1]) + (uint32_t)(a[1] == b[0] || a[1] == b[1]);
}

int bo_classify_pairs(const bo_graph* g, uint32_t max_side, uint64_t max_bfly, uint64_t* out) {
  if (g->L > max_side || g->R > max_side) return BO_ARG;
  uint64_t n = 0, cap = 64;
  bo_bfly* list = (bo_bfly*)malloc(cap * sizeof(bo_bfly));
  if (!list) return BO_INTERNAL;
  uint32_t* common = (uint32_t*)malloc(sizeof(uint32_t) * (g->R + 1));
  for (uint32_t a = 0; a < g->L; ++a)
    for (uint32_t b = a + 1; b < g->L; ++b) {
      uint64_t da, db, k = 0, i = 0, j = 0;
      const uint32_t* na = nbr(g, 0, a, &da);
      const uint32_t* nb = nbr(g, 0, b, &db);
      while (i < da && j < db) { /* std::set_intersection */
        if (na[i] < nb[j]) ++i;
        else if (nb[j] < na[i]) ++j;
        else {
          common[k++] = na[i];
          ++i;
          ++j;
        }
      }
      for (uint64_t x = 0; x < k; ++x)
        for (uint64_t y = x + 1; y < k; ++y) {
          if (n == cap) {
            cap *= 2;
            bo_bfly* t = (bo_bfly*)realloc(list, cap * sizeof(bo_bfly));
            if (!t) {
              free(list);
              free(common);
              return BO_INTERNAL;
            }
            list = t;
          }
          bo_bfly f = {{a, b}, {common[x], common[y]}};
          list[n++] = f;
        }
    }
  free(common);
  if (n > max_bfly) {
    free(list);
    return BO_ARG;
  }
  uint64_t c[6] = {n, 0, 0, 0, 0, 0};
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = i + 1; j < n; ++j) {
      const uint32_t sl = shared2(list[i].l, list[j].l), sr = shared2(list[i].r, list[j].r);
      const uint32_t sv = sl + sr, se = sl * sr;
      if (sv == 0) ++c[1];
      else if (sv == 1) ++c[2];
      else if (sv == 2 && se == 0) ++c[3];
      else if (sv == 2 && se == 1) ++c[4];
      else if (sv == 3 && se == 2) ++c[5];
      else {
        free(list);
        return BO_INTERNAL; /* InternalError: impossible pair */
      }
    }
  free(list);
  memcpy(out, c, sizeof(c));
  return BO_OK;
}

/* out[5] = vsamp, esamp, wsamp, espar, clrspar (oracle.cpp:96-116; same operation order) */
int bo_variance_bounds(uint64_t n_v, uint64_t m, uint64_t wedges, const uint64_t* counts,
                       double p, double* out) {
  if (!(p > 0.0 && p <= 1.0)) return BO_ARG;
  const double bfly = (double)counts[0], n = (double)n_v, mm = (double)m, w = (double)wedges;
  const uint64_t pV = counts[2] + counts[3] + counts[4] + counts[5], pE = counts[4] + counts[5];
  out[0] = n * (bfly + (double)pV) / 4.0;
  out[1] = mm * (bfly + (double)pE) / 4.0;
  out[2] = w * (bfly + (double)counts[5]) / 4.0;
  const double inv = 1.0 / p, p1w2 = 2.0 * (double)counts[5], p1e2 = 2.0 * (double)counts[4],
               p2v2 = 2.0 * (double)counts[3];
  out[3] = bfly * inv * inv * inv * inv + p1w2 * inv * inv + p1e2 * inv;
  out[4] = bfly * inv * inv * inv + p1w2 * inv * inv + (p1e2 + p2v2) * inv;
  return BO_OK;
}

/* Independent checker for the GPU's identity-based pair counts at sizes the enumeration
 * cannot reach: the same five counts from per-pair common-neighbour counts c (all
 * same-side pairs, sorted-merge intersections: O(side^2 * degree)) and the all-subject
 * local counts, in 128-bit arithmetic. out[11] = bfly, then (lo, hi) words of p_0v, p_1v,
 * p_2v, p_1e, p_1w. */
int bo_pair_counts_by_moments(const bo_graph* g, int threads, uint64_t* out) {
  typedef unsigned __int128 u128;
  u128 s2 = 0, s3 = 0, s4 = 0;
  for (int side = 0; side < 2; ++side) {
    const uint32_t cnt = side == 0 ? g->L : g->R;
    for (uint32_t a = 0; a < cnt; ++a) {
      uint64_t da;
      const uint32_t* na = nbr(g, side, a, &da);
      for (uint32_t b = a + 1; b < cnt; ++b) {
        uint64_t db;
        const uint32_t* nb = nbr(g, side, b, &db);
        const u128 c = bo_intersection_size(na, da, nb, db);
        if (c >= 2) s2 += c * (c - 1) / 2;
        if (c >= 3) s3 += c * (c - 1) * (c - 2) / 6;
        if (c >= 4) s4 += c * (c - 1) * (c - 2) * (c - 3) / 24;
      }
    }
  }
  const uint64_t n = (uint64_t)g->L + g->R;
  uint64_t* lv = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  uint64_t* le = (uint64_t*)malloc(sizeof(uint64_t) * (g->m ? g->m : 1));
  if (!lv || !le) {
    free(lv);
    free(le);
    return BO_INTERNAL;
  }
  int st = bo_count_all_vertices(g, threads, lv);
  if (st == BO_OK) st = bo_count_all_edges(g, threads, le);
  u128 v2 = 0, e2 = 0;
  for (uint64_t i = 0; st == BO_OK && i < n; ++i) v2 += (u128)lv[i] * (lv[i] ? lv[i] - 1 : 0) / 2;
  for (uint64_t i = 0; st == BO_OK && i < g->m; ++i) e2 += (u128)le[i] * (le[i] ? le[i] - 1 : 0) / 2;
  free(lv);
  free(le);
  if (st != BO_OK) return st;
  if (s2 % 2) return BO_INTERNAL;
  const u128 b = s2 / 2, p1w = 3 * s3, p2v = 3 * s4;
  if (e2 < 2 * p1w) return BO_INTERNAL;
  const u128 p1e = e2 - 2 * p1w, sh = 2 * p2v + 2 * p1e + 3 * p1w;
  if (v2 < sh) return BO_INTERNAL;
  const u128 p1v = v2 - sh, all = b * (b ? b - 1 : 0) / 2, t = p1v + p2v + p1e + p1w;
  if (all < t || (b >> 64)) return BO_INTERNAL;
  const u128 v[5] = {all - t, p1v, p2v, p1e, p1w};
  out[0] = (uint64_t)b;
  for (int q = 0; q < 5; ++q) {
    out[1 + 2 * q] = (uint64_t)v[q];
    out[2 + 2 * q] = (uint64_t)(v[q] >> 64);
  }
  return BO_OK;
}
