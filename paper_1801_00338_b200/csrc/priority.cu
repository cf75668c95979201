// priority.cu -- degree-priority relabelling and the wedge plan of the exact kernels.
//
// Every vertex of both sides gets a priority id p: degree descending, ties by global index
// ascending (a strict total order). The merged-side CSR lists neighbours in ascending p.
// A butterfly is counted once, at its highest-priority vertex u ("start"): wedges
// (u, v, w) with v > u and w > u in priority order. The reference anchors at every vertex
// of one side and walks w < v in dense-id order (exact.cpp:29-41); both enumerate every
// butterfly exactly once, so the uint64 totals are identical.
//
// Build (no per-list sort):  the sequence of (src = rank[x], dst = p) entries is emitted in
// dst-major order (segment of dst p at poff[p]); a STABLE radix sort by src then yields
// every src list already ascending in dst.
#include "cubwrap.cuh"
#include "graph.cuh"

namespace bflyd {
namespace {

__global__ void k_degkeys(const uint64_t* __restrict__ loff, const uint64_t* __restrict__ roff,
                          uint32_t L, uint32_t R, uint32_t* __restrict__ key,
                          uint32_t* __restrict__ gid) {
  uint64_t n = uint64_t{L} + R;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t d = g < L ? loff[g + 1] - loff[g] : roff[g - L + 1] - roff[g - L];
    key[g] = 0xFFFFFFFFu - static_cast<uint32_t>(d);
    gid[g] = static_cast<uint32_t>(g);
  }
}

__global__ void k_rank(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ inv,
                       uint64_t n, uint32_t* __restrict__ rank, uint64_t* __restrict__ pdeg) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p <= n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    if (p == n) {
      pdeg[n] = 0;
    } else {
      rank[inv[p]] = static_cast<uint32_t>(p);
      pdeg[p] = 0xFFFFFFFFu - skey[p];
    }
  }
}

// mark[off[r]] = r for every row with entries (rows are never empty in canonical CSRs)
__global__ void k_mark_rows(const uint64_t* __restrict__ off, uint32_t rows,
                            uint32_t* __restrict__ mark) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    if (off[r + 1] > off[r]) mark[off[r]] = static_cast<uint32_t>(r);
}

// side 0: left CSR entries (dst = left row l, src = right col); side 1: right CSR entries.
template <bool EID>
__global__ void k_fill(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                       const uint32_t* __restrict__ rowof, const uint32_t* __restrict__ eid_of,
                       uint64_t m, uint32_t row_base, uint32_t col_base,
                       const uint32_t* __restrict__ rank, const uint64_t* __restrict__ poff,
                       uint32_t* __restrict__ seq_src, uint64_t* __restrict__ seq_val,
                       uint32_t* __restrict__ seq_val32) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t row = rowof[k];
    uint32_t p = rank[row_base + row];
    uint64_t slot = poff[p] + (k - off[row]);
    seq_src[slot] = rank[col_base + adj[k]];
    if (EID) {
      uint32_t e = eid_of ? eid_of[k] : static_cast<uint32_t>(k);
      seq_val[slot] = static_cast<uint64_t>(p) | (static_cast<uint64_t>(e) << 32);
    } else {
      seq_val32[slot] = p;
    }
  }
}

__global__ void k_unpack(const uint64_t* __restrict__ v, uint64_t n, uint32_t* __restrict__ adj,
                         uint32_t* __restrict__ eid) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = v[i];
    adj[i] = static_cast<uint32_t>(x);
    eid[i] = static_cast<uint32_t>(x >> 32);
  }
}

__global__ void k_fwd_init(const uint64_t* __restrict__ poff, uint64_t n,
                           uint64_t* __restrict__ fwd, uint64_t* __restrict__ work) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    fwd[u] = poff[u + 1];
    work[u] = 0;
  }
}

// One thread per directed entry e = (u -> v). Forward entries (v > u) locate u inside the
// ascending list N(v) by binary search; the wedge suffix is N(v) after u.
__global__ void k_plan(const uint64_t* __restrict__ poff, const uint32_t* __restrict__ padj,
                       const uint32_t* __restrict__ psrc, uint64_t nnz,
                       uint2* __restrict__ fseg, uint64_t* __restrict__ fwd,
                       unsigned long long* __restrict__ work) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t stride = ((uint64_t)gridDim.x * blockDim.x) & ~31ull;
  for (uint64_t base = warp * 32; base < nnz; base += stride) {
    const uint64_t e = base + lane;
    bool valid = e < nnz;
    uint32_t u = valid ? psrc[e] : 0xFFFFFFFFu;
    unsigned long long wk = 0;
    if (valid) {
      uint32_t v = padj[e];
      if (v > u) {
        uint64_t lo = poff[v], hi = poff[v + 1], end = hi;
        while (lo < hi) {
          uint64_t mid = (lo + hi) >> 1;
          if (padj[mid] < u) lo = mid + 1;
          else hi = mid;
        }
        wk = end - lo - 1;
        // wedge suffix of N(v) after u: absolute start and length (m < 2^31: fits u32)
        fseg[e] = make_uint2(static_cast<uint32_t>(lo + 1), static_cast<uint32_t>(wk));
        if (e == poff[u] || padj[e - 1] < u) fwd[u] = e;
      }  // backward entries keep no suffix: nothing reads fseg there
    }
    // warp-segmented sum of wk over runs of equal u, one atomic per run
    unsigned full = 0xffffffffu;
    uint32_t up = __shfl_up_sync(full, u, 1);
    bool head = lane == 0 || up != u;
    unsigned heads = __ballot_sync(full, head);
    int my_head = 31 - __clz(heads & ((2u << lane) - 1u));
    for (int off = 1; off < 32; off <<= 1) {
      unsigned long long y = __shfl_up_sync(full, wk, off);
      if ((int)lane - off >= my_head) wk += y;
    }
    uint32_t dn = __shfl_down_sync(full, u, 1);
    bool tail = lane == 31 || dn != u;
    if (valid && tail && wk) atomicAdd(&work[u], wk);
  }
}

}  // namespace

void ensure_priority(bfly_graph* g, bool with_eid) {
  if (g->prio_ready && (!with_eid || g->prio_has_eid)) return;
  cudaStream_t s = g->stream;
  const uint64_t n = g->n(), nnz = 2 * g->m;
  g->prio_ready = false;
  g->hub_ready = false;  // the hub plan indexes priority-CSR entries
  if (n == 0) {
    g->poff.alloc(1, s);
    g->poff.zero();
    g->rank.alloc(1, s);
    g->inv.alloc(1, s);
    g->padj.alloc(1, s);
    g->psrc.alloc(1, s);
    g->fseg.alloc(1, s);
    g->work.alloc(1, s);
    g->fwd.alloc(1, s);
    g->total_work = 0;
    g->prio_ready = true;
    g->prio_has_eid = with_eid;
    return;
  }
  // 1. priority order: degree descending, ties by global id (stable sort of ~degree)
  {
    DBuf<uint32_t> key(n, s), gid(n, s), skey(n, s);
    launch("prio_degkeys", k_degkeys, grid_for(n, 256), 256, 0, s, g->loff.p, g->roff.p, g->L,
           g->R, key.p, gid.p);
    g->inv.alloc(n, s);
    sort_pairs(key.p, skey.p, gid.p, g->inv.p, n, 0, 32, s, "sort_priority_order");
    g->rank.alloc(n, s);
    DBuf<uint64_t> pdeg(n + 1, s);
    launch("prio_rank", k_rank, grid_for(n + 1, 256), 256, 0, s, skey.p, g->inv.p, n, g->rank.p,
           pdeg.p);
    g->poff.alloc(n + 1, s);
    exclusive_sum(pdeg.p, g->poff.p, n + 1, s);
  }
  // 2. dst-major entry sequence, then stable sort by src
  {
    DBuf<uint32_t> seq_src(nnz, s), lrow_tmp, rrow_tmp;
    // rows of the CSR entries: kept from the build, else rebuilt (mark row starts + max-scan)
    const uint32_t* lrow = g->lrow.p;
    const uint32_t* rrow = g->rrow.p;
    auto rows = [&](const uint64_t* off, uint32_t nrows, DBuf<uint32_t>& out) {
      DBuf<uint32_t> mark(g->m, s);
      mark.zero();
      out.alloc(g->m, s);
      launch("prio_mark_rows", k_mark_rows, grid_for(nrows, 256), 256, 0, s, off, nrows, mark.p);
      inclusive_max(mark.p, out.p, g->m, s);
    };
    if (!lrow) {
      rows(g->loff.p, g->L, lrow_tmp);
      lrow = lrow_tmp.p;
    }
    if (!rrow) {
      rows(g->roff.p, g->R, rrow_tmp);
      rrow = rrow_tmp.p;
    }
    int nb = bits_for(n - 1);
    if (nb == 0) nb = 1;
    g->psrc.alloc(nnz, s);
    g->padj.alloc(nnz, s);
    if (with_eid) {
      DBuf<uint64_t> val(nnz, s), sval(nnz, s);
      launch("prio_fill", k_fill<true>, grid_for(g->m, 256), 256, 0, s, g->loff.p, g->ladj.p,
             lrow, (const uint32_t*)nullptr, g->m, 0u, g->L, g->rank.p, g->poff.p, seq_src.p,
             val.p, (uint32_t*)nullptr);
      launch("prio_fill", k_fill<true>, grid_for(g->m, 256), 256, 0, s, g->roff.p, g->radj.p,
             rrow, g->reid.p, g->m, g->L, 0u, g->rank.p, g->poff.p, seq_src.p, val.p,
             (uint32_t*)nullptr);
      lrow_tmp.release();
      rrow_tmp.release();
      sort_pairs(seq_src.p, g->psrc.p, val.p, sval.p, nnz, 0, nb, s, "sort_priority_csr");
      g->peid.alloc(nnz, s);
      launch("prio_unpack", k_unpack, grid_for(nnz, 256), 256, 0, s, sval.p, nnz, g->padj.p,
             g->peid.p);
    } else {
      DBuf<uint32_t> val(nnz, s);
      launch("prio_fill", k_fill<false>, grid_for(g->m, 256), 256, 0, s, g->loff.p, g->ladj.p,
             lrow, (const uint32_t*)nullptr, g->m, 0u, g->L, g->rank.p, g->poff.p, seq_src.p,
             (uint64_t*)nullptr, val.p);
      launch("prio_fill", k_fill<false>, grid_for(g->m, 256), 256, 0, s, g->roff.p, g->radj.p,
             rrow, g->reid.p, g->m, g->L, 0u, g->rank.p, g->poff.p, seq_src.p,
             (uint64_t*)nullptr, val.p);
      lrow_tmp.release();
      rrow_tmp.release();
      sort_pairs(seq_src.p, g->psrc.p, val.p, g->padj.p, nnz, 0, nb, s, "sort_priority_csr");
    }
  }
  // 3. wedge plan: suffix positions, first forward entry, work per start
  g->fseg.alloc(nnz, s);
  g->fwd.alloc(n, s);
  g->work.alloc(n, s);
  launch("prio_fwd_init", k_fwd_init, grid_for(n, 256), 256, 0, s, g->poff.p, n, g->fwd.p,
         g->work.p);
  launch("prio_plan", k_plan, grid_for(nnz, 256, 148u * 64u), 256, 0, s, g->poff.p, g->padj.p,
         g->psrc.p, nnz, g->fseg.p, g->fwd.p, reinterpret_cast<unsigned long long*>(g->work.p));
  trace_mark("priority csr + plan (queued)");
  g->prio_ready = true;
  g->prio_has_eid = with_eid;
}

}  // namespace bflyd
