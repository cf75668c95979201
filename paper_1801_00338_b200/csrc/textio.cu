// textio.cu -- edge-list text ingestion and serialisation on the device:
// load_edge_list (graph.cpp:75-99) and serialize_edge_list (graph.cpp:107-112).
//
// Parse: the text goes to the GPU in chunks of at most 1 GiB split after a newline. Per chunk
// a flag pass marks line starts, a scan numbers the lines, and one thread per line applies
// the reference's rules: a line whose first byte outside " \t\r" is absent, '%' or '#' is
// skipped; otherwise two whitespace-separated tokens (isspace) must each be a complete
// decimal uint64 (std::from_chars: digits only, overflow is an error); further tokens are
// ignored. Edges are compacted in line order, so the edge list -- and therefore the
// first-seen vertex numbering -- equals the reference's. The first malformed line (lowest
// line number, where the reference stops) is reported; its message is rebuilt on the host
// from that one line.
//
// Serialise: "% bip\n", then "lid rid\n" per canonical edge (left CSR order, external ids):
// per-edge byte lengths, a scan, and one thread per edge writing its digits.
#include <cstring>
#include <string>

#include "cubwrap.cuh"
#include "graph.cuh"
#include "local.cuh"

namespace bflyd {
namespace {

__device__ __forceinline__ bool lead_blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }
__device__ __forceinline__ bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

__global__ void k_line_flags(const char* __restrict__ t, uint64_t len, uint32_t* __restrict__ f) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
       i += (uint64_t)gridDim.x * blockDim.x)
    f[i] = (i == 0 || t[i - 1] == '\n') ? 1u : 0u;
}

__global__ void k_line_starts(const uint32_t* __restrict__ f, const uint32_t* __restrict__ idx,
                              uint64_t len, uint32_t* __restrict__ starts) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (f[i]) starts[idx[i]] = static_cast<uint32_t>(i);
}

// status per line: 0 skipped, 1 edge, 2 malformed
__global__ void k_parse_lines(const char* __restrict__ t, uint64_t len,
                              const uint32_t* __restrict__ starts, uint32_t nlines,
                              uint64_t* __restrict__ ol, uint64_t* __restrict__ orr,
                              uint32_t* __restrict__ edge_flag,
                              unsigned long long* __restrict__ first_err) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x) {
    const uint32_t a = starts[j];
    uint32_t b = j + 1 < nlines ? starts[j + 1] : static_cast<uint32_t>(len);
    if (b > a && t[b - 1] == '\n') --b;
    uint32_t p = a;
    while (p < b && lead_blank(t[p])) ++p;
    edge_flag[j] = 0;
    if (p == b || t[p] == '%' || t[p] == '#') continue;  // graph.cpp:81-83
    uint64_t ids[2] = {0, 0};
    bool ok = true;
    uint32_t q = a;
    for (int k = 0; k < 2 && ok; ++k) {  // graph.cpp:86-94
      while (q < b && is_space(t[q])) ++q;
      if (q == b) {
        ok = false;
        break;
      }
      uint64_t v = 0;
      for (; q < b && !is_space(t[q]); ++q) {
        const int d = t[q] - '0';
        if (d < 0 || d > 9 || v > (~0ull - d) / 10) {
          ok = false;
          break;
        }
        v = v * 10 + d;
      }
      ids[k] = v;
    }
    if (!ok) {
      atomicMin(first_err, (unsigned long long)j);
      continue;
    }
    ol[j] = ids[0];
    orr[j] = ids[1];
    edge_flag[j] = 1;
  }
}

__global__ void k_compact_edges(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                const uint64_t* __restrict__ ol, const uint64_t* __restrict__ orr,
                                uint32_t nlines, uint64_t base, uint64_t* __restrict__ dl,
                                uint64_t* __restrict__ dr) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x)
    if (flag[j]) {
      dl[base + pos[j]] = ol[j];
      dr[base + pos[j]] = orr[j];
    }
}

__device__ __forceinline__ uint32_t digits(uint64_t x) {
  uint32_t d = 1;
  while (x >= 10) {
    x /= 10;
    ++d;
  }
  return d;
}

__device__ __forceinline__ void put_u64(char* out, uint64_t x, uint32_t nd) {
  for (uint32_t i = nd; i-- > 0;) {
    out[i] = static_cast<char>('0' + x % 10);
    x /= 10;
  }
}

__global__ void k_mark_rows(const uint64_t* __restrict__ off, uint32_t rows,
                            uint32_t* __restrict__ mark) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    if (off[r + 1] > off[r]) mark[off[r]] = static_cast<uint32_t>(r);
}

__global__ void k_edge_text_len(const uint32_t* __restrict__ rowof, const uint32_t* __restrict__ ladj,
                                const uint64_t* __restrict__ lids, const uint64_t* __restrict__ rids,
                                uint64_t m, unsigned long long* __restrict__ lenk) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x)
    lenk[k] = digits(lids[rowof[k]]) + 1 + digits(rids[ladj[k]]) + 1;
}

__global__ void k_edge_text(const uint32_t* __restrict__ rowof, const uint32_t* __restrict__ ladj,
                            const uint64_t* __restrict__ lids, const uint64_t* __restrict__ rids,
                            uint64_t m, const unsigned long long* __restrict__ off, uint64_t head,
                            char* __restrict__ out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x) {
    char* o = out + head + off[k];
    const uint64_t a = lids[rowof[k]], b = rids[ladj[k]];
    const uint32_t da = digits(a), db = digits(b);
    put_u64(o, a, da);
    o[da] = ' ';
    put_u64(o + da + 1, b, db);
    o[da + 1 + db] = '\n';
  }
}

}  // namespace

// The reference's message for one malformed line (graph.cpp:86-94), without the line suffix.
std::string parse_error_message(const char* line, size_t n) {
  auto sp = [](char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
  };
  size_t q = 0;
  for (int k = 0; k < 2; ++k) {
    while (q < n && sp(line[q])) ++q;
    if (q == n) return "expected two vertex ids, got " + std::to_string(k);
    const size_t s0 = q;
    while (q < n && !sp(line[q])) ++q;
    bool ok = true;
    uint64_t v = 0;
    for (size_t i = s0; i < q && ok; ++i) {
      const int d = line[i] - '0';
      if (d < 0 || d > 9 || v > (~0ull - d) / 10) ok = false;
      else v = v * 10 + d;
    }
    if (!ok) return "bad vertex id '" + std::string(line + s0, q - s0) + "'";
  }
  return "malformed line";
}

// Parses `len` bytes into device edge arrays (grown as needed). Returns the edge count;
// *err_line = 1-based number of the first malformed line, 0 when there is none.
uint64_t parse_text_device(cudaStream_t s, const char* text, uint64_t len,
                           DBuf<uint64_t>& dl, DBuf<uint64_t>& dr, uint64_t* err_line) {
  constexpr uint64_t kChunk = 1ull << 30;
  uint64_t edges = 0, cap = 0, line0 = 0;
  *err_line = 0;
  DBuf<unsigned long long> ferr(1, s);
  DBuf<unsigned long long> cnt(1, s);
  for (uint64_t c0 = 0; c0 < len;) {
    uint64_t c1 = std::min(len, c0 + kChunk);
    if (c1 < len) {  // end the chunk after its last newline
      const void* nl = nullptr;
      for (uint64_t back = c1; back > c0 && !nl; --back)
        if (text[back - 1] == '\n') nl = text + back - 1;
      if (nl) c1 = static_cast<const char*>(nl) - text + 1;
      else {
        const void* fwd = std::memchr(text + c1, '\n', len - c1);
        c1 = fwd ? static_cast<const char*>(fwd) - text + 1 : len;
      }
      if (c1 - c0 >= (1ull << 31)) fail(kArgument, "edge-list line longer than 2 GiB");
    }
    const uint64_t n = c1 - c0;
    DBuf<char> dt(n, s);
    BFLY_CUDA(cudaMemcpyAsync(dt.p, text + c0, n, cudaMemcpyHostToDevice, s));
    DBuf<uint32_t> flag(n, s), idx(n, s);
    launch("text_line_flags", k_line_flags, grid_for(n, 256), 256, 0, s, dt.p, n, flag.p);
    exclusive_sum(flag.p, idx.p, n, s);
    uint32_t hl[2];
    BFLY_CUDA(cudaMemcpyAsync(&hl[0], idx.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaMemcpyAsync(&hl[1], flag.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
    const uint32_t nlines = hl[0] + hl[1];
    DBuf<uint32_t> starts(nlines, s), eflag(nlines, s), pos(nlines, s);
    DBuf<uint64_t> ol(nlines, s), orr(nlines, s);
    launch("text_line_starts", k_line_starts, grid_for(n, 256), 256, 0, s, flag.p, idx.p, n,
           starts.p);
    const unsigned long long none = ~0ull;
    BFLY_CUDA(cudaMemcpyAsync(ferr.p, &none, 8, cudaMemcpyHostToDevice, s));
    launch("text_parse_lines", k_parse_lines, grid_for(nlines, 256), 256, 0, s, dt.p, n, starts.p,
           nlines, ol.p, orr.p, eflag.p, ferr.p);
    exclusive_sum(eflag.p, pos.p, nlines, s);
    unsigned long long fe = 0;
    uint32_t hp[2];
    BFLY_CUDA(cudaMemcpyAsync(&fe, ferr.p, 8, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaMemcpyAsync(&hp[0], pos.p + nlines - 1, 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaMemcpyAsync(&hp[1], eflag.p + nlines - 1, 4, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
    if (fe != ~0ull) {
      *err_line = line0 + fe + 1;
      uint32_t ab[2];
      BFLY_CUDA(cudaMemcpyAsync(ab, starts.p + fe, (fe + 1 < nlines ? 8 : 4),
                                cudaMemcpyDeviceToHost, s));
      BFLY_CUDA(cudaStreamSynchronize(s));
      const uint64_t a = ab[0], b = fe + 1 < nlines ? ab[1] : n;
      std::string msg = parse_error_message(text + c0 + a, b - a);
      fail(kParse, msg + " (line " + std::to_string(*err_line) + ")");
    }
    const uint64_t ne = uint64_t{hp[0]} + hp[1];
    if (edges + ne > cap) {  // grow (geometric) the device edge arrays
      const uint64_t ncap = std::max<uint64_t>(edges + ne, cap * 2);
      DBuf<uint64_t> nl2(ncap, s), nr2(ncap, s);
      if (edges) {
        BFLY_CUDA(cudaMemcpyAsync(nl2.p, dl.p, edges * 8, cudaMemcpyDeviceToDevice, s));
        BFLY_CUDA(cudaMemcpyAsync(nr2.p, dr.p, edges * 8, cudaMemcpyDeviceToDevice, s));
      }
      dl = std::move(nl2);
      dr = std::move(nr2);
      cap = ncap;
    }
    if (ne)
      launch("text_compact_edges", k_compact_edges, grid_for(nlines, 256), 256, 0, s, eflag.p,
             pos.p, ol.p, orr.p, nlines, edges, dl.p, dr.p);
    edges += ne;
    line0 += nlines;
    c0 = c1;
  }
  return edges;
}

// Bytes of serialize_edge_list(g); writes them to host `out` when it is non-null.
uint64_t serialize_device(bfly_graph* g, char* out) {
  static const char kHead[] = "% bip\n";
  const uint64_t head = sizeof(kHead) - 1;
  cudaStream_t s = g->stream;
  const uint64_t m = g->m;
  if (m == 0) {
    if (out) std::memcpy(out, kHead, head);
    return head;
  }
  DBuf<uint32_t> rowof_tmp;
  const uint32_t* rowof = g->lrow.p;  // left row of each canonical edge, from the build
  if (!rowof) {
    DBuf<uint32_t> mark(m, s);
    rowof_tmp.alloc(m, s);
    mark.zero();
    launch("text_mark_rows", k_mark_rows, grid_for(g->L, 256), 256, 0, s, g->loff.p, g->L,
           mark.p);
    inclusive_max(mark.p, rowof_tmp.p, m, s);
    rowof = rowof_tmp.p;
  }
  DBuf<unsigned long long> lenk(m, s), off(m, s);
  launch("text_edge_len", k_edge_text_len, grid_for(m, 256), 256, 0, s, rowof, g->ladj.p,
         g->lids.p, g->rids.p, m, lenk.p);
  exclusive_sum(lenk.p, off.p, m, s);
  unsigned long long tail[2];
  BFLY_CUDA(cudaMemcpyAsync(&tail[0], off.p + m - 1, 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaMemcpyAsync(&tail[1], lenk.p + m - 1, 8, cudaMemcpyDeviceToHost, s));
  BFLY_CUDA(cudaStreamSynchronize(s));
  const uint64_t total = head + tail[0] + tail[1];
  if (out) {
    DBuf<char> dt(total, s);
    BFLY_CUDA(cudaMemcpyAsync(dt.p, kHead, head, cudaMemcpyHostToDevice, s));
    launch("text_edge_write", k_edge_text, grid_for(m, 256), 256, 0, s, rowof, g->ladj.p,
           g->lids.p, g->rids.p, m, off.p, head, dt.p);
    BFLY_CUDA(cudaMemcpyAsync(out, dt.p, total, cudaMemcpyDeviceToHost, s));
    BFLY_CUDA(cudaStreamSynchronize(s));
  }
  return total;
}

}  // namespace bflyd
