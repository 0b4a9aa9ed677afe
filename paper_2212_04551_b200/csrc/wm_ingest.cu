// wm_ingest.cu — graph ingest on the device: the step before the hot path.
//
// Reference: CsrGraph construction (pkg/src/warpmine/graph.py:44-78:
// symmetrise, drop self-loops and duplicates, rows strictly ascending) and the
// edge-list reader (graph.py:139-188: '#'/'%' comments and blank lines
// skipped, exactly two integer tokens per line, negative ids rejected, ids
// remapped to 0..n-1 in ascending order).  The reference builds Python tuples
// (`sorted(set(pairs))`), minutes at R-MAT scale 22; here both steps are
// data-parallel passes over HBM:
//
//   text bytes --(newline select, one thread per line)--> (u, v) + status
//   ids --(radix sort, unique, binary search)--> dense 0..n-1
//   (u, v) --(u64 key (min<<32|max), radix sort, unique)--> undirected edges
//   --(both directions, radix sort)--> rows ascending --(row histogram, scan)--> CSR
//
// Output is bit-identical to the host construction (tests/test_gpu_ingest.py).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "wm_common.cuh"

namespace wm {

namespace {

struct DevMem {
  void *p = nullptr;
  ~DevMem() { if (p) cudaFree(p); }
  template <typename T> T *as() const { return static_cast<T *>(p); }
};

#define WM_DALLOC(mem, bytes) WM_CUDA(cudaMalloc(&(mem).p, (bytes) > 0 ? (bytes) : 16))

constexpr unsigned long long kNoEdge = ~0ull;

// undirected key of each endpoint pair; self-loops map to kNoEdge
__global__ void edge_keys_kernel(int64_t m, const int64_t *__restrict__ src,
                                 const int64_t *__restrict__ dst, int64_t n,
                                 unsigned long long *__restrict__ keys, int *__restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = src[i], v = dst[i];
    if (u < 0 || v < 0 || u >= n || v >= n) {
      atomicExch(bad, 1);
      keys[i] = kNoEdge;
      continue;
    }
    const int64_t lo = u < v ? u : v, hi = u < v ? v : u;
    keys[i] = (u == v) ? kNoEdge : (((unsigned long long)lo << 32) | (unsigned long long)hi);
  }
}

// both directions of every unique undirected edge
__global__ void expand_kernel(int64_t e, const unsigned long long *__restrict__ und,
                              unsigned long long *__restrict__ dir) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = und[i];
    dir[2 * i] = k;
    dir[2 * i + 1] = (k << 32) | (k >> 32);
  }
}

__global__ void split_kernel(int64_t nnz, const unsigned long long *__restrict__ dir,
                             int32_t *__restrict__ nbr, int64_t *__restrict__ deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = dir[i];
    nbr[i] = (int32_t)(k & 0xffffffffull);
    atomicAdd(reinterpret_cast<unsigned long long *>(deg + (k >> 32)), 1ull);
  }
}

int grid_for(const Workspace *ws, int64_t items) {
  const int64_t b = (items + 255) / 256;
  const int64_t cap = (int64_t)ws->num_sms * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 32 && (1ll << b) < n) ++b;
  return b;
}

// Device endpoints -> CSR on the host (out->offsets / out->neighbors malloc'd).
int csr_from_device_pairs(Workspace *ws, int64_t n, const int64_t *d_src, const int64_t *d_dst,
                          int64_t m, wm_csr_out *out, cudaStream_t s) {
  DevMem keys, keys2, und, dir, dir2, nbr, deg, off, tmp, cnt, bad;
  WM_DALLOC(keys, sizeof(unsigned long long) * m);
  WM_DALLOC(keys2, sizeof(unsigned long long) * m);
  WM_DALLOC(cnt, sizeof(int64_t) * 2);
  WM_DALLOC(bad, sizeof(int));
  WM_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
  if (m > 0)
    edge_keys_kernel<<<grid_for(ws, m), 256, 0, s>>>(m, d_src, d_dst, n, keys.as<unsigned long long>(),
                                                      bad.as<int>());
  WM_CUDA(cudaGetLastError());
  const int vb = bits_for(n);
  // sort + unique the undirected keys (kNoEdge sorts last)
  size_t t1 = 0, t2 = 0, t3 = 0;
  WM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys.as<unsigned long long>(),
                                         keys2.as<unsigned long long>(), m, 0, 64, s));
  WM_CUDA(cub::DeviceSelect::Unique(nullptr, t2, keys2.as<unsigned long long>(),
                                    keys.as<unsigned long long>(), cnt.as<int64_t>(), m, s));
  WM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t3, keys.as<unsigned long long>(),
                                         keys2.as<unsigned long long>(), 2 * m, 0, 32 + vb, s));
  size_t tb = t1 > t2 ? t1 : t2;
  if (t3 > tb) tb = t3;
  WM_DALLOC(tmp, tb);
  size_t t = tb;
  WM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t, keys.as<unsigned long long>(),
                                         keys2.as<unsigned long long>(), m, 0, 64, s));
  t = tb;
  WM_CUDA(cub::DeviceSelect::Unique(tmp.p, t, keys2.as<unsigned long long>(),
                                    keys.as<unsigned long long>(), cnt.as<int64_t>(), m, s));
  int64_t e = 0;
  int hbad = 0;
  WM_CUDA(cudaMemcpyAsync(&e, cnt.p, sizeof e, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof hbad, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  if (hbad) return fail(WM_EINVAL, "edge endpoint outside vertex range 0..%lld", (long long)n - 1);
  if (e > 0) {
    unsigned long long last = 0;
    WM_CUDA(cudaMemcpy(&last, keys.as<unsigned long long>() + e - 1, sizeof last,
                       cudaMemcpyDeviceToHost));
    if (last == kNoEdge) --e;
  }
  const int64_t nnz = 2 * e;
  WM_DALLOC(dir, sizeof(unsigned long long) * nnz);
  WM_DALLOC(dir2, sizeof(unsigned long long) * nnz);
  WM_DALLOC(nbr, sizeof(int32_t) * nnz);
  WM_DALLOC(deg, sizeof(int64_t) * (n + 1));
  WM_DALLOC(off, sizeof(int64_t) * (n + 1));
  WM_CUDA(cudaMemsetAsync(deg.p, 0, sizeof(int64_t) * (n + 1), s));
  if (e > 0) {
    expand_kernel<<<grid_for(ws, e), 256, 0, s>>>(e, keys.as<unsigned long long>(),
                                                   dir.as<unsigned long long>());
    t = tb;
    WM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t, dir.as<unsigned long long>(),
                                           dir2.as<unsigned long long>(), nnz, 0, 32 + vb, s));
    split_kernel<<<grid_for(ws, nnz), 256, 0, s>>>(nnz, dir2.as<unsigned long long>(),
                                                    nbr.as<int32_t>(), deg.as<int64_t>());
    WM_CUDA(cudaGetLastError());
  }
  size_t ts = 0;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, ts, deg.as<int64_t>(), off.as<int64_t>(),
                                        n + 1, s));
  DevMem tmp2;
  WM_DALLOC(tmp2, ts);
  WM_CUDA(cub::DeviceScan::ExclusiveSum(tmp2.p, ts, deg.as<int64_t>(), off.as<int64_t>(),
                                        n + 1, s));
  out->n = n;
  out->nnz = nnz;
  out->offsets = static_cast<int64_t *>(malloc(sizeof(int64_t) * (n + 1)));
  out->neighbors = static_cast<int32_t *>(malloc(sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
  if (!out->offsets || !out->neighbors) return fail(WM_ECAPACITY, "host allocation failed");
  WM_CUDA(cudaMemcpyAsync(out->offsets, off.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost,
                          s));
  if (nnz > 0)
    WM_CUDA(cudaMemcpyAsync(out->neighbors, nbr.p, sizeof(int32_t) * nnz,
                            cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  return WM_OK;
}

// ---- edge-list text -------------------------------------------------------

enum : int { kSkip = 0, kEdge = 1, kErrTokens = 2, kErrNonInt = 3, kErrNegative = 4,
             kErrRange = 5 };

__device__ __forceinline__ bool is_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f' ||
         c == 0x1c || c == 0x1d || c == 0x1e || c == 0x1f;
}

// Python int() of one token: optional sign, digits, single underscores
// between digits.  Returns false when the token is not an integer.
__device__ bool parse_int(const unsigned char *p, const unsigned char *e, long long &val,
                          bool &overflow) {
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) { neg = *p == '-'; ++p; }
  if (p == e) return false;
  unsigned long long v = 0;
  bool prev_digit = false;
  overflow = false;
  for (; p < e; ++p) {
    const unsigned char c = *p;
    if (c >= '0' && c <= '9') {
      if (v > (0x7fffffffffffffffull - (c - '0')) / 10) overflow = true;
      else v = v * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  val = neg ? -(long long)v : (long long)v;
  return true;
}

// one thread per line (graph.py:150-182 per-line rules)
__global__ void parse_lines_kernel(const unsigned char *__restrict__ text, int64_t len,
                                   const int64_t *__restrict__ nl, int64_t lines,
                                   int64_t *__restrict__ us, int64_t *__restrict__ vs,
                                   int *__restrict__ status,
                                   unsigned long long *__restrict__ first_err) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < lines;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = j == 0 ? 0 : nl[j - 1] + 1;
    const int64_t e = nl[j];  // exclusive (a '\n' or len)
    const unsigned char *p = text + b, *end = text + e;
    while (p < end && is_space(*p)) ++p;
    while (end > p && is_space(end[-1])) --end;
    int st = kSkip;
    if (p < end && *p != '#' && *p != '%') {
      const unsigned char *tok[3], *tend[3];
      int nt = 0;
      const unsigned char *q = p;
      while (q < end && nt < 3) {
        while (q < end && is_space(*q)) ++q;
        if (q >= end) break;
        tok[nt] = q;
        while (q < end && !is_space(*q)) ++q;
        tend[nt] = q;
        ++nt;
      }
      if (nt != 2) {
        st = kErrTokens;
      } else {
        long long u = 0, v = 0;
        bool ou = false, ov = false;
        if (!parse_int(tok[0], tend[0], u, ou) || !parse_int(tok[1], tend[1], v, ov)) st = kErrNonInt;
        else if (u < 0 || v < 0) st = kErrNegative;
        else if (ou || ov) st = kErrRange;
        else if (u == v) st = kSkip;
        else {
          st = kEdge;
          us[j] = u;
          vs[j] = v;
        }
      }
    }
    status[j] = st;
    if (st >= kErrTokens) atomicMin(first_err, (unsigned long long)j);
  }
}

struct IsNewline {
  const unsigned char *text;
  __device__ bool operator()(const int64_t &i) const { return text[i] == '\n'; }
};

struct IsEdge {
  const int *status;
  __device__ bool operator()(const int64_t &j) const { return status[j] == kEdge; }
};

__global__ void gather_kernel(int64_t e, const int64_t *__restrict__ sel,
                              const int64_t *__restrict__ us, const int64_t *__restrict__ vs,
                              int64_t *__restrict__ ids, int64_t *__restrict__ su,
                              int64_t *__restrict__ sv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = sel[i];
    su[i] = us[j];
    sv[i] = vs[j];
    ids[i] = us[j];
    ids[e + i] = vs[j];
  }
}

// dense id = rank of the raw id among the sorted unique ids
__global__ void remap_kernel(int64_t e, const int64_t *__restrict__ uniq, int64_t n,
                             int64_t *__restrict__ su, int64_t *__restrict__ sv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * e;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t *p = i < e ? su + i : sv + (i - e);
    const int64_t x = *p;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (uniq[mid] < x) lo = mid + 1; else hi = mid;
    }
    *p = lo;
  }
}

int parse_edge_list(Workspace *ws, const char *text, uint64_t len, wm_csr_out *out,
                    cudaStream_t s) {
  DevMem dtext, flags, nl, cnt, us, vs, status, ferr, sel, ids, ids2, uniq, su, sv, tmp;
  WM_DALLOC(dtext, len);
  if (len) WM_CUDA(cudaMemcpyAsync(dtext.p, text, len, cudaMemcpyHostToDevice, s));
  // newline positions: select i where text[i] == '\n'
  WM_DALLOC(nl, sizeof(int64_t) * (len + 1));
  WM_DALLOC(cnt, sizeof(int64_t));
  thrust::counting_iterator<int64_t> iota(0);
  const unsigned char *dt = dtext.as<unsigned char>();
  const IsNewline is_nl{dt};
  size_t t1 = 0;
  WM_CUDA(cub::DeviceSelect::If(nullptr, t1, iota, nl.as<int64_t>(), cnt.as<int64_t>(),
                                (int64_t)len, is_nl, s));
  WM_DALLOC(tmp, t1);
  WM_CUDA(cub::DeviceSelect::If(tmp.p, t1, iota, nl.as<int64_t>(), cnt.as<int64_t>(),
                                (int64_t)len, is_nl, s));
  int64_t nnl = 0;
  WM_CUDA(cudaMemcpyAsync(&nnl, cnt.p, sizeof nnl, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  // a final line without '\n' ends at len
  int64_t lines = nnl;
  char lastc = len ? text[len - 1] : '\n';
  if (lastc != '\n') {
    WM_CUDA(cudaMemcpyAsync(nl.as<int64_t>() + nnl, &len, sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
    ++lines;
  }
  WM_DALLOC(us, sizeof(int64_t) * lines);
  WM_DALLOC(vs, sizeof(int64_t) * lines);
  WM_DALLOC(status, sizeof(int) * lines);
  WM_DALLOC(ferr, sizeof(unsigned long long));
  WM_CUDA(cudaMemsetAsync(ferr.p, 0xff, sizeof(unsigned long long), s));
  if (lines)
    parse_lines_kernel<<<grid_for(ws, lines), 256, 0, s>>>(
        dt, (int64_t)len, nl.as<int64_t>(), lines, us.as<int64_t>(), vs.as<int64_t>(),
        status.as<int>(), ferr.as<unsigned long long>());
  WM_CUDA(cudaGetLastError());
  unsigned long long fe = 0;
  WM_CUDA(cudaMemcpyAsync(&fe, ferr.p, sizeof fe, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  if (fe != ~0ull) {
    int st = 0;
    WM_CUDA(cudaMemcpy(&st, status.as<int>() + fe, sizeof st, cudaMemcpyDeviceToHost));
    out->error_line = (int64_t)fe + 1;
    const char *why = st == kErrTokens ? "expected two integer tokens"
                    : st == kErrNonInt ? "non-integer token"
                    : st == kErrNegative ? "negative vertex id"
                                         : "vertex id exceeds int64";
    return fail(WM_EPARSE, "line %lld: %s", (long long)fe + 1, why);
  }
  // compact the edge lines
  WM_DALLOC(sel, sizeof(int64_t) * lines);
  IsEdge pred{status.as<int>()};
  size_t t2 = 0;
  WM_CUDA(cub::DeviceSelect::If(nullptr, t2, iota, sel.as<int64_t>(), cnt.as<int64_t>(), lines,
                                pred, s));
  DevMem tmp3;
  WM_DALLOC(tmp3, t2);
  WM_CUDA(cub::DeviceSelect::If(tmp3.p, t2, iota, sel.as<int64_t>(), cnt.as<int64_t>(), lines,
                                pred, s));
  int64_t e = 0;
  WM_CUDA(cudaMemcpyAsync(&e, cnt.p, sizeof e, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  if (e == 0) {
    out->error_line = 0;
    return fail(WM_EPARSE, "empty graph: no valid edges in input");
  }
  WM_DALLOC(ids, sizeof(int64_t) * 2 * e);
  WM_DALLOC(ids2, sizeof(int64_t) * 2 * e);
  WM_DALLOC(uniq, sizeof(int64_t) * 2 * e);
  WM_DALLOC(su, sizeof(int64_t) * e);
  WM_DALLOC(sv, sizeof(int64_t) * e);
  gather_kernel<<<grid_for(ws, e), 256, 0, s>>>(e, sel.as<int64_t>(), us.as<int64_t>(),
                                                vs.as<int64_t>(), ids.as<int64_t>(),
                                                su.as<int64_t>(), sv.as<int64_t>());
  // ids remapped to 0..n-1 preserving ascending order (graph.py:183-187)
  size_t t4 = 0, t5 = 0;
  WM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t4, ids.as<int64_t>(), ids2.as<int64_t>(),
                                         2 * e, 0, 64, s));
  WM_CUDA(cub::DeviceSelect::Unique(nullptr, t5, ids2.as<int64_t>(), uniq.as<int64_t>(),
                                    cnt.as<int64_t>(), 2 * e, s));
  DevMem tmp4;
  WM_DALLOC(tmp4, t4 > t5 ? t4 : t5);
  WM_CUDA(cub::DeviceRadixSort::SortKeys(tmp4.p, t4, ids.as<int64_t>(), ids2.as<int64_t>(),
                                         2 * e, 0, 64, s));
  WM_CUDA(cub::DeviceSelect::Unique(tmp4.p, t5, ids2.as<int64_t>(), uniq.as<int64_t>(),
                                    cnt.as<int64_t>(), 2 * e, s));
  int64_t n = 0;
  WM_CUDA(cudaMemcpyAsync(&n, cnt.p, sizeof n, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  if (n >= (1ll << 31) - 1) return fail(WM_EINVAL, "n=%lld exceeds int32 vertex ids", (long long)n);
  remap_kernel<<<grid_for(ws, 2 * e), 256, 0, s>>>(e, uniq.as<int64_t>(), n, su.as<int64_t>(),
                                                    sv.as<int64_t>());
  WM_CUDA(cudaGetLastError());
  return csr_from_device_pairs(ws, n, su.as<int64_t>(), sv.as<int64_t>(), e, out, s);
}

}  // namespace

}  // namespace wm

using namespace wm;

extern "C" {

int wm_csr_build(int64_t n, const int64_t *src, const int64_t *dst, int64_t m,
                 wm_csr_out *out) {
  clear_error();
  if (!out || (m > 0 && (!src || !dst))) return fail(WM_EINVAL, "null argument");
  memset(out, 0, sizeof *out);
  if (n < 1) return fail(WM_EINVAL, "graph needs at least one vertex, got n=%lld", (long long)n);
  if (n >= (1ll << 31) - 1) return fail(WM_EINVAL, "n=%lld exceeds int32 vertex ids",
                                        (long long)n);
  if (m < 0) return fail(WM_EINVAL, "negative edge count");
  Workspace *ws = nullptr;
  int st = workspace_get(&ws);
  if (st) return st;
  WsLock lk(ws);
  if ((st = lk.status())) return st;
  cudaStream_t s = ws->own_stream;
  cudaEvent_t a = ws->ev[4], b = ws->ev[5];
  WM_CUDA(cudaEventRecord(a, s));
  DevMem ds, dd;
  WM_DALLOC(ds, sizeof(int64_t) * m);
  WM_DALLOC(dd, sizeof(int64_t) * m);
  if (m > 0) {
    WM_CUDA(cudaMemcpyAsync(ds.p, src, sizeof(int64_t) * m, cudaMemcpyHostToDevice, s));
    WM_CUDA(cudaMemcpyAsync(dd.p, dst, sizeof(int64_t) * m, cudaMemcpyHostToDevice, s));
  }
  st = csr_from_device_pairs(ws, n, ds.as<int64_t>(), dd.as<int64_t>(), m, out, s);
  if (st) { wm_csr_free(out); return st; }
  WM_CUDA(cudaEventRecord(b, s));
  WM_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  WM_CUDA(cudaEventElapsedTime(&ms, a, b));
  out->device_ms = ms;
  return WM_OK;
}

int wm_edge_list_parse(const char *text, uint64_t len, wm_csr_out *out) {
  clear_error();
  if (!out || (len > 0 && !text)) return fail(WM_EINVAL, "null argument");
  memset(out, 0, sizeof *out);
  Workspace *ws = nullptr;
  int st = workspace_get(&ws);
  if (st) return st;
  WsLock lk(ws);
  if ((st = lk.status())) return st;
  cudaStream_t s = ws->own_stream;
  cudaEvent_t a = ws->ev[4], b = ws->ev[5];
  WM_CUDA(cudaEventRecord(a, s));
  st = parse_edge_list(ws, text, len, out, s);
  if (st) {
    const int64_t line = out->error_line;
    wm_csr_free(out);
    out->error_line = line;
    return st;
  }
  WM_CUDA(cudaEventRecord(b, s));
  WM_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  WM_CUDA(cudaEventElapsedTime(&ms, a, b));
  out->device_ms = ms;
  return WM_OK;
}

void wm_csr_free(wm_csr_out *out) {
  if (!out) return;
  free(out->offsets);
  free(out->neighbors);
  out->offsets = nullptr;
  out->neighbors = nullptr;
  out->n = out->nnz = 0;
}

}  // extern "C"
