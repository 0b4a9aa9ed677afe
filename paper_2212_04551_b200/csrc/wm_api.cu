// wm_api.cu — the C-ABI entry points of libwm_b200.so (include/warpmine_b200.h).
//
// wm_run replaces the body of warpmine.engine.run (reference
// pkg/src/warpmine/engine.py:781-843): argument checks mirror :791-798 and
// Application validation :72-80; dispatch picks the clique kernel for the
// clique_app pipeline (apps.py:43-47) and the motif kernel for motif_app
// (apps.py:50-58).  Any other pipeline is rejected with WM_EINVAL — there is
// no CPU fallback.
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <string>

#include "wm_common.cuh"

namespace wm {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int DeviceBuffer::ensure(size_t want) {
  if (want <= bytes && ptr) return WM_OK;
  release();
  size_t b = want < 256 ? 256 : want;
  cudaError_t e = cudaMalloc(&ptr, b);
  if (e != cudaSuccess) {
    ptr = nullptr;
    bytes = 0;
    return fail(WM_ECUDA, "cudaMalloc(%zu) failed: %s", b, cudaGetErrorString(e));
  }
  bytes = b;
  return WM_OK;
}

void DeviceBuffer::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

__global__ void lb_init_kernel(LbState *lb, int total_warps, uint32_t *ring, uint32_t cap) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) {
    LbState z;
    memset(&z, 0, sizeof z);
    z.active = total_warps;
    z.total_warps = total_warps;
    z.t_start_min = ~0ull;
    z.t_tail_min = ~0ull;
    z.t_base = globaltimer_ns();
    *lb = z;
  }
  if (ring)
    for (uint32_t i = tid; i < cap; i += gridDim.x * blockDim.x) ring[(size_t)i * kSlotWords] = 0u;
}

int lb_prepare(Graph *g, LbState *lb, int warps, uint32_t words, LbShared *out, cudaStream_t s) {
  uint32_t cap = 1;
  while (cap < 8u * (uint32_t)warps) cap <<= 1;
  int st;
  if ((st = g->ws->ring.ensure(sizeof(uint32_t) * kSlotWords * (size_t)cap))) return st;
  out->lb = lb;
  out->ring = g->ws->ring.as<uint32_t>();
  out->cap = cap;
  out->words = words;
  lb_init_kernel<<<(int)((cap + 255) / 256), 256, 0, s>>>(lb, warps, out->ring, cap);
  WM_CUDA(cudaGetLastError());
  return WM_OK;
}

void finish_lb_stats(const LbState &h, wm_result *res) {
  const double W = (double)h.total_warps;
  const double T0 = (double)h.t_start_min, T1 = (double)h.t_end_max;
  if (W <= 0 || T1 <= T0) {
    res->idle_warp_fraction = 0;
    res->idle_warp_fraction_tail = 0;
    return;
  }
  // idle = waiting in acquire_work + after exit + before first start
  const double after_exit = W * T1 - (double)h.sum_end;
  const double before_start = (double)h.sum_start - W * T0;
  const double idle = (double)h.sum_idle_ns + after_exit + before_start;
  res->idle_warp_fraction = idle / (W * (T1 - T0));
  double Tt = (double)h.t_tail_min;
  if (Tt < T0 || Tt > T1 || h.t_tail_min == ~0ull) Tt = T1;
  res->idle_warp_fraction_tail =
      (T1 > Tt) ? ((double)h.sum_tail_idle_ns + after_exit) / (W * (T1 - Tt)) : 0.0;
  if (res->idle_warp_fraction_tail > 1.0) res->idle_warp_fraction_tail = 1.0;
  res->migrations = h.migrations;
  res->rebalance_count = h.donation_polls;
  res->peak_ext = h.peak_ext;
}

// ---------------------------------------------------------------------------
// device result vector (wm_cfg.reduce_out, include/warpmine_b200.h): every
// word is a sum over runs and ranks, so packing adds into it

__global__ void red_pack_kernel(unsigned long long *__restrict__ out,
                                const unsigned long long *__restrict__ ctr, int is_clique,
                                int alg_bytes, int add_tasks, const LbState *__restrict__ lbs,
                                int nlb, const unsigned long long *__restrict__ hist, uint32_t P) {
  if (threadIdx.x == 0) {
    const unsigned long long c = ctr[0];
    if (is_clique) out[WM_RED_CLIQUES] += c;
    out[WM_RED_LEAVES] += c;
    if (alg_bytes) out[WM_RED_ALG_BYTES] += ctr[1];
    if (add_tasks) out[WM_RED_TASKS] += ctr[2];
    for (int i = 0; i < nlb; ++i) {
      out[WM_RED_MIGRATIONS] += lbs[i].migrations;
      out[WM_RED_DONATIONS] += lbs[i].donation_polls;
    }
  }
  if (hist)
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) out[WM_RED_HIST + i] += hist[i];
}

// out[i] += v[i - idx] for four host-known words (timing slots, task counts)
__global__ void red_add_kernel(unsigned long long *out, unsigned long long a,
                               unsigned long long b, unsigned long long c, unsigned long long d) {
  if (threadIdx.x == 0) {
    out[0] += a;
    out[1] += b;
    out[2] += c;
    out[3] += d;
  }
}

// the 2-cliques of a wide root's induced subgraph are its edges: nnz / 2
__global__ void red_edges_kernel(unsigned long long *out, const int64_t *nnz) {
  if (threadIdx.x == 0) {
    const unsigned long long e = (unsigned long long)(*nnz) / 2ull;
    out[WM_RED_CLIQUES] += e;
    out[WM_RED_LEAVES] += e;
  }
}

int red_pack(const wm_cfg *cfg, cudaStream_t s, const unsigned long long *ctr, bool is_clique,
             bool alg_bytes, bool add_tasks, const LbState *lbs, int nlb,
             const unsigned long long *hist, uint32_t P) {
  if (!cfg->reduce_out) return WM_OK;
  red_pack_kernel<<<1, 256, 0, s>>>(reinterpret_cast<unsigned long long *>(cfg->reduce_out),
                                    ctr, is_clique, alg_bytes, add_tasks, lbs, nlb, hist, P);
  WM_CUDA(cudaGetLastError());
  return WM_OK;
}

int red_add(const wm_cfg *cfg, cudaStream_t s, uint64_t idx, unsigned long long a,
            unsigned long long b, unsigned long long c, unsigned long long d) {
  if (!cfg->reduce_out) return WM_OK;
  red_add_kernel<<<1, 32, 0, s>>>(reinterpret_cast<unsigned long long *>(cfg->reduce_out) + idx,
                                  a, b, c, d);
  WM_CUDA(cudaGetLastError());
  return WM_OK;
}

int red_edges(const wm_cfg *cfg, cudaStream_t s, const int64_t *nnz) {
  if (!cfg->reduce_out) return WM_OK;
  red_edges_kernel<<<1, 32, 0, s>>>(reinterpret_cast<unsigned long long *>(cfg->reduce_out), nnz);
  WM_CUDA(cudaGetLastError());
  return WM_OK;
}

// ---------------------------------------------------------------------------
// CsrGraph.validate (graph.py:122-133) on the device, one thread per stored
// entry (hub rows spread over the grid).  The first violation in the
// reference's check order wins: vertex u ascending, then per u: range,
// strictly ascending, self-loop, symmetry (first v in row order).  Key =
// u << 33 | code << 31 | detail; atomicMin.  Offsets that decrease are
// reported first (the reference checks them before any row, graph.py:124-125):
// their own word.  Symmetry is searched only for entries (u, v) with v > u;
// with rows strictly ascending, "every such entry has its reverse" plus
// "#(v > u) == #(v < u)" is symmetry.  Only an invalid graph gets a second
// pass over the v < u entries (to name the first offending edge).
enum : unsigned long long { kCsrRange = 0, kCsrAscend = 1, kCsrLoop = 2, kCsrSym = 3 };

// offsets: [0] first decreasing / out-of-range vertex, [1] max degree (the
// capacity planning of the motif arena), [2] non-zero when offsets[0] != 0
// or offsets[n] != nnz
__global__ void csr_offsets_kernel(int64_t n, int64_t nnz, const int64_t *__restrict__ off,
                                   unsigned long long *__restrict__ bad_off,
                                   unsigned long long *__restrict__ max_deg,
                                   unsigned long long *__restrict__ bad_ends) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != nnz)) *bad_ends = 1ull;
  unsigned long long md = 0;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[u], e = off[u + 1];
    if (e < b || b < 0 || e > nnz) atomicMin(bad_off, (unsigned long long)u);
    else if ((unsigned long long)(e - b) > md) md = (unsigned long long)(e - b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, md, o);
    md = y > md ? y : md;
  }
  if (lane_id() == 0 && md) atomicMax(max_deg, md);
}

// bad[0] first violation key, bad[2] / bad[3] entries with v > u / v < u
__global__ void csr_check_kernel(int64_t n, int64_t nnz, const int64_t *__restrict__ off,
                                 const int32_t *__restrict__ nbr, int lower_pass,
                                 unsigned long long *__restrict__ bad) {
  unsigned long long up = 0, down = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    // u = the row holding entry p: last u with off[u] <= p
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(off + mid) <= p) lo = mid; else hi = mid;
    }
    const int64_t u = lo, b = __ldg(off + u);
    const int32_t v = __ldg(nbr + p);
    unsigned long long k = ~0ull;
    if (v < 0 || v >= n) {
      k = ((unsigned long long)u << 33) | (kCsrRange << 31) |
          ((unsigned long long)(p - b + 1) & 0x7FFFFFFFull);
    } else if (p > b && __ldg(nbr + p - 1) >= v) {
      k = ((unsigned long long)u << 33) | (kCsrAscend << 31);
    } else if (v == u) {
      k = ((unsigned long long)u << 33) | (kCsrLoop << 31);
    } else if ((v > u) != (lower_pass != 0)) {
      int64_t rl = __ldg(off + v), rh = __ldg(off + v + 1);
      if (rl < 0) rl = 0;
      if (rh > nnz) rh = nnz;
      // interpolation + binary search (a hub row of 41K ids: ~5 loads); a
      // miss is re-checked by a linear scan, so an unsorted row of v (reported
      // at v) never masquerades as an asymmetric edge — the reference tests
      // membership in a set (graph.py:132-133)
      bool found = rl < rh && row_contains(nbr, rl, rh, (int32_t)u);
      for (int64_t q = rl; q < rh && !found; ++q) found = __ldg(nbr + q) == (int32_t)u;
      if (!found) k = ((unsigned long long)u << 33) | (kCsrSym << 31) | (unsigned long long)v;
    }
    if (v > (int32_t)u) ++up; else if (v < (int32_t)u) ++down;
    if (k != ~0ull) atomicMin(bad, k);
  }
  up = warp_sum_u64(up);
  down = warp_sum_u64(down);
  if (lane_id() == 0 && !lower_pass) {
    if (up) atomicAdd(bad + 2, up);
    if (down) atomicAdd(bad + 3, down);
  }
}

// Runs the checks on stream s (graph arrays already on the device) and sets
// g->max_degree.
static int csr_validate(Graph *g, cudaStream_t s) {
  int st = g->ws->counters.ensure(sizeof(unsigned long long) * 64);
  if (st) return st;
  // [key, first bad offset, up, down, max degree, bad ends]
  unsigned long long *bad = g->ws->counters.as<unsigned long long>() + 56;
  WM_CUDA(cudaMemsetAsync(bad, 0xff, 2 * sizeof(unsigned long long), s));
  WM_CUDA(cudaMemsetAsync(bad + 2, 0, 4 * sizeof(unsigned long long), s));
  const int64_t ns = (int64_t)g->num_sms;
  const int vb = (int)((g->n + 255) / 256 < ns * 8 ? (g->n + 255) / 256 : ns * 8);
  csr_offsets_kernel<<<vb > 0 ? vb : 1, 256, 0, s>>>(g->n, g->nnz, g->offsets, bad + 1, bad + 4,
                                                     bad + 5);
  unsigned long long hb[6] = {~0ull, ~0ull, 0, 0, 0, 0};
  WM_CUDA(cudaMemcpyAsync(hb, bad, sizeof hb, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  if (hb[5]) return fail(WM_EINVAL, "offsets do not span nnz=%lld", (long long)g->nnz);
  if (hb[1] != ~0ull)
    return fail(WM_EINVAL, "offsets must be non-decreasing (vertex %lld)", (long long)hb[1]);
  g->max_degree = (int64_t)hb[4];
  const int eb = (int)((g->nnz + 255) / 256 < ns * 32 ? (g->nnz + 255) / 256 : ns * 32);
  for (int pass = 0; pass < 2; ++pass) {
    if (g->nnz > 0)
      csr_check_kernel<<<eb > 0 ? eb : 1, 256, 0, s>>>(g->n, g->nnz, g->offsets, g->neighbors,
                                                       pass, bad);
    WM_CUDA(cudaGetLastError());
    WM_CUDA(cudaMemcpyAsync(hb, bad, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaStreamSynchronize(s));
    // a valid graph stops after pass 0; any violation also searches the
    // v < u entries so the reported one is the first in the reference's order
    if (hb[0] == ~0ull && hb[2] == hb[3]) break;
  }
  const unsigned long long h = hb[0];
  if (h == ~0ull) return WM_OK;
  const long long u = (long long)(h >> 33);
  const unsigned long long code = (h >> 31) & 3ull, det = h & 0x7FFFFFFFull;
  switch (code) {
    case kCsrRange:
      return fail(WM_EINVAL, "neighbour #%llu of vertex %lld is outside [0, %lld)", det - 1, u,
                  (long long)g->n);
    case kCsrAscend:
      return fail(WM_EINVAL, "adjacency of %lld not strictly ascending", u);
    case kCsrLoop:
      return fail(WM_EINVAL, "self-loop at %lld", u);
    default:
      return fail(WM_EINVAL, "edge (%lld,%llu) not symmetric", u, det);
  }
}

static std::mutex g_ws_mu;
static Workspace *g_ws[64];

int workspace_get(Workspace **out) {
  int dev = 0;
  WM_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(WM_EINVAL, "device %d out of range", dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (!g_ws[dev]) {
    Workspace *w = new Workspace();
    w->device = dev;
    cudaError_t e = cudaDeviceGetAttribute(&w->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->own_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&w->pool, dev);
    if (e == cudaSuccess) {
      uint64_t thr = ~0ull;
      e = cudaMemPoolSetAttribute(w->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    for (int i = 0; i < 6 && e == cudaSuccess; ++i) e = cudaEventCreate(&w->ev[i]);
    if (e != cudaSuccess) {
      delete w;
      return fail(WM_ECUDA, "workspace init failed: %s", cudaGetErrorString(e));
    }
    g_ws[dev] = w;
  }
  *out = g_ws[dev];
  return WM_OK;
}

}  // namespace wm

using namespace wm;

extern "C" {

int wm_abi_version(void) { return WM_ABI_VERSION; }

const char *wm_last_error(void) { return g_last_error.c_str(); }

static int graph_init(Graph *g) {
  int st = workspace_get(&g->ws);
  if (st) return st;
  g->device = g->ws->device;
  g->num_sms = g->ws->num_sms;
  return WM_OK;
}

// graph arrays come from the device's stream-ordered pool (release threshold
// = unlimited), so create/destroy cycles reuse memory without device syncs
static cudaError_t graph_alloc(Graph *g) {
  cudaStream_t s = g->ws->own_stream;
  cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void **>(&g->offsets),
                                          sizeof(int64_t) * (g->n + 1), g->ws->pool, s);
  if (e == cudaSuccess)
    e = cudaMallocFromPoolAsync(reinterpret_cast<void **>(&g->neighbors),
                                sizeof(int32_t) * (g->nnz > 0 ? g->nnz : 1), g->ws->pool, s);
  return e;
}

int wm_graph_create(const wm_csr *csr, void **out) {
  g_last_error.clear();
  if (!csr || !out) return fail(WM_EINVAL, "null argument");
  if (csr->n < 1) return fail(WM_EINVAL, "graph needs at least one vertex, got n=%lld",
                              (long long)csr->n);
  if (csr->n >= (1ll << 31) - 1) return fail(WM_EINVAL, "n=%lld exceeds int32 vertex ids",
                                             (long long)csr->n);
  if (!csr->offsets || (csr->nnz > 0 && !csr->neighbors))
    return fail(WM_EINVAL, "null CSR arrays");
  if (csr->offsets[0] != 0 || csr->offsets[csr->n] != csr->nnz)
    return fail(WM_EINVAL, "offsets do not span nnz=%lld", (long long)csr->nnz);
  Graph *g = new Graph();
  int st = graph_init(g);
  if (st) { delete g; return st; }
  WsLock lk(g->ws);
  if ((st = lk.status())) { delete g; return st; }
  g->n = csr->n;
  g->nnz = csr->nnz;
  cudaStream_t s = g->ws->own_stream;
  cudaError_t e = graph_alloc(g);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(g->offsets, csr->offsets, sizeof(int64_t) * (g->n + 1),
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && g->nnz > 0)
    e = cudaMemcpyAsync(g->neighbors, csr->neighbors, sizeof(int32_t) * g->nnz,
                        cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    wm_graph_destroy(g);
    return fail(WM_ECUDA, "graph upload failed: %s", cudaGetErrorString(e));
  }
  if ((st = csr_validate(g, s))) {
    wm_graph_destroy(g);
    return st;
  }
  *out = g;
  return WM_OK;
}


int wm_graph_create_device(int64_t n, int64_t nnz, const int64_t *d_offsets,
                           const int32_t *d_neighbors, void **out) {
  g_last_error.clear();
  if (!out || !d_offsets || n < 1) return fail(WM_EINVAL, "bad device graph arguments");
  if (n >= (1ll << 31) - 1) return fail(WM_EINVAL, "n=%lld exceeds int32 vertex ids",
                                        (long long)n);
  if (nnz < 0) return fail(WM_EINVAL, "negative nnz");
  Graph *g = new Graph();
  int st = graph_init(g);
  if (st) { delete g; return st; }
  WsLock lk(g->ws);
  if ((st = lk.status())) { delete g; return st; }
  g->n = n;
  g->nnz = nnz;
  cudaStream_t s = g->ws->own_stream;
  cudaError_t e = graph_alloc(g);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(g->offsets, d_offsets, sizeof(int64_t) * (n + 1),
                        cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && nnz > 0)
    e = cudaMemcpyAsync(g->neighbors, d_neighbors, sizeof(int32_t) * nnz,
                        cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    wm_graph_destroy(g);
    return fail(WM_ECUDA, "device graph copy failed: %s", cudaGetErrorString(e));
  }
  if ((st = csr_validate(g, s))) {
    wm_graph_destroy(g);
    return st;
  }
  *out = g;
  return WM_OK;
}

void wm_graph_destroy(void *gp) {
  Graph *g = static_cast<Graph *>(gp);
  if (!g) return;
  if (g->ws) {
    cudaStream_t s = g->ws->own_stream;
    if (g->offsets) cudaFreeAsync(g->offsets, s);
    if (g->neighbors) cudaFreeAsync(g->neighbors, s);
    if (g->ehash) cudaFreeAsync(g->ehash, s);
  }
  clique_index_free(g);
  delete g;
}

// engine.py:791-798 / balance.py:48-52, shared by wm_run and wm_run_listing
static int check_run_args(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res) {
  if (!g || !app || !cfg || !res) return fail(WM_EINVAL, "null argument");
  if (cfg->mode != WM_MODE_WC && cfg->mode != WM_MODE_OPT && cfg->mode != WM_MODE_DFS)
    return fail(WM_EINVAL, "mode must be one of dfs, wc, opt");
  if (cfg->mode == WM_MODE_DFS && cfg->count_bytes)
    return fail(WM_EINVAL, "count_bytes is measured on the warp-centric tree (wc/opt)");
  if (cfg->mode == WM_MODE_OPT && !(cfg->lb_threshold > 0.0 && cfg->lb_threshold <= 1.0))
    return fail(WM_EINVAL, "threshold must be in (0, 1]");
  if (cfg->mode == WM_MODE_OPT && cfg->lb_poll < 1)
    return fail(WM_EINVAL, "poll_interval must be >= 1");
  if (cfg->shard_count < 1 || cfg->shard_rank < 0 || cfg->shard_rank >= cfg->shard_count)
    return fail(WM_EINVAL, "bad shard %d/%d", cfg->shard_rank, cfg->shard_count);
  // engine.py:72-80, apps.py:38-58
  if (app->k < 3) return fail(WM_EINVAL, "need k >= 3");
  int dev = 0;
  WM_CUDA(cudaGetDevice(&dev));
  if (dev != g->device)
    return fail(WM_EINVAL, "graph lives on device %d, current device is %d", g->device, dev);
  return WM_OK;
}

uint64_t wm_reduce_words(uint32_t pattern_count, int shard_count) {
  return (uint64_t)WM_RED_HIST + pattern_count +
         (uint64_t)WM_RED_SLOT_WORDS * (uint64_t)(shard_count > 0 ? shard_count : 1);
}

static unsigned long long dbits(double x) {
  unsigned long long u;
  memcpy(&u, &x, sizeof u);
  return u;
}

static int wm_run_locked(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res);

int wm_run(void *gp, const wm_app *app, const wm_cfg *cfg, wm_result *res) {
  g_last_error.clear();
  Graph *g = static_cast<Graph *>(gp);
  int st = check_run_args(g, app, cfg, res);
  if (st) return st;
  WsLock lk(g->ws);
  if ((st = lk.status())) return st;
  cudaStream_t s = cfg->stream ? static_cast<cudaStream_t>(cfg->stream) : g->ws->own_stream;
  const uint32_t P = app->aggregator == WM_AGG_PATTERN ? app->pattern_count : 0;
  if (cfg->reduce_out) {
    if (reinterpret_cast<uintptr_t>(cfg->reduce_out) & 7u)
      return fail(WM_EINVAL, "reduce_out must be 8-byte aligned");
    WM_CUDA(cudaMemsetAsync(cfg->reduce_out, 0,
                            sizeof(uint64_t) * wm_reduce_words(P, cfg->shard_count), s));
  }
  st = wm_run_locked(g, app, cfg, res);
  if (st == WM_OK && cfg->reduce_out)
    st = red_add(cfg, s, (uint64_t)WM_RED_HIST + P +
                             (uint64_t)WM_RED_SLOT_WORDS * (uint64_t)cfg->shard_rank,
                 dbits(res->kernel_ms), dbits(res->device_ms), dbits(res->idle_warp_fraction),
                 dbits(res->idle_warp_fraction_tail));
  return st;
}

static int wm_run_locked(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res) {
  const bool clique = app->aggregator == WM_AGG_COUNTER && !app->extend_all &&
                      (app->filters & WM_F_CLIQUE) && (app->filters & WM_F_LOWER) &&
                      !(app->filters & WM_F_CANONICAL);
  const bool motif = app->aggregator == WM_AGG_PATTERN && app->extend_all && app->genedges &&
                     app->filters == WM_F_CANONICAL;
  uint64_t *user_hist = res->pattern_counts;
  memset(res, 0, sizeof *res);
  res->pattern_counts = user_hist;
  cudaStream_t s = cfg->stream ? static_cast<cudaStream_t>(cfg->stream) : g->ws->own_stream;
  if (clique) {
    if (app->k > 12) return fail(WM_EINVAL, "k must be in [3, 12], got %d", app->k);
    return run_clique(g, app, cfg, res, s);
  }
  if (motif) {
    if (app->k > 8) return fail(WM_EINVAL, "k must be in [3, 8], got %d", app->k);
    if ((!app->dict_table && !app->dict_device) ||
        app->dict_len != (1ull << (app->k * (app->k - 1) / 2 - 1)) || app->pattern_count < 1 ||
        (app->dict_device && app->dict_device_bits != 16 && app->dict_device_bits != 32) ||
        (app->dict_device && app->dict_device_bits == 16 && app->pattern_count >= 0xFFFFu))
      return fail(WM_EINVAL, "pattern aggregation requires the k=%d dictionary", app->k);
    if (!user_hist) return fail(WM_EINVAL, "pattern_counts buffer required");
    return run_motif(g, app, cfg, res, s);
  }
  if (app->aggregator == WM_AGG_STORE)
    return fail(WM_EINVAL, "store aggregation runs through wm_run_listing");
  return fail(WM_EINVAL,
              "pipeline not supported on the device: only the built-in clique_app and "
              "motif_app pipelines run (no CPU fallback)");
}

int wm_run_listing(void *gp, const wm_app *app, const wm_cfg *cfg, wm_listing *lst,
                   wm_result *res) {
  g_last_error.clear();
  Graph *g = static_cast<Graph *>(gp);
  int st = check_run_args(g, app, cfg, res);
  if (st) return st;
  if (!lst) return fail(WM_EINVAL, "null listing");
  if (cfg->reduce_out)
    return fail(WM_EINVAL, "listing results (records, checksum) are produced on the host; "
                           "reduce_out is not supported for wm_run_listing");
  WsLock lk(g->ws);
  if ((st = lk.status())) return st;
  // listing_app (apps.py:61-67): extend(0,len), canonical, store
  if (!(app->aggregator == WM_AGG_STORE && app->extend_all && app->genedges &&
        app->filters == WM_F_CANONICAL))
    return fail(WM_EINVAL, "wm_run_listing needs the listing_app pipeline");
  if (app->k > 12) return fail(WM_EINVAL, "k must be in [3, 12], got %d", app->k);
  if (lst->capacity < 1) return fail(WM_EINVAL, "capacity must be positive");
  if (lst->filter != WM_LIST_ALL && lst->filter != WM_LIST_COMPLETE)
    return fail(WM_EINVAL, "unknown listing filter %u", lst->filter);
  if (cfg->count_bytes) return fail(WM_EINVAL, "count_bytes is not available for listing");
  memset(res, 0, sizeof *res);
  lst->emitted = 0;
  lst->checksum = 0;
  cudaStream_t s = cfg->stream ? static_cast<cudaStream_t>(cfg->stream) : g->ws->own_stream;
  return run_motif(g, app, cfg, res, s, lst);
}

}  // extern "C"
