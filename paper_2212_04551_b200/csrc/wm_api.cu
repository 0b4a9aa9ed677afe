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
  int64_t md = 0;
  for (int64_t v = 0; v < csr->n; ++v) {
    int64_t d = csr->offsets[v + 1] - csr->offsets[v];
    if (d < 0) return fail(WM_EINVAL, "offsets decrease at vertex %lld", (long long)v);
    if (d > md) md = d;
  }
  Graph *g = new Graph();
  int st = graph_init(g);
  if (st) { delete g; return st; }
  g->n = csr->n;
  g->nnz = csr->nnz;
  g->max_degree = md;
  cudaStream_t s = g->ws->own_stream;
  cudaError_t e = graph_alloc(g);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(g->offsets, csr->offsets, sizeof(int64_t) * (g->n + 1),
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && g->nnz > 0)
    e = cudaMemcpyAsync(g->neighbors, csr->neighbors, sizeof(int32_t) * g->nnz,
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    wm_graph_destroy(g);
    return fail(WM_ECUDA, "graph upload failed: %s", cudaGetErrorString(e));
  }
  *out = g;
  return WM_OK;
}

__global__ void max_degree_kernel(int64_t n, const int64_t *__restrict__ off,
                                  unsigned long long *__restrict__ out) {
  unsigned long long m = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
    m = d > m ? d : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

int wm_graph_create_device(int64_t n, int64_t nnz, const int64_t *d_offsets,
                           const int32_t *d_neighbors, void **out) {
  g_last_error.clear();
  if (!out || !d_offsets || n < 1) return fail(WM_EINVAL, "bad device graph arguments");
  if (n >= (1ll << 31) - 1) return fail(WM_EINVAL, "n=%lld exceeds int32 vertex ids",
                                        (long long)n);
  Graph *g = new Graph();
  int st = graph_init(g);
  if (st) { delete g; return st; }
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
  // max degree for capacity planning, reduced on the device
  if (e == cudaSuccess) {
    const int r = g->ws->counters.ensure(sizeof(unsigned long long) * 64);
    if (r) { wm_graph_destroy(g); return r; }
    unsigned long long *md = g->ws->counters.as<unsigned long long>();
    e = cudaMemsetAsync(md, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) {
      const int64_t blocks = (n + 255) / 256 < (int64_t)g->num_sms * 8 ? (n + 255) / 256
                                                                      : (int64_t)g->num_sms * 8;
      max_degree_kernel<<<(int)blocks, 256, 0, s>>>(n, g->offsets, md);
      e = cudaGetLastError();
    }
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, md, sizeof h, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    g->max_degree = (int64_t)h;
  }
  if (e != cudaSuccess) {
    wm_graph_destroy(g);
    return fail(WM_ECUDA, "device graph copy failed: %s", cudaGetErrorString(e));
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

int wm_run(void *gp, const wm_app *app, const wm_cfg *cfg, wm_result *res) {
  g_last_error.clear();
  Graph *g = static_cast<Graph *>(gp);
  int st = check_run_args(g, app, cfg, res);
  if (st) return st;
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
