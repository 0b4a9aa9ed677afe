// wm_common.cuh — shared device/host plumbing for libwm_b200.so.
//
// * error capture for the C-ABI (wm_last_error)
// * warp primitives (ballot/popc compaction, reductions)
// * the on-device load balancer.  It replaces the reference's host-side
//   Coordinator (pkg/src/warpmine/balance.py:163-194), which stops every warp
//   at a consistent state and hands one pending extension to each idle warp
//   in order (balance.py:80-128).  On the device it is a ticketed rendezvous
//   ring that needs only fetch-and-add (no CAS retry loops):
//     - a warp whose stack is empty and finds the root cursor drained takes an
//       idle ticket t = FAA(tail) and spins on slot t of the ring (its own
//       line: thousands of idle warps cost no shared traffic);
//     - busy warps poll (tail - head) every `poll` DFS steps; when
//       active/total < threshold (balance.py:63-66) a busy warp takes a donor
//       ticket h = FAA(head) and writes its donation record into slot h —
//       tickets pair donors and idle warps FIFO, like the reference's
//       round-robin over the idle list, and nobody is ever stopped;
//     - `active` counts busy warps plus records in flight, so active == 0 is a
//       stable termination condition.
//   This is the paper's stated future work: balancing
//   without stopping and relaunching the kernel.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <cuda_runtime.h>
#include <cuda/atomic>

#include "../../include/warpmine_b200.h"

namespace wm {

// ---------------------------------------------------------------------------
// error capture

void set_error(const std::string &msg);
void clear_error();
int fail(int code, const char *fmt, ...);

#define WM_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess)                                                   \
      return ::wm::fail(WM_ECUDA, "%s failed at %s:%d: %s", #call, __FILE__, \
                        __LINE__, cudaGetErrorString(_e));                   \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers

constexpr int kWarp = 32;
#ifndef WM_INTERP_MIN
#define WM_INTERP_MIN 16  // rows longer than this start with interpolation probes
#endif
constexpr int kMaxK = 12;
constexpr int kSlotWords = 128;  // ring slot: [0] seq (ticket+1), [32..127] record

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// first index in sorted a[0..n) with a[i] >= x (shared or global)
template <typename T>
__device__ __forceinline__ int lower_bound_i(const T *a, int n, T x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// membership of x in the ascending CSR row [b, e) of nbr (global, read-only).
// Long rows start with interpolation probes: ids are (randomly permuted)
// vertex numbers, so a row is close to a uniform sample of [0, n) and each
// probe shrinks the range to ~sqrt of itself — a 64K-entry hub row takes
// ~5 dependent loads instead of 16.  Binary search finishes (and bounds the
// cost on skewed rows).
__device__ __forceinline__ bool row_contains(const int32_t *__restrict__ nbr, int64_t b,
                                             int64_t e, int32_t x) {
  if (e - b > WM_INTERP_MIN) {
    int64_t lo = b, hi = e - 1;
    int32_t vlo = __ldg(nbr + lo), vhi = __ldg(nbr + hi);
    if (x <= vlo) return x == vlo;
    if (x >= vhi) return x == vhi;
    // invariant: vlo < x < vhi, candidates strictly inside (lo, hi)
#pragma unroll 1
    for (int it = 0; it < 3 && hi - lo > 8; ++it) {
      const float f = (float)(x - vlo) / (float)(vhi - vlo);
      int64_t pos = lo + 1 + (int64_t)(f * (float)(hi - lo - 1));
      pos = pos < lo + 1 ? lo + 1 : (pos > hi - 1 ? hi - 1 : pos);
      const int32_t y = __ldg(nbr + pos);
      if (y == x) return true;
      if (y < x) { lo = pos; vlo = y; } else { hi = pos; vhi = y; }
    }
    b = lo + 1;
    e = hi;
  }
  while (b < e) {
    int64_t mid = (b + e) >> 1;
    int32_t y = __ldg(nbr + mid);
    if (y == x) return true;
    if (y < x) b = mid + 1; else e = mid;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Edge hash set: every undirected edge {u, v} of the CSR as the key
// min << 32 | max in an open-addressed table of 32-byte buckets (4 keys, one
// L2 sector), load factor <= 1/2, linear probing over buckets.  Keys fill a
// bucket's slots in order and are never deleted, so a bucket whose last slot
// is empty ends the probe.  An adjacency test is one sector load (rarely two)
// with no dependence on either endpoint's CSR row — against log2(degree)
// dependent loads for a binary search — and the tests of one candidate
// against several traversal vertices are independent loads in flight together.
constexpr unsigned long long kEhEmpty = ~0ull;

struct EdgeHash {
  const ulonglong2 *b;        // bucket i = b[2i], b[2i+1]; null = no table (binary search)
  unsigned long long bmask;
};

__device__ __host__ __forceinline__ unsigned long long eh_key(int32_t u, int32_t v) {
  const uint32_t lo = (uint32_t)(u < v ? u : v), hi = (uint32_t)(u < v ? v : u);
  return ((unsigned long long)lo << 32) | hi;
}

__device__ __host__ __forceinline__ unsigned long long eh_bucket(unsigned long long key,
                                                                 unsigned long long bmask) {
  unsigned long long z = key + 0x9E3779B97F4A7C15ull;  // splitmix64 finaliser
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (z ^ (z >> 31)) & bmask;
}

__device__ __forceinline__ bool edge_hash_contains(const EdgeHash &H, int32_t u, int32_t v) {
  const unsigned long long key = eh_key(u, v);
  unsigned long long b = eh_bucket(key, H.bmask);
  for (;;) {
    const ulonglong2 p = __ldg(H.b + 2 * b), q = __ldg(H.b + 2 * b + 1);
    if (p.x == key || p.y == key || q.x == key || q.y == key) return true;
    if (q.y == kEhEmpty) return false;
    b = (b + 1) & H.bmask;
  }
}

using aref_u64 = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
using aref_i32 = cuda::atomic_ref<int, cuda::thread_scope_device>;
using aref_u32 = cuda::atomic_ref<uint32_t, cuda::thread_scope_device>;

// ---------------------------------------------------------------------------
// load-balancing state (one per enumeration launch); hot fields on their own
// 128-byte lines so polls never queue behind another field's atomics

struct alignas(128) LbState {
  alignas(128) unsigned long long task_cursor;  // next root task (engine.py:187 deque)
  alignas(128) int active;                      // busy warps + records in flight
  int total_warps;
  alignas(128) unsigned long long head;         // donor tickets
  alignas(128) unsigned long long tail;         // idle-warp tickets
  alignas(128) unsigned long long migrations;   // donated prefixes (balance.py:192-193)
  unsigned long long donation_polls;            // donations made (rebalance_count)
  // t_base is the globaltimer at lb_init; every other time is relative to it
  // (absolute ns summed over thousands of warps would overflow u64)
  unsigned long long t_base, t_start_min, t_end_max, t_tail_min;
  unsigned long long sum_start, sum_end, sum_idle_ns, sum_tail_idle_ns;
  unsigned long long peak_ext;
  int error;                                    // WM_E* raised on device
};

struct LbShared {
  LbState *lb;
  uint32_t *ring;     // [cap * kSlotWords]
  uint32_t cap;       // power of two >= 2 * warps
  uint32_t words;     // record words (<= 96)
};

__device__ __forceinline__ unsigned long long ld_relaxed(unsigned long long *p) {
  return aref_u64(*p).load(cuda::std::memory_order_relaxed);
}
__device__ __forceinline__ int ld_relaxed(int *p) {
  return aref_i32(*p).load(cuda::std::memory_order_relaxed);
}

__device__ __forceinline__ void raise_error(LbState *lb, int code) {
  atomicCAS(&lb->error, 0, code);
}

// A record is up to 96 u32 held lane-distributed: lane l holds word 32r+l in w[r].
struct Rec3 {
  uint32_t w[3];
};

// word `idx` of a lane-distributed record (warp-collective; idx may differ per lane)
__device__ __forceinline__ uint32_t rec_word(const Rec3 &r, int idx) {
  const int src = idx & 31, reg = (idx >> 5) & 3;
  const uint32_t a = __shfl_sync(0xffffffffu, r.w[0], src);
  const uint32_t b = __shfl_sync(0xffffffffu, r.w[1], src);
  const uint32_t c = __shfl_sync(0xffffffffu, r.w[2], src);
  return reg == 0 ? a : (reg == 1 ? b : c);
}

__global__ void lb_init_kernel(LbState *lb, int total_warps, uint32_t *ring, uint32_t cap);

// Donor side: write `rec` into the next donor ticket's slot.  Warp-collective.
// Only called after donation_wanted() saw waiting idle tickets; a rare
// overshoot (two donors racing for one waiting warp) leaves the record for
// the next warp that goes idle — possibly the donor itself.
__device__ __forceinline__ void donate_record(const LbShared &L, const Rec3 &rec) {
  const int lane = lane_id();
  unsigned long long h = 0;
  if (lane == 0) {
    atomicAdd(&L.lb->active, 1);  // the record is work in flight
    h = atomicAdd(&L.lb->head, 1ull);
  }
  h = __shfl_sync(0xffffffffu, h, 0);
  uint32_t *slot = L.ring + (size_t)(h & (L.cap - 1)) * kSlotWords;
  if (lane == 0) {
    // slot reuse guard: the record of ticket h - cap must have been consumed
    // (cap >= 8 x warps makes this wait practically never taken)
    // relaxed polling: an acquire load per spin would invalidate the SM's L1
    // (CCTL.IVALL) under the busy warps sharing it
    while (aref_u32(slot[0]).load(cuda::std::memory_order_relaxed) != 0u) __nanosleep(64);
    __threadfence();
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 3; ++r)
    if ((uint32_t)(lane + 32 * r) < L.words) __stcg(slot + 32 + 32 * r + lane, rec.w[r]);
  __threadfence();
  __syncwarp();
  if (lane == 0) aref_u32(slot[0]).store((uint32_t)(h + 1), cuda::std::memory_order_release);
}

// Per-warp bookkeeping of idle time (for idle_warp_fraction).
struct WarpClock {
  unsigned long long t_start, idle_ns, tail_idle_ns;
};

// Warp-collective work acquisition shared by the clique and motif kernels.
//   returns 1: root task (task index in *task_idx)
//           2: donated record (lane-distributed in rec)
//           0: no work left — exit
// `roots_left` is warp-uniform state owned by the caller.
__device__ __forceinline__ int acquire_work(const LbShared &L, bool lb_on,
                                            unsigned long long ntasks, bool &roots_left,
                                            unsigned long long &task_idx, Rec3 &rec,
                                            WarpClock &clk) {
  const int lane = lane_id();
  LbState *lb = L.lb;
  if (roots_left) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&lb->task_cursor, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx < ntasks) {
      task_idx = idx;
      return 1;
    }
    roots_left = false;
    if (lane == 0) {
      const unsigned long long ta = globaltimer_ns(), base = lb->t_base;
      atomicMin(&lb->t_tail_min, ta > base ? ta - base : 0ull);
    }
  }
  if (!lb_on) return 0;
  const unsigned long long t0 = globaltimer_ns();
  unsigned long long t = 0;
  if (lane == 0) {
    t = atomicAdd(&lb->tail, 1ull);
    atomicSub(&lb->active, 1);
  }
  t = __shfl_sync(0xffffffffu, t, 0);
  uint32_t *slot = L.ring + (size_t)(t & (L.cap - 1)) * kSlotWords;
  unsigned backoff = 32;
  int result = 0;
  for (;;) {
    int state = 0;  // 1 record, 2 exit
    if (lane == 0) {
      // relaxed spin (no per-iteration L1 invalidation); the fence below
      // orders the record reads after the observed sequence word
      if (aref_u32(slot[0]).load(cuda::std::memory_order_relaxed) == (uint32_t)(t + 1)) state = 1;
      else if (ld_relaxed(&lb->active) <= 0 || ld_relaxed(&lb->error)) state = 2;
    }
    state = __shfl_sync(0xffffffffu, state, 0);
    if (state == 1) {
      __threadfence();
#pragma unroll
      for (int r = 0; r < 3; ++r)
        if ((uint32_t)(lane + 32 * r) < L.words) rec.w[r] = __ldcg(slot + 32 + 32 * r + lane);
      __syncwarp();
      if (lane == 0) aref_u32(slot[0]).store(0u, cuda::std::memory_order_release);
      result = 2;
      break;
    }
    if (state == 2) { result = 0; break; }
    __nanosleep(backoff);
    if (backoff < 1024) backoff <<= 1;
  }
  const unsigned long long dt = globaltimer_ns() - t0;
  clk.idle_ns += dt;
  clk.tail_idle_ns += dt;
  return result;
}

__device__ __forceinline__ void warp_clock_begin(WarpClock &clk, LbState *lb) {
  const unsigned long long base = lb->t_base;
  const unsigned long long t = globaltimer_ns();
  clk.t_start = t > base ? t - base : 0ull;
  clk.idle_ns = 0;
  clk.tail_idle_ns = 0;
}

__device__ __forceinline__ void warp_clock_end(LbState *lb, const WarpClock &clk) {
  if (lane_id() == 0) {
    const unsigned long long base = lb->t_base;
    const unsigned long long ta = globaltimer_ns();
    const unsigned long long t = ta > base ? ta - base : 0ull;
    atomicMin(&lb->t_start_min, clk.t_start);
    atomicMax(&lb->t_end_max, t);
    atomicAdd(&lb->sum_start, clk.t_start);
    atomicAdd(&lb->sum_end, t);
    atomicAdd(&lb->sum_idle_ns, clk.idle_ns);
    atomicAdd(&lb->sum_tail_idle_ns, clk.tail_idle_ns);
  }
}

// Should a busy warp donate now?  balance.py:63-66: rebalance when
// active/total < threshold  <=>  idle > total * (1 - threshold); idle =
// idle tickets not yet served by a donor ticket.
__device__ __forceinline__ bool donation_wanted(const LbShared &L, int idle_min) {
  int want = 0;
  if (lane_id() == 0) {
    const unsigned long long t = ld_relaxed(&L.lb->tail);
    const unsigned long long h = ld_relaxed(&L.lb->head);
    want = (long long)(t - h) >= (long long)idle_min;
  }
  return __shfl_sync(0xffffffffu, want, 0) != 0;
}

// ---------------------------------------------------------------------------
// host-side helpers

struct DeviceBuffer {
  void *ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t want);
  void release();
  ~DeviceBuffer() { release(); }
  template <typename T> T *as() const { return static_cast<T *>(ptr); }
};

// Per-device scratch, shared by every graph handle on that device: grow-only
// buffers reused across runs and across graphs, so a fresh upload (the e2e
// path) pays no cudaMalloc/cudaFree.  Every C-ABI entry point that touches it
// holds `mu` for the whole call (WsLock), so concurrent callers on one device
// (ctypes releases the GIL) are serialised; a nested call from the same
// thread (a listing sink calling back into the library) is refused.
struct Workspace {
  std::mutex mu;
  std::atomic<std::thread::id> owner{};
  int device = 0;
  int num_sms = 0;
  cudaStream_t own_stream = nullptr;
  cudaMemPool_t pool = nullptr;  // stream-ordered pool for graph arrays
  DeviceBuffer dag_off, dag_nbr, outdeg, keys_in, keys_out, vals_in, vals_out, cub_tmp;
  DeviceBuffer lb, ring, counters, hist, arena, table, listing, listing_ring;
  DeviceBuffer edge_src, edge_flag, edge_pos;  // clique orientation, per directed edge
  DeviceBuffer claims;  // motif B_alg claim slots (count_bytes with the balancer on)
  DeviceBuffer ehash_local;  // motif root-suffix runs: edge hash of the induced subgraph
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
};

// Stream-ordered phase timing of the host-side run setup (WM_PHASES=1 prints
// the per-phase device time to stderr; off by default).
struct PhaseTimer {
  bool on = false;
  cudaEvent_t ev[12];
  const char *name[12];
  int n = 0;
  cudaStream_t s;
  explicit PhaseTimer(cudaStream_t st) : s(st) {
    const char *e = getenv("WM_PHASES");
    on = e && *e == '1';
  }
  void mark(const char *nm) {
    if (!on || n >= 12) return;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], s);
    name[n++] = nm;
  }
  ~PhaseTimer() {
    if (!on || n < 2) return;
    cudaEventSynchronize(ev[n - 1]);
    for (int i = 1; i < n; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, "[wm phases] %-14s %8.3f ms\n", name[i], ms);
    }
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
};

// returns the workspace of the current device (created on first use)
int workspace_get(Workspace **out);

// Scoped hold of a workspace for one C-ABI call.  status() is WM_EINVAL when
// the calling thread already holds it (re-entry from a sink callback).
class WsLock {
 public:
  explicit WsLock(Workspace *w) : w_(w) {
    if (!w_) return;
    if (w_->owner.load() == std::this_thread::get_id()) {
      reentrant_ = true;
      return;
    }
    w_->mu.lock();
    w_->owner.store(std::this_thread::get_id());
    held_ = true;
  }
  ~WsLock() {
    if (held_) {
      w_->owner.store(std::thread::id());
      w_->mu.unlock();
    }
  }
  int status() const {
    return reentrant_ ? fail(WM_EINVAL, "re-entrant call into libwm_b200 on device %d (a "
                                        "listing sink may not start another run)", w_->device)
                      : WM_OK;
  }
  WsLock(const WsLock &) = delete;
  WsLock &operator=(const WsLock &) = delete;

 private:
  Workspace *w_ = nullptr;
  bool held_ = false, reentrant_ = false;
};

struct Graph {
  int64_t n = 0, nnz = 0;
  int64_t max_degree = 0;
  int device = 0;
  int num_sms = 0;
  int64_t *offsets = nullptr;   // device [n+1]
  int32_t *neighbors = nullptr; // device [nnz]
  Workspace *ws = nullptr;
  // edge hash set (motif adjacency probes), built on first use; owned by the graph
  unsigned long long *ehash = nullptr;
  unsigned long long ehash_bmask = 0;  // bucket count - 1 (4 keys per bucket)
  // clique index per orientation (id, degree), built on first use (wm_clique.cu)
  void *cidx[2] = {nullptr, nullptr};
};

// frees g's clique indexes (wm_clique.cu)
void clique_index_free(Graph *g);

// Task sort keys are (out-)degree + 1 <= max_degree + 1: radix-sort only those
// bits (same stable order as a 32-bit sort, fewer passes).
inline int task_key_bits(const Graph *g) {
  unsigned long long v = (unsigned long long)g->max_degree + 1ull;
  int b = 1;
  while (b < 32 && (v >> b)) ++b;
  return b;
}

// builds g->ehash on stream s if absent (wm_motif.cu)
int graph_edge_hash(Graph *g, cudaStream_t s);

// Allocates the balancer's ring for `warps` and initialises lb (one
// LbState) on stream s.
int lb_prepare(Graph *g, LbState *lb, int warps, uint32_t words, LbShared *out, cudaStream_t s);

int run_clique(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res, cudaStream_t s);
int run_motif(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res, cudaStream_t s,
              wm_listing *lst = nullptr);

// device result vector (wm_cfg.reduce_out; no-ops when it is NULL):
// adds one run's counters (ctr[0] count/leaves, ctr[1] B_alg, ctr[2] tasks),
// its balancer statistics and histogram on stream s
int red_pack(const wm_cfg *cfg, cudaStream_t s, const unsigned long long *ctr, bool is_clique,
             bool alg_bytes, bool add_tasks, const LbState *lbs, int nlb,
             const unsigned long long *hist, uint32_t P);
// adds four host-known words at reduce_out[idx .. idx+4)
int red_add(const wm_cfg *cfg, cudaStream_t s, uint64_t idx, unsigned long long a,
            unsigned long long b, unsigned long long c, unsigned long long d);
// adds *nnz / 2 cliques and leaves (device-resident edge count)
int red_edges(const wm_cfg *cfg, cudaStream_t s, const int64_t *nnz);

// fills the idle fractions and LB stats of `res` from a device LbState copy
void finish_lb_stats(const LbState &h, wm_result *res);

}  // namespace wm
