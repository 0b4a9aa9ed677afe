// wm_motif.cu — warp-centric k-motif counting (motif_app, reference
// pkg/src/warpmine/apps.py:50-58) for sm_100a.
//
// Reference pipeline per traversal tr[0..L) (engine.py:214-241):
//   extend(0,L)        union of N(tr[0..L)) minus tr, deduplicated  engine.py:245-327
//   filter_canonical   keep e iff e > tr[0] and e > tr[j] for every j
//                      after the first position adjacent to e     engine.py:424-513,
//                                                                  canon.py:190-210
//   aggregate_pattern  at L == k-1: bits = bitmap | mask << off(k-1),
//                      pid = table[bits], counts[pid]++            aggregate.py:174-196
//   move_step+induce   pop, append, bitmap[L] = extend_bits(...)   engine.py:643-705
//
// B200 restatement.  The canonical extension set obeys an exact recurrence
// (the filters are conjunctive and only tighten as the traversal grows):
//   E_1     = { e in N(r) : e > r },                         mask 1
//   E_{L+1} = { e in E_L : e > w }                (A part),  mask |= adj(e,w) << L
//           ∪ { e in N(w) : e > tr[0], e adjacent to none of tr[0..L) }
//                                                 (B part),  mask  = 1 << L
// with w = tr[L].  Each level is one warp pass: lanes take 32 entries, probe
// adjacency by binary search in the shorter CSR row, and compact survivors
// with __ballot_sync/__popc into the next level of a per-warp HBM arena
// (DFS-wide: level L holds at most L * max_degree entries, the reference's
// capacity rule engine.py:319).  Entries pack vertex | mask << vbits.
// Leaves (L == k-1) are never materialised: A-part leaves are classified with
// one dictionary lookup each and bucketed with __match_any_sync into a
// shared-memory u64 histogram; all B-part leaves share mask 1 << (k-2), so they
// are counted with ballot+popc and added with a single lookup.
//
// Load balancing: as for cliques, busy warps donate half of the pending
// entries of their shallowest level through the ticket ring; a record holds
// (root, level, prefix, bitmap, [lo, hi)) and the thief deterministically
// rebuilds E_1..E_level for that prefix (same order, so the index range is
// meaningful), exactly the reference's "inherited levels are generated but
// empty" install (balance.py:131-155).
#include <chrono>
#include <cub/cub.cuh>

#include "wm_common.cuh"

namespace wm {

// sort keys of the root range [rb, re) only (entry i = vertex rb + i):
// degree + 1 for roots with an edge, 0 otherwise; warp-aggregated count
__global__ void motif_task_keys_kernel(const int64_t *__restrict__ off, int64_t rb, int64_t re,
                                       uint32_t *__restrict__ keys,
                                       int32_t *__restrict__ vals,
                                       unsigned long long *__restrict__ ntask) {
  const int64_t R = re - rb;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < R; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    bool ok = false;
    if (i < R) {
      const int64_t v = rb + i;
      const int64_t d = off[v + 1] - off[v];
      ok = d > 0;
      keys[i] = ok ? (uint32_t)d + 1u : 0u;
      vals[i] = (int32_t)v;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    if (lane_id() == 0 && bal) atomicAdd(ntask, (unsigned long long)__popc(bal));
  }
}

// Listing ring (aggregate_store, aggregate.py:199-223): records are staged in
// an HBM ring; `head` (device) hands out record tickets; each block of
// 2^block_shift tickets has a completion counter the producers bump after
// their records are written (and fenced).  The host copies completed blocks
// with the copy engine and publishes its tail with a small H2D copy into
// device memory (ctl[0]; ctl[1] = consumer failed) — producers waiting for
// space poll L2, never host memory (thousands of warps reading sysmem would
// starve the very copies they wait for).  A producer blocks while its ticket is more than
// `cap` ahead of the tail (StoreBuffer back-pressure, aggregate.py:69-99).
// Small scattered stores straight into mapped host memory ran at ~1.4 GB/s
// over PCIe; the HBM ring + bulk DMA runs at copy-engine speed.
struct ListRing {
  uint32_t *slots;                 // device [cap * stride]
  uint32_t *blockdone;             // device [cap >> block_shift] records written per block
  uint32_t block_shift;
  unsigned long long *ctl;         // device [0] tail [1] failed (written by host DMA)
  unsigned long long *head;        // device ticket counter
  unsigned long long cap_mask;
  uint32_t stride;                 // words per record (k + 4)
  uint32_t filter;                 // WM_LIST_*
  unsigned long long full_prefix;  // bitmap of a complete (k-1)-prefix
  uint32_t full_mask;              // mask of e adjacent to all of tr[0..k-1)
};

struct MotifArgs {
  const int64_t *off;
  const int32_t *nbr;
  const int32_t *tasks;
  unsigned long long ntasks, task_offset, task_stride;
  // multi-GPU: every shard walks every root but descends only into the
  // level-1 entries with index + root = l1_offset (mod l1_stride) (edge tasks
  // (r, u) dealt cyclically, rotated by the root so the many one-child roots
  // spread too); a hub root's subtree no longer lands on one
  // GPU.  l1_stride = 1: no filter.  shard_level 2 (k >= 6) deals the
  // level-2 entries (root, child, grandchild) instead, by a hash of the three
  // vertex ids: one hub child's subtree no longer lands on one GPU either;
  // every rank then builds E_2 of every child (a small share at k >= 6).
  uint32_t l1_offset, l1_stride;
  int shard_level;
  int k;
  int vbits;
  uint32_t vmask;
  const uint32_t *table;            // u32 dictionary, or
  const uint16_t *table16;          // u16 dictionary (SENTINEL 0xFFFF)
  uint32_t pattern_count;
  uint32_t *arena;
  unsigned long long warp_stride;  // arena words per warp
  long long maxdeg;
  unsigned long long *hist;        // global [pattern_count]
  unsigned long long *counters;    // [0] leaves [1] B_alg [2] tasks [3] nodes [4] polls [5] peak
  int lb_on, lb_poll, idle_min;
  int smem_hist;
  // B_alg claim slots (BYTES): one u32 flag per shared (donated-across) node
  uint32_t *claims;
  unsigned long long *claim_ctr;
  uint32_t claim_cap;
  EdgeHash H;                      // adjacency probes (null table: CSR binary search)
  LbShared L;
  ListRing ring;
};

struct MotifWarp {
  int32_t tr[kMaxK];
  long long tb[kMaxK], te[kMaxK];   // CSR row bounds of tr[j]
  unsigned long long bm[kMaxK];     // bm[L-1] = bitmap of tr[0..L) (<= 54 bits, k <= 12)
  unsigned long long tail_cache;    // listing: last consumer tail seen (lane 0)
  union {
    struct {
      int32_t le[32];               // listing: leaf vertex of record rank r
      uint32_t lm[32];              //          and its adjacency mask
    };
    struct {                        // counting: leaf_bulk's pair rings
      uint2 ra[64];                 //   A leaves (x entry, e entry)
      uint2 rb[64];                 //   B leaves (x entry, e vertex)
    };
  };
  uint32_t size[kMaxK], cur[kMaxK], lo[kMaxK];
  // B_alg: the node of length L is productive iff a leaf lies
  // below it.  claimed bit L: this warp knows the node's bytes are counted
  // (by itself or another warp); claim[L]: global claim slot of a node shared
  // with other warps through a donation (kNoClaim: private to this warp).
  uint32_t claim[kMaxK];
  uint32_t claimed;
  // per-warp counters (lane 0), in shared memory rather than registers: the
  // k >= 6 kernel runs at 40 registers (6 blocks/SM) and spills
  unsigned long long n_leaves, n_nodes, n_polls, n_peak, n_tasks;
  uint32_t lbt, lbh;  // poll_donate's pipelined ticket counters (lane 0)
};

constexpr uint32_t kNoClaim = 0xFFFFFFFFu;

__device__ __forceinline__ int group_off(int i) { return i * (i - 1) / 2 - 1; }

// adjacency of e (row [eb,ee)) and x (row [xb,xe)): search the shorter row
__device__ __forceinline__ bool adj_probe(const int32_t *__restrict__ nbr, int32_t e, long long eb,
                                          long long ee, int32_t x, long long xb, long long xe) {
  return (ee - eb <= xe - xb) ? row_contains(nbr, eb, ee, x) : row_contains(nbr, xb, xe, e);
}

// Adjacency of candidate e with traversal vertex tr[j]: one edge-hash probe.
// Without a table (allocation failed): binary search in the shorter CSR row,
// out of line — a cold path whose interpolation search would otherwise be
// inlined at every probe site of the hot loops.
__device__ __noinline__ bool adj_csr(const MotifArgs &a, const MotifWarp &w, int j, int32_t e) {
  const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
  return adj_probe(a.nbr, e, eb, ee, w.tr[j], w.tb[j], w.te[j]);
}

__device__ __forceinline__ bool adj_tr(const MotifArgs &a, const MotifWarp &w, int j, int32_t e) {
  if (a.H.b) return edge_hash_contains(a.H, e, w.tr[j]);
  return adj_csr(a, w, j, e);
}

#ifndef WM_BPART_UNROLL
#define WM_BPART_UNROLL 6  // motif k <= 8 has L <= 6; deeper listing levels loop
#endif

// e adjacent to none of tr[0..L): the B-part test.  With the hash table the L
// probes are independent loads (no early exit), all in flight at once.
__device__ __forceinline__ bool adj_none(const MotifArgs &a, const MotifWarp &w, int L, int32_t e) {
  if (a.H.b) {
    bool hit = false;
#pragma unroll
    for (int j = 0; j < WM_BPART_UNROLL; ++j)
      if (j < L) hit |= edge_hash_contains(a.H, e, w.tr[j]);
    for (int j = WM_BPART_UNROLL; j < L; ++j) hit |= edge_hash_contains(a.H, e, w.tr[j]);
    return !hit;
  }
  bool keep = true;
  for (int j = 0; j < L && keep; ++j) keep = !adj_csr(a, w, j, e);
  return keep;
}

__device__ __forceinline__ uint32_t *level_ptr(const MotifArgs &a, uint32_t *base, int L) {
  // level L (1..k-2) starts at maxdeg * (L-1)L/2
  return base + (unsigned long long)a.maxdeg * (unsigned long long)((L - 1) * L / 2);
}


// Warp-cooperative lower bound: first position in the ascending CSR row
// [b, e) holding a value > key.  Canonical candidates must exceed tr[0]
// (canon.py:190-210), so row scans start there instead of filtering a hub's
// whole row element by element.  32-ary search: <= 4 dependent loads for a
// 64K-entry row.
__device__ __forceinline__ long long row_first_above(const int32_t *__restrict__ nbr, long long b,
                                                     long long e, int32_t key) {
  const int lane = lane_id();
  while (e - b > 32) {
    const long long step = (e - b + 31) / 32;
    const long long pos = b + step * lane;
    const bool le = pos < e && __ldg(nbr + pos) <= key;
    const unsigned bal = __ballot_sync(0xffffffffu, le);
    const int cnt = __popc(bal);  // rows are ascending: the <= key prefix is lanes [0, cnt)
    if (cnt == 0) return b;
    const long long nb = b + step * (cnt - 1) + 1;
    const long long ne = b + step * cnt;
    b = nb;
    e = ne < e ? ne : e;
  }
  const long long pos = b + lane;
  const bool le = pos < e && __ldg(nbr + pos) <= key;
  return b + __popc(__ballot_sync(0xffffffffu, le));
}

// warp-collective append with ballot+popc compaction
__device__ __forceinline__ void emit(uint32_t *dst, uint32_t &cnt, bool keep, uint32_t val) {
  const int lane = lane_id();
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (keep) dst[cnt + __popc(bal & ((1u << lane) - 1u))] = val;
  cnt += __popc(bal);
}

// E_1 for root r
__device__ __forceinline__ uint32_t build_first(const MotifArgs &a, MotifWarp &w, uint32_t *base) {
  const int lane = lane_id();
  uint32_t *dst = level_ptr(a, base, 1);
  const int32_t r = w.tr[0];
  uint32_t cnt = 0;
  for (long long p0 = row_first_above(a.nbr, w.tb[0], w.te[0], r); p0 < w.te[0]; p0 += 32) {
    const long long p = p0 + lane;
    bool keep = false;
    uint32_t val = 0;
    if (p < w.te[0]) {
      const int32_t e = __ldg(a.nbr + p);
      keep = e > r;
      val = (uint32_t)e | (1u << a.vbits);
    }
    emit(dst, cnt, keep, val);
  }
  return cnt;
}

// E_{L+1} from E_L and w = tr[L]
__device__ __forceinline__ uint32_t build_next(const MotifArgs &a, MotifWarp &w, uint32_t *base,
                                               int L) {
  const int lane = lane_id();
  const uint32_t *src = level_ptr(a, base, L);
  uint32_t *dst = level_ptr(a, base, L + 1);
  const int32_t x = w.tr[L];
  const long long xb = w.tb[L], xe = w.te[L];
  const int32_t t0 = w.tr[0];
  const uint32_t n_src = w.size[L];
  uint32_t cnt = 0;
  // A part: surviving canonical candidates, mask gains bit L
  for (uint32_t i0 = 0; i0 < n_src; i0 += 32) {
    const uint32_t i = i0 + lane;
    bool keep = false;
    uint32_t val = 0;
    if (i < n_src) {
      const uint32_t ent = __ldcg(src + i);
      const int32_t e = (int32_t)(ent & a.vmask);
      if (e > x) {
        const bool hit = adj_tr(a, w, L, e);
        val = ent | ((uint32_t)hit << (a.vbits + L));
        keep = true;
      }
    }
    emit(dst, cnt, keep, val);
  }
  // B part: neighbours of w new to the traversal's neighbourhood
  for (long long p0 = row_first_above(a.nbr, xb, xe, t0); p0 < xe; p0 += 32) {
    const long long p = p0 + lane;
    bool keep = false;
    uint32_t val = 0;
    if (p < xe) {
      const int32_t e = __ldg(a.nbr + p);
      if (e > t0) {
        keep = adj_none(a, w, L, e);
        val = (uint32_t)e | (1u << (a.vbits + L));
      }
    }
    emit(dst, cnt, keep, val);
  }
  return cnt;
}

// WM_MOTIF_PROF=1 (tuning builds only): per-phase SM cycles summed over warps
// into counters[20..27] — [20] idle (acquire_work) [21] donated-prefix
// rebuild [22] level builds [23] leaf aggregation [24] leaf steps [25] max
// single leaf step [26] records received; [28..31] leaf-step candidates:
// A scanned, A kept (e > x), B scanned, B kept — printed by run_motif.
#ifndef WM_MOTIF_PROF
#define WM_MOTIF_PROF 0
#endif
#if WM_MOTIF_PROF
#define WM_PT(v) const long long v = clock64()
#define WM_PACC(slot, t0) (prof[slot] += (unsigned long long)(clock64() - (t0)))
#else
#define WM_PT(v)
#define WM_PACC(slot, t0)
#endif

// dictionary lookup (aggregate.py:189); SENTINEL >= pattern_count either way
__device__ __forceinline__ uint32_t dict_lookup(const MotifArgs &a, uint32_t bits) {
  return a.table16 ? (uint32_t)__ldg(a.table16 + bits) : __ldg(a.table + bits);
}

// bump hist[pid] by the number of lanes sharing pid (lanes with valid)
__device__ __forceinline__ void hist_add(const MotifArgs &a, unsigned long long *sh, bool valid,
                                         uint32_t pid) {
  const int lane = lane_id();
  const uint32_t key = valid ? pid : 0xFFFFFFFEu;
  const unsigned mm = __match_any_sync(0xffffffffu, key);
  if (valid && lane == __ffs(mm) - 1) {
    if (a.smem_hist) atomicAdd(sh + pid, (unsigned long long)__popc(mm));
    else atomicAdd(a.hist + pid, (unsigned long long)__popc(mm));
  }
}

// leaves of the traversal tr[0..k-1) (w = tr[k-2]); returns the warp total
__device__ __forceinline__ unsigned long long aggregate_leaves(const MotifArgs &a, MotifWarp &w,
                                                               uint32_t *base,
                                                               unsigned long long *sh) {
  const int lane = lane_id();
  const int L = a.k - 2;  // E_L holds the candidates of tr[0..L)
  const uint32_t *src = level_ptr(a, base, L);
  const int32_t x = w.tr[L];
  const long long xb = w.tb[L], xe = w.te[L];
  const int32_t t0 = w.tr[0];
  const uint32_t bits = (uint32_t)w.bm[L];  // bitmap of tr[0..k-1) (k <= 8 here)
  const int off = group_off(a.k - 1);
  const uint32_t n_src = w.size[L];
  unsigned long long total = 0;
  bool bad = false;
  for (uint32_t i0 = 0; i0 < n_src; i0 += 32) {
    const uint32_t i = i0 + lane;
    bool valid = false;
    uint32_t pid = 0;
    if (i < n_src) {
      const uint32_t ent = __ldcg(src + i);
      const int32_t e = (int32_t)(ent & a.vmask);
      if (e > x) {
        const uint32_t mask = (ent >> a.vbits) | ((uint32_t)adj_tr(a, w, L, e) << L);
        pid = dict_lookup(a, bits | (mask << off));
        valid = true;
        bad |= pid >= a.pattern_count;
      }
    }
    total += __popc(__ballot_sync(0xffffffffu, valid));
    hist_add(a, sh, valid && pid < a.pattern_count, pid);
  }
  unsigned long long nb = 0;
  const long long pb = row_first_above(a.nbr, xb, xe, t0);
#if WM_MOTIF_PROF
  if (lane == 0) {
    atomicAdd(&a.counters[28], (unsigned long long)n_src);
    atomicAdd(&a.counters[29], total);
    atomicAdd(&a.counters[30], (unsigned long long)(xe - pb));
  }
#endif
  for (long long p0 = pb; p0 < xe; p0 += 32) {
    const long long p = p0 + lane;
    bool keep = false;
    if (p < xe) {
      const int32_t e = __ldg(a.nbr + p);
      if (e > t0) keep = adj_none(a, w, L, e);
    }
    nb += __popc(__ballot_sync(0xffffffffu, keep));
  }
  if (nb) {
    const uint32_t pid = dict_lookup(a, bits | ((1u << L) << off));
    if (pid >= a.pattern_count) bad = true;
    else if (lane == 0) {
      if (a.smem_hist) atomicAdd(sh + pid, nb);
      else atomicAdd(a.hist + pid, nb);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_error(a.L.lb, WM_EINVARIANT);
#if WM_MOTIF_PROF
  if (lane == 0) atomicAdd(&a.counters[31], nb);
#endif
  return total + nb;
}


using aref_sys_u64 = cuda::atomic_ref<unsigned long long, cuda::thread_scope_system>;
using aref_sys_u32 = cuda::atomic_ref<uint32_t, cuda::thread_scope_system>;

// Warp-collective: stream one record per lane with `keep` (leaf e with
// adjacency mask) to the host ring, in rank order.  Returns false once the
// consumer has failed (aggregate.py:88-99); the warp then stops producing.
__device__ __forceinline__ bool emit_records(const MotifArgs &a, MotifWarp &w, bool keep,
                                             int32_t e, uint32_t mask) {
  const ListRing &R = a.ring;
  const int lane = lane_id();
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (!bal) return true;
  const int n = __popc(bal);
  const int rank = __popc(bal & ((1u << lane) - 1u));
  if (keep) {
    w.le[rank] = e;
    w.lm[rank] = mask;
  }
  unsigned long long base = 0;
  int ok = 1;
  if (lane == 0) {
    base = atomicAdd(R.head, (unsigned long long)n);
    // back-pressure: tickets [base, base+n) need free slots.  The consumer's
    // tail lives in host memory; it is read only when the cached copy says
    // the ring may be full.
    const unsigned long long need = base + (unsigned long long)n;
    unsigned sl = 128;
    while (need > w.tail_cache + R.cap_mask + 1ull) {
      w.tail_cache = aref_u64(R.ctl[0]).load(cuda::std::memory_order_relaxed);
      if (need <= w.tail_cache + R.cap_mask + 1ull) break;
      if (aref_u64(R.ctl[1]).load(cuda::std::memory_order_relaxed) ||
          ld_relaxed(&a.L.lb->error)) {
        ok = 0;
        break;
      }
      __nanosleep(sl);
      if (sl < 8192) sl <<= 1;
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (!ok) {
    if (lane == 0) raise_error(a.L.lb, WM_ESHUTDOWN);
    return false;
  }
  __syncwarp();
  // record payload, coalesced over the warp
  const uint32_t st = R.stride;
  const int nw = n * (int)st;
  const unsigned long long bm = w.bm[a.k - 2];
  for (int i = lane; i < nw; i += 32) {
    const int r = i / (int)st, j = i - r * (int)st;
    uint32_t v;
    if (j == 0) v = (uint32_t)(base + (unsigned long long)r + 1ull);  // ticket + 1
    else if (j == 1) v = (uint32_t)w.le[r];
    else if (j == 2) v = w.lm[r];
    else if (j == 3) v = (uint32_t)bm;
    else if (j == 4) v = (uint32_t)(bm >> 32);
    else v = (uint32_t)w.tr[j - 5];
    R.slots[((base + (unsigned long long)r) & R.cap_mask) * st + j] = v;
  }
  __threadfence();
  __syncwarp();
  // completion counts per ring block (a warp's tickets span at most two)
  if (lane == 0) {
    const unsigned long long b0 = base >> R.block_shift, b1 = (base + n - 1) >> R.block_shift;
    const uint32_t nblk = (uint32_t)(R.cap_mask >> R.block_shift);  // block count - 1
    if (b0 == b1) {
      atomicAdd(R.blockdone + (b0 & nblk), (uint32_t)n);
    } else {
      const uint32_t n0 = (uint32_t)((b1 << R.block_shift) - base);
      atomicAdd(R.blockdone + (b0 & nblk), n0);
      atomicAdd(R.blockdone + (b1 & nblk), (uint32_t)n - n0);
    }
  }
  return true;
}

// listing leaves of tr[0..k-1): same candidates as aggregate_leaves, every
// one streamed as a record (aggregate_store, aggregate.py:199-223).  Returns
// the leaves found (aggregated_total); *emitted counts records that passed
// the device filter; *ok turns false when the consumer failed.
__device__ __forceinline__ unsigned long long list_leaves(const MotifArgs &a, MotifWarp &w,
                                                          uint32_t *base,
                                                          unsigned long long &emitted,
                                                          bool &ok) {
  const int lane = lane_id();
  const int L = a.k - 2;
  const uint32_t *src = level_ptr(a, base, L);
  const int32_t x = w.tr[L];
  const long long xb = w.tb[L], xe = w.te[L];
  const int32_t t0 = w.tr[0];
  const uint32_t n_src = w.size[L];
  const bool complete_only = a.ring.filter == WM_LIST_COMPLETE;
  const bool prefix_full = w.bm[L] == a.ring.full_prefix;
  unsigned long long total = 0;
  for (uint32_t i0 = 0; i0 < n_src && ok; i0 += 32) {
    const uint32_t i = i0 + lane;
    bool valid = false;
    int32_t e = 0;
    uint32_t mask = 0;
    if (i < n_src) {
      const uint32_t ent = __ldcg(src + i);
      e = (int32_t)(ent & a.vmask);
      if (e > x) {
        mask = (ent >> a.vbits) | ((uint32_t)adj_tr(a, w, L, e) << L);
        valid = true;
      }
    }
    total += __popc(__ballot_sync(0xffffffffu, valid));
    const bool keep = valid && (!complete_only || (prefix_full && mask == a.ring.full_mask));
    emitted += __popc(__ballot_sync(0xffffffffu, keep));
    ok = emit_records(a, w, keep, e, mask);
  }
  // B part (mask = 1 << L: e sees only tr[L], never complete for k >= 3)
  for (long long p0 = row_first_above(a.nbr, xb, xe, t0); p0 < xe && ok; p0 += 32) {
    const long long p = p0 + lane;
    bool keep = false;
    int32_t e = 0;
    if (p < xe) {
      e = __ldg(a.nbr + p);
      if (e > t0) keep = adj_none(a, w, L, e);
    }
    total += __popc(__ballot_sync(0xffffffffu, keep));
    const bool out = keep && (!complete_only || (prefix_full && (1u << L) == a.ring.full_mask));
    emitted += __popc(__ballot_sync(0xffffffffu, out));
    ok = emit_records(a, w, out, e, 1u << L);
  }
  return total;
}

__device__ __forceinline__ void set_tr(const MotifArgs &a, MotifWarp &w, int j, int32_t v) {
  if (lane_id() == 0) {
    w.tr[j] = v;
    w.tb[j] = __ldg(a.off + v);
    w.te[j] = __ldg(a.off + v + 1);
  }
  __syncwarp();
}

constexpr int kMotifHdr = 6;  // [root, level, lo, hi, bitmap lo, bitmap hi] then tr[1..level)
// BYTES records also carry the donor's claimed mask and claim slots of the
// shared nodes 1..level: word kMotifClaimMask, then kMotifClaim + L - 1
constexpr int kMotifClaimMask = kMotifHdr + kMaxK - 1;
constexpr int kMotifClaim = kMotifHdr + kMaxK;
constexpr int kMotifRecWords = kMotifClaim + kMaxK;

// A leaf-parent node of length L produced leaves: it and every ancestor are
// productive.  Count each node's 4 * deg(last) exactly once over all warps:
// private nodes directly, shared nodes through their claim slot (first
// atomicExch wins).  A claimed node's ancestors are claimed already, so the
// walk stops at the first one.  Lane 0.
__device__ __forceinline__ void claim_path(const MotifArgs &a, MotifWarp &w, int L,
                                           unsigned long long &bytes) {
  for (; L >= 1; --L) {
    if ((w.claimed >> L) & 1u) break;
    w.claimed |= 1u << L;
    const uint32_t c = w.claim[L];
    if (c == kNoClaim || atomicExch(a.claims + c, 1u) == 0u) {
      bytes += 4ull * (unsigned long long)(w.te[L - 1] - w.tb[L - 1]);
    } else {
      w.claimed |= (1u << L) - 1u;  // another warp claimed this node and its ancestors
      break;
    }
  }
}

// Before donating children of the node of length sd: give every unclaimed
// private node 1..sd a global claim slot (the thief shares them).  Lane 0;
// false when the slot table is full (the caller then skips the donation).
__device__ __forceinline__ bool share_claims(const MotifArgs &a, MotifWarp &w, int sd) {
  int need = 0;
  for (int L = 1; L <= sd; ++L)
    if (!((w.claimed >> L) & 1u) && w.claim[L] == kNoClaim) ++need;
  if (!need) return true;
  const unsigned long long base = atomicAdd(a.claim_ctr, (unsigned long long)need);
  if (base + need > a.claim_cap) return false;
  uint32_t c = (uint32_t)base;
  for (int L = 1; L <= sd; ++L)
    if (!((w.claimed >> L) & 1u) && w.claim[L] == kNoClaim) w.claim[L] = c++;
  return true;
}

// a leaf-level range is donated only if it carries >= this many candidate scans
// (4,096 after leaf_bulk: cfg5 k=7 26.7 -> 26.0 ms, cfg4 k=6 83.9 -> 83.5, k=5
// unchanged; 16,384 and 256 slower, profiles/r02_ab_motif_donate.log)
#ifndef WM_MOTIF_DONATE_MIN
#define WM_MOTIF_DONATE_MIN 4096ull
#endif
// blocks per SM the register budget must allow.  Before leaf_bulk: 4 (64
// registers) for k <= 5, 6 (40 registers) for k >= 6 (profiles/r02_ab_motif_mb.log).
// With leaf_bulk and the per-warp counters in shared memory, 5 (48 registers)
// for every k: cfg4 k=5 2.83 -> 2.69 ms, k=6 83.0 -> 79.9, cfg5 k=7 25.5 -> 25.2
// (profiles/r02_ab_motif_occupancy_v2.log)
#ifndef WM_MOTIF_MINBLOCKS
#define WM_MOTIF_MINBLOCKS 5
#endif
#ifndef WM_MOTIF_MINBLOCKS_DEEP
#define WM_MOTIF_MINBLOCKS_DEEP 5
#endif
#ifndef WM_MOTIF_LEAF_BULK
#define WM_MOTIF_LEAF_BULK 1
#endif


// multi-GPU dealing (MotifArgs::l1_offset): true when the entry popped at
// level s (vertex v, index cur - 1) belongs to another shard
__device__ __forceinline__ bool other_shard(const MotifArgs &a, const MotifWarp &w, int s,
                                            uint32_t cur, int32_t v) {
  if (a.l1_stride <= 1) return false;
  if (s == 1 && a.shard_level == 1)
    return ((cur - 1) + (uint32_t)w.tr[0]) % a.l1_stride != a.l1_offset;
  if (s == 2 && a.shard_level == 2) {
    uint32_t h = (uint32_t)w.tr[0] * 0x9E3779B1u ^ (uint32_t)w.tr[1] * 0x85EBCA77u ^
                 (uint32_t)v * 0xC2B2AE3Du;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    return h % a.l1_stride != a.l1_offset;
  }
  return false;
}

// On-device load balancing, one poll (after each node): when enough warps are
// idle, donate half of the pending entries of the shallowest level s0..s that
// has >= 2 (reference balance.py:102-128 steals the shallowest pending entry).
// The poll is software-pipelined: the idle/donor ticket counters loaded at
// one poll (lane 0, into lbt/lbh) are consumed at the next, so the L2 round
// trip never stalls the enumeration (cfg4 k=6 87.9 -> 84.9 ms, idle fraction
// 0.098 -> 0.026; cfg5 k=7 28.3 -> 26.2, profiles/r02_ab_motif_v2.log).
template <bool BYTES>
__device__ __forceinline__ void poll_donate(const MotifArgs &a, MotifWarp &w, int s0, int s,
                                            int &poll) {
  const int lane = lane_id();
  if (!(a.lb_on && ++poll >= a.lb_poll)) return;
  poll = 0;
  int want = 0;
  if (lane == 0) {
    ++w.n_polls;
    want = (int)(w.lbt - w.lbh) >= a.idle_min;
    w.lbt = (uint32_t)ld_relaxed(&a.L.lb->tail);
    w.lbh = (uint32_t)ld_relaxed(&a.L.lb->head);
  }
  if (!__shfl_sync(0xffffffffu, want, 0)) return;
  int sd = -1;
  for (int j = s0; j <= s; ++j)
    if (w.cur[j] - w.lo[j] >= 2u) { sd = j; break; }
  if (sd < 0) return;
  const uint32_t pend = w.cur[sd] - w.lo[sd];
  bool worth = sd < a.k - 2 || (unsigned long long)pend * w.size[sd] >= WM_MOTIF_DONATE_MIN;
  if (BYTES && worth) {
    int ok_share = 0;
    if (lane == 0) ok_share = share_claims(a, w, sd);
    worth = __shfl_sync(0xffffffffu, ok_share, 0) != 0;
    __syncwarp();  // lane 0's claim slots visible to the record build
  }
  if (!worth) return;
  const uint32_t half = pend / 2;
  const uint32_t lo = w.lo[sd];
  Rec3 r;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int idx = 32 * q + lane;
    uint32_t val = 0;
    if (idx == 0) val = (uint32_t)w.tr[0];
    else if (idx == 1) val = (uint32_t)sd;
    else if (idx == 2) val = lo;
    else if (idx == 3) val = lo + half;
    else if (idx == 4) val = (uint32_t)w.bm[sd - 1];
    else if (idx == 5) val = (uint32_t)(w.bm[sd - 1] >> 32);
    else if (idx >= kMotifHdr && idx < kMotifHdr + sd - 1) val = (uint32_t)w.tr[idx - kMotifHdr + 1];
    else if (BYTES && idx == kMotifClaimMask) val = w.claimed & ((2u << sd) - 1u);
    else if (BYTES && idx >= kMotifClaim && idx < kMotifClaim + sd)
      val = w.claim[idx - kMotifClaim + 1];
    r.w[q] = val;
  }
  donate_record(a.L, r);
  if (lane == 0) {
    w.lo[sd] = lo + half;
    atomicAdd(&a.L.lb->migrations, (unsigned long long)half);
    atomicAdd(&a.L.lb->donation_polls, 1ull);
  }
  __syncwarp();
}

// One round of leaf_bulk's A ring: each lane takes one leaf (x, e) with e in
// E_L, e > x — the A part of aggregate_leaves for its own x — probes
// adj(e, x), looks the leaf's bitmap up and bumps the histogram.
__device__ __forceinline__ uint32_t leaf_round_a(const MotifArgs &a, const uint2 *ring, int head,
                                                 int cnt, uint32_t bml, int offL, int offK,
                                                 int L, unsigned long long *sh, bool &bad) {
  const int lane = lane_id();
  bool valid = false;
  uint32_t pid = 0;
  if (lane < cnt) {
    const uint2 p = ring[(head + lane) & 63];
    const int32_t x = (int32_t)(p.x & a.vmask), e = (int32_t)(p.y & a.vmask);
    const uint32_t adj = edge_hash_contains(a.H, e, x) ? 1u : 0u;
    const uint32_t mask = (p.y >> a.vbits) | (adj << L);
    pid = dict_lookup(a, bml | ((p.x >> a.vbits) << offL) | (mask << offK));
    valid = true;
    bad |= pid >= a.pattern_count;
  }
  hist_add(a, sh, valid && pid < a.pattern_count, pid);
  return __popc(__ballot_sync(0xffffffffu, valid));
}

// One round of the B ring: lane takes one (x, e), e in N(x), e > tr[0]; e is
// a leaf iff it is adjacent to none of tr[0..L) (its mask is 1 << L).
__device__ __forceinline__ uint32_t leaf_round_b(const MotifArgs &a, const MotifWarp &w,
                                                 const uint2 *ring, int head, int cnt,
                                                 uint32_t bml, int offL, int offK, int L,
                                                 unsigned long long *sh, bool &bad) {
  const int lane = lane_id();
  bool keep = false;
  uint32_t pid = 0;
  if (lane < cnt) {
    const uint2 p = ring[(head + lane) & 63];
    keep = adj_none(a, w, L, (int32_t)p.y);
    if (keep) {
      pid = dict_lookup(a, bml | ((p.x >> a.vbits) << offL) | ((1u << L) << offK));
      bad |= pid >= a.pattern_count;
    }
  }
  hist_add(a, sh, keep && pid < a.pattern_count, pid);
  return __popc(__ballot_sync(0xffffffffu, keep));
}

// All pending children x of a node of length L = k-2 (entries [lo, cur) of
// E_L), i.e. every leaf-parent below it, in one pass.  aggregate_leaves per x
// leaves most lanes idle: E_L holds ~30-70 entries of which half exceed x, and
// N(x) above tr[0] ~10 (cfg4/cfg5 counters, profiles/r02_motif_prof.log).
// Here the leaves of successive x are flattened through two 64-entry rings
// in shared memory — A leaves (x, e in E_L, e > x) and B leaves (x, e in
// N(x), e > tr[0]) — and resolved 32 at a time, one leaf per lane: the
// probes, dictionary lookups and histogram updates run with full lanes.
// Same leaves, same patterns as the per-x pass (the histogram is a sum);
// balancer polls and shard dealing stay per x.
template <bool BYTES>
__device__ __forceinline__ unsigned long long leaf_bulk(const MotifArgs &a, MotifWarp &w,
                                                        uint32_t *base, unsigned long long *sh,
                                                        int s0, int &poll) {
  const int lane = lane_id();
  const uint32_t lt = (1u << lane) - 1u;
  const int L = a.k - 2;
  const uint32_t *src = level_ptr(a, base, L);
  const uint32_t n = w.size[L];
  const uint32_t bml = (uint32_t)w.bm[L - 1];  // bitmap of tr[0..L) (k <= 8)
  const int offL = group_off(L), offK = group_off(L + 1);
  const int32_t t0 = w.tr[0];
  unsigned long long total = 0;
  bool bad = false;
  int ha = 0, na = 0, hb = 0, nb = 0;  // warp-uniform ring state
  for (;;) {
    const uint32_t cur = w.cur[L];
    if (cur == w.lo[L]) break;
    const uint32_t ex = __ldcg(src + (cur - 1));
    const int32_t x = (int32_t)(ex & a.vmask);
    __syncwarp();  // every lane's read of w.cur precedes lane 0's write
    if (lane == 0) w.cur[L] = cur - 1;
    __syncwarp();
    if (other_shard(a, w, L, cur, x)) continue;
    if (lane == 0) ++w.n_nodes;
    // A leaves: e in E_L above x
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint32_t ent = i < n ? __ldcg(src + i) : 0u;
      const bool keep = i < n && (int32_t)(ent & a.vmask) > x;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) w.ra[(ha + na + __popc(bal & lt)) & 63] = make_uint2(ex, ent);
      na += __popc(bal);
      if (na >= 32) {
        __syncwarp();
        total += leaf_round_a(a, w.ra, ha, 32, bml, offL, offK, L, sh, bad);
        __syncwarp();
        ha = (ha + 32) & 63;
        na -= 32;
      }
    }
    // B leaves: N(x) above tr[0] (rows ascending; a scan from the row start
    // with an e > tr[0] test measured the same, profiles/r02_ab_motif_v2.log)
    const long long xb = __ldg(a.off + x), xe = __ldg(a.off + x + 1);
    for (long long p0 = row_first_above(a.nbr, xb, xe, t0); p0 < xe; p0 += 32) {
      const long long p = p0 + lane;
      const bool keep = p < xe;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) w.rb[(hb + nb + lane) & 63] = make_uint2(ex, (uint32_t)__ldg(a.nbr + p));
      nb += __popc(bal);
      if (nb >= 32) {
        __syncwarp();
        total += leaf_round_b(a, w, w.rb, hb, 32, bml, offL, offK, L, sh, bad);
        __syncwarp();
        hb = (hb + 32) & 63;
        nb -= 32;
      }
    }
    poll_donate<BYTES>(a, w, s0, L, poll);
  }
  __syncwarp();
  if (na) total += leaf_round_a(a, w.ra, ha, na, bml, offL, offK, L, sh, bad);
  if (nb) total += leaf_round_b(a, w, w.rb, hb, nb, bml, offL, offK, L, sh, bad);
  __syncwarp();
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_error(a.L.lb, WM_EINVARIANT);
  return total;
}

template <bool BYTES, bool LIST, int MINB>
__global__ void __launch_bounds__(256, MINB) motif_enum_kernel(MotifArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned long long *sh = reinterpret_cast<unsigned long long *>(smraw);
  MotifWarp *warps = reinterpret_cast<MotifWarp *>(
      smraw + (a.smem_hist ? ((size_t)a.pattern_count * 8 + 15) / 16 * 16 : 0));
  MotifWarp &w = warps[threadIdx.x >> 5];
  const int lane = lane_id();
  const int k = a.k;
  if (a.smem_hist) {
    for (uint32_t i = threadIdx.x; i < a.pattern_count; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  const unsigned long long gw = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  uint32_t *base = a.arena + gw * a.warp_stride;
  WarpClock clk;
  warp_clock_begin(clk, a.L.lb);
  bool roots_left = true;
  unsigned long long bytes = 0;
  unsigned long long emitted = 0;
  bool ok = true;
  if (LIST && lane == 0) w.tail_cache = 0;
  int poll = 0;
  if (lane == 0) {
    w.n_leaves = w.n_nodes = w.n_polls = w.n_peak = w.n_tasks = 0;
    w.lbt = w.lbh = 0;
  }
  __syncwarp();
#if WM_MOTIF_PROF
  unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  while (ok) {
    unsigned long long ti = 0;
    Rec3 rec = {{0u, 0u, 0u}};
    WM_PT(tq);
    const int kind = acquire_work(a.L, a.lb_on, a.ntasks, roots_left, ti, rec, clk);
    WM_PACC(0, tq);
    if (kind == 0) break;
    int s0;
    WM_PT(tr0);
    if (kind == 1) {
      set_tr(a, w, 0, __ldg(a.tasks + a.task_offset + ti * a.task_stride));
      if (lane == 0) {
        w.bm[0] = 0;
        w.claimed = 0;
        w.claim[1] = kNoClaim;
      }
      __syncwarp();
      const uint32_t n1 = build_first(a, w, base);
      if (lane == 0) {
        w.size[1] = n1;
        w.cur[1] = n1;
        w.lo[1] = 0;
      }
      s0 = 1;
      if (lane == 0) ++w.n_tasks;
    } else {
      // donated prefix: rebuild E_1..E_s0 deterministically, then own [lo, hi)
      s0 = (int)rec_word(rec, 1);
      const uint32_t lo = rec_word(rec, 2), hi = rec_word(rec, 3);
      const unsigned long long bm =
          (unsigned long long)rec_word(rec, 4) | ((unsigned long long)rec_word(rec, 5) << 32);
      set_tr(a, w, 0, (int32_t)rec_word(rec, 0));
      for (int j = 1; j < s0; ++j) set_tr(a, w, j, (int32_t)rec_word(rec, kMotifHdr + j - 1));
      uint32_t n = build_first(a, w, base);
      if (lane == 0) w.size[1] = n;
      __syncwarp();
      for (int j = 1; j < s0; ++j) {
        n = build_next(a, w, base, j);
        if (lane == 0) w.size[j + 1] = n;
        __syncwarp();
      }
      if (BYTES) {
        const uint32_t cm = rec_word(rec, kMotifClaimMask);
        uint32_t cl[kMaxK];
#pragma unroll
        for (int j = 1; j < kMaxK; ++j) cl[j] = rec_word(rec, kMotifClaim + j - 1);
        if (lane == 0) {
          w.claimed = cm;
          for (int j = 1; j <= s0; ++j) w.claim[j] = cl[j];
        }
      }
      if (lane == 0) {
        w.bm[s0 - 1] = bm;
        w.cur[s0] = hi;
        w.lo[s0] = lo;
      }
#if WM_MOTIF_PROF
      prof[6] += 1;
#endif
    }
    __syncwarp();
    WM_PACC(kind == 1 ? 2 : 1, tr0);
    int s = s0;
    for (;;) {
      const uint32_t cur = w.cur[s];
      if (cur == w.lo[s]) {
        // level exhausted: the node of length s is complete
        if (s == s0) break;
        --s;
        continue;
      }
#if WM_MOTIF_LEAF_BULK
      if (!BYTES && !LIST && s == k - 2 && k >= 4 && a.H.b) {
        // the node's children are leaf-parents: all of them in one pass
        WM_PT(tl);
        const unsigned long long got = leaf_bulk<BYTES>(a, w, base, sh, s0, poll);
        if (lane == 0) w.n_leaves += got;
        WM_PACC(3, tl);
        continue;
      }
#endif
      // move_step: pop the highest pending entry (engine.py:652-669)
      const uint32_t ent = __ldcg(level_ptr(a, base, s) + (cur - 1));
      const int32_t v = (int32_t)(ent & a.vmask);
      if (other_shard(a, w, s, cur, v)) {
        // another shard's edge task / (root, child, grandchild): consume without descending
        if (lane == 0) w.cur[s] = cur - 1;
        __syncwarp();
        continue;
      }
      const uint32_t m = ent >> a.vbits;
      set_tr(a, w, s, v);
      if (lane == 0) {
        if (BYTES) {  // a fresh node of length s + 1
          w.claimed &= ~(1u << (s + 1));
          w.claim[s + 1] = kNoClaim;
        }
        w.cur[s] = cur - 1;
        // induce (engine.py:678-705): bitmap of tr[0..s] (s+1 vertices)
        w.bm[s] = (s == 1) ? 0ull
                           : (w.bm[s - 1] | ((unsigned long long)m << group_off(s)));
      }
      __syncwarp();
      if (lane == 0) ++w.n_nodes;
      if (s + 1 == k - 1) {
        unsigned long long got;
        WM_PT(tl);
        if (LIST) {
          got = list_leaves(a, w, base, emitted, ok);
          if (!ok) break;
        } else {
          got = aggregate_leaves(a, w, base, sh);
        }
#if WM_MOTIF_PROF
        {
          const unsigned long long d = (unsigned long long)(clock64() - tl);
          prof[3] += d;
          prof[4] += 1;
          if (d > prof[5]) prof[5] = d;
        }
#endif
        if (lane == 0) w.n_leaves += got;
        if (BYTES && lane == 0 && got) claim_path(a, w, s + 1, bytes);
        __syncwarp();
      } else {
        WM_PT(tb);
        const uint32_t n = build_next(a, w, base, s);
        WM_PACC(2, tb);
        if ((long long)n > (long long)(s + 1) * a.maxdeg && lane == 0)
          raise_error(a.L.lb, WM_ECAPACITY);
        if (lane == 0) {
          w.size[s + 1] = n;
          w.cur[s + 1] = n;
          w.lo[s + 1] = 0;
        }
        if (lane == 0) {
          unsigned long long live = 0;
          for (int j = 1; j <= s + 1; ++j) live += w.size[j];
          if (live > w.n_peak) w.n_peak = live;
        }
        __syncwarp();
        ++s;
      }
      // on-device load balancing: donate half of the shallowest pending range
      poll_donate<BYTES>(a, w, s0, s, poll);
    }
  }
  __syncwarp();
  if (lane == 0) {
    atomicAdd(&a.counters[0], w.n_leaves);
    if (BYTES) atomicAdd(&a.counters[1], bytes);
    atomicAdd(&a.counters[2], w.n_tasks);
    atomicAdd(&a.counters[3], w.n_nodes);
    atomicAdd(&a.counters[4], w.n_polls);
    atomicMax(&a.counters[5], w.n_peak);
    if (LIST) atomicAdd(&a.counters[6], emitted);
#if WM_MOTIF_PROF
    for (int q = 0; q < 7; ++q) {
      if (q == 5) atomicMax(&a.counters[25], prof[5]);
      else atomicAdd(&a.counters[20 + q], prof[q]);
    }
#endif
  }
  warp_clock_end(a.L.lb, clk);
  if (a.smem_hist) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < a.pattern_count; i += blockDim.x)
      if (sh[i]) atomicAdd(a.hist + i, sh[i]);
  }
}


// --------------------------------------------------------------------------
// DM_DFS ablation (mode "dfs", reference engine.py:13-16, :274-294): one
// THREAD per traversal running the same E-recurrence as the warp kernel with
// scalar loops — no ballot compaction, no cooperative probes, per-leaf
// histogram atomics.  Same tree, same histograms / records.

// scalar record emission (one ticket per record)
__device__ __forceinline__ bool emit_one(const MotifArgs &a, unsigned long long &tail_cache,
                                         const int32_t *tr, unsigned long long bm, int32_t e,
                                         uint32_t mask) {
  const ListRing &R = a.ring;
  const unsigned long long idx = atomicAdd(R.head, 1ull);
  unsigned sl = 128;
  while (idx + 1ull > tail_cache + R.cap_mask + 1ull) {
    tail_cache = aref_u64(R.ctl[0]).load(cuda::std::memory_order_relaxed);
    if (idx + 1ull <= tail_cache + R.cap_mask + 1ull) break;
    if (aref_u64(R.ctl[1]).load(cuda::std::memory_order_relaxed) ||
        ld_relaxed(&a.L.lb->error)) {
      raise_error(a.L.lb, WM_ESHUTDOWN);
      return false;
    }
    __nanosleep(sl);
    if (sl < 8192) sl <<= 1;
  }
  uint32_t *slot = R.slots + (idx & R.cap_mask) * R.stride;
  slot[0] = (uint32_t)(idx + 1ull);
  slot[1] = (uint32_t)e;
  slot[2] = mask;
  slot[3] = (uint32_t)bm;
  slot[4] = (uint32_t)(bm >> 32);
  for (int j = 0; j < a.k - 1; ++j) slot[5 + j] = (uint32_t)tr[j];
  __threadfence();
  atomicAdd(R.blockdone + ((idx >> R.block_shift) & (R.cap_mask >> R.block_shift)), 1u);
  return true;
}

template <bool LIST>
__global__ void __launch_bounds__(256) motif_dfs_kernel(MotifArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned long long *sh = reinterpret_cast<unsigned long long *>(smraw);
  if (a.smem_hist) {
    for (uint32_t i = threadIdx.x; i < a.pattern_count; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t *base = a.arena + tid * a.warp_stride;
  const int k = a.k;
  const int L = k - 2;  // leaf level: E_L holds the candidates of tr[0..k-1)
  const int off = group_off(k - 1);
  const bool complete_only = LIST && a.ring.filter == WM_LIST_COMPLETE;
  int32_t tr[kMaxK];
  long long tb[kMaxK], te[kMaxK];
  unsigned long long bm[kMaxK];
  uint32_t size[kMaxK], cur[kMaxK];
  unsigned long long leaves = 0, emitted = 0, nodes = 0, done = 0, tail_cache = 0;
  bool ok = true, bad = false;
  while (ok) {
    const unsigned long long ti = atomicAdd(&a.counters[16], 1ull);  // engine.py:187
    if (ti >= a.ntasks) break;
    ++done;
    const int32_t r = __ldg(a.tasks + a.task_offset + ti * a.task_stride);
    tr[0] = r;
    tb[0] = __ldg(a.off + r);
    te[0] = __ldg(a.off + r + 1);
    bm[0] = 0;
    uint32_t *l1 = level_ptr(a, base, 1);
    uint32_t n1 = 0;
    for (long long p = tb[0]; p < te[0]; ++p) {
      const int32_t e = __ldg(a.nbr + p);
      if (e > r) l1[n1++] = (uint32_t)e | (1u << a.vbits);
    }
    size[1] = cur[1] = n1;
    int s = 1;
    while (ok) {
      if (cur[s] == 0) {
        if (s == 1) break;
        --s;
        continue;
      }
      const uint32_t ent = level_ptr(a, base, s)[--cur[s]];
      const int32_t x = (int32_t)(ent & a.vmask);
      tr[s] = x;
      tb[s] = __ldg(a.off + x);
      te[s] = __ldg(a.off + x + 1);
      bm[s] = (s == 1) ? 0ull
                       : (bm[s - 1] | ((unsigned long long)(ent >> a.vbits) << group_off(s)));
      ++nodes;
      const uint32_t *src = level_ptr(a, base, s);
      if (s == L) {
        // leaves of tr[0..k-1): A part (E_L, mask gains bit L), B part (N(x))
        for (uint32_t i = 0; i < size[s] && ok; ++i) {
          const uint32_t en = src[i];
          const int32_t e = (int32_t)(en & a.vmask);
          if (e <= x) continue;
          const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
          const uint32_t mask =
              (en >> a.vbits) | ((uint32_t)adj_probe(a.nbr, e, eb, ee, x, tb[s], te[s]) << L);
          ++leaves;
          if (LIST) {
            if (!complete_only || (bm[L] == a.ring.full_prefix && mask == a.ring.full_mask)) {
              ok = emit_one(a, tail_cache, tr, bm[L], e, mask);
              ++emitted;
            }
          } else {
            const uint32_t pid = dict_lookup(a, (uint32_t)bm[L] | (mask << off));
            if (pid >= a.pattern_count) bad = true;
            else if (a.smem_hist) atomicAdd(sh + pid, 1ull);
            else atomicAdd(a.hist + pid, 1ull);
          }
        }
        unsigned long long nb = 0;
        for (long long p = tb[s]; p < te[s] && ok; ++p) {
          const int32_t e = __ldg(a.nbr + p);
          if (e <= r) continue;
          const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
          bool keep = true;
          for (int j = 0; j < L && keep; ++j)
            keep = !adj_probe(a.nbr, e, eb, ee, tr[j], tb[j], te[j]);
          if (!keep) continue;
          ++nb;
          if (LIST && !complete_only) {
            ok = emit_one(a, tail_cache, tr, bm[L], e, 1u << L);
            ++emitted;
          }
        }
        leaves += nb;
        if (!LIST && nb) {
          const uint32_t pid = dict_lookup(a, (uint32_t)bm[L] | ((1u << L) << off));
          if (pid >= a.pattern_count) bad = true;
          else if (a.smem_hist) atomicAdd(sh + pid, nb);
          else atomicAdd(a.hist + pid, nb);
        }
        continue;
      }
      // E_{s+1} from E_s and x = tr[s]
      uint32_t *dst = level_ptr(a, base, s + 1);
      uint32_t n = 0;
      for (uint32_t i = 0; i < size[s]; ++i) {
        const uint32_t en = src[i];
        const int32_t e = (int32_t)(en & a.vmask);
        if (e <= x) continue;
        const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
        dst[n++] = en | ((uint32_t)adj_probe(a.nbr, e, eb, ee, x, tb[s], te[s]) << (a.vbits + s));
      }
      for (long long p = tb[s]; p < te[s]; ++p) {
        const int32_t e = __ldg(a.nbr + p);
        if (e <= r) continue;
        const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
        bool keep = true;
        for (int j = 0; j < s && keep; ++j)
          keep = !adj_probe(a.nbr, e, eb, ee, tr[j], tb[j], te[j]);
        if (keep) dst[n++] = (uint32_t)e | (1u << (a.vbits + s));
      }
      ++s;
      size[s] = cur[s] = n;
    }
  }
  if (bad) raise_error(a.L.lb, WM_EINVARIANT);
  leaves = warp_sum_u64(leaves);
  emitted = warp_sum_u64(emitted);
  nodes = warp_sum_u64(nodes);
  done = warp_sum_u64(done);
  if (lane_id() == 0) {
    atomicAdd(&a.counters[0], leaves);
    atomicAdd(&a.counters[2], done);
    atomicAdd(&a.counters[3], nodes);
    if (LIST) atomicAdd(&a.counters[6], emitted);
  }
  if (a.smem_hist) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < a.pattern_count; i += blockDim.x)
      if (sh[i]) atomicAdd(a.hist + i, sh[i]);
  }
}

// Edge hash set construction (see EdgeHash): one warp per vertex u inserts the
// keys of its neighbours v > u with atomicCAS, slots in order within a bucket.
// every edge {u, v} with lo <= u < v (lo = 0: the whole graph)
__global__ void edge_hash_build_kernel(int64_t lo, int64_t n, const int64_t *__restrict__ off,
                                       const int32_t *__restrict__ nbr,
                                       unsigned long long *__restrict__ keys,
                                       unsigned long long bmask) {
  const int lane = lane_id();
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = lo + wid; u < n; u += nw) {
    const int64_t b = off[u], e = off[u + 1];
    for (int64_t p = b + lane; p < e; p += 32) {
      const int32_t v = nbr[p];
      if (v <= (int32_t)u) continue;
      const unsigned long long key = eh_key((int32_t)u, v);
      unsigned long long bk = eh_bucket(key, bmask);
      for (bool done = false; !done; bk = (bk + 1) & bmask) {
        for (int sl = 0; sl < 4; ++sl) {
          const unsigned long long prev = atomicCAS(keys + 4 * bk + sl, kEhEmpty, key);
          if (prev == kEhEmpty || prev == key) { done = true; break; }
        }
      }
    }
  }
}

int graph_edge_hash(Graph *g, cudaStream_t s) {
  if (g->ehash) return WM_OK;
  const unsigned long long m = (unsigned long long)(g->nnz / 2);
  unsigned long long slots = 64;
  while (slots < 2 * m) slots <<= 1;  // load factor <= 1/2
  const size_t bytes = slots * sizeof(unsigned long long);
  void *p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, g->ws->pool, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return WM_ECAPACITY;  // caller keeps the binary-search probes
  }
  WM_CUDA(cudaMemsetAsync(p, 0xFF, bytes, s));
  const int64_t blocks = ((g->n * 32 + 255) / 256) < (int64_t)g->num_sms * 16
                             ? (g->n * 32 + 255) / 256
                             : (int64_t)g->num_sms * 16;
  edge_hash_build_kernel<<<(int)(blocks > 0 ? blocks : 1), 256, 0, s>>>(
      0, g->n, g->offsets, g->neighbors, static_cast<unsigned long long *>(p), slots / 4 - 1);
  WM_CUDA(cudaGetLastError());
  g->ehash = static_cast<unsigned long long *>(p);
  g->ehash_bmask = slots / 4 - 1;
  return WM_OK;
}

template <bool LIST>
static int launch_motif_dfs(Graph *g, MotifArgs a, cudaStream_t s, int *warps_out, bool launch,
                            cudaEvent_t k0) {
  const size_t smem = a.smem_hist ? ((size_t)a.pattern_count * 8 + 15) / 16 * 16 : 0;
  const unsigned long long per = a.warp_stride * sizeof(uint32_t);
  size_t free_b = 0, total_b = 0;
  WM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const unsigned long long budget = (unsigned long long)(free_b * 0.6) + g->ws->arena.bytes;
  unsigned long long threads = (unsigned long long)g->num_sms * 2048ull;
  if (threads > a.ntasks) threads = a.ntasks > 0 ? a.ntasks : 1;
  while (threads > 256 && threads * per > budget) threads >>= 1;
  const int blocks = (int)((threads + 255) / 256);
  int st = g->ws->arena.ensure((size_t)blocks * 256 * per);
  if (st) return st;
  if (!launch) return WM_OK;
  a.arena = g->ws->arena.as<uint32_t>();
  WM_CUDA(cudaMemsetAsync(a.counters + 16, 0, sizeof(unsigned long long), s));
  if ((st = lb_prepare(g, a.L.lb, 1, 1u, &a.L, s))) return st;  // error flag only
  auto kern = motif_dfs_kernel<LIST>;
  if (smem > 48 * 1024)
    WM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  WM_CUDA(cudaEventRecord(k0, s));  // after all host-side setup: kernel time only
  kern<<<blocks, 256, smem, s>>>(a);
  WM_CUDA(cudaGetLastError());
  *warps_out = blocks * 8;
  return WM_OK;
}

template <bool BYTES, bool LIST>
static int launch_motif(Graph *g, const wm_cfg *cfg, MotifArgs a, cudaStream_t s, int *warps_out,
                        bool launch, cudaEvent_t k0) {
  int wpb = cfg->warps_per_block > 0 ? cfg->warps_per_block : 8;
  const size_t hist_bytes = a.smem_hist ? ((size_t)a.pattern_count * 8 + 15) / 16 * 16 : 0;
  const size_t smem = hist_bytes + sizeof(MotifWarp) * wpb;
  auto kern = (a.k >= 6 && !LIST) ? motif_enum_kernel<BYTES, LIST, WM_MOTIF_MINBLOCKS_DEEP>
                                  : motif_enum_kernel<BYTES, LIST, WM_MOTIF_MINBLOCKS>;
  WM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int bps = 0;
  WM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, wpb * 32, smem));
  if (cfg->blocks_per_sm > 0 && cfg->blocks_per_sm < bps) bps = cfg->blocks_per_sm;
  if (bps < 1) return fail(WM_ECAPACITY, "motif kernel does not fit on an SM");
  long long blocks = (long long)g->num_sms * bps;
  // arena budget: per-warp levels 1..k-2 hold sum_L L*maxdeg entries.  The
  // free-memory query (a driver round trip) only when the grow-only arena
  // does not already hold the full grid.
  const unsigned long long per_warp = a.warp_stride * sizeof(uint32_t);
  if ((unsigned long long)blocks * wpb * per_warp > g->ws->arena.bytes) {
    size_t free_b = 0, total_b = 0;
    WM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const unsigned long long budget = (unsigned long long)(free_b * 0.6) + g->ws->arena.bytes;
    while (blocks > 1 && (unsigned long long)blocks * wpb * per_warp > budget) blocks >>= 1;
  }
  if (!a.lb_on) {
    const unsigned long long need = (a.ntasks + wpb - 1) / wpb;
    if ((unsigned long long)blocks > need) blocks = (long long)(need > 0 ? need : 1);
  }
  const int warps = (int)blocks * wpb;
  int st = g->ws->arena.ensure((size_t)per_warp * warps);
  if (st) return st;
  if (!launch) {  // allocation pass, outside the timed region
    uint32_t cap = 1;
    while (cap < 8u * (uint32_t)warps) cap <<= 1;
    return g->ws->ring.ensure(sizeof(uint32_t) * kSlotWords * (size_t)cap);
  }
  a.arena = g->ws->arena.as<uint32_t>();
  if ((st = lb_prepare(g, a.L.lb, warps, (uint32_t)(BYTES ? kMotifRecWords : kMotifHdr + kMaxK),
                      &a.L, s)))
    return st;
  a.idle_min = (int)((1.0 - cfg->lb_threshold) * warps);
  if (a.idle_min < 1) a.idle_min = 1;
  WM_CUDA(cudaEventRecord(k0, s));  // after all host-side setup: kernel time only
  kern<<<(int)blocks, wpb * 32, smem, s>>>(a);
  WM_CUDA(cudaGetLastError());
  *warps_out = warps;
  return WM_OK;
}

// Host side of the listing ring, cached per device: a mapped control block
// (tail, failure flag), pinned staging for records and block counters, and a
// copy stream so the copy engine drains the HBM ring while the kernel runs.
struct HostRing {
  unsigned long long *ctl = nullptr;  // mapped [0] tail [1] failed
  uint32_t *stage = nullptr;          // pinned [cap * stride]
  uint32_t *counts = nullptr;         // pinned [cap >> block_shift]
  size_t stage_bytes = 0, count_bytes = 0;
  cudaStream_t copy = nullptr;
};
static HostRing g_hring[64];

static int host_ring_get(Graph *g, unsigned long long cap, uint32_t stride, uint32_t nblk,
                         HostRing **out) {
  HostRing &h = g_hring[g->device];
  if (!h.ctl) {
    void *p = nullptr;
    WM_CUDA(cudaHostAlloc(&p, 256, cudaHostAllocMapped | cudaHostAllocPortable));
    h.ctl = static_cast<unsigned long long *>(p);
    WM_CUDA(cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking));
  }
  const size_t want = sizeof(uint32_t) * (size_t)cap * stride;
  if (h.stage_bytes < want) {
    if (h.stage) cudaFreeHost(h.stage);
    h.stage = nullptr;
    h.stage_bytes = 0;
    void *p = nullptr;
    WM_CUDA(cudaHostAlloc(&p, want, cudaHostAllocPortable));
    h.stage = static_cast<uint32_t *>(p);
    h.stage_bytes = want;
  }
  if (h.count_bytes < sizeof(uint32_t) * nblk) {
    if (h.counts) cudaFreeHost(h.counts);
    h.counts = nullptr;
    h.count_bytes = 0;
    void *p = nullptr;
    WM_CUDA(cudaHostAlloc(&p, sizeof(uint32_t) * nblk, cudaHostAllocPortable));
    h.counts = static_cast<uint32_t *>(p);
    h.count_bytes = sizeof(uint32_t) * nblk;
  }
  *out = &h;
  return WM_OK;
}

// splitmix64 finaliser and the record checksum of include/warpmine_b200.h
static inline uint64_t smix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t record_hash(const uint32_t *r, int k) {
  uint64_t h = 0;
  for (int j = 0; j < k - 1; ++j) h = smix(h ^ (uint64_t)r[5 + j]);
  h = smix(h ^ (uint64_t)r[1]);
  const int off = (k - 1) * (k - 2) / 2 - 1;
  const unsigned __int128 bits = ((unsigned __int128)r[3] | ((unsigned __int128)r[4] << 32)) |
                                 ((unsigned __int128)r[2] << off);
  h = smix(h ^ (uint64_t)bits);
  h = smix(h ^ (uint64_t)(bits >> 64));
  return h;
}

// Consume records [0, n) of the staging buffer: checksum (all host cores)
// and the sink; returns false when the sink failed.
static bool consume(const uint32_t *recs, unsigned long long n, uint32_t stride, int k,
                    wm_listing *lst, uint64_t &sum) {
  uint64_t bsum = 0;
  const long long nn = (long long)n;
#pragma omp parallel for reduction(+ : bsum) schedule(static) if (nn >= 4096)
  for (long long r = 0; r < nn; ++r) bsum += record_hash(recs + r * stride, k);
  sum += bsum;
  return !(lst->sink && lst->sink(lst->user, recs, n, stride) != 0);
}

// Drain the HBM ring while the kernel (event `done`) runs: poll the block
// counters from the tail, copy every run of completed blocks with the copy
// engine, reset their counters, publish the new tail.  After the kernel has
// finished, the last partial block is copied up to the device head.
static int drain_listing(HostRing *h, unsigned long long cap, uint32_t stride, int k,
                         wm_listing *lst, cudaEvent_t done, const uint32_t *dring,
                         uint32_t *dcounts, uint32_t block_shift,
                         const unsigned long long *dhead, unsigned long long *dctl) {
  const unsigned long long G = 1ull << block_shift, mask = cap - 1;
  const uint32_t nblk = (uint32_t)(cap >> block_shift);
  cudaStream_t cs = h->copy;
  unsigned long long tail = 0;
  bool failed = false;
  uint64_t sum = 0, emitted = 0;
  int idle = 0;
  const char *dbg = getenv("WM_LIST_DEBUG");
  double t_poll = 0, t_copy = 0, t_consume = 0;
  long iters = 0, copies = 0;
  auto now = []() {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
  };
  double t0 = now();
  for (;;) {
    ++iters;
    if (!failed) {
      double ta = now();
      const uint32_t b0 = (uint32_t)((tail >> block_shift) & (nblk - 1));
      const uint32_t nchk = nblk - b0 < 64u ? nblk - b0 : 64u;  // no wrap inside one copy
      WM_CUDA(cudaMemcpyAsync(h->counts, dcounts + b0, sizeof(uint32_t) * nchk,
                              cudaMemcpyDeviceToHost, cs));
      WM_CUDA(cudaStreamSynchronize(cs));
      // counters accumulate G per lap and are never reset during the run (a
      // reset would be a kernel on the copy stream, queued behind the
      // persistent enumeration kernel): block b0 + i of lap L is complete
      // when its counter reaches (L + 1) * G
      const uint32_t want = (uint32_t)(((tail >> block_shift) / nblk + 1) * G);
      uint32_t full = 0;
      while (full < nchk && h->counts[full] == want) ++full;
      double tb = now();
      t_poll += tb - ta;
      if (full) {
        const unsigned long long n = (unsigned long long)full * G;
        WM_CUDA(cudaMemcpyAsync(h->stage, dring + (tail & mask) * stride,
                                sizeof(uint32_t) * stride * n, cudaMemcpyDeviceToHost, cs));
        WM_CUDA(cudaStreamSynchronize(cs));
        double tc = now();
        t_copy += tc - tb;
        ++copies;
        const bool ok_c = consume(h->stage, n, stride, k, lst, sum);
        t_consume += now() - tc;
        if (ok_c) {
          emitted += n;
          tail += n;
          h->ctl[0] = tail;  // pinned source of the H2D publish
          WM_CUDA(cudaMemcpyAsync(dctl, &h->ctl[0], sizeof(unsigned long long),
                                  cudaMemcpyHostToDevice, cs));
        } else {
          failed = true;  // the tail stops: producers block, see ctl[1], stop
          h->ctl[1] = 1ull;
          WM_CUDA(cudaMemcpyAsync(dctl + 1, &h->ctl[1], sizeof(unsigned long long),
                                  cudaMemcpyHostToDevice, cs));
          WM_CUDA(cudaStreamSynchronize(cs));
        }
        idle = 0;
        continue;
      }
    }
    const cudaError_t q = cudaEventQuery(done);
    if (q == cudaSuccess) {
      if (!failed) {
        unsigned long long head = 0;
        WM_CUDA(cudaMemcpyAsync(&head, dhead, sizeof head, cudaMemcpyDeviceToHost, cs));
        WM_CUDA(cudaStreamSynchronize(cs));
        // several blocks may have completed between the last counter poll
        // and the event query, so [tail, head) can span the ring's end (and
        // exceed one block): drain it in pieces that stop at the wrap (the
        // staging buffer holds a whole ring, cap records)
        while (head > tail && !failed) {
          const unsigned long long to_end = cap - (tail & mask);
          unsigned long long n = head - tail;
          if (n > to_end) n = to_end;
          WM_CUDA(cudaMemcpyAsync(h->stage, dring + (tail & mask) * stride,
                                  sizeof(uint32_t) * stride * n, cudaMemcpyDeviceToHost, cs));
          WM_CUDA(cudaStreamSynchronize(cs));
          if (consume(h->stage, n, stride, k, lst, sum)) emitted += n;
          else failed = true;
          tail += n;
        }
      }
      break;
    }
    if (q != cudaErrorNotReady)
      return fail(WM_ECUDA, "listing kernel failed: %s", cudaGetErrorString(q));
    if (++idle > 4) {
      struct timespec ts = {0, 10000};
      nanosleep(&ts, nullptr);
    }
  }
  if (dbg && *dbg == '1')
    fprintf(stderr, "[wm listing] %.3f ms total, %ld iters, %ld copies, poll %.3f copy %.3f consume %.3f ms\n",
            1e3 * (now() - t0), iters, copies, 1e3 * t_poll, 1e3 * t_copy, 1e3 * t_consume);
  lst->emitted = emitted;
  lst->checksum = sum;
  lst->stride_words = stride;
  return failed ? WM_ESHUTDOWN : WM_OK;
}

int run_motif(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res, cudaStream_t s,
              wm_listing *lst) {
  const int64_t n = g->n;
  const int k = app->k;
  const bool bytes = cfg->count_bytes != 0;
  // B_alg works with the balancer on (claim slots, motif_enum_kernel<true>)
  const bool lb_on = cfg->mode == WM_MODE_OPT;
  const int vbits = 32 - (k - 2);
  if (n > (1ll << vbits))
    return fail(WM_EINVAL, "motif kernel packs vertex ids in %d bits; n=%lld too large for k=%d",
                vbits, (long long)n, k);
  int st;
  if ((st = g->ws->keys_in.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->keys_out.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->vals_in.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->vals_out.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->counters.ensure(sizeof(unsigned long long) * 64))) return st;
  if ((st = g->ws->lb.ensure(sizeof(LbState) * 8))) return st;
  const bool dict_dev = app->dict_device != nullptr;
  if (!dict_dev && (st = g->ws->table.ensure(sizeof(uint32_t) * app->dict_len))) return st;
  if ((st = g->ws->hist.ensure(sizeof(unsigned long long) * app->pattern_count))) return st;
  size_t tmp_sort = 0;
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      nullptr, tmp_sort, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), g->ws->vals_out.as<int32_t>(), (int)n, 0, 32, s));
  if ((st = g->ws->cub_tmp.ensure(tmp_sort))) return st;

  cudaEvent_t e0 = g->ws->ev[0], e1 = g->ws->ev[1], k0 = g->ws->ev[2], k1 = g->ws->ev[3];
  PhaseTimer pt(s);
  WM_CUDA(cudaEventRecord(e0, s));
  pt.mark("start");
  unsigned long long *ctr = g->ws->counters.as<unsigned long long>();
  WM_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * 64, s));
  if (!lst) {
    WM_CUDA(cudaMemsetAsync(g->ws->hist.ptr, 0, sizeof(unsigned long long) * app->pattern_count,
                            s));
    if (!dict_dev)
      WM_CUDA(cudaMemcpyAsync(g->ws->table.ptr, app->dict_table,
                              sizeof(uint32_t) * app->dict_len, cudaMemcpyHostToDevice, s));
  }
  const int tpb = 256;
  const int64_t rb = cfg->root_begin < 0 ? 0 : cfg->root_begin;
  const int64_t re = (cfg->root_end < 0 || cfg->root_end > n) ? n : cfg->root_end;
  const int64_t nr = re > rb ? re - rb : 0;  // only the root range is keyed and sorted
  const int rblocks = (int)((nr + tpb - 1) / tpb < (int64_t)g->num_sms * 16
                                ? (nr + tpb - 1) / tpb
                                : (int64_t)g->num_sms * 16);
  if (nr > 0) {
    motif_task_keys_kernel<<<rblocks, tpb, 0, s>>>(g->offsets, rb, re,
                                                   g->ws->keys_in.as<uint32_t>(),
                                                   g->ws->vals_in.as<int32_t>(), ctr + 8);
    size_t tb = g->ws->cub_tmp.bytes;
    WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
        g->ws->cub_tmp.ptr, tb, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
        g->ws->vals_in.as<int32_t>(), g->ws->vals_out.as<int32_t>(), (int)nr, 0,
        task_key_bits(g), s));
  }
  // a root suffix run touches only the induced subgraph on [rb, n): every
  // traversal vertex exceeds its root (canon.py:190-210), so every adjacency
  // probe is an edge of that subgraph.  Its edges get their own hash set, built
  // here (inside the timed run): rows of [rb, n) hold at most 2x its edges.
  int64_t span[2] = {0, 0};
  if (rb > 0) {
    WM_CUDA(cudaMemcpyAsync(&span[0], g->offsets + rb, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaMemcpyAsync(&span[1], g->offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  }
  pt.mark("task sort");
  unsigned long long ntask = 0;
  WM_CUDA(cudaMemcpyAsync(&ntask, ctr + 8, sizeof ntask, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  pt.mark("sync");
  res->launches = 2;
  MotifArgs a;
  a.off = g->offsets;
  a.nbr = g->neighbors;
  a.tasks = g->ws->vals_out.as<int32_t>();
  if (cfg->mode == WM_MODE_DFS) {  // the ablation kernel shards whole roots
    a.task_offset = (unsigned long long)cfg->shard_rank;
    a.task_stride = (unsigned long long)cfg->shard_count;
    a.l1_offset = 0;
    a.l1_stride = 1;
    a.shard_level = 1;
  } else {
    a.task_offset = 0;
    a.task_stride = 1;
    a.l1_offset = (uint32_t)cfg->shard_rank;
    a.l1_stride = (uint32_t)cfg->shard_count;
    // WM_MOTIF_SHARD_LEVEL=1|2 overrides (A/B); default level 2 from k = 6
    const char *sl = getenv("WM_MOTIF_SHARD_LEVEL");
    a.shard_level = (sl && (*sl == '1' || *sl == '2')) ? (*sl - '0') : (k >= 6 ? 2 : 1);
  }
  a.ntasks = ntask > a.task_offset ? (ntask - a.task_offset + a.task_stride - 1) / a.task_stride : 0;
  a.k = k;
  a.vbits = vbits;
  a.vmask = (1u << vbits) - 1u;
  a.table = nullptr;
  a.table16 = nullptr;
  if (!dict_dev) a.table = g->ws->table.as<uint32_t>();
  else if (app->dict_device_bits == 16) a.table16 = static_cast<const uint16_t *>(app->dict_device);
  else a.table = static_cast<const uint32_t *>(app->dict_device);
  a.pattern_count = app->pattern_count;
  a.maxdeg = g->max_degree > 0 ? g->max_degree : 1;
  a.warp_stride = (unsigned long long)a.maxdeg * (unsigned long long)((k - 2) * (k - 1) / 2);
  a.hist = g->ws->hist.as<unsigned long long>();
  a.counters = ctr;
  a.lb_on = lb_on;
  a.lb_poll = cfg->lb_poll > 0 ? cfg->lb_poll : 1;
  a.idle_min = 1;
  a.smem_hist = app->pattern_count <= 2048;
  a.claims = nullptr;
  a.claim_ctr = ctr + 16;
  a.claim_cap = 0;
  if (bytes) {
    // claim slots for nodes shared through donations (untimed allocation)
    const uint32_t cap = 1u << 24;
    if ((st = g->ws->claims.ensure(sizeof(uint32_t) * cap))) return st;
    WM_CUDA(cudaMemsetAsync(g->ws->claims.ptr, 0, sizeof(uint32_t) * cap, s));
    a.claims = g->ws->claims.as<uint32_t>();
    a.claim_cap = cap;
  }
  a.H.b = nullptr;
  a.H.bmask = 0;
  // WM_NO_EDGE_HASH=1 forces the CSR binary-search probes (fallback-path tests)
  const char *no_hash = getenv("WM_NO_EDGE_HASH");
  const char *no_local = getenv("WM_NO_LOCAL_HASH");  // A/B: global table for suffix runs
  if (cfg->mode != WM_MODE_DFS && !(no_hash && *no_hash == '1')) {
    const unsigned long long local_m = (unsigned long long)(span[1] - span[0]) / 2;
    if (rb > 0 && !(no_local && *no_local == '1') && 4 * local_m < (unsigned long long)g->nnz) {
      unsigned long long slots = 64;
      while (slots < 2 * local_m) slots <<= 1;  // load factor <= 1/2
      if ((st = g->ws->ehash_local.ensure(slots * sizeof(unsigned long long)))) return st;
      WM_CUDA(cudaMemsetAsync(g->ws->ehash_local.ptr, 0xFF, slots * sizeof(unsigned long long), s));
      const int64_t lw = (n - rb) * 32;
      const int64_t lblocks = (lw + 255) / 256 < (int64_t)g->num_sms * 16 ? (lw + 255) / 256
                                                                          : (int64_t)g->num_sms * 16;
      edge_hash_build_kernel<<<(int)(lblocks > 0 ? lblocks : 1), 256, 0, s>>>(
          rb, n, g->offsets, g->neighbors, g->ws->ehash_local.as<unsigned long long>(),
          slots / 4 - 1);
      WM_CUDA(cudaGetLastError());
      a.H.b = reinterpret_cast<const ulonglong2 *>(g->ws->ehash_local.ptr);
      a.H.bmask = slots / 4 - 1;
      res->launches += 1;
    } else if (graph_edge_hash(g, s) == WM_OK) {
      // the whole graph's table: built once per graph (first motif run)
      a.H.b = reinterpret_cast<const ulonglong2 *>(g->ehash);
      a.H.bmask = g->ehash_bmask;
    }
  }
  a.L.lb = g->ws->lb.as<LbState>();
  memset(&a.ring, 0, sizeof a.ring);
  HostRing *hr = nullptr;
  unsigned long long cap = 0;
  uint32_t block_shift = 0;
  if (lst) {
    cap = 4096;
    while (cap < lst->capacity && cap < (1ull << 26)) cap <<= 1;
    block_shift = 10;  // 1024-record completion blocks
    const uint32_t nblk = (uint32_t)(cap >> block_shift);
    const uint32_t stride = (uint32_t)k + 4u;
    if ((st = host_ring_get(g, cap, stride, nblk, &hr))) return st;
    memset(hr->ctl, 0, 256);
    // device block: [head u64][tail u64][failed u64][counters u32 x nblk]
    if ((st = g->ws->listing.ensure(3 * sizeof(unsigned long long) +
                                    sizeof(uint32_t) * (nblk + 2)))) return st;
    if ((st = g->ws->listing_ring.ensure(sizeof(uint32_t) * cap * stride))) return st;
    WM_CUDA(cudaMemsetAsync(g->ws->listing.ptr, 0,
                            3 * sizeof(unsigned long long) + sizeof(uint32_t) * (nblk + 2), s));
    unsigned long long *dctl = g->ws->listing.as<unsigned long long>() + 1;
    a.ring.slots = g->ws->listing_ring.as<uint32_t>();
    a.ring.head = g->ws->listing.as<unsigned long long>();
    a.ring.blockdone = reinterpret_cast<uint32_t *>(g->ws->listing.as<char>() + 24);
    a.ring.block_shift = block_shift;
    a.ring.ctl = dctl;
    a.ring.cap_mask = cap - 1;
    a.ring.stride = stride;
    a.ring.filter = lst->filter;
    const int sp = (k - 1) * (k - 2) / 2 - 1;  // stored_bits(k-1), canon.py:42-48
    a.ring.full_prefix = sp > 0 ? ((sp >= 64) ? ~0ull : ((1ull << sp) - 1ull)) : 0ull;
    a.ring.full_mask = (1u << (k - 1)) - 1u;
    a.smem_hist = 0;
  }
  int warps = 0;
  const bool dfs = cfg->mode == WM_MODE_DFS;
#define WM_LAUNCH(GO)                                                            \
  (dfs ? (lst ? launch_motif_dfs<true>(g, a, s, &warps, GO, k0)                  \
              : launch_motif_dfs<false>(g, a, s, &warps, GO, k0)) :              \
  bytes ? launch_motif<true, false>(g, cfg, a, s, &warps, GO, k0)                \
         : (lst ? launch_motif<false, true>(g, cfg, a, s, &warps, GO, k0)        \
                : launch_motif<false, false>(g, cfg, a, s, &warps, GO, k0)))
  pt.mark("hash/claims");
  const auto hp0 = std::chrono::steady_clock::now();
  if (a.ntasks) {
    if ((st = WM_LAUNCH(false))) return st;
  }
  if (pt.on)
    fprintf(stderr, "[wm phases] plan (host)     %8.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hp0).count());
  pt.mark("plan");
  WM_CUDA(cudaEventRecord(k0, s));
  if (a.ntasks) {
    if ((st = WM_LAUNCH(true))) return st;
    res->launches += 2;
  }
#undef WM_LAUNCH
  WM_CUDA(cudaEventRecord(k1, s));
  pt.mark("lb init+kernel");
  int drain_st = WM_OK;
  if (lst) {
    // consume while the kernel produces (the host copies below would block)
    drain_st = drain_listing(hr, cap, a.ring.stride, k, lst, k1, a.ring.slots,
                             a.ring.blockdone, block_shift, a.ring.head, a.ring.ctl);
    if (drain_st == WM_ECUDA) return drain_st;
  }
  if (!lst && (st = red_pack(cfg, s, ctr, false, bytes, true, a.L.lb, a.ntasks ? 1 : 0,
                             g->ws->hist.as<unsigned long long>(), app->pattern_count)))
    return st;
  unsigned long long hc[8];
  WM_CUDA(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, s));
#if WM_MOTIF_PROF
  unsigned long long hp[12];
  WM_CUDA(cudaMemcpyAsync(hp, ctr + 20, sizeof hp, cudaMemcpyDeviceToHost, s));
#endif
  if (!lst)
    WM_CUDA(cudaMemcpyAsync(res->pattern_counts, g->ws->hist.ptr,
                            sizeof(unsigned long long) * app->pattern_count,
                            cudaMemcpyDeviceToHost, s));
  LbState hl;
  WM_CUDA(cudaMemcpyAsync(&hl, a.L.lb, sizeof hl, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaEventRecord(e1, s));
  pt.mark("readback");
  WM_CUDA(cudaStreamSynchronize(s));
  float kms = 0, dms = 0;
  WM_CUDA(cudaEventElapsedTime(&kms, k0, k1));
  WM_CUDA(cudaEventElapsedTime(&dms, e0, e1));
  res->h2d_bytes = (lst || dict_dev) ? 0 : sizeof(uint32_t) * app->dict_len;
  res->d2h_bytes = sizeof ntask + sizeof hc + sizeof hl +
                   (lst ? (uint64_t)lst->emitted * a.ring.stride * 4
                        : sizeof(unsigned long long) * app->pattern_count);
#if WM_MOTIF_PROF
  fprintf(stderr,
          "[motif prof] Gcycles idle %.3f rebuild %.3f build %.3f leaf %.3f | leaf steps %llu "
          "max leaf step %.3f Mcycles | records %llu | A scanned %llu kept %llu B scanned %llu "
          "kept %llu\n",
          hp[0] * 1e-9, hp[1] * 1e-9, hp[2] * 1e-9, hp[3] * 1e-9, hp[4], hp[5] * 1e-6, hp[6],
          hp[8], hp[9], hp[10], hp[11]);
#endif
  res->leaves = hc[0];
  res->alg_bytes = bytes ? hc[1] : 0;
  res->tasks = hc[2];
  res->nodes = hc[3];
  res->polls = hc[4];
  res->kernel_ms = kms;
  res->device_ms = dms;
  res->warps = warps;
  res->peak_ext = hc[5];
  if (a.ntasks) {
    finish_lb_stats(hl, res);
    res->peak_ext = hc[5];
    if (drain_st == WM_ESHUTDOWN || hl.error == WM_ESHUTDOWN)
      return fail(WM_ESHUTDOWN, "store consumer terminated");
    if (hl.error) {
      return fail(hl.error, hl.error == WM_EINVARIANT
                                ? "completed subgraph mapped to an unreachable bitmap"
                                : "extension array exceeded its capacity");
    }
  }
  if (drain_st) return fail(drain_st, "store consumer terminated");
  return WM_OK;
}

}  // namespace wm
