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
#include <cub/cub.cuh>

#include "wm_common.cuh"

namespace wm {

__global__ void degree_kernel(int64_t n, const int64_t *__restrict__ off,
                              int32_t *__restrict__ deg) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    deg[v] = (int32_t)(off[v + 1] - off[v]);
}

// sort keys for root tasks: degree+1 inside the root range (deterministic)
__global__ void motif_task_keys_kernel(int64_t n, const int32_t *__restrict__ deg, int64_t rb,
                                       int64_t re, uint32_t *__restrict__ keys,
                                       int32_t *__restrict__ vals,
                                       unsigned long long *__restrict__ ntask) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = v >= rb && v < re && deg[v] > 0;
    keys[v] = ok ? (uint32_t)deg[v] + 1u : 0u;
    vals[v] = (int32_t)v;
    if (ok) atomicAdd(ntask, 1ull);
  }
}

struct MotifArgs {
  const int64_t *off;
  const int32_t *nbr;
  const int32_t *tasks;
  unsigned long long ntasks, task_offset, task_stride;
  int k;
  int vbits;
  uint32_t vmask;
  const uint32_t *table;
  uint32_t pattern_count;
  uint32_t *arena;
  unsigned long long warp_stride;  // arena words per warp
  long long maxdeg;
  unsigned long long *hist;        // global [pattern_count]
  unsigned long long *counters;    // [0] leaves [1] B_alg [2] tasks [3] nodes [4] polls [5] peak
  int lb_on, lb_poll, idle_min;
  int smem_hist;
  LbShared L;
};

struct MotifWarp {
  int32_t tr[kMaxK];
  long long tb[kMaxK], te[kMaxK];   // CSR row bounds of tr[j]
  uint32_t bm[kMaxK];               // bm[L-1] = bitmap of tr[0..L)
  uint32_t size[kMaxK], cur[kMaxK], lo[kMaxK];
  unsigned long long below[kMaxK];  // leaves under the node of length L
};

__device__ __forceinline__ int group_off(int i) { return i * (i - 1) / 2 - 1; }

// adjacency of e (row [eb,ee)) and x (row [xb,xe)): search the shorter row
__device__ __forceinline__ bool adj_probe(const int32_t *__restrict__ nbr, int32_t e, long long eb,
                                          long long ee, int32_t x, long long xb, long long xe) {
  return (ee - eb <= xe - xb) ? row_contains(nbr, eb, ee, x) : row_contains(nbr, xb, xe, e);
}

__device__ __forceinline__ uint32_t *level_ptr(const MotifArgs &a, uint32_t *base, int L) {
  // level L (1..k-2) starts at maxdeg * (L-1)L/2
  return base + (unsigned long long)a.maxdeg * (unsigned long long)((L - 1) * L / 2);
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
  for (long long p0 = w.tb[0]; p0 < w.te[0]; p0 += 32) {
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
        const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
        const bool hit = adj_probe(a.nbr, e, eb, ee, x, xb, xe);
        val = ent | ((uint32_t)hit << (a.vbits + L));
        keep = true;
      }
    }
    emit(dst, cnt, keep, val);
  }
  // B part: neighbours of w new to the traversal's neighbourhood
  for (long long p0 = xb; p0 < xe; p0 += 32) {
    const long long p = p0 + lane;
    bool keep = false;
    uint32_t val = 0;
    if (p < xe) {
      const int32_t e = __ldg(a.nbr + p);
      if (e > t0) {
        const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
        keep = true;
        for (int j = 0; j < L && keep; ++j)
          keep = !adj_probe(a.nbr, e, eb, ee, w.tr[j], w.tb[j], w.te[j]);
        val = (uint32_t)e | (1u << (a.vbits + L));
      }
    }
    emit(dst, cnt, keep, val);
  }
  return cnt;
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
  const uint32_t bits = w.bm[L];  // bitmap of tr[0..k-1)
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
        const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
        const uint32_t mask =
            (ent >> a.vbits) | ((uint32_t)adj_probe(a.nbr, e, eb, ee, x, xb, xe) << L);
        pid = __ldg(a.table + (bits | (mask << off)));
        valid = true;
        bad |= pid >= a.pattern_count;
      }
    }
    total += __popc(__ballot_sync(0xffffffffu, valid));
    hist_add(a, sh, valid && pid < a.pattern_count, pid);
  }
  unsigned long long nb = 0;
  for (long long p0 = xb; p0 < xe; p0 += 32) {
    const long long p = p0 + lane;
    bool keep = false;
    if (p < xe) {
      const int32_t e = __ldg(a.nbr + p);
      if (e > t0) {
        const long long eb = __ldg(a.off + e), ee = __ldg(a.off + e + 1);
        keep = true;
        for (int j = 0; j < L && keep; ++j)
          keep = !adj_probe(a.nbr, e, eb, ee, w.tr[j], w.tb[j], w.te[j]);
      }
    }
    nb += __popc(__ballot_sync(0xffffffffu, keep));
  }
  if (nb) {
    const uint32_t pid = __ldg(a.table + (bits | ((1u << L) << off)));
    if (pid >= a.pattern_count) bad = true;
    else if (lane == 0) {
      if (a.smem_hist) atomicAdd(sh + pid, nb);
      else atomicAdd(a.hist + pid, nb);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_error(a.L.lb, WM_EINVARIANT);
  return total + nb;
}

__device__ __forceinline__ void set_tr(const MotifArgs &a, MotifWarp &w, int j, int32_t v) {
  if (lane_id() == 0) {
    w.tr[j] = v;
    w.tb[j] = __ldg(a.off + v);
    w.te[j] = __ldg(a.off + v + 1);
  }
  __syncwarp();
}

constexpr int kMotifHdr = 5;  // [root, level, lo, hi, bitmap] then tr[1..level)

template <bool BYTES>
__global__ void __launch_bounds__(256) motif_enum_kernel(MotifArgs a) {
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
  unsigned long long leaves = 0, bytes = 0, tasks_done = 0, nodes = 0, polls = 0, peak = 0;
  int poll = 0;
  for (;;) {
    unsigned long long ti = 0;
    Rec3 rec = {{0u, 0u, 0u}};
    const int kind = acquire_work(a.L, a.lb_on, a.ntasks, roots_left, ti, rec, clk);
    if (kind == 0) break;
    int s0;
    if (kind == 1) {
      set_tr(a, w, 0, __ldg(a.tasks + a.task_offset + ti * a.task_stride));
      if (lane == 0) {
        w.bm[0] = 0;
        w.below[1] = 0;
      }
      __syncwarp();
      const uint32_t n1 = build_first(a, w, base);
      if (lane == 0) {
        w.size[1] = n1;
        w.cur[1] = n1;
        w.lo[1] = 0;
      }
      s0 = 1;
      ++tasks_done;
    } else {
      // donated prefix: rebuild E_1..E_s0 deterministically, then own [lo, hi)
      s0 = (int)rec_word(rec, 1);
      const uint32_t lo = rec_word(rec, 2), hi = rec_word(rec, 3), bm = rec_word(rec, 4);
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
      if (lane == 0) {
        w.bm[s0 - 1] = bm;
        w.cur[s0] = hi;
        w.lo[s0] = lo;
        w.below[s0] = 0;
      }
    }
    __syncwarp();
    int s = s0;
    for (;;) {
      const uint32_t cur = w.cur[s];
      if (cur == w.lo[s]) {
        // level exhausted: the node of length s is complete
        if (BYTES && lane == 0) {
          const unsigned long long b = w.below[s];
          if (b) {
            bytes += 4ull * (unsigned long long)(w.te[s - 1] - w.tb[s - 1]);
            if (s > s0) w.below[s - 1] += b;
          }
        }
        __syncwarp();
        if (s == s0) break;
        --s;
        continue;
      }
      // move_step: pop the highest pending entry (engine.py:652-669)
      const uint32_t ent = __ldcg(level_ptr(a, base, s) + (cur - 1));
      const int32_t v = (int32_t)(ent & a.vmask);
      const uint32_t m = ent >> a.vbits;
      set_tr(a, w, s, v);
      if (lane == 0) {
        w.cur[s] = cur - 1;
        // induce (engine.py:678-705): bitmap of tr[0..s] (s+1 vertices)
        w.bm[s] = (s == 1) ? 0u : (w.bm[s - 1] | (m << group_off(s)));
      }
      __syncwarp();
      ++nodes;
      if (s + 1 == k - 1) {
        const unsigned long long got = aggregate_leaves(a, w, base, sh);
        leaves += got;
        if (BYTES && lane == 0 && got) {
          bytes += 4ull * (unsigned long long)(w.te[s] - w.tb[s]);
          w.below[s] += got;
        }
        __syncwarp();
      } else {
        const uint32_t n = build_next(a, w, base, s);
        if ((long long)n > (long long)(s + 1) * a.maxdeg && lane == 0)
          raise_error(a.L.lb, WM_ECAPACITY);
        if (lane == 0) {
          w.size[s + 1] = n;
          w.cur[s + 1] = n;
          w.lo[s + 1] = 0;
          w.below[s + 1] = 0;
        }
        __syncwarp();
        unsigned long long live = 0;
        for (int j = 1; j <= s + 1; ++j) live += w.size[j];
        if (live > peak) peak = live;
        ++s;
      }
      // on-device load balancing: donate half of the shallowest pending range
      if (!BYTES && a.lb_on && ++poll >= a.lb_poll) {
        poll = 0;
        ++polls;
        if (donation_wanted(a.L, a.idle_min)) {
          int sd = -1;
          for (int j = s0; j <= s; ++j)
            if (w.cur[j] - w.lo[j] >= 2u) { sd = j; break; }
          if (sd >= 0) {
            const uint32_t pend = w.cur[sd] - w.lo[sd];
            const bool worth = sd < k - 2 || (unsigned long long)pend * w.size[sd] >= 4096ull;
            if (worth) {
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
                else if (idx == 4) val = w.bm[sd - 1];
                else if (idx >= kMotifHdr && idx < kMotifHdr + sd - 1) val = (uint32_t)w.tr[idx - kMotifHdr + 1];
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
          }
        }
      }
    }
  }
  leaves = __shfl_sync(0xffffffffu, leaves, 0);
  if (lane == 0) {
    atomicAdd(&a.counters[0], leaves);
    if (BYTES) atomicAdd(&a.counters[1], bytes);
    atomicAdd(&a.counters[2], tasks_done);
    atomicAdd(&a.counters[3], nodes);
    atomicAdd(&a.counters[4], polls);
    atomicMax(&a.counters[5], peak);
  }
  warp_clock_end(a.L.lb, clk);
  if (a.smem_hist) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < a.pattern_count; i += blockDim.x)
      if (sh[i]) atomicAdd(a.hist + i, sh[i]);
  }
}

template <bool BYTES>
static int launch_motif(Graph *g, const wm_cfg *cfg, MotifArgs a, cudaStream_t s, int *warps_out,
                        bool launch) {
  int wpb = cfg->warps_per_block > 0 ? cfg->warps_per_block : 8;
  const size_t hist_bytes = a.smem_hist ? ((size_t)a.pattern_count * 8 + 15) / 16 * 16 : 0;
  const size_t smem = hist_bytes + sizeof(MotifWarp) * wpb;
  auto kern = motif_enum_kernel<BYTES>;
  WM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int bps = 0;
  WM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, wpb * 32, smem));
  if (cfg->blocks_per_sm > 0 && cfg->blocks_per_sm < bps) bps = cfg->blocks_per_sm;
  if (bps < 1) return fail(WM_ECAPACITY, "motif kernel does not fit on an SM");
  long long blocks = (long long)g->num_sms * bps;
  // arena budget: per-warp levels 1..k-2 hold sum_L L*maxdeg entries
  const unsigned long long per_warp = a.warp_stride * sizeof(uint32_t);
  size_t free_b = 0, total_b = 0;
  WM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const unsigned long long budget = (unsigned long long)(free_b * 0.6) + g->ws->arena.bytes;
  while (blocks > 1 && (unsigned long long)blocks * wpb * per_warp > budget) blocks >>= 1;
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
  if ((st = lb_prepare(g, a.L.lb, warps, (uint32_t)(kMotifHdr + kMaxK), &a.L, s))) return st;
  a.idle_min = (int)((1.0 - cfg->lb_threshold) * warps);
  if (a.idle_min < 1) a.idle_min = 1;
  kern<<<(int)blocks, wpb * 32, smem, s>>>(a);
  WM_CUDA(cudaGetLastError());
  *warps_out = warps;
  return WM_OK;
}

int run_motif(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res, cudaStream_t s) {
  const int64_t n = g->n;
  const int k = app->k;
  const bool bytes = cfg->count_bytes != 0;
  const bool lb_on = cfg->mode == WM_MODE_OPT && !bytes;
  const int vbits = 32 - (k - 2);
  if (n > (1ll << vbits))
    return fail(WM_EINVAL, "motif kernel packs vertex ids in %d bits; n=%lld too large for k=%d",
                vbits, (long long)n, k);
  int st;
  if ((st = g->ws->outdeg.ensure(sizeof(int32_t) * (n + 1)))) return st;
  if ((st = g->ws->keys_in.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->keys_out.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->vals_in.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->vals_out.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->counters.ensure(sizeof(unsigned long long) * 64))) return st;
  if ((st = g->ws->lb.ensure(sizeof(LbState) * 8))) return st;
  if ((st = g->ws->table.ensure(sizeof(uint32_t) * app->dict_len))) return st;
  if ((st = g->ws->hist.ensure(sizeof(unsigned long long) * app->pattern_count))) return st;
  size_t tmp_sort = 0;
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      nullptr, tmp_sort, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), g->ws->vals_out.as<int32_t>(), (int)n, 0, 32, s));
  if ((st = g->ws->cub_tmp.ensure(tmp_sort))) return st;

  cudaEvent_t e0 = g->ws->ev[0], e1 = g->ws->ev[1], k0 = g->ws->ev[2], k1 = g->ws->ev[3];
  WM_CUDA(cudaEventRecord(e0, s));
  unsigned long long *ctr = g->ws->counters.as<unsigned long long>();
  WM_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * 64, s));
  WM_CUDA(cudaMemsetAsync(g->ws->hist.ptr, 0, sizeof(unsigned long long) * app->pattern_count, s));
  WM_CUDA(cudaMemcpyAsync(g->ws->table.ptr, app->dict_table, sizeof(uint32_t) * app->dict_len,
                          cudaMemcpyHostToDevice, s));
  const int tpb = 256;
  const int eblocks = (int)((n + tpb - 1) / tpb < (int64_t)g->num_sms * 16
                                ? (n + tpb - 1) / tpb
                                : (int64_t)g->num_sms * 16);
  degree_kernel<<<eblocks, tpb, 0, s>>>(n, g->offsets, g->ws->outdeg.as<int32_t>());
  const int64_t rb = cfg->root_begin < 0 ? 0 : cfg->root_begin;
  const int64_t re = (cfg->root_end < 0 || cfg->root_end > n) ? n : cfg->root_end;
  motif_task_keys_kernel<<<eblocks, tpb, 0, s>>>(n, g->ws->outdeg.as<int32_t>(), rb, re,
                                                 g->ws->keys_in.as<uint32_t>(),
                                                 g->ws->vals_in.as<int32_t>(), ctr + 8);
  size_t tb = g->ws->cub_tmp.bytes;
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      g->ws->cub_tmp.ptr, tb, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), g->ws->vals_out.as<int32_t>(), (int)n, 0, 32, s));
  unsigned long long ntask = 0;
  WM_CUDA(cudaMemcpyAsync(&ntask, ctr + 8, sizeof ntask, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  res->launches = 2;
  MotifArgs a;
  a.off = g->offsets;
  a.nbr = g->neighbors;
  a.tasks = g->ws->vals_out.as<int32_t>();
  a.task_offset = (unsigned long long)cfg->shard_rank;
  a.task_stride = (unsigned long long)cfg->shard_count;
  a.ntasks = ntask > a.task_offset ? (ntask - a.task_offset + a.task_stride - 1) / a.task_stride : 0;
  a.k = k;
  a.vbits = vbits;
  a.vmask = (1u << vbits) - 1u;
  a.table = g->ws->table.as<uint32_t>();
  a.pattern_count = app->pattern_count;
  a.maxdeg = g->max_degree > 0 ? g->max_degree : 1;
  a.warp_stride = (unsigned long long)a.maxdeg * (unsigned long long)((k - 2) * (k - 1) / 2);
  a.hist = g->ws->hist.as<unsigned long long>();
  a.counters = ctr;
  a.lb_on = lb_on;
  a.lb_poll = cfg->lb_poll > 0 ? cfg->lb_poll : 1;
  a.idle_min = 1;
  a.smem_hist = app->pattern_count <= 2048;
  a.L.lb = g->ws->lb.as<LbState>();
  int warps = 0;
  if (a.ntasks) {
    st = bytes ? launch_motif<true>(g, cfg, a, s, &warps, false)
               : launch_motif<false>(g, cfg, a, s, &warps, false);
    if (st) return st;
  }
  WM_CUDA(cudaEventRecord(k0, s));
  if (a.ntasks) {
    st = bytes ? launch_motif<true>(g, cfg, a, s, &warps, true)
               : launch_motif<false>(g, cfg, a, s, &warps, true);
    if (st) return st;
    res->launches += 2;
  }
  WM_CUDA(cudaEventRecord(k1, s));
  unsigned long long hc[8];
  WM_CUDA(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaMemcpyAsync(res->pattern_counts, g->ws->hist.ptr,
                          sizeof(unsigned long long) * app->pattern_count,
                          cudaMemcpyDeviceToHost, s));
  LbState hl;
  WM_CUDA(cudaMemcpyAsync(&hl, a.L.lb, sizeof hl, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaEventRecord(e1, s));
  WM_CUDA(cudaStreamSynchronize(s));
  float kms = 0, dms = 0;
  WM_CUDA(cudaEventElapsedTime(&kms, k0, k1));
  WM_CUDA(cudaEventElapsedTime(&dms, e0, e1));
  res->h2d_bytes = sizeof(uint32_t) * app->dict_len;
  res->d2h_bytes = sizeof ntask + sizeof hc + sizeof(unsigned long long) * app->pattern_count +
                   sizeof hl;
  res->leaves = hc[0];
  res->alg_bytes = bytes ? hc[1] : 0;
  res->tasks = hc[2];
  res->nodes = hc[3];
  res->polls = hc[4];
  res->kernel_ms = kms;
  res->device_ms = dms;
  res->warps = warps;
  if (a.ntasks) {
    finish_lb_stats(hl, res);
    if (hl.error) {
      return fail(hl.error, hl.error == WM_EINVARIANT
                                ? "completed subgraph mapped to an unreachable bitmap"
                                : "extension array exceeded its capacity");
    }
  }
  res->peak_ext = hc[5];
  return WM_OK;
}

}  // namespace wm
