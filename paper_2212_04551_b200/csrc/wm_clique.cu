// wm_clique.cu — warp-centric k-clique counting (clique_app, reference
// pkg/src/warpmine/apps.py:43-47) for sm_100a.
//
// Reference pipeline per traversal (engine.py:214-241):
//   extend(0,1)      N(tr[0]) minus tr                    engine.py:245-327
//   filter_lower     drop e <= tr[len-1]                  engine.py:331-353
//   compact          stable removal of invalid entries    engine.py:544-564
//   filter_clique    keep e adjacent to every tr[j]       engine.py:355-422
//   aggregate        count_valid at len == k-1            engine.py:568-592,
//                                                         aggregate.py:155-171
//   move_step        pop one pending extension, descend   engine.py:643-676
//
// B200 restatement.  The clique tree's level-L extension set is
//   C_L = { e in N(tr[0]) : e above tr[L-1], e adjacent to tr[0..L) }
// which, since the filters are conjunctive, equals C_{L-1} ∩ N+(tr[L-1])
// with N+ the out-neighbours of an orientation ("lower" = above in the
// order).  A preprocessing kernel builds, once per root, the induced DAG on
// the d = |N+(root)| candidates as a d x d bitmap (sorted-set intersections
// of N+(u_i) against N+(root) by binary search in shared memory) into an HBM
// arena.  Every later extension is one W-word AND (extend + lower + clique
// fused), compaction is implicit in the bitmap, and the last three levels are
// aggregated in bulk: for a node at traversal length k-3 with candidates C,
//   leaves = sum_{j in C} sum_{l in C&A[j]} popc(C & A[j] & A[l])
// with one lane per j (k = 3 uses the two-level form sum_j popc(C & A[j])).
// Counts are orientation-invariant; WM_ORDER_ID
// reproduces the reference's id order exactly, WM_ORDER_DEGREE bounds d by
// the degeneracy.
//
// Work distribution: persistent warps pull root tasks (cost-sorted, largest
// first) from a global cursor (the engine's root deque, engine.py:187).  In
// opt mode busy warps poll the idle-warp ring and donate half of their
// shallowest pending extensions (balance.py:102-155 semantics: the thief owns
// exactly the stolen branches; inherited levels are never regenerated).
#include <algorithm>
#include <cub/cub.cuh>
#include <vector>

#include "wm_common.cuh"

namespace wm {

// --------------------------------------------------------------------------
// orientation: u is "above" v

__device__ __forceinline__ bool above(int order, int64_t du, int32_t u, int64_t dv, int32_t v) {
  if (order == WM_ORDER_ID) return u > v;
  return du > dv || (du == dv && u > v);
}

__global__ void orient_count_kernel(int64_t n, const int64_t *__restrict__ off,
                                    const int32_t *__restrict__ nbr, int order,
                                    int32_t *__restrict__ outdeg) {
  const int lane = lane_id();
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = off[v], e = off[v + 1], dv = e - b;
    int cnt = 0;
    for (int64_t p = b + lane; p < e; p += 32) {
      const int32_t u = __ldg(nbr + p);
      const int64_t du = order == WM_ORDER_ID ? 0 : __ldg(off + u + 1) - __ldg(off + u);
      cnt += above(order, du, u, dv, (int32_t)v);
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) outdeg[v] = cnt;
  }
}

// ballot+popc stream compaction of the "above" neighbours, order preserved
__global__ void orient_fill_kernel(int64_t n, const int64_t *__restrict__ off,
                                   const int32_t *__restrict__ nbr, int order,
                                   const int64_t *__restrict__ doff, int32_t *__restrict__ dnbr) {
  const int lane = lane_id();
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = off[v], e = off[v + 1], dv = e - b;
    int64_t w = doff[v];
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const int64_t p = p0 + lane;
      bool keep = false;
      int32_t u = 0;
      if (p < e) {
        u = __ldg(nbr + p);
        const int64_t du = order == WM_ORDER_ID ? 0 : __ldg(off + u + 1) - __ldg(off + u);
        keep = above(order, du, u, dv, (int32_t)v);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) dnbr[w + __popc(bal & ((1u << lane) - 1))] = u;
      w += __popc(bal);
    }
  }
}


// Edge-parallel orientation (the reference's filter_lower, engine.py:331-353,
// applied once per edge): flag every directed edge (v, u) with u above v,
// exclusive-scan the flags, scatter.  Rows stay ascending (the CSR is
// row-major) and every hub row is spread over many threads instead of being
// walked by one warp — the warp-per-vertex form spent 0.5 ms on cfg3, bound by
// the 20K-entry hub rows' dependent loads.
__global__ void orient_src_kernel(int64_t n, const int64_t *__restrict__ off,
                                  int32_t *__restrict__ src) {
  const int lane = lane_id();
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = off[v], e = off[v + 1];
    for (int64_t p = b + lane; p < e; p += 32) src[p] = (int32_t)v;
  }
}

__global__ void orient_flag_kernel(int64_t nnz, const int64_t *__restrict__ off,
                                   const int32_t *__restrict__ nbr,
                                   const int32_t *__restrict__ src, int order,
                                   int32_t *__restrict__ flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (p == nnz) { flag[p] = 0; continue; }
    const int32_t u = __ldg(nbr + p), v = __ldg(src + p);
    int64_t du = 0, dv = 0;
    if (order != WM_ORDER_ID) {
      du = __ldg(off + u + 1) - __ldg(off + u);
      dv = __ldg(off + v + 1) - __ldg(off + v);
    }
    flag[p] = above(order, du, u, dv, v) ? 1 : 0;
  }
}

__global__ void orient_scatter_kernel(int64_t nnz, const int32_t *__restrict__ nbr,
                                      const int32_t *__restrict__ flag,
                                      const int32_t *__restrict__ pos,
                                      int32_t *__restrict__ dnbr) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    if (flag[p]) dnbr[pos[p]] = __ldg(nbr + p);
}

__global__ void orient_off_kernel(int64_t n, const int64_t *__restrict__ off,
                                  const int32_t *__restrict__ pos, int64_t *__restrict__ doff,
                                  int32_t *__restrict__ outdeg) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = pos[off[v]];
    doff[v] = a;
    outdeg[v] = v < n ? (int32_t)(pos[off[v + 1]] - a) : 0;
  }
}

// sort keys: eligible roots (out-degree >= k-1, inside the root range) get
// outdeg+1, others 0; values are vertex ids in ascending order so the stable
// descending sort is deterministic (identical task lists on every rank).
__global__ void task_keys_kernel(int64_t n, const int32_t *__restrict__ outdeg, int k,
                                 int64_t rb, int64_t re, uint32_t *__restrict__ keys,
                                 int32_t *__restrict__ vals) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = v >= rb && v < re && outdeg[v] >= k - 1;
    keys[v] = ok ? (uint32_t)outdeg[v] + 1u : 0u;
    vals[v] = (int32_t)v;
  }
}

// counts[c] = number of eligible tasks whose bitmap needs 2^c words per row
// (c = 0..5 -> W = 1..32, d <= 32W); counts[6] = over-capacity (d > 1024).
__global__ void bucket_count_kernel(int64_t n, const uint32_t *__restrict__ keys,
                                    unsigned long long *__restrict__ counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = keys[i];
    if (!key) continue;
    const uint32_t d = key - 1;
    int c = 0;
    while (c < 6 && d > (32u << c)) ++c;
    atomicAdd(&counts[c], 1ull);
  }
}

// words of the compact local bitmap of a root with out-degree d
__device__ __host__ __forceinline__ unsigned long long bm_words(int d) {
  return (unsigned long long)d * (unsigned long long)((d + 31) >> 5);
}

__global__ void task_words_kernel(unsigned long long ntask, const uint32_t *__restrict__ keys,
                                  unsigned long long *__restrict__ words) {
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       t < ntask; t += (unsigned long long)gridDim.x * blockDim.x)
    words[t] = bm_words((int)keys[t] - 1);
}

// --------------------------------------------------------------------------
// 1) per-root local DAG bitmaps, built once into an HBM arena
//
// Root task t (vertex v, d = |N+(v)|) owns rows [bm_off[t], bm_off[t] + d*Wv)
// with Wv = ceil(d/32): row i = N+(u_i) ∩ N+(v) as local bit positions, u_i
// the i-th out-neighbour of v in ascending id.  These rows are the reference's
// filter_clique + filter_lower predicates (engine.py:331-422) precomputed for
// every pair inside the root's extension set, so every later extension is a
// W-word AND.  Total size is sum_v d_v * ceil(d_v/32) words (2.6 MB at cfg3).

template <int W> struct BuildSmem {
  static constexpr int D = 32 * W;
  unsigned long long key[D];  // orientation key of member i (rank-ordered bitmaps)
  int32_t rk[D];              // member i's local index: its rank among the members
  int32_t list[D];
  uint32_t adj[D * W];
  int32_t pre[D + 1];
  int64_t rowbeg[D];
#ifndef WM_BUILD_BATCH
#define WM_BUILD_BATCH 8
#endif
#ifndef WM_BUILD_BSEARCH
  int32_t hkey[2 * D];        // member id -> local index, open addressing (load <= 1/2)
  int32_t hval[2 * D];
#endif
};

template <int W>
__global__ void __launch_bounds__(256) clique_build_kernel(const int64_t *__restrict__ doff,
                                                           const int32_t *__restrict__ dnbr,
                                                           const int32_t *__restrict__ tasks,
                                                           unsigned long long ntask,
                                                           const unsigned long long *__restrict__ bm_off,
                                                           uint32_t *__restrict__ bm,
                                                           unsigned long long below,
                                                           unsigned long long first,
                                                           unsigned long long stride,
                                                           const int64_t *__restrict__ goff,
                                                           int order, int rank_order) {
  extern __shared__ __align__(16) unsigned char smraw[];
  BuildSmem<W> &sm = reinterpret_cast<BuildSmem<W> *>(smraw)[threadIdx.x >> 5];
  const int lane = lane_id();
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  // only this shard's tasks need a bitmap: every t < below (split over the
  // shards at level 1), then t = first + j * stride
  const unsigned long long wid = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nmine = below + (first < ntask ? (ntask - first + stride - 1) / stride : 0);
  for (unsigned long long j = wid; j < nmine; j += nwarps) {
    const unsigned long long t = j < below ? j : first + (j - below) * stride;
    const int32_t v = __ldg(tasks + t);
    const int64_t b = __ldg(doff + v);
    const int d = (int)(__ldg(doff + v + 1) - b);
    const int wv = (d + 31) >> 5;
    for (int i = lane; i < d; i += 32) {
      const int32_t u = __ldg(dnbr + b + i);
      const int64_t rb = __ldg(doff + u), re = __ldg(doff + u + 1);
      sm.list[i] = u;
      sm.rowbeg[i] = rb;
      sm.pre[i] = (int)(re - rb);
      if (rank_order) {
        const unsigned long long gd = order == WM_ORDER_ID ? 0ull
                                          : (unsigned long long)(__ldg(goff + u + 1) - __ldg(goff + u));
        sm.key[i] = (gd << 32) | (uint32_t)u;  // the orientation order of above()
      }
    }
    for (int i = lane; i < d * wv; i += 32) sm.adj[i] = 0u;
    __syncwarp();
    // Local indices in descending orientation order make every row strictly
    // lower-triangular (row i holds only members ranked above u_i, i.e. at
    // smaller local indices), which the bulk loops exploit: the lowest member
    // of a candidate set has no neighbour in it.
    for (int i = lane; i < d; i += 32) {
      int r = i;
      if (rank_order) {
        const unsigned long long ki = sm.key[i];
        r = 0;
        for (int j = 0; j < d; ++j) r += sm.key[j] > ki;
      }
      sm.rk[i] = r;
    }
    __syncwarp();
    int carry = 0;
    for (int base = 0; base < d; base += 32) {
      const int i = base + lane;
      const int x = i < d ? sm.pre[i] : 0;
      int y = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      if (i < d) sm.pre[i] = carry + y - x;
      carry += __shfl_sync(0xffffffffu, y, 31);
    }
    __syncwarp();
    const int total = carry;
#ifndef WM_BUILD_BSEARCH
    // members into a small hash table (member id -> local index): one or two
    // shared loads per membership test instead of a log2(d) binary search;
    // each lane walks the flattened (row, element) pairs with a row cursor
    // that only moves forward instead of searching the row per element, 8
    // elements per batch so their loads are in flight together: cfg5 k=8
    // build 30.7 -> 23.5 ms (profiles/r02_ab_bhash2.log; WM_BUILD_BSEARCH=1
    // restores the binary searches)
    int tb = 5;
    while ((1 << tb) < 2 * d) ++tb;
    const int T = 1 << tb;
    for (int i = lane; i < T; i += 32) sm.hkey[i] = -1;
    __syncwarp();
    for (int i = lane; i < d; i += 32) {
      const int32_t x = sm.list[i];
      uint32_t h = ((uint32_t)x * 0x9E3779B1u) >> (32 - tb);
      while (atomicCAS(&sm.hkey[h], -1, x) != -1) h = (h + 1) & (uint32_t)(T - 1);
      sm.hval[h] = sm.rk[i];
    }
    __syncwarp();
    int r = 0;
    for (int f0 = lane; f0 < total; f0 += 32 * WM_BUILD_BATCH) {
      // the batch's rows (cursor moves forward), then all its loads in flight
      int rows[WM_BUILD_BATCH];
      int32_t xs[WM_BUILD_BATCH];
#pragma unroll
      for (int j = 0; j < WM_BUILD_BATCH; ++j) {
        const int f = f0 + 32 * j;
        rows[j] = -1;
        if (f < total) {
          while (r + 1 < d && sm.pre[r + 1] <= f) ++r;
          rows[j] = r;
          xs[j] = __ldg(dnbr + sm.rowbeg[r] + (f - sm.pre[r]));
        }
      }
#pragma unroll
      for (int j = 0; j < WM_BUILD_BATCH; ++j) {
        if (rows[j] < 0) continue;
        const int32_t x = xs[j];
        uint32_t h = ((uint32_t)x * 0x9E3779B1u) >> (32 - tb);
        int32_t kx;
        while ((kx = sm.hkey[h]) != x && kx != -1) h = (h + 1) & (uint32_t)(T - 1);
        if (kx == x) {
          const int b = sm.hval[h];
          atomicOr(&sm.adj[sm.rk[rows[j]] * wv + (b >> 5)], 1u << (b & 31));
        }
      }
    }
#else
    // flattened (row, element) pairs: every lane busy regardless of row length
    for (int f0 = 0; f0 < total; f0 += 128) {
      int32_t xs[4];
      int rows[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int f = f0 + j * 32 + lane;
        rows[j] = -1;
        if (f < total) {
          int lo = 0, hi = d;  // last row with pre <= f
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (sm.pre[mid] <= f) lo = mid; else hi = mid;
          }
          rows[j] = sm.rk[lo];
          xs[j] = __ldg(dnbr + sm.rowbeg[lo] + (f - sm.pre[lo]));
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (rows[j] >= 0) {
          const int pos = lower_bound_i(sm.list, d, xs[j]);
          if (pos < d && sm.list[pos] == xs[j]) {
            const int b = sm.rk[pos];
            atomicOr(&sm.adj[rows[j] * wv + (b >> 5)], 1u << (b & 31));
          }
        }
      }
    }
#endif
    __syncwarp();
    uint32_t *out = bm + bm_off[t];
    for (int i = lane; i < d * wv; i += 32) out[i] = sm.adj[i];
    __syncwarp();
  }
}

// --------------------------------------------------------------------------
// 2) enumeration: per-warp DFS-wide stack in shared memory
//
// One launch per width class WMAX (4, 8, 16, 32).  The class-4 launch runs
// every task with d <= 128; each task is processed by the instantiation for
// its own word count (1, 2 or 4) over a shared per-warp buffer, so small
// roots pay for narrow rows only.

template <int WMAX> struct alignas(16) CliqueSmem {  // 16B: uint4 row loads
  static constexpr int D = 32 * WMAX;
  static constexpr int S = WMAX;
  uint32_t adj[D * S];                 // local DAG rows, stride w (16B-aligned vector loads)
  uint32_t C[kMaxK * WMAX];            // candidate set per level  [s * w + x]
  uint32_t P[kMaxK * WMAX];            // unconsumed members       [s * w + x]
  unsigned long long below[kMaxK];     // leaves under the level's node (B_alg)
  int32_t last[kMaxK];                 // vertex appended at the level
  uint32_t queue[96];                  // bulk4/5 ring (64) + a scratch slot per lane
  uint32_t pq[64];                     // bulk5 (h, i) pair ring
  uint32_t crow[32];                   // bulk4 node compacted to <= 32 members
  // per-warp node/poll counters (lane 0): off the register budget, cfg3 k=9
  // 18.95 -> 18.59 ms, k=10 81.7 -> 80.0 (profiles/r02_ab_clique_smem_counters.log;
  // the poll's ticket words there too were slower)
  unsigned long long n_nodes, n_polls;
};

struct CliqueArgs {
  const int64_t *doff;
  const int32_t *dnbr;
  const int32_t *tasks;              // class's cost-sorted roots
  const unsigned long long *bm_off;  // class's bitmap offsets (per task)
  const uint32_t *bm;                // bitmap arena
  unsigned long long ntasks;         // tasks of this shard in the class
  unsigned long long task_offset;    // shard rank
  unsigned long long task_stride;    // shard count
  // multi-GPU: the class's first `heavy` (costliest) tasks are processed by
  // EVERY shard, each over its own level-1 members (member i + task = rank
  // mod N) — one hub root's subtree no longer lands on one GPU; the others are
  // dealt whole, task index = rank (mod N), from rem_first on
  unsigned long long heavy;
  unsigned long long rem_first;
  int k;
  int lb_on;
  int lb_poll;
  int idle_min;
  LbShared L;
  unsigned long long *counters;      // [0] cliques [1] B_alg [2] tasks [3] nodes [4] polls
};

template <int w> struct Width {
  static constexpr int S = w;
};

// one local-DAG row into registers with 64/128-bit shared loads
template <int w>
__device__ __forceinline__ void load_row(const uint32_t *p, uint32_t (&r)[w]) {
  if constexpr (w % 4 == 0) {
#pragma unroll
    for (int q = 0; q < w / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4 *>(p)[q];
      r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
    }
  } else if constexpr (w == 2) {
    const uint2 v = *reinterpret_cast<const uint2 *>(p);
    r[0] = v.x; r[1] = v.y;
  } else {
    r[0] = p[0];
  }
}

__device__ __forceinline__ unsigned long long outdeg_bytes(const CliqueArgs &a, int32_t u) {
  return 4ull * (unsigned long long)(__ldg(a.doff + u + 1) - __ldg(a.doff + u));
}

// Pop the highest member of m (one FLO via bfind; __ffs needs BREV + FLO and
// 31 - __clz is not folded back).  Sums of popcounts do not depend on the
// member order.
__device__ __forceinline__ int pop_hi(uint32_t &m) {
  int l;
  asm("bfind.u32 %0, %1;" : "=r"(l) : "r"(m));
  m ^= 1u << l;
  return l;
}

// Branch-free ring push: the lanes whose bit is set in `word` take the next
// ring positions in lane order; the others write their scratch slot 64 + lane.
__device__ __forceinline__ int ring_slot(uint32_t word, int tail) {
  const int lane = lane_id();
  const uint32_t lt = (1u << lane) - 1u;
  return ((word >> lane) & 1u) ? ((tail + __popc(word & lt)) & 63) : 64 + lane;
}

// Two-level bulk (traversal length k-2, k == 3 roots): sum_j popc(C & A[j]).
template <int w, bool BYTES>
__device__ __forceinline__ unsigned long long bulk2(const uint32_t *adj, const uint32_t *Cs,
                                                    const CliqueArgs &a, int64_t lb,
                                                    unsigned long long &bytes) {
  constexpr int S = Width<w>::S;
  const int lane = lane_id();
  uint32_t c[w];
#pragma unroll
  for (int x = 0; x < w; ++x) c[x] = Cs[x];
  unsigned long long part = 0;
#pragma unroll
  for (int q = 0; q < w; ++q) {
    if (c[q] == 0u) continue;
    if ((c[q] >> lane) & 1u) {
      const int j = q * 32 + lane;
      uint32_t row[w];
      load_row<w>(adj + j * S, row);
      uint32_t t = 0;
#pragma unroll
      for (int x = 0; x < w; ++x) t += __popc(c[x] & row[x]);
      part += t;
      if (BYTES && t) bytes += outdeg_bytes(a, __ldg(a.dnbr + lb + j));
    }
  }
  return part;
}

// Three-level bulk for a node at traversal length k-3 with candidates C and
// members to expand J (J == C except for donated partial levels): one lane per
// j in J; the lane walks the members l of Cj = C & A[j] and adds
// popc(Cj & A[l]).  Returns this lane's partial; with BYTES, adds B_alg of the
// productive length k-2 and k-1 nodes and reports the warp total.
template <int w, bool BYTES>
__device__ __forceinline__ unsigned long long bulk3(const uint32_t *adj, const uint32_t *Cs,
                                                    const uint32_t *Js, const CliqueArgs &a,
                                                    int64_t lb, unsigned long long &bytes) {
  constexpr int S = Width<w>::S;
  const int lane = lane_id();
  uint32_t c[w];
#pragma unroll
  for (int x = 0; x < w; ++x) c[x] = Cs[x];
  unsigned long long part = 0;
#pragma unroll
  for (int q = 0; q < w; ++q) {
    const uint32_t jw = Js[q];
    if (jw == 0u) continue;
    if ((jw >> lane) & 1u) {
      const int j = q * 32 + lane;
      uint32_t rj[w];
      load_row<w>(adj + j * S, rj);
      uint32_t cj[w];
      int cnt = 0;
#pragma unroll
      for (int x = 0; x < w; ++x) {
        cj[x] = c[x] & rj[x];
        cnt += __popc(cj[x]);
      }
      if (cnt >= 2) {
        uint32_t sub = 0;  // <= (32 w)^2
#pragma unroll
        for (int y = 0; y < w; ++y) {
          uint32_t m = cj[y];
          while (m) {
            const int l = y * 32 + pop_hi(m);
            uint32_t rl[w];
            load_row<w>(adj + l * S, rl);
            uint32_t t = 0;
#pragma unroll
            for (int x = 0; x < w; ++x) t += __popc(cj[x] & rl[x]);
            sub += t;
            if (BYTES && t) bytes += outdeg_bytes(a, __ldg(a.dnbr + lb + l));
          }
        }
        part += sub;
        if (BYTES && sub) bytes += outdeg_bytes(a, __ldg(a.dnbr + lb + j));
      }
    }
  }
  return part;
}


#ifndef WM_BULK4_MINK
#define WM_BULK4_MINK 5
#endif
#ifndef WM_BULK5_MINK
#define WM_BULK5_MINK 6
#endif
#ifndef WM_BULK5_POLL_MIN
#define WM_BULK5_POLL_MIN 4
#endif
#ifndef WM_BULK5_POLL_EVERY
#define WM_BULK5_POLL_EVERY 8  // with donate min 32K: k=8 4.63 -> 4.37 ms, k=9 18.53 -> 18.24 (r02_ab_clique_knobs.log)
#endif
#ifndef WM_COMPACT_POLL_MIN
#define WM_COMPACT_POLL_MIN 16
#endif

// Four-level bulk for a node at traversal length k-4 with candidates C and
// children to expand P: leaves = sum_{i in P} sum_{j in C_i} sum_{l in C_ij}
// popc(C_ij & A[l]) with C_i = C & A[i], C_ij = C_i & A[j].  The (i, j)
// pairs — the grandchildren, i.e. the (k-2)-cliques below the node — are
// flattened through a 64-entry ring in shared memory so that all 32 lanes
// take one pair each per round; bulk3's lane-per-j mapping leaves most
// lanes idle once candidate sets are small (deep k).  Each lane then walks
// the members l of its C_ij (the reference's last two extend/filter levels
// done as one AND + popc per l).
template <int w>
__device__ __forceinline__ unsigned long long bulk4_round(const uint32_t *adj, const uint32_t (&c)[w],
                                                          const uint32_t *queue, int head, int nq) {
  constexpr int S = Width<w>::S;
  const int lane = lane_id();
  uint32_t part = 0;  // <= 32 * 32 * w per round: no 64-bit adds in the loop
  if (lane < nq) {
    const uint32_t e = queue[(head + lane) & 63];
    const int i = (int)(e >> 16), j = (int)(e & 0xffffu);
    uint32_t ri[w], rj[w], cij[w];
    load_row<w>(adj + i * S, ri);
    load_row<w>(adj + j * S, rj);
#pragma unroll
    for (int x = 0; x < w; ++x) cij[x] = c[x] & ri[x] & rj[x];
    bool low = true;  // rows are lower-triangular: the lowest member adds nothing
#pragma unroll
    for (int y = 0; y < w; ++y) {
      uint32_t m = cij[y];
      if (low && m) {
        m &= m - 1u;
        low = false;
      }
      while (m) {
        const int l = y * 32 + pop_hi(m);
        uint32_t rl[w];
        load_row<w>(adj + l * S, rl);
#pragma unroll
        for (int x = 0; x < w; ++x) part += __popc(cij[x] & rl[x]);
      }
    }
  }
  return part;
}

// Donate the upper half of the pending members of the shallowest level that
// has any (reference balance.py:102-128 steals the shallowest pending entry;
// one record here carries half of that level so a thief gets a large
// subtree).  Record: [task, level, C[level] (w words), donated P (w words)].
// Subtrees estimated below ~32K nodes are not worth a move and stay (16K before the
// per-warp counters and bulk5 poll every 8 children, profiles/r02_ab_clique_knobs.log).
constexpr int kRecHdr = 2;
#ifndef WM_CLIQUE_DONATE_MIN
#define WM_CLIQUE_DONATE_MIN 32768.f
#endif

template <int w>
__device__ __forceinline__ void try_donate(uint32_t *C, uint32_t *P, const CliqueArgs &a, int s0,
                                           int s, unsigned long long task) {
  const int lane = lane_id();
  int sd = -1;
  uint32_t pw = 0u;
  for (int t = s0; t <= s; ++t) {
    const uint32_t w2 = lane < w ? P[t * w + lane] : 0u;
    if (__ballot_sync(0xffffffffu, w2 != 0u)) { sd = t; pw = w2; break; }
  }
  if (sd < 0) return;
  const uint32_t cw = lane < w ? C[sd * w + lane] : 0u;
  const int cnt = __popc(pw);
  int pre = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int z = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += z;
  }
  const int total = __shfl_sync(0xffffffffu, pre, 31);
  const int csize = __reduce_add_sync(0xffffffffu, __popc(cw));
  const int depth = a.k - 2 - sd;  // levels below, bulk levels included
  const float est = (float)total * __powf((float)csize, (float)(depth - 1));
  if (est < WM_CLIQUE_DONATE_MIN) return;
  pre -= cnt;  // exclusive prefix
  const int keep = total / 2;
  uint32_t give;
  if (pre >= keep) give = pw;
  else if (pre + cnt <= keep) give = 0u;
  else {
    uint32_t w2 = pw;
    for (int r = keep - pre; r > 0; --r) w2 &= w2 - 1u;
    give = w2;
  }
  Rec3 rec;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int idx = 32 * r + lane;
    const uint32_t cv = __shfl_sync(0xffffffffu, cw, (idx - kRecHdr) & 31);
    const uint32_t gv = __shfl_sync(0xffffffffu, give, (idx - kRecHdr - w) & 31);
    rec.w[r] = idx == 0 ? (uint32_t)task
             : idx == 1 ? (uint32_t)sd
             : (idx - kRecHdr < w ? cv : (idx - kRecHdr - w < w ? gv : 0u));
  }
  donate_record(a.L, rec);
  if (lane < w) P[sd * w + lane] = pw & ~give;
  const int moved = __reduce_add_sync(0xffffffffu, __popc(give));
  if (lane == 0) {
    atomicAdd(&a.L.lb->migrations, (unsigned long long)moved);
    atomicAdd(&a.L.lb->donation_polls, 1ull);
  }
  __syncwarp();
}

struct TaskCounters {
  unsigned long long acc, bytes, nodes, polls;
  int poll;
};

// A wide (w > 1) four-level bulk node whose candidate set has m <= 32
// members is first compacted to an m x m one-word bitmap (row r = members
// above member r: one ballot per row), so the pair ring and the popc loop run
// at w = 1 — a single AND + POPC per step instead of w of each.  For a
// donation the pending compact children are mapped back to their original
// bit positions in P[lv] (one OR-reduction per word) and re-read afterwards.
template <int w, int WMAX>
__device__ __forceinline__ unsigned long long bulk4_compact(CliqueSmem<WMAX> &sm, const CliqueArgs &a,
                                                            int lv, int m, int s0,
                                                            unsigned long long task,
                                                            TaskCounters &tc, uint32_t &pt,
                                                            uint32_t &ph) {
  const int lane = lane_id();
  // member r's original bit position, scattered by bit lanes (crow is
  // scratch until the compact rows are written)
  {
    int before = 0;
#pragma unroll
    for (int x = 0; x < w; ++x) {
      const uint32_t cw = sm.C[lv * w + x];
      if ((cw >> lane) & 1u)
        sm.crow[before + __popc(cw & ((1u << lane) - 1u))] = (uint32_t)(x * 32 + lane);
      before += __popc(cw);
    }
  }
  __syncwarp();
  const int pos = lane < m ? (int)sm.crow[lane] : -1;  // this lane's member
  __syncwarp();
  for (int r = 0; r < m; ++r) {
    const int pr = __shfl_sync(0xffffffffu, pos, r);
    const uint32_t *row = sm.adj + pr * w;
    const bool bit = lane < m && ((row[pos >> 5] >> (pos & 31)) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) sm.crow[r] = bal;
  }
  uint32_t pc = __ballot_sync(0xffffffffu, lane < m && ((sm.P[lv * w + (pos >> 5)] >> (pos & 31)) & 1u));
  const uint32_t c1[1] = {m == 32 ? 0xffffffffu : ((1u << m) - 1u)};
  // only nodes with many members carry enough work to be worth splitting
  const bool pollable = a.lb_on && m >= WM_COMPACT_POLL_MIN;
  __syncwarp();
  unsigned long long part = 0;
  int head = 0, nq = 0;
  while (pc) {
    const int i = pop_hi(pc);
    const uint32_t word = sm.crow[i];  // row i is already restricted to C
    sm.queue[ring_slot(word, head + nq)] = ((uint32_t)i << 16) | (uint32_t)lane;
    nq += __popc(word);
    if (nq >= 32) {
      __syncwarp();
      part += bulk4_round<1>(sm.crow, c1, sm.queue, head, 32);
      __syncwarp();
      head = (head + 32) & 63;
      nq -= 32;
    }
    if (pollable && ++tc.poll >= a.lb_poll) {
      tc.poll = 0;
      if (lane == 0) ++sm.n_polls;
      int want = 0;
      if (lane == 0) {
        want = (int)(pt - ph) >= a.idle_min;
        pt = (uint32_t)ld_relaxed(&a.L.lb->tail);
        ph = (uint32_t)ld_relaxed(&a.L.lb->head);
      }
      if (__shfl_sync(0xffffffffu, want, 0)) {
        const bool mine = lane < m && ((pc >> lane) & 1u);
#pragma unroll
        for (int x = 0; x < w; ++x) {
          const uint32_t v = __reduce_or_sync(0xffffffffu, (mine && (pos >> 5) == x) ? 1u << (pos & 31) : 0u);
          if (lane == 0) sm.P[lv * w + x] = v;
        }
        __syncwarp();
        try_donate<w>(sm.C, sm.P, a, s0, lv, task);
        pc = __ballot_sync(0xffffffffu,
                           lane < m && ((sm.P[lv * w + (pos >> 5)] >> (pos & 31)) & 1u));
        __syncwarp();
      }
    }
  }
  if (nq) {
    __syncwarp();
    part += bulk4_round<1>(sm.crow, c1, sm.queue, head, nq);
    __syncwarp();
  }
  return part;
}

// The pending children of a four-level bulk node stay in the stack's P[lv]
// (popped one at a time, like move_step), so the balancer can donate half of
// them mid-node: with whole bulk nodes as the unit of work the tail of a
// small-k run would otherwise wait on the largest node.  Polls happen per
// child, software-pipelined as in run_task.
template <int w, int WMAX>
__device__ __forceinline__ unsigned long long bulk4(CliqueSmem<WMAX> &sm, const CliqueArgs &a,
                                                    int lv, int s0, unsigned long long task,
                                                    TaskCounters &tc, uint32_t &pt,
                                                    uint32_t &ph) {
  constexpr int S = Width<w>::S;
  const int lane = lane_id();
  if (w > 1) {
    int m = 0;
#pragma unroll
    for (int x = 0; x < w; ++x) m += __popc(sm.C[lv * w + x]);
    if (m <= 32) return bulk4_compact<w, WMAX>(sm, a, lv, m, s0, task, tc, pt, ph);
  }
  const uint32_t *adj = sm.adj;
  uint32_t *queue = sm.queue;
  uint32_t *Ps = sm.P + lv * w;
  uint32_t c[w];
#pragma unroll
  for (int x = 0; x < w; ++x) c[x] = sm.C[lv * w + x];
  unsigned long long part = 0;
  int head = 0, nq = 0;  // warp-uniform ring state
  for (int q = 0; q < w; ++q) {
    uint32_t pm = Ps[q];  // pending children of word q, in a register between polls
    while (pm) {
      const int i = q * 32 + pop_hi(pm);
      uint32_t ci[w];
      load_row<w>(adj + i * S, ci);  // broadcast read
#pragma unroll
      for (int x = 0; x < w; ++x) {
        const uint32_t word = ci[x] & c[x];  // the child's candidates: its own ballot
        if (word == 0u) continue;
        queue[ring_slot(word, head + nq)] = ((uint32_t)i << 16) | (uint32_t)(x * 32 + lane);
        nq += __popc(word);
        if (nq >= 32) {
          __syncwarp();
          part += bulk4_round<w>(adj, c, queue, head, 32);
          __syncwarp();
          head = (head + 32) & 63;
          nq -= 32;
        }
      }
      if (a.lb_on && ++tc.poll >= a.lb_poll) {
        tc.poll = 0;
        if (lane == 0) ++sm.n_polls;
        int want = 0;
        if (lane == 0) {
          want = (int)(pt - ph) >= a.idle_min;
          pt = (uint32_t)ld_relaxed(&a.L.lb->tail);
          ph = (uint32_t)ld_relaxed(&a.L.lb->head);
        }
        if (__shfl_sync(0xffffffffu, want, 0)) {
          // expose the pending children, donate, take back what is left
          __syncwarp();  // every lane's read of Ps[q] precedes lane 0's write
          if (lane == 0) Ps[q] = pm;
          __syncwarp();
          try_donate<w>(sm.C, sm.P, a, s0, lv, task);
          pm = Ps[q];
          __syncwarp();
        }
      }
    }
    __syncwarp();  // (racecheck) reads of Ps[q] before the reset
    if (lane == 0) Ps[q] = 0u;
  }
  if (nq) {
    __syncwarp();
    part += bulk4_round<w>(adj, c, queue, head, nq);
    __syncwarp();
  }
  return part;
}

// Five-level bulk for a node at traversal length k-5 whose candidate set has
// m <= 32 members (always true for one-word roots): with R[x] the node's
// one-word rows (the root's own rows when w = 1, else the compacted rows),
//   leaves = sum_{h in P} sum_{i in C_h} sum_{j in C_hi} sum_{l in C_hij} popc(C_hij & R[l])
// The (h, i, j) triples of ALL children h share one 64-entry ring, so rounds
// stay full across sibling subtrees and the per-(k-4)-node work of bulk4
// (compaction, child pops, partial rounds) disappears: the bulk4 node of each
// child h is just the word C_h = c & R[h].  Returns false (nothing done) when
// the node is too wide to compact; the DFS then continues to bulk4.
// One round: each lane takes one queued candidate set C_hij (its (h, i, j)
// triple's set, computed at push time) and counts the edges inside it.
__device__ __forceinline__ unsigned long long bulk5_round(const uint32_t *R,
                                                          const uint32_t *queue, int head,
                                                          int nq) {
  const int lane = lane_id();
  uint32_t part = 0;  // <= 32 * 32 per round
  if (lane < nq) {
    const uint32_t cij = queue[(head + lane) & 63];
    uint32_t m = cij;
    m &= m - 1u;  // rows are lower-triangular: the lowest member adds nothing
    while (m) part += __popc(cij & R[pop_hi(m)]);
  }
  return part;
}

template <int w, int WMAX>
__device__ __forceinline__ bool bulk5(CliqueSmem<WMAX> &sm, const CliqueArgs &a, int lv, int s0,
                                      unsigned long long task, TaskCounters &tc, uint32_t &pt,
                                      uint32_t &ph, unsigned long long &out) {
  const int lane = lane_id();
  const uint32_t *R;
  uint32_t c, pc;
  int m = 0, pos = -1;
  if (w == 1) {
    R = sm.adj;  // stride 1: the root's rows are already one word
    c = sm.C[lv];
    pc = sm.P[lv];
  } else {
#pragma unroll
    for (int x = 0; x < w; ++x) m += __popc(sm.C[lv * w + x]);
    if (m > 32) return false;
    {
      int before = 0;
#pragma unroll
      for (int x = 0; x < w; ++x) {
        const uint32_t cw = sm.C[lv * w + x];
        if ((cw >> lane) & 1u)
          sm.crow[before + __popc(cw & ((1u << lane) - 1u))] = (uint32_t)(x * 32 + lane);
        before += __popc(cw);
      }
    }
    __syncwarp();
    pos = lane < m ? (int)sm.crow[lane] : -1;
    __syncwarp();
    for (int r = 0; r < m; ++r) {
      const int pr = __shfl_sync(0xffffffffu, pos, r);
      const uint32_t *row = sm.adj + pr * w;
      const bool bit = lane < m && ((row[pos >> 5] >> (pos & 31)) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) sm.crow[r] = bal;
    }
    pc = __ballot_sync(0xffffffffu,
                       lane < m && ((sm.P[lv * w + (pos >> 5)] >> (pos & 31)) & 1u));
    R = sm.crow;
    c = m == 32 ? 0xffffffffu : ((1u << m) - 1u);
    __syncwarp();
  }
  const bool pollable = a.lb_on && __popc(pc) >= WM_BULK5_POLL_MIN;
  unsigned long long part = 0;
  int head = 0, nq = 0;
  // (h, i) pairs of several children flattened through a 64-entry pair ring,
  // 32 per batch (one per lane, word = C_hi): push rounds then run with most
  // lanes busy instead of |C_h| of them (a child has few members: the
  // per-child rounds pushed ~4 triples each).  cfg3 k=8 5.85 -> 5.22 ms, k=9
  // 26.46 -> 21.43, k=10 118.7 -> 93.3, cfg5 k=8 67.9 -> 53.5
  // (profiles/r02_ab_pairq.log).  The rings hold the candidate sets themselves
  // (C_hi, C_hij, computed at push) and skip every set too small to reach a
  // counted edge (child < 4, pair < 3, triple < 2 members): k=9 21.4 -> 19.0
  // ms, k=10 93.2 -> 81.8 (profiles/r02_ab_cijq.log, r02_ab_cijq2.log).
  const uint32_t lt = (1u << lane) - 1u;
  int phead = 0, pn = 0;
  while (pc || pn) {
    while (pc && pn < 32) {
      const int h = pop_hi(pc);
      const uint32_t ch = c & R[h];
      // a child needs >= 4 candidates and a pair >= 3 to reach a counted edge:
      // queue C_hi itself for the pairs that can
      const uint32_t ci = ((ch >> lane) & 1u) ? (ch & R[lane]) : 0u;
      const bool pk = __popc(ch) >= 4 && __popc(ci) >= 3;
      const unsigned pb = __ballot_sync(0xffffffffu, pk);
      if (pk) sm.pq[(phead + pn + __popc(pb & lt)) & 63] = ci;
      pn += __popc(pb);
      // a bulk5 child is a whole (k-4)-node: poll every WM_BULK5_POLL_EVERY
      // children (the pipelined loads keep it cheap; every child over-donates)
      if (pollable && ++tc.poll >= WM_BULK5_POLL_EVERY) {
        tc.poll = 0;
        if (lane == 0) ++sm.n_polls;
        int want = 0;
        if (lane == 0) {
          want = (int)(pt - ph) >= a.idle_min;
          pt = (uint32_t)ld_relaxed(&a.L.lb->tail);
          ph = (uint32_t)ld_relaxed(&a.L.lb->head);
        }
        if (__shfl_sync(0xffffffffu, want, 0)) {
          // expose the pending children in the original bit space, donate,
          // take back what is left
          if (w == 1) {
            if (lane == 0) sm.P[lv] = pc;
            __syncwarp();
            try_donate<w>(sm.C, sm.P, a, s0, lv, task);
            pc = sm.P[lv];
          } else {
            const bool mine = lane < m && ((pc >> lane) & 1u);
#pragma unroll
            for (int x = 0; x < w; ++x) {
              const uint32_t v =
                  __reduce_or_sync(0xffffffffu, (mine && (pos >> 5) == x) ? 1u << (pos & 31) : 0u);
              if (lane == 0) sm.P[lv * w + x] = v;
            }
            __syncwarp();
            try_donate<w>(sm.C, sm.P, a, s0, lv, task);
            pc = __ballot_sync(0xffffffffu,
                               lane < m && ((sm.P[lv * w + (pos >> 5)] >> (pos & 31)) & 1u));
          }
          __syncwarp();
        }
      }
    }
    __syncwarp();
    const int take = pn < 32 ? pn : 32;
    const uint32_t ci = lane < take ? sm.pq[(phead + lane) & 63] : 0u;  // C_hi
    phead = (phead + take) & 63;
    pn -= take;
    __syncwarp();
    // each j of C_hi: C_hij = C_hi & R[j] goes into the ring unless it has
    // fewer than two members (no edge inside: nothing to count)
    uint32_t word = ci;
    for (;;) {
      if (!__any_sync(0xffffffffu, word != 0u)) break;
      uint32_t t = 0u;
      if (word) t = ci & R[pop_hi(word)];
      const bool keep = (t & (t - 1u)) != 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) sm.queue[(head + nq + __popc(bal & lt)) & 63] = t;
      nq += __popc(bal);
      if (nq >= 32) {
        __syncwarp();
        part += bulk5_round(R, sm.queue, head, 32);
        __syncwarp();
        head = (head + 32) & 63;
        nq -= 32;
      }
    }
  }
  if (nq) {
    __syncwarp();
    part += bulk5_round(R, sm.queue, head, nq);
    __syncwarp();
  }
  out = part;
  return true;
}

// Process one task (root or donated level) of word width w.
template <int w, int WMAX, bool BYTES>
// inlined into the kernel (its three width instantiations): the out-of-line
// form's call ABI kept a 272-byte local stack frame per thread (20.7 MB of
// DRAM writes per launch) and cost cfg3 k=8 6.45 -> 5.77 ms, k=9 28.9 -> 26.6
// (B200 A/B, profiles/r02_ab_clique1.log)
#ifndef WM_RUNTASK_NOINLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void run_task(CliqueSmem<WMAX> &sm, const CliqueArgs &a, int kind,
                                      unsigned long long task, int s0, int32_t root, int d,
                                      int64_t lb, const Rec3 &rec, bool stage, bool split,
                                      TaskCounters &tcio) {
  constexpr int S = Width<w>::S;
  const int lane = lane_id();
  TaskCounters tc = tcio;  // registers for the hot loop (tcio lives in local memory)
  const int k = a.k;
  uint32_t *C = sm.C;
  uint32_t *P = sm.P;
  uint32_t *adj = sm.adj;
  if (stage) {
    // stage the root's rows from the arena (L2-resident) into smem
    // (arena rows hold wv = ceil(d/32) words; words wv..w-1 of a row are
    // never read unmasked: C is zero there)
    const uint32_t *src = a.bm + __ldg(a.bm_off + task);
    const int wv = (d + 31) >> 5;
    if (w == 1) {
      for (int i = lane; i < d; i += 32) adj[i] = __ldg(src + i);
    } else if (wv == w) {
      for (int i = lane; i < d * w; i += 32) {
        const int r = i / w, x = i - r * w;
        adj[r * S + x] = __ldg(src + i);
      }
    } else {
      for (int i = lane; i < d * wv; i += 32) {
        const int r = i / wv, x = i - r * wv;
        adj[r * S + x] = __ldg(src + i);
      }
    }
  }
  {
    // donated record: words 2..w+1 = C[s0], w+2..2w+1 = pending subset
    const uint32_t cv = rec_word(rec, kRecHdr + lane);
    const uint32_t pv = rec_word(rec, kRecHdr + w + lane);
    if (lane < w) {
      uint32_t cword, pword;
      if (kind == 1) {
        const int lo = lane * 32;
        cword = d >= lo + 32 ? 0xffffffffu : (d > lo ? (1u << (d - lo)) - 1u : 0u);
        pword = cword;
        if (split) {  // this shard's level-1 members: (member + task) = rank (mod N)
          const uint32_t N = (uint32_t)a.task_stride;
          const uint32_t base = (uint32_t)(((unsigned long long)lo + task) % N);
          uint32_t mine = 0u;
          for (uint32_t j = ((uint32_t)a.task_offset + N - base) % N; j < 32u; j += N)
            mine |= 1u << j;
          pword &= mine;
        }
      } else {
        cword = cv;
        pword = pv;
      }
      C[s0 * w + lane] = cword;
      P[s0 * w + lane] = pword;
    }
  }
  if (BYTES && lane == 0) {
    sm.below[s0] = 0;
    sm.last[s0] = root;
  }
  __syncwarp();
  // balancer poll, software-pipelined: the idle-ticket counters loaded at one
  // poll are consumed at the next, so the L2 round trip never stalls the DFS
  uint32_t pt = 0, ph = 0;  // low words suffice: tail - head is small
  if (!BYTES && a.lb_on && lane == 0) {
    pt = (uint32_t)ld_relaxed(&a.L.lb->tail);
    ph = (uint32_t)ld_relaxed(&a.L.lb->head);
  }
  if (!BYTES && k >= WM_BULK5_MINK && s0 == k - 5) {
    // the task itself is a five-level bulk node (if it compacts)
    unsigned long long part = 0;
    if (bulk5<w, WMAX>(sm, a, s0, s0, task, tc, pt, ph, part)) {
      tc.acc += part;
      tcio = tc;
      return;
    }
  }
  if (!BYTES && k >= WM_BULK4_MINK && s0 == k - 4) {
    // the task itself is a four-level bulk node
    tc.acc += bulk4<w, WMAX>(sm, a, s0, s0, task, tc, pt, ph);
    tcio = tc;
    return;
  }
  if (s0 >= k - 3) {
    // the task itself is a bulk node
    unsigned long long bytes = 0;
    const unsigned long long part =
        (s0 == k - 2) ? bulk2<w, BYTES>(adj, C + s0 * w, a, lb, bytes)
                      : bulk3<w, BYTES>(adj, C + s0 * w, P + s0 * w, a, lb, bytes);
    tc.acc += part;
    if (BYTES) {
      tc.bytes += bytes;
      if (warp_sum_u64(part) && lane == 0) tc.bytes += outdeg_bytes(a, root);
    }
    tcio = tc;
    return;
  }
  int s = s0;
  for (;;) {
    // move_step: next unconsumed member at level s (lowest set bit)
    const uint32_t pw = lane < w ? P[s * w + lane] : 0u;
    const unsigned nz = __ballot_sync(0xffffffffu, pw != 0u);
    if (nz == 0u) {
      if (BYTES && lane == 0) {
        const unsigned long long b = sm.below[s];
        if (b) {
          tc.bytes += outdeg_bytes(a, sm.last[s]);
          if (s > s0) sm.below[s - 1] += b;
        }
      }
      __syncwarp();
      if (s == s0) break;
      --s;
      continue;
    }
    const int wl = __ffs(nz) - 1;
    const uint32_t word = __shfl_sync(0xffffffffu, pw, wl);
    const int i = wl * 32 + __ffs(word) - 1;
    if (lane == wl) P[s * w + wl] = word & (word - 1u);
    // extend + lower + clique, fused: C_{s+1} = C_s & A[i]
    uint32_t cw = 0u;
    if (lane < w) {
      cw = C[s * w + lane] & adj[i * S + lane];
      C[(s + 1) * w + lane] = cw;
    }
    const int cnt = __reduce_add_sync(0xffffffffu, __popc(cw));
    __syncwarp();
    if (lane == 0) ++sm.n_nodes;
    unsigned long long part5 = 0;
    bool done5 = false;
    if (!BYTES && k >= WM_BULK5_MINK && s + 1 == k - 5 && cnt >= k - s - 1) {
      if (lane < w) P[(s + 1) * w + lane] = cw;
      __syncwarp();
      done5 = bulk5<w, WMAX>(sm, a, s + 1, s0, task, tc, pt, ph, part5);
      tc.acc += part5;
    }
    if (done5) {
      // the child node was finished in bulk
    } else if (cnt >= k - s - 1) {
      if (!BYTES && k >= WM_BULK4_MINK && s + 1 == k - 4) {
        if (lane < w) P[(s + 1) * w + lane] = cw;
        __syncwarp();
        tc.acc += bulk4<w, WMAX>(sm, a, s + 1, s0, task, tc, pt, ph);
      } else if (s + 1 == k - 3) {
        unsigned long long bytes = 0;
        const unsigned long long part =
            bulk3<w, BYTES>(adj, C + (s + 1) * w, C + (s + 1) * w, a, lb, bytes);
        tc.acc += part;
        if (BYTES) {
          tc.bytes += bytes;
          const unsigned long long tot = warp_sum_u64(part);
          if (lane == 0 && tot) {
            tc.bytes += outdeg_bytes(a, __ldg(a.dnbr + lb + i));
            sm.below[s] += tot;
          }
        }
        __syncwarp();
      } else {
        ++s;
        if (lane < w) P[s * w + lane] = cw;
        if (BYTES && lane == 0) {
          sm.below[s] = 0;
          sm.last[s] = __ldg(a.dnbr + lb + i);
        }
        __syncwarp();
      }
    }
    // on-device load balancing (opt mode): poll the idle-warp ring
    if (!BYTES && a.lb_on && ++tc.poll >= a.lb_poll) {
      tc.poll = 0;
      if (lane == 0) ++sm.n_polls;
      int want = 0;
      if (lane == 0) {
        want = (int)(pt - ph) >= a.idle_min;
        pt = (uint32_t)ld_relaxed(&a.L.lb->tail);
        ph = (uint32_t)ld_relaxed(&a.L.lb->head);
      }
      if (__shfl_sync(0xffffffffu, want, 0)) try_donate<w>(C, P, a, s0, s, task);
    }
  }
  tcio = tc;
}

// <= 51 registers for the narrow classes: 5 blocks (40 warps) per SM
#ifndef WM_ENUM_MINBLOCKS
#define WM_ENUM_MINBLOCKS 5
#endif
// (W = 8: <= 128 registers keeps two blocks per SM)
#ifndef WM_ENUM_MINBLOCKS_W8
#define WM_ENUM_MINBLOCKS_W8 2
#endif
template <int WMAX, bool BYTES>
__global__ void __launch_bounds__(256, WMAX <= 4 ? WM_ENUM_MINBLOCKS
                                                 : (WMAX == 8 ? WM_ENUM_MINBLOCKS_W8 : 1))
    clique_enum_kernel(CliqueArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  CliqueSmem<WMAX> &sm = reinterpret_cast<CliqueSmem<WMAX> *>(smraw)[threadIdx.x >> 5];
  const int lane = lane_id();
  WarpClock clk;
  warp_clock_begin(clk, a.L.lb);
  bool roots_left = true;
  TaskCounters tc = {0, 0, 0, 0, 0};
  if (lane == 0) sm.n_nodes = sm.n_polls = 0;
  __syncwarp();
  unsigned long long tasks_done = 0;
  unsigned long long cached = ~0ull;
  for (;;) {
    unsigned long long ti = 0;
    Rec3 rec = {{0u, 0u, 0u}};
    const int kind = acquire_work(a.L, a.lb_on, a.ntasks, roots_left, ti, rec, clk);
    if (kind == 0) break;
    unsigned long long task;
    int s0;
    bool split = false;
    if (kind == 1) {
      if (ti < a.heavy) {
        task = ti;
        split = true;
        tasks_done += (task % a.task_stride == a.task_offset);  // count each task once
      } else {
        task = a.rem_first + (ti - a.heavy) * a.task_stride;
        ++tasks_done;
      }
      s0 = 1;
    } else {
      task = __shfl_sync(0xffffffffu, rec.w[0], 0);
      s0 = (int)__shfl_sync(0xffffffffu, rec.w[0], 1);
    }
    const int32_t root = __ldg(a.tasks + task);
    const int64_t lb = __ldg(a.doff + root);
    const int d = (int)(__ldg(a.doff + root + 1) - lb);
    const bool stage = task != cached;
    cached = task;
    const int wv = (d + 31) >> 5;
    if (WMAX <= 4) {
      if (wv <= 1) run_task<1, WMAX, BYTES>(sm, a, kind, task, s0, root, d, lb, rec, stage, split, tc);
      else if (wv <= 2) run_task<(WMAX >= 2 ? 2 : 1), WMAX, BYTES>(sm, a, kind, task, s0, root, d, lb, rec, stage, split, tc);
      else run_task<WMAX, WMAX, BYTES>(sm, a, kind, task, s0, root, d, lb, rec, stage, split, tc);
    } else {
      run_task<WMAX, WMAX, BYTES>(sm, a, kind, task, s0, root, d, lb, rec, stage, split, tc);
    }
  }
  const unsigned long long acc = warp_sum_u64(tc.acc);
  const unsigned long long bytes = BYTES ? warp_sum_u64(tc.bytes) : 0;
  if (lane == 0) {
    atomicAdd(&a.counters[0], acc);
    if (BYTES) atomicAdd(&a.counters[1], bytes);
    atomicAdd(&a.counters[2], tasks_done);
    atomicAdd(&a.counters[3], sm.n_nodes);
    atomicAdd(&a.counters[4], sm.n_polls);
  }
  warp_clock_end(a.L.lb, clk);
}


// --------------------------------------------------------------------------
// 3) DM_DFS ablation (mode "dfs", reference engine.py:13-16, :274-294): one
// THREAD per traversal, the paper's baseline that DFS-wide is measured
// against (Table 4).  Each thread owns a root, keeps its candidate
// lists C_L = C_{L-1} ∩ N+(tr[L-1]) in a private HBM arena and intersects
// sorted lists by a scalar merge — uncoalesced, divergent, no warp
// cooperation.  Same tree, same counts.

// |a ∩ b| (both ascending), optionally writing the intersection to out
__device__ __forceinline__ int merge_intersect(const int32_t *__restrict__ a, int na,
                                               const int32_t *__restrict__ b, int nb,
                                               int32_t *__restrict__ out) {
  int i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    const int32_t x = a[i], y = __ldg(b + j);
    if (x == y) {
      if (out) out[c] = x;
      ++c; ++i; ++j;
    } else if (x < y) {
      ++i;
    } else {
      ++j;
    }
  }
  return c;
}

__global__ void __launch_bounds__(256) clique_dfs_kernel(
    const int64_t *__restrict__ doff, const int32_t *__restrict__ dnbr,
    const int32_t *__restrict__ tasks, unsigned long long ntasks, unsigned long long task_offset,
    unsigned long long task_stride, int k, int32_t *__restrict__ arena, int cap,
    unsigned long long *__restrict__ counters) {
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t *base = arena + tid * (unsigned long long)(k - 2) * (unsigned long long)cap;
  unsigned long long acc = 0, nodes = 0, done = 0;
  const int32_t *ptr[kMaxK];
  int len[kMaxK], pos[kMaxK];
  for (;;) {
    const unsigned long long ti = atomicAdd(&counters[16], 1ull);  // root cursor (engine.py:187)
    if (ti >= ntasks) break;
    ++done;
    const int32_t root = __ldg(tasks + task_offset + ti * task_stride);
    const int64_t rb = __ldg(doff + root);
    ptr[1] = dnbr + rb;
    len[1] = (int)(__ldg(doff + root + 1) - rb);
    pos[1] = 0;
    int L = 1;
    while (L >= 1) {
      if (pos[L] == len[L]) { --L; continue; }
      const int32_t v = ptr[L][pos[L]++];
      const int64_t vb = __ldg(doff + v);
      const int vd = (int)(__ldg(doff + v + 1) - vb);
      ++nodes;
      if (L == k - 2) {
        acc += (unsigned long long)merge_intersect(ptr[L], len[L], dnbr + vb, vd, nullptr);
      } else {
        int32_t *out = base + (size_t)(L - 1) * cap;
        const int c = merge_intersect(ptr[L], len[L], dnbr + vb, vd, out);
        if (c >= k - L - 1) {
          ++L;
          ptr[L] = out;
          len[L] = c;
          pos[L] = 0;
        }
      }
    }
  }
  acc = warp_sum_u64(acc);
  nodes = warp_sum_u64(nodes);
  done = warp_sum_u64(done);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&counters[0], acc);
    atomicAdd(&counters[2], done);
    atomicAdd(&counters[3], nodes);
  }
}

static int run_clique_dfs(Graph *g, const wm_cfg *cfg, int k, unsigned long long ntask,
                          int maxout, wm_result *res, cudaStream_t s, cudaEvent_t k0,
                          cudaEvent_t k1) {
  unsigned long long *ctr = g->ws->counters.as<unsigned long long>();
  const unsigned long long ro = (unsigned long long)cfg->shard_rank;
  const unsigned long long nt =
      ntask > ro ? (ntask - ro + cfg->shard_count - 1) / cfg->shard_count : 0;
  // private arenas: (k-2) levels of maxout entries per thread; thread count
  // bounded by the memory budget (a scaled-down copy of the reference's
  // per-lane TE, engine.py:83-152)
  const int cap = maxout > 0 ? maxout : 1;
  const unsigned long long per = (unsigned long long)(k - 2) * cap * sizeof(int32_t);
  size_t free_b = 0, total_b = 0;
  WM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const unsigned long long budget = (unsigned long long)(free_b * 0.5) + g->ws->arena.bytes;
  unsigned long long threads = (unsigned long long)g->num_sms * 2048ull;
  if (threads > nt) threads = nt > 0 ? nt : 1;
  while (threads > 256 && threads * per > budget) threads >>= 1;
  const int blocks = (int)((threads + 255) / 256);
  int st = g->ws->arena.ensure((size_t)blocks * 256 * per);
  if (st) return st;
  WM_CUDA(cudaEventRecord(k0, s));
  if (nt)
    clique_dfs_kernel<<<blocks, 256, 0, s>>>(
        g->ws->dag_off.as<int64_t>(), g->ws->dag_nbr.as<int32_t>(), g->ws->vals_out.as<int32_t>(),
        nt, ro, (unsigned long long)cfg->shard_count, k, g->ws->arena.as<int32_t>(), cap, ctr);
  WM_CUDA(cudaGetLastError());
  WM_CUDA(cudaEventRecord(k1, s));
  res->warps = blocks * 8;
  res->launches += nt ? 1 : 0;
  return WM_OK;
}

// --------------------------------------------------------------------------
// host launcher

template <int W>
static int launch_build(Graph *g, const CliqueArgs &a, unsigned long long ntask,
                        unsigned long long all_below, unsigned long long first,
                        unsigned long long stride, int order, int rank_order, cudaStream_t s) {
  const size_t per_warp = sizeof(BuildSmem<W>);
  int wpb = 8;
  while (wpb > 1 && per_warp * wpb > 200 * 1024) wpb >>= 1;
  const size_t smem = per_warp * wpb;
  auto kern = clique_build_kernel<W>;
  WM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int bps = 0;
  WM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, wpb * 32, smem));
  if (bps < 1) return fail(WM_ECAPACITY, "clique build kernel W=%d does not fit on an SM", W);
  unsigned long long blocks = (unsigned long long)g->num_sms * bps;
  const unsigned long long below = all_below < ntask ? all_below : ntask;
  const unsigned long long mine =
      below + (first < ntask ? (ntask - first + stride - 1) / stride : 0);
  if (!mine) return WM_OK;
  const unsigned long long need = (mine + wpb - 1) / wpb;
  if (blocks > need) blocks = need;
  kern<<<(int)blocks, wpb * 32, smem, s>>>(a.doff, a.dnbr, a.tasks, ntask, a.bm_off,
                                           const_cast<uint32_t *>(a.bm), below, first, stride,
                                           g->offsets, order, rank_order);
  WM_CUDA(cudaGetLastError());
  return WM_OK;
}

struct EnumPlan {
  int wpb = 0, blocks = 0, warps = 0;
  size_t smem = 0;
};

template <int WMAX, bool BYTES>
static int plan_enum(Graph *g, const wm_cfg *cfg, unsigned long long ntasks, bool lb_on,
                     EnumPlan *p) {
  const size_t per_warp = sizeof(CliqueSmem<WMAX>);
  int wpb = cfg->warps_per_block > 0 ? cfg->warps_per_block : 8;
  while (wpb > 1 && per_warp * wpb > 200 * 1024) wpb >>= 1;
  const size_t smem = per_warp * wpb;
  auto kern = clique_enum_kernel<WMAX, BYTES>;
  WM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int bps = 0;
  WM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, wpb * 32, smem));
  if (cfg->blocks_per_sm > 0 && cfg->blocks_per_sm < bps) bps = cfg->blocks_per_sm;
  if (bps < 1) return fail(WM_ECAPACITY, "clique kernel W=%d does not fit on an SM", WMAX);
  int blocks = g->num_sms * bps;
  if (!lb_on) {  // no stealing: no point in more warps than tasks
    const unsigned long long need = (ntasks + wpb - 1) / wpb;
    if ((unsigned long long)blocks > need) blocks = (int)(need > 0 ? need : 1);
  }
  p->wpb = wpb;
  p->blocks = blocks;
  p->warps = blocks * wpb;
  p->smem = smem;
  return WM_OK;
}

template <int WMAX, bool BYTES>
static int launch_enum(Graph *g, const wm_cfg *cfg, CliqueArgs a, const EnumPlan &p,
                       cudaStream_t s) {
  int st = lb_prepare(g, a.L.lb, p.warps, (uint32_t)(kRecHdr + 2 * WMAX), &a.L, s);
  if (st) return st;
  a.idle_min = (int)((1.0 - cfg->lb_threshold) * p.warps);
  if (a.idle_min < 1) a.idle_min = 1;
  clique_enum_kernel<WMAX, BYTES><<<p.blocks, p.wpb * 32, p.smem, s>>>(a);
  WM_CUDA(cudaGetLastError());
  return WM_OK;
}

// WM_PHASES=1: print per-phase device times of run_clique to stderr (tuning aid)

// --------------------------------------------------------------------------
// Roots wider than the W=32 class (> 1024 out-neighbours): the k-cliques whose
// lowest vertex is v are exactly {v} + the (k-1)-cliques of the subgraph
// induced on N+(v), counted in any orientation.  Such roots are taken out of
// the bitmap launch and each one's induced subgraph is counted by a nested
// run (degree orientation inside it; nested wide roots recurse the same way).

// warp per member i of the ascending member list M: how many of N(M[i]) are in M
__global__ void induced_count_kernel(int d, const int32_t *__restrict__ M,
                                     const int64_t *__restrict__ off,
                                     const int32_t *__restrict__ nbr, int64_t *__restrict__ cnt) {
  const int lane = lane_id();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < d; i += nw) {
    const int32_t u = M[i];
    int64_t c = 0;
    for (int64_t p0 = off[u]; p0 < off[u + 1]; p0 += 32) {
      const int64_t p = p0 + lane;
      bool in = false;
      if (p < off[u + 1]) {
        const int32_t v = nbr[p];
        const int j = lower_bound_i(M, d, v);
        in = j < d && M[j] == v;
      }
      c += __popc(__ballot_sync(0xffffffffu, in));
    }
    if (lane == 0) cnt[i] = c;
  }
}

// same walk, writing local ids in row order (ballot+popc keeps them ascending)
__global__ void induced_fill_kernel(int d, const int32_t *__restrict__ M,
                                    const int64_t *__restrict__ off,
                                    const int32_t *__restrict__ nbr,
                                    const int64_t *__restrict__ pos, int32_t *__restrict__ out) {
  const int lane = lane_id();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < d; i += nw) {
    const int32_t u = M[i];
    int64_t w = pos[i];
    for (int64_t p0 = off[u]; p0 < off[u + 1]; p0 += 32) {
      const int64_t p = p0 + lane;
      int j = d;
      if (p < off[u + 1]) {
        const int32_t v = nbr[p];
        j = lower_bound_i(M, d, v);
        if (j < d && M[j] != v) j = d;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, j < d);
      if (j < d) out[w + __popc(bal & ((1u << lane) - 1u))] = j;
      w += __popc(bal);
    }
  }
}

static int run_clique_impl(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res,
                           cudaStream_t s, std::vector<std::vector<int32_t>> *wide, bool top);

// count the (k-1)-cliques of G[M] for every wide root's member list and add
// them (and the nested runs' statistics) into res
static int clique_wide_roots(Graph *g, const wm_app *app, const wm_cfg *cfg,
                             const std::vector<std::vector<int32_t>> &wide, wm_result *res,
                             cudaStream_t s) {
  for (const auto &M : wide) {
    const int d = (int)M.size();
    int32_t *dM = nullptr, *dnbr = nullptr;
    int64_t *cnt = nullptr, *doff = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, doff, d + 1, s));
    WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&dM), sizeof(int32_t) * d,
                                    g->ws->pool, s));
    WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&cnt), sizeof(int64_t) * (d + 1),
                                    g->ws->pool, s));
    WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&doff), sizeof(int64_t) * (d + 1),
                                    g->ws->pool, s));
    WM_CUDA(cudaMallocFromPoolAsync(&tmp, tb, g->ws->pool, s));
    WM_CUDA(cudaMemcpyAsync(dM, M.data(), sizeof(int32_t) * d, cudaMemcpyHostToDevice, s));
    WM_CUDA(cudaMemsetAsync(cnt + d, 0, sizeof(int64_t), s));
    const int blocks = (d * 32 + 255) / 256 < g->num_sms * 16 ? (d * 32 + 255) / 256
                                                                : g->num_sms * 16;
    induced_count_kernel<<<blocks, 256, 0, s>>>(d, dM, g->offsets, g->neighbors, cnt);
    WM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, doff, d + 1, s));
    std::vector<int64_t> hcnt(d + 1);
    int64_t nnz = 0;
    WM_CUDA(cudaMemcpyAsync(hcnt.data(), cnt, sizeof(int64_t) * d, cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaMemcpyAsync(&nnz, doff + d, sizeof nnz, cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaStreamSynchronize(s));
    res->h2d_bytes += sizeof(int32_t) * d;
    res->d2h_bytes += sizeof(int64_t) * (d + 1);
    res->launches += 2;
    int st = WM_OK;
    if (app->k - 1 == 2) {
      res->clique_count += (uint64_t)nnz / 2;  // 2-cliques of G[M]: its edges
      res->leaves += (uint64_t)nnz / 2;
      st = red_edges(cfg, s, doff + d);
    } else if (nnz > 0) {
      WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&dnbr), sizeof(int32_t) * nnz,
                                      g->ws->pool, s));
      induced_fill_kernel<<<blocks, 256, 0, s>>>(d, dM, g->offsets, g->neighbors, doff, dnbr);
      WM_CUDA(cudaGetLastError());
      Graph sub;
      sub.n = d;
      sub.nnz = nnz;
      for (int i = 0; i < d; ++i) sub.max_degree = hcnt[i] > sub.max_degree ? hcnt[i] : sub.max_degree;
      sub.device = g->device;
      sub.num_sms = g->num_sms;
      sub.offsets = doff;
      sub.neighbors = dnbr;
      sub.ws = g->ws;
      wm_app sa = *app;
      sa.k = app->k - 1;
      wm_cfg sc = *cfg;
      sc.root_begin = sc.root_end = -1;
      sc.shard_rank = 0;
      sc.shard_count = 1;
      sc.order = WM_ORDER_DEGREE;
      wm_result r = {};
      std::vector<std::vector<int32_t>> nested;
      st = run_clique_impl(&sub, &sa, &sc, &r, s, &nested, false);
      if (st == WM_OK && !nested.empty()) st = clique_wide_roots(&sub, &sa, &sc, nested, &r, s);
      res->clique_count += r.clique_count;
      res->leaves += r.leaves;
      res->alg_bytes += r.alg_bytes;
      res->nodes += r.nodes;
      res->polls += r.polls;
      res->kernel_ms += r.kernel_ms;
      res->device_ms += r.device_ms;
      res->build_ms += r.build_ms;
      res->launches += r.launches + 1;
      res->migrations += r.migrations;
      res->rebalance_count += r.rebalance_count;
      res->h2d_bytes += r.h2d_bytes;
      res->d2h_bytes += r.d2h_bytes;
    }
    res->tasks += 1;
    if (dnbr) cudaFreeAsync(dnbr, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(doff, s);
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(dM, s);
    if (st) return st;
  }
  return WM_OK;
}


// --------------------------------------------------------------------------
// Per-(graph, orientation) clique index.  Everything the root tasks need that
// depends only on the graph and the orientation — the oriented DAG (the
// reference's filter_lower, engine.py:331-353, as a CSR), the cost-sorted
// task order (all vertices by out-degree desc, id asc), the bitmap-arena
// offsets of every task, and the member lists of the wide roots — is built
// on the first clique run over all roots and kept on the graph handle, the
// way the reference's CsrGraph keeps its adjacency lists/sets for every later
// run (graph.py:93-103, used by engine.py:167-171).  A run over all roots
// then plans on the host from the cached sorted out-degrees: the tasks of
// k are the prefix with out-degree >= k-1, the width classes are sub-ranges
// of it, and the run needs ONE host synchronisation (the result read-back).
// Root-range runs, the DFS ablation and nested wide-root runs keep the
// per-run path below.
struct CliqueIndex {
  int64_t *dag_off = nullptr;          // [n+1]
  int32_t *dag_nbr = nullptr;          // [m]
  int32_t *tasks = nullptr;            // [n] vertices by (out-degree desc, id asc)
  unsigned long long *bm_off = nullptr;  // [n+1] arena offsets over `tasks` (wide: 0 words)
  unsigned long long arena_words = 0;
  std::vector<int32_t> sorted_deg;     // host: out-degree of tasks[i] (descending)
  std::vector<std::vector<int32_t>> wide;  // host: members of the roots with d > 1024
  // Union graph of the roots with 128 < d <= 1024 (clique_union_get): the
  // disjoint union of their out-neighbourhoods' induced subgraphs; its
  // (k-1)-cliques are exactly the k-cliques rooted at those roots.
  Graph *ug = nullptr;
  bool union_tried = false;
};

void clique_index_free(Graph *g) {
  for (int o = 0; o < 2; ++o) {
    CliqueIndex *ix = static_cast<CliqueIndex *>(g->cidx[o]);
    if (!ix) continue;
    if (g->ws) {
      cudaStream_t s = g->ws->own_stream;
      cudaFreeAsync(ix->dag_off, s);
      cudaFreeAsync(ix->dag_nbr, s);
      cudaFreeAsync(ix->tasks, s);
      cudaFreeAsync(ix->bm_off, s);
      if (ix->ug) {
        cudaFreeAsync(ix->ug->offsets, s);
        cudaFreeAsync(ix->ug->neighbors, s);
      }
    }
    if (ix->ug) {
      clique_index_free(ix->ug);
      delete ix->ug;
    }
    delete ix;
    g->cidx[o] = nullptr;
  }
}

// Union-graph rows of one wide-class root per warp: local member i's row is
// A[i] | A^T[i] over the root's bitmap (A lower-triangular: members ranked
// above i; the transpose adds those ranked below), i.e. i's neighbours inside
// the root's out-neighbourhood, emitted in ascending local index = ascending
// union id (moff[r] + local).  Pass 1 (out == nullptr) writes the degrees.
__global__ void union_rows_kernel(const int32_t *__restrict__ tasks,
                                  const int64_t *__restrict__ doff,
                                  const unsigned long long *__restrict__ bm_off,
                                  const uint32_t *__restrict__ bm, unsigned long long first,
                                  unsigned long long cnt, const int64_t *__restrict__ moff,
                                  int64_t *__restrict__ udeg, const int64_t *__restrict__ uoff,
                                  int32_t *__restrict__ out) {
  const int lane = lane_id();
  const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  for (unsigned long long r = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
       r < cnt; r += nw) {
    const unsigned long long t = first + r;
    const int32_t v = __ldg(tasks + t);
    const int d = (int)(__ldg(doff + v + 1) - __ldg(doff + v));
    const int wv = (d + 31) >> 5;
    const uint32_t *A = bm + __ldg(bm_off + t);
    const int64_t base = __ldg(moff + r);
    for (int i = 0; i < d; ++i) {
      uint32_t mine = 0u;  // lane x < wv: word x of row i of A | A^T
      for (int x = 0; x < wv; ++x) {
        const int j = 32 * x + lane;
        const bool tb = j < d && ((__ldg(A + (size_t)j * wv + (i >> 5)) >> (i & 31)) & 1u);
        const uint32_t tw = __ballot_sync(0xffffffffu, tb);
        if (lane == x) mine = __ldg(A + (size_t)i * wv + x) | tw;
      }
      const int c = __popc(mine);
      if (!out) {
        const int deg = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) udeg[base + i] = deg;
      } else {
        int pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int z = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += z;
        }
        int64_t pos = uoff[base + i] + (pre - c);
        uint32_t m = mine;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1u;
          out[pos++] = (int32_t)(base + 32 * lane + b);
        }
      }
    }
  }
}

__global__ void index_words_kernel(int64_t n, const uint32_t *__restrict__ keys,
                                   unsigned long long *__restrict__ words) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int d = t < n ? (int)keys[t] - 1 : 0;
    words[t] = d > 1024 ? 0ull : bm_words(d);  // wide roots live outside the arena
  }
}

static int clique_index_get(Graph *g, int order, cudaStream_t s, CliqueIndex **out) {
  const int o = order == WM_ORDER_ID ? 0 : 1;
  if (g->cidx[o]) {
    *out = static_cast<CliqueIndex *>(g->cidx[o]);
    return WM_OK;
  }
  const int64_t n = g->n, nnz = g->nnz;
  int st;
  if ((st = g->ws->keys_in.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->keys_out.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->vals_in.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->outdeg.ensure(sizeof(int32_t) * (n + 1)))) return st;
  if ((st = g->ws->hist.ensure(sizeof(unsigned long long) * (n + 1)))) return st;
  if ((st = g->ws->edge_src.ensure(sizeof(int32_t) * (nnz + 1)))) return st;
  if ((st = g->ws->edge_flag.ensure(sizeof(int32_t) * (nnz + 1)))) return st;
  if ((st = g->ws->edge_pos.ensure(sizeof(int32_t) * (nnz + 1)))) return st;
  size_t t1 = 0, t2 = 0, t3 = 0;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, g->ws->edge_flag.as<int32_t>(),
                                        g->ws->edge_pos.as<int32_t>(), (int)(nnz + 1), s));
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      nullptr, t2, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), g->ws->vals_in.as<int32_t>(), (int)n, 0, 32, s));
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, g->ws->hist.as<unsigned long long>(),
                                        g->ws->hist.as<unsigned long long>(), (int)(n + 1), s));
  size_t tmp = t1 > t2 ? t1 : t2;
  if (t3 > tmp) tmp = t3;
  if ((st = g->ws->cub_tmp.ensure(tmp))) return st;
  CliqueIndex *ix = new CliqueIndex();
  auto alloc = [&](void **p, size_t b) {
    return cudaMallocFromPoolAsync(p, b > 0 ? b : 4, g->ws->pool, s);
  };
  cudaError_t e = alloc(reinterpret_cast<void **>(&ix->dag_off), sizeof(int64_t) * (n + 1));
  if (e == cudaSuccess)
    e = alloc(reinterpret_cast<void **>(&ix->dag_nbr), sizeof(int32_t) * (nnz / 2 + 1));
  if (e == cudaSuccess) e = alloc(reinterpret_cast<void **>(&ix->tasks), sizeof(int32_t) * n);
  if (e == cudaSuccess)
    e = alloc(reinterpret_cast<void **>(&ix->bm_off), sizeof(unsigned long long) * (n + 1));
  if (e != cudaSuccess) {
    g->cidx[o] = ix;
    clique_index_free(g);
    return fail(WM_ECUDA, "clique index allocation failed: %s", cudaGetErrorString(e));
  }
  g->cidx[o] = ix;  // owned by the graph from here on (freed with it)
  const int tpb = 256;
  const int64_t ns = (int64_t)g->num_sms;
  const int vblocks = (int)((n * 32 + tpb - 1) / tpb < ns * 64 ? (n * 32 + tpb - 1) / tpb : ns * 64);
  const int pblocks = (int)((nnz + tpb) / tpb < ns * 32 ? (nnz + tpb) / tpb : ns * 32);
  const int nblocks = (int)((n + tpb) / tpb < ns * 16 ? (n + tpb) / tpb : ns * 16);
  int32_t *esrc = g->ws->edge_src.as<int32_t>(), *eflag = g->ws->edge_flag.as<int32_t>(),
          *epos = g->ws->edge_pos.as<int32_t>();
  orient_src_kernel<<<vblocks, tpb, 0, s>>>(n, g->offsets, esrc);
  orient_flag_kernel<<<pblocks, tpb, 0, s>>>(nnz, g->offsets, g->neighbors, esrc, order, eflag);
  size_t tb = g->ws->cub_tmp.bytes;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(g->ws->cub_tmp.ptr, tb, eflag, epos, (int)(nnz + 1), s));
  orient_scatter_kernel<<<pblocks, tpb, 0, s>>>(nnz, g->neighbors, eflag, epos, ix->dag_nbr);
  orient_off_kernel<<<nblocks, tpb, 0, s>>>(n, g->offsets, epos, ix->dag_off,
                                            g->ws->outdeg.as<int32_t>());
  // every vertex is a task candidate (k = 1 keys: out-degree + 1)
  task_keys_kernel<<<nblocks, tpb, 0, s>>>(n, g->ws->outdeg.as<int32_t>(), 1, 0, n,
                                           g->ws->keys_in.as<uint32_t>(),
                                           g->ws->vals_in.as<int32_t>());
  tb = g->ws->cub_tmp.bytes;
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      g->ws->cub_tmp.ptr, tb, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), ix->tasks, (int)n, 0, task_key_bits(g), s));
  unsigned long long *words = g->ws->hist.as<unsigned long long>();
  index_words_kernel<<<nblocks, tpb, 0, s>>>(n, g->ws->keys_out.as<uint32_t>(), words);
  tb = g->ws->cub_tmp.bytes;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(g->ws->cub_tmp.ptr, tb, words, ix->bm_off, (int)(n + 1), s));
  std::vector<uint32_t> keys((size_t)n);
  WM_CUDA(cudaMemcpyAsync(keys.data(), g->ws->keys_out.ptr, sizeof(uint32_t) * n,
                          cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaMemcpyAsync(&ix->arena_words, ix->bm_off + n, sizeof ix->arena_words,
                          cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  ix->sorted_deg.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) ix->sorted_deg[i] = (int32_t)keys[i] - 1;
  // wide roots: the sorted prefix with d > 1024
  int64_t nw = 0;
  while (nw < n && ix->sorted_deg[nw] > 1024) ++nw;
  if (nw) {
    std::vector<int32_t> ids((size_t)nw);
    std::vector<int64_t> off((size_t)n + 1);
    WM_CUDA(cudaMemcpyAsync(ids.data(), ix->tasks, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaMemcpyAsync(off.data(), ix->dag_off, sizeof(int64_t) * (n + 1),
                            cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < nw; ++i) {
      std::vector<int32_t> M((size_t)(off[ids[i] + 1] - off[ids[i]]));
      WM_CUDA(cudaMemcpyAsync(M.data(), ix->dag_nbr + off[ids[i]], sizeof(int32_t) * M.size(),
                              cudaMemcpyDeviceToHost, s));
      ix->wide.push_back(std::move(M));
    }
    WM_CUDA(cudaStreamSynchronize(s));
  }
  *out = ix;
  return WM_OK;
}

// Builds (once per graph and orientation) the union graph of the roots whose
// out-degree is in (128, 1024]: their bitmaps (the same per-root build as a
// run) turned into the symmetric adjacency of each out-neighbourhood, one
// disjoint component per root.  Such roots otherwise run in the W = 8..32
// enumeration classes (106+ registers, 9+ KB of shared memory per warp: 16
// warps per SM); the union's own tasks are narrow and run in the W <= 4 class
// at 40 warps per SM.
static int clique_union_get(Graph *g, CliqueIndex *ix, int order, cudaStream_t s) {
  if (ix->ug || ix->union_tried) return WM_OK;
  ix->union_tried = true;
  const std::vector<int32_t> &sd = ix->sorted_deg;
  unsigned long long nwide = 0, nunion = 0;
  while (nwide < sd.size() && sd[nwide] > 1024) ++nwide;
  while (nwide + nunion < sd.size() && sd[nwide + nunion] > 128) ++nunion;
  if (!nunion) return WM_OK;
  // member offsets (host; sorted degrees are cached)
  std::vector<int64_t> moff(nunion + 1, 0);
  for (unsigned long long r = 0; r < nunion; ++r) moff[r + 1] = moff[r] + sd[nwide + r];
  const int64_t U = moff[nunion];
  int st;
  if ((st = g->ws->arena.ensure(sizeof(uint32_t) * (ix->arena_words + 1)))) return st;
  // bitmaps of the union roots, bucket by bucket (c = 5, 4, 3: W = 32, 16, 8)
  {
    unsigned long long begin = nwide;
    for (int c = 5; c >= 3; --c) {
      unsigned long long cnt = 0;
      while (begin + cnt < nwide + nunion && sd[begin + cnt] > (32 << (c - 1))) ++cnt;
      if (!cnt) continue;
      CliqueArgs a;
      a.doff = ix->dag_off;
      a.dnbr = ix->dag_nbr;
      a.tasks = ix->tasks + begin;
      a.bm_off = ix->bm_off + begin;
      a.bm = g->ws->arena.as<uint32_t>();
      switch (c) {
        case 5: st = launch_build<32>(g, a, cnt, cnt, cnt, 1, order, 1, s); break;
        case 4: st = launch_build<16>(g, a, cnt, cnt, cnt, 1, order, 1, s); break;
        default: st = launch_build<8>(g, a, cnt, cnt, cnt, 1, order, 1, s); break;
      }
      if (st) return st;
      begin += cnt;
    }
  }
  int64_t *dmoff = nullptr, *udeg = nullptr, *uoff = nullptr;
  void *tmp = nullptr;
  size_t tb = 0;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, udeg, uoff, (int)(U + 1), s));
  WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&dmoff), sizeof(int64_t) * (nunion + 1),
                                  g->ws->pool, s));
  WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&udeg), sizeof(int64_t) * (U + 1),
                                  g->ws->pool, s));
  WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&uoff), sizeof(int64_t) * (U + 1),
                                  g->ws->pool, s));
  WM_CUDA(cudaMallocFromPoolAsync(&tmp, tb > 0 ? tb : 16, g->ws->pool, s));
  WM_CUDA(cudaMemcpyAsync(dmoff, moff.data(), sizeof(int64_t) * (nunion + 1),
                          cudaMemcpyHostToDevice, s));
  WM_CUDA(cudaMemsetAsync(udeg + U, 0, sizeof(int64_t), s));
  const int64_t want = ((int64_t)nunion * 32 + 255) / 256;
  const int blocks = (int)(want < (int64_t)g->num_sms * 16 ? want : (int64_t)g->num_sms * 16);
  union_rows_kernel<<<blocks, 256, 0, s>>>(ix->tasks, ix->dag_off, ix->bm_off,
                                           g->ws->arena.as<uint32_t>(), nwide, nunion, dmoff,
                                           udeg, nullptr, nullptr);
  WM_CUDA(cudaGetLastError());
  WM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, udeg, uoff, (int)(U + 1), s));
  int64_t nnz = 0;
  WM_CUDA(cudaMemcpyAsync(&nnz, uoff + U, sizeof nnz, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  int32_t *unbr = nullptr;
  WM_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&unbr),
                                  sizeof(int32_t) * (nnz > 0 ? nnz : 1), g->ws->pool, s));
  union_rows_kernel<<<blocks, 256, 0, s>>>(ix->tasks, ix->dag_off, ix->bm_off,
                                           g->ws->arena.as<uint32_t>(), nwide, nunion, dmoff,
                                           nullptr, uoff, unbr);
  WM_CUDA(cudaGetLastError());
  cudaFreeAsync(dmoff, s);
  cudaFreeAsync(udeg, s);
  cudaFreeAsync(tmp, s);
  Graph *ug = new Graph();
  ug->n = U;
  ug->nnz = nnz;
  ug->device = g->device;
  ug->num_sms = g->num_sms;
  ug->ws = g->ws;
  ug->offsets = uoff;
  ug->neighbors = unbr;
  ug->max_degree = sd[nwide];  // a component has at most d vertices
  ix->ug = ug;
  return WM_OK;
}

int run_clique(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res, cudaStream_t s) {
  std::vector<std::vector<int32_t>> wide;
  int st = run_clique_impl(g, app, cfg, res, s, &wide, true);
  if (st || wide.empty()) return st;
  // each top-level wide root is one task of this shard (nested runs add none)
  if ((st = red_add(cfg, s, WM_RED_TASKS, (unsigned long long)wide.size(), 0, 0, 0))) return st;
  return clique_wide_roots(g, app, cfg, wide, res, s);
}

static int run_clique_impl(Graph *g, const wm_app *app, const wm_cfg *cfg, wm_result *res,
                           cudaStream_t s, std::vector<std::vector<int32_t>> *wide, bool top) {
  PhaseTimer pt(s);
  const int64_t n = g->n;
  const int k = app->k;
  const int order = cfg->order == WM_ORDER_ID ? WM_ORDER_ID : WM_ORDER_DEGREE;
  const bool bytes = cfg->count_bytes != 0;
  const bool lb_on = cfg->mode == WM_MODE_OPT && !bytes;
  int st;
  // all roots, warp-centric, a user graph: plan from the cached index
  const bool all_roots = (cfg->root_begin <= 0) &&
                         (cfg->root_end < 0 || cfg->root_end >= n);
  CliqueIndex *ix = nullptr;
  if (top && all_roots && cfg->mode != WM_MODE_DFS) {
    if ((st = clique_index_get(g, order, s, &ix))) return st;
  }
  if ((st = g->ws->counters.ensure(sizeof(unsigned long long) * 64))) return st;
  if ((st = g->ws->lb.ensure(sizeof(LbState) * 8))) return st;
  cudaEvent_t e0 = g->ws->ev[0], e1 = g->ws->ev[1], k0 = g->ws->ev[2], k1 = g->ws->ev[3], kb = g->ws->ev[4];
  unsigned long long *ctr = g->ws->counters.as<unsigned long long>();
  const int tpb = 256;
  const int eblocks = (int)((n + tpb - 1) / tpb < (int64_t)g->num_sms * 16
                                ? (n + tpb - 1) / tpb
                                : (int64_t)g->num_sms * 16);
  unsigned long long hb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long skip = 0, ntask = 0, arena_words = 0;
  const int64_t *doff_p = nullptr;
  const int32_t *dnbr_p = nullptr;
  Graph *union_g = nullptr;  // set: the wide classes run as this graph's (k-1)-cliques
  int32_t *tasks_sorted = nullptr;
  const unsigned long long *bm_off = nullptr;
  if (ix) {
    WM_CUDA(cudaEventRecord(e0, s));
    pt.mark("start");
    WM_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * 64, s));
    // eligible tasks: the sorted prefix with out-degree >= k-1; buckets by
    // width (d <= 32 << c), wide roots (d > 1024) first
    const std::vector<int32_t> &sd = ix->sorted_deg;
    auto count_ge = [&](int64_t x) {  // entries with degree >= x (descending order)
      return (unsigned long long)(std::upper_bound(sd.begin(), sd.end(), (int32_t)x,
                                                   [](int32_t v, int32_t e) { return v > e; }) -
                                  sd.begin());
    };
    const unsigned long long E = count_ge(k - 1);
    unsigned long long above = count_ge(1025);
    if (above > E) above = E;
    hb[6] = above;
    for (int c = 5; c >= 0; --c) {
      // bucket c: 32 << (c-1) < d <= 32 << c (bucket 0: d <= 32)
      const unsigned long long lo_excl = c > 0 ? count_ge((32ll << (c - 1)) + 1) : E;
      unsigned long long hi_incl = count_ge((32ll << c) + 1);
      unsigned long long lo = lo_excl < E ? lo_excl : E;
      if (hi_incl > E) hi_incl = E;
      hb[c] = lo > hi_incl ? lo - hi_incl : 0;
    }
    skip = hb[6];
    for (unsigned long long i = (unsigned long long)cfg->shard_rank; i < skip;
         i += (unsigned long long)cfg->shard_count)
      wide->push_back(ix->wide[i]);
    for (int c = 0; c < 6; ++c) ntask += hb[c];
    doff_p = ix->dag_off;
    dnbr_p = ix->dag_nbr;
    tasks_sorted = ix->tasks + skip;
    bm_off = ix->bm_off + skip;
    arena_words = ix->arena_words;
    res->launches = 1;
    // the W = 8..32 classes run as the union graph's (k-1)-cliques instead
    // (clique_union_get); not for the B_alg pass (its bytes are the parent's
    // tree) or k = 3 (no level left to split).  WM_CLIQUE_UNION=0 disables.
    const char *un = getenv("WM_CLIQUE_UNION");
    if (!bytes && k >= 4 && !(un && *un == '0') && (hb[3] || hb[4] || hb[5])) {
      if ((st = clique_union_get(g, ix, order, s))) return st;
      if (ix->ug) {
        union_g = ix->ug;
        // the union roots are the sorted prefix with 128 < d <= 1024; with
        // hb[3..5] cleared, tasks_sorted + (hb[5]+hb[4]+hb[3]) is the W <= 4 range
        const unsigned long long shift = hb[5] + hb[4] + hb[3];
        tasks_sorted += shift;
        bm_off += shift;
        ntask -= shift;
        hb[3] = hb[4] = hb[5] = 0;
      }
    }
    pt.mark("plan");
  } else {
  if ((st = g->ws->dag_off.ensure(sizeof(int64_t) * (n + 1)))) return st;
  if ((st = g->ws->outdeg.ensure(sizeof(int32_t) * (n + 1)))) return st;
  if ((st = g->ws->dag_nbr.ensure(sizeof(int32_t) * (g->nnz / 2 + 1)))) return st;
  if ((st = g->ws->keys_in.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->keys_out.ensure(sizeof(uint32_t) * n))) return st;
  if ((st = g->ws->vals_in.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->vals_out.ensure(sizeof(int32_t) * n))) return st;
  if ((st = g->ws->hist.ensure(sizeof(unsigned long long) * (n + 1)))) return st;  // task words
  if ((st = g->ws->table.ensure(sizeof(unsigned long long) * (n + 1)))) return st; // bm_off
  const int64_t nnz = g->nnz;
  if ((st = g->ws->edge_src.ensure(sizeof(int32_t) * (nnz + 1)))) return st;
  if ((st = g->ws->edge_flag.ensure(sizeof(int32_t) * (nnz + 1)))) return st;
  if ((st = g->ws->edge_pos.ensure(sizeof(int32_t) * (nnz + 1)))) return st;
  size_t tmp_scan = 0, tmp_sort = 0, tmp_scan2 = 0, tmp_scan3 = 0;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan3, g->ws->edge_flag.as<int32_t>(),
                                        g->ws->edge_pos.as<int32_t>(), (int)(nnz + 1), s));
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, g->ws->outdeg.as<int32_t>(),
                                        g->ws->dag_off.as<int64_t>(), (int)(n + 1), s));
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      nullptr, tmp_sort, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), g->ws->vals_out.as<int32_t>(), (int)n, 0, 32, s));
  WM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan2, g->ws->hist.as<unsigned long long>(),
                                        g->ws->table.as<unsigned long long>(), (int)(n + 1), s));
  size_t tmp = tmp_scan > tmp_sort ? tmp_scan : tmp_sort;
  if (tmp_scan2 > tmp) tmp = tmp_scan2;
  if (tmp_scan3 > tmp) tmp = tmp_scan3;
  if ((st = g->ws->cub_tmp.ensure(tmp))) return st;

  WM_CUDA(cudaEventRecord(e0, s));
  pt.mark("start");
  WM_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * 64, s));
  const int vblocks = (int)((n * 32 + tpb - 1) / tpb < (int64_t)g->num_sms * 64
                                ? (n * 32 + tpb - 1) / tpb
                                : (int64_t)g->num_sms * 64);
  const int pblocks = (int)((nnz + tpb) / tpb < (int64_t)g->num_sms * 32
                                ? (nnz + tpb) / tpb
                                : (int64_t)g->num_sms * 32);
  const int nblocks = (int)((n + tpb) / tpb < (int64_t)g->num_sms * 16 ? (n + tpb) / tpb
                                                                      : (int64_t)g->num_sms * 16);
  int32_t *esrc = g->ws->edge_src.as<int32_t>(), *eflag = g->ws->edge_flag.as<int32_t>(),
          *epos = g->ws->edge_pos.as<int32_t>();
  orient_src_kernel<<<vblocks, tpb, 0, s>>>(n, g->offsets, esrc);
  orient_flag_kernel<<<pblocks, tpb, 0, s>>>(nnz, g->offsets, g->neighbors, esrc, order, eflag);
  size_t tb = g->ws->cub_tmp.bytes;
  WM_CUDA(cub::DeviceScan::ExclusiveSum(g->ws->cub_tmp.ptr, tb, eflag, epos, (int)(nnz + 1), s));
  orient_scatter_kernel<<<pblocks, tpb, 0, s>>>(nnz, g->neighbors, eflag, epos,
                                                g->ws->dag_nbr.as<int32_t>());
  orient_off_kernel<<<nblocks, tpb, 0, s>>>(n, g->offsets, epos, g->ws->dag_off.as<int64_t>(),
                                            g->ws->outdeg.as<int32_t>());
  pt.mark("orient");
  const int64_t rb = cfg->root_begin < 0 ? 0 : cfg->root_begin;
  const int64_t re = (cfg->root_end < 0 || cfg->root_end > n) ? n : cfg->root_end;
  task_keys_kernel<<<eblocks, tpb, 0, s>>>(n, g->ws->outdeg.as<int32_t>(), k, rb, re,
                                           g->ws->keys_in.as<uint32_t>(), g->ws->vals_in.as<int32_t>());
  tb = g->ws->cub_tmp.bytes;
  WM_CUDA(cub::DeviceRadixSort::SortPairsDescending(
      g->ws->cub_tmp.ptr, tb, g->ws->keys_in.as<uint32_t>(), g->ws->keys_out.as<uint32_t>(),
      g->ws->vals_in.as<int32_t>(), g->ws->vals_out.as<int32_t>(), (int)n, 0,
      task_key_bits(g), s));
  bucket_count_kernel<<<eblocks, tpb, 0, s>>>(n, g->ws->keys_out.as<uint32_t>(), ctr + 8);
  pt.mark("task sort");
  WM_CUDA(cudaMemcpyAsync(hb, ctr + 8, sizeof hb, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  res->launches = 5;
  if (cfg->mode == WM_MODE_DFS) {
    unsigned long long ntask = 0;
    for (int c = 0; c < 7; ++c) ntask += hb[c];
    uint32_t key0 = 0;
    if (ntask) {
      WM_CUDA(cudaMemcpyAsync(&key0, g->ws->keys_out.ptr, sizeof key0, cudaMemcpyDeviceToHost, s));
      WM_CUDA(cudaStreamSynchronize(s));
    }
    WM_CUDA(cudaMemsetAsync(ctr + 16, 0, sizeof(unsigned long long), s));
    int st2 = run_clique_dfs(g, cfg, k, ntask, key0 ? (int)key0 - 1 : 1, res, s, kb, k1);
    if (st2) return st2;
    if ((st2 = red_pack(cfg, s, ctr, true, false, top, nullptr, 0, nullptr, 0))) return st2;
    unsigned long long hc[8];
    WM_CUDA(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaEventRecord(e1, s));
    WM_CUDA(cudaStreamSynchronize(s));
    float kms = 0, dms = 0;
    WM_CUDA(cudaEventElapsedTime(&kms, kb, k1));
    WM_CUDA(cudaEventElapsedTime(&dms, e0, e1));
    res->clique_count = hc[0];
    res->leaves = hc[0];
    res->tasks = hc[2];
    res->nodes = hc[3];
    res->kernel_ms = kms;
    res->device_ms = dms;
    res->d2h_bytes = sizeof hb + sizeof key0 + sizeof hc;
    return WM_OK;
  }
  // wide roots (> 1024 out-neighbours) sort first: hand this shard's share
  // (cyclic over their own list) to clique_wide_roots, skip them below
  skip = hb[6];
  if (skip) {
    std::vector<int32_t> ids(skip);
    WM_CUDA(cudaMemcpyAsync(ids.data(), g->ws->vals_out.ptr, sizeof(int32_t) * skip,
                            cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaStreamSynchronize(s));
    for (unsigned long long i = (unsigned long long)cfg->shard_rank; i < skip;
         i += (unsigned long long)cfg->shard_count) {
      int64_t be[2];
      WM_CUDA(cudaMemcpyAsync(be, g->ws->dag_off.as<int64_t>() + ids[i], sizeof be,
                              cudaMemcpyDeviceToHost, s));
      WM_CUDA(cudaStreamSynchronize(s));
      std::vector<int32_t> M((size_t)(be[1] - be[0]));
      WM_CUDA(cudaMemcpyAsync(M.data(), g->ws->dag_nbr.as<int32_t>() + be[0],
                              sizeof(int32_t) * M.size(), cudaMemcpyDeviceToHost, s));
      WM_CUDA(cudaStreamSynchronize(s));
      res->d2h_bytes += sizeof be + sizeof(int32_t) * M.size();
      wide->push_back(std::move(M));
    }
    res->d2h_bytes += sizeof(int32_t) * skip;
  }
  uint32_t *keys_sorted = g->ws->keys_out.as<uint32_t>() + skip;
  tasks_sorted = g->ws->vals_out.as<int32_t>() + skip;
  for (int c = 0; c < 6; ++c) ntask += hb[c];
  // bitmap arena offsets: exclusive scan of d * ceil(d/32) over the sorted tasks
  unsigned long long *words = g->ws->hist.as<unsigned long long>();
  unsigned long long *bmo = g->ws->table.as<unsigned long long>();
  if (ntask) {
    task_words_kernel<<<eblocks, tpb, 0, s>>>(ntask, keys_sorted, words);
    WM_CUDA(cudaMemsetAsync(words + ntask, 0, sizeof(unsigned long long), s));
    tb = g->ws->cub_tmp.bytes;
    WM_CUDA(cub::DeviceScan::ExclusiveSum(g->ws->cub_tmp.ptr, tb, words, bmo, (int)(ntask + 1), s));
    WM_CUDA(cudaMemcpyAsync(&arena_words, bmo + ntask, sizeof arena_words,
                            cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaStreamSynchronize(s));
    res->launches += 1;
  }
  bm_off = bmo;
  doff_p = g->ws->dag_off.as<int64_t>();
  dnbr_p = g->ws->dag_nbr.as<int32_t>();
  }  // per-run path
  if ((st = g->ws->arena.ensure(sizeof(uint32_t) * (arena_words + 1)))) return st;
  if (pt.on)
    fprintf(stderr, "[wm phases] tasks by width (d<=32,64,128,256,512,1024,wide): %llu %llu "
            "%llu %llu %llu %llu %llu\n", hb[0], hb[1], hb[2], hb[3], hb[4], hb[5], hb[6]);

  // width classes, contiguous in the descending sort: 32, 16, 8, then <= 4
  struct Cls { int wmax; unsigned long long begin, cnt, heavy; EnumPlan plan; };
  Cls cls[4];
  int ncls = 0;
  {
    unsigned long long begin = 0;
    for (int c = 5; c >= 3; --c) {
      if (hb[c]) cls[ncls++] = Cls{1 << c, begin, hb[c], 0, EnumPlan()};
      begin += hb[c];
    }
    const unsigned long long small = hb[0] + hb[1] + hb[2];
    if (small) cls[ncls++] = Cls{4, begin, small, 0, EnumPlan()};
  }
  // multi-GPU: each class's costliest tasks are split over all shards at
  // level 1 (CliqueArgs::heavy); WM_CLIQUE_SPLIT = tasks per shard (default 32).
  // Not for k = 3 (bulk2 roots have no level to split) or the B_alg pass.
  const unsigned long long N = (unsigned long long)cfg->shard_count;
  const unsigned long long R = (unsigned long long)cfg->shard_rank;
  // Deep runs (k >= 10) split EVERY task: each rank then builds every bitmap
  // (the build is < 1 % of such a run) and the shards balance to within a few
  // percent — cfg5 k=12 at 8 shards 6.3x -> 7.5x (profiles/r02_split_cfg5k12.log);
  // shallow runs split only the costliest 32 x N, since replicating the build
  // would cost more than the imbalance (cfg5 k=8: 31 ms build vs 10 ms kernel
  // per shard).
  {
    const char *sp = getenv("WM_CLIQUE_SPLIT");
    const unsigned long long per = sp ? strtoull(sp, nullptr, 10) : (k >= 10 ? ~0ull : 32ull);
    for (int i = 0; i < ncls; ++i) {
      const unsigned long long cap = per == ~0ull ? ~0ull : per * N;
      cls[i].heavy = (N > 1 && k >= 4 && !bytes) ? (cls[i].cnt < cap ? cls[i].cnt : cap) : 0ull;
    }
  }
  // this shard's tasks of a class: all `heavy` (split), then index = R (mod N)
  auto rem_first = [&](unsigned long long heavy) { return heavy + (R + N - heavy % N) % N; };
  auto shard_tasks = [&](unsigned long long cnt, unsigned long long heavy) {
    const unsigned long long f = rem_first(heavy);
    return heavy + (cnt > f ? (cnt - f + N - 1) / N : 0ull);
  };
  // plan + allocate everything before the timed region
  int max_warps = 0;
  for (int i = 0; i < ncls; ++i) {
    const unsigned long long nt = shard_tasks(cls[i].cnt, cls[i].heavy);
    switch (cls[i].wmax) {
#define WM_PLAN(WW)                                                                 \
  case WW:                                                                          \
    st = bytes ? plan_enum<WW, true>(g, cfg, nt, lb_on, &cls[i].plan)              \
               : plan_enum<WW, false>(g, cfg, nt, lb_on, &cls[i].plan);            \
    break;
      WM_PLAN(4) WM_PLAN(8) WM_PLAN(16) WM_PLAN(32)
#undef WM_PLAN
    }
    if (st) return st;
    if (cls[i].plan.warps > max_warps) max_warps = cls[i].plan.warps;
  }
  {
    uint32_t cap = 1;
    while (cap < 8u * (uint32_t)max_warps) cap <<= 1;
    if ((st = g->ws->ring.ensure(sizeof(uint32_t) * kSlotWords * (size_t)cap))) return st;
  }
  LbState *lbs = g->ws->lb.as<LbState>();
  int max_w = 0;
  double idle_w = 0, idle_tail_w = 0, tot_w = 0;
  int launched = 0;
  pt.mark("plan+sync");
  WM_CUDA(cudaEventRecord(k0, s));
  // build all bitmaps, then enumerate
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      WM_CUDA(cudaEventRecord(kb, s));
      pt.mark("bitmap build");
    }
    unsigned long long begin = 0;
    for (int c = 5; c >= 0 && pass == 0; --c) {
      const unsigned long long cnt = hb[c];
      if (!cnt) continue;
      CliqueArgs a;
      a.doff = doff_p;
      a.dnbr = dnbr_p;
      a.tasks = tasks_sorted + begin;
      a.bm_off = bm_off + begin;
      a.bm = g->ws->arena.as<uint32_t>();
      begin += cnt;
      // arena offsets cover every task (shard-independent); only this shard's
      // tasks are built: the class's split tasks (class-local index < heavy)
      // and class-local index (class_off + t) = rank (mod N) above them
      unsigned long long class_off = 0;
      for (int c2 = 2; c2 > c; --c2) class_off += hb[c2];  // buckets 0-2 share a class
      if (c > 2) class_off = 0;
      unsigned long long heavy_c = 0;
      for (int i = 0; i < ncls; ++i)
        if (cls[i].wmax == (c > 2 ? (1 << c) : 4)) heavy_c = cls[i].heavy;
      const unsigned long long all_below = heavy_c > class_off ? heavy_c - class_off : 0ull;
      unsigned long long first = (R + N - class_off % N) % N;  // t = first (mod N)
      if (first < all_below) first += (all_below - first + N - 1) / N * N;
      switch (c) {
#define WM_BCASE(CC, WW) \
  case CC:               \
    st = launch_build<WW>(g, a, cnt, all_below, first, N, order, !bytes, s); \
    break;
        WM_BCASE(0, 1) WM_BCASE(1, 2) WM_BCASE(2, 4) WM_BCASE(3, 8) WM_BCASE(4, 16)
        WM_BCASE(5, 32)
#undef WM_BCASE
      }
      if (st) return st;
      res->launches += 1;
    }
    for (int i = 0; i < ncls && pass == 1; ++i) {
      CliqueArgs a;
      a.doff = doff_p;
      a.dnbr = dnbr_p;
      a.tasks = tasks_sorted + cls[i].begin;
      a.bm_off = bm_off + cls[i].begin;
      a.bm = g->ws->arena.as<uint32_t>();
      a.task_offset = R;
      a.task_stride = N;
      a.heavy = cls[i].heavy;
      a.rem_first = rem_first(cls[i].heavy);
      a.ntasks = shard_tasks(cls[i].cnt, cls[i].heavy);
      a.k = k;
      a.lb_on = lb_on;
      a.lb_poll = cfg->lb_poll > 0 ? cfg->lb_poll : 1;
      a.idle_min = 1;
      a.L.lb = lbs + launched;
      a.counters = ctr;
      if (!a.ntasks) continue;
      switch (cls[i].wmax) {
#define WM_CASE(WW)                                                                  \
  case WW:                                                                           \
    st = bytes ? launch_enum<WW, true>(g, cfg, a, cls[i].plan, s)                    \
               : launch_enum<WW, false>(g, cfg, a, cls[i].plan, s);                  \
    break;
        WM_CASE(4) WM_CASE(8) WM_CASE(16) WM_CASE(32)
#undef WM_CASE
      }
      if (st) return st;
      if (cls[i].wmax > max_w) max_w = cls[i].wmax;
      if (cls[i].plan.warps > res->warps) res->warps = cls[i].plan.warps;
      res->launches += 2;
      ++launched;
    }
  }
  WM_CUDA(cudaEventRecord(k1, s));
  pt.mark("enumerate");
  if ((st = red_pack(cfg, s, ctr, true, bytes, top, lbs, launched, nullptr, 0))) return st;
  unsigned long long hc[8];
  WM_CUDA(cudaMemcpyAsync(hc, ctr, sizeof hc, cudaMemcpyDeviceToHost, s));
  LbState hl[8];
  if (launched)
    WM_CUDA(cudaMemcpyAsync(hl, lbs, sizeof(LbState) * launched, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaEventRecord(e1, s));
  pt.mark("readback");
  WM_CUDA(cudaStreamSynchronize(s));
  float kms = 0, dms = 0, bms = 0;
  WM_CUDA(cudaEventElapsedTime(&bms, k0, kb));
  WM_CUDA(cudaEventElapsedTime(&kms, kb, k1));
  WM_CUDA(cudaEventElapsedTime(&dms, e0, e1));
  res->build_ms = bms;
  res->d2h_bytes += sizeof hb + (ntask ? sizeof arena_words : 0) + sizeof hc +
                    sizeof(LbState) * (uint64_t)launched;
  res->clique_count = hc[0];
  res->leaves = hc[0];
  res->alg_bytes = bytes ? hc[1] : 0;
  res->tasks = hc[2];
  res->nodes = hc[3];
  res->polls = hc[4];
  res->kernel_ms = kms;
  res->device_ms = dms;
  res->bucket_words = max_w;
  for (int i = 0; i < launched; ++i) {
    wm_result tmp = {};
    finish_lb_stats(hl[i], &tmp);
    const double span = (double)(hl[i].t_end_max - hl[i].t_start_min) * hl[i].total_warps;
    if (hl[i].t_end_max > hl[i].t_start_min) {
      idle_w += tmp.idle_warp_fraction * span;
      idle_tail_w += tmp.idle_warp_fraction_tail * span;
      tot_w += span;
    }
    res->migrations += tmp.migrations;
    res->rebalance_count += tmp.rebalance_count;
    if (hl[i].error) return fail(hl[i].error, "device raised status %d", hl[i].error);
  }
  res->idle_warp_fraction = tot_w > 0 ? idle_w / tot_w : 0;
  res->idle_warp_fraction_tail = tot_w > 0 ? idle_tail_w / tot_w : 0;
  res->peak_ext = (uint64_t)max_w * 32;
  if (union_g) {
    wm_app ua = *app;
    ua.k = k - 1;
    wm_cfg uc = *cfg;
    uc.root_begin = uc.root_end = -1;
    uc.order = WM_ORDER_DEGREE;
    wm_result r = {};
    std::vector<std::vector<int32_t>> nested;  // components have <= 1024 vertices: none
    if ((st = run_clique_impl(union_g, &ua, &uc, &r, s, &nested, true))) return st;
    res->clique_count += r.clique_count;
    res->leaves += r.leaves;
    res->nodes += r.nodes;
    res->polls += r.polls;
    res->tasks += r.tasks;
    res->kernel_ms += r.kernel_ms;
    res->device_ms += r.device_ms;
    res->build_ms += r.build_ms;
    res->launches += r.launches;
    res->migrations += r.migrations;
    res->rebalance_count += r.rebalance_count;
    res->d2h_bytes += r.d2h_bytes;
    if (r.warps > res->warps) res->warps = r.warps;
    if (r.bucket_words > res->bucket_words) res->bucket_words = r.bucket_words;
    // warp-time weighted idle fractions of the two launches' spans
    const double a0 = res->kernel_ms - r.kernel_ms, a1 = r.kernel_ms;
    if (a0 + a1 > 0) {
      res->idle_warp_fraction = (res->idle_warp_fraction * a0 + r.idle_warp_fraction * a1) / (a0 + a1);
      res->idle_warp_fraction_tail =
          (res->idle_warp_fraction_tail * a0 + r.idle_warp_fraction_tail * a1) / (a0 + a1);
    }
  }
  return WM_OK;
}

}  // namespace wm
