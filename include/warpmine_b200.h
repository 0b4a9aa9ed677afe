/*
 * warpmine_b200.h — C-ABI of libwm_b200.so, the B200-native replacement for
 * the body of the reference's engine entry point
 *
 *     warpmine.engine.run(g: CsrGraph, app: Application, *, mode="wc",
 *                         warps=4, lane_width=32, balance_config=None)
 *         -> RunResult                 (pkg/src/warpmine/engine.py:781-843)
 *
 * Plain pointers and sizes only.  Host pointers are borrowed for the duration
 * of the call; device memory is owned by the library.  Calls are blocking;
 * the library's per-device scratch is held for the whole of each call, so
 * concurrent calls on one device are serialised (a call from inside a listing
 * sink callback is refused with WM_EINVAL).  Status codes map onto the reference's
 * exception taxonomy (pkg/src/warpmine/errors.py:4-31) in
 * paper_2212_04551_b200/_native.py:
 *
 *   WM_EINVAL      -> ValueError              (engine.py:791-798, :72-80;
 *                                              apps.py:38-40, :52-54)
 *   WM_ECAPACITY   -> CapacityError           (engine.py:319-323)
 *   WM_EINVARIANT  -> InternalInvariantError  (engine.py:258-261, :472-473;
 *                                              aggregate.py:190-193)
 *   WM_ESHUTDOWN   -> StoreShutdownError      (aggregate.py:88-99: the store
 *                                              consumer is gone)
 *   WM_EPARSE      -> GraphParseError         (graph.py:139-188, errors.py:4-11)
 *   WM_ECUDA       -> DeviceError (RuntimeError); no reference counterpart.
 */
#ifndef WARPMINE_B200_H
#define WARPMINE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WM_ABI_VERSION 2

#define WM_OK 0
#define WM_EINVAL (-1)
#define WM_ECAPACITY (-2)
#define WM_EINVARIANT (-3)
#define WM_ECUDA (-4)
#define WM_ESHUTDOWN (-5)
#define WM_EPARSE (-6)

/* Pipeline filter tags (engine.py:227-237); order-insensitive bit set. */
#define WM_F_LOWER 1u
#define WM_F_COMPACT 2u
#define WM_F_CLIQUE 4u
#define WM_F_CANONICAL 8u

#define WM_AGG_COUNTER 0 /* aggregate_counter, aggregate.py:169-171 */
#define WM_AGG_PATTERN 1 /* aggregate_pattern, aggregate.py:174-196 */
#define WM_AGG_STORE 2   /* aggregate_store, aggregate.py:199-223 (wm_run_listing) */

#define WM_MODE_WC 1  /* warp-centric, load balancing off  (engine.py:18-19) */
#define WM_MODE_OPT 2 /* warp-centric + on-device balancer (engine.py:20-21) */
#define WM_MODE_DFS 3 /* thread-per-traversal DFS ablation, DM_DFS (engine.py:13-16) */

#define WM_ORDER_ID 0     /* clique orientation by vertex id (reference order) */
#define WM_ORDER_DEGREE 1 /* clique orientation by (degree, id) */

/* CsrGraph (graph.py:28-78): rows ascending, symmetric, no self-loops. */
typedef struct {
  int64_t n;                /* vertices */
  int64_t nnz;              /* 2 * undirected edges */
  const int64_t *offsets;   /* [n + 1] host */
  const int32_t *neighbors; /* [nnz] host */
} wm_csr;

/* Application (engine.py:53-80) as built by clique_app / motif_app
 * (apps.py:43-58). */
typedef struct {
  int k;
  int extend_all;           /* extend(0, len) vs extend(0, 1) */
  int genedges;             /* maintain induced-edge bitmaps */
  int aggregator;           /* WM_AGG_* */
  uint32_t filters;         /* WM_F_* */
  const uint32_t *dict_table; /* host, [dict_len]; pattern aggregator only */
  uint64_t dict_len;
  uint32_t pattern_count;
  const void *dict_device;  /* optional device-resident copy of the table (then
                               dict_table may be NULL): u16 entries with
                               SENTINEL 0xFFFF (pattern_count < 65535) or u32 */
  uint32_t dict_device_bits; /* 16 or 32 */
} wm_app;

/* Run configuration: mode / balance_config (balance.py:36-60) plus the
 * B200-only knobs (root range, sharding, orientation, instrumentation). */
typedef struct {
  int mode;                 /* WM_MODE_WC | WM_MODE_OPT | WM_MODE_DFS */
  double lb_threshold;      /* donate when active/total warps < threshold
                               (balance.py:63-66); (0, 1] */
  int lb_poll;              /* DFS steps between idle-warp polls (>= 1) */
  int64_t root_begin;       /* root range [root_begin, root_end) over vertex */
  int64_t root_end;         /*   ids; -1,-1 = all (engine.py:187)           */
  int shard_rank;           /* cyclic shard of the cost-sorted root tasks */
  int shard_count;          /*   (multi-GPU, one process per GPU); 1 = all */
  int order;                /* WM_ORDER_* (clique only) */
  int count_bytes;          /* 1: instrumented pass computing B_alg (SURVEY
                               8(d)); cliques run it with LB off, motifs
                               with the balancer as configured */
  int warps_per_block;      /* 0 = auto */
  int blocks_per_sm;        /* 0 = auto (occupancy) */
  void *stream;             /* cudaStream_t to run on; NULL = library stream */
  uint64_t *reduce_out;     /* optional DEVICE buffer of wm_reduce_words() u64:
                               the run's result vector, written on `stream`
                               (layout below) so one collective on that stream
                               sums every rank's results (aggregate.py:39-55)
                               with no host round trip.  NULL = not written. */
} wm_cfg;

/* Device result vector (wm_cfg.reduce_out), u64 words:
 *   [WM_RED_CLIQUES] clique_count   [WM_RED_LEAVES] leaves (aggregated_total)
 *   [WM_RED_ALG_BYTES] B_alg        [WM_RED_MIGRATIONS] migrations
 *   [WM_RED_DONATIONS] rebalance_count  [WM_RED_TASKS] root tasks
 *   [WM_RED_RECORDS] [WM_RED_CHECKSUM] listing (0 for wm_run)
 *   [WM_RED_HIST .. +pattern_count) pattern histogram
 *   then shard_count slots of WM_RED_SLOT_WORDS: slot shard_rank holds this
 *   rank's kernel_ms, device_ms, idle_warp_fraction, idle_warp_fraction_tail
 *   as IEEE-754 double bit patterns; other slots are 0.
 * Every word is a sum over ranks: counters add (mod 2^64), and each timing
 * slot has exactly one non-zero contributor, so ncclAllReduce(ncclUint64,
 * ncclSum) over the whole vector leaves every rank's timings intact for a
 * max on the host. */
#define WM_RED_CLIQUES 0
#define WM_RED_LEAVES 1
#define WM_RED_ALG_BYTES 2
#define WM_RED_MIGRATIONS 3
#define WM_RED_DONATIONS 4
#define WM_RED_TASKS 5
#define WM_RED_RECORDS 6
#define WM_RED_CHECKSUM 7
#define WM_RED_HIST 8
#define WM_RED_SLOT_WORDS 4

/* words of the reduce_out vector for `pattern_count` patterns (0 for the
 * counter aggregator) and `shard_count` ranks */
uint64_t wm_reduce_words(uint32_t pattern_count, int shard_count);

/* RunResult (engine.py:747-762) plus device evidence. */
typedef struct {
  uint64_t clique_count;        /* counter aggregator */
  uint64_t leaves;              /* aggregated_total (engine.py:581, :604) */
  uint64_t alg_bytes;           /* B_alg when count_bytes, else 0 */
  uint64_t rebalance_count;     /* donation rounds (idle-triggered polls) */
  uint64_t migrations;          /* prefixes moved between warps */
  uint64_t peak_ext;            /* peak extension entries held by one warp */
  uint64_t *pattern_counts;     /* caller-allocated [pattern_count] or NULL */
  uint64_t tasks;               /* root tasks processed by this shard */
  uint64_t launches;            /* kernels launched by this call */
  uint64_t nodes;               /* internal search-tree nodes expanded */
  uint64_t polls;               /* idle-counter polls by busy warps (opt) */
  uint64_t h2d_bytes;           /* host->device bytes copied by this call */
  uint64_t d2h_bytes;           /* device->host bytes copied by this call */
  double kernel_ms;             /* enumeration kernel(s), CUDA events */
  double build_ms;              /* per-root bitmap build kernels (clique) */
  double device_ms;             /* whole call on the device incl. preprocessing */
  double idle_warp_fraction;    /* idle warp-time / (warps * kernel time) */
  double idle_warp_fraction_tail; /* same, from the first root-queue drain */
  int warps;                    /* resident warps of the enumeration kernel */
  int bucket_words;             /* clique bitmap words per row (max bucket) */
} wm_result;

/* ---- subgraph listing (listing_app / subgraph_listing, apps.py:61-67,
 * :94-118; aggregate_store, aggregate.py:199-223) ------------------------
 *
 * Every completed k-subgraph is streamed to the host as one record through a
 * bounded ring in mapped pinned memory: producers (device warps) block while
 * the ring is full, exactly the StoreBuffer back-pressure of
 * aggregate.py:69-147.  The calling thread drains the ring and hands batches
 * of records to `sink`; a non-zero return from `sink` is the dead consumer of
 * aggregate.py:88-99: producers stop and wm_run_listing returns WM_ESHUTDOWN.
 *
 * Record layout (u32 words, `stride` words per record):
 *   [0] sequence (internal)      [1] e, the k-th vertex
 *   [2] mask: bit j set iff tr[j] is adjacent to e (adjacency_mask, :160-166)
 *   [3] prefix bitmap low word   [4] prefix bitmap high word  (bitmap of tr[0..k-1))
 *   [5 .. 5+k-1) tr[0..k-1)      (traversal order)
 * The reference record is (tr[0..k-1) + (e,), bits) with
 *   bits = prefix | mask << ((k-1)(k-2)/2 - 1)          (extend_bits, canon.py:76-90)
 * which needs up to 65 bits at k = 12, so it is left to the consumer.
 *
 * Record checksum (order-independent, for parity at scale): with
 *   smix(x) = splitmix64 finaliser of x + 0x9E3779B97F4A7C15,
 *   h = 0; for v in vertices: h = smix(h ^ v);
 *   h = smix(h ^ (bits mod 2^64)); h = smix(h ^ (bits >> 64)),
 * checksum = sum of h over all emitted records mod 2^64. */
#define WM_LIST_ALL 0      /* emit every connected induced k-subgraph */
#define WM_LIST_COMPLETE 1 /* device-side complete_subgraph predicate (apps.py:121-123) */

typedef int (*wm_sink_fn)(void *user, const uint32_t *records, uint64_t count,
                          uint32_t stride_words);

typedef struct {
  uint32_t capacity;        /* ring records (rounded up to a power of two) */
  uint32_t filter;          /* WM_LIST_* */
  wm_sink_fn sink;          /* NULL: records are only counted and checksummed */
  void *user;
  uint64_t emitted;         /* out: records handed to the consumer */
  uint64_t checksum;        /* out: record checksum (above) */
  uint32_t stride_words;    /* out: record stride */
  uint32_t reserved;
} wm_listing;

/* engine.run with the store aggregator (listing_app pipeline: extend(0,len),
 * canonical, store).  Blocks until every record has been consumed. */
int wm_run_listing(void *graph, const wm_app *app, const wm_cfg *cfg, wm_listing *listing,
                   wm_result *result);

/* ---- graph ingest on the device (the step before the path) ------------
 * CsrGraph construction (graph.py:44-78) and the edge-list reader
 * (graph.py:139-188) as data-parallel sort/unique/scan passes.  Outputs are
 * malloc'd host arrays owned by the caller (release with wm_csr_free). */
typedef struct {
  int64_t n;                /* vertices */
  int64_t nnz;              /* 2 * undirected edges */
  int64_t *offsets;         /* [n + 1] */
  int32_t *neighbors;       /* [nnz], rows strictly ascending */
  int64_t error_line;       /* WM_EPARSE: 1-based offending line (0: whole input) */
  double device_ms;
} wm_csr_out;

/* CsrGraph.from_arrays: endpoint arrays (any direction / multiplicity) on
 * 0..n-1 -> symmetric CSR without self-loops or duplicates. */
int wm_csr_build(int64_t n, const int64_t *src, const int64_t *dst, int64_t m,
                 wm_csr_out *out);

/* load_edge_list: whitespace edge-list text -> CSR with ids remapped to
 * 0..n-1 in ascending order.  WM_EPARSE + out->error_line on the first
 * malformed line (two integer tokens, non-negative). */
int wm_edge_list_parse(const char *text, uint64_t len, wm_csr_out *out);

void wm_csr_free(wm_csr_out *out);

/* ---- pattern dictionary on the device --------------------------------
 * build_dictionary (canon.py:315-343): table[b] = pattern id of every
 * reachable k-vertex bitmap b (SENTINEL 0xFFFFFFFF otherwise), ids ascending
 * with the canonical (minimum) bitmap, byte-identical to the reference.
 * table_out holds 2^(k(k-1)/2-1) entries (2^27 at k = 8); bitmaps_out
 * receives the canonical bitmaps (bitmaps_cap entries at most). */
int wm_dictionary_build(int k, uint32_t *table_out, uint64_t *bitmaps_out, uint32_t bitmaps_cap,
                        uint32_t *pattern_count);

/* Upload a CSR graph to the current device (cudaSetDevice beforehand).
 * The CsrGraph contract (graph.py:122-133) is checked on the device after the
 * upload: offsets span nnz and never decrease, every neighbour id is in
 * [0, n), rows are strictly ascending, there are no self-loops and every edge
 * is symmetric.  A violation returns WM_EINVAL naming the first offending
 * vertex/edge, in the reference's wording. */
int wm_graph_create(const wm_csr *csr, void **graph);

/* Same, from device-resident arrays (copied device-to-device; same checks). */
int wm_graph_create_device(int64_t n, int64_t nnz, const int64_t *d_offsets,
                           const int32_t *d_neighbors, void **graph);

/* engine.run: enumerate every canonical size-k traversal rooted in the
 * configured root set.  Fills *result; pattern_counts must hold
 * app->pattern_count entries for the pattern aggregator. */
int wm_run(void *graph, const wm_app *app, const wm_cfg *cfg, wm_result *result);

void wm_graph_destroy(void *graph);

/* Message of the last failing call on this thread ("" if none). */
const char *wm_last_error(void);

int wm_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* WARPMINE_B200_H */
