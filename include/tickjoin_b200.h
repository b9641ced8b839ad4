/*
 * tickjoin_b200.h — C ABI of the B200-native QUAD tick pipeline.
 *
 * Drop-in boundary for the reference's QUAD path (arXiv 1411.3212,
 * `tickjoin` package).  The reference has no FFI: its boundary is the Python
 * tick API `Engine(MethodConfig(method="quad")).process_tick(batch)`
 * (tickjoin/engine.py:137-259).  Each entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only; no torch types.
 *
 * Status codes: 0 = OK, negative = error.  The error codes map 1:1 onto the
 * reference exception classes (tickjoin/errors.py:4-45) plus device errors.
 * A context is single-threaded (like `Engine`); distinct
 * contexts may run concurrently on distinct devices.
 */
#ifndef TICKJOIN_B200_H
#define TICKJOIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TJ_ABI_VERSION 4

/* status codes — errors.py:4-45 */
#define TJ_OK 0
#define TJ_E_EMPTY_BATCH (-1)      /* EmptyBatch        errors.py:7   */
#define TJ_E_OUT_OF_BOUNDS (-2)    /* OutOfBounds       errors.py:11  */
#define TJ_E_TILING_GAP (-5)       /* TilingGap         errors.py:23  */
#define TJ_E_COUNT_MISMATCH (-6)   /* CountMismatch     errors.py:27  */
#define TJ_E_DUPLICATE_RESULT (-7) /* DuplicateResult   errors.py:31  */
#define TJ_E_BAD_CONFIG (-8)       /* BadConfig         errors.py:35  */
#define TJ_E_INVALID_ARG (-20)     /* ValueError (bad rect, null ptr)  */
#define TJ_E_CUDA (-100)
#define TJ_E_NCCL (-101)
#define TJ_E_OOM (-102)
#define TJ_E_NO_DEVICE (-103)

/* memory spaces of caller buffers */
#define TJ_MEM_HOST 0   /* pageable or pinned host memory                  */
#define TJ_MEM_DEVICE 1 /* device memory on the context's CUDA device      */
/* tj_tick_in.out_mem flag: compact 32-bit delivery.  Result ids come as int32
 * (tj_tick_out.ids32, id_bytes = 4) when every result id of the tick fits in
 * int32, else as int64 (id_bytes = 8); CSR offsets come as int32
 * (offsets32, offset_bytes = 4) when the tick has fewer than 2^31 results,
 * else as int64.  Halves the bytes a host caller downloads per tick; the
 * values are the same. */
#define TJ_OUT_IDS32 0x100

/* rebuild policies — MethodConfig.rebuild, engine.py:70,163-170 */
#define TJ_REBUILD_EVERY_TICK 0
#define TJ_REBUILD_ADAPTIVE 1

typedef struct tj_ctx tj_ctx;

/* MethodConfig fields read by the QUAD and UG paths (engine.py:57-96). */
typedef struct tj_config {
  int32_t th_quad;               /* occupancy threshold, >= 1 (default 384)  */
  int32_t l_max;                 /* deepest level, 1..12 (default 12)        */
  int32_t covering_optimization; /* 1: covering subqueries skip bitmaps      */
  int32_t rebuild;               /* TJ_REBUILD_*                             */
  int32_t device;                /* CUDA device ordinal                      */
  int32_t split_factor;          /* 0: QUAD (quadtree index).  1..4096: the
                                    uniform-grid method "ug" with this many
                                    columns and rows (grid.py:35-40); th_quad,
                                    l_max and rebuild are then unused         */
} tj_config;

/* One tick of input as structure-of-arrays (TickBatch, geometry.py:58-64,
 * converted AoS->SoA as in geometry.py:91-110).  Pointers live in `mem`. */
typedef struct tj_tick_in {
  int64_t n_obj;
  const int64_t* obj_id;
  const double* obj_x;
  const double* obj_y;
  int64_t n_q;
  const int64_t* q_issuer;
  const double* q_xa;
  const double* q_ya;
  const double* q_xb;
  const double* q_yb;
  int32_t mem;     /* TJ_MEM_HOST / TJ_MEM_DEVICE for the inputs        */
  int32_t out_mem; /* where tj_tick_out buffers should be delivered,
                      optionally | TJ_OUT_IDS32                          */
} tj_tick_in;

/* Per-query results as CSR in input-query order; ids ascending per query
 * (ResultSet.by_query, decode.py:23-37).  Library-owned; valid until the
 * next tj_tick or tj_destroy on the same context. */
typedef struct tj_tick_out {
  int64_t n_q;
  int64_t n_results;
  const int64_t* offsets; /* n_q + 1 (offset_bytes == 8; else NULL) */
  const int64_t* ids;     /* n_results (id_bytes == 8; else NULL) */
  int32_t mem;
  int32_t id_bytes;       /* 8: ids holds the results; 4: ids32 does  */
  const int32_t* ids32;   /* n_results (id_bytes == 4; else NULL) */
  const int32_t* offsets32; /* n_q + 1 (offset_bytes == 4; else NULL) */
  int32_t offset_bytes;   /* 8: offsets holds the CSR offsets; 4: offsets32 does */
  int32_t reserved;
} tj_tick_out;

/* TickStats counters (engine.py:99-121) plus device stage times. */
typedef struct tj_stats {
  int64_t n_objects, n_queries;
  int64_t containment_tests;   /* engine.py:225 */
  int64_t decoded_bits;        /* engine.py:279 */
  int64_t subq_intersecting;   /* engine.py:213 */
  int64_t subq_covering;       /* engine.py:214 */
  int64_t covering_results;    /* engine.py:245 */
  int64_t active_cells;        /* engine.py:263 */
  int64_t results_total;       /* engine.py:248 */
  int64_t occ_sum, occ_sumsq;  /* occupancy moments over non-empty leaves */
  int64_t n_leaves, l_deep, n_tasks, bitmap_words, n_subqueries, work_units;
  int32_t rebuilt;             /* 1 if the index was (re)built this tick */
  int32_t retries;             /* capacity-growth replays of this tick    */
  double t_index_ms, t_filter_ms, t_decode_ms, t_merge_ms, t_total_ms; /* CUDA events */
  double mbr[4];
  double t_join_ms;            /* the per-leaf join kernel alone (CUDA events) */
  int64_t task_objects;        /* P_a: objects in leaves that are join tasks   */
  int64_t task_subqueries;     /* S_a: intersecting subqueries in join tasks   */
  int64_t kernel_launches;     /* kernels this call launched (all attempts)    */
  double t_build_ms;           /* index build alone (K0 + K1: MBR .. leaf directory of objects) */
  double t_scatter_ms;         /* query -> leaf scatter + subquery directory (K2) */
  double t_sort_ms;            /* objects into leaf order (K1's last part, concurrent with K2) */
  int32_t id_order;            /* how result lists were put in id order (decode.py:117):
                                  TJ_IDS_MONOTONE, TJ_IDS_KEYED or TJ_IDS_SORTED */
  int32_t reserved2;
  double t_decode_kernel_ms;   /* the per-query decode kernel alone (K4 without the offsets scan) */
} tj_stats;

/* tj_stats.id_order */
enum {
  TJ_IDS_MONOTONE = 0, /* ids increase with the input row: runs merge by row                    */
  TJ_IDS_KEYED = 1,    /* ids are not the rows: objects ranked by id (counting sort over a
                          presence bitmap), leaf blocks in id order with 32-bit id offsets,
                          runs merge by offset                                                */
  TJ_IDS_SORTED = 2    /* each multi-result list sorted by id: the first such tick of a
                          context, duplicate ids, or an id range of 2^28 or more             */
};

/* Reference-order index view (QuadIndex, quadtree.py:41-67). */
typedef struct tj_index_info {
  double mbr[4];
  int32_t th_quad, l_max, l_deep, reserved;
  int64_t n_leaves; /* len(leaves) */
  int64_t n_cells;  /* len(zmap) = 4**l_deep */
} tj_index_info;

/* ---- lifecycle -------------------------------------------------------- */
int tj_abi_version(void);
int tj_device_count(int* count);
/* Engine.__init__ + MethodConfig.validate (engine.py:73-88,140-145). */
int tj_create(const tj_config* cfg, tj_ctx** out);
int tj_destroy(tj_ctx* ctx);
/* Last error message of a context (or of the last failed tj_create if ctx is NULL). */
const char* tj_last_error(const tj_ctx* ctx);

/* ---- the hot path ------------------------------------------------------ */
/* Engine.process_tick for method "quad" (engine.py:178-259): index build,
 * query->leaf scatter, per-leaf bitmap join, decode, canonical merge. */
int tj_tick(tj_ctx* ctx, const tj_tick_in* in, tj_tick_out* out, tj_stats* stats);

/* ---- introspection (parity tests; host copies, reference order) ------- */
/* build_quadtree result: leaves ascending packed (level << 2*l_max | z),
 * zmap packed ids per deepest cell (quadtree.py:74-158).  Null buffers: info only. */
int tj_get_index(tj_ctx* ctx, tj_index_info* info, int64_t* leaves, int64_t leaves_cap,
                 int64_t* zmap, int64_t zmap_cap);
/* map_objects_quad (quadtree.py:161-165): packed leaf per input object. */
int tj_get_object_cells(tj_ctx* ctx, int64_t* cells, int64_t cap);
/* split_queries_quad output (quadtree.py:168-240), per query in ascending
 * packed-leaf order: input query row, packed leaf, covering flag. */
int tj_get_subqueries(tj_ctx* ctx, int64_t* count, int64_t* q_row, int64_t* cell,
                      uint8_t* covering, int64_t cap);
/* sort_by_cell (directory.py:119-158): objects' input rows in directory order;
 * indices into the subquery list for the intersecting / covering blocks. */
int tj_get_directory(tj_ctx* ctx, int64_t* obj_rows, int64_t obj_cap, int64_t* isq, int64_t* n_isq,
                     int64_t* cov, int64_t* n_cov, int64_t sq_cap);
/* Per-task linear bitmaps + popcounts (bitmap.py:70-119) for tasks in
 * ascending packed cell order; task_woff has n_tasks + 1 entries. */
int tj_get_bitmaps(tj_ctx* ctx, int64_t* n_tasks, int64_t* n_words, int64_t* task_cell,
                   int64_t* task_nobj, int64_t* task_nisq, int64_t* task_woff, uint32_t* words,
                   int64_t* counts, int64_t task_cap, int64_t word_cap, int64_t count_cap);
/* simulate_assignment over heaviest-first tasks (scheduler.py:31-54):
 * greedy least-loaded assignment of task weights n_isq*n_obj. */
int tj_get_imbalance(tj_ctx* ctx, int32_t sim_processors, int32_t heaviest_first, double* imbalance);
/* Object counts of the non-empty leaves in ascending packed cell order: the
 * array the reference's _occupancy_stats reduces (engine.py:261-267), so the
 * host computes occupancy mean / var / dispersion exactly as NumPy does.
 * counts == NULL: only *n_active is returned. */
int tj_get_occupancy(tj_ctx* ctx, int64_t* counts, int64_t cap, int64_t* n_active);

/* Method "ug_baseline" (baseline.py:26-121): the reference's direct-emission
 * filter stages each task cell's (query, object) pairs privately and flushes
 * full stages to a locked shared buffer.  The B200 path produces the same
 * results through the bitmap pipeline; this returns the contention counter the
 * reference reports for the last tick (flushes = sync_ops): the sum over task
 * cells of ceil(intersecting pairs / staging_capacity), counted on the device. */
int tj_get_staging_flushes(tj_ctx* ctx, int32_t staging_capacity, int64_t* flushes);

/* Multi-GPU leaf-range sharding (no reference counterpart —
 * the reference is single-process).  With nranks > 1 every
 * tick builds the full index, then scatters, joins and decodes only the
 * (query, leaf) pairs of this rank's contiguous Morton range of leaves
 * (balanced by object count); the output CSR holds each query's results
 * restricted to those leaves.  Partial lists of the ranks are disjoint and individually sorted;
 * their per-query merge is the full result.  nranks == 1 (default): off. */
int tj_set_shard(tj_ctx* ctx, int32_t rank, int32_t nranks);

/* ---- multi-GPU data plane (one process or thread per GPU) ---------------
 * tj_tick_sharded takes this rank's slice of the tick's objects and queries
 * (any sizes per rank) and returns the complete result lists of this rank's
 * queries: the slices are gathered into the full tick on every rank, the
 * tick runs on the rank's contiguous Morton range of leaves (tj_set_shard),
 * each query's partial lists go to its home rank (all-to-all), and the home
 * rank merges them on the device.  Concatenating the ranks' outputs in rank
 * order gives tj_tick's output for the concatenated slices.  Transports:
 * NCCL (the caller shares one tj_nccl_unique_id among the ranks, e.g. over
 * its own bootstrap; libnccl.so.2 is loaded at run time) or an in-process
 * group of contexts driven from one thread each. */
typedef struct tj_group tj_group;
int tj_nccl_unique_id(void* id, int32_t bytes); /* bytes >= 128 (ncclUniqueId) */
int tj_comm_init(tj_ctx* ctx, const void* nccl_unique_id, int32_t rank, int32_t nranks);
int tj_group_create(int32_t nranks, tj_group** out);
int tj_group_destroy(tj_group* group);
int tj_comm_init_local(tj_ctx* ctx, tj_group* group, int32_t rank);
int tj_tick_sharded(tj_ctx* ctx, const tj_tick_in* in, tj_tick_out* out, tj_stats* stats);

/* The context's CUDA stream (cudaStream_t), for callers that time or order
 * work against the tick with their own events. */
int tj_get_stream(tj_ctx* ctx, void** stream);

/* ---- pinned host buffers for end-to-end callers ------------------------ */
int tj_host_alloc(int64_t bytes, void** ptr);
int tj_host_free(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* TICKJOIN_B200_H */
