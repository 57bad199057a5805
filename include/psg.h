/*
 * psg — perfslice-gpu: the thin C ABI between the perfslice host layer and the
 * hand-written sm_100a kernels of the trace query path (SURVEY.md §8(b) "New
 * thin C ABI into CUDA").  Plain C types only; no exceptions cross it.
 *
 * Status codes are the reference's ps_status values (perfslice.h:24-40,
 * reproduced in perfslice_gpu.h) so callers map errors exactly as they do for
 * the reference C API; CUDA / NCCL failures map to PS_E_INTERNAL with the CUDA
 * error string in psg_last_error() (thread-local, like capi.cpp:33).
 *
 * Ownership (SURVEY.md §8(b) "Ownership"): every device buffer belongs to the
 * psg_context; results stay resident in HBM until the next query of the same
 * kind and are copied out through the psg_get_* calls into caller-allocated
 * host arrays (sizes are reported by the query call first — the two-call
 * pattern).  A context is single-threaded (serialise like a ps_session) and
 * issues all work on one CUDA stream; every call returns after its outputs
 * are complete on that stream unless documented otherwise.
 *
 * Multi-GPU: one process per GPU.  Each rank opens a context on its device,
 * loads (or generates) its own shard of traces, and joins a communicator with
 * psg_comm_init(); queries then all-reduce only the per-shard summaries
 * (iteration counts, per-(iteration,node) cross-rank sums, per-node outlier
 * sums) over NCCL.  Trace events never cross GPUs.
 */
#ifndef PSG_H
#define PSG_H

#include <stddef.h>
#include <stdint.h>

#include "perfslice_gpu.h" /* ps_status */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psg_context psg_context;

/* ---- context ------------------------------------------------------------ */
const char* psg_version(void);
const char* psg_last_error(void);
/* stream: a cudaStream_t to issue on, or NULL for a context-owned stream. */
ps_status psg_open(int device, void* stream, psg_context** out);
void psg_close(psg_context* ctx);
/* The cudaStream_t every kernel of this context is launched on. */
void* psg_stream(psg_context* ctx);
/* Device bytes currently held by the context (traces + results). */
uint64_t psg_device_bytes(const psg_context* ctx);

/* ---- multi-GPU (NCCL over NVLink; loaded at runtime) ------ */
ps_status psg_comm_unique_id(uint8_t out_id[128]);
ps_status psg_comm_init(psg_context* ctx, int nranks, int rank, const uint8_t id[128]);
/* Host-side summary exchange instead of NCCL (an MPI or torch.distributed
 * process group, or several ranks sharing one GPU): the library calls
 * fn(buf, count, dtype, op, user) with a HOST buffer of `count` elements
 * (dtype 0 = uint64, 1 = float64; op 0 = sum, 1 = max, 2 = min), expects the
 * element-wise reduction over all ranks in place, and treats a nonzero return
 * as an error.  Every rank must issue the same queries in the same order. */
typedef int (*psg_allreduce_fn)(void* buf, uint64_t count, int dtype, int op, void* user);
ps_status psg_comm_init_host(psg_context* ctx, int nranks, int rank, psg_allreduce_fn fn,
                             void* user);

/* ---- calling-context tree (meta.bin contexts, store.hpp:70-75) ----------- */
/* parent[0] must be 0xFFFFFFFF; parent[c] < c for c > 0 (topological ids). */
ps_status psg_set_cct(psg_context* ctx, const uint32_t* parent, uint32_t n_ctx);

/* ---- trace loading ------------------------------------------------------ */
/* Replaces db_handle::read_trace_full's per-event decode (store.cpp:573-580,
 * 678-692): `body` holds the packed 12-byte little-endian trace.db events
 * {u64 ts, u32 ctx} of n_traces traces back to back (host memory, pinned or
 * pageable), event_off[n_traces+1] their event offsets, profile_ids and
 * t_end_ns the trace.db index fields.  Copies to HBM, transposes to SoA and
 * validates (non-decreasing ts, ctx < n_ctx, t_end >= last ts); an invalid
 * body fails with PS_E_FORMAT like validate_database (store.cpp:713-764). */
ps_status psg_load_traces_aos(psg_context* ctx, const void* body, uint64_t n_events,
                              const uint64_t* event_off, const uint32_t* profile_ids,
                              const uint64_t* t_end_ns, uint32_t n_traces);

/* Starts the host->device copy of the first staging chunks (up to 1.5 GB) of
 * the NEXT psg_load_traces_aos call's body while the device works on the
 * current traces (PCIe is otherwise idle during a query): call it after
 * loading, before querying.  Only pinned bodies are prefetched (pageable ones:
 * a no-op).  The bytes are read at prefetch time; a later
 * psg_load_traces_aos with the same body pointer and n_events uses them, any
 * other staging user drops them.  No reference counterpart: a pipelining
 * hint under the drop-in of store.cpp:678-692 / ingest.cpp:178-208. */
ps_status psg_prefetch_aos(psg_context* ctx, const void* body, uint64_t n_events);
/* The mmap reader path: opens <dir>/meta.bin + trace.db (format store.hpp:5-23)
 * and loads the traces whose profile id is listed (NULL = every trace),
 * setting the CCT and the rank->host mapping from meta.bin as well. */
ps_status psg_load_trace_db(psg_context* ctx, const char* dir, const uint32_t* pids,
                            uint32_t n_pids);

/* Device synthetic generator: byte-identical to the reference
 * synthgen::generate_iterative_scenario (synthgen.cpp:146-246) for ranks
 * [rank_lo, rank_hi) of an n_ranks scenario (the xorshift64* stream of
 * util.hpp:18-42 is jumped ahead on the GPU).  spread is
 * [n_kernels][n_ranks] (spread_rank_stride = n_ranks) or one shared
 * [n_ranks] ladder (spread_rank_stride = 0 → index by rank only); NULL means
 * factor 1.0.  Also installs the scenario's CCT. */
typedef struct psg_iter_scenario {
  uint32_t n_ranks;
  uint32_t n_iterations;
  uint32_t n_kernels;
  const double* mean_time_s;   /* [n_kernels] */
  const double* jitter_frac;   /* [n_kernels] */
  const double* spread;        /* see above, may be NULL */
  uint64_t spread_kernel_stride; /* 0: the same ladder for every kernel */
  double copy_segment_s;
  uint64_t seed;
} psg_iter_scenario;
ps_status psg_generate_iterative(psg_context* ctx, const psg_iter_scenario* s,
                                 uint32_t rank_lo, uint32_t rank_hi);

/* Rank -> node (hostname) mapping for node_correlate / topology: node_of_trace
 * is indexed by loaded-trace position; rack/chassis per node are the parsed
 * x<rack>c<chassis>... coordinates (topology.cpp:33-46). */
ps_status psg_set_nodes(psg_context* ctx, const uint32_t* node_of_trace, uint32_t n_nodes,
                        const uint32_t* node_rack, const uint32_t* node_chassis);

/* Loaded shard shape. */
typedef struct psg_shard_info {
  uint32_t n_traces;
  uint32_t n_ctx;
  uint64_t n_events;
  uint64_t t_min;      /* min first timestamp */
  uint64_t t_max;      /* max t_end */
} psg_shard_info;
ps_status psg_shard(psg_context* ctx, psg_shard_info* out);
/* Copies the loaded SoA back (tests): ts[n_events], ctx[n_events], event_off[n+1],
 * t_end[n], profile_ids[n]; any pointer may be NULL. */
ps_status psg_get_traces(psg_context* ctx, uint64_t* ts, uint32_t* ctx_ids, uint64_t* event_off,
                         uint64_t* t_end, uint32_t* profile_ids);

/* Writes the loaded traces back as a packed trace.db body (12-byte AoS,
 * n_events * 12 bytes) into host memory (the inverse of K1). */
ps_status psg_export_aos(psg_context* ctx, void* body);
/* The same for the loaded traces [t_lo, t_hi) only (their events back to
 * back: (event_off[t_hi] - event_off[t_lo]) * 12 bytes). */
ps_status psg_export_aos_range(psg_context* ctx, uint32_t t_lo, uint32_t t_hi, void* body);
/* Process-wide number of psg kernel launches so far (CUB library kernels
 * are not counted). */
uint64_t psg_kernel_launches(void);

/* ---- query ------------------------------------------------------------- */
enum {
  PSG_Q_WINDOW = 1u << 0,      /* (1)+(2): window filter + per-(trace,ctx) aggregates */
  PSG_Q_CUBE = 1u << 1,        /* (3): iteration detection + trace x iteration x node cube */
  PSG_Q_STATS = 1u << 2,       /* cross-rank savings / CV over the cube (needs CUBE) */
  PSG_Q_OUTLIERS = 1u << 3,    /* (4): balance ratios, node means, z-score / top-k, topology (needs WINDOW) */
  PSG_Q_NO_CUBE_STORE = 1u << 8, /* store only the incl half of the cube (excl is dropped) */
  PSG_Q_CLAMP_TEND = 1u << 9,    /* window end = min(t1, trace t_end) per trace: whole-trace
                                    integration equals the trace's profile record exactly */
  PSG_Q_CUBE64 = 1u << 10,       /* keep 64-bit cube cells in HBM even when every stored
                                    iteration spans < 2^32 ns (default there: 32-bit cells,
                                    exact, widened to int64 on copy-out) */
  PSG_Q_EXACT_BOUNDS = 1u << 11, /* run pass 1 in its exact mode (boundary timestamps loaded
                                    and deduplicated there) instead of the optimistic one
                                    verified by pass 2 */
  PSG_Q_SPARSE = 1u << 12,       /* window as sparse (trace, ctx) rows (psg_get_window_groups /
                                    psg_get_remat_rows) instead of dense [trace][ctx]; taken
                                    anyway when the tree is too large for the fused kernel's
                                    per-warp window records or the dense result for HBM */
  PSG_Q_ALL = PSG_Q_WINDOW | PSG_Q_CUBE | PSG_Q_STATS | PSG_Q_OUTLIERS
};

#define PSG_ANCHOR_AUTO 0xFFFFFFFFu

typedef struct psg_query_spec {
  uint32_t flags;
  uint64_t t0_ns, t1_ns;         /* window [t0, t1); t0 > t1 is PS_E_INVALID_ARGUMENT */
  uint32_t anchor_ctx;           /* explicit anchor (itermodel anchor_policy::explicit_ctx), or
                                    PSG_ANCHOR_AUTO: suggest_anchor on the trace with the
                                    smallest profile id, on the device (itermodel.cpp:45-109,
                                    253-255) */
  /* outliers: candidate call-site contexts (the worst balance ratio wins,
   * workflows.cpp:442-459), then node means of its per-rank window-inclusive
   * time, z-scores, and the top-k (value desc, node id asc) among z >= z_min
   * (k = 0: no cap). */
  const uint32_t* site_ctx;
  uint32_t n_sites;
  uint32_t top_k;
  double z_min;
} psg_query_spec;

typedef struct psg_query_info {
  /* window */
  uint64_t n_window_groups;      /* rows of the group_aggregate result (count > 0) */
  uint64_t n_window_rows;        /* events with t0 <= ts < t1 */
  /* cube (global over all ranks where noted) */
  uint32_t n_nodes;              /* anchor subtree size */
  uint32_t n_kept;               /* local traces with >= 1 iteration */
  uint32_t n_skipped;            /* local traces without iterations */
  uint32_t min_iterations;       /* global ordinal intersection (diagnostics use it) */
  uint32_t n_kept_global;
  uint64_t n_cells;              /* local cube cells (sum iter_counts * n_nodes) */
  uint32_t n_leaves;
  uint32_t n_internal;           /* internal nodes of the subtree (the cube stores excl only for these) */
  uint32_t anchor;               /* the anchor used (the suggested one for PSG_ANCHOR_AUTO) */
  /* outliers */
  uint32_t worst_site;           /* ctx id */
  double worst_ratio;
  uint32_t n_outliers;
  uint32_t n_racks;
  /* timing of the last query on the device (CUDA events on psg_stream) */
  float ms_total;
  float ms_main;                 /* pass 2: the fused window+cube kernel (k_trace_query) */
  float ms_bounds;               /* pass 1: iteration boundaries (k_bounds), 0 without CUBE */
  /* device cube storage: bytes per cell (4 when every stored iteration spans
   * < 2^32 ns, else 8) and total bytes incl. the per-row pad column */
  uint32_t cube_cell_bytes;
  uint64_t cube_store_bytes;
  /* host round trips (stream synchronisations) the query made: 1 once an
   * earlier query on the same traces has sized the device buffers */
  uint32_t host_syncs;
  /* the window's layout: 1 = sparse rows (PSG_Q_SPARSE or a large tree), and
   * the rematerialize rows (incl or excl nonzero) it holds */
  uint32_t window_sparse;
  uint64_t n_remat_rows;
} psg_query_info;

ps_status psg_query(psg_context* ctx, const psg_query_spec* spec, psg_query_info* info);

/* ---- result copy-out (caller-allocated host arrays; NULL skips a column) -- */
/* Dense per-(trace, ctx) window aggregates, trace-major [n_traces][n_ctx]:
 * count, sum/min/max of clipped row durations (ns), mean = sum/count,
 * excl/incl = time-integrated exclusive/inclusive ns incl. the carry-in
 * segment (itermodel::rematerialize over [t0,t1)). */
ps_status psg_get_window(psg_context* ctx, uint64_t* count, int64_t* sum, int64_t* min,
                         int64_t* max, double* mean, int64_t* excl, int64_t* incl);
/* The window as sparse rows sorted by (trace, ctx), for either layout:
 * group_aggregate over the window rows keyed by (pid, ctx) (frame.cpp:290-408)
 * — *n rows with count > 0: loaded-trace index, ctx, count, sum / min / max of
 * the clipped row durations (ns), mean; and itermodel::rematerialize over
 * [t0, t1) per trace (itermodel.cpp:145-183) — *n rows with incl or excl
 * nonzero.  Call with NULL arrays to size. */
ps_status psg_get_window_groups(psg_context* ctx, uint64_t* n, uint32_t* trace, uint32_t* ctx_ids,
                                uint64_t* count, int64_t* sum, int64_t* min, int64_t* max, double* mean);
ps_status psg_get_remat_rows(psg_context* ctx, uint64_t* n, uint32_t* trace, uint32_t* ctx_ids,
                             int64_t* incl, int64_t* excl);
/* Per trace carry-in (store.cpp:667-670): has (0/1), ts, ctx. */
ps_status psg_get_carry(psg_context* ctx, uint8_t* has, uint64_t* ts, uint32_t* ctx_ids);
/* tri_model (itermodel.hpp:78-116): node_ids[n_nodes], per loaded trace
 * iter_counts[n_traces] (0 = skipped), block_offset[n_kept], dense cube
 * incl/excl[n_cells] (iteration-major, node-minor per kept trace, kept traces
 * in load order) and gap rows [n_kept][n_nodes]. */
ps_status psg_get_cube(psg_context* ctx, uint32_t* node_ids, uint32_t* iter_counts,
                       uint64_t* block_offset, int64_t* incl, int64_t* excl,
                       int64_t* gap_incl, int64_t* gap_excl);
/* The cube exactly as stored in HBM, copied without conversion (lossless;
 * the fast copy-out for host consumers that read the compact form): the
 * incl cells (*cell_bytes = 4 or 8) in rows of stride *row_stride (n_nodes + 1
 * rounded up to even; column n_nodes is padding), each kept trace's
 * iter_counts[t] rows starting at cell stored_off[t] (loaded-trace index;
 * undefined for skipped traces), and the exclusive time of the anchor
 * subtree's internal nodes [rows][n_internal] (rows in trace order; a leaf's
 * excl is its incl) when the query stored it.  Sizes are set first; any
 * output pointer may be NULL. */
ps_status psg_get_cube_stored(psg_context* ctx, uint32_t* cell_bytes, uint32_t* row_stride,
                              uint64_t* incl_bytes, void* incl, uint64_t* stored_off,
                              uint64_t* xint_cells, int64_t* xint);
/* The same copy, enqueued on the context's copy-out stream and returned at
 * once (pinned destinations): it overlaps whatever the host does next, e.g.
 * loading the next batch of traces (the H2D and D2H directions run on
 * separate copy engines).  The next psg_query waits for it on the device;
 * psg_wait_copies blocks the host until the data has landed. */
ps_status psg_get_cube_stored_async(psg_context* ctx, void* incl, uint64_t* stored_off, int64_t* xint);
ps_status psg_wait_copies(psg_context* ctx);
/* The same dense layout for the loaded traces [t_lo, t_hi) only (the kept
 * ones, in load order, relative to the range): *n_cells and *n_kept are set
 * first (any output pointer may be NULL, e.g. to size the arrays), then
 * incl / excl [*n_cells] and gap rows [*n_kept][n_nodes].  Cells are widened
 * to int64 on the device; no host buffer of the whole cube is needed. */
ps_status psg_get_cube_range(psg_context* ctx, uint32_t t_lo, uint32_t t_hi, uint64_t* n_cells,
                             uint32_t* n_kept, int64_t* incl, int64_t* excl, int64_t* gap_incl,
                             int64_t* gap_excl);
/* detect_iterations' boundaries (itermodel.cpp:111-143) of loaded trace
 * `trace` after a PSG_Q_CUBE query: *n boundary timestamps (strictly
 * increasing; the last may equal t_end, an empty interval the cube drops).
 * ts = NULL sizes. */
ps_status psg_get_boundaries(psg_context* ctx, uint32_t trace, uint32_t* n, uint64_t* ts);
/* topology::parse_node_name (topology.cpp:14-46): rack and chassis of an
 * x<r>c<c>s<s>b<b>n<n> hostname, else PS_E_PARSE with the reference's message. */
ps_status psg_node_name(const char* name, uint32_t* rack, uint32_t* chassis);
/* savings_report / iteration_cv_report per subtree leaf (diagnostics.cpp:100-158):
 * leaves[n_leaves]; savings rows [n_leaves][4] = avg_mean_s, avg_max_s,
 * savings_per_iter_s, total_reduction_s; summary[4] = n_iterations,
 * total_savings_s, total_time_s (as given), speedup_frac; cv [n_leaves][2] =
 * across, within; cv_ok[n_leaves] (0 = the reference would raise). */
ps_status psg_get_stats(psg_context* ctx, double total_time_s, uint32_t* leaves, double* savings,
                        double* summary, double* cv, int32_t* cv_ok);
/* Outliers: per site balance ratio [n_sites]; node means [n_nodes] (s);
 * node z-scores; selected node ids [n_outliers] (value desc, id asc); topology
 * rows [n_racks][3] = rack, affected nodes, n_chassis and chassis masks per
 * rack: affected [n_racks], fully affected [n_racks] (bit c = chassis c).
 * Outlier queries raise PS_E_PARSE when a hostname of the node universe read
 * from a database is not a Slingshot name (topology.cpp:14-46). */
ps_status psg_get_outliers(psg_context* ctx, double* site_ratio, double* node_mean, double* node_z,
                           uint32_t* selected, uint32_t* rack_rows, uint64_t* chassis_mask,
                           uint64_t* full_mask);

/* localize_outliers' rows (topology.cpp:54-92) for any chassis ids: one row
 * [rack, chassis, outlier nodes, fully affected 0/1] per affected (rack,
 * chassis), ascending.  Call with rows = NULL for *n_rows first.  (The masks of
 * psg_get_outliers have bit c = chassis c and need chassis ids < 64.) */
ps_status psg_get_topology(psg_context* ctx, uint32_t* n_rows, uint32_t* rows);

/* ingest::ingest_traces (ingest.cpp:178-208) on the device: the events with
 * t0 <= ts < t1 of every loaded trace in load order, as SoA rows, plus the
 * carry-ins.  Call with NULL arrays to get *n_rows, then again to copy. */
ps_status psg_window_rows(psg_context* ctx, uint64_t t0_ns, uint64_t t1_ns, uint64_t* n_rows,
                          uint32_t* row_pid, uint64_t* row_ts, uint32_t* row_ctx);

/* ---- profile records (profile.db) ---------------- */
/* Loads profile-record bodies into HBM.  `records` holds the packed 14-byte
 * records {u32 ctx, u16 metric, f64 value} of n_profiles profiles back to back
 * (host or device memory; each profile's run sorted by ctx, as the reference's
 * binary search requires, store.cpp:601-613 -- else PS_E_FORMAT),
 * rec_off[n_profiles + 1] their record offsets, pid[] strictly ascending
 * profile ids, rank[] their MPI ranks (-1: not a rank, e.g. the summary
 * profile), node_of_profile[] their node ids in the psg_set_nodes numbering
 * (NULL: no psg_profile_outliers). */
ps_status psg_load_profiles(psg_context* ctx, const void* records, const uint64_t* rec_off,
                            const uint32_t* pid, const int32_t* rank,
                            const uint32_t* node_of_profile, uint32_t n_profiles);
/* meta.bin + profile.db of a reference database directory (db_handle::open,
 * store.cpp:484-503): all profiles; nodes = the hostnames of the ranks, sorted
 * (node_correlate's order), with rack / chassis parsed from Slingshot names. */
ps_status psg_load_profile_db(psg_context* ctx, const char* dir);
/* ingest::ingest_profiles / read_slices (ingest.cpp:122-176) on the device:
 * the records of the requested profiles (sorted, deduplicated; an unknown id
 * is PS_E_NOT_FOUND) whose ctx is in ctx_ids (NULL: all) and metric in
 * metric_ids (NULL: all), profile-id ascending, record order within a profile.
 * Call with NULL row arrays to get *n_rows, then again to copy. */
ps_status psg_slice(psg_context* ctx, const uint32_t* pids, uint32_t n_pids, const uint32_t* ctx_ids,
                    uint32_t n_ctx_ids, const uint16_t* metric_ids, uint32_t n_metrics,
                    uint64_t* n_rows, uint32_t* row_pid, uint32_t* row_ctx, uint16_t* row_metric,
                    double* row_value);
/* congestion_report's numeric core over profile records (workflows.cpp:413-539):
 * per candidate site the rank_vector of `metric` (rank profiles in rank order,
 * absent records as 0; workflows.cpp:42-62), its balance ratio
 * (diagnostics.cpp:10-19), the worst (first minimal) site, the node means of
 * its values (node_correlate, diagnostics.cpp:378-403), then z-scores and the
 * top-k (mean desc, node asc) among z >= z_min, and the rack / chassis
 * localisation.  Results: info (worst_site, worst_ratio, n_outliers, n_racks,
 * ms_total) and psg_get_outliers. */
ps_status psg_profile_outliers(psg_context* ctx, uint16_t metric, const uint32_t* site_ctx,
                               uint32_t n_sites, uint32_t top_k, double z_min, psg_query_info* info);

/* ---- device buffers and small diagnostics (the binding's hot-path
 * signatures) ------------------------------------------- */
/* Device memory on the context's device (e.g. frame columns uploaded by a
 * host caller); psg_copy is cudaMemcpy in any direction, synchronous. */
ps_status psg_dev_alloc(psg_context* ctx, uint64_t bytes, void** out);
void psg_dev_free(psg_context* ctx, void* p);
ps_status psg_copy(psg_context* ctx, void* dst, const void* src, uint64_t bytes);
/* what = 0: diagnostics::balance_ratio, (Σ/n)/max or 1.0 when max == 0;
 * what = 1: cv_percent, 100 * population std / mean (diagnostics.cpp:10-31).
 * values: host or device f64.  Empty input is PS_E_INVALID_ARGUMENT
 * (empty_input); a zero mean is PS_E_INSUFFICIENT_DATA (undefined_cv). */
ps_status psg_vector_stats(psg_context* ctx, const double* values, uint64_t n, uint32_t what,
                           double* result);
/* node_correlate's sums (diagnostics.cpp:378-403): per node the mean of its
 * values summed in input order (bit-identical to the reference's fold) and
 * the count; node_of[i] < n_nodes.  Host or device values; host outputs. */
ps_status psg_node_means(psg_context* ctx, const double* values, const uint32_t* node_of, uint64_t n,
                         uint32_t n_nodes, double* mean, uint32_t* count);
/* localize_outliers' counts (topology.cpp:54-92): nodes [0, n_universe) are
 * the universe, further nodes are outliers outside it; outliers[] are node
 * indices (distinct).  Rows as psg_get_topology: [rack, chassis, outlier
 * nodes, fully affected] ascending; call with rows = NULL for *n_rows. */
ps_status psg_localize(psg_context* ctx, const uint32_t* node_rack, const uint32_t* node_chassis,
                       uint32_t n_nodes, uint32_t n_universe, const uint32_t* outliers, uint32_t n_out,
                       uint32_t* n_rows, uint32_t* rows);

/* ---- frame operators (frame.hpp) ------------------
 * The reference's columnar engine for numeric columns on the device, with its
 * determinism contract (frame.hpp:3-10): every result is the reference's,
 * bit for bit.  Column data pointers are DEVICE pointers (e.g. CUDA tensors);
 * n = rows.  Index outputs (perm, starts, idx, lidx, ridx) are device u64. */
enum { PSG_I64 = 0, PSG_U64 = 1, PSG_F64 = 2 };                      /* frame::dtype */
enum { PSG_LT = 0, PSG_LE = 1, PSG_EQ = 2, PSG_GE = 3, PSG_GT = 4, PSG_NE = 5 }; /* frame::cmp_op */
enum { PSG_AGG_SUM = 0, PSG_AGG_MIN = 1, PSG_AGG_MAX = 2, PSG_AGG_MEAN = 3, PSG_AGG_COUNT = 4 };
typedef struct psg_col {
  uint32_t dtype;
  const void* data;
} psg_col;
/* sort's permutation (frame.cpp:62-117, 410-422): stable multi-key argsort,
 * ascending[k] = 0 for a descending key (NULL: all ascending). */
ps_status psg_frame_argsort(psg_context* ctx, const psg_col* keys, uint32_t n_keys,
                            const uint8_t* ascending, uint64_t n, uint64_t* perm);
/* group_aggregate's grouping (frame.cpp:290-318): perm[n] sorted by the key
 * tuple, starts[*n_groups] = first sorted position of each group. */
ps_status psg_frame_group(psg_context* ctx, const psg_col* keys, uint32_t n_keys, uint64_t n,
                          uint64_t* perm, uint64_t* starts, uint64_t* n_groups);
/* one aggregate column per group (frame.cpp:320-392): sum / min / max in the
 * source dtype (integer sums wrap), mean in f64, count in u64; NaN in an f64
 * source is PS_E_INVALID_ARGUMENT (require_numeric). */
ps_status psg_frame_group_agg(psg_context* ctx, psg_col src, const uint64_t* perm,
                              const uint64_t* starts, uint64_t n_groups, uint64_t n, uint32_t fn,
                              void* out);
/* out[i] = src[idx[i]] (any 8-byte dtype). */
ps_status psg_frame_gather(psg_context* ctx, psg_col src, const uint64_t* idx, uint64_t n_idx,
                           void* out);
/* filter (frame.cpp:424-470): idx[*n_out] = rows with (col <op> *literal), in
 * order; literal is a host i64 / u64 / f64 of the column's dtype. */
ps_status psg_frame_filter(psg_context* ctx, psg_col col, uint32_t op, const void* literal,
                           uint64_t n, uint64_t* idx, uint64_t* n_out);
/* merge (frame.cpp:472-572): inner-join row pairs ordered by (left row, right
 * row).  *n_out is always set; the pairs are written when it fits capacity. */
ps_status psg_frame_merge(psg_context* ctx, const psg_col* lkeys, const psg_col* rkeys,
                          uint32_t n_keys, uint64_t n_left, uint64_t n_right, uint64_t capacity,
                          uint64_t* lidx, uint64_t* ridx, uint64_t* n_out);
/* vector_add, in_place_multiply, scalar_compare (0/1 i64), reduce_sum and
 * cumulative_sum (fold-left in 4096-element blocks, then across blocks;
 * frame.cpp:574-657) over f64 columns. */
ps_status psg_frame_vector_add(psg_context* ctx, const double* a, const double* b, uint64_t n,
                               double* out);
ps_status psg_frame_multiply(psg_context* ctx, const double* a, double scalar, uint64_t n,
                             double* out);
ps_status psg_frame_scalar_compare(psg_context* ctx, const double* a, uint32_t op, double scalar,
                                   uint64_t n, int64_t* out);
ps_status psg_frame_reduce_sum(psg_context* ctx, const double* a, uint64_t n, double* result);
ps_status psg_frame_cumsum(psg_context* ctx, const double* a, uint64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PSG_H */
