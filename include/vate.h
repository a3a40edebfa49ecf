/*
 * vate.h -- C ABI of the B200-native VATE hot path (libvate_b200.so).
 *
 * The reference package (slidecard, pure Python + numpy) has no native
 * interface; its "plugin" boundary is the duck-typed pool protocol plus the
 * estimator / pipeline functions.  Each entry point below names the reference
 * symbol it replaces (paths relative to /root/reference/pkg/src/slidecard/).
 * The Python host layer paper_1812_00282_b200/ binds these through ctypes and
 * re-exposes the reference's names; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Every function returns int: VATE_OK (0) or a negative code.  The text of
 *     the last error on the calling thread is vate_last_error().
 *     VATE_ECONFIG maps to slidecard's ConfigError (errors.py:9-10),
 *     VATE_EVALUE to ValueError (precondition violations, e.g. pools.py:215-217),
 *     VATE_ECUDA / VATE_ENOMEM to RuntimeError / MemoryError.
 *   - A vate_pool owns one CUDA stream on one device; calls on one pool are
 *     stream-ordered and must not be made concurrently from several threads.
 *   - `where` says whether an input pointer is host memory (VATE_HOST) or
 *     device memory on the pool's device (VATE_DEVICE).  Output pointers are
 *     host memory unless the name ends in _dev.
 *   - Plain pointers and sizes only; no torch or numpy types.
 */
#ifndef VATE_H
#define VATE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VATE_ABI_VERSION 1

enum vate_status {
  VATE_OK = 0,
  VATE_ECONFIG = -1, /* ConfigError: bad shape / config / snapshot      */
  VATE_EVALUE = -2,  /* ValueError: precondition violated               */
  VATE_ECUDA = -3,   /* CUDA runtime failure                            */
  VATE_ENOMEM = -4   /* device or pinned allocation failed              */
};

enum vate_where { VATE_HOST = 0, VATE_DEVICE = 1, VATE_STAGED = 2 };
enum vate_partition { VATE_TAIL = 0, VATE_LOWDEV = 1 }; /* pools.py:27-29 */
enum vate_kind { VATE_AT = 0, VATE_DR = 1, VATE_TS = 2 };  /* estimator.py COUNTER_KINDS */

typedef struct vate_pool vate_pool;   /* AtPool on one device               */
typedef struct vate_hosts vate_hosts; /* SlidingHostSet on the same device  */

/* ---- library ---------------------------------------------------------- */
const char* vate_last_error(void);
int vate_abi_version(void);
int vate_device_count(int* n);

/* ---- pool lifecycle: AtPool.__init__ (pools.py:72-100), make_pool
 *      (pools.py:413-421), _validate_pool_shape (pools.py:57-64) --------- */
int vate_pool_create(vate_pool** out, int c, int k, int partition, int device);
/* make_pool(kind, ...) (pools.py:413-421) for every counter kind: VATE_AT as
 * above, or the comparators VATE_DR (DrPool, pools.py:301-353) and VATE_TS
 * (TsPool, pools.py:356-410), which share the scan, registry, g0 and float
 * path but not snapshots or the replica merge (VATE_ECONFIG).  partition is
 * ignored for DR/TS, as make_pool ignores it. */
int vate_pool_create_kind(vate_pool** out, int kind, int c, int k, int partition, int device);
/* the pool's kind and, for TS, its own slice index (TsPool.t, pools.py:360) */
int vate_pool_kind(const vate_pool* p, int* kind, uint64_t* slice_index);
int vate_pool_destroy(vate_pool* p);
/* bact0 (pools.py:96), cell storage bytes (1, 2 or 4), the stream (cudaStream_t) */
int vate_pool_info(const vate_pool* p, int32_t* bact0, int32_t* cell_bytes, void** stream);
/* HBM the pool's cells occupy (unpacked) plus a deferred pool's pending-set
 * bitmap; the reference's packed accounting (pools.py:257-259) is host-side. */
int vate_pool_device_bytes(const vate_pool* p, int64_t* bytes);
/* Per-slice estimate latency of the slice steps (vate_slice_step and the
 * lagged step): with on = 1, CUDA events mark the end of each slice's scan
 * (compute stream) and the landing of its report rows in host memory (copy
 * stream).  out = [slices measured, mean ms, max ms, last ms]. */
int vate_pool_set_latency(vate_pool* p, int on);
int vate_pool_latency(vate_pool* p, double out[4]);
/* The same marks for a slice driven by separate calls (scan, then the
 * estimate's begin/finish): which = 0 after the scan, 1 after the finish. */
int vate_pool_lat_mark(vate_pool* p, int64_t t, int which);
/* out = [deferred scatter on, bit-plane mode on, its window k', its ring
 * slots, the last packed scan's form (1: the per-CTA stamp filter + mark-word
 * check for skewed traffic, 0: plain)]. */
int vate_pool_mode(const vate_pool* p, int32_t out[5]);
/* CUDA runtime calls other than launches made by this thread so far (the
 * library's host cost per slice, with vate_pool_launches). */
int vate_api_calls(uint64_t* n);
int vate_pool_sync(vate_pool* p);
/* cumulative count of kernels this pool (and its registries) launched */
int vate_pool_launches(const vate_pool* p, uint64_t* n);
/* per-kernel CUDA-event timing (bench only): kind ids in vate_kernel_kind */
int vate_pool_set_timing(vate_pool* p, int on);
int vate_pool_timing(vate_pool* p, int kind, double* total_ms, uint64_t* launches);
/* the timed launches since timing was switched on: out[3i..3i+2] = (kind, start
 * ms, end ms) relative to the switch-on; *n = count (may exceed cap).  Gaps
 * between consecutive launches are device idle time (bench diagnostics). */
int vate_pool_timeline(vate_pool* p, double* out, uint64_t cap, uint64_t* n);

/* stream-ordered timestamps for benchmarking: mark(id) records CUDA event id
 * (0..15) on the pool's stream; elapsed waits for both and returns ms. */
int vate_mark(vate_pool* p, int id);
int vate_mark_elapsed(vate_pool* p, int id0, int id1, double* ms);

/* tuning switches (bench / tests): VATE_OPT_G0 = 0 auto, 1 L2-gather kernel,
 * 2 shared-memory / cluster-DSMEM kernel (c <= 24 only).  VATE_OPT_INCREMENTAL
 * = 1 (default) lets the fused estimate update g0 through an inverse index
 * (exact), 0 recomputes every g0 by a full gather. */
enum vate_option { VATE_OPT_G0 = 0, VATE_OPT_INCREMENTAL = 1, VATE_OPT_SCAN_FILTER = 2,
                   VATE_OPT_CONCURRENT = 3, VATE_OPT_INC_SORT = 4, VATE_OPT_FUSE_SWEEP = 5,
                   VATE_OPT_DEFERRED = 6, VATE_OPT_BITPLANE = 7, VATE_OPT_L2_KEEP = 8 };
/* VATE_OPT_L2_KEEP: -1 auto (default: on for deferred pools), 0 off, 1 on --
 * the scan's registry sector loads, stamps and marks carry the L2 evict_last
 * policy so the table and the marks outlive the slice's streaming passes. */
/* VATE_OPT_BITPLANE: -1 auto (default: on for deferred pools, when the HBM
 * fits it), 0 off, 1 on.  On: the pool keeps one mark bitmap per epoch, the
 * estimate for k' = the first estimate's k' reads ~(S | P | M_e) instead of
 * the cells, and the cells are brought up to date block by block as blocks
 * fall due.  Identical results. */
/* VATE_OPT_SCAN_FILTER: -1 auto (default: the per-CTA registry-stamp filter
 * when the last compacted slice saw >= 8 packets per distinct host, else
 * plain stamps), 0 off, 1 on.  Both forms leave identical state. */
/* VATE_OPT_FUSE_SWEEP (default 1): in the slice step the advance's two-block
 * sweep runs inside the bitmap pass (after each word's bits are taken). */
/* VATE_OPT_INC_SORT (default 1): when few hosts join or leave the window, the
 * sorted active set (SlidingHostSet.active, pipeline.py:54-58) is updated by
 * merging the sorted arrivals and removing the departures instead of a full
 * radix sort. */
/* VATE_OPT_CONCURRENT (default 1): the estimate's registry compaction runs
 * beside the bitmap pass, and the slice advance beside g0 + float path, on a
 * second stream of the pool (fork/join by events; results unchanged). */
/* VATE_OPT_DEFERRED: -1 auto (default: on for AT pools whose cells exceed
 * 16 MiB or more), 0 off, 1 on.  On: scans and set_many set one bit per cell in an
 * L2-resident pending-set bitmap; the next pool pass stores the block clocks
 * (identical state). */
int vate_pool_set_option(vate_pool* p, int option, int64_t value);
/* incremental-estimate counters: [rebuilds, delta slices, refresh slices, full
 * slices, last delta cells, last delta work, identity slices, hosts indexed,
 * total index-rebuild time in microseconds, misses gathered since the rebuild,
 * extensions (previous misses merged into the index)] */
int vate_pool_inc_stats(vate_pool* p, uint64_t out[11]);
/* active-set ordering work: [full radix sorts, incremental merges, reuses] */
int vate_pool_sort_stats(const vate_pool* p, uint64_t out[3]);
/* key sorts of the active set (radix): calls, keys sorted in total, the largest */
int vate_pool_sort_sizes(const vate_pool* p, uint64_t out[3]);

/* cudaProfilerStart/Stop, so `ncu --profile-from-start off` captures exactly a
 * timed region (bench.py with VATE_PROFILE_REGION=1). */
int vate_profiler(int on);

enum vate_kernel_kind {
  VATE_K_SCAN = 0,     /* record_pairs / set_many scatter      */
  VATE_K_REGISTRY = 1, /* host-registry update / compaction    */
  VATE_K_BITMAP = 2,   /* Z_p count + inactive bitmap          */
  VATE_K_G0 = 3,       /* per-host g0 gather                   */
  VATE_K_FINAL = 4,    /* estimate LUT + floor compaction      */
  VATE_K_SWEEP = 5,    /* two-block maintenance                */
  VATE_K_SORT = 6,     /* active-host radix sort               */
  VATE_K_OTHER = 7,
  VATE_K_COUNT = 8
};

/* ---- ingest ------------------------------------------------------------ */
/* AtPool.set_many (pools.py:164-178): cells[idx] <- clock of idx's block.
 * Indices >= 2^c fail with VATE_EVALUE (checked on the host for host input). */
int vate_set_cells(vate_pool* p, const uint64_t* idx, uint64_t n, int where);

/* record_pairs (estimator.py:102-104) = pair_cells (:96-99) + set_many, fused.
 * g, cell_stream, group_stream are EstimatorConfig's (estimator.py:32-61).
 * If hosts != NULL the distinct aips are also registered as last seen in
 * slice t (SlidingHostSet.update, pipeline.py:50-52, called from
 * Pipeline.process_slice pipeline.py:146-147). */
int vate_scan_pairs(vate_pool* p, uint64_t g, uint64_t cell_stream, uint64_t group_stream,
                    const uint64_t* aips, const uint64_t* bips, uint64_t n, int where,
                    vate_hosts* hosts, int64_t t);
/* Same, on packed 8-byte records {uint32 aip, uint32 bip}. */
int vate_scan_packed(vate_pool* p, uint64_t g, uint64_t cell_stream, uint64_t group_stream,
                     const uint32_t* pairs, uint64_t n, int where, vate_hosts* hosts,
                     int64_t t);
/* H2D prefetch: stage packed records from (pinned) host memory on the pool's
 * copy stream into one of two device buffers (*slot), overlapping the
 * current slice's kernels; vate_scan_staged scans a staged buffer once its
 * copy has landed (stream-ordered, no host wait). */
int vate_stage_packed(vate_pool* p, const uint32_t* pairs, uint64_t n, int* slot);
int vate_scan_staged(vate_pool* p, uint64_t g, uint64_t cell_stream, uint64_t group_stream,
                     int slot, uint64_t n, vate_hosts* hosts, int64_t t);
/* pair_cells (estimator.py:96-99) without touching the pool; c <= 32. */
int vate_pair_cells(vate_pool* p, uint64_t g, int c, uint64_t cell_stream,
                    uint64_t group_stream, const uint64_t* aips, const uint64_t* bips,
                    uint64_t n, int where, uint64_t* out_cells);

/* host_cells (estimator.py:107-111): all g cells of each host, host-major;
 * out_cells holds n*g values. */
int vate_host_cells(vate_pool* p, uint64_t g, int c, uint64_t cell_stream, const uint64_t* aips,
                    uint64_t n, int where, uint64_t* out_cells);

/* ---- maintenance: AtPool.advance_slice (pools.py:221-249) -------------- */
/* blocks[0] = block now at clock 0, blocks[1] = block at clock k;
 * maintained = cells visited, cleared = cells turned inactive. */
int vate_advance(vate_pool* p, int32_t blocks[2], uint64_t* maintained, uint64_t* cleared);
/* Stream-ordered variant: enqueue now, collect with vate_advance_result. */
int vate_advance_async(vate_pool* p);
int vate_advance_result(vate_pool* p, int32_t blocks[2], uint64_t* maintained,
                        uint64_t* cleared);
/* PackedArray write API on the device cells (bitpack.py:57-78, :97-140):
 * put: cells[idx[i]] = values[i] & (2^width - 1) (set / set_one / set_range;
 * duplicate indices must carry equal values); fill: every cell = value
 * (ValueError if value exceeds the width).  Any AT/DR/TS pool. */
int vate_put_cells(vate_pool* p, const uint64_t* idx, const uint64_t* values, uint64_t n,
                   int where);
int vate_fill_cells(vate_pool* p, uint64_t value);

/* ---- queries ----------------------------------------------------------- */
/* AtPool.count_inactive (pools.py:195-210); 1 <= k_prime <= k. */
int vate_count_inactive(vate_pool* p, int k_prime, uint64_t* out);
/* AtPool.inactive_mask (pools.py:187-193): out[i] = 1 if idx[i] inactive. */
int vate_inactive_mask(vate_pool* p, const uint64_t* idx, uint64_t n, int k_prime,
                       uint8_t* out, int where);
/* PackedArray.get through AtPool.cells (bitpack.py:88-95). */
int vate_get_cells(vate_pool* p, const uint64_t* idx, uint64_t n, uint32_t* out, int where);
/* the same for every kind, 64-bit values (TS cells hold u64 slice indices,
 * TS_UNSET = 2^64-1, counters.py:159) */
int vate_get_cells64(vate_pool* p, const uint64_t* idx, uint64_t n, uint64_t* out, int where);
/* inactive_virtual_counts (estimator.py:114-123): g0 per host. */
int vate_host_g0(vate_pool* p, uint64_t g, uint64_t cell_stream, const uint64_t* aips,
                 uint64_t n, int k_prime, int32_t* g0, int where);

/* ---- float path: reports_from_counts (estimator.py:138-162) ------------
 * log_zv[j] = np.log(j == 0 ? 1/(2g) : j/g) for j in [0, g], computed by the
 * host with numpy so the device reproduces numpy's logarithm bit for bit;
 * set once per g.  log_zp is np.log of the clamped pool fraction. */
int vate_set_log_table(vate_pool* p, uint64_t g, const double* log_zv);
int vate_reports_from_counts(vate_pool* p, uint64_t g, const int32_t* g0, uint64_t n,
                             uint64_t pool_inactive, double log_zp, double* est,
                             double* z_v, uint8_t* saturated);

/* ---- fused per-slice estimate: Pipeline._estimate (pipeline.py:120-138) -
 * begin: sorted active hosts (SlidingHostSet.active, pipeline.py:54-58),
 *        pool_inactive (count_inactive) and g0 of every active host are
 *        computed on the device; returns once the host count and P are known
 *        (the g0 gather may still be running).  nhosts == 0 means no report
 *        and no P (pipeline.py:122-123).
 * finish: estimates, z_v, saturation and the `estimate >= floor` filter
 *        (pipeline.py:136-137) on the device; kept rows land in the host
 *        arrays (capacity cap) in ascending host order. */
int vate_estimate_begin(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                        int64_t t, int k_prime, uint64_t* nhosts, uint64_t* pool_inactive);
/* begin for an explicit host list (ascending, no duplicates) instead of the
 * registry's active set -- the aip-range split of a multi-GPU estimate. */
int vate_estimate_begin_hosts(vate_pool* p, const uint64_t* hosts, uint64_t n, int where,
                              uint64_t g, uint64_t cell_stream, int k_prime,
                              uint64_t* pool_inactive);
/* vate_estimate_begin restricted to share `part` of `nparts` of the sorted
 * active set (positions [n*part/nparts, n*(part+1)/nparts)): the multi-GPU
 * split of Pipeline._estimate (pipeline.py:120-138) when every rank's
 * registry holds the same hosts (vate_hosts_touched exchange). *nhosts is the
 * share's size. */
int vate_estimate_begin_part(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                             int64_t t, int k_prime, int part, int nparts, uint64_t* nhosts,
                             uint64_t* pool_inactive);
int vate_estimate_finish(vate_pool* p, uint64_t g, uint64_t pool_inactive, double log_zp,
                         double floor, uint64_t* out_host, double* out_est,
                         double* out_zv, uint8_t* out_sat, uint64_t cap, uint64_t* nkept);

/* async form: the report rows are copied on the pool's D2H stream (double-
 * buffered), overlapping the next slice; *nkept is final on return, the host
 * arrays are complete after vate_estimate_wait. */
int vate_estimate_finish_async(vate_pool* p, uint64_t g, uint64_t pool_inactive, double log_zp,
                               double floor, uint64_t* out_host, double* out_est,
                               double* out_zv, uint8_t* out_sat, uint64_t cap, uint64_t* nkept);
int vate_estimate_wait(vate_pool* p);
/* Device addresses of the last finished report rows (for GPU consumers; with
 * null host output arrays the rows stay in HBM and nothing crosses PCIe).
 * Valid until the next-but-one finish (two report sets alternate). */
/* Multi-GPU lagged step: with a peer exchange set, every lagged slice step
 * (vate_slice_step_lagged, vate_slice_lagged_begin/_end) runs the replica
 * exchange (vate_peer_exchange) between the slice's scan and its pool pass,
 * and this rank's reports are share `part` of `nparts` of the sorted active
 * set.  x = NULL restores the single-GPU step.  Set between lagged runs. */
int vate_pool_set_peer(vate_pool* p, struct vate_peer* x, int part, int nparts);
int vate_reports_device(vate_pool* p, uint64_t** host, double** est, double** zv,
                        uint8_t** sat);

/* Synchronous copy of rows [first, first+n) of the last finished report set
 * (the rows a caller's too-small output arrays did not receive: the async
 * forms copy at most `cap` rows and report the full count in *nkept). */
int vate_reports_copy(vate_pool* p, uint64_t first, uint64_t n, uint64_t* host, double* est,
                      double* zv, uint8_t* sat);

/* ---- one whole slice (pipeline.py:142-160) in one call, streaming form ---
 * scan (pairs: host/device pointer, or the staging slot when where ==
 * VATE_STAGED) -> estimate begin -> the slice's single host round trip ->
 * the previous slice's advance result (collected into res->prev_*) -> g0 ->
 * advance (enqueued) -> float path + async D2H of the report rows (complete
 * after vate_estimate_wait or the next call's round trip).
 * log_zp_table[P] = np.log(clamped P / 2^c) for P in [0, 2^c] (numpy-made,
 * estimator.py:148-151).  The advance of this slice is collected by the next
 * call or by vate_advance_result. */
typedef struct vate_step_result {
  uint64_t nhosts, nkept, pool_inactive;
  int32_t prev_collected;
  int32_t prev_blocks[2];
  uint64_t prev_maintained, prev_cleared;
  int64_t prev_t;      /* lagged step: the slice these results belong to */
  int32_t prev_valid;  /* lagged step: 1 if a slice was completed by this call */
} vate_step_result;
int vate_slice_step(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                    uint64_t group_stream, const uint32_t* pairs, uint64_t n, int where,
                    int64_t t, int k_prime, double floor, const double* log_zp_table,
                    uint64_t* out_host, double* out_est, double* out_zv, uint8_t* out_sat,
                    uint64_t cap, vate_step_result* res);

/* Software-pipelined form of vate_slice_step: enqueues slice t's scan, then
 * completes the PREVIOUS slice (reports into the out arrays, its counts and
 * maintenance in res, res->prev_t / prev_valid say which slice; its g0 lookups,
 * float path and copies run on a second stream beside slice t's scan), then
 * enqueues slice t's bitmap pass, registry compaction, delta apply and sweep.
 * Results are those of vate_slice_step, one call later; vate_slice_flush
 * completes the last slice.  Use one or the other per pool, not both. */
int vate_slice_step_lagged(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                           uint64_t group_stream, const uint32_t* pairs, uint64_t n, int where,
                           int64_t t, int k_prime, double floor, const double* log_zp_table,
                           uint64_t* out_host, double* out_est, double* out_zv,
                           uint8_t* out_sat, uint64_t cap, vate_step_result* res);
int vate_slice_flush(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                     double floor, const double* log_zp_table, uint64_t* out_host,
                     double* out_est, double* out_zv, uint8_t* out_sat, uint64_t cap,
                     vate_step_result* res);
/* The same in two halves, for pools too large for a log table: begin enqueues
 * slice t's scan and completes the previous slice up to g0 (res->nhosts,
 * res->pool_inactive); the caller takes log_zp = np.log of the clamped pool
 * fraction (estimator.py:148-151) and end runs the previous slice's float path
 * and enqueues slice t's estimate front and sweep.  flush_begin + end (with any
 * group_stream) complete the last slice. */
int vate_slice_lagged_begin(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                            uint64_t group_stream, const uint32_t* pairs, uint64_t n, int where,
                            int64_t t, int k_prime, vate_step_result* res);
int vate_slice_lagged_end(vate_pool* p, vate_hosts* hosts, uint64_t g, uint64_t cell_stream,
                          uint64_t group_stream, double floor, double log_zp, uint64_t* out_host,
                          double* out_est, double* out_zv, uint8_t* out_sat, uint64_t cap,
                          vate_step_result* res);
int vate_slice_lagged_flush_begin(vate_pool* p, vate_hosts* hosts, uint64_t g,
                                  uint64_t cell_stream, vate_step_result* res);

/* ---- snapshots: AtPool.snapshot_bytes / load (pools.py:261-298) -------- */
int vate_snapshot_size(const vate_pool* p, uint64_t* nbytes);
int vate_snapshot(vate_pool* p, uint8_t* buf, uint64_t cap, uint64_t* len);
/* Restores payload + bact0 into a pool of the snapshot's (c, k, partition). */
int vate_load(vate_pool* p, const uint8_t* buf, uint64_t len);

/* ---- host registry: SlidingHostSet (pipeline.py:43-64) ------------------ */
int vate_hosts_create(vate_hosts** out, vate_pool* p, int k);
int vate_hosts_destroy(vate_hosts* h);
int vate_hosts_update(vate_hosts* h, const uint64_t* aips, uint64_t n, int64_t t, int where);
/* sorted hosts with last-seen > t - k_prime; *n = count (may exceed cap) */
int vate_hosts_active(vate_hosts* h, int64_t t, int k_prime, uint64_t* out, uint64_t cap,
                      uint64_t* n);
/* drop hosts last seen at or before t - k (SlidingHostSet.prune) */
int vate_hosts_prune(vate_hosts* h, int64_t t);
int vate_hosts_size(vate_hosts* h, uint64_t* n);
/* keys last seen exactly in slice t (what this rank's scans registered in t),
 * into device memory out_dev[cap]; *n = count (VATE_EVALUE if > cap). The
 * multi-GPU exchange all-gathers these so every registry holds the union
 * (SlidingHostSet.update, pipeline.py:50-52, over the sharded stream). */
int vate_hosts_touched(vate_hosts* h, int64_t t, uint64_t* out_dev, uint64_t cap, uint64_t* n);

/* ---- multi-GPU replica merge ---------------------------
 * Replicas share bact0 and hold identical cells at slice start, so a cell
 * differs only if some replica set it this slice (value == its block clock).
 * dirty: 1 bit per cell, words of 32 cells, (2^c + 31) / 32 uint32 words.
 * merge: OR of nranks such bitmaps laid end to end; dirty cells take their
 * block clock.  Both pointers are device memory (e.g. NCCL buffers). */
int vate_dirty_bitmap(vate_pool* p, uint32_t* bitmap_dev);
int vate_merge_dirty(vate_pool* p, const uint32_t* bitmaps_dev, int nranks);

/* ---- multi-GPU exchange over peer memory (option P2P) -----
 * Replaces the all-gather + vate_merge_dirty + touched-host all-gather of the
 * NCCL path with one window per rank in its own HBM, mapped by every peer over
 * NVLink (CUDA IPC), and kernels that OR the peers' dirty bitmaps straight
 * into the cells.  Per slice: vate_peer_exchange after this rank's scans and
 * before its estimate (vate_estimate_begin_part).  key_cap bounds the hosts one
 * rank registers per slice (at most its packets per slice) and must be equal on
 * every rank.
 *   create: allocates the window; handle_out receives 64 bytes (cudaIpcMemHandle_t)
 *           that the launcher all-gathers in rank order.
 *   open:   maps the peers' windows (handles: world * 64 bytes); every rank must
 *           have created its window before any rank exchanges (launcher barrier).
 *   mode:   0 auto (one-shot for world <= 2, else two-shot), 1 one-shot (read every
 *           peer's bitmap), 2 two-shot (reduce own segment, then gather the ORs).
 *   exchange: dirty bitmap + touched keys published, arrival flags, fused OR-and-
 *           apply, peers' keys into the registry; *touched_total = hosts registered
 *           in slice t over all ranks (with repeats across ranks). */
typedef struct vate_peer vate_peer;
int vate_peer_create(vate_peer** out, vate_pool* p, vate_hosts* h, int rank, int world,
                     uint64_t key_cap, uint8_t* handle_out);
int vate_peer_open(vate_peer* x, const uint8_t* handles);
int vate_peer_set_mode(vate_peer* x, int mode);
int vate_peer_exchange(vate_peer* x, int64_t t, uint64_t* touched_total);
int vate_peer_info(const vate_peer* x, uint64_t* window_bytes, uint64_t* nvlink_bytes,
                   int* two_shot);
int vate_peer_destroy(vate_peer* x);


/* ---- line-rate trace ingest (traceio.DeviceSlices; traceio.py:77-106,
 * :188-230): two pinned staging buffers the reader fills from the file, async
 * H2D, packing + slice runs on the device, carried slices across chunks. */
typedef struct vate_tracer vate_tracer;
int vate_tracer_create(vate_tracer** out, vate_pool* p, uint64_t chunk_records,
                       uint64_t slice_us);
int vate_tracer_destroy(vate_tracer* x);
/* the slot's pinned staging buffer (16-byte records), once its last H2D is done */
int vate_tracer_buffer(vate_tracer* x, int slot, uint8_t** host);
int vate_tracer_submit(vate_tracer* x, int slot, uint64_t n, int64_t first_slice,
                       uint64_t prev_ts, int has_prev, uint64_t carry_off, uint64_t carry_n);
/* runs = (slice - first_slice, pair offset) per slice change, unsorted */
int vate_tracer_collect(vate_tracer* x, int slot, uint64_t* runs, uint64_t cap,
                        uint64_t* nruns, int64_t* violation, uint32_t** pairs_dev);
int vate_tracer_release(vate_tracer* x, int slot);
/* L2 ceilings for bench.py's rooflines (measurement only): over an
 * L2-resident buffer of buf_bytes (power of two), n random accesses per
 * launch, reps timed launches after a warm-up; out = [random 32-B sector
 * reads G/s, random 2-byte stores G/s, random 32-bit red.or G/s, streaming
 * read GB/s]. */
int vate_bench_l2(vate_pool* p, uint64_t buf_bytes, uint64_t n, int reps, double out[4]);
/* Measurement only: ms per launch of the scan's memory skeleton (per packet one
 * streamed 8-B read, one random red.or into a 2^mark_log2-bit bitmap, one random
 * 32-B read of a table_bytes table) on the scan's grid. */
int vate_bench_scan_skeleton(vate_pool* p, int mark_log2, uint64_t table_bytes, uint64_t n,
                             int reps, double* ms_out);
/* The same with ablation flags (vate_probe.cu): 1 the scan's 64-bit hashing,
 * 2 stamp stores, 4 dependent second reads, 8 256-bit loads. */
int vate_bench_scan_ablation(vate_pool* p, int mark_log2, uint64_t table_bytes, uint64_t n,
                             int reps, int flags, double* ms_out);

/* ---- speed-of-light probe (bench only) -----------------------------------
 * n "packets" of the scan's memory pattern without its arithmetic or input
 * stream: one random 32-B load from a table_bytes table and one random byte
 * store into the pool's cells (power-of-two spans; clobbers the cells -- use a
 * scratch pool).  Mean ms per launch over reps. */
int vate_bench_sol_scatter(vate_pool* p, uint64_t n, uint64_t table_bytes, int reps,
                           double* ms_per_rep);

/* ---- synthetic traffic (bench / tests): oracle.synthetic_slice ---------- */
int vate_synth_packets(vate_pool* p, int64_t t, uint64_t n, uint64_t hosts,
                       uint64_t base_aip, uint64_t trace_seed, uint32_t* pairs_dev);
/* cfg 3 (oracle.synthetic_zipf_slice): Zipf host ranks from a fixed-point CDF
 * table, plus spread_q16/65536 of packets from nspread super-spreaders with
 * random peers (tables on the device, built by the caller). */
int vate_synth_zipf(vate_pool* p, int64_t t, uint64_t n, uint64_t hosts, uint64_t base_aip,
                    uint64_t trace_seed, const uint64_t* zipf_cdf_dev,
                    const uint64_t* spread_cdf_dev, uint64_t nspread, uint32_t spread_q16,
                    uint32_t* pairs_dev);

#ifdef __cplusplus
}
#endif
#endif /* VATE_H */
