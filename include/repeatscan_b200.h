/*
 * repeatscan_b200.h -- C-ABI of the B200-native longest-repeat path.
 *
 * Drop-in boundary for the reference package `repeatscan`
 * (/root/reference/pkg/src/repeatscan, cited below as <file>:<line>).  The
 * reference has no FFI: its data-parallel path goes through the operator API
 * `_backend.kernels` (11 chunked numba kernels, _kernels_numba.py:15-195)
 * driven by `engine.parallel_for/parallel_scan` (engine.py:55-110).  Each
 * entry point below replaces one reference call site; the ctypes binding in
 * paper_1501_06663_b200/_native.py mirrors the reference Python API on top.
 *
 * Conventions (the reference's host layouts, suffixes.py:3-8, query.py:130-168):
 *   - every host array is int64, 1-based with an unused pad slot 0:
 *       sa[n+1], rank[n+1], lcp[n+2], raw[n+1], flags[n+1], ps[n+1],
 *       leftmost starts/lengths[n+1], all lengths[n+1], offsets[n+2];
 *     compact starts/lengths and flat tie starts are 0-based [m] / [T].
 *   - plain host pointers and sizes; no device or torch types cross the ABI.
 *   - every call is synchronous w.r.t. its host outputs and returns a status;
 *     rs_last_error() explains a non-zero status.
 *   - mode: 0 = leftmost, 1 = all ties.   path: 0 = raw, 1 = compact.
 *   - n <= 2^31 - 2 (device indices are 32-bit; tie totals are 64-bit).
 */
#ifndef REPEATSCAN_B200_H
#define REPEATSCAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (0 = ok) */
#define RS_OK 0
#define RS_EINVAL -1 /* bad argument / malformed input -> ValueError  */
#define RS_ERANGE -2 /* position / size out of range   -> IndexError  */
#define RS_ENOMEM -3 /* device or host allocation failed -> MemoryError */
#define RS_ECUDA -4  /* CUDA runtime error              -> RuntimeError */
#define RS_ENCCL -5  /* NCCL error                      -> RuntimeError */
#define RS_ESTATE -6 /* call out of order (e.g. fetch before query)   */

#define RS_MODE_LEFTMOST 0
#define RS_MODE_ALL 1
#define RS_PATH_RAW 0
#define RS_PATH_COMPACT 1

/* stage timers (milliseconds, CUDA events on the context stream) */
#define RS_STAGE_H2D 0
#define RS_STAGE_SA 1
#define RS_STAGE_LCP 2
#define RS_STAGE_RAW_LLR 3
#define RS_STAGE_COMPACT 4
#define RS_STAGE_QUERY 5
#define RS_STAGE_D2H 6
#define RS_NUM_STAGES 7

typedef struct rs_ctx rs_ctx;

/* ---- context ------------------------------------------------------------ */
const char *rs_version(void);
int rs_device_count(int *count);
/* One context per process and device: a CUDA stream, a device buffer arena
 * and the device-resident pipeline state.  Replaces the thread pool of
 * engine.py:71-74 / :92-109 as the "concurrency boundary". */
int rs_create(int device, rs_ctx **out);
int rs_destroy(rs_ctx *ctx);
const char *rs_last_error(const rs_ctx *ctx);
int rs_synchronize(rs_ctx *ctx);
/* number of kernels this context launched so far */
int rs_launch_count(const rs_ctx *ctx, int64_t *count);
/* bytes this context copied host -> device and device -> host so far (every
 * transfer the library issues: inputs, wire words / bytes, small readbacks) */
int rs_transfer_bytes(const rs_ctx *ctx, int64_t *h2d_bytes, int64_t *d2h_bytes);
/* last per-stage device times (RS_NUM_STAGES doubles) */
int rs_stage_times(const rs_ctx *ctx, double *ms);
/* CUDA-event timing on the context stream (slots 0..63) */
int rs_record_event(rs_ctx *ctx, int slot);
int rs_elapsed_ms(rs_ctx *ctx, int slot_a, int slot_b, float *ms);
/* bytes of device memory currently held by the arena */
int rs_device_bytes(const rs_ctx *ctx, int64_t *bytes);
/* release every device buffer of the arena */
int rs_release(rs_ctx *ctx);
/* pinned host memory for zero-staging D2H outputs (cudaHostAlloc) */
int rs_host_alloc(int64_t bytes, void **out);
int rs_host_free(void *p);

/* ---- array-level operators (host int64 in / host int64 out) -------------
 * Each replaces one reference function on caller-allocated arrays. */

/* suffixes.py:56-66 build_suffix_structures: sa[n+1], rank[n+1], lcp[n+2]
 * (zero-filled pads) from text[n]; prefix doubling + LSD radix sort on device,
 * rank by inversion, Kasai/PLCP LCP. */
int rs_suffix_structures(rs_ctx *ctx, const uint8_t *text, int64_t n, int64_t *sa,
                         int64_t *rank, int64_t *lcp);
/* llr.py:63-72 build_raw_llr -> _kernels_numba.py:33-38 fill_raw_llr */
int rs_raw_llr(rs_ctx *ctx, const int64_t *rank, const int64_t *lcp, int64_t n, int64_t *raw);
/* llr.py:84-89 compute_flags -> _kernels_numba.py:41-46 fill_flags */
int rs_flags(rs_ctx *ctx, const int64_t *raw, int64_t n, int64_t *flags);
/* llr.py:92-96 prefix_sum -> engine.py:77-110 parallel_scan (inclusive over
 * slots 1..n of an (n+1)-array; ps[0] = 0) */
int rs_prefix_sum(rs_ctx *ctx, const int64_t *flags, int64_t n, int64_t *ps);
/* engine.py:77-110 parallel_scan on a plain 0-based array of `count` values */
int rs_inclusive_scan(rs_ctx *ctx, const int64_t *values, int64_t count, int64_t *out);
/* llr.py:99-116 scatter_compact -> _kernels_numba.py:49-55 scatter_chunk;
 * starts/lengths hold ps[n] entries */
int rs_scatter_compact(rs_ctx *ctx, const int64_t *raw, const int64_t *flags, const int64_t *ps,
                       int64_t n, int64_t *starts, int64_t *lengths);
/* llr.py:119-123 build_compact_llr (fused flag -> scan -> scatter) and
 * llr.py:75-81 compact_llr_sequential (same result).  starts/lengths must
 * hold n entries; *m receives the entry count. */
int rs_compact(rs_ctx *ctx, const int64_t *raw, int64_t n, int64_t *starts, int64_t *lengths,
               int64_t *m);

/* ---- device-resident pipeline (query.py:218-239 all_positions) ----------
 * load text or structures once, run the query on device, fetch results. */

/* Text bytes (text.py:21-23 uint8 buffer), H2D. */
int rs_set_text(rs_ctx *ctx, const uint8_t *text, int64_t n);
/* query.py:234 `structures=` input (range-checked on device).  sa may be
 * NULL: the query path only reads rank and lcp (_kernels_numba.py:33-38). */
int rs_set_structures(rs_ctx *ctx, const int64_t *sa, const int64_t *rank, const int64_t *lcp,
                      int64_t n);
/* suffixes.py:69-103 verify_suffix_structures, on device; *ok = 1 iff valid.
 * (size and sentinel checks are the caller's, as in the reference). */
int rs_verify_structures(rs_ctx *ctx, const uint8_t *text, int64_t n, const int64_t *sa,
                         const int64_t *rank, const int64_t *lcp, int64_t *ok);
/* Independent check of query answers against compact entries starts/lengths[m]
 * (the reference's Algorithm 4 as written, _kernels_numba.py:74-85 +
 * :158-195: binary search + forward walk per position, no code shared with
 * the scan kernels).  All-ties arrays (a_lengths[n+1], a_offsets[n+2],
 * a_flat[total]) and/or leftmost arrays (l_starts/l_lengths[n+1]) may be
 * NULL.  *bad receives the number of positions whose answer differs. */
int rs_check_answers(rs_ctx *ctx, const int64_t *starts, const int64_t *lengths, int64_t m, int64_t n,
                     const int64_t *a_lengths, const int64_t *a_offsets, const int64_t *a_flat,
                     int64_t total, const int64_t *l_starts, const int64_t *l_lengths, int64_t *bad);
/* query.py:234 build_suffix_structures on device from the loaded text. */
int rs_build_structures(rs_ctx *ctx);
int rs_get_structures(rs_ctx *ctx, int64_t *sa, int64_t *rank, int64_t *lcp);
/* query.py:171-215 `raw` / `c` inputs given by the caller. */
int rs_set_raw(rs_ctx *ctx, const int64_t *raw, int64_t n);
int rs_set_compact(rs_ctx *ctx, const int64_t *starts, const int64_t *lengths, int64_t m,
                   int64_t n);
/* query.py:235-239: raw LLR (if absent) -> compaction (compact path, if
 * absent) -> per-position scan.  For mode=all, *total receives T, the
 * number of tie starts (may be NULL). */
int rs_query(rs_ctx *ctx, int mode, int path, int64_t *total);
/* Leftmost results: starts[n+1] (starts[0] = -1), lengths[n+1]. */
int rs_fetch_leftmost(rs_ctx *ctx, int64_t *starts, int64_t *lengths);
/* All-ties results: lengths[n+1], offsets[n+2], flat[T]. */
int rs_fetch_all(rs_ctx *ctx, int64_t *lengths, int64_t *offsets, int64_t *flat);
/* Intermediate arrays of the pipeline (for build_raw_llr / build_compact_llr). */
int rs_get_raw(rs_ctx *ctx, int64_t *raw);
int rs_get_compact_size(rs_ctx *ctx, int64_t *m);
int rs_get_compact(rs_ctx *ctx, int64_t *starts, int64_t *lengths);
/* Invalidate the pipeline state (keeps the buffer arena). */
int rs_reset(rs_ctx *ctx);
/* Drop everything derived from the loaded text (keeps the text resident). */
int rs_clear_derived(rs_ctx *ctx);
/* Drop the raw LLR / compact entries but keep the suffix structures on
 * device: the next rs_query recomputes llr.py:63-123 from them, like the
 * reference's all_positions(text, structures=s) (query.py:234-239). */
int rs_clear_llr(rs_ctx *ctx);
/* Per-kernel profiling: while enabled every launch is bracketed by CUDA
 * events on the context stream and tagged with its algorithmic HBM bytes.
 * rs_profile_end aggregates per kernel name; read them with rs_profile_kernel. */
int rs_profile_begin(rs_ctx *ctx);
int rs_profile_end(rs_ctx *ctx, int *kinds);
int rs_profile_kernel(rs_ctx *ctx, int i, char *name, int cap, int64_t *launches,
                      double *total_ms, double *bytes);
/* Number of prefix-doubling rounds of the last on-device suffix sort. */
int rs_sa_rounds(const rs_ctx *ctx, int *rounds);

/* ---- TSV wire format (cli.py:62-93) ------------------------
 * Serialize positions [lo, hi] (1-based, inclusive) of the last rs_query
 * result on device, byte-identical to the reference CLI; *nbytes receives the
 * size; rs_fetch_serialized copies the bytes out. */
int rs_serialize(rs_ctx *ctx, int64_t lo, int64_t hi, int64_t *nbytes);
int rs_fetch_serialized(rs_ctx *ctx, uint8_t *out);

/* ---- walk-step statistics (stats.py:21-76) ---------------
 * Steps of the raw / compact query walk at every position (= candidates
 * covering it) for the loaded raw array or compact entries: steps[n+1]
 * (may be NULL), stats[4] = {min, max, sum, count} over positions with
 * steps > 0 (min = 0 when count = 0). */
int rs_walk_steps(rs_ctx *ctx, int path, int64_t *steps, int64_t *stats);
/* summarize_steps (stats.py:58-68) of a caller-given steps array of `count` values. */
int rs_summarize_steps(rs_ctx *ctx, const int64_t *steps, int64_t count, int64_t *stats);

/* ---- sharded query (multi-GPU) ------------------------------
 * One process per GPU.  The compact entries of the WHOLE text live in every
 * rank's device buffer (rank 0 builds them, torch.distributed/NCCL broadcasts
 * them straight into the buffer returned by rs_device_buffer).  Each rank
 * answers its position shard [lo, hi) (1-based); the shard's left halo is
 * implicit: the per-tile windows are found by binary search over the global
 * entry array (ends strictly increasing), so entries that start before lo
 * but still cover it are included.  Shard outputs are shard-local:
 * leftmost starts/lengths[hi-lo]; all lengths[hi-lo], offsets[hi-lo+1]
 * (offsets[0] = 0, local), flat[T_shard]. */
#define RS_BUF_LLRC 0  /* uint32 pairs (start, length), 8 bytes per entry */
#define RS_BUF_OUT0 1  /* int64 */
#define RS_BUF_OUT1 2  /* int64 */
#define RS_BUF_FLAT 3  /* int64 */
#define RS_BUF_TEXT 4  /* uint8 text (n + 128 bytes; rs_set_text_device) */
#define RS_BUF_SEND 5  /* distributed sort: (position, raw) uint32 pairs bound for other ranks */
#define RS_BUF_RAW 6   /* distributed sort: this rank's raw LLR shard incl. its left halo */
/* Ensure >= bytes of device buffer `which` and return its device pointer; a request
 * within the current capacity never reallocates (contents stay valid). */
int rs_device_buffer(rs_ctx *ctx, int which, int64_t bytes, void **ptr);
/* Declare that RS_BUF_LLRC holds m valid entries of a text of length n
 * (validated on device like rs_set_compact). */
int rs_set_compact_device(rs_ctx *ctx, int64_t m, int64_t n);
/* cudaStream_t of the context (for torch.cuda.ExternalStream). */
int rs_stream(rs_ctx *ctx, void **stream);
int rs_query_shard(rs_ctx *ctx, int mode, int64_t lo, int64_t hi, int64_t *total);
/* Position shard [lo, hi) (1-based) answered from the suffix structures on
 * the device (rs_set_structures or rs_build_structures): raw LLR for the
 * shard's slots and its left halo (slots >= lo - max LCP, the only ones that
 * can reach lo) by the reference formula (_kernels_numba.py:33-38), then the
 * fused compact scan.  Shard outputs as rs_query_shard (rebase / fetch with
 * rs_shard_rebase, rs_fetch_shard).  Multi-GPU query-from-structures: every
 * rank holds the structures and answers its own shard, no exchange. */
int rs_query_structures_shard(rs_ctx *ctx, int mode, int64_t lo, int64_t hi, int64_t *total);
/* Add `base` (the ties of all earlier shards) to the shard's offsets on device. */
int rs_shard_rebase(rs_ctx *ctx, int64_t base);
/* D2H of the shard results (a, b, flat as described above). */
int rs_fetch_shard(rs_ctx *ctx, int mode, int64_t *a, int64_t *b, int64_t *flat);

/* ---- distributed suffix sort ------------------------------
 * Replaces the serial suffix sort of suffixes.py:31-66 when it is split over
 * `world` ranks: every rank holds the whole text (rs_set_text, or
 * rs_device_buffer(RS_BUF_TEXT) + NCCL broadcast + rs_set_text_device) and
 * sorts the suffixes whose top round-0 key digit falls in its range (ranges
 * balanced on the digit histogram), i.e. one contiguous segment of the SA.
 * Raw LLR leaves in text order through an all-to-all of (position, raw)
 * pairs into bucket-aligned position shards, each rank then scans its shard
 * (left halo of `halo` raw values received from the nearest earlier rank
 * with a non-empty shard; `halo` may not exceed that shard's length).
 * Supported regime: 32-bit symbol-aligned round-0 keys and tied groups of at
 * most 1025 suffixes whose common prefixes stay below 4096 symbols (i.i.d. or
 * planted-repeat DNA); info[0] = 0 otherwise and the caller runs the
 * single-GPU path.
 *   rs_dist_sort   info[16]: [ok, m, S (first SA slot), first key, first
 *                  suffix, last key, last suffix, bits, K]
 *   rs_dist_update nbr[6] = prev rank's (last key, last suffix, has_prev),
 *                  next rank's (first key, first suffix, has_next);
 *                  send_counts[world] = entries of RS_BUF_SEND per destination
 *                  (concatenated in rank order); info[0] = ok, info[1] = total
 *   rs_dist_apply  recv = device array of `count` (position, raw) uint32 pairs;
 *                  halo_cap = halo slots reserved before the shard;
 *                  info = [ok, P0, P1 (0-based shard), max raw, R0]; the
 *                  shard's raw array (RS_BUF_RAW) holds raw[i] at [i - R0]
 *   rs_dist_scan   all-ties / leftmost scan of the shard (fused compact
 *                  scan; raw-path scan when a window exceeds its shared
 *                  stage), outputs as rs_query_shard (rebase / fetch with
 *                  rs_shard_rebase, rs_fetch_shard). */
int rs_set_text_device(rs_ctx *ctx, int64_t n);
int rs_dist_sort(rs_ctx *ctx, int32_t rank, int32_t world, int64_t *info);
int rs_dist_update(rs_ctx *ctx, int32_t rank, int32_t world, const int64_t *nbr, int64_t *send_counts,
                   int64_t *info);
int rs_dist_apply(rs_ctx *ctx, int32_t rank, int32_t world, const void *recv, int64_t count, int64_t halo_cap,
                  int64_t *info);
int rs_dist_scan(rs_ctx *ctx, int mode, int64_t halo, int64_t *total);

/* ---- NCCL inside the library ------------------------------
 * The multi-GPU data plane runs as NCCL collectives on each context's stream
 * between the library's device buffers.  Rank 0 creates the 128-byte id
 * (rs_nccl_unique_id) and hands it to the other ranks by any channel
 * (torch.distributed in distributed.py); every rank then calls rs_nccl_init.
 *   rs_nccl_broadcast_text  the text (RS_BUF_TEXT, n bytes) from `root` to
 *                           every rank; leaves the text loaded (as rs_set_text)
 *   rs_nccl_allgather_i64   one int64 per rank (the shards' tie totals) ->
 *                           out[world] in rank order on every rank */
int rs_nccl_unique_id(uint8_t *id128);
int rs_nccl_init(rs_ctx *ctx, const uint8_t *id128, int32_t rank, int32_t world);
int rs_nccl_destroy(rs_ctx *ctx);
int rs_nccl_broadcast_text(rs_ctx *ctx, int64_t n, int32_t root);
int rs_nccl_allgather_i64(rs_ctx *ctx, int64_t value, int64_t *out);

#ifdef __cplusplus
}
#endif
#endif
