/*
 * repeatscan_oracle.c -- CPU restatement of the reference longest-repeat path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_1501_06663_b200/csrc/ and the CPU baseline leg of
 * bench.py.  Nothing in the product package links or calls it; the product
 * path fails loudly when its CUDA library is missing instead of falling back
 * here.
 *
 * Every function restates one piece of the reference package `repeatscan`
 * (paths relative to /root/reference/pkg/src/repeatscan/) with the same
 * 1-based padded int64 layouts:
 *   sa[1..n], rank[1..n], lcp[1..n+1] (lcp[1] = lcp[n+1] = 0),
 *   raw[0..n] (raw[0] = 0 pad), compact starts/lengths 0-based [0, m).
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py) plus the reference's own hard-coded
 * known-answer tests (mississippi / aaaa / Figure-4 / abcabcddbca).
 *
 * Threaded drivers (or_*_par) mirror engine.py:43-110 (contiguous chunks,
 * chunked inclusive scan with a serial carry) using OpenMP threads; the
 * chunk kernels themselves are the sequential loops of _kernels_numba.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

/* ------------------------------------------------------------------------ */
/* Suffix array by prefix doubling -- suffixes.py:31-53.                     */
/* numpy: order = argsort(data, stable); dense ranks by cumsum of changes;   */
/* per round key2 = rank[i+k] or -1 past the end, order = lexsort((key2,    */
/* rank)), dense re-rank, k *= 2, until ranks are all distinct.  lexsort is  */
/* a stable sort by (rank, key2); we restate it as two stable counting       */
/* sorts (LSD: key2 first, then rank), both keys being dense in [-1, n).     */
/* ------------------------------------------------------------------------ */
static void counting_sort_by(const i64 *key, i64 shift, i64 nkeys, const i64 *in,
                             i64 *out, i64 n, i64 *cnt) {
    memset(cnt, 0, sizeof(i64) * (size_t)(nkeys + 1));
    for (i64 t = 0; t < n; ++t) cnt[key[in[t]] + shift + 1]++;
    for (i64 b = 1; b <= nkeys; ++b) cnt[b] += cnt[b - 1];
    for (i64 t = 0; t < n; ++t) out[cnt[key[in[t]] + shift]++] = in[t];
}

/* Returns 0-based SA in order[0..n). */
int or_suffix_array_0based(const uint8_t *data, i64 n, i64 *order) {
    if (n <= 0) return 0;
    i64 *rank = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *key2 = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *tmp = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *cnt = (i64 *)malloc(sizeof(i64) * (size_t)(n + 258));
    if (!rank || !key2 || !tmp || !cnt) {
        free(rank); free(key2); free(tmp); free(cnt);
        return -1;
    }
    /* suffixes.py:34 stable argsort of the bytes */
    {
        i64 c256[257];
        memset(c256, 0, sizeof(c256));
        for (i64 i = 0; i < n; ++i) c256[data[i] + 1]++;
        for (int b = 1; b <= 256; ++b) c256[b] += c256[b - 1];
        for (i64 i = 0; i < n; ++i) order[c256[data[i]]++] = i;
    }
    /* suffixes.py:35-38 dense ranks = cumsum of "byte changed" */
    {
        i64 r = 0;
        rank[order[0]] = 0;
        for (i64 t = 1; t < n; ++t) {
            if (data[order[t]] != data[order[t - 1]]) ++r;
            rank[order[t]] = r;
        }
    }
    i64 k = 1;
    /* suffixes.py:40 while rank[order[-1]] != n - 1 */
    while (rank[order[n - 1]] != n - 1) {
        /* :41-42 key2 = rank[i+k] or -1 past the end */
        for (i64 i = 0; i < n; ++i) key2[i] = (i + k < n) ? rank[i + k] : -1;
        /* :43 lexsort((key2, rank)): stable by key2 over index order, then rank */
        for (i64 i = 0; i < n; ++i) tmp[i] = i;
        counting_sort_by(key2, 1, n + 1, tmp, order, n, cnt);
        counting_sort_by(rank, 0, n, order, tmp, n, cnt);
        memcpy(order, tmp, sizeof(i64) * (size_t)n);
        /* :44-51 dense re-rank on (rank, key2) changes */
        i64 r = 0;
        tmp[order[0]] = 0;
        for (i64 t = 1; t < n; ++t) {
            i64 a = order[t], b = order[t - 1];
            if (rank[a] != rank[b] || key2[a] != key2[b]) ++r;
            tmp[a] = r;
        }
        memcpy(rank, tmp, sizeof(i64) * (size_t)n);
        k *= 2; /* :52 */
    }
    free(rank); free(key2); free(tmp); free(cnt);
    return 0;
}

/* kasai_lcp -- _kernels_numba.py:15-30 (1-based padded sa/rank, lcp[n+2]). */
void or_kasai_lcp(const uint8_t *data, const i64 *sa, const i64 *rank, i64 *lcp, i64 n) {
    i64 h = 0;
    for (i64 i = 1; i <= n; ++i) {
        i64 r = rank[i];
        if (r == 1) { h = 0; continue; }
        i64 j = sa[r - 1];
        while (i + h <= n && j + h <= n && data[i + h - 1] == data[j + h - 1]) ++h;
        lcp[r] = h;
        if (h > 0) --h;
    }
}

/* build_suffix_structures -- suffixes.py:56-66.  sa/rank are n+1, lcp n+2;  */
/* the caller zero-fills them (suffixes.py:59-61).                           */
int or_build_structures(const uint8_t *data, i64 n, i64 *sa, i64 *rank, i64 *lcp) {
    if (n <= 0) return 0;
    if (or_suffix_array_0based(data, n, sa + 1) != 0) return -1;
    for (i64 j = 1; j <= n; ++j) sa[j] += 1;        /* :63 */
    for (i64 j = 1; j <= n; ++j) rank[sa[j]] = j;   /* :64 */
    or_kasai_lcp(data, sa, rank, lcp, n);           /* :65 */
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Chunk kernels over a 1-based half-open range [lo, hi).                   */
/* ------------------------------------------------------------------------ */

/* fill_raw_llr -- _kernels_numba.py:33-38 */
void or_fill_raw_llr(i64 lo, i64 hi, const i64 *rank, const i64 *lcp, i64 *out) {
    for (i64 i = lo; i < hi; ++i) {
        i64 a = lcp[rank[i]], b = lcp[rank[i] + 1];
        out[i] = a > b ? a : b;
    }
}

/* fill_flags -- _kernels_numba.py:41-46 */
void or_fill_flags(i64 lo, i64 hi, const i64 *llr, i64 *out) {
    for (i64 i = lo; i < hi; ++i) {
        i64 len = llr[i];
        out[i] = (len > 0 && len >= llr[i - 1]) ? 1 : 0;
    }
}

/* scatter_chunk -- _kernels_numba.py:49-55 */
void or_scatter_chunk(i64 lo, i64 hi, const i64 *llr, const i64 *flags, const i64 *ps,
                      i64 *starts, i64 *lengths) {
    for (i64 i = lo; i < hi; ++i) {
        if (flags[i] == 1) {
            i64 t = ps[i] - 1;
            starts[t] = i;
            lengths[t] = llr[i];
        }
    }
}

/* compact_sequential -- _kernels_numba.py:58-71; returns m */
i64 or_compact_sequential(const i64 *llr, i64 n, i64 *starts, i64 *lengths) {
    i64 j = 0, prev = 0;
    for (i64 i = 1; i <= n; ++i) {
        i64 len = llr[i];
        if (len > 0 && len >= prev) {
            starts[j] = i;
            lengths[j] = len;
            ++j;
        }
        prev = len;
    }
    return j;
}

/* _first_end_at_or_after -- _kernels_numba.py:74-85 */
static i64 first_end_at_or_after(const i64 *ends, i64 size, i64 k) {
    i64 lo = 0, hi = size;
    while (lo < hi) {
        i64 mid = (lo + hi) / 2;
        if (ends[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* leftmost_raw_chunk -- _kernels_numba.py:88-102 */
void or_leftmost_raw_chunk(i64 lo, i64 hi, const i64 *llr, i64 *out_start, i64 *out_len) {
    for (i64 k = lo; k < hi; ++k) {
        i64 best_start = -1, best_len = 0;
        for (i64 i = k; i >= 1; --i) {
            if (i + llr[i] - 1 < k) break;
            if (llr[i] >= best_len) { best_len = llr[i]; best_start = i; }
        }
        out_start[k] = best_start;
        out_len[k] = best_len;
    }
}

/* leftmost_compact_chunk -- _kernels_numba.py:105-118 */
void or_leftmost_compact_chunk(i64 lo, i64 hi, const i64 *starts, const i64 *lengths,
                               const i64 *ends, i64 size, i64 *out_start, i64 *out_len) {
    for (i64 k = lo; k < hi; ++k) {
        i64 best_start = -1, best_len = 0;
        for (i64 t = first_end_at_or_after(ends, size, k); t < size && starts[t] <= k; ++t) {
            if (lengths[t] > best_len) { best_len = lengths[t]; best_start = starts[t]; }
        }
        out_start[k] = best_start;
        out_len[k] = best_len;
    }
}

/* all_raw_count_chunk -- _kernels_numba.py:121-138 */
void or_all_raw_count_chunk(i64 lo, i64 hi, const i64 *llr, i64 *out_len, i64 *out_cnt) {
    for (i64 k = lo; k < hi; ++k) {
        i64 best = 0;
        for (i64 i = k; i >= 1 && i + llr[i] - 1 >= k; --i)
            if (llr[i] > best) best = llr[i];
        i64 cnt = 0;
        if (best > 0)
            for (i64 i = k; i >= 1 && i + llr[i] - 1 >= k; --i)
                if (llr[i] == best) ++cnt;
        out_len[k] = best;
        out_cnt[k] = cnt;
    }
}

/* all_raw_fill_chunk -- _kernels_numba.py:141-155 (writes backwards) */
void or_all_raw_fill_chunk(i64 lo, i64 hi, const i64 *llr, const i64 *best_len,
                           const i64 *offsets, i64 *flat) {
    for (i64 k = lo; k < hi; ++k) {
        i64 len = best_len[k];
        if (len == 0) continue;
        i64 idx = offsets[k + 1];
        for (i64 i = k; i >= 1 && i + llr[i] - 1 >= k; --i)
            if (llr[i] == len) flat[--idx] = i;
    }
}

/* all_compact_count_chunk -- _kernels_numba.py:158-177 */
void or_all_compact_count_chunk(i64 lo, i64 hi, const i64 *starts, const i64 *lengths,
                                const i64 *ends, i64 size, i64 *out_len, i64 *out_cnt) {
    for (i64 k = lo; k < hi; ++k) {
        i64 best = 0;
        i64 t0 = first_end_at_or_after(ends, size, k);
        for (i64 t = t0; t < size && starts[t] <= k; ++t)
            if (lengths[t] > best) best = lengths[t];
        i64 cnt = 0;
        if (best > 0)
            for (i64 t = t0; t < size && starts[t] <= k; ++t)
                if (lengths[t] == best) ++cnt;
        out_len[k] = best;
        out_cnt[k] = cnt;
    }
}

/* all_compact_fill_chunk -- _kernels_numba.py:180-195 (writes forwards) */
void or_all_compact_fill_chunk(i64 lo, i64 hi, const i64 *starts, const i64 *lengths,
                               const i64 *ends, i64 size, const i64 *best_len,
                               const i64 *offsets, i64 *flat) {
    for (i64 k = lo; k < hi; ++k) {
        i64 len = best_len[k];
        if (len == 0) continue;
        i64 idx = offsets[k];
        for (i64 t = first_end_at_or_after(ends, size, k); t < size && starts[t] <= k; ++t)
            if (lengths[t] == len) flat[idx++] = starts[t];
    }
}

/* ------------------------------------------------------------------------ */
/* Threaded drivers -- engine.py:43-110 + llr.py / query.py call sequences.  */
/* ------------------------------------------------------------------------ */

/* engine.py:43-52 contiguous split of [lo, hi) into <= parts chunks */
static void chunk_bounds(i64 lo, i64 hi, int parts, int p, i64 *a, i64 *b) {
    i64 total = hi - lo;
    i64 base = total / parts, extra = total % parts;
    i64 start = lo + p * base + (p < extra ? p : extra);
    *a = start;
    *b = start + base + (p < extra ? 1 : 0);
}

static int clamp_parts(int workers, i64 total) {
    if (workers < 1) workers = 1;
    if (total < workers) workers = (int)(total > 0 ? total : 1);
    return workers;
}

/* engine.py:77-110 parallel_scan (chunk cumsum, serial carry, offset pass) */
void or_parallel_scan(const i64 *values, i64 n, i64 *out, int workers) {
    if (n <= 0) return;
    int parts = clamp_parts(workers, n);
    i64 *carry = (i64 *)calloc((size_t)parts + 1, sizeof(i64));
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b, s = 0;
        chunk_bounds(0, n, parts, p, &a, &b);
        for (i64 i = a; i < b; ++i) { s += values[i]; out[i] = s; }
    }
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(0, n, parts, p, &a, &b);
        carry[p + 1] = carry[p] + (b > a ? out[b - 1] : 0);
    }
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(0, n, parts, p, &a, &b);
        if (carry[p])
            for (i64 i = a; i < b; ++i) out[i] += carry[p];
    }
    free(carry);
}

/* llr.py:63-72 build_raw_llr: out[0..n] */
void or_build_raw_llr_par(const i64 *rank, const i64 *lcp, i64 n, i64 *out, int workers) {
    out[0] = 0;
    if (n <= 0) return;
    int parts = clamp_parts(workers, n);
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(1, n + 1, parts, p, &a, &b);
        or_fill_raw_llr(a, b, rank, lcp, out);
    }
}

/* llr.py:119-123 build_compact_llr: flags -> prefix sum -> scatter.        */
/* starts/lengths must hold n entries; returns m.                           */
i64 or_build_compact_llr_par(const i64 *raw, i64 n, i64 *starts, i64 *lengths, int workers) {
    if (n <= 0) return 0;
    int parts = clamp_parts(workers, n);
    i64 *flags = (i64 *)calloc((size_t)n + 1, sizeof(i64));
    i64 *ps = (i64 *)calloc((size_t)n + 1, sizeof(i64));
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(1, n + 1, parts, p, &a, &b);
        or_fill_flags(a, b, raw, flags);
    }
    or_parallel_scan(flags + 1, n, ps + 1, workers); /* llr.py:92-96 */
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(1, n + 1, parts, p, &a, &b);
        or_scatter_chunk(a, b, raw, flags, ps, starts, lengths);
    }
    i64 m = ps[n];
    free(flags);
    free(ps);
    return m;
}

/* query.py:171-184 _leftmost_all_positions; path 0 = raw, 1 = compact.     */
/* out_start/out_len are n+1; ends is the compact ends array.               */
void or_leftmost_all_par(i64 n, int path, const i64 *raw, const i64 *cs, const i64 *cl,
                         const i64 *ce, i64 m, i64 *out_start, i64 *out_len, int workers) {
    out_start[0] = -1;
    out_len[0] = 0;
    if (n <= 0) return;
    int parts = clamp_parts(workers, n);
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(1, n + 1, parts, p, &a, &b);
        if (path == 0) or_leftmost_raw_chunk(a, b, raw, out_start, out_len);
        else or_leftmost_compact_chunk(a, b, cs, cl, ce, m, out_start, out_len);
    }
}

/* query.py:187-204 _all_all_positions, first half: lengths, counts, offsets. */
/* lengths n+1, offsets n+2 (zeroed by caller); returns T = offsets[n+1].   */
i64 or_all_count_par(i64 n, int path, const i64 *raw, const i64 *cs, const i64 *cl,
                     const i64 *ce, i64 m, i64 *lengths, i64 *offsets, int workers) {
    if (n <= 0) return 0;
    int parts = clamp_parts(workers, n);
    i64 *counts = (i64 *)calloc((size_t)n + 1, sizeof(i64));
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(1, n + 1, parts, p, &a, &b);
        if (path == 0) or_all_raw_count_chunk(a, b, raw, lengths, counts);
        else or_all_compact_count_chunk(a, b, cs, cl, ce, m, lengths, counts);
    }
    or_parallel_scan(counts + 1, n, offsets + 2, workers); /* query.py:201-204 */
    offsets[0] = 0;
    offsets[1] = 0;
    free(counts);
    return offsets[n + 1];
}

/* query.py:205-215 _all_all_positions, second half: fill flat starts. */
void or_all_fill_par(i64 n, int path, const i64 *raw, const i64 *cs, const i64 *cl,
                     const i64 *ce, i64 m, const i64 *lengths, const i64 *offsets,
                     i64 *flat, int workers) {
    if (n <= 0) return;
    int parts = clamp_parts(workers, n);
#pragma omp parallel for num_threads(parts) schedule(static, 1)
    for (int p = 0; p < parts; ++p) {
        i64 a, b;
        chunk_bounds(1, n + 1, parts, p, &a, &b);
        if (path == 0) or_all_raw_fill_chunk(a, b, raw, lengths, offsets, flat);
        else or_all_compact_fill_chunk(a, b, cs, cl, ce, m, lengths, offsets, flat);
    }
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Threaded build_suffix_structures (same output as or_build_structures).    */
/* Used only to give the CPU baseline / reference arm of bench.py its        */
/* `structures=` input at 256 Mi in seconds instead of minutes (the query    */
/* path the arm times starts from given structures, query.py:234).  Same     */
/* prefix doubling as suffixes.py:31-53 -- per round sort by (rank[i],       */
/* rank[i+k] or -1), dense re-rank, double k until ranks are distinct --    */
/* with the sort done as a parallel LSD radix sort of packed 64-bit keys    */
/* (the SA is unique, so any correct sort yields the reference's SA), then  */
/* rank inversion and Kasai's LCP (_kernels_numba.py:15-30) over T chunks   */
/* of text positions, each restarting h at 0 (h is only a lower bound).     */
/* ------------------------------------------------------------------------ */
typedef uint32_t u32;
typedef uint64_t u64;

static int bits_for(u64 x) { int b = 0; while (b < 64 && (x >> b)) ++b; return b; }

int or_build_structures_par(const uint8_t *data, i64 n, i64 *sa, i64 *rank_out, i64 *lcp, int workers) {
    if (n <= 0) return 0;
    if (n >= (1ll << 32) - 2) return -2;
    int T = clamp_parts(workers, n);
    u64 *keyA = (u64 *)malloc(sizeof(u64) * (size_t)n), *keyB = (u64 *)malloc(sizeof(u64) * (size_t)n);
    u32 *valA = (u32 *)malloc(sizeof(u32) * (size_t)n), *valB = (u32 *)malloc(sizeof(u32) * (size_t)n);
    u32 *rank = (u32 *)malloc(sizeof(u32) * (size_t)n);
    i64 *cnt = (i64 *)malloc(sizeof(i64) * (size_t)(T + 1));
    if (!keyA || !keyB || !valA || !valB || !rank || !cnt) {
        free(keyA); free(keyB); free(valA); free(valB); free(rank); free(cnt);
        return -1;
    }
#pragma omp parallel for num_threads(T) schedule(static)
    for (i64 i = 0; i < n; ++i) rank[i] = data[i]; /* order-equivalent to :34-38 */
    u32 maxrank = 255;
    for (i64 k = 1;; k *= 2) {
        int rb = bits_for((u64)maxrank + 1);
#pragma omp parallel for num_threads(T) schedule(static)
        for (i64 i = 0; i < n; ++i) {
            u64 k2 = (i + k < n) ? (u64)rank[i + k] + 1 : 0; /* -1 past the end -> 0 */
            keyA[i] = ((u64)rank[i] << rb) | k2;
            valA[i] = (u32)i;
        }
        /* radix sort in place (ping-pong tracked locally) */
        {
            u64 *kin = keyA, *kout = keyB;
            u32 *vin = valA, *vout = valB;
            const int DB = 11, NB = 1 << DB;
            int bits = 2 * rb + 1;
            i64 *hist = (i64 *)calloc((size_t)T * NB, sizeof(i64));
            for (int shift = 0; shift < bits; shift += DB) {
                memset(hist, 0, sizeof(i64) * (size_t)T * NB);
#pragma omp parallel num_threads(T)
                {
                    int t = 0;
#ifdef _OPENMP
                    t = omp_get_thread_num();
#endif
                    i64 a, b;
                    chunk_bounds(0, n, T, t, &a, &b);
                    i64 *h = hist + (size_t)t * NB;
                    for (i64 i = a; i < b; ++i) h[(kin[i] >> shift) & (NB - 1)]++;
                }
                int distinct = 0;
                for (int d = 0; d < NB && distinct < 2; ++d) {
                    i64 s = 0;
                    for (int t = 0; t < T; ++t) s += hist[(size_t)t * NB + d];
                    distinct += s > 0;
                }
                if (distinct < 2) continue;
                i64 run = 0;
                for (int d = 0; d < NB; ++d)
                    for (int t = 0; t < T; ++t) {
                        i64 c = hist[(size_t)t * NB + d];
                        hist[(size_t)t * NB + d] = run;
                        run += c;
                    }
#pragma omp parallel num_threads(T)
                {
                    int t = 0;
#ifdef _OPENMP
                    t = omp_get_thread_num();
#endif
                    i64 a, b;
                    chunk_bounds(0, n, T, t, &a, &b);
                    i64 *h = hist + (size_t)t * NB;
                    for (i64 i = a; i < b; ++i) {
                        i64 p = h[(kin[i] >> shift) & (NB - 1)]++;
                        kout[p] = kin[i];
                        vout[p] = vin[i];
                    }
                }
                u64 *tk = kin; kin = kout; kout = tk;
                u32 *tv = vin; vin = vout; vout = tv;
            }
            free(hist);
            if (kin != keyA) { /* result lives in the B buffers: swap roles */
                u64 *tk = keyA; keyA = keyB; keyB = tk;
                u32 *tv = valA; valA = valB; valB = tv;
            }
        }
        /* :44-51 dense re-rank by key changes (parallel count + carry) */
#pragma omp parallel num_threads(T)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            i64 a, b, c = 0;
            chunk_bounds(0, n, T, t, &a, &b);
            for (i64 j = (a == 0 ? 1 : a); j < b; ++j) c += keyA[j] != keyA[j - 1];
            cnt[t + 1] = c;
        }
        cnt[0] = 0;
        for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
#pragma omp parallel num_threads(T)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            i64 a, b, r;
            chunk_bounds(0, n, T, t, &a, &b);
            r = cnt[t];
            for (i64 j = a; j < b; ++j) {
                if (j > 0 && keyA[j] != keyA[j - 1]) ++r;
                rank[valA[j]] = (u32)r;
            }
        }
        maxrank = (u32)cnt[T];
        if ((i64)maxrank == n - 1) break; /* :40 all ranks distinct */
    }
#pragma omp parallel for num_threads(T) schedule(static)
    for (i64 j = 0; j < n; ++j) {
        sa[j + 1] = (i64)valA[j] + 1;        /* :63 */
        rank_out[valA[j] + 1] = j + 1;       /* :64 */
    }
    free(keyA); free(keyB); free(valA); free(valB); free(rank); free(cnt);
    /* :65 kasai_lcp over T chunks of text positions */
#pragma omp parallel num_threads(T)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        i64 a, b, h = 0;
        chunk_bounds(1, n + 1, T, t, &a, &b);
        for (i64 i = a; i < b; ++i) {
            i64 r = rank_out[i];
            if (r == 1) { h = 0; continue; }
            i64 j = sa[r - 1];
            while (i + h <= n && j + h <= n && data[i + h - 1] == data[j + h - 1]) ++h;
            lcp[r] = h;
            if (h > 0) --h;
        }
    }
    return 0;
}
