/*
 * oracle32.c -- 32-bit-index restatement of the reference path for the
 * full-size parity digests (n up to 2^31 - 2).
 *
 * TEST INFRASTRUCTURE ONLY (like repeatscan_oracle.c): used by
 * tests/golden/make_fullsize.py to produce the committed C5 (1 GiB) digests,
 * and by tests/test_oracle_golden.py, which pins it to the reference's own
 * digests and to the int64 oracle.  The product library never links it.
 *
 * Same algorithm and same results as repeatscan_oracle.c (which restates
 * /root/reference/pkg/src/repeatscan line by line), with uint32 arrays so
 * that a 1 GiB text fits in 62 GB of host RAM (~21 B/symbol peak instead of
 * ~64), and with every reference-layout int64 array produced in chunks so
 * Python can stream it into sha256 without materialising it:
 *   o32_sa        suffixes.py:31-53 prefix doubling (argsort of bytes, dense
 *                 ranks, per round key2 = rank[i+k] or -1 -> lexsort((key2,
 *                 rank)) as two stable counting sorts -> dense re-rank)
 *   o32_lcp       suffixes.py:63-65 rank inversion + kasai_lcp
 *                 (_kernels_numba.py:15-30)
 *   o32_raw       fill_raw_llr (_kernels_numba.py:33-38)
 *   o32_compact   compact_sequential (_kernels_numba.py:58-71) == flags ->
 *                 prefix_sum -> scatter (llr.py:119-123)
 *   o32_chunk     int64 ref-layout slices of sa/rank/lcp/raw/flags/starts/lengths
 *   o32_leftmost  leftmost_compact_chunk (_kernels_numba.py:105-118)
 *   o32_all_count all_compact_count_chunk (_kernels_numba.py:158-177)
 *   o32_all_fill  all_compact_fill_chunk (_kernels_numba.py:180-195)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;
typedef uint32_t u32;

typedef struct {
    i64 n;
    const uint8_t *data;
    u32 *sa;   /* 0-based SA, n entries */
    u32 *rank; /* 1-based rank of text position i+1 at [i], n entries */
    u32 *lcp;  /* reference layout lcp[0..n+1] */
    u32 *raw;  /* raw[0..n] */
    u32 *cs, *cl;
    i64 m;
} o32;

o32 *o32_create(const uint8_t *data, i64 n) {
    o32 *h = (o32 *)calloc(1, sizeof(o32));
    if (!h) return NULL;
    h->n = n;
    h->data = data;
    return h;
}

void o32_destroy(o32 *h) {
    if (!h) return;
    free(h->sa); free(h->rank); free(h->lcp); free(h->raw); free(h->cs); free(h->cl);
    free(h);
}

/* stable counting sort of in[] by key[in[t]] (dense in [0, nkeys)) */
static void csort(const u32 *key, u32 nkeys, const u32 *in, u32 *out, i64 n, u32 *cnt) {
    memset(cnt, 0, sizeof(u32) * ((size_t)nkeys + 1));
    for (i64 t = 0; t < n; ++t) cnt[key[in[t]] + 1]++;
    for (u32 b = 1; b <= nkeys; ++b) cnt[b] += cnt[b - 1];
    for (i64 t = 0; t < n; ++t) out[cnt[key[in[t]]]++] = in[t];
}

/* suffixes.py:31-53; returns the number of doubling rounds, -1 on OOM */
int o32_sa(o32 *h) {
    i64 n = h->n;
    const uint8_t *data = h->data;
    if (n <= 0) return 0;
    u32 *order = (u32 *)malloc(sizeof(u32) * (size_t)n);
    u32 *rank = (u32 *)malloc(sizeof(u32) * (size_t)n);
    u32 *key2 = (u32 *)malloc(sizeof(u32) * (size_t)n);
    u32 *tmp = (u32 *)malloc(sizeof(u32) * (size_t)n);
    u32 *cnt = (u32 *)malloc(sizeof(u32) * ((size_t)n + 2));
    if (!order || !rank || !key2 || !tmp || !cnt) {
        free(order); free(rank); free(key2); free(tmp); free(cnt);
        return -1;
    }
    { /* :34 stable argsort of the bytes */
        i64 c256[257];
        memset(c256, 0, sizeof(c256));
        for (i64 i = 0; i < n; ++i) c256[data[i] + 1]++;
        for (int b = 1; b <= 256; ++b) c256[b] += c256[b - 1];
        for (i64 i = 0; i < n; ++i) order[c256[data[i]]++] = (u32)i;
    }
    { /* :35-38 dense ranks */
        u32 r = 0;
        rank[order[0]] = 0;
        for (i64 t = 1; t < n; ++t) {
            if (data[order[t]] != data[order[t - 1]]) ++r;
            rank[order[t]] = r;
        }
    }
    int rounds = 0;
    i64 k = 1;
    while ((i64)rank[order[n - 1]] != n - 1) { /* :40 */
        /* :41-42 key2 = rank[i+k] or -1 past the end, shifted by +1 */
#pragma omp parallel for schedule(static)
        for (i64 i = 0; i < n; ++i) key2[i] = (i + k < n) ? rank[i + k] + 1 : 0;
        /* :43 lexsort((key2, rank)): stable by key2 over index order, then by rank */
        for (i64 i = 0; i < n; ++i) tmp[i] = (u32)i;
        csort(key2, (u32)(n + 1), tmp, order, n, cnt);
        csort(rank, (u32)n, order, tmp, n, cnt);
        memcpy(order, tmp, sizeof(u32) * (size_t)n);
        /* :44-51 dense re-rank on (rank, key2) changes */
        u32 r = 0;
        tmp[order[0]] = 0;
        for (i64 t = 1; t < n; ++t) {
            u32 a = order[t], b = order[t - 1];
            if (rank[a] != rank[b] || key2[a] != key2[b]) ++r;
            tmp[a] = r;
        }
        memcpy(rank, tmp, sizeof(u32) * (size_t)n);
        k *= 2; /* :52 */
        ++rounds;
    }
    free(rank); free(key2); free(tmp); free(cnt);
    h->sa = order;
    return rounds;
}

/* suffixes.py:63-65: rank by inversion, kasai_lcp (_kernels_numba.py:15-30) */
int o32_lcp(o32 *h) {
    i64 n = h->n;
    h->rank = (u32 *)malloc(sizeof(u32) * (size_t)(n > 0 ? n : 1));
    h->lcp = (u32 *)calloc((size_t)n + 2, sizeof(u32));
    if (!h->rank || !h->lcp) return -1;
    if (n <= 0) return 0;
    const u32 *sa = h->sa;
    u32 *rank = h->rank, *lcp = h->lcp;
    const uint8_t *data = h->data;
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < n; ++j) rank[sa[j]] = (u32)(j + 1);
    i64 hh = 0;
    for (i64 i = 1; i <= n; ++i) {
        i64 r = rank[i - 1];
        if (r == 1) { hh = 0; continue; }
        i64 j = (i64)sa[r - 2] + 1; /* sa[r-1] in 1-based terms */
        while (i + hh <= n && j + hh <= n && data[i + hh - 1] == data[j + hh - 1]) ++hh;
        lcp[r] = (u32)hh;
        if (hh > 0) --hh;
    }
    return 0;
}

/* fill_raw_llr (_kernels_numba.py:33-38) */
int o32_raw(o32 *h) {
    i64 n = h->n;
    h->raw = (u32 *)calloc((size_t)n + 1, sizeof(u32));
    if (!h->raw) return -1;
    const u32 *rank = h->rank, *lcp = h->lcp;
    u32 *raw = h->raw;
#pragma omp parallel for schedule(static)
    for (i64 i = 1; i <= n; ++i) {
        u32 a = lcp[rank[i - 1]], b = lcp[rank[i - 1] + 1];
        raw[i] = a > b ? a : b;
    }
    return 0;
}

void o32_free_structures(o32 *h) {
    free(h->sa); free(h->rank); free(h->lcp);
    h->sa = h->rank = h->lcp = NULL;
}

/* compact_sequential (_kernels_numba.py:58-71); returns m or -1 */
i64 o32_compact(o32 *h) {
    i64 n = h->n, m = 0;
    const u32 *raw = h->raw;
    for (i64 i = 1; i <= n; ++i) m += (raw[i] > 0 && raw[i] >= raw[i - 1]);
    h->cs = (u32 *)malloc(sizeof(u32) * (size_t)(m > 0 ? m : 1));
    h->cl = (u32 *)malloc(sizeof(u32) * (size_t)(m > 0 ? m : 1));
    if (!h->cs || !h->cl) return -1;
    i64 j = 0;
    u32 prev = 0;
    for (i64 i = 1; i <= n; ++i) {
        u32 len = raw[i];
        if (len > 0 && len >= prev) { h->cs[j] = (u32)i; h->cl[j] = len; ++j; }
        prev = len;
    }
    h->m = m;
    return m;
}

enum { W_SA = 0, W_RANK, W_LCP, W_RAW, W_FLAGS, W_CSTARTS, W_CLENGTHS };

/* int64 reference-layout slice [lo, lo+count) of one array */
int o32_chunk(const o32 *h, int which, i64 lo, i64 count, i64 *out) {
    i64 n = h->n;
#pragma omp parallel for schedule(static)
    for (i64 t = 0; t < count; ++t) {
        i64 j = lo + t, v = 0;
        switch (which) {
        case W_SA: v = j == 0 ? 0 : (i64)h->sa[j - 1] + 1; break;
        case W_RANK: v = j == 0 ? 0 : (i64)h->rank[j - 1]; break;
        case W_LCP: v = (i64)h->lcp[j]; break;
        case W_RAW: v = (i64)h->raw[j]; break;
        case W_FLAGS: v = j == 0 ? 0 : (h->raw[j] > 0 && h->raw[j] >= h->raw[j - 1]); break;
        case W_CSTARTS: v = (i64)h->cs[j]; break;
        case W_CLENGTHS: v = (i64)h->cl[j]; break;
        }
        out[t] = v;
    }
    (void)n;
    return 0;
}

/* _first_end_at_or_after (_kernels_numba.py:74-85), ends = starts + lengths - 1 */
static i64 first_end(const o32 *h, i64 k) {
    i64 lo = 0, hi = h->m;
    while (lo < hi) {
        i64 mid = (lo + hi) / 2;
        if ((i64)h->cs[mid] + (i64)h->cl[mid] - 1 < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* leftmost_compact_chunk (_kernels_numba.py:105-118) for k in [lo, hi) */
void o32_leftmost(const o32 *h, i64 lo, i64 hi, i64 *starts, i64 *lengths) {
#pragma omp parallel for schedule(dynamic, 4096)
    for (i64 k = lo; k < hi; ++k) {
        i64 bs = -1, bl = 0;
        for (i64 t = first_end(h, k); t < h->m && (i64)h->cs[t] <= k; ++t)
            if ((i64)h->cl[t] > bl) { bl = h->cl[t]; bs = h->cs[t]; }
        starts[k - lo] = bs;
        lengths[k - lo] = bl;
    }
}

/* all_compact_count_chunk (_kernels_numba.py:158-177) for k in [lo, hi) */
void o32_all_count(const o32 *h, i64 lo, i64 hi, i64 *lengths, i64 *counts) {
#pragma omp parallel for schedule(dynamic, 4096)
    for (i64 k = lo; k < hi; ++k) {
        i64 best = 0, t0 = first_end(h, k), cnt = 0;
        for (i64 t = t0; t < h->m && (i64)h->cs[t] <= k; ++t)
            if ((i64)h->cl[t] > best) best = h->cl[t];
        if (best > 0)
            for (i64 t = t0; t < h->m && (i64)h->cs[t] <= k; ++t)
                if ((i64)h->cl[t] == best) ++cnt;
        lengths[k - lo] = best;
        counts[k - lo] = cnt;
    }
}

/* all_compact_fill_chunk (_kernels_numba.py:180-195): local_offsets[k - lo]
 * is the chunk-relative offset of position k's block */
void o32_all_fill(const o32 *h, i64 lo, i64 hi, const i64 *lengths, const i64 *local_offsets,
                  i64 *flat) {
#pragma omp parallel for schedule(dynamic, 4096)
    for (i64 k = lo; k < hi; ++k) {
        i64 len = lengths[k - lo];
        if (len == 0) continue;
        i64 idx = local_offsets[k - lo];
        for (i64 t = first_end(h, k); t < h->m && (i64)h->cs[t] <= k; ++t)
            if ((i64)h->cl[t] == len) flat[idx++] = h->cs[t];
    }
}
