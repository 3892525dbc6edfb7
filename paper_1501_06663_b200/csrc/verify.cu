// verify.cu -- on-device check of suffix structures (suffixes.py:69-103).
//
// The reference verifier is an O(n^2) host loop: sa is a permutation of
// 1..n, rank[sa[j]] == j, and for every adjacent pair (sa[j-1], sa[j]) the
// stored lcp equals the common-prefix length and the suffixes are in strict
// lexicographic order (mismatch byte decides; otherwise the shorter suffix,
// the one that ran out, comes first).  Here every check is one thread per j.
#include "common.cuh"

namespace rsb {

namespace {

__device__ __forceinline__ u64 vload8(const unsigned char *t, long long p) {
    const u64 *w = reinterpret_cast<const u64 *>(t + (p & ~7ll));
    unsigned sh = (unsigned)(p & 7) * 8;
    u64 lo = w[0], hi = w[1];
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

__global__ void k_mark(const long long *__restrict__ sa, long long n, unsigned *__restrict__ seen,
                       unsigned *err) {
    long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1;
    if (j > n) return;
    long long p = sa[j];
    if (p < 1 || p > n) {
        atomicOr(err, 1u);
        return;
    }
    atomicAdd(&seen[p], 1u);
}

__global__ void k_check(const unsigned char *__restrict__ text, const long long *__restrict__ sa,
                        const long long *__restrict__ rank, const long long *__restrict__ lcp, long long n,
                        const unsigned *__restrict__ seen, unsigned *err) {
    long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1;
    if (j > n) return;
    if (seen[j] != 1) {
        atomicOr(err, 1u);
        return;
    }
    long long p = sa[j];
    if (rank[p] != j) {
        atomicOr(err, 1u);
        return;
    }
    if (j < 2) return;
    long long a = sa[j - 1] - 1, b = p - 1;
    long long lim = n - (a > b ? a : b);
    long long h = 0;
    while (h < lim) {
        u64 x = vload8(text, a + h) ^ vload8(text, b + h);
        if (x == 0) {
            h += 8;
        } else {
            h += (__ffsll((long long)x) - 1) >> 3;
            break;
        }
    }
    if (h > lim) h = lim;
    if (lcp[j] != h) {
        atomicOr(err, 1u);
        return;
    }
    if (a + h < n && b + h < n) {
        if (text[a + h] >= text[b + h]) atomicOr(err, 1u);
    } else if (a + h < n) {
        atomicOr(err, 1u);
    }
}

// Independent answer checker (the reference's Algorithm 4 taken literally,
// _kernels_numba.py:74-85 + :158-195): one thread per position k binary
// searches the first compact entry whose end reaches k, walks the window
// forward while start <= k, and checks that the results claim exactly the
// maximum length over the window (lengths), exactly the entries of that
// length in increasing start order (offsets, flat) and, when given, the
// first of them as the leftmost answer.  Shares no code with the scan
// kernels of scan_query.cu (no window bounds, no staging, no tile lists).
__global__ void k_check_answers(const long long *__restrict__ cs, const long long *__restrict__ cl,
                                long long m, long long n, const long long *__restrict__ L,
                                const long long *__restrict__ O, const long long *__restrict__ F,
                                long long T, const long long *__restrict__ ls,
                                const long long *__restrict__ ll, unsigned long long *bad) {
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1;
    if (k > n) return;
    long long lo = 0, hi = m;
    while (lo < hi) {
        long long mid = (lo + hi) >> 1;
        if (cs[mid] + cl[mid] - 1 < k) lo = mid + 1; else hi = mid;
    }
    long long best = 0, first = -1;
    for (long long t = lo; t < m && cs[t] <= k; ++t)
        if (cl[t] > best) { best = cl[t]; first = cs[t]; }
    bool ok = true;
    if (L) {
        ok = L[k] == best;
        long long o0 = O[k], o1 = O[k + 1];
        ok = ok && 0 <= o0 && o0 <= o1 && o1 <= T;
        if (ok) {
            long long idx = o0;
            if (best > 0)
                for (long long t = lo; t < m && cs[t] <= k && ok; ++t)
                    if (cl[t] == best) ok = idx < o1 && F[idx++] == cs[t];
            ok = ok && idx == o1;
        }
        if (k == 1) ok = ok && O[0] == 0 && O[1] == 0 && L[0] == 0;
        if (k == n) ok = ok && O[n + 1] == T;
    }
    if (ls) {
        ok = ok && ls[k] == first && ll[k] == best;
        if (k == 1) ok = ok && ls[0] == -1 && ll[0] == 0;
    }
    if (!ok) atomicAdd(bad, 1ull);
}

}  // namespace

long long check_answers(rs_ctx *c, const long long *d_cs, const long long *d_cl, long long m, long long n,
                        const long long *d_L, const long long *d_O, const long long *d_F, long long T,
                        const long long *d_ls, const long long *d_ll) {
    if (n <= 0) return 0;
    unsigned long long *bad = (unsigned long long *)((char *)buf(c, B_SMALL, 4096) + 256);
    RS_CUDA(cudaMemsetAsync(bad, 0, sizeof(*bad), c->stream));
    RS_LAUNCH(c, k_check_answers, grid_for(n, 256), 256, 0, d_cs, d_cl, m, n, d_L, d_O, d_F, T, d_ls, d_ll,
              bad);
    unsigned long long h = 0;
    fetch_small(c, &h, bad, sizeof(h));
    return (long long)h;
}

bool verify_structures(rs_ctx *c, const unsigned char *d_text, long long n, const long long *d_sa,
                       const long long *d_rank, const long long *d_lcp) {
    if (n <= 0) return true;
    unsigned *seen = (unsigned *)buf(c, B_T0, sizeof(unsigned) * (size_t)(n + 1));
    RS_CUDA(cudaMemsetAsync(seen, 0, sizeof(unsigned) * (size_t)(n + 1), c->stream));
    unsigned *err = (unsigned *)((char *)buf(c, B_SMALL, 4096) + 128);
    RS_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned), c->stream));
    RS_LAUNCH(c, k_mark, grid_for(n, 256), 256, 0, d_sa, n, seen, err);
    unsigned h = 0;
    fetch_small(c, &h, err, sizeof(h));
    if (h) return false;
    RS_LAUNCH(c, k_check, grid_for(n, 256), 256, 0, d_text, d_sa, d_rank, d_lcp, n, seen, err);
    fetch_small(c, &h, err, sizeof(h));
    return h == 0;
}

}  // namespace rsb
