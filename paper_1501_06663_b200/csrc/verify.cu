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

}  // namespace

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
