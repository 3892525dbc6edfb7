// suffix_array.cu -- on-device suffix array, rank (ISA) and LCP (north-star subsystem 1).
//
// Reference: suffixes.py:31-53 (prefix doubling with np.argsort/np.lexsort),
// suffixes.py:64 (rank inversion), _kernels_numba.py:15-30 (Kasai LCP).
//
// B200 design (prefix doubling with group-head ranks, Larsson-Sadakane style):
//   round 0: every suffix gets a packed key of its first K symbols, each an
//            order-preserving code 1..sigma (0 = past the end) of b bits,
//            K = floor(64 / b)  (DNA: b = 3, K = 21; sigma<=127: K = 9; bytes: K = 7).
//            One LSD radix sort of (key, position) pairs gives the SA order.
//   k_update: SA/ISA write-back, ISA = SA index of the suffix's group head
//            (single-pass max-scan with look-back) and compaction of the
//            still-unsorted positions (sum-scan with look-back) in ONE kernel.
//   round r>=1 (h = K * 2^(r-1)): only unsorted suffixes get a key
//            (ISA[i], ISA[i+h]+1 or 0 past the end) and are re-sorted; their
//            groups occupy the same SA slots, so results write straight back.
//   Rank = ISA (ranks are the final group heads), inversion is free.
//   LCP: Phi array (scatter), PLCP by Kasai's carry over text-order chunks
//   with 8-byte word compares, then LCP[r] = PLCP[SA[r]] (gather).
// Device layouts: sa/isa u32[n] 0-based; lcp_d u32[n+2] with lcp_d[r] =
// reference lcp[r+1] (lcp_d[0] = lcp_d[n] = 0).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace rsb {

size_t raw_slots(long long n);

namespace {

constexpr unsigned kNone = 0xffffffffu;

struct CodeTable {
    unsigned short code[256];  // 1..sigma; sigma may be 256, so 9 bits
};

__global__ void k_byte_hist(const unsigned char *__restrict__ text, long long n,
                            unsigned long long *__restrict__ hist) {
    __shared__ unsigned s[256];
    s[threadIdx.x] = 0;
    __syncthreads();
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&s[text[i]], 1u);
    __syncthreads();
    if (s[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)s[threadIdx.x]);
}

// key[i] = sum_j code(text[i+j]) << (b*(K-1-j)), j < K, code 0 past the end.
__global__ void __launch_bounds__(256) k_init_keys(const unsigned char *__restrict__ text, long long n, CodeTable ct,
                                                   int b, int K, u64 *__restrict__ keys,
                                                   unsigned *__restrict__ vals) {
    __shared__ unsigned short s[256 + 64];
    long long base = blockIdx.x * 256ll;
    for (int j = threadIdx.x; j < 256 + K; j += 256) {
        long long p = base + j;
        s[j] = p < n ? ct.code[text[p]] : 0;
    }
    __syncthreads();
    long long i = base + threadIdx.x;
    if (i >= n) return;
    u64 key = 0;
    for (int j = 0; j < K; ++j) key = (key << b) | s[threadIdx.x + j];
    keys[i] = key;
    vals[i] = (unsigned)i;
}

// Round r >= 1 keys for the unsorted positions P[0..U).
__global__ void k_make_keys(const unsigned *__restrict__ P, long long U, const unsigned *__restrict__ sa,
                            const unsigned *__restrict__ isa, long long n, long long h,
                            u64 *__restrict__ keys, unsigned *__restrict__ vals) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= U) return;
    unsigned i = sa[P[t]];
    u64 hi = isa[i];
    u64 lo = ((long long)i + h < n) ? (u64)isa[i + h] + 1 : 0;
    keys[t] = hi * (u64)(n + 1) + lo;
    vals[t] = i;
}

constexpr int kUNT = 256;
constexpr int kUIPT = 8;
constexpr int kUTile = kUNT * kUIPT;

// Write back one sorted run of (key, suffix) pairs occupying SA slots Pos(t)
// (P[t], or t when P is null): sa[Pos(t)] = suffix, isa[suffix] = SA slot of
// its new group head, and the positions still in non-singleton groups are
// compacted into P_next.
__global__ void __launch_bounds__(kUNT) k_update(const u64 *__restrict__ keys, const unsigned *__restrict__ vals,
                                                 const unsigned *__restrict__ P, long long U,
                                                 unsigned *__restrict__ sa, unsigned *__restrict__ isa,
                                                 unsigned *__restrict__ P_next,
                                                 unsigned long long *U_next, unsigned *counter,
                                                 u64 *status_max, u64 *status_sum, long long tiles) {
    __shared__ unsigned s_tile;
    __shared__ u64 s_warp[kUNT / 32];
    __shared__ unsigned s_warp32[kUNT / 32];
    __shared__ u64 s_head_prefix;
    __shared__ u64 s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const int lane = threadIdx.x & 31;
    const long long t0 = tile * kUTile + (long long)threadIdx.x * kUIPT;
    u64 k[kUIPT];
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) k[j] = (t0 + j < U) ? keys[t0 + j] : ~0ull;
    u64 kprev = __shfl_up_sync(0xffffffffu, k[kUIPT - 1], 1);
    u64 knext = __shfl_down_sync(0xffffffffu, k[0], 1);
    if (lane == 0) kprev = (t0 > 0 && t0 - 1 < U) ? keys[t0 - 1] : 0;
    if (lane == 31) knext = (t0 + kUIPT < U) ? keys[t0 + kUIPT] : 0;
    bool newf[kUIPT + 1];
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        newf[j] = (t == 0) || (k[j] != (j ? k[j - 1] : kprev));
    }
    newf[kUIPT] = (t0 + kUIPT >= U) || (knext != k[kUIPT - 1]);
    // last valid element's successor flag
#pragma unroll
    for (int j = 0; j < kUIPT; ++j)
        if (t0 + j + 1 == U) newf[j + 1] = true;

    unsigned pos[kUIPT];
    u64 hmax = 0;
    unsigned unsorted = 0, ucnt = 0;
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        if (t < U) {
            pos[j] = P ? P[t] : (unsigned)t;
            if (newf[j]) hmax = (u64)pos[j];
            bool un = !(newf[j] && newf[j + 1]);
            unsorted |= (unsigned)un << j;
            ucnt += un;
        }
    }
    // heads: inclusive max-scan across the block, then look-back over tiles
    u64 incl;
    u64 tile_max = block_inclusive_max64<kUNT>(hmax, incl, s_warp);
    u64 excl_in_block = __shfl_up_sync(0xffffffffu, incl, 1);
    // inclusive of previous thread within the block:
    // (block_inclusive_max64 returned this thread's inclusive value; derive the
    //  exclusive one for thread 0 of each warp from the warp totals.)
    unsigned excl_u;
    unsigned utotal = block_exclusive_sum<kUNT>(ucnt, excl_u, s_warp32);
    if (threadIdx.x < 32) {
        u64 hp = lookback_warp(status_max, tile, tile_max, OpMax());
        u64 up = lookback_warp(status_sum, tile, (u64)utotal, OpSum());
        if (threadIdx.x == 0) {
            s_head_prefix = hp;
            s_base = up;
            if (tile == tiles - 1) *U_next = up + utotal;
        }
    }
    __syncthreads();
    // exclusive max for this thread = max(tile prefix, inclusive value of previous thread)
    u64 run = s_head_prefix;
    {
        const int warp = threadIdx.x >> 5;
        u64 prev_incl;
        if (lane > 0) prev_incl = excl_in_block;
        else prev_incl = warp ? s_warp[warp - 1] : 0;
        if (threadIdx.x > 0 && prev_incl > run) run = prev_incl;
    }
    u64 o = s_base + excl_u;
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        if (t >= U) break;
        if (newf[j]) run = pos[j];
        unsigned v = vals[t];
        sa[pos[j]] = v;
        isa[v] = (unsigned)run;
        if (unsorted >> j & 1) P_next[o++] = pos[j];
    }
}

// phi[sa[j]] = sa[j-1] (kNone for j = 0)
__global__ void k_phi(const unsigned *__restrict__ sa, long long n, unsigned *__restrict__ phi) {
    long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j >= n) return;
    phi[sa[j]] = j ? sa[j - 1] : kNone;
}

__device__ __forceinline__ u64 load8(const unsigned char *t, long long p) {
    const u64 *w = reinterpret_cast<const u64 *>(t + (p & ~7ll));
    unsigned sh = (unsigned)(p & 7) * 8;
    u64 lo = __ldg(w), hi = __ldg(w + 1);
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

// Kasai over text-order chunks: PLCP[i] = lcp(i, phi[i]); carry h-1 within a chunk.
__global__ void k_plcp(const unsigned char *__restrict__ text, const unsigned *__restrict__ phi, long long n,
                       long long chunk, unsigned *__restrict__ plcp) {
    long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long i0 = c * chunk;
    if (i0 >= n) return;
    long long i1 = i0 + chunk < n ? i0 + chunk : n;
    long long h = 0;
    for (long long i = i0; i < i1; ++i) {
        unsigned j = phi[i];
        if (j == kNone) {
            h = 0;
            plcp[i] = 0;
            continue;
        }
        long long lim = n - (i > (long long)j ? i : (long long)j);  // min remaining length
        while (h < lim) {
            u64 x = load8(text, i + h) ^ load8(text, (long long)j + h);
            if (x == 0) {
                h += 8;
            } else {
                h += (__ffsll((long long)x) - 1) >> 3;
                break;
            }
        }
        if (h > lim) h = lim;
        plcp[i] = (unsigned)h;
        if (h > 0) --h;
    }
}

// lcp_d[r] = PLCP[sa[r]] for 1 <= r < n; lcp_d[0] = lcp_d[n] = lcp_d[n+1] = 0.
__global__ void k_lcp_gather(const unsigned *__restrict__ sa, const unsigned *__restrict__ plcp, long long n,
                             unsigned *__restrict__ lcp_d) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r > n + 1) return;
    lcp_d[r] = (r == 0 || r >= n) ? 0u : plcp[sa[r]];
}

}  // namespace

void build_suffix_array(rs_ctx *c, long long n) {
    const unsigned char *text = (const unsigned char *)c->bufs[B_TEXT].p;
    unsigned *sa = (unsigned *)buf(c, B_SA, sizeof(unsigned) * (size_t)(n + 4));
    unsigned *isa = (unsigned *)buf(c, B_ISA, sizeof(unsigned) * (size_t)(n + 4));
    c->sa_rounds = 0;
    if (n <= 0) return;
    // alphabet -> order-preserving codes 1..sigma
    unsigned long long *hist = (unsigned long long *)buf(c, B_HIST, sizeof(unsigned long long) * 8 * 256);
    RS_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 256, c->stream));
    unsigned hb = (unsigned)std::min<long long>((n + 256 * 64 - 1) / (256 * 64), c->sm_count * 4);
    RS_LAUNCH(c, k_byte_hist, hb, 256, 0, text, n, hist);
    std::vector<unsigned long long> h(256);
    fetch_small(c, h.data(), hist, sizeof(unsigned long long) * 256);
    CodeTable ct;
    int sigma = 0;
    for (int b = 0; b < 256; ++b) ct.code[b] = h[b] ? (unsigned short)(++sigma) : 0;
    int bits = 1;
    while ((1 << bits) < sigma + 1) ++bits;
    int K = 64 / bits;

    u64 *k0 = (u64 *)buf(c, B_KEYS0, sizeof(u64) * (size_t)n);
    u64 *k1 = (u64 *)buf(c, B_KEYS1, sizeof(u64) * (size_t)n);
    unsigned *v0 = (unsigned *)buf(c, B_VALS0, sizeof(unsigned) * (size_t)n);
    unsigned *v1 = (unsigned *)buf(c, B_VALS1, sizeof(unsigned) * (size_t)n);
    unsigned *Pa = (unsigned *)buf(c, B_T0, sizeof(unsigned) * (size_t)n);
    unsigned *Pb = (unsigned *)buf(c, B_T1, sizeof(unsigned) * (size_t)n);
    unsigned long long *u_dev = (unsigned long long *)buf(c, B_SMALL, 4096) + 4;

    RS_LAUNCH(c, k_init_keys, grid_for(n, 256), 256, 0, text, n, ct, bits, K, k0, v0);
    u64 *ks;
    unsigned *vs;
    radix_sort_pairs(c, k0, k1, v0, v1, n, bits * K, &ks, &vs);

    long long U = n;
    const unsigned *P = nullptr;
    long long depth = K;
    // bits of a round key hi*(n+1)+lo < n*(n+1)
    int rbits = (int)std::ceil(std::log2((double)n * (double)(n + 1)));
    if (rbits < 1) rbits = 1;
    while (true) {
        ++c->sa_rounds;
        long long tiles = (U + kUTile - 1) / kUTile;
        Scratch s = scratch(c, 2 * tiles);
        RS_LAUNCH(c, k_update, (unsigned)tiles, kUNT, 0, ks, vs, P, U, sa, isa, Pa, u_dev, s.counter, s.status,
                  s.status + tiles, tiles);
        unsigned long long un = 0;
        fetch_small(c, &un, u_dev, sizeof(un));
        U = (long long)un;
        if (U == 0) break;
        if (depth >= n) fail(RS_ECUDA, "suffix sort did not converge");
        std::swap(Pa, Pb);  // Pb now holds the unsorted list
        P = Pb;
        RS_LAUNCH(c, k_make_keys, grid_for(U, 256), 256, 0, P, U, sa, isa, n, depth, k0, v0);
        radix_sort_pairs(c, k0, k1, v0, v1, U, rbits, &ks, &vs);
        depth *= 2;
    }
}

void build_lcp(rs_ctx *c, long long n) {
    unsigned *lcp_d = (unsigned *)buf(c, B_LCP, sizeof(unsigned) * (size_t)(n + 4));
    if (n <= 0) {
        RS_CUDA(cudaMemsetAsync(lcp_d, 0, sizeof(unsigned) * 4, c->stream));
        return;
    }
    const unsigned char *text = (const unsigned char *)c->bufs[B_TEXT].p;
    const unsigned *sa = (const unsigned *)c->bufs[B_SA].p;
    unsigned *phi = (unsigned *)buf(c, B_PHI, sizeof(unsigned) * (size_t)n);
    unsigned *plcp = (unsigned *)buf(c, B_PLCP, sizeof(unsigned) * (size_t)n);
    RS_LAUNCH(c, k_phi, grid_for(n, 256), 256, 0, sa, n, phi);
    long long chunk = std::max<long long>(32, n >> 19);
    long long chunks = (n + chunk - 1) / chunk;
    RS_LAUNCH(c, k_plcp, grid_for(chunks, 128), 128, 0, text, phi, n, chunk, plcp);
    RS_LAUNCH(c, k_lcp_gather, grid_for(n + 2, 256), 256, 0, sa, plcp, n, lcp_d);
}

}  // namespace rsb
