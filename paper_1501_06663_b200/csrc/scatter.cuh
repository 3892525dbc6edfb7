// scatter.cuh -- bucketed permutation scatter (see scatter.cu).
#pragma once
#include "common.cuh"

namespace rsb {

constexpr int kMaxBuckets = 256;
constexpr unsigned kNoDest = 0xffffffffu;
// one cursor per 128-byte line: the per-(block, bucket) atomics of different
// buckets then go to different L2 slices instead of serialising on one line
constexpr int kCursorStride = 32;

struct BucketEmit {
    uint2 *stage;       // (dest, val) pairs, bucket b owns [b << shift, (b + 1) << shift)
    unsigned *cursor;   // per-bucket fill counts
    int shift;
    long long nb;
    unsigned *stage2;   // optional second value per pair (same slot), or null
};

// Shared memory for bucket_emit with NT threads x IPT items.
template <int NT, int IPT>
struct EmitSmem {
    unsigned cnt[kMaxBuckets];           // block bucket counts
    unsigned bstart[kMaxBuckets];        // block-local start of each bucket run
    unsigned gbase[kMaxBuckets];         // global slot reserved for the block's run
    unsigned dest[NT * IPT];             // items exchanged into bucket order
    unsigned val[NT * IPT];
    unsigned val2[NT * IPT];
    unsigned warp_tot[NT / 32];
};

// Phase 1, called by every thread of a 256-thread block (contains
// __syncthreads): append this thread's IPT (dest, val[, val2]) items (dest ==
// kNoDest: none) to their buckets.  Order inside a bucket is free, so items are
// ranked with one shared atomic each (no MATCH, no per-warp counter
// chain), one global atomicAdd per (block, bucket), and an
// exchange through shared memory so each bucket's run is written by
// consecutive threads (coalesced) instead of one scattered store per item.
template <int NT, int IPT>
__device__ __forceinline__ void bucket_emit(const BucketEmit &be, const unsigned *dest, const unsigned *val,
                                            EmitSmem<NT, IPT> &sm, const unsigned *val2 = nullptr) {
    static_assert(NT == 256, "one thread per bucket");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    sm.cnt[threadIdx.x] = 0;
    __syncthreads();
    unsigned short rank[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j)
        if (dest[j] != kNoDest) rank[j] = (unsigned short)atomicAdd(&sm.cnt[dest[j] >> be.shift], 1u);
    __syncthreads();
    {
        const int b = threadIdx.x;
        const unsigned run = sm.cnt[b];
        // block-exclusive scan of the bucket totals (bucket order)
        unsigned x = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sm.warp_tot[warp] = x;
        __syncthreads();
        unsigned wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += sm.warp_tot[w];
        sm.bstart[b] = wbase + x - run;
        if (b < be.nb && run) sm.gbase[b] = atomicAdd(&be.cursor[b * kCursorStride], run);
    }
    __syncthreads();
    unsigned total = 0;
    for (int w = 0; w < NT / 32; ++w) total += sm.warp_tot[w];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (dest[j] == kNoDest) continue;
        const unsigned b = dest[j] >> be.shift;
        const unsigned p = sm.bstart[b] + rank[j];
        sm.dest[p] = dest[j];
        sm.val[p] = val[j];
        if (val2) sm.val2[p] = val2[j];
    }
    __syncthreads();
    for (unsigned i = threadIdx.x; i < total; i += NT) {
        const unsigned d = sm.dest[i];
        const unsigned b = d >> be.shift;
        const unsigned within = sm.gbase[b] + (i - sm.bstart[b]);
        // dest not injective (caller data): never write past the bucket's region
        if (within >> be.shift) continue;
        const long long slot = ((long long)b << be.shift) + within;
        be.stage[slot] = make_uint2(d, sm.val[i]);
        if (val2) be.stage2[slot] = sm.val2[i];
    }
}

BucketEmit bucket_setup(rs_ctx *c, long long n_out, int slot = 0, bool two = false);
// out[dest] = val; if out2: out2[dest + out2_shift] = val2 (second stage array).
void bucket_apply(rs_ctx *c, const BucketEmit &be, unsigned *out, long long elems, unsigned *out2 = nullptr,
                  int out2_shift = 0);
void raw_from_sa_lcp(rs_ctx *c, long long n, size_t raw_slots_n);
void raw_from_sa_lcp_range(rs_ctx *c, long long n, size_t raw_slots_n, long long first, long long last);
// phi[sa[j]] = sa[j-1] (0xffffffff at j = 0) through the bucketed scatter.
void scatter_phi(rs_ctx *c, const unsigned *sa, long long n, unsigned *phi);
// isa[sa[r]] = r through the bucketed scatter.
void scatter_rank(rs_ctx *c, const unsigned *sa, long long n, unsigned *isa);
// isa == inverse permutation of sa (0-based, n entries)?
bool check_rank_inverse(rs_ctx *c, const unsigned *sa, const unsigned *isa, long long n);
// out[dest[i]] = val[i], i < n; dest a permutation into [0, n_out).
void scatter_by(rs_ctx *c, const unsigned *dest, const unsigned *val, long long n, unsigned *out, long long n_out);

}  // namespace rsb
