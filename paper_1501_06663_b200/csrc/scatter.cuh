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

// Phase 1, called by every thread of a 256-thread block (contains
// __syncthreads): append this thread's IPT (dest, val) pairs (dest ==
// kNoDest: none) to their buckets.  Ranking is warp-synchronous
// (match_any + per-warp counters, no shared-memory atomics); one global
// atomicAdd per (block, bucket) reserves the block's run.
// s_cnt must hold 8 * 256 u16 counters, s_base 256 u32.
template <int IPT>
__device__ __forceinline__ void bucket_emit(const BucketEmit &be, const unsigned *dest, const unsigned *val,
                                            unsigned short *s_cnt, unsigned *s_base,
                                            const unsigned *val2 = nullptr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned short *wc = s_cnt + warp * 256;
    for (int i = lane; i < 256; i += 32) wc[i] = 0;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1;
    unsigned short rank[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const bool valid = dest[j] != kNoDest;
        const unsigned b = valid ? dest[j] >> be.shift : 0x100u;
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const unsigned short before = valid ? wc[b & 0xff] : 0;
        __syncwarp();
        if (valid) {
            rank[j] = before + (unsigned short)__popc(peers & lt);
            if ((peers & lt) == 0) wc[b] = before + (unsigned short)__popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    {
        const int b = threadIdx.x;  // one thread per bucket (nb <= 256)
        if (b < be.nb) {
            unsigned run = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const unsigned c = s_cnt[w * 256 + b];
                s_cnt[w * 256 + b] = (unsigned short)run;
                run += c;
            }
            if (run) s_base[b] = atomicAdd(&be.cursor[b * kCursorStride], run);
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (dest[j] == kNoDest) continue;
        const unsigned b = dest[j] >> be.shift;
        const long long slot = ((long long)b << be.shift) + s_base[b] + wc[b] + rank[j];
        be.stage[slot] = make_uint2(dest[j], val[j]);
        if (val2) be.stage2[slot] = val2[j];
    }
}

BucketEmit bucket_setup(rs_ctx *c, long long n_out, int slot = 0, bool two = false);
// out[dest] = val; if out2: out2[dest + out2_shift] = val2 (second stage array).
void bucket_apply(rs_ctx *c, const BucketEmit &be, unsigned *out, long long elems, unsigned *out2 = nullptr,
                  int out2_shift = 0);
void raw_from_sa_lcp(rs_ctx *c, long long n, size_t raw_slots_n);

}  // namespace rsb
