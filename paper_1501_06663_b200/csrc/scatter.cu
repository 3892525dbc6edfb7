// scatter.cu -- L2-local permutation scatter: out[dest[i]] = val[i].
//
// Measured on B200 (ncu, profiles/): a random 4-byte store costs ~64 B of HBM
// traffic (sector read-modify-write) and a random 4-byte load ~128 B, so the
// two permutation steps of the path -- ISA[SA[r]] = r after the first sort
// round and raw[SA[r]] = max(LCP[r], LCP[r+1]) -- were the slowest kernels.
// Here they become two streaming passes:
//   phase 1 (fused into the producer): (dest, val) pairs are appended to
//     bucket dest >> S of a staging array.  dest is injective, so bucket b
//     holds at most 2^S pairs and owns the fixed region [b*2^S, (b+1)*2^S);
//     a block reserves its per-bucket run with one atomicAdd per bucket.
//   phase 2 (k_bucket_apply): blocks walk the staging array bucket-major, so
//     the few buckets in flight span a few MB of `out` and every random store
//     merges in L2 before its line is written back once.
// ~20 B of HBM traffic per element instead of ~64-128 B.
#include "common.cuh"
#include "scatter.cuh"

namespace rsb {

namespace {

constexpr int kApplyNT = 256;
constexpr int kApplyIPT = 4;  // tools/micro/scatter_bench.cu: 4 -> 1.42 ms, 8 -> 1.46, 16 -> 1.53 (2^28 pairs)

__global__ void __launch_bounds__(kApplyNT) k_bucket_apply(const uint2 *__restrict__ stage,
                                                           const unsigned *__restrict__ cursor, int shift,
                                                           long long chunks_per_bucket,
                                                           unsigned *__restrict__ out,
                                                           const unsigned *__restrict__ stage2,
                                                           unsigned *__restrict__ out2, int out2_shift) {
    const long long b = blockIdx.x / chunks_per_bucket;
    const long long chunk = blockIdx.x % chunks_per_bucket;
    long long count = cursor[b * kCursorStride];
    if (count > (1ll << shift)) count = 1ll << shift;  // overfull bucket: non-injective dest (caller data)
    const long long begin = chunk * (kApplyNT * kApplyIPT);
    if (begin >= count) return;
    const uint2 *src = stage + (b << shift);
    const unsigned *src2 = stage2 + (b << shift);
    uint2 v[kApplyIPT];
    unsigned w[kApplyIPT];
    // every load of the chunk in flight before the first store
#pragma unroll
    for (int j = 0; j < kApplyIPT; ++j) {
        long long i = begin + j * kApplyNT + threadIdx.x;
        v[j] = i < count ? __ldcs(src + i) : make_uint2(0xffffffffu, 0);
        if (stage2) w[j] = i < count ? __ldcs(src2 + i) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kApplyIPT; ++j)
        if (v[j].x != 0xffffffffu) out[v[j].x] = v[j].y;
    if (stage2) {
#pragma unroll
        for (int j = 0; j < kApplyIPT; ++j)
            if (v[j].x != 0xffffffffu) out2[v[j].x + out2_shift] = w[j];
    }
}

// SA-order raw LLR (device-built structures): raw[sa[r] + 1] = max(lcp_d[r], lcp_d[r+1]).
constexpr int kRNT = 256;
constexpr int kRIPT = 8;
__global__ void __launch_bounds__(kRNT) k_raw_sa_emit(const unsigned *__restrict__ sa, const unsigned *__restrict__ lcp_d,
                                                     long long n, BucketEmit be, unsigned dlo = 0,
                                                     unsigned dhi = 0xffffffffu) {
    __shared__ EmitSmem<kRNT, kRIPT> sm;
    const long long r0 = (blockIdx.x * (long long)kRNT + threadIdx.x) * kRIPT;
    unsigned dest[kRIPT], val[kRIPT];
    if (r0 + kRIPT < n && !((reinterpret_cast<uintptr_t>(sa) | reinterpret_cast<uintptr_t>(lcp_d)) & 15)) {
        // 16-byte vector loads (r0 is a multiple of 8): 5 loads instead of 17
        const uint4 s0 = *reinterpret_cast<const uint4 *>(sa + r0), s1 = *reinterpret_cast<const uint4 *>(sa + r0 + 4);
        const uint4 l0 = *reinterpret_cast<const uint4 *>(lcp_d + r0), l1 = *reinterpret_cast<const uint4 *>(lcp_d + r0 + 4);
        const unsigned l8 = lcp_d[r0 + 8];
        const unsigned sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const unsigned lv[9] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w, l8};
#pragma unroll
        for (int j = 0; j < kRIPT; ++j) {
            dest[j] = sv[j] + 1;
            val[j] = lv[j] > lv[j + 1] ? lv[j] : lv[j + 1];
        }
    } else {
#pragma unroll
        for (int j = 0; j < kRIPT; ++j) {
            long long r = r0 + j;
            if (r < n) {
                dest[j] = sa[r] + 1;
                unsigned a = lcp_d[r], c = lcp_d[r + 1];
                val[j] = a > c ? a : c;
            } else {
                dest[j] = 0xffffffffu;
            }
        }
    }
    if (dlo != 0 || dhi != 0xffffffffu) {  // a position shard: only slots [dlo, dhi]
#pragma unroll
        for (int j = 0; j < kRIPT; ++j)
            if (dest[j] < dlo || dest[j] > dhi) dest[j] = 0xffffffffu;
    }
    bucket_emit<kRNT, kRIPT>(be, dest, val, sm);
}

// 8 consecutive u32 from a 32-byte aligned address (i0 multiple of 8)
__device__ __forceinline__ void load8(const unsigned *__restrict__ a, long long i0, unsigned (&v)[8]) {
    const uint4 x = *reinterpret_cast<const uint4 *>(a + i0), y = *reinterpret_cast<const uint4 *>(a + i0 + 4);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
}

// phi[sa[j]] = sa[j-1] (kNone at j = 0), emitted in SA order.
__global__ void __launch_bounds__(kRNT) k_phi_emit(const unsigned *__restrict__ sa, long long n, BucketEmit be) {
    __shared__ EmitSmem<kRNT, kRIPT> sm;
    const long long j0 = (blockIdx.x * (long long)kRNT + threadIdx.x) * kRIPT;
    unsigned dest[kRIPT], val[kRIPT];
    if (j0 + kRIPT <= n && !(reinterpret_cast<uintptr_t>(sa) & 15)) {
        load8(sa, j0, dest);
        val[0] = j0 > 0 ? sa[j0 - 1] : 0xffffffffu;
#pragma unroll
        for (int q = 1; q < kRIPT; ++q) val[q] = dest[q - 1];
    } else {
#pragma unroll
        for (int q = 0; q < kRIPT; ++q) {
            const long long j = j0 + q;
            dest[q] = j < n ? sa[j] : kNoDest;
            val[q] = (j < n && j > 0) ? sa[j - 1] : 0xffffffffu;
        }
    }
    bucket_emit<kRNT, kRIPT>(be, dest, val, sm);
}

// isa[sa[r]] = r, emitted in SA order.
__global__ void __launch_bounds__(kRNT) k_rank_emit(const unsigned *__restrict__ sa, long long n, BucketEmit be) {
    __shared__ EmitSmem<kRNT, kRIPT> sm;
    const long long r0 = (blockIdx.x * (long long)kRNT + threadIdx.x) * kRIPT;
    unsigned dest[kRIPT], val[kRIPT];
    if (r0 + kRIPT <= n && !(reinterpret_cast<uintptr_t>(sa) & 15)) {
        load8(sa, r0, dest);
    } else {
#pragma unroll
        for (int q = 0; q < kRIPT; ++q) dest[q] = r0 + q < n ? sa[r0 + q] : kNoDest;
    }
#pragma unroll
    for (int q = 0; q < kRIPT; ++q) val[q] = (unsigned)(r0 + q);
    bucket_emit<kRNT, kRIPT>(be, dest, val, sm);
}

// out[dest[i]] = val[i] for i < n (dest a permutation of its range).
__global__ void __launch_bounds__(kRNT) k_pair_emit(const unsigned *__restrict__ dest_in,
                                                   const unsigned *__restrict__ val_in, long long n, BucketEmit be) {
    __shared__ EmitSmem<kRNT, kRIPT> sm;
    const long long i0 = (blockIdx.x * (long long)kRNT + threadIdx.x) * kRIPT;
    unsigned dest[kRIPT], val[kRIPT];
    if (i0 + kRIPT <= n && !((reinterpret_cast<uintptr_t>(dest_in) | reinterpret_cast<uintptr_t>(val_in)) & 15)) {
        load8(dest_in, i0, dest);
        load8(val_in, i0, val);
    } else {
#pragma unroll
        for (int q = 0; q < kRIPT; ++q) {
            const long long i = i0 + q;
            dest[q] = i < n ? dest_in[i] : kNoDest;
            val[q] = i < n ? val_in[i] : 0u;
        }
    }
    bucket_emit<kRNT, kRIPT>(be, dest, val, sm);
}

__global__ void k_equal_u32(const unsigned *__restrict__ a, const unsigned *__restrict__ b, long long n,
                            unsigned *err) {
    long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
    bool bad = false;
    if (i + 3 < n) {
        const uint4 x = *reinterpret_cast<const uint4 *>(a + i), y = *reinterpret_cast<const uint4 *>(b + i);
        bad = (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
    } else {
        for (; i < n; ++i) bad |= a[i] != b[i];
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

}  // namespace

// True iff isa is the inverse permutation of sa (both 0-based, n entries):
// isa'[sa[r]] = r through the bucketed scatter into a cleared buffer (holes
// and duplicates of a non-permutation stay 0xffffffff), then one coalesced
// comparison with isa.
bool check_rank_inverse(rs_ctx *c, const unsigned *sa, const unsigned *isa, long long n) {
    if (n <= 0) return true;
    unsigned *tmp = (unsigned *)buf(c, B_T0, sizeof(unsigned) * (size_t)(n + 4));
    RS_CUDA(cudaMemsetAsync(tmp, 0xff, sizeof(unsigned) * (size_t)n, c->stream));
    scatter_rank(c, sa, n, tmp);
    unsigned *err = (unsigned *)((char *)buf(c, B_SMALL, 4096) + 192);
    RS_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned), c->stream));
    RS_LAUNCH_B(c, 8.0 * n, k_equal_u32, grid_for((n + 3) / 4, 256), 256, 0, tmp, isa, n, err);
    unsigned h = 0;
    fetch_small(c, &h, err, sizeof(h));
    return h == 0;
}

BucketEmit bucket_setup(rs_ctx *c, long long n_out, int slot, bool two) {
    // <= 256 buckets: a block's items spread over few buckets (long runs), and
    // the buckets in flight during phase 2 cover a few MB of `out` (L2-resident).
    int shift = 12;
    while (((n_out + (1ll << shift) - 1) >> shift) > kMaxBuckets && shift < 30) ++shift;
    long long nb = (n_out + (1ll << shift) - 1) >> shift;
    if (nb < 1) nb = 1;
    if (nb > kMaxBuckets) fail(RS_EINVAL, "too many scatter buckets");
    uint2 *stage = (uint2 *)buf(c, slot == 0 ? B_T2 : B_T3, sizeof(uint2) * (size_t)(nb << shift));
    unsigned *cur = (unsigned *)buf(c, B_CURSOR, sizeof(unsigned) * 2 * kMaxBuckets * kCursorStride) +
                    (size_t)slot * kMaxBuckets * kCursorStride;
    RS_CUDA(cudaMemsetAsync(cur, 0, sizeof(unsigned) * (size_t)nb * kCursorStride, c->stream));
    unsigned *stage2 = two ? (unsigned *)buf(c, slot == 0 ? B_T4 : B_T5, sizeof(unsigned) * (size_t)(nb << shift))
                           : nullptr;
    return BucketEmit{stage, cur, shift, nb, stage2};
}

void bucket_apply(rs_ctx *c, const BucketEmit &be, unsigned *out, long long elems, unsigned *out2,
                  int out2_shift) {
    long long per_block = kApplyNT * kApplyIPT;
    long long chunks = ((1ll << be.shift) + per_block - 1) / per_block;
    RS_LAUNCH_B(c, (out2 ? 20.0 : 12.0) * (double)elems, k_bucket_apply, (unsigned)(be.nb * chunks), kApplyNT, 0,
                be.stage, be.cursor, be.shift, chunks, out, out2 ? be.stage2 : nullptr, out2, out2_shift);
}

// raw (B_RAW, 1-based u32) from device-built SA + SA-order LCP, via the bucketed scatter.
void raw_from_sa_lcp(rs_ctx *c, long long n, size_t raw_slots_n) {
    unsigned *raw = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots_n);
    RS_CUDA(cudaMemsetAsync(raw, 0, sizeof(unsigned), c->stream));
    BucketEmit be = bucket_setup(c, n + 1, 0);
    RS_LAUNCH_B(c, 16.0 * n, k_raw_sa_emit, grid_for((n + kRIPT - 1) / kRIPT, kRNT), kRNT, 0,
                (const unsigned *)c->bufs[B_SA].p, (const unsigned *)c->bufs[B_LCP].p, n, be);
    bucket_apply(c, be, raw, n);
}

// raw slots [first, last] only (a position shard + its halo), SA order: every
// rank reads the whole SA / LCP once but emits and scatters only its slots
void raw_from_sa_lcp_range(rs_ctx *c, long long n, size_t raw_slots_n, long long first, long long last) {
    unsigned *raw = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots_n);
    RS_CUDA(cudaMemsetAsync(raw, 0, sizeof(unsigned), c->stream));
    BucketEmit be = bucket_setup(c, n + 1, 0);
    RS_LAUNCH_B(c, 8.0 * n + 8.0 * (double)(last - first + 1), k_raw_sa_emit,
                grid_for((n + kRIPT - 1) / kRIPT, kRNT), kRNT, 0, (const unsigned *)c->bufs[B_SA].p,
                (const unsigned *)c->bufs[B_LCP].p, n, be, (unsigned)first, (unsigned)last);
    bucket_apply(c, be, raw, last - first + 1);
}

void scatter_phi(rs_ctx *c, const unsigned *sa, long long n, unsigned *phi) {
    BucketEmit be = bucket_setup(c, n, 0);
    RS_LAUNCH_B(c, 12.0 * n, k_phi_emit, grid_for((n + kRIPT - 1) / kRIPT, kRNT), kRNT, 0, sa, n, be);
    bucket_apply(c, be, phi, n);
}

void scatter_by(rs_ctx *c, const unsigned *dest, const unsigned *val, long long n, unsigned *out, long long n_out) {
    BucketEmit be = bucket_setup(c, n_out, 0);
    RS_LAUNCH_B(c, 16.0 * n, k_pair_emit, grid_for((n + kRIPT - 1) / kRIPT, kRNT), kRNT, 0, dest, val, n, be);
    bucket_apply(c, be, out, n);
}

void scatter_rank(rs_ctx *c, const unsigned *sa, long long n, unsigned *isa) {
    BucketEmit be = bucket_setup(c, n, 0);
    RS_LAUNCH_B(c, 12.0 * n, k_rank_emit, grid_for((n + kRIPT - 1) / kRIPT, kRNT), kRNT, 0, sa, n, be);
    bucket_apply(c, be, isa, n);
}

}  // namespace rsb
