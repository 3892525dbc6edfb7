// scan_query.cu -- per-position covering-repeat scan (north-star subsystem 3).
//
// Reference semantics (1-based positions k):
//   leftmost, raw     _kernels_numba.py:88-102   (Alg. 1, leftward walk, ties -> smallest start)
//   leftmost, compact _kernels_numba.py:105-118  (Alg. 2, binary search + rightward walk)
//   all, raw          _kernels_numba.py:121-155  (Alg. 3: max, count, fill; block sorted by start)
//   all, compact      _kernels_numba.py:158-195  (Alg. 4)
//   CSR assembly      query.py:187-215 (offsets[0]=offsets[1]=0, offsets[k+1]=offsets[k]+cnt[k])
//
// Both walks visit exactly the candidates covering k, and those form one
// contiguous window [lo(k), hi(k)) of the candidate array (compact: starts and
// ends strictly increasing; raw: ends i+raw[i]-1 nondecreasing).  So a tile of
// G consecutive positions needs one contiguous candidate range, found once per
// tile by k_bounds (binary search, all tiles in parallel), staged into shared
// memory with a single TMA bulk copy (cp.async.bulk + mbarrier), and every
// thread then walks its positions' windows in shared memory.  The all-ties
// variant is single-pass: per-position tie counts -> block scan -> decoupled
// look-back for the tile's global CSR base -> offsets and tie starts written
// directly in the reference int64 layout.
#include "common.cuh"

namespace rsb {

namespace {

constexpr int kNT = 256;
constexpr int kPPT = 8;
constexpr int kG = kNT * kPPT;           // positions per tile
constexpr int kCapC = kG + 1024;         // staged compact entries (uint2)
constexpr int kCapR = 2 * kG + 2048;     // staged raw values (u32)
constexpr int kStageBytes = 8 * kCapC + 64;

// ---- TMA (1-D bulk copy) + mbarrier ------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes,
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Candidate window view: compact entries (start, len) or raw values (start = base + t).
template <bool RAW>
struct Cand {
    const uint2 *e;       // compact
    const unsigned *r;    // raw
    long long base;       // raw: text index of r[0]
    __device__ __forceinline__ long long start(long long t) const { return RAW ? base + t : (long long)e[t].x; }
    __device__ __forceinline__ unsigned len(long long t) const { return RAW ? r[t] : e[t].y; }
    __device__ __forceinline__ long long end(long long t) const {
        return RAW ? base + t + (long long)r[t] - 1 : (long long)e[t].x + (long long)e[t].y - 1;
    }
};

// Per-tile candidate range.  Tiles cover positions [kb + g*G, kb + g*G + G - 1] ∩ [kb, ke].
// Compact: lo = first t with end_t >= kfirst, hi = #{t : start_t <= klast}.
// Raw:     lo = first i in [1, kfirst] with i + raw[i] - 1 >= kfirst (else kfirst + 1),
//          hi = klast + 1 (window indices are text indices).
template <bool RAW>
__global__ void k_bounds(const uint2 *__restrict__ e, const unsigned *__restrict__ raw, long long count,
                         long long kb, long long ke, long long tiles, long long *__restrict__ bounds) {
    long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g >= tiles) return;
    long long kfirst = kb + g * kG;
    long long klast = kfirst + kG - 1;
    if (klast > ke) klast = ke;
    long long lo, hi;
    if (RAW) {
        long long a = 1, b = kfirst + 1;  // search in [1, kfirst]; answer kfirst+1 if none
        while (a < b) {
            long long mid = (a + b) >> 1;
            if (mid + (long long)__ldg(raw + mid) - 1 >= kfirst) b = mid; else a = mid + 1;
        }
        lo = a;
        hi = klast + 1;
    } else {
        long long a = 0, b = count;
        while (a < b) {
            long long mid = (a + b) >> 1;
            uint2 x = __ldg(e + mid);
            if ((long long)x.x + x.y - 1 >= kfirst) b = mid; else a = mid + 1;
        }
        lo = a;
        a = lo;
        b = count;
        while (a < b) {
            long long mid = (a + b) >> 1;
            if ((long long)__ldg(&e[mid].x) <= klast) a = mid + 1; else b = mid;
        }
        hi = a;
    }
    bounds[2 * g] = lo;
    bounds[2 * g + 1] = hi;
}

// Query kernel.  out_off = 1 writes the reference 1-based padded layout
// (slot k), out_off = 0 writes a shard-local layout (slot k - kb).
template <bool RAW, bool ALL>
__global__ void __launch_bounds__(kNT) k_query(const uint2 *__restrict__ e, const unsigned *__restrict__ raw,
                                               long long kb, long long ke, const long long *__restrict__ bounds,
                                               int out_off, long long *__restrict__ out0,
                                               long long *__restrict__ out1, long long *__restrict__ flat,
                                               long long flat_cap, unsigned *counter, u64 *status,
                                               long long tiles, unsigned long long *total_out) {
    __shared__ __align__(128) unsigned char s_stage[kStageBytes];
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ unsigned s_tile;
    __shared__ u64 s_warp[kNT / 32];
    __shared__ u64 s_base;

    long long tile;
    if (ALL) {
        if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
        __syncthreads();
        tile = s_tile;
    } else {
        tile = blockIdx.x;
    }
    const long long lo = bounds[2 * tile], hi = bounds[2 * tile + 1];
    const long long cnt = hi - lo;

    // ---- stage the tile's candidate range [lo, hi) ----
    Cand<RAW> c;
    c.e = nullptr;
    c.r = nullptr;
    c.base = lo;
    if (RAW) {
        long long a = lo & ~3ll, b = (hi + 3) & ~3ll;
        if (cnt > 0 && b - a <= kCapR) {
            if (threadIdx.x == 0) {
                mbar_init(&s_bar, 1);
                unsigned bytes = (unsigned)((b - a) * 4);
                mbar_expect_tx(&s_bar, bytes);
                tma_load_1d(s_stage, raw + a, bytes, &s_bar);
            }
            __syncthreads();
            mbar_wait(&s_bar, 0);
            c.r = reinterpret_cast<const unsigned *>(s_stage) + (lo - a);
        } else {
            c.r = raw + lo;
        }
    } else {
        long long a = lo & ~1ll, b = (hi + 1) & ~1ll;
        if (cnt > 0 && b - a <= kCapC) {
            if (threadIdx.x == 0) {
                mbar_init(&s_bar, 1);
                unsigned bytes = (unsigned)((b - a) * 8);
                mbar_expect_tx(&s_bar, bytes);
                tma_load_1d(s_stage, e + a, bytes, &s_bar);
            }
            __syncthreads();
            mbar_wait(&s_bar, 0);
            c.e = reinterpret_cast<const uint2 *>(s_stage) + (lo - a);
        } else {
            c.e = e + lo;
        }
    }

    // ---- per-thread positions ----
    const long long k0 = kb + tile * kG + (long long)threadIdx.x * kPPT;
    unsigned best[kPPT];
    unsigned ties[kPPT];
    long long bstart[kPPT];
    long long w_lo = 0, w_hi = 0;
    if (k0 <= ke) {
        long long a = 0, b = cnt;  // first t with end >= k0
        while (a < b) {
            long long mid = (a + b) >> 1;
            if (c.end(mid) >= k0) b = mid; else a = mid + 1;
        }
        w_lo = a;
        if (RAW) {
            w_hi = k0 - lo + 1;
        } else {
            a = w_lo;
            b = cnt;
            while (a < b) {
                long long mid = (a + b) >> 1;
                if (c.start(mid) <= k0) a = mid + 1; else b = mid;
            }
            w_hi = a;
        }
    }
    unsigned my_total = 0;
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const long long k = k0 + j;
        best[j] = 0;
        ties[j] = 0;
        bstart[j] = -1;
        if (k > ke) continue;
        while (w_lo < cnt && c.end(w_lo) < k) ++w_lo;
        if (RAW) {
            w_hi = k - lo + 1;
        } else {
            while (w_hi < cnt && c.start(w_hi) <= k) ++w_hi;
        }
        unsigned bl = 0, nt = 0;
        long long bs = -1;
        for (long long t = w_lo; t < w_hi; ++t) {
            unsigned L = c.len(t);
            if (L > bl) {
                bl = L;
                bs = c.start(t);
                nt = 1;
            } else if (L == bl) {
                ++nt;
            }
        }
        best[j] = bl;
        bstart[j] = bl ? bs : -1;
        ties[j] = bl ? nt : 0;
        my_total += ties[j];
    }

    if (!ALL) {
#pragma unroll
        for (int j = 0; j < kPPT; ++j) {
            const long long k = k0 + j;
            if (k > ke) break;
            const long long slot = k - kb + out_off;
            out0[slot] = bstart[j];
            out1[slot] = best[j];
        }
        if (tile == 0 && threadIdx.x == 0 && out_off) {
            out0[0] = -1;
            out1[0] = 0;
        }
        return;
    }

    // ---- all ties: CSR offsets via block scan + look-back ----
    u64 excl;
    u64 block_total = block_exclusive_sum64<kNT>((u64)my_total, excl, s_warp);
    if (threadIdx.x < 32) {
        u64 base = lookback_warp(status, tile, block_total, OpSum());
        if (threadIdx.x == 0) {
            s_base = base;
            if (tile == tiles - 1) *total_out = base + block_total;
        }
    }
    __syncthreads();
    u64 o = s_base + excl;
    // window pointers again from the thread's first position
    if (k0 <= ke) {
        long long a = 0, b = cnt;
        while (a < b) {
            long long mid = (a + b) >> 1;
            if (c.end(mid) >= k0) b = mid; else a = mid + 1;
        }
        w_lo = a;
    }
    if (tile == 0 && threadIdx.x == 0) {
        if (out_off) {
            out0[0] = 0;   // lengths[0]
            out1[0] = 0;   // offsets[0]
        }
        out1[out_off] = 0;  // offsets[k=kb] (exclusive prefix of the first position)
    }
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const long long k = k0 + j;
        if (k > ke) break;
        const long long slot = k - kb + out_off;
        out0[slot] = best[j];
        out1[slot + 1] = (long long)(o + ties[j]);
        if (ties[j]) {
            while (w_lo < cnt && c.end(w_lo) < k) ++w_lo;
            long long t = w_lo;
            long long w = (long long)o;
            const unsigned bl = best[j];
            // walk forward until ties[j] starts are written (all lie in the window)
            for (unsigned got = 0; got < ties[j]; ++t) {
                if (c.len(t) == bl) {
                    if (w < flat_cap) flat[w] = c.start(t);
                    ++w;
                    ++got;
                }
            }
        }
        o += ties[j];
    }
}

}  // namespace

// Run the scan for positions [kb, ke] over candidates (compact entries or raw),
// writing into B_OUT0/B_OUT1/B_FLAT.  out_off: 1 = reference layout.
void query_range(rs_ctx *c, int mode, int path, const uint2 *d_e, long long count, const unsigned *d_raw,
                 long long kb, long long ke, int out_off, long long n_slots) {
    const bool all = mode == RS_MODE_ALL;
    const bool rawp = path == RS_PATH_RAW;
    long long npos = ke - kb + 1;
    if (npos <= 0) return;
    long long tiles = (npos + kG - 1) / kG;
    long long *bounds = (long long *)buf(c, B_BOUNDS, sizeof(long long) * 2 * (size_t)tiles);
    if (rawp)
        RS_LAUNCH(c, k_bounds<true>, grid_for(tiles, 128), 128, 0, d_e, d_raw, count, kb, ke, tiles, bounds);
    else
        RS_LAUNCH(c, k_bounds<false>, grid_for(tiles, 128), 128, 0, d_e, d_raw, count, kb, ke, tiles, bounds);

    long long *out0 = (long long *)buf(c, B_OUT0, sizeof(long long) * (size_t)(n_slots + 1));
    long long *out1 = (long long *)buf(c, B_OUT1, sizeof(long long) * (size_t)(n_slots + 2));
    unsigned long long *tot = (unsigned long long *)buf(c, B_SMALL, 4096) + 2;
    if (!all) {
        if (rawp)
            RS_LAUNCH(c, (k_query<true, false>), (unsigned)tiles, kNT, 0, d_e, d_raw, kb, ke, bounds, out_off,
                      out0, out1, nullptr, 0, nullptr, nullptr, tiles, tot);
        else
            RS_LAUNCH(c, (k_query<false, false>), (unsigned)tiles, kNT, 0, d_e, d_raw, kb, ke, bounds,
                      out_off, out0, out1, nullptr, 0, nullptr, nullptr, tiles, tot);
        c->out_mode = 0;
        return;
    }
    // Tie total is unknown before the scan: size flat for the worst case seen
    // so far and re-run if it overflows (T <= sum of window sizes; in practice
    // T/n is 1.0-1.9).  Capacity starts at 2n + 64 slots.
    size_t cap_slots = c->bufs[B_FLAT].cap / sizeof(long long);
    size_t want = (size_t)(2 * npos + 64);
    if (cap_slots < want) cap_slots = want;
    for (int attempt = 0; attempt < 3; ++attempt) {
        long long *flat = (long long *)buf(c, B_FLAT, sizeof(long long) * cap_slots);
        Scratch s = scratch(c, tiles);
        if (rawp)
            RS_LAUNCH(c, (k_query<true, true>), (unsigned)tiles, kNT, 0, d_e, d_raw, kb, ke, bounds, out_off,
                      out0, out1, flat, (long long)cap_slots, s.counter, s.status, tiles, tot);
        else
            RS_LAUNCH(c, (k_query<false, true>), (unsigned)tiles, kNT, 0, d_e, d_raw, kb, ke, bounds,
                      out_off, out0, out1, flat, (long long)cap_slots, s.counter, s.status, tiles, tot);
        unsigned long long T = 0;
        fetch_small(c, &T, tot, sizeof(T));
        c->total = (long long)T;
        c->out_mode = 1;
        if ((size_t)T <= cap_slots) return;
        cap_slots = (size_t)T + 64;
    }
    fail(RS_ECUDA, "tie buffer sizing did not converge");
}

}  // namespace rsb
