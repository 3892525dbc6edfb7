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
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace rsb {

namespace {

constexpr int kNT = 256;
constexpr int kPPT = 4;
constexpr int kG = kNT * kPPT;           // positions per tile
constexpr int kCapC = kG + 1024;         // staged compact entries (uint2)
constexpr int kCapR = 2 * kG + 2048;     // staged raw values (u32)
constexpr int kStageBytes = 8 * kCapC + 128;
constexpr int kQuerySmem = kStageBytes + 3 * 4 * kG;  // dynamic shared memory: stage + lo/hi/count

// Candidate window view: compact entries (start, len) or raw values (start = base + t).
// Positions are < 2^31, so candidate starts/ends are 32-bit.
template <bool RAW>
struct Cand {
    const uint2 *e;       // compact
    const unsigned *r;    // raw
    unsigned base;        // raw: text index of r[0]
    __device__ __forceinline__ unsigned start(unsigned t) const { return RAW ? base + t : e[t].x; }
    __device__ __forceinline__ unsigned len(unsigned t) const { return RAW ? r[t] : e[t].y; }
    __device__ __forceinline__ int end(unsigned t) const {
        if (RAW) return (int)(base + t + r[t]) - 1;
        const uint2 v = e[t];
        return (int)(v.x + v.y) - 1;
    }
};

// Compact candidates as two shared arrays (starts, lengths): the window walks
// read lengths of neighbouring entries, 4-byte words in consecutive banks
// (the interleaved uint2 layout put two entries per bank pair: 2-way conflicts).
struct CandSoA {
    const unsigned *st, *ln;
    __device__ __forceinline__ unsigned start(unsigned t) const { return st[t]; }
    __device__ __forceinline__ unsigned len(unsigned t) const { return ln[t]; }
    __device__ __forceinline__ int end(unsigned t) const { return (int)(st[t] + ln[t]) - 1; }
};

// Per-tile candidate range.  Tiles cover positions [kb + g*G, kb + g*G + G - 1] ∩ [kb, ke].
// Compact: lo = first t with end_t >= kfirst, hi = #{t : start_t <= klast}.
// Raw:     lo = first i in [1, kfirst] with i + raw[i] - 1 >= kfirst (else kfirst + 1),
//          hi = klast + 1 (window indices are text indices).
template <bool RAW>
__global__ void k_bounds(const uint2 *__restrict__ e, const unsigned *__restrict__ raw, long long count,
                         long long kb, long long ke, long long tiles, long long *__restrict__ bounds,
                         long long min_lo) {
    long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g >= tiles) return;
    long long kfirst = kb + g * kG;
    long long klast = kfirst + kG - 1;
    if (klast > ke) klast = ke;
    long long lo, hi;
    if (RAW) {
        // search in [min_lo, kfirst]; answer kfirst+1 if none (min_lo > 1: a
        // shard's raw array starts there -- it is below every covering start)
        // i + raw[i] - 1 >= kfirst is monotone in i; gallop left from kfirst
        // (the answer lies within the longest repeat length of it) before
        // bisecting: ~2 log2(LLR) probes instead of log2(n)
        const long long a0 = min_lo > 1 ? min_lo : 1;
        long long a = a0, b = kfirst + 1;
        if (kfirst < a0) {
            // (empty search range: as the plain bisection, lo = a0)
        } else if (kfirst + (long long)__ldg(raw + kfirst) - 1 >= kfirst) {
            b = kfirst;
            long long step = 1;
            while (true) {
                const long long probe = kfirst - step;
                if (probe < a0) { a = a0; break; }
                if (probe + (long long)__ldg(raw + probe) - 1 >= kfirst) {
                    b = probe;
                    step <<= 1;
                } else {
                    a = probe + 1;
                    break;
                }
            }
        } else {
            a = b;  // nothing at or before kfirst reaches it
        }
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

// Window bounds per position: every position's window is the contiguous
// candidate range [lo(k), hi(k)); lo(k) = first candidate with end >= k,
// hi(k) = #candidates with start <= k.  Both are nondecreasing, so each
// candidate fills the positions where it is the boundary -- O(tile +
// candidates), no searches -- unless candidates are few and long
// (repetitive text), then one binary search per position.
template <typename C, typename IdxT>
__device__ __forceinline__ void fill_windows(const C &c, unsigned cnt, int tile_k0, int tile_k1, int npos,
                                             IdxT *s_lo, IdxT *s_hi) {
    if (cnt * 8 < (unsigned)npos) {
        for (int p = threadIdx.x; p < npos; p += kNT) {
            const int k = tile_k0 + p;
            unsigned a = 0, b = cnt;
            while (a < b) {
                const unsigned mid = (a + b) >> 1;
                if (c.end(mid) >= k) b = mid; else a = mid + 1;
            }
            s_lo[p] = (IdxT)a;
            b = cnt;
            while (a < b) {
                const unsigned mid = (a + b) >> 1;
                if ((int)c.start(mid) <= k) a = mid + 1; else b = mid;
            }
            s_hi[p] = (IdxT)a;
        }
    } else {
        // every position gets both bounds (no prior initialisation needed):
        // lo = cnt after the last end, hi = 0 before the first start
        if (cnt == 0) {
            for (int p = threadIdx.x; p < npos; p += kNT) {
                s_lo[p] = (IdxT)0;
                s_hi[p] = (IdxT)0;
            }
        } else if (threadIdx.x == 0) {
            const int el = c.end(cnt - 1);
#pragma unroll 1
            for (int k = (el + 1 > tile_k0 ? el + 1 : tile_k0); k <= tile_k1; ++k) s_lo[k - tile_k0] = (IdxT)cnt;
            const int s0 = (int)c.start(0);
#pragma unroll 1
            for (int k = tile_k0; k < s0 && k <= tile_k1; ++k) s_hi[k - tile_k0] = (IdxT)0;
        }
        for (unsigned t = threadIdx.x; t < cnt; t += kNT) {
            const int ep = t ? c.end(t - 1) : tile_k0 - 1;
            const int e_t = c.end(t);
            int a = ep + 1 > tile_k0 ? ep + 1 : tile_k0;
            int b = e_t < tile_k1 ? e_t : tile_k1;
#pragma unroll 1
            for (int k = a; k <= b; ++k) s_lo[k - tile_k0] = (IdxT)t;
            const int st = (int)c.start(t);
            const int sn = (t + 1 < cnt) ? (int)c.start(t + 1) : tile_k1 + 1;
            a = st > tile_k0 ? st : tile_k0;
            b = sn - 1 < tile_k1 ? sn - 1 : tile_k1;
#pragma unroll 1
            for (int k = a; k <= b; ++k) s_hi[k - tile_k0] = (IdxT)(t + 1);
        }
    }
    __syncthreads();
}

// IdxT: per-position window bounds (u16 in the fused kernel, whose windows
// index a shared stage of < 2^16 entries: smaller footprint, 8 CTAs per SM)
template <typename IdxT>
struct TileCtx {
    long long tile, cnt, tile_k0, tile_k1, slot0, tiles, flat_cap;
    int npos, out_off;
    IdxT *s_lo, *s_hi;
    unsigned *s_cnt, *s_warp;
    unsigned short *s_ties;  // tile-local tie list (candidate indices), or null
    unsigned ties_cap;       // its capacity
    u64 *s_base;
    long long *out0, *out1, *flat;
    u64 *status;
    unsigned long long *total_out;
};

// Everything after staging.  Inlined twice (candidates in shared memory or,
// for oversized windows, in global memory) so each copy uses the right
// address space (LDS instead of generic loads).
template <typename C, bool ALL, typename IdxT>
__device__ __forceinline__ void query_tile(const C &c, const TileCtx<IdxT> &x) {
    const unsigned cnt = (unsigned)x.cnt;
    fill_windows<C, IdxT>(c, cnt, (int)x.tile_k0, (int)x.tile_k1, x.npos, x.s_lo, x.s_hi);

    // ---- per position (lane-interleaved: consecutive threads, consecutive positions) ----
    // Windows of up to 32 candidates (the common case) record their ties as a
    // bit mask relative to the window start while finding the maximum, so the
    // tie starts are later read by iterating set bits (nt steps) instead of
    // re-walking the window; longer windows (repetitive text) re-walk.
    unsigned tmask[kPPT];  // tie mask; 0 with ties means "re-walk"
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const int p = threadIdx.x + j * kNT;
        tmask[j] = 0;
        if (p >= x.npos) continue;
        const unsigned wl = x.s_lo[p], wh = x.s_hi[p];
        unsigned bl = 0, nt = 0, bs = 0;
        if (wh - wl <= 32u) {
            unsigned tm = 0, bit = 1;
            unsigned t = wl;
            // two candidates per iteration (branch-free updates), then the odd one
#pragma unroll 1
            for (; t + 1 < wh; t += 2, bit <<= 2) {
                const unsigned L0 = c.len(t), L1 = c.len(t + 1);
                tm = L0 > bl ? bit : (L0 == bl ? tm | bit : tm);
                bl = L0 > bl ? L0 : bl;
                tm = L1 > bl ? bit << 1 : (L1 == bl ? tm | (bit << 1) : tm);
                bl = L1 > bl ? L1 : bl;
            }
            if (t < wh) {
                const unsigned L0 = c.len(t);
                tm = L0 > bl ? bit : (L0 == bl ? tm | bit : tm);
                bl = L0 > bl ? L0 : bl;
            }
            nt = __popc(tm);
            if (tm) bs = c.start(wl + __ffs(tm) - 1);
            tmask[j] = tm;
        } else {
#pragma unroll 1
            for (unsigned t = wl; t < wh; ++t) {
                const unsigned L = c.len(t);
                if (L > bl) {
                    bl = L;
                    bs = c.start(t);
                    nt = 1;
                } else if (L == bl) {
                    ++nt;
                }
            }
        }
        if (ALL) {
            x.out0[x.slot0 + p] = bl;
            x.s_cnt[p] = bl ? nt : 0;
        } else {
            x.out0[x.slot0 + p] = bl ? (long long)bs : -1ll;
            x.out1[x.slot0 + p] = bl;
        }
    }
    if (!ALL) {
        if (x.tile == 0 && threadIdx.x == 0 && x.out_off) {
            x.out0[0] = -1;
            x.out1[0] = 0;
        }
        return;
    }

    // ---- all ties: exclusive scan of the tile's counts (position order) ----
    __syncthreads();
    unsigned mine[kPPT], msum = 0;
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const int p = threadIdx.x * kPPT + j;
        mine[j] = p < x.npos ? x.s_cnt[p] : 0;
        msum += mine[j];
    }
    unsigned excl;
    const unsigned block_total = block_exclusive_sum<kNT, false>(msum, excl, x.s_warp);
    // publish the tile's aggregate at once (successors stop waiting on it),
    // but resolve this tile's own base only after listing the ties: by then
    // the predecessors have had the listing's time to publish theirs
    if (threadIdx.x == 0) lookback_publish(x.status, x.tile, (u64)block_total);
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const int p = threadIdx.x * kPPT + j;
        if (p < x.npos) x.s_cnt[p] = excl;
        excl += mine[j];
    }
    __syncthreads();
    // Every warp lists its positions' ties in shared memory (candidate indices
    // in output order); then warp 0 resolves the tile's global base (decoupled
    // look-back); after the barrier the list is written out coalesced.  Tiles
    // whose ties overflow the list write directly.
    const bool staged = x.s_ties != nullptr && block_total <= x.ties_cap;
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const int p = threadIdx.x + j * kNT;
        if (!staged || p >= x.npos) continue;
        const unsigned ex = x.s_cnt[p];
        const unsigned nxt = (p + 1 < x.npos) ? x.s_cnt[p + 1] : block_total;
        if (nxt == ex) continue;
        const unsigned wl = x.s_lo[p];
        unsigned tm = tmask[j];
        unsigned w = ex;
        if (tm) {
            do {
                const unsigned b = __ffs(tm) - 1;
                tm &= tm - 1;
                x.s_ties[w++] = (unsigned short)(wl + b);
            } while (tm);
        } else {
            const unsigned wh = x.s_hi[p];
            unsigned bl = 0;  // long window (> 32): maximum again, then the ties
#pragma unroll 1
            for (unsigned t = wl; t < wh; ++t) bl = max(bl, c.len(t));
#pragma unroll 1
            for (unsigned t = wl; t < wh; ++t)
                if (c.len(t) == bl) x.s_ties[w++] = (unsigned short)t;
        }
    }
    if (threadIdx.x < 32) {
        u64 base = lookback_warp(x.status, x.tile, (u64)block_total, OpSum(), true);
        if (threadIdx.x == 0) {
            *x.s_base = base;
            if (x.tile == x.tiles - 1) *x.total_out = base + block_total;
        }
    }
    __syncthreads();
    const u64 tile_base = *x.s_base;
    if (x.tile == 0 && threadIdx.x == 0) {
        if (x.out_off) {
            x.out0[0] = 0;  // lengths[0]
            x.out1[0] = 0;  // offsets[0]
        }
        x.out1[x.out_off] = 0;  // offsets of the first position
    }
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const int p = threadIdx.x + j * kNT;
        if (p < x.npos)  // offsets[k+1] = inclusive prefix
            x.out1[x.slot0 + 1 + p] = (long long)(tile_base + ((p + 1 < x.npos) ? x.s_cnt[p + 1] : block_total));
    }
    const bool cap_ok = (long long)(tile_base + block_total) <= x.flat_cap;
    long long *const flat_tile = x.flat + tile_base;
    if (staged) {
        if (cap_ok) {
            for (unsigned i = threadIdx.x; i < block_total; i += kNT) flat_tile[i] = c.start(x.s_ties[i]);
        } else {
            for (unsigned i = threadIdx.x; i < block_total; i += kNT)
                if ((long long)(tile_base + i) < x.flat_cap) flat_tile[i] = c.start(x.s_ties[i]);
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
        const int p = threadIdx.x + j * kNT;
        if (p >= x.npos) continue;
        const unsigned ex = x.s_cnt[p];
        const unsigned nt = ((p + 1 < x.npos) ? x.s_cnt[p + 1] : block_total) - ex;
        if (nt == 0) continue;
        const unsigned wl = x.s_lo[p];
        unsigned tm = tmask[j];
        if (tm && cap_ok) {  // 32-bit tile-local slots, no per-store capacity test
            unsigned w = ex;
            do {
                const unsigned b = __ffs(tm) - 1;
                tm &= tm - 1;
                flat_tile[w++] = c.start(wl + b);
            } while (tm);
            continue;
        }
        long long w = (long long)(tile_base + ex);
        if (tm) {
            do {
                const unsigned b = __ffs(tm) - 1;
                tm &= tm - 1;
                if (w < x.flat_cap) x.flat[w] = c.start(wl + b);
                ++w;
            } while (tm);
            continue;
        }
        const unsigned wh = x.s_hi[p];
        unsigned bl = 0;
#pragma unroll 1
        for (unsigned t = wl; t < wh; ++t) bl = max(bl, c.len(t));
#pragma unroll 1
        for (unsigned t = wl; t < wh; ++t) {
            if (c.len(t) == bl) {
                if (w < x.flat_cap) x.flat[w] = c.start(t);
                ++w;
            }
        }
    }
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
    extern __shared__ __align__(128) unsigned char dsm[];
    unsigned char *s_stage = dsm;
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[kNT / 32];
    __shared__ u64 s_base;

    // tile = blockIdx.x also for the look-back of the all variant (dispatch
    // order, as k_query_fused; see lookback_warp)
    (void)counter;
    (void)s_tile;
    const long long tile = blockIdx.x;
    TileCtx<unsigned> x;
    x.tile = tile;
    const long long lo = bounds[2 * tile], hi = bounds[2 * tile + 1];
    x.cnt = hi - lo;
    x.tile_k0 = kb + tile * kG;
    x.npos = (int)((ke - x.tile_k0 + 1) < kG ? (ke - x.tile_k0 + 1) : kG);
    x.tile_k1 = x.tile_k0 + x.npos - 1;
    x.slot0 = x.tile_k0 - kb + out_off;
    x.out_off = out_off;
    x.tiles = tiles;
    x.flat_cap = flat_cap;
    x.s_lo = reinterpret_cast<unsigned *>(dsm + kStageBytes);  // window start per position
    x.s_hi = x.s_lo + kG;                                       // window end (exclusive)
    x.s_cnt = x.s_hi + kG;                                      // tie counts -> exclusive offsets
    x.s_warp = s_warp;
    x.s_ties = nullptr;  // candidates may be > 2^16: direct tie stores
    x.ties_cap = 0;
    x.s_base = &s_base;
    x.out0 = out0;
    x.out1 = out1;
    x.flat = flat;
    x.status = status;
    x.total_out = total_out;

    // ---- stage the tile's candidate range [lo, hi) with one TMA bulk copy ----
    const int esz = RAW ? 4 : 8;
    const long long align = 16 / esz;
    const long long a = lo & ~(align - 1), b = (hi + align - 1) & ~(align - 1);
    const bool fits = x.cnt > 0 && b - a <= (RAW ? kCapR : kCapC);
    if (fits && threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        unsigned bytes = (unsigned)((b - a) * esz);
        mbar_expect_tx(&s_bar, bytes);
        tma_load_1d(s_stage, RAW ? (const void *)(raw + a) : (const void *)(e + a), bytes, &s_bar);
    }
    // window bounds per position: every position's window is the contiguous
    // candidate range [lo(k), hi(k)); lo(k) = first candidate with end >= k,
    // hi(k) = #candidates with start <= k.  Both are nondecreasing, so each
    // candidate fills the positions where it is the boundary -- O(tile +
    // candidates), no searches.
    for (int i = threadIdx.x; i < x.npos; i += kNT) {
        x.s_lo[i] = (unsigned)x.cnt;
        x.s_hi[i] = 0;
    }
    __syncthreads();
    Cand<RAW> c;
    c.base = (unsigned)lo;
    if (fits) {
        mbar_wait(&s_bar, 0);
        c.e = RAW ? nullptr : reinterpret_cast<const uint2 *>(s_stage) + (lo - a);
        c.r = RAW ? reinterpret_cast<const unsigned *>(s_stage) + (lo - a) : nullptr;
        query_tile<Cand<RAW>, ALL>(c, x);
    } else {
        c.e = RAW ? nullptr : e + lo;
        c.r = RAW ? raw + lo : nullptr;
        query_tile<Cand<RAW>, ALL>(c, x);
    }
}

// Compact path with the compaction fused into the scan.  A tile's compact
// candidates are exactly the flagged raw slots i in [lo, klast] (flag(i) =
// raw[i] > 0 && raw[i] >= raw[i-1]; lo = first i whose raw end reaches the
// tile, from k_bounds<true>): flagged slots before lo end before the tile,
// every flagged slot from lo on reaches it (raw ends are nondecreasing).  So
// the tile stages raw[lo-1, klast] with one TMA copy, compacts it in shared
// memory (block scan, order kept) and runs the compact walk on that list --
// the global LLRc is never written nor read back.  The host only takes this
// path when every tile's raw range fits the stage (short repeats).
constexpr int kFStage = kG + 768 + 16;  // staged raw values incl. alignment slack and slot lo-1
constexpr int kFRawBytes = ((4 * kFStage + 127) / 128) * 128;
// the raw stage is dead after compaction: the per-position window bounds
// (u16) and tie counts reuse it (region A); then the compacted starts and
// lengths (B) and the tile's tie list (C, u16 candidate indices: ~2.2 ties
// per position of headroom over i.i.d. DNA's 1.9) -> 27.5 KB, 8 CTAs per SM
constexpr int kFRegionA = kFRawBytes > 8 * kG ? kFRawBytes : 8 * kG;
constexpr int kFTiesCap = 2688;
static_assert(kFStage < 65536, "u16 window bounds and tie indices");
constexpr int kFusedSmem = kFRegionA + 8 * kFStage + 2 * kFTiesCap;
static_assert(kFusedSmem + 128 <= 233472 / 8 - 1024, "8 CTAs per SM");

template <bool ALL>
__global__ void __launch_bounds__(kNT, 8) k_query_fused(const unsigned *__restrict__ raw, long long kb, long long ke,
                                                     const long long *__restrict__ bounds, int out_off,
                                                     long long *__restrict__ out0, long long *__restrict__ out1,
                                                     long long *__restrict__ flat, long long flat_cap,
                                                     unsigned *counter, u64 *status, long long tiles,
                                                     unsigned long long *total_out, unsigned ties_cap) {
    extern __shared__ __align__(128) unsigned char dsm[];
    unsigned *s_raw = reinterpret_cast<unsigned *>(dsm);
    unsigned *s_st = reinterpret_cast<unsigned *>(dsm + kFRegionA);  // compacted starts
    unsigned *s_ln = s_st + kFStage;                                   // compacted lengths
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[kNT / 32];
    __shared__ unsigned s_warp_c[kNT / 32];  // the compaction scan's own (no barrier between the scans)
    __shared__ u64 s_base;

    // tile = blockIdx.x also for the look-back of the all variant (blocks
    // are dispatched in index order, as CUB's single-pass scan relies on):
    // saves the tile counter's round trip before the bounds load and TMA
    (void)counter;
    (void)s_tile;
    const long long tile = blockIdx.x;
    TileCtx<unsigned short> x;
    x.tile = tile;
    const long long lo = bounds[2 * tile], hi = bounds[2 * tile + 1];  // raw slots [lo, hi)
    x.tile_k0 = kb + tile * kG;
    x.npos = (int)((ke - x.tile_k0 + 1) < kG ? (ke - x.tile_k0 + 1) : kG);
    x.tile_k1 = x.tile_k0 + x.npos - 1;
    x.slot0 = x.tile_k0 - kb + out_off;
    x.out_off = out_off;
    x.tiles = tiles;
    x.flat_cap = flat_cap;
    x.s_lo = reinterpret_cast<unsigned short *>(dsm);  // aliases s_raw (dead after compaction)
    x.s_hi = x.s_lo + kG;
    x.s_cnt = reinterpret_cast<unsigned *>(dsm + 4 * kG);
    x.s_warp = s_warp;
    x.s_ties = reinterpret_cast<unsigned short *>(dsm + kFRegionA + 8 * kFStage);
    x.ties_cap = ties_cap;
    x.s_base = &s_base;
    x.out0 = out0;
    x.out1 = out1;
    x.flat = flat;
    x.status = status;
    x.total_out = total_out;

    const long long a = (lo - 1) & ~3ll, b = (hi + 3) & ~3ll;  // stage raw[a, b), 16-byte aligned
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        const unsigned bytes = (unsigned)((b - a) * 4);
        mbar_expect_tx(&s_bar, bytes);
        tma_load_1d(s_raw, raw + a, bytes, &s_bar);
    }
    __syncthreads();
    mbar_wait(&s_bar, 0);
    // tile-local compaction: thread-contiguous runs, block scan, order kept
    const int nr = (int)(hi - lo);
    const int per = (nr + kNT - 1) / kNT;
    const int o0 = threadIdx.x * per;
    const unsigned *r0 = s_raw + (lo - a);  // r0[o] = raw[lo + o], r0[-1] = raw[lo - 1]
    unsigned nf = 0;
    for (int q = 0; q < per; ++q) {
        const int o = o0 + q;
        if (o < nr) nf += (r0[o] > 0u && r0[o] >= r0[o - 1]);
    }
    unsigned w;
    const unsigned cnt = block_exclusive_sum<kNT, false>(nf, w, s_warp_c);
    for (int q = 0; q < per; ++q) {
        const int o = o0 + q;
        if (o < nr && r0[o] > 0u && r0[o] >= r0[o - 1]) {
            s_st[w] = (unsigned)(lo + o);
            s_ln[w++] = r0[o];
        }
    }
    x.cnt = cnt;
    __syncthreads();  // s_raw dead from here: the window bounds take its place (fill_windows writes all)
    CandSoA c;
    c.st = s_st;
    c.ln = s_ln;
    query_tile<CandSoA, ALL>(c, x);
}

// max over tiles of the staged raw range (hi - lo + 8) -> *out
__global__ void k_max_span(const long long *__restrict__ bounds, long long tiles, unsigned long long *out) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long v = 0;
    if (t < tiles) v = (unsigned long long)(bounds[2 * t + 1] - bounds[2 * t] + 8);
    for (int o = 16; o; o >>= 1) {
        unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
        v = v > y ? v : y;
    }
    if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// Walk-step statistics (stats.py:30-76): the steps of a query walk at k are
// exactly the candidates covering k, i.e. the window size hi(k) - lo(k)
// (raw: k - #{i : i + raw[i] - 1 < k}; compact: max(upto - below, 0)).
// Writes steps[k] (optional) and accumulates min/max/sum/count over k with
// steps > 0 into acc[4].
template <bool RAW>
__global__ void __launch_bounds__(kNT) k_steps(const uint2 *__restrict__ e, const unsigned *__restrict__ raw,
                                               long long kb, long long ke, const long long *__restrict__ bounds,
                                               long long *__restrict__ steps, unsigned long long *acc) {
    extern __shared__ __align__(128) unsigned char dsm[];
    unsigned char *s_stage = dsm;
    unsigned *s_lo = reinterpret_cast<unsigned *>(dsm + kStageBytes);
    unsigned *s_hi = s_lo + kG;
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ unsigned long long s_red[4];
    const long long tile = blockIdx.x;
    const long long lo = bounds[2 * tile], hi = bounds[2 * tile + 1];
    const long long cnt = hi - lo;
    const long long tile_k0 = kb + tile * kG;
    const int npos = (int)((ke - tile_k0 + 1) < kG ? (ke - tile_k0 + 1) : kG);
    if (threadIdx.x < 4) s_red[threadIdx.x] = threadIdx.x == 0 ? ~0ull : 0ull;
    for (int i = threadIdx.x; i < npos; i += kNT) {
        s_lo[i] = (unsigned)cnt;
        s_hi[i] = 0;
    }
    const int esz = RAW ? 4 : 8;
    const long long align = 16 / esz;
    const long long a = lo & ~(align - 1), b = (hi + align - 1) & ~(align - 1);
    const bool fits = cnt > 0 && b - a <= (RAW ? kCapR : kCapC);
    if (fits && threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        unsigned bytes = (unsigned)((b - a) * esz);
        mbar_expect_tx(&s_bar, bytes);
        tma_load_1d(s_stage, RAW ? (const void *)(raw + a) : (const void *)(e + a), bytes, &s_bar);
    }
    __syncthreads();
    Cand<RAW> c;
    c.base = (unsigned)lo;
    if (fits) {
        mbar_wait(&s_bar, 0);
        c.e = RAW ? nullptr : reinterpret_cast<const uint2 *>(s_stage) + (lo - a);
        c.r = RAW ? reinterpret_cast<const unsigned *>(s_stage) + (lo - a) : nullptr;
    } else {
        c.e = RAW ? nullptr : e + lo;
        c.r = RAW ? raw + lo : nullptr;
    }
    fill_windows<Cand<RAW>, unsigned>(c, (unsigned)(cnt > 0 ? cnt : 0), (int)tile_k0, (int)(tile_k0 + npos - 1), npos, s_lo, s_hi);
    unsigned long long mn = ~0ull, mx = 0, sum = 0, n = 0;
    for (int p = threadIdx.x; p < npos; p += kNT) {
        const long long w = (long long)s_hi[p] - (long long)s_lo[p];
        const unsigned long long st = w > 0 ? (unsigned long long)w : 0ull;
        if (steps) steps[tile_k0 + p] = (long long)st;
        if (st) {
            mn = st < mn ? st : mn;
            mx = st > mx ? st : mx;
            sum += st;
            ++n;
        }
    }
    atomicMin(&s_red[0], mn);
    atomicMax(&s_red[1], mx);
    atomicAdd(&s_red[2], sum);
    atomicAdd(&s_red[3], n);
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicMin(&acc[0], s_red[0]);
        atomicMax(&acc[1], s_red[1]);
        atomicAdd(&acc[2], s_red[2]);
        atomicAdd(&acc[3], s_red[3]);
    }
}

// Summary of a caller-given steps array (summarize_steps, stats.py:58-68).
__global__ void k_summarize(const long long *__restrict__ steps, long long n, unsigned long long *acc) {
    unsigned long long mn = ~0ull, mx = 0, sum = 0, cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long v = steps[i];
        if (v > 0) {
            const unsigned long long u = (unsigned long long)v;
            mn = u < mn ? u : mn;
            mx = u > mx ? u : mx;
            sum += u;
            ++cnt;
        }
    }
    if (cnt) {
        atomicMin(&acc[0], mn);
        atomicMax(&acc[1], mx);
        atomicAdd(&acc[2], sum);
        atomicAdd(&acc[3], cnt);
    }
}

}  // namespace

// Run the scan for positions [kb, ke] over candidates (compact entries or raw),
// writing into B_OUT0/B_OUT1/B_FLAT.  out_off: 1 = reference layout.
bool query_range(rs_ctx *c, int mode, int path, const uint2 *d_e, long long count, const unsigned *d_raw,
                 long long kb, long long ke, int out_off, long long n_slots, long long min_lo) {
    const bool all = mode == RS_MODE_ALL;
    // compact path without a materialised LLRc: compaction fused into the scan
    const bool fused = path == RS_PATH_COMPACT && d_e == nullptr;
    const bool rawp = path == RS_PATH_RAW;
    long long npos = ke - kb + 1;
    if (npos <= 0) return true;
    long long tiles = (npos + kG - 1) / kG;
    long long *bounds = (long long *)buf(c, B_BOUNDS, sizeof(long long) * 2 * (size_t)tiles);
    if (rawp || fused)
        RS_LAUNCH(c, k_bounds<true>, grid_for(tiles, 128), 128, 0, d_e, d_raw, count, kb, ke, tiles, bounds, min_lo);
    else
        RS_LAUNCH(c, k_bounds<false>, grid_for(tiles, 128), 128, 0, d_e, d_raw, count, kb, ke, tiles, bounds, 1ll);
    if (fused) {
        unsigned long long *span = (unsigned long long *)buf(c, B_SMALL, 4096) + 6;
        RS_CUDA(cudaMemsetAsync(span, 0, sizeof(*span), c->stream));
        RS_LAUNCH(c, k_max_span, grid_for(tiles, 256), 256, 0, bounds, tiles, span);
        unsigned long long mx = 0;
        fetch_small(c, &mx, span, sizeof(mx));
        if (mx > (unsigned long long)kFStage) return false;  // long repeats: the caller materialises LLRc
        static unsigned long long fattr = 0;
        once_per_device(fattr, c->device, [] {
            RS_CUDA(cudaFuncSetAttribute(k_query_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem));
            RS_CUDA(cudaFuncSetAttribute(k_query_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem));
        });
    }

    static unsigned long long attr = 0;
    once_per_device(attr, c->device, [] {
        RS_CUDA(cudaFuncSetAttribute(k_query<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQuerySmem));
        RS_CUDA(cudaFuncSetAttribute(k_query<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQuerySmem));
        RS_CUDA(cudaFuncSetAttribute(k_query<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQuerySmem));
        RS_CUDA(cudaFuncSetAttribute(k_query<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQuerySmem));
    });
    long long *out0 = (long long *)buf(c, B_OUT0, sizeof(long long) * (size_t)(n_slots + 1));
    long long *out1 = (long long *)buf(c, B_OUT1, sizeof(long long) * (size_t)(n_slots + 2));
    unsigned long long *tot = (unsigned long long *)buf(c, B_SMALL, 4096) + 2;
    // algorithmic bytes: candidates read once (compact 8 B/entry, raw 4 B/slot),
    // int64 outputs written once (leftmost 16 B/pos; all 16 B/pos + 8 B/tie).
    const double cand_bytes = (rawp || fused) ? 4.0 * (double)npos : 8.0 * (double)count;
    const double qbytes = cand_bytes + 16.0 * (double)npos;
    if (!all) {
        if (fused)
            RS_LAUNCH_B(c, qbytes, (k_query_fused<false>), (unsigned)tiles, kNT, kFusedSmem, d_raw, kb, ke, bounds,
                        out_off, out0, out1, nullptr, 0, nullptr, nullptr, tiles, tot, 0u);
        else if (rawp)
            RS_LAUNCH_B(c, qbytes, (k_query<true, false>), (unsigned)tiles, kNT, kQuerySmem, d_e, d_raw, kb, ke, bounds, out_off,
                      out0, out1, nullptr, 0, nullptr, nullptr, tiles, tot);
        else
            RS_LAUNCH_B(c, qbytes, (k_query<false, false>), (unsigned)tiles, kNT, kQuerySmem, d_e, d_raw, kb, ke, bounds,
                      out_off, out0, out1, nullptr, 0, nullptr, nullptr, tiles, tot);
        c->out_mode = 0;
        return true;
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
        if (fused) {
            // RS_FUSED_TIES_CAP (tests only) shrinks the shared tie list so
            // the direct-store fallback of overflowing tiles gets exercised
            unsigned ties_cap = kFTiesCap;
            if (const char *e = std::getenv("RS_FUSED_TIES_CAP")) {
                const long v = std::strtol(e, nullptr, 10);
                if (v >= 0 && v < ties_cap) ties_cap = (unsigned)v;
            }
            RS_LAUNCH_B(c, qbytes, (k_query_fused<true>), (unsigned)tiles, kNT, kFusedSmem, d_raw, kb, ke, bounds,
                        out_off, out0, out1, flat, (long long)cap_slots, s.counter, s.status, tiles, tot, ties_cap);
        }
        else if (rawp)
            RS_LAUNCH_B(c, qbytes, (k_query<true, true>), (unsigned)tiles, kNT, kQuerySmem, d_e, d_raw, kb, ke, bounds, out_off,
                      out0, out1, flat, (long long)cap_slots, s.counter, s.status, tiles, tot);
        else
            RS_LAUNCH_B(c, qbytes, (k_query<false, true>), (unsigned)tiles, kNT, kQuerySmem, d_e, d_raw, kb, ke, bounds,
                      out_off, out0, out1, flat, (long long)cap_slots, s.counter, s.status, tiles, tot);
        unsigned long long T = 0;
        fetch_small(c, &T, tot, sizeof(T));
        add_bytes_last(c, 8.0 * (double)T);
        c->total = (long long)T;
        c->out_mode = 1;
        if ((size_t)T <= cap_slots) return true;
        cap_slots = (size_t)T + 64;
    }
    fail(RS_ECUDA, "tie buffer sizing did not converge");
}

// Walk steps / statistics over positions [1, n] of the loaded candidates.
// steps_out: device int64[n+1] or null; acc_host receives {min, max, sum, count}.
void walk_steps(rs_ctx *c, int path, long long n, long long *d_steps, unsigned long long *acc_host) {
    const bool rawp = path == RS_PATH_RAW;
    unsigned long long *acc = (unsigned long long *)buf(c, B_SMALL, 4096) + 16;
    unsigned long long init[4] = {~0ull, 0, 0, 0};
    RS_CUDA(cudaMemcpyAsync(acc, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    if (d_steps) RS_CUDA(cudaMemsetAsync(d_steps, 0, sizeof(long long), c->stream));
    if (n > 0) {
        const uint2 *d_e = (const uint2 *)c->bufs[B_LLRC].p;
        const unsigned *d_raw = (const unsigned *)c->bufs[B_RAW].p;
        const long long count = rawp ? 0 : c->m;
        long long tiles = (n + kG - 1) / kG;
        long long *bounds = (long long *)buf(c, B_BOUNDS, sizeof(long long) * 2 * (size_t)tiles);
        static unsigned long long attr = 0;
        once_per_device(attr, c->device, [] {
            const int sm = kStageBytes + 2 * 4 * kG;
            RS_CUDA(cudaFuncSetAttribute(k_steps<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            RS_CUDA(cudaFuncSetAttribute(k_steps<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        });
        const int sm = kStageBytes + 2 * 4 * kG;
        if (rawp) {
            RS_LAUNCH(c, k_bounds<true>, grid_for(tiles, 128), 128, 0, d_e, d_raw, count, 1, n, tiles, bounds, 1ll);
            RS_LAUNCH(c, k_steps<true>, (unsigned)tiles, kNT, sm, d_e, d_raw, 1, n, bounds, d_steps, acc);
        } else {
            RS_LAUNCH(c, k_bounds<false>, grid_for(tiles, 128), 128, 0, d_e, d_raw, count, 1, n, tiles, bounds, 1ll);
            RS_LAUNCH(c, k_steps<false>, (unsigned)tiles, kNT, sm, d_e, d_raw, 1, n, bounds, d_steps, acc);
        }
    }
    fetch_small(c, acc_host, acc, 4 * sizeof(unsigned long long));
}

void summarize(rs_ctx *c, const long long *d_steps, long long count, unsigned long long *acc_host) {
    unsigned long long *acc = (unsigned long long *)buf(c, B_SMALL, 4096) + 16;
    unsigned long long init[4] = {~0ull, 0, 0, 0};
    RS_CUDA(cudaMemcpyAsync(acc, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    if (count > 0)
        RS_LAUNCH(c, k_summarize, (unsigned)std::min<long long>(grid_for(count, 256), (long long)c->sm_count * 8), 256, 0,
                  d_steps, count, acc);
    fetch_small(c, acc_host, acc, 4 * sizeof(unsigned long long));
}

}  // namespace rsb
