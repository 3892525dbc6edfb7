// suffix_array.cu -- on-device suffix array, rank (ISA) and LCP (north-star subsystem 1).
//
// Reference: suffixes.py:31-53 (prefix doubling with np.argsort/np.lexsort),
// suffixes.py:64 (rank inversion), _kernels_numba.py:15-30 (Kasai LCP).
//
// B200 design (prefix doubling with group-head ranks, Larsson-Sadakane style):
//   round 0: every suffix gets a packed key of its first K symbols, each an
//            order-preserving code 0..sigma-1 of b = ceil(log2 sigma) bits
//            (2 bits for DNA); past the end pads with code 0, and the ties
//            that creates are broken by suffix length in the next round.
//            K is the largest count that fits the fewest 8-bit radix passes
//            while sigma^K >= 16 n (DNA at 256 Mi: b = 2, K = 16, 4 passes).
//            One LSD radix sort of (key, position) pairs gives the SA order.
//   k_update: SA write-back, ISA = SA slot of the suffix's group head
//            (max-scan) and compaction of the still-unsorted slots (sum-scan),
//            both through ONE decoupled look-back.  In round 0 it also emits
//            the LCP of adjacent suffixes straight from their keys (exact
//            when the keys differ) and each suffix's raw-LLR candidate
//            max(LCP to predecessor, LCP to successor); ISA and raw go to text
//            order through the bucketed scatter (scatter.cu).
//   round r>=1 (h = K * 2^(r-1)): only unsorted suffixes get a key
//            (ISA[i], ISA[i+h]+1 or 0 past the end) and are re-sorted; their
//            groups occupy the same SA slots, so results write straight back.
//   Rank = ISA (ranks are the final group heads), inversion is free.
//   LCP: pairs tied after round 0 (LCP >= K) are finished by direct word
//   compares, which also fixes the raw LLR of their two suffixes.  When that
//   would be expensive (repetitive text), Kasai over text-order chunks (PLCP
//   via the Phi array) recomputes every LCP, and raw is rebuilt from SA order.
// Device layouts: sa/isa u32[n] 0-based; lcp_d u32[n+2] with lcp_d[r] =
// reference lcp[r+1] (lcp_d[0] = lcp_d[n] = 0); raw u32 1-based (raw[0] = 0).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "scatter.cuh"

namespace rsb {

size_t raw_slots(long long n);

namespace {

constexpr unsigned kNone = 0xffffffffu;
constexpr unsigned kLcpUnknown = 0xfffffffeu;

struct CodeTable {
    unsigned short code[256];  // 1..sigma; sigma may be 256, so 9 bits
};

__device__ __forceinline__ u64 load8(const unsigned char *t, long long p) {
    const u64 *w = reinterpret_cast<const u64 *>(t + (p & ~7ll));
    unsigned sh = (unsigned)(p & 7) * 8;
    u64 lo = __ldg(w), hi = __ldg(w + 1);
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

// Which byte values occur (the code table needs presence only): 16-byte
// loads and one shared byte flag store per text byte (benign same-value
// races, no atomics), then one global atomicOr per present value and block.
__global__ void k_byte_present(const unsigned char *__restrict__ text, long long n, unsigned *__restrict__ present) {
    __shared__ unsigned s_flag[64];  // 256 byte flags
    if (threadIdx.x < 64) s_flag[threadIdx.x] = 0;
    __syncthreads();
    unsigned char *flag = reinterpret_cast<unsigned char *>(s_flag);
    const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const bool vec = ((unsigned long long)text & 15) == 0;
    const long long nv = vec ? n / 16 : 0;
    const uint4 *tv = reinterpret_cast<const uint4 *>(text);
    for (long long v = gid; v < nv; v += stride) {
        const uint4 q = tv[v];
        const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j) flag[(w[k] >> (8 * j)) & 0xff] = 1;
    }
    for (long long i = nv * 16 + gid; i < n; i += stride) flag[text[i]] = 1;
    __syncthreads();
    if (threadIdx.x < 256 && flag[threadIdx.x]) atomicOr(&present[threadIdx.x >> 5], 1u << (threadIdx.x & 31));
}

// Text -> big-endian bit stream of b-bit codes (one 64-bit word per thread),
// zero padded past the end.  Code table in shared memory (a table indexed by
// data in the parameter/constant space serialises divergent lanes); for
// b in {1, 2, 4, 8} a word covers whole 16-byte (8-byte) vectors of text.
__global__ void k_pack_text(const unsigned char *__restrict__ text, long long n, CodeTable ct, int b,
                            long long words, u64 *__restrict__ stream) {
    __shared__ unsigned char s_code[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_code[i] = (unsigned char)ct.code[i];
    __syncthreads();
    long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (w >= words) return;
    const long long bit0 = w * 64;
    const int cpw = 64 / b;  // codes per word when b divides 64
    const bool fast = (64 % b) == 0 && cpw >= 8 && ((unsigned long long)text & 15) == 0 &&
                      (w + 1) * (long long)cpw <= n;
    u64 x = 0;
    if (fast) {
        const unsigned char *src = text + w * (long long)cpw;
        int j = 0;
        for (int v = 0; v < cpw; v += 8) {  // 8 bytes per step (16-byte vectors pair up)
            const uint2 q = *reinterpret_cast<const uint2 *>(src + v);
#pragma unroll
            for (int k = 0; k < 8; ++k, ++j) {
                const unsigned byte = ((k < 4 ? q.x : q.y) >> (8 * (k & 3))) & 0xff;
                x |= (u64)s_code[byte] << (64 - b * (j + 1));
            }
        }
        stream[w] = x;
        return;
    }
    long long p = bit0 / b;
    for (; p * b < bit0 + 64; ++p) {
        const u64 code = p < n ? s_code[text[p]] : 0;
        const long long off = p * b - bit0;  // bit offset of this code's MSB within the word (may be < 0)
        const int sh = 64 - b - (int)off;     // left shift placing the code
        if (sh >= 0) x |= code << sh;
        else x |= code >> (-sh);
    }
    stream[w] = x;
}

// Round r >= 1 keys for the unsorted slots P[0..U): (group, lo) packed as
// group << lo_bits | lo, the group given either as its head slot or as its
// dense ordinal (the list is in slot order, so groups are consecutive runs
// of equal heads); both orders agree.
// During the doubling rounds the ISA entry of a suffix whose group is still
// tied carries this flag over its group head (slots are < 2^31); sorted
// suffixes hold their final slot.  Lets the round keys be built in text order.
constexpr unsigned kUnsortedBit = 0x80000000u;

__global__ void k_make_keys(const unsigned *__restrict__ G, const unsigned *__restrict__ V, long long U,
                            const unsigned *__restrict__ isa, long long n, long long h, int lo_bits,
                            u64 *__restrict__ keys, unsigned *__restrict__ vals) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= U) return;
    const unsigned i = V[t];
    // Suffixes shorter than h (padded with the smallest code) order by length
    // before every longer member of their group: lo = remaining length in
    // [1, h]; otherwise h + 1 + rank of suffix i + h.
    u64 lo = ((long long)i + h < n) ? (u64)(h + 1) + (isa[i + h] & ~kUnsortedBit) : (u64)(n - i);
    keys[t] = ((u64)G[t] << lo_bits) | lo;
    vals[t] = i;
}

// The same round keys built in TEXT order (large rounds: repetitive text keeps
// most suffixes tied for many rounds).  isa[i] (the group head, flagged while
// tied) and isa[i + h] are both read coalesced -- the list version gathers
// isa[i + h] at random, ~136 B of DRAM per 4-byte key on a 1 GiB text.  The
// tied suffixes are appended in any order (warp-aggregated counter): the sort
// orders them by (head, lo), and suffixes with equal keys stay tied.
constexpr int kMKNT = 256, kMKIPT = 4, kMKTile = kMKNT * kMKIPT;
__global__ void __launch_bounds__(kMKNT) k_make_keys_text(const unsigned *__restrict__ isa, long long n, long long h,
                                                        int lo_bits, u64 *__restrict__ keys,
                                                        unsigned *__restrict__ vals,
                                                        unsigned long long *__restrict__ counter) {
    __shared__ u64 s_key[kMKTile];
    __shared__ unsigned s_val[kMKTile];
    __shared__ unsigned s_warp[kMKNT / 32];
    __shared__ unsigned long long s_base;
    const long long i0 = (blockIdx.x * (long long)kMKNT + threadIdx.x) * kMKIPT;
    unsigned hd[kMKIPT];
    if (i0 + kMKIPT <= n) {
        const uint4 q = *reinterpret_cast<const uint4 *>(isa + i0);
        hd[0] = q.x, hd[1] = q.y, hd[2] = q.z, hd[3] = q.w;
    } else {
#pragma unroll
        for (int j = 0; j < kMKIPT; ++j) hd[j] = (i0 + j < n) ? isa[i0 + j] : 0u;
    }
    unsigned cnt = 0;
#pragma unroll
    for (int j = 0; j < kMKIPT; ++j) cnt += hd[j] >> 31;
    unsigned excl;
    const unsigned total = block_exclusive_sum<kMKNT>(cnt, excl, s_warp);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(counter, (unsigned long long)total) : 0;
#pragma unroll
    for (int j = 0; j < kMKIPT; ++j) {
        if (!(hd[j] & kUnsortedBit)) continue;
        const long long i = i0 + j;
        const u64 lo = (i + h < n) ? (u64)(h + 1) + (isa[i + h] & ~kUnsortedBit) : (u64)(n - i);
        s_key[excl] = ((u64)(hd[j] & ~kUnsortedBit) << lo_bits) | lo;
        s_val[excl] = (unsigned)i;
        ++excl;
    }
    __syncthreads();
    const unsigned long long base = s_base;
    for (unsigned t = threadIdx.x; t < total; t += kMKNT) {
        keys[base + t] = s_key[t];
        vals[base + t] = s_val[t];
    }
}

// Dense ordinal of each list entry's group (runs of equal heads): exclusive
// count of run starts, block scan + decoupled look-back; total -> *groups.
// 32 entries per thread: one look-back per 8192 entries (8 per thread left the
// tiles waiting on their predecessors)
constexpr int kGNT = 256, kGIPT = 32, kGTile = kGNT * kGIPT;
__global__ void __launch_bounds__(kGNT) k_group_ordinals(const unsigned *__restrict__ H, long long U,
                                                       unsigned *__restrict__ G, unsigned long long *groups,
                                                       unsigned *counter, u64 *status, long long tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[kGNT / 32];
    __shared__ u64 s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long t0 = tile * kGTile + (long long)threadIdx.x * kGIPT;
    unsigned starts = 0, cnt = 0;
    unsigned prev = (t0 > 0 && t0 - 1 < U) ? H[t0 - 1] : 0xffffffffu;
    unsigned hv[kGIPT];
    const bool full = t0 + kGIPT <= U;
    if (full) {  // 16-byte loads
        const uint4 *q = reinterpret_cast<const uint4 *>(H + t0);
#pragma unroll
        for (int w = 0; w < kGIPT / 4; ++w) {
            const uint4 a = q[w];
            hv[4 * w] = a.x; hv[4 * w + 1] = a.y; hv[4 * w + 2] = a.z; hv[4 * w + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kGIPT; ++j) hv[j] = t0 + j < U ? H[t0 + j] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kGIPT; ++j) {
        const long long t = t0 + j;
        if (t < U) {
            const bool f = t == 0 || hv[j] != prev;
            starts |= (unsigned)f << j;
            cnt += f;
            prev = hv[j];
        }
    }
    unsigned excl;
    const unsigned tot = block_exclusive_sum<kGNT>(cnt, excl, s_warp);
    if (threadIdx.x < 32) {
        const u64 base = lookback_warp(status, tile, (u64)tot, OpSum());
        if (threadIdx.x == 0) {
            s_base = base;
            if (tile == tiles - 1) *groups = base + tot;
        }
    }
    __syncthreads();
    u64 g = s_base + excl;  // run starts before this thread's items
    unsigned gv[kGIPT];
#pragma unroll
    for (int j = 0; j < kGIPT; ++j) {
        if (starts >> j & 1) ++g;
        gv[j] = (unsigned)(g - 1);
    }
    if (full) {
        uint4 *q = reinterpret_cast<uint4 *>(G + t0);
#pragma unroll
        for (int w = 0; w < kGIPT / 4; ++w) q[w] = make_uint4(gv[4 * w], gv[4 * w + 1], gv[4 * w + 2], gv[4 * w + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < kGIPT; ++j)
            if (t0 + j < U) G[t0 + j] = gv[j];
    }
}

constexpr int kUNT = 256;
constexpr int kUIPT = 8;
constexpr int kUTile = kUNT * kUIPT;

// LCP of two suffixes from their packed K-symbol keys (codes 0..sigma-1, the
// smallest code also pads past the end), capped by their remaining lengths.
// Equal keys with both suffixes >= K long: unknown (>= K), fixed later.
__device__ __forceinline__ unsigned key_lcp(u64 a, u64 b, int code_bits, int key_bits, unsigned K,
                                            unsigned rem_a, unsigned rem_b) {
    const u64 x = a ^ b;
    const unsigned m = rem_a < rem_b ? rem_a : rem_b;
    if (x) {
        const unsigned z = (unsigned)(__clzll((long long)x) - (64 - key_bits));
        // code_bits is 2 for DNA: avoid the integer division there
        const unsigned l = code_bits == 2 ? z >> 1 : (code_bits == 1 ? z : z / (unsigned)code_bits);
        return l < m ? l : m;
    }
    return m < K ? m : kLcpUnknown;
}

// Write back one sorted run of (key, suffix) pairs occupying SA slots Pos(t)
// (P[t], or t itself in round 0 when P is null): sa[Pos(t)] = suffix,
// isa[suffix] = SA slot of its new group head, and the slots still in
// non-singleton groups are compacted into P_next.
template <typename KeyT>
__device__ __forceinline__ void load_keys(const KeyT *__restrict__ keys, long long t0, long long U, u64 *k) {
    if (t0 + kUIPT <= U) {
        if (sizeof(KeyT) == 8) {
            const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(keys + t0);
#pragma unroll
            for (int j = 0; j < kUIPT / 2; ++j) {
                ulonglong2 q = p[j];
                k[2 * j] = q.x;
                k[2 * j + 1] = q.y;
            }
        } else {
            const uint4 *p = reinterpret_cast<const uint4 *>(keys + t0);
#pragma unroll
            for (int j = 0; j < kUIPT / 4; ++j) {
                uint4 q = p[j];
                k[4 * j] = q.x;
                k[4 * j + 1] = q.y;
                k[4 * j + 2] = q.z;
                k[4 * j + 3] = q.w;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < kUIPT; ++j) k[j] = (t0 + j < U) ? (u64)keys[t0 + j] : ~0ull;
    }
}

// u32 keys: 5 CTAs/SM (a few spilled bytes, measured 2.34 -> 2.26 ms on C3);
// u64 keys stay at 4 (5 measured slower)
template <bool REDUCE, typename KeyT>
__global__ void __launch_bounds__(kUNT, sizeof(KeyT) == 4 ? 5 : 4) k_update(const KeyT *__restrict__ keys, const unsigned *__restrict__ vals,
                                                 const unsigned *__restrict__ P, long long U,
                                                 unsigned *__restrict__ sa, unsigned *__restrict__ isa,
                                                 unsigned *__restrict__ P_next, unsigned *__restrict__ H_next,
                                                 unsigned *__restrict__ V_next, u64 *__restrict__ tile_agg,
                                                 const u64 *__restrict__ tile_prefix,
                                                 unsigned *__restrict__ lcp_d, int code_bits, int key_bits,
                                                 BucketEmit be, SegBoundary sb) {
    __shared__ u64 s_warp[kUNT / 32];
    __shared__ unsigned s_warp32[kUNT / 32];
    __shared__ u64 s_head_prefix;
    __shared__ u64 s_base;
    __shared__ EmitSmem<kUNT, kUIPT> s_emit;
    const long long tile = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const long long t0 = tile * kUTile + (long long)threadIdx.x * kUIPT;
    u64 k[kUIPT];
    load_keys<KeyT>(keys, t0, U, k);
    u64 kprev = __shfl_up_sync(0xffffffffu, k[kUIPT - 1], 1);
    u64 knext = __shfl_down_sync(0xffffffffu, k[0], 1);
    if (lane == 0) kprev = (t0 > 0 && t0 - 1 < U) ? (u64)keys[t0 - 1] : 0;
    if (lane == 31) knext = (t0 + kUIPT < U) ? (u64)keys[t0 + kUIPT] : 0;
    // Round 0: a suffix shorter than K symbols (padded key) may tie with the
    // longer suffixes it is a prefix of.  It sorts first among them (the input
    // order puts short suffixes first, shortest first) and stays there, so the
    // key LCPs next to it (capped by its length) are final; the group is then
    // resolved like any other (the direct comparison stops at its end, later
    // rounds key it by its length).
    bool newf[kUIPT + 1];
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        newf[j] = (t == 0) || (k[j] != (j ? k[j - 1] : kprev));
    }
    newf[kUIPT] = (t0 + kUIPT >= U) || (knext != k[kUIPT - 1]);
#pragma unroll
    for (int j = 0; j < kUIPT; ++j)
        if (t0 + j + 1 == U) newf[j + 1] = true;

    unsigned pos[kUIPT];
    u64 hmax = 0;
    unsigned unsorted = 0, ucnt = 0;
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        pos[j] = 0;
        if (t < U) {
            pos[j] = P ? P[t] : (unsigned)t;
            if (newf[j]) hmax = (u64)pos[j];
            bool un = !(newf[j] && newf[j + 1]);
            unsorted |= (unsigned)un << j;
            ucnt += un;
        }
    }
    u64 incl;
    const u64 tile_max = block_inclusive_max64<kUNT>(hmax, incl, s_warp);
    const u64 excl_in_block = __shfl_up_sync(0xffffffffu, incl, 1);
    unsigned excl_u;
    const unsigned utotal = block_exclusive_sum<kUNT>(ucnt, excl_u, s_warp32);
    if (REDUCE) {
        // pass 1 of reduce-then-scan: this tile's (max head, unsorted count)
        if (threadIdx.x == 0) tile_agg[tile] = (tile_max << 31) | (u64)utotal;
        return;
    }
    if (threadIdx.x == 0) {
        const u64 both = tile_prefix[tile];  // exclusive (max, sum) over earlier tiles
        s_head_prefix = both >> 31;
        s_base = both & ((1ull << 31) - 1);
    }
    __syncthreads();
    // exclusive max for this thread = max(tile prefix, inclusive value of previous thread)
    u64 run = s_head_prefix;
    {
        const int warp = threadIdx.x >> 5;
        u64 prev_incl = (lane > 0) ? excl_in_block : (warp ? s_warp[warp - 1] : 0);
        if (threadIdx.x > 0 && prev_incl > run) run = prev_incl;
    }
    u64 o = s_base + excl_u;
    unsigned vv[kUIPT], hh[kUIPT];
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        vv[j] = kNoDest;
        hh[j] = 0;
        if (t >= U) continue;
        if (newf[j]) run = pos[j];
        unsigned v = vals[t];
        vv[j] = v;
        hh[j] = (unsigned)run | ((unsorted >> j & 1) ? kUnsortedBit : 0u);  // ISA value (flag: still tied)
        if (P) {
            sa[pos[j]] = v;
            if (!be.stage) isa[v] = hh[j];
        }
        if (unsorted >> j & 1) {
            // next round's inputs: slot, group head (= new isa) and suffix,
            // so k_make_keys needs only the one random gather isa[i + h]
            P_next[o] = pos[j];
            if (H_next) {  // null: the next round builds its keys in text order
                H_next[o] = (unsigned)run;
                V_next[o] = v;
            }
            ++o;
        }
    }
    if (sb.group_count) {  // still-tied groups (sizes the next round's keys)
        unsigned gs = 0;
#pragma unroll
        for (int j = 0; j < kUIPT; ++j) gs += (t0 + j < U) && newf[j] && (unsorted >> j & 1);
        gs = __reduce_add_sync(0xffffffffu, gs);
        if (lane == 0 && gs) atomicAdd(sb.group_count, (unsigned long long)gs);
    }
    if (P) {
        if (be.stage) {  // large later rounds: ISA through the bucketed scatter too
            __syncthreads();
            bucket_emit<kUNT, kUIPT>(be, vv, hh, s_emit);
        }
        return;
    }
    // ---- round 0: SA slots are t itself -> each thread stores its 8 slots as
    //      two 16-byte vectors (a warp covers 1 KB contiguously) ----
    //      (sa == null: the sorted suffix array itself becomes the SA)
    const bool full = t0 + kUIPT <= U;
    if (sa) {
        if (full) {
            uint4 *d = reinterpret_cast<uint4 *>(sa + t0);
            d[0] = make_uint4(vv[0], vv[1], vv[2], vv[3]);
            d[1] = make_uint4(vv[4], vv[5], vv[6], vv[7]);
        } else {
#pragma unroll
            for (int j = 0; j < kUIPT; ++j)
                if (t0 + j < U) sa[t0 + j] = vv[j];
        }
    }
    // LCP of adjacent suffixes from their packed K-symbol keys (capped by the
    // suffix lengths); kLcpUnknown (true LCP >= K) when undecided.
    const unsigned K = (unsigned)(key_bits / code_bits);
    unsigned vprev = __shfl_up_sync(0xffffffffu, vv[kUIPT - 1], 1);
    unsigned vnext = __shfl_down_sync(0xffffffffu, vv[0], 1);
    if (lane == 0) vprev = t0 > 0 ? vals[t0 - 1] : 0;
    if (lane == 31) vnext = (t0 + kUIPT < U) ? vals[t0 + kUIPT] : 0;
    // text length (remaining lengths cap the key LCPs); U == n unless this is
    // one rank's segment of a distributed sort, whose first slot and the slot
    // after its last hold the LCPs with the neighbouring segments (sb)
    const unsigned nn = (unsigned)sb.n_text;
    unsigned lk[kUIPT + 1];
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        long long t = t0 + j;
        const unsigned vp = j ? vv[j - 1] : vprev;
        lk[j] = (t > 0 && t < U) ? key_lcp(k[j], j ? k[j - 1] : kprev, code_bits, key_bits, K, nn - vv[j], nn - vp)
                : t == 0 ? sb.lcp_first : sb.lcp_last;
    }
    lk[kUIPT] = (t0 + kUIPT < U)
                    ? key_lcp(knext, k[kUIPT - 1], code_bits, key_bits, K, nn - vnext, nn - vv[kUIPT - 1])
                    : sb.lcp_last;
    if (full) {
        uint4 *d = reinterpret_cast<uint4 *>(lcp_d + t0);
        d[0] = make_uint4(lk[0], lk[1], lk[2], lk[3]);
        d[1] = make_uint4(lk[4], lk[5], lk[6], lk[7]);
    } else {
#pragma unroll
        for (int j = 0; j < kUIPT; ++j)
            if (t0 + j < U) lcp_d[t0 + j] = lk[j];
    }
    // raw LLR candidate of each suffix: max(LCP with SA predecessor, with
    // successor); still-unknown pairs count as 0 and are fixed by k_lcp_patch
    // (every suffix of a tied group is next to one such pair).
    unsigned rr[kUIPT];
#pragma unroll
    for (int j = 0; j < kUIPT; ++j) {
        unsigned a = lk[j] == kLcpUnknown ? 0 : lk[j];
        unsigned b = lk[j + 1] == kLcpUnknown ? 0 : lk[j + 1];
        rr[j] = a > b ? a : b;
    }
    __syncthreads();
    if (be.stage2) {
        bucket_emit<kUNT, kUIPT>(be, vv, hh, s_emit, rr);  // (ISA, raw) into text order
    } else {
        // raw only (ISA is filled from SA if ever needed); the tied suffixes'
        // raw is emitted by k_small_groups into the same buckets
#pragma unroll
        for (int j = 0; j < kUIPT; ++j)
            if (unsorted >> j & 1) hh[j] = kNoDest;
            else hh[j] = vv[j];
        bucket_emit<kUNT, kUIPT>(be, hh, rr, s_emit);
    }
}

// Pass 2 of reduce-then-scan over the k_update tiles: exclusive OpMaxSum
// prefix per tile and the total unsorted count.  256 threads x 4 aggregates
// per block, block scan, decoupled look-back across blocks (a single-block
// scan was latency-bound at ~0.25 ms for 131k tiles).
constexpr int kTSNT = 256, kTSIPT = 4, kTSTile = kTSNT * kTSIPT;
__global__ void __launch_bounds__(kTSNT) k_tile_scan_lb(const u64 *__restrict__ agg, long long tiles,
                                                        u64 *__restrict__ prefix, unsigned long long *U_next,
                                                        unsigned *counter, u64 *status, long long blocks) {
    __shared__ unsigned s_blk;
    __shared__ u64 s_warp[kTSNT / 32];
    __shared__ u64 s_base;
    const OpMaxSum op;
    if (threadIdx.x == 0) s_blk = atomicAdd(counter, 1u);
    __syncthreads();
    const long long blk = s_blk;
    const long long i0 = blk * kTSTile + (long long)threadIdx.x * kTSIPT;
    u64 v[kTSIPT], acc = 0;
#pragma unroll
    for (int j = 0; j < kTSIPT; ++j) {
        v[j] = i0 + j < tiles ? agg[i0 + j] : 0ull;
        acc = op(acc, v[j]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u64 x = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = op(x, y);
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        u64 w = lane < kTSNT / 32 ? s_warp[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u64 y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w = op(w, y);
        }
        if (lane < kTSNT / 32) s_warp[lane] = w;
        const u64 total = __shfl_sync(0xffffffffu, w, kTSNT / 32 - 1);
        const u64 base = lookback_warp(status, blk, total, op);
        if (lane == 0) {
            s_base = base;
            if (blk == blocks - 1) *U_next = op(base, total) & ((1ull << 31) - 1);
        }
    }
    __syncthreads();
    // exclusive prefix of this thread's first aggregate
    u64 run = op(s_base, warp ? s_warp[warp - 1] : 0ull);
    const u64 xprev = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane) run = op(run, xprev);
#pragma unroll
    for (int j = 0; j < kTSIPT; ++j) {
        if (i0 + j < tiles) prefix[i0 + j] = run;
        run = op(run, v[j]);
    }
}

// 64 bits of the packed symbol stream starting at symbol p.
__device__ __forceinline__ u64 load_sym64(const u64 *__restrict__ stream, int b, long long p) {
    const long long o = (long long)b * p;
    const u64 *w = stream + (o >> 6);
    const unsigned sh = (unsigned)(o & 63);
    const u64 lo = __ldg(w);
    return sh ? (lo << sh) | (__ldg(w + 1) >> (64 - sh)) : lo;
}

// Common prefix length of the suffixes at i and j, starting the comparison at
// offset h0 and capped by lim = n - max(i, j).  Compares 64 / b symbols per
// step on the packed stream (code equality == byte equality; the stream is
// L2-resident at 256 Mi DNA), instead of 8 bytes of the raw text.
__device__ __forceinline__ long long packed_lcp(const u64 *__restrict__ stream, int b, long long i, long long j,
                                                long long h0, long long lim) {
    long long h = h0;
    const int per = 64 / b;
    while (h < lim) {
        const u64 x = load_sym64(stream, b, i + h) ^ load_sym64(stream, b, j + h);
        if (x == 0) {
            h += per;
        } else {
            h += __clzll((long long)x) / b;
            break;
        }
    }
    return h > lim ? lim : h;
}

// LCP of the adjacent suffixes at SA slots r-1, r, known to be >= K.
__device__ __forceinline__ unsigned lcp_from_depth(const u64 *__restrict__ stream, int b,
                                                   const unsigned *__restrict__ sa, long long n, long long K,
                                                   long long r) {
    const long long a = sa[r - 1], c = sa[r];
    const long long lim = n - (a > c ? a : c);
    return (unsigned)packed_lcp(stream, b, a, c, K < lim ? K : lim, lim);
}

// Adjacent pairs whose round-0 keys were equal: lcp >= K, finished by 8-byte
// word compares from depth K.  The raw LLR of both suffixes of a patched pair
// is recomputed here; a neighbouring pair that is itself still unknown is
// computed redundantly (the same value its own thread writes), so threads
// need no ordering.
// slots: the SA slots of the suffixes tied after round 0 (only their pairs can
// be unknown), or null to scan every slot.
__global__ void k_lcp_patch(const u64 *__restrict__ stream, int b, const unsigned *__restrict__ sa, long long n,
                            long long K, unsigned *__restrict__ lcp_d, unsigned *__restrict__ raw,
                            const unsigned *__restrict__ slots, long long nslots) {
    long long stride = (long long)gridDim.x * blockDim.x;
    const long long total = slots ? nslots : n;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x + (slots ? 0 : 1); q < total; q += stride) {
        const long long r = slots ? (long long)slots[q] : q;
        if (r < 1 || lcp_d[r] != kLcpUnknown) continue;
        const unsigned h = lcp_from_depth(stream, b, sa, n, K, r);
        lcp_d[r] = h;
        unsigned lp = lcp_d[r - 1];
        if (lp == kLcpUnknown) lp = lcp_from_depth(stream, b, sa, n, K, r - 1);
        unsigned ln = lcp_d[r + 1];
        if (ln == kLcpUnknown) ln = lcp_from_depth(stream, b, sa, n, K, r + 1);
        raw[sa[r - 1] + 1] = lp > h ? lp : h;
        raw[sa[r] + 1] = h > ln ? h : ln;
    }
}

// isa[V[t]] = H[t] (flagged): members of groups still tied keep their group head.
__global__ void k_isa_heads(const unsigned *__restrict__ V, const unsigned *__restrict__ H, long long U,
                            unsigned *__restrict__ isa) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t < U) isa[V[t]] = H[t] | kUnsortedBit;
}

// ---- small tied groups after round 0 ------------------------------------
// Suffixes whose round-0 keys are equal share their first K symbols.  On
// i.i.d.-like text these groups have 2-3 members: sorting each one directly by
// comparing the suffixes on the packed stream (from depth K) gives their final
// order AND the LCPs between them, which replaces a whole doubling round
// (keys, 64-bit radix sort, update) and the LCP patch for them.  Larger groups
// stay in the list for the doubling rounds.
constexpr int kSmallGroup = 8;

// suffix a < suffix c, given >= K equal leading symbols; l = their LCP.  The
// 64-bit windows are big-endian code strings, so at the first difference the
// smaller window is the smaller suffix (no extra symbol loads).
__device__ __forceinline__ bool suffix_less(const u64 *__restrict__ stream, int b, long long n, long long K,
                                            unsigned a, unsigned c, unsigned &l) {
    const long long lim = n - (long long)(a > c ? a : c);
    long long h = K < lim ? K : lim;
    const int per = 64 / b;
    while (h < lim) {
        const u64 wa = load_sym64(stream, b, (long long)a + h), wc = load_sym64(stream, b, (long long)c + h);
        const u64 x = wa ^ wc;
        if (x == 0) {
            h += per;
            continue;
        }
        h += __clzll((long long)x) / b;
        if (h >= lim) break;  // first difference lies past the end of the shorter suffix
        l = (unsigned)h;
        return wa < wc;
    }
    l = (unsigned)lim;
    return a > c;  // one is a prefix of the other: the shorter (later start) sorts first
}

// One thread per list entry (groups are runs of equal heads; a group's slots
// are head .. head+s-1).  Each entry classifies its group by looking at most
// kSmallGroup entries each way; the first entry of a small group sorts it.
// keep[t] = 1 marks entries of groups left to the doubling rounds.  The raw
// LLR corrections (text order, random) leave through the bucketed scatter:
// each member's (suffix, raw) is handed to its own entry's thread in shared
// memory and the block emits them together (be; applied after round 0's raw).
constexpr int kSGNT = 256;
__device__ __forceinline__ void sg_put(long long e, long long tb, unsigned v, unsigned r, unsigned *s_dest,
                                       unsigned *s_val, unsigned *__restrict__ raw) {
    if (e - tb < kSGNT) {
        s_dest[e - tb] = v;
        s_val[e - tb] = r;
    } else {
        raw[v + 1] = r;  // member beyond this block (rare): direct store
    }
}

__global__ void __launch_bounds__(kSGNT) k_small_groups(const unsigned *__restrict__ P,
                                                        const unsigned *__restrict__ H,
                                                        const unsigned *__restrict__ V, long long U,
                                                        const u64 *__restrict__ stream, int b, long long n,
                                                        long long K, unsigned *__restrict__ sa,
                                                        unsigned *__restrict__ isa, unsigned *__restrict__ lcp_d,
                                                        unsigned *__restrict__ raw, unsigned *__restrict__ keep,
                                                        BucketEmit be) {
    __shared__ EmitSmem<kSGNT, 1> s_emit;
    __shared__ unsigned s_dest[kSGNT], s_val[kSGNT];
    const long long tb = blockIdx.x * (long long)kSGNT;
    const long long t = tb + threadIdx.x;
    s_dest[threadIdx.x] = kNoDest;
    __syncthreads();
    if (t < U) {
        const unsigned head = H[t];
        int back = 0, fwd = 0;
        while (back < kSmallGroup && t - back - 1 >= 0 && H[t - back - 1] == head) ++back;
        while (fwd < kSmallGroup && t + fwd + 1 < U && H[t + fwd + 1] == head) ++fwd;
        const bool small = back + fwd + 1 <= kSmallGroup;
        keep[t] = small ? 0u : 1u;
        if (!small) {  // left to the doubling rounds: round-0 raw candidate (unknown LCPs as 0)
            const unsigned slot = P[t];
            unsigned a = lcp_d[slot], c2 = lcp_d[slot + 1];
            a = a == kLcpUnknown ? 0u : a;
            c2 = c2 == kLcpUnknown ? 0u : c2;
            s_dest[threadIdx.x] = V[t];
            s_val[threadIdx.x] = a > c2 ? a : c2;
        }
        if (small && !back) {
            const int s = fwd + 1;
            const unsigned lb = lcp_d[head];  // group boundaries: keys differ there, LCP known from round 0
            if (s == 2) {
                // round 0 left sa[head..head+1] = (x, y), isa = head for both, and
                // raw without the (unknown) inner LCP; write only what changes
                const unsigned x = V[t], y = V[t + 1];
                const unsigned le = lcp_d[head + 2];
                unsigned l;
                const bool swap = suffix_less(stream, b, n, K, y, x, l);
                const unsigned first = swap ? y : x, second = swap ? x : y;
                if (swap) {
                    sa[head] = y;
                    sa[head + 1] = x;
                    if (isa) isa[y] = head;
                }
                if (isa) isa[second] = head + 1;
                lcp_d[head + 1] = l;
                sg_put(t, tb, first, lb > l ? lb : l, s_dest, s_val, raw);
                sg_put(t + 1, tb, second, l > le ? l : le, s_dest, s_val, raw);
            } else {
                unsigned v[kSmallGroup];
                unsigned lc[kSmallGroup + 1];
                lc[0] = lb;
                lc[s] = lcp_d[head + s];
                for (int j = 0; j < s; ++j) v[j] = V[t + j];
                unsigned l;
                for (int i = 1; i < s; ++i) {  // insertion sort by suffix comparison
                    const unsigned x = v[i];
                    int j = i;
                    while (j > 0 && suffix_less(stream, b, n, K, x, v[j - 1], l)) {
                        v[j] = v[j - 1];
                        --j;
                    }
                    v[j] = x;
                }
                for (int j = 1; j < s; ++j) {
                    suffix_less(stream, b, n, K, v[j - 1], v[j], l);
                    lc[j] = l;
                }
                for (int j = 0; j < s; ++j) {
                    const unsigned slot = head + j;
                    sa[slot] = v[j];
                    if (isa) isa[v[j]] = slot;
                    if (j) lcp_d[slot] = lc[j];
                    sg_put(t + j, tb, v[j], lc[j] > lc[j + 1] ? lc[j] : lc[j + 1], s_dest, s_val, raw);
                }
            }
        }
    }
    __syncthreads();
    const unsigned d = s_dest[threadIdx.x], vl = s_val[threadIdx.x];
    bucket_emit<kSGNT, 1>(be, &d, &vl, s_emit);
}

// Distributed-segment variant of k_small_groups: no direct raw stores at all
// (a rank holds no global raw array).  keep[t] = 1 marks entries of groups left to
// the doubling rounds.  Raw LLR (text order, random) leaves through the
// bucketed scatter: each member's (suffix, raw) is handed to its own entry's
// thread in shared memory and the block emits them together; a group that
// began in the previous block is re-sorted by this block's first thread for
// its members here (identical result), so no member is ever stored directly.

__global__ void __launch_bounds__(kSGNT) k_small_groups_seg(const unsigned *__restrict__ P,
                                                        const unsigned *__restrict__ H,
                                                        const unsigned *__restrict__ V, long long U,
                                                        const u64 *__restrict__ stream, int b, long long n,
                                                        long long K, unsigned *__restrict__ sa,
                                                        unsigned *__restrict__ isa, unsigned *__restrict__ lcp_d,
                                                        unsigned *__restrict__ keep, BucketEmit be) {
    __shared__ EmitSmem<kSGNT, 1> s_emit;
    __shared__ unsigned s_dest[kSGNT], s_val[kSGNT];
    const long long tb = blockIdx.x * (long long)kSGNT;
    const long long t = tb + threadIdx.x;
    s_dest[threadIdx.x] = kNoDest;
    __syncthreads();
    if (t < U) {
        const unsigned head = H[t];
        int back = 0, fwd = 0;
        while (back < kSmallGroup && t - back - 1 >= 0 && H[t - back - 1] == head) ++back;
        while (fwd < kSmallGroup && t + fwd + 1 < U && H[t + fwd + 1] == head) ++fwd;
        const bool small = back + fwd + 1 <= kSmallGroup;
        keep[t] = small ? 0u : 1u;  // larger groups: k_large_groups_seg sorts and emits them
        const bool starter = small && back == 0;
        if (starter || (small && back > 0 && t == tb)) {
            const long long g0 = t - back;  // first entry of the group
            const int s = back + fwd + 1;
            const unsigned lb = lcp_d[head];  // group boundaries: keys differ there, LCP known from round 0
            const unsigned le = lcp_d[head + s];
            if (s == 2) {  // the common case, in registers
                unsigned x = V[g0], y = V[g0 + 1], l;
                const bool moved = suffix_less(stream, b, n, K, y, x, l);
                if (moved) {
                    const unsigned z = x;
                    x = y;
                    y = z;
                }
                if (starter) {  // round 0 left the pair in input order, ISA = head for both
                    if (moved) {
                        sa[head] = x;
                        sa[head + 1] = y;
                        if (isa) isa[x] = head;
                    }
                    if (isa) isa[y] = head + 1;
                    lcp_d[head + 1] = l;
                }
                if (g0 >= tb) {
                    s_dest[g0 - tb] = x;
                    s_val[g0 - tb] = lb > l ? lb : l;
                }
                if (g0 + 1 < tb + kSGNT) {
                    s_dest[g0 + 1 - tb] = y;
                    s_val[g0 + 1 - tb] = l > le ? l : le;
                }
            } else {
                unsigned v[kSmallGroup];
                unsigned lc[kSmallGroup + 1];
                lc[0] = lb;
                lc[s] = le;
                for (int j = 0; j < s; ++j) v[j] = V[g0 + j];
                unsigned l;
                for (int i = 1; i < s; ++i) {  // insertion sort by suffix comparison
                    const unsigned x = v[i];
                    int j = i;
                    while (j > 0 && suffix_less(stream, b, n, K, x, v[j - 1], l)) {
                        v[j] = v[j - 1];
                        --j;
                    }
                    v[j] = x;
                }
                for (int j = 1; j < s; ++j) {
                    suffix_less(stream, b, n, K, v[j - 1], v[j], l);
                    lc[j] = l;
                }
                for (int j = 0; j < s; ++j) {
                    if (starter) {
                        const unsigned slot = head + j;
                        sa[slot] = v[j];
                        if (isa) isa[v[j]] = slot;
                        if (j) lcp_d[slot] = lc[j];
                    }
                    const long long e = g0 + j;
                    if (e >= tb && e < tb + kSGNT) {
                        s_dest[e - tb] = v[j];
                        s_val[e - tb] = lc[j] > lc[j + 1] ? lc[j] : lc[j + 1];
                    }
                }
            }
        }
    }
    __syncthreads();
    const unsigned d = s_dest[threadIdx.x], vl = s_val[threadIdx.x];
    bucket_emit<kSGNT, 1>(be, &d, &vl, s_emit);
}

// Order-preserving compaction of the (slot, head, suffix) lists to the kept
// entries: block scan + decoupled look-back, one pass.
constexpr int kKNT = 256, kKIPT = 8, kKTile = kKNT * kKIPT;
__global__ void __launch_bounds__(kKNT) k_keep_compact(const unsigned *__restrict__ keep, const unsigned *__restrict__ P,
                                                     const unsigned *__restrict__ H, const unsigned *__restrict__ V,
                                                     long long U, unsigned *__restrict__ P2, unsigned *__restrict__ H2,
                                                     unsigned *__restrict__ V2, unsigned long long *total,
                                                     unsigned *counter, u64 *status, long long tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[kKNT / 32];
    __shared__ u64 s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long i0 = tile * kKTile + (long long)threadIdx.x * kKIPT;
    unsigned flags = 0, cnt = 0;
#pragma unroll
    for (int j = 0; j < kKIPT; ++j) {
        const bool f = i0 + j < U && keep[i0 + j];
        flags |= (unsigned)f << j;
        cnt += f;
    }
    unsigned excl;
    const unsigned tot = block_exclusive_sum<kKNT>(cnt, excl, s_warp);
    if (threadIdx.x < 32) {
        const u64 base = lookback_warp(status, tile, (u64)tot, OpSum());
        if (threadIdx.x == 0) {
            s_base = base;
            if (tile == tiles - 1) *total = base + tot;
        }
    }
    __syncthreads();
    u64 o = s_base + excl;
#pragma unroll
    for (int j = 0; j < kKIPT; ++j) {
        if (flags >> j & 1) {
            P2[o] = P[i0 + j];
            H2[o] = H[i0 + j];
            V2[o] = V[i0 + j];
            ++o;
        }
    }
}

// phi[sa[j]] = sa[j-1] (kNone for j = 0)
__global__ void k_phi(const unsigned *__restrict__ sa, long long n, unsigned *__restrict__ phi) {
    long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j >= n) return;
    phi[sa[j]] = j ? sa[j - 1] : kNone;
}

// PLCP[i] = lcp(i, phi[i]) from scratch, one thread per position (short LCPs).
__global__ void k_plcp_flat(const u64 *__restrict__ stream, int b, const unsigned *__restrict__ phi, long long n,
                            unsigned *__restrict__ plcp) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned j = phi[i];
    if (j == kNone) {
        plcp[i] = 0;
        return;
    }
    const long long lim = n - (i > (long long)j ? i : (long long)j);
    plcp[i] = (unsigned)packed_lcp(stream, b, i, (long long)j, 0, lim);
}

// Kasai over text-order chunks: PLCP[i] = lcp(i, phi[i]); carry h-1 within a chunk.
__global__ void k_plcp(const unsigned char *__restrict__ text, const u64 *__restrict__ stream, int b,
                       const unsigned *__restrict__ phi, long long n, long long chunk, unsigned *__restrict__ plcp) {
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
        if (stream) {
            h = packed_lcp(stream, b, i, (long long)j, h, lim);
        } else {
            while (h < lim) {
                u64 x = load8(text, i + h) ^ load8(text, (long long)j + h);
                if (x == 0) {
                    h += 8;
                } else {
                    h += (__ffsll((long long)x) - 1) >> 3;
                    break;
                }
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

// ---- distributed suffix sort -------------------------------
// Order-preserving filter of the round-0 (key, suffix) pairs, in sort input
// order, whose top key digit lies in [dlo, dhi): one rank's share of the
// suffixes (MSD split by the top digit).  Block scan + decoupled look-back.
constexpr int kFNT = 256, kFIPT = 8, kFTile = kFNT * kFIPT;
__global__ void __launch_bounds__(kFNT) k_filter_keys(TextKeys tk, long long count, int top_shift, unsigned dlo,
                                                      unsigned dhi, unsigned *__restrict__ keys,
                                                      unsigned *__restrict__ vals, unsigned long long *total,
                                                      unsigned *counter, u64 *status, long long tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[kFNT / 32];
    __shared__ u64 s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long e0 = tile * kFTile + (long long)threadIdx.x * kFIPT;
    unsigned k[kFIPT], v[kFIPT], flags = 0, cnt = 0;
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) {
        const long long e = e0 + j;
        bool f = false;
        if (e < count) {
            const long long pos = text_pos(tk, e);
            k[j] = (unsigned)text_key(tk, pos);
            v[j] = (unsigned)pos;
            const unsigned d = (k[j] >> top_shift) & 0xffu;
            f = d >= dlo && d < dhi;
        }
        flags |= (unsigned)f << j;
        cnt += f;
    }
    unsigned excl;
    const unsigned tot = block_exclusive_sum<kFNT>(cnt, excl, s_warp);
    if (threadIdx.x < 32) {
        const u64 base = lookback_warp(status, tile, (u64)tot, OpSum());
        if (threadIdx.x == 0) {
            s_base = base;
            if (tile == tiles - 1) *total = base + tot;
        }
    }
    __syncthreads();
    u64 o = s_base + excl;
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) {
        if (flags >> j & 1) {
            keys[o] = k[j];
            vals[o] = v[j];
            ++o;
        }
    }
}

// The staged (position, raw) entries of each bucket, concatenated in bucket
// order (= destination-rank order) into the send buffer; blockIdx.x = chunk
// of 4096 entries, blockIdx.y = bucket.
__global__ void k_pack_send(const uint2 *__restrict__ stage, const unsigned *__restrict__ cursor, int shift,
                            const long long *__restrict__ off, uint2 *__restrict__ send) {
    const long long b = blockIdx.y;
    const unsigned cnt = cursor[b * kCursorStride];
    const unsigned begin = blockIdx.x * 4096u;
    if (begin >= cnt) return;
    const unsigned end = cnt - begin < 4096u ? cnt : begin + 4096u;
    const uint2 *src = stage + (b << shift);
    uint2 *dst = send + off[b];
    for (unsigned i = begin + threadIdx.x; i < end; i += blockDim.x) dst[i] = src[i];
}

// Received (position, raw) entries -> this rank's raw shard (raw[i] at
// rawbuf[i - R0]); max raw for the halo width (one atomic per block).
constexpr int kARNT = 256, kARIPT = 8;
__global__ void __launch_bounds__(kARNT) k_apply_recv(const uint2 *__restrict__ recv, long long cnt, long long R0,
                                                      unsigned *__restrict__ rawbuf, unsigned *maxraw) {
    __shared__ unsigned s_max[kARNT / 32];
    const long long i0 = blockIdx.x * (long long)(kARNT * kARIPT) + threadIdx.x;
    uint2 e[kARIPT];
#pragma unroll
    for (int j = 0; j < kARIPT; ++j) {  // all loads in flight before the stores
        const long long i = i0 + (long long)j * kARNT;
        e[j] = i < cnt ? recv[i] : make_uint2(0xffffffffu, 0u);
    }
    unsigned v = 0;
#pragma unroll
    for (int j = 0; j < kARIPT; ++j) {
        if (e[j].x != 0xffffffffu) {
            rawbuf[(long long)e[j].x + 1 - R0] = e[j].y;
            v = v > e[j].y ? v : e[j].y;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned y = __shfl_xor_sync(0xffffffffu, v, o);
        v = v > y ? v : y;
    }
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned m = 0;
        for (int w = 0; w < kARNT / 32; ++w) m = m > s_max[w] ? m : s_max[w];
        if (m) atomicMax(maxraw, m);
    }
}

}  // namespace

// Alphabet -> order-preserving codes, round-0 key length K, and the text
// packed once as a big-endian stream of b-bit codes (n b/8 bytes, L2-resident
// at 256 Mi DNA); the sort's histogram and first pass generate (key, suffix)
// pairs from it directly.
TextPrep prepare_text(rs_ctx *c, long long n) {
    const unsigned char *text = (const unsigned char *)c->bufs[B_TEXT].p;
    // alphabet -> order-preserving codes 0..sigma-1 (presence of each byte value)
    unsigned *present = (unsigned *)buf(c, B_HIST, sizeof(unsigned long long) * 8 * 256);
    RS_CUDA(cudaMemsetAsync(present, 0, sizeof(unsigned) * 8, c->stream));
    unsigned hb = (unsigned)std::min<long long>((n + 256 * 64 - 1) / (256 * 64), c->sm_count * 8);
    RS_LAUNCH_B(c, 1.0 * n, k_byte_present, hb, 256, 0, text, n, present);
    unsigned pres[8];
    fetch_small(c, pres, present, sizeof(pres));
    CodeTable ct;
    int sigma = 0;
    // order-preserving codes 0..sigma-1; past the end pads with code 0 too
    // (ties this creates are broken by suffix length in the next rounds)
    for (int b = 0; b < 256; ++b) ct.code[b] = (pres[b >> 5] >> (b & 31) & 1) ? (unsigned short)(sigma++) : 0;
    int bits = 1;
    while ((1 << bits) < sigma) ++bits;
    // Round-0 key length: all Kmax symbols that fit in 64 bits, unless fewer
    // already separate i.i.d. text (sigma^K >= 16 n) with fewer 8-bit radix
    // passes; the prefix-doubling rounds resolve whatever stays tied.
    const int Kmax = 64 / bits;
    int K = Kmax;
    if (sigma >= 2) {
        double need = std::log2((double)n) + 4.0;
        int Kr = (int)std::ceil(need / std::log2((double)sigma));
        if (Kr < Kmax) {
            int kb = ((Kr * bits + 7) / 8) * 8;
            K = std::min(Kmax, std::max(1, kb / bits));
        }
    }
    c->sa_key_symbols = K;

    const long long words = (n * bits + 63) / 64 + 4;
    u64 *stream = (u64 *)buf(c, B_PACKED, sizeof(u64) * (size_t)words);
    RS_LAUNCH_B(c, (double)n + 8.0 * words, k_pack_text, grid_for(words, 256), 256, 0, text, n, ct, bits, words,
                stream);
    c->packed_bits = bits;
    return TextPrep{stream, words, bits, K, sigma};
}

// ---- distributed path: tied groups larger than kSmallGroup -----------------
// suffix_less with a depth cap: `over` is set when the common prefix reaches
// `cap` symbols (the caller then declines the whole text).
__device__ __forceinline__ bool suffix_less_capped(const u64 *__restrict__ stream, int b, long long n, long long K,
                                                   unsigned a, unsigned c, long long cap, bool &over) {
    const long long lim = n - (long long)(a > c ? a : c);
    long long h = K < lim ? K : lim;
    const int per = 64 / b;
    while (h < lim) {
        if (h >= cap) {
            over = true;
            return a < c;
        }
        const u64 wa = load_sym64(stream, b, (long long)a + h), wc = load_sym64(stream, b, (long long)c + h);
        const u64 x = wa ^ wc;
        if (x == 0) {
            h += per;
            continue;
        }
        h += __clzll((long long)x) / b;
        if (h >= lim) break;
        return wa < wc;
    }
    return a > c;  // one is a prefix of the other: the shorter (later start) sorts first
}

constexpr int kLGB = 1024;         // list entries per block (rounded out to whole groups)
constexpr int kLGSlots = 2 * kLGB; // sort capacity: groups of up to kLGB + 1 members always fit
constexpr int kLGCap = 4096;       // longest common prefix (symbols) inside a group
constexpr int kLGNT = 256;

// First group boundary (head change; U counts as one) at or after x.
__device__ __forceinline__ long long next_group_start(const unsigned *__restrict__ H, long long U, long long x,
                                                      int *s_min) {
    long long base = x;
    while (true) {
        if (threadIdx.x == 0) *s_min = 0x7fffffff;
        __syncthreads();
        const long long t = base + threadIdx.x;
        const bool f = t >= U || t == 0 || H[t] != H[t - 1];
        if (f) atomicMin(s_min, (int)threadIdx.x);
        __syncthreads();
        const int m = *s_min;
        __syncthreads();
        if (m != 0x7fffffff) return base + m;
        base += kLGNT;
    }
}

// Tied groups above kSmallGroup members after round 0 (runs of equal heads in
// the (slot, head, suffix) lists).  Block b takes the whole groups that start
// in list entries [b kLGB, (b + 1) kLGB) and bitonic-sorts them together by
// (head, suffix) -- members compared by their cached first window past the
// shared key, else by packed-text comparison -- then writes SA slots, the LCPs
// of adjacent members and their raw LLR values (group boundary LCPs are known
// from round 0) into the bucketed scatter.  A group of more than kLGB + 1
// members or with a common prefix of kLGCap symbols sets *decline.
__global__ void __launch_bounds__(kLGNT) k_large_groups_seg(const unsigned *__restrict__ P,
                                                        const unsigned *__restrict__ H,
                                                        const unsigned *__restrict__ V, long long U,
                                                        const u64 *__restrict__ stream, int b, long long n,
                                                        long long K, unsigned *__restrict__ sa,
                                                        unsigned *__restrict__ lcp_d, BucketEmit be,
                                                        unsigned *decline) {
    __shared__ EmitSmem<kLGNT, 1> s_emit;
    __shared__ unsigned s_v[kLGSlots], s_h[kLGSlots];
    __shared__ u64 s_w[kLGSlots];  // first window past the shared round-0 key
    __shared__ unsigned s_l[kLGSlots + 1];
    __shared__ int s_min, s_over;
    const long long lo = (long long)blockIdx.x * kLGB;
    const long long hi = lo + kLGB < U ? lo + kLGB : U;
    const long long s0 = next_group_start(H, U, lo, &s_min);
    if (s0 >= hi) return;  // every entry here belongs to a group started earlier
    const long long s1 = next_group_start(H, U, hi, &s_min);
    const int m = (int)(s1 - s0);
    if (m > kLGSlots) {
        if (threadIdx.x == 0) atomicOr(decline, 1u);
        return;
    }
    int p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += kLGNT) {
        const bool real = i < m;
        const unsigned v = real ? V[s0 + i] : 0xffffffffu;
        s_v[i] = v;
        s_h[i] = real ? H[s0 + i] : 0xffffffffu;
        s_w[i] = real ? load_sym64(stream, b, (long long)v + K) : 0;
    }
    if (threadIdx.x == 0) s_over = 0;
    __syncthreads();
    bool over = false;
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < p2; i += kLGNT) {
                const int q = i ^ j;
                if (q <= i) continue;
                const unsigned x = s_v[i], y = s_v[q], hx = s_h[i], hy = s_h[q];
                const u64 wx = s_w[i], wy = s_w[q];
                // (head, suffix) order; padding (head 0xffffffff) sorts last
                bool lt;
                if (hx != hy) {
                    lt = hx < hy;
                } else if (hx == 0xffffffffu) {
                    lt = false;
                } else {
                    const long long lim = n - (long long)(x > y ? x : y);
                    const u64 d = wx ^ wy;
                    if (d != 0 && K + __clzll((long long)d) / b < lim) lt = wx < wy;
                    else lt = suffix_less_capped(stream, b, n, K, x, y, kLGCap, over);
                }
                const bool up = (i & k) == 0;  // ascending half of the bitonic merge
                if (up ? !lt : lt) {
                    s_v[i] = y;
                    s_v[q] = x;
                    s_h[i] = hy;
                    s_h[q] = hx;
                    s_w[i] = wy;
                    s_w[q] = wx;
                }
            }
            __syncthreads();
        }
    }
    if (over) s_over = 1;
    __syncthreads();
    if (s_over) {
        if (threadIdx.x == 0) atomicOr(decline, 1u);
        return;
    }
    // s_l[i] = LCP of sorted members i-1, i; at a group's first member (and
    // past the last) the boundary LCP with the neighbouring slot, from round 0
    for (int i = threadIdx.x; i <= m; i += kLGNT) {
        unsigned l;
        if (i == m) {
            l = lcp_d[P[s1 - 1] + 1];
        } else if (i == 0 || s_h[i] != s_h[i - 1]) {
            l = lcp_d[P[s0 + i]];
        } else {
            const long long a = s_v[i - 1], c = s_v[i];
            const long long lim = n - (a > c ? a : c);
            l = (unsigned)packed_lcp(stream, b, a, c, K < lim ? K : lim, lim);
        }
        s_l[i] = l;
    }
    __syncthreads();
    for (int i0 = 0; i0 < m; i0 += kLGNT) {  // uniform trip count: bucket_emit is block-collective
        const int i = i0 + threadIdx.x;
        unsigned d = kNoDest, vl = 0;
        if (i < m) {
            d = s_v[i];
            const unsigned slot = P[s0 + i];  // groups keep their slot ranges: list order is slot order
            sa[slot] = d;
            if (i > 0 && s_h[i] == s_h[i - 1]) lcp_d[slot] = s_l[i];
            vl = s_l[i] > s_l[i + 1] ? s_l[i] : s_l[i + 1];
        }
        bucket_emit<kLGNT, 1>(be, &d, &vl, s_emit);
    }
}

void ensure_isa(rs_ctx *c);

void build_suffix_array(rs_ctx *c, long long n) {
    unsigned *sa = (unsigned *)buf(c, B_SA, sizeof(unsigned) * (size_t)(n + 16));  // round 0 swaps it with a vals buffer
    unsigned *isa = (unsigned *)buf(c, B_ISA, sizeof(unsigned) * (size_t)(n + 4));
    c->sa_rounds = 0;
    c->lcp_from_keys = false;
    c->sa_device_built = false;
    c->raw_from_round0 = false;
    c->patch_slots = 0;
    if (n <= 0) return;
    const TextPrep tp = prepare_text(c, n);
    const int bits = tp.bits, K = tp.K;
    u64 *stream = tp.stream;
    u64 *k0 = (u64 *)buf(c, B_KEYS0, sizeof(u64) * (size_t)n + 16);
    u64 *k1 = (u64 *)buf(c, B_KEYS1, sizeof(u64) * (size_t)n + 16);
    unsigned *v0 = (unsigned *)buf(c, B_VALS0, sizeof(unsigned) * (size_t)(n + 16));
    unsigned *v1 = (unsigned *)buf(c, B_VALS1, sizeof(unsigned) * (size_t)(n + 16));
    unsigned *Pa = (unsigned *)buf(c, B_T0, sizeof(unsigned) * (size_t)n);
    unsigned *Pb = (unsigned *)buf(c, B_T1, sizeof(unsigned) * (size_t)n);
    unsigned *Ha = (unsigned *)buf(c, B_H0, sizeof(unsigned) * (size_t)n);
    unsigned *Hb = (unsigned *)buf(c, B_H1, sizeof(unsigned) * (size_t)n);
    unsigned *Va = (unsigned *)buf(c, B_V0, sizeof(unsigned) * (size_t)n);
    unsigned *Vb = (unsigned *)buf(c, B_V1, sizeof(unsigned) * (size_t)n);
    unsigned long long *u_dev = (unsigned long long *)buf(c, B_SMALL, 4096) + 4;
    unsigned *lcp_d = (unsigned *)buf(c, B_LCP, sizeof(unsigned) * (size_t)(n + 4));
    RS_CUDA(cudaMemsetAsync(lcp_d + n, 0, sizeof(unsigned) * 4, c->stream));
    unsigned *raw = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots(n));
    RS_CUDA(cudaMemsetAsync(raw, 0, sizeof(unsigned), c->stream));

    const TextKeys tk{stream, n, bits, K, std::min<long long>(K - 1, n)};
    // round-0 keys of <= 32 bits (DNA) travel as u32: 8 instead of 12 bytes per pair and pass
    const bool key32 = bits * K <= 32;
    u64 *ks = nullptr;
    unsigned *ks32 = nullptr;
    bool text_keys = false;  // the keys being consumed were built in text order
    bool lists_ok = true;    // Ha / Va hold the head / suffix lists of the tied suffixes
    unsigned *vs;
    if (key32)
        radix_sort_pairs<unsigned>(c, (unsigned *)k0, (unsigned *)k1, v0, v1, n, bits * K, &ks32, &vs, &tk);
    else
        radix_sort_pairs<u64>(c, k0, k1, v0, v1, n, bits * K, &ks, &vs, &tk);

    long long U = n;
    const unsigned *P = nullptr;
    long long depth = K;
    SegBoundary sb_whole{n, 0, 0, nullptr};
    c->isa_lazy = false;
    while (true) {
        ++c->sa_rounds;
        long long tiles = (U + kUTile - 1) / kUTile;
        u64 *tagg = (u64 *)buf(c, B_BOUNDS, sizeof(u64) * 2 * (size_t)(tiles + 1));
        u64 *tpre = tagg + tiles + 1;
        BucketEmit be{nullptr, nullptr, 0, 0, nullptr};
        bool skip_isa = false;
        RS_CUDA(cudaMemsetAsync(u_dev + 1, 0, sizeof(unsigned long long), c->stream));
        sb_whole.group_count = u_dev + 1;
        if (P && U >= n / 16) be = bucket_setup(c, n, 0, false);
        // Round 0: the tied count is known after the reduce pass.  With few
        // ties (i.i.d.-like text) the SA after round 0 + the small-group sort
        // is final and the query pipeline never reads ISA -> scatter only raw
        // and fill ISA from SA if it is ever needed.
        auto tile_scan = [&](const u64 *agg, long long nt, u64 *pre) {
            const long long blocks = (nt + kTSTile - 1) / kTSTile;
            Scratch sc = scratch(c, blocks);
            RS_LAUNCH(c, k_tile_scan_lb, (unsigned)blocks, kTSNT, 0, agg, nt, pre, u_dev, sc.counter, sc.status,
                      blocks);
        };
        auto setup_round0_emit = [&]() {
            unsigned long long u0 = 0;
            fetch_small(c, &u0, u_dev, sizeof(u0));
            skip_isa = u0 <= (unsigned long long)(n / 8);
            be = bucket_setup(c, n, 0, !skip_isa);
        };
        // reduce-then-scan instead of a look-back: the heavy pass never waits
        if (ks32) {
            RS_LAUNCH_B(c, 4.0 * U, (k_update<true, unsigned>), (unsigned)tiles, kUNT, 0, ks32, vs, P, U, sa, isa, Pa,
                        Ha, Va, tagg, tpre, lcp_d, bits, bits * K, be, sb_whole);
            tile_scan(tagg, tiles, tpre);
            if (!P) setup_round0_emit();
            // round 0: 8 B (key, suffix) in; 4 B SA + 4 B LCP + 12 B (ISA, raw) staging out
            RS_LAUNCH_B(c, 24.0 * U, (k_update<false, unsigned>), (unsigned)tiles, kUNT, 0, ks32, vs, P, U,
                        (unsigned *)nullptr, isa, Pa, Ha, Va, tagg, tpre, lcp_d, bits, bits * K, be, sb_whole);
            ks32 = nullptr;
        } else {
            RS_LAUNCH_B(c, 8.0 * U, (k_update<true, u64>), (unsigned)tiles, kUNT, 0, ks, vs, P, U, sa, isa, Pa, Ha,
                        Va, tagg, tpre, lcp_d, bits, bits * K, be, sb_whole);
            tile_scan(tagg, tiles, tpre);
            if (!P) setup_round0_emit();
            // head / suffix lists only when the next round may use the list
            // gather (text-order rounds with more than n/2 tied skip them)
            const bool lists = !P || !text_keys || 2 * U <= n;
            RS_LAUNCH_B(c, (P ? 24.0 : 28.0) * U, (k_update<false, u64>), (unsigned)tiles, kUNT, 0, ks, vs, P, U,
                        P ? sa : (unsigned *)nullptr, isa, Pa, lists ? Ha : nullptr, lists ? Va : nullptr, tagg,
                        tpre, P ? nullptr : lcp_d, bits, bits * K, be, sb_whole);
            lists_ok = lists;
        }
        if (!P) {  // round 0: the sorted suffixes are the SA -- adopt their buffer instead of copying
            const BufId idv = (vs == (const unsigned *)c->bufs[B_VALS0].p) ? B_VALS0 : B_VALS1;
            std::swap(c->bufs[B_SA], c->bufs[idv]);
            sa = (unsigned *)c->bufs[B_SA].p;
            if (idv == B_VALS0) v0 = (unsigned *)c->bufs[B_VALS0].p;
            else v1 = (unsigned *)c->bufs[B_VALS1].p;
        }
        unsigned long long un = 0, ngroups = 0;
        {
            unsigned long long two[2];
            fetch_small(c, two, u_dev, sizeof(two));
            un = two[0];
            ngroups = two[1];
        }
        add_bytes_last(c, 4.0 * (double)un);
        // skip_isa (few ties): raw is applied after k_small_groups added the tied suffixes
        if (!P) {
            if (!skip_isa) bucket_apply(c, be, isa, n, raw, 1);
            else if (un == 0) bucket_apply(c, be, raw + 1, n);
        } else if (be.stage) {
            bucket_apply(c, be, isa, U);
        }
        if (!P) c->isa_lazy = skip_isa;
        U = (long long)un;
        if (std::getenv("RS_DEBUG_ROUNDS")) std::fprintf(stderr, "round %d depth %lld unsorted %lld\n", c->sa_rounds, depth, U);
        if (c->sa_rounds == 1 && U > 0 && U <= n / 8) {  // mostly small groups (i.i.d.-like text)
            // small tied groups: final order + LCP + raw by direct comparison;
            // the lists keep only the larger groups (order preserved)
            unsigned *keep = (unsigned *)buf(c, B_T4, sizeof(unsigned) * (size_t)U);
            // lazy ISA (rebuilt from the final SA if ever needed): no ISA stores here
            // (the tied suffixes' raw goes into round 0's buckets, applied once below)
            RS_LAUNCH_B(c, 16.0 * U, k_small_groups, grid_for(U, kSGNT), kSGNT, 0, Pa, Ha, Va, U, stream, bits, n,
                        (long long)K, sa, c->isa_lazy ? nullptr : isa, lcp_d, raw, keep, be);
            bucket_apply(c, be, raw + 1, n);
            const long long ktiles = (U + kKTile - 1) / kKTile;
            Scratch ks_ = scratch(c, ktiles);
            RS_LAUNCH_B(c, 16.0 * U, k_keep_compact, (unsigned)ktiles, kKNT, 0, keep, Pa, Ha, Va, U, Pb, Hb, Vb, u_dev,
                        ks_.counter, ks_.status, ktiles);
            fetch_small(c, &un, u_dev, sizeof(un));
            U = (long long)un;
            std::swap(Pa, Pb);
            std::swap(Ha, Hb);
            std::swap(Va, Vb);
        }
        if (c->sa_rounds == 1) {
            c->sa_unsorted_after_round0 = U;
            // keep the tied slots of round 0: the LCP patch visits only them
            c->patch_slots = 0;
            if (U > 0 && U <= n / 4) {
                unsigned *keep = (unsigned *)buf(c, B_PATCH, sizeof(unsigned) * (size_t)U);
                RS_CUDA(cudaMemcpyAsync(keep, Pa, sizeof(unsigned) * (size_t)U, cudaMemcpyDeviceToDevice, c->stream));
                c->patch_slots = U;
            }
        }
        if (U == 0) break;
        if (c->isa_lazy) {  // more rounds: they read ISA (group heads for the tied)
            scatter_rank(c, sa, n, isa);
            RS_LAUNCH(c, k_isa_heads, grid_for(U, 256), 256, 0, Va, Ha, U, isa);
            c->isa_lazy = false;
        }
        if (depth > 2 * n + 64) fail(RS_ECUDA, "suffix sort did not converge");  // depth >= n resolves every group
        std::swap(Pa, Pb);  // Pb/Hb/Vb now hold the unsorted slots, heads, suffixes
        std::swap(Ha, Hb);
        std::swap(Va, Vb);
        P = Pb;
        // round key (group, lo): the group as its head slot, or -- when it
        // saves radix passes (few large groups, e.g. periodic text) -- as the
        // group's dense ordinal (Pa is free here: the lists live in Pb/Hb/Vb)
        int lo_bits = 1;
        while ((1ull << lo_bits) <= (unsigned long long)(n + depth + 1)) ++lo_bits;
        int g_bits = 0;
        while ((1ull << g_bits) < ngroups) ++g_bits;
        int h_bits = 0;
        while ((1ull << h_bits) < (unsigned long long)n) ++h_bits;
        // large rounds (most suffixes still tied): keys in text order, grouped
        // by head slot; smaller rounds: the list gather (dense ordinals when
        // they save radix passes)
        const bool text_order = (4 * U > n || !lists_ok) && !std::getenv("RS_SA_LIST_KEYS");
        text_keys = text_order;
        if (text_order) {
            unsigned long long *kc = (unsigned long long *)buf(c, B_SMALL, 4096) + 100;
            RS_CUDA(cudaMemsetAsync(kc, 0, sizeof(*kc), c->stream));
            RS_LAUNCH_B(c, 8.0 * n + 12.0 * U, k_make_keys_text, (unsigned)((n + kMKTile - 1) / kMKTile), kMKNT,
                        0, isa, n, depth, lo_bits, k0, v0, kc);
            unsigned long long got = 0;
            fetch_small(c, &got, kc, sizeof(got));
            if ((long long)got != U) fail(RS_ECUDA, "text-order round keys: tied-suffix count mismatch");
            radix_sort_pairs<u64>(c, k0, k1, v0, v1, U, std::max(1, lo_bits + h_bits), &ks, &vs);
            depth *= 2;
            continue;
        }
        const bool dense = (lo_bits + g_bits + 7) / 8 < (lo_bits + h_bits + 7) / 8;
        if (dense) {
            const long long gt = (U + kGTile - 1) / kGTile;
            Scratch sc = scratch(c, gt);
            RS_LAUNCH_B(c, 8.0 * U, k_group_ordinals, (unsigned)gt, kGNT, 0, Hb, U, Pa, u_dev, sc.counter, sc.status,
                        gt);
        }
        RS_LAUNCH_B(c, 20.0 * U, k_make_keys, grid_for(U, 256), 256, 0, dense ? Pa : Hb, Vb, U, isa, n, depth,
                    lo_bits, k0, v0);
        const int rbits = std::max(1, lo_bits + (dense ? g_bits : h_bits));
        radix_sort_pairs<u64>(c, k0, k1, v0, v1, U, rbits, &ks, &vs);
        depth *= 2;
    }
    c->lcp_from_keys = true;
    c->sa_final_depth = depth;
    c->sa_device_built = true;
}

void build_lcp(rs_ctx *c, long long n) {
    unsigned *lcp_d = (unsigned *)buf(c, B_LCP, sizeof(unsigned) * (size_t)(n + 4));
    if (n <= 0) {
        RS_CUDA(cudaMemsetAsync(lcp_d, 0, sizeof(unsigned) * 4, c->stream));
        return;
    }
    const unsigned char *text = (const unsigned char *)c->bufs[B_TEXT].p;
    const unsigned *sa = (const unsigned *)c->bufs[B_SA].p;
    // Patch work is at most (tied suffixes) x (final depth / 8 + 1) word
    // compares; take it when that is cheaper than a full Kasai pass.
    double patch_work = (double)c->sa_unsorted_after_round0 * (1.0 + (double)c->sa_final_depth / 8.0);
    if (c->lcp_from_keys && c->sa_unsorted_after_round0 == 0) {  // every LCP known after round 0
        c->raw_from_round0 = true;
        return;
    }
    if (c->lcp_from_keys && patch_work <= 2.0 * (double)n) {
        const bool list = c->patch_slots > 0;
        const long long work = list ? c->patch_slots : n;
        unsigned blocks = (unsigned)std::min<long long>(grid_for(work, 256), (long long)c->sm_count * 16);
        RS_LAUNCH_B(c, list ? 8.0 * work : 4.0 * n, k_lcp_patch, blocks, 256, 0,
                    (const u64 *)c->bufs[B_PACKED].p, c->packed_bits, sa, n,
                    (long long)c->sa_key_symbols, lcp_d, (unsigned *)c->bufs[B_RAW].p,
                    list ? (const unsigned *)c->bufs[B_PATCH].p : nullptr, work);
        c->raw_from_round0 = true;  // B_RAW is final
        return;
    }
    c->raw_from_round0 = false;
    unsigned *phi = (unsigned *)buf(c, B_PHI, sizeof(unsigned) * (size_t)n);
    unsigned *plcp = (unsigned *)buf(c, B_PLCP, sizeof(unsigned) * (size_t)n);
    // Device-built structures: the two permutation steps (phi by SA order,
    // PLCP -> SA order by ISA) go through the bucketed L2-local scatter
    // instead of one random 4-byte store/load per suffix.
    const bool bucketed = c->sa_device_built;
    if (bucketed) ensure_isa(c);
    if (bucketed)
        scatter_phi(c, sa, n, phi);
    else
        RS_LAUNCH_B(c, 8.0 * n, k_phi, grid_for(n, 256), 256, 0, sa, n, phi);
    const u64 *stream = c->packed_bits ? (const u64 *)c->bufs[B_PACKED].p : nullptr;
    // Short LCPs (the doubling depth bounds the longest: < 1024 symbols here):
    // every position compares from scratch, one thread each, instead of
    // Kasai's carried h along a sequential chunk -- far more parallelism for
    // the same few packed-window compares.  Long repeats keep the carry.
    if (stream && c->sa_device_built && c->sa_final_depth <= 1024) {
        RS_LAUNCH_B(c, 8.0 * n, k_plcp_flat, grid_for(n, 256), 256, 0, stream, c->packed_bits, phi, n, plcp);
    } else {
        long long chunk = std::max<long long>(32, n >> 19);
        long long chunks = (n + chunk - 1) / chunk;
        RS_LAUNCH_B(c, 10.0 * n, k_plcp, grid_for(chunks, 128), 128, 0, text, stream, c->packed_bits, phi, n, chunk,
                    plcp);
    }
    if (bucketed) {
        RS_CUDA(cudaMemsetAsync(lcp_d + n, 0, sizeof(unsigned) * 2, c->stream));
        scatter_by(c, (const unsigned *)c->bufs[B_ISA].p, plcp, n, lcp_d, n);
    } else {
        RS_LAUNCH_B(c, 12.0 * n, k_lcp_gather, grid_for(n + 2, 256), 256, 0, sa, plcp, n, lcp_d);
    }
}


// ---- distributed suffix sort: host side ---------------------------------
// Rank r of `world` owns the suffixes whose top round-0 key digit falls in its
// range (ranges balanced on the digit histogram every rank computes from its
// copy of the text), i.e. one contiguous segment [S, S + m) of the suffix
// array; the text-order outputs (raw LLR, then the query) are split into
// bucket-aligned position shards.  Distributed regime: 32-bit symbol-aligned
// round-0 keys and tied groups that k_small_groups_seg / k_large_groups_seg
// sort by direct comparison (<= kLGB + 1 members, common prefix < kLGCap);
// otherwise the caller runs the single-GPU path.

static unsigned host_key_lcp(unsigned long long a, unsigned long long b, int code_bits, int key_bits, unsigned K,
                             unsigned rem_a, unsigned rem_b) {
    const unsigned long long x = a ^ b;
    const unsigned m = rem_a < rem_b ? rem_a : rem_b;
    if (x) {
        const unsigned z = (unsigned)(__builtin_clzll(x) - (64 - key_bits));
        const unsigned l = z / (unsigned)code_bits;
        return l < m ? l : m;
    }
    return m < K ? m : kLcpUnknown;
}

static void dist_buckets(long long n, int *shift, long long *nb) {
    // the same rule as bucket_setup(c, n, ...)
    int sh = 12;
    while (((n + (1ll << sh) - 1) >> sh) > kMaxBuckets && sh < 30) ++sh;
    *shift = sh;
    *nb = std::max<long long>(1, (n + (1ll << sh) - 1) >> sh);
}

void dist_shard(long long n, int rank, int world, long long *P0, long long *P1) {
    int shift;
    long long nb;
    dist_buckets(n, &shift, &nb);
    const long long b0 = (long long)rank * nb / world, b1 = (long long)(rank + 1) * nb / world;
    *P0 = std::min<long long>(b0 << shift, n);
    *P1 = std::min<long long>(b1 << shift, n);
}

void dist_sort(rs_ctx *c, long long n, int rank, int world, long long *info) {
    for (int i = 0; i < 16; ++i) info[i] = 0;
    c->dist.stage = 0;
    if (n < 4096 || world < 1 || rank < 0 || rank >= world) return;
    const TextPrep tp = prepare_text(c, n);
    const int bits = tp.bits, K = tp.K, key_bits = bits * K;
    if (key_bits > 32) return;
    const TextKeys tk{tp.stream, n, bits, K, std::min<long long>(K - 1, n)};
    std::vector<unsigned long long> h;
    if (!text_digit_histograms(c, tk, key_bits, h)) return;
    const int passes = (key_bits + 7) / 8, top = passes - 1;
    unsigned long long cum[257];
    cum[0] = 0;
    for (int d = 0; d < 256; ++d) cum[d + 1] = cum[d] + h[(size_t)top * 256 + d];
    auto split = [&](int r) {  // first digit whose prefix reaches r/world of the suffixes
        if (r <= 0) return 0;
        if (r >= world) return 256;
        const unsigned long long target = (unsigned long long)((__int128)n * r / world);
        int d = 0;
        while (d < 256 && cum[d] < target) ++d;
        return d;
    };
    const int dlo = split(rank), dhi = split(rank + 1);
    const long long S = (long long)cum[dlo], m = (long long)(cum[dhi] - cum[dlo]);
    unsigned *k0 = (unsigned *)buf(c, B_KEYS0, sizeof(unsigned) * (size_t)(m + 16));
    unsigned *k1 = (unsigned *)buf(c, B_KEYS1, sizeof(unsigned) * (size_t)(m + 16));
    unsigned *v0 = (unsigned *)buf(c, B_VALS0, sizeof(unsigned) * (size_t)(m + 16));
    unsigned *v1 = (unsigned *)buf(c, B_VALS1, sizeof(unsigned) * (size_t)(m + 16));
    unsigned long long *tot = (unsigned long long *)buf(c, B_SMALL, 4096) + 12;
    const long long tiles = (n + kFTile - 1) / kFTile;
    Scratch sc = scratch(c, tiles);
    RS_LAUNCH_B(c, 0.25 * n + 8.0 * m, k_filter_keys, (unsigned)tiles, kFNT, 0, tk, n, 8 * top, (unsigned)dlo,
                (unsigned)dhi, k0, v0, tot, sc.counter, sc.status, tiles);
    unsigned long long got = 0;
    fetch_small(c, &got, tot, sizeof(got));
    if ((long long)got != m) fail(RS_ECUDA, "distributed sort: filtered count mismatch");
    unsigned *ks = k0, *vs = v0;
    if (m > 1) radix_sort_pairs<unsigned>(c, k0, k1, v0, v1, m, key_bits, &ks, &vs, nullptr);
    c->dist.m = m;
    c->dist.S = S;
    c->dist.keys = ks;
    c->dist.vals = vs;
    c->dist.bits = bits;
    c->dist.K = K;
    if (m > 0) {
        unsigned a[2], b2[2];
        fetch_small(c, &a[0], ks, 4);
        fetch_small(c, &a[1], ks + m - 1, 4);
        fetch_small(c, &b2[0], vs, 4);
        fetch_small(c, &b2[1], vs + m - 1, 4);
        c->dist.first_key = a[0];
        c->dist.last_key = a[1];
        c->dist.first_pos = b2[0];
        c->dist.last_pos = b2[1];
    }
    c->dist.stage = 1;
    info[0] = 1;
    info[1] = m;
    info[2] = S;
    info[3] = (long long)c->dist.first_key;
    info[4] = c->dist.first_pos;
    info[5] = (long long)c->dist.last_key;
    info[6] = c->dist.last_pos;
    info[7] = bits;
    info[8] = K;
}

void dist_update(rs_ctx *c, long long n, int rank, int world, const long long *nbr, long long *send_counts,
                 long long *info) {
    for (int i = 0; i < 16; ++i) info[i] = 0;
    if (c->dist.stage < 1) fail(RS_ESTATE, "rs_dist_sort first");
    const long long m = c->dist.m;
    const int bits = c->dist.bits, K = c->dist.K, key_bits = bits * K;
    const u64 *stream = (const u64 *)c->bufs[B_PACKED].p;
    BucketEmit be = bucket_setup(c, n, 0, false);
    if (m > 0) {
        SegBoundary sb{n, 0u, 0u, nullptr};
        if (nbr[2])
            sb.lcp_first = host_key_lcp(c->dist.first_key, (unsigned long long)nbr[0], bits, key_bits, (unsigned)K,
                                        (unsigned)(n - c->dist.first_pos), (unsigned)(n - nbr[1]));
        if (nbr[5])
            sb.lcp_last = host_key_lcp((unsigned long long)nbr[3], c->dist.last_key, bits, key_bits, (unsigned)K,
                                       (unsigned)(n - nbr[4]), (unsigned)(n - c->dist.last_pos));
        unsigned *sa = (unsigned *)buf(c, B_SA, sizeof(unsigned) * (size_t)(m + 4));
        unsigned *lcp_d = (unsigned *)buf(c, B_LCP, sizeof(unsigned) * (size_t)(m + 4));
        RS_CUDA(cudaMemsetAsync(lcp_d + m, 0, sizeof(unsigned) * 4, c->stream));
        unsigned *Pa = (unsigned *)buf(c, B_T0, sizeof(unsigned) * (size_t)m);
        unsigned *Ha = (unsigned *)buf(c, B_H0, sizeof(unsigned) * (size_t)m);
        unsigned *Va = (unsigned *)buf(c, B_V0, sizeof(unsigned) * (size_t)m);
        unsigned long long *u_dev = (unsigned long long *)buf(c, B_SMALL, 4096) + 4;
        const long long tiles = (m + kUTile - 1) / kUTile;
        u64 *tagg = (u64 *)buf(c, B_BOUNDS, sizeof(u64) * 2 * (size_t)(tiles + 1));
        u64 *tpre = tagg + tiles + 1;
        RS_LAUNCH_B(c, 4.0 * m, (k_update<true, unsigned>), (unsigned)tiles, kUNT, 0, c->dist.keys, c->dist.vals,
                    nullptr, m, sa, nullptr, Pa, Ha, Va, tagg, tpre, lcp_d, bits, key_bits, be, sb);
        {
            const long long blocks = (tiles + kTSTile - 1) / kTSTile;
            Scratch sc = scratch(c, blocks);
            RS_LAUNCH(c, k_tile_scan_lb, (unsigned)blocks, kTSNT, 0, tagg, tiles, tpre, u_dev, sc.counter, sc.status,
                      blocks);
        }
        RS_LAUNCH_B(c, 24.0 * m, (k_update<false, unsigned>), (unsigned)tiles, kUNT, 0, c->dist.keys, c->dist.vals,
                    nullptr, m, sa, nullptr, Pa, Ha, Va, tagg, tpre, lcp_d, bits, key_bits, be, sb);
        unsigned long long un = 0;
        fetch_small(c, &un, u_dev, sizeof(un));
        info[2] = (long long)un;
        if (un > 0) {
            unsigned *keep = (unsigned *)buf(c, B_T4, sizeof(unsigned) * (size_t)un);
            RS_LAUNCH_B(c, 16.0 * un, k_small_groups_seg, grid_for((long long)un, kSGNT), kSGNT, 0, Pa, Ha, Va,
                        (long long)un, stream, bits, n, (long long)K, sa, nullptr, lcp_d, keep, be);
            unsigned long long big = 0;
            unsigned *Pb = (unsigned *)buf(c, B_T1, sizeof(unsigned) * (size_t)un);
            unsigned *Hb = (unsigned *)buf(c, B_H1, sizeof(unsigned) * (size_t)un);
            unsigned *Vb = (unsigned *)buf(c, B_V1, sizeof(unsigned) * (size_t)un);
            const long long ktiles = (un + kKTile - 1) / kKTile;
            Scratch ks_ = scratch(c, ktiles);
            RS_LAUNCH_B(c, 16.0 * un, k_keep_compact, (unsigned)ktiles, kKNT, 0, keep, Pa, Ha, Va, (long long)un,
                        Pb, Hb, Vb, u_dev, ks_.counter, ks_.status, ktiles);
            fetch_small(c, &big, u_dev, sizeof(big));
            info[3] = (long long)big;
            if (big > 0) {  // groups above kSmallGroup: sorted per block of whole groups on this rank
                unsigned *decline = (unsigned *)((unsigned long long *)buf(c, B_SMALL, 4096) + 9);
                RS_CUDA(cudaMemsetAsync(decline, 0, sizeof(unsigned), c->stream));
                const long long blocks = ((long long)big + kLGB - 1) / kLGB;
                RS_LAUNCH_B(c, 28.0 * big, k_large_groups_seg, (unsigned)blocks, kLGNT, 0, Pb, Hb, Vb,
                            (long long)big, stream, bits, n, (long long)K, sa, lcp_d, be, decline);
                unsigned dec = 0;
                fetch_small(c, &dec, decline, sizeof(dec));
                if (std::getenv("RS_DEBUG_ROUNDS"))
                    std::fprintf(stderr, "dist rank %d: %llu suffixes in tied groups above %d%s\n", rank, big,
                                 kSmallGroup, dec ? " (declined)" : "");
                if (dec) return;  // a group too large or too repetitive: not distributed (info[0] = 0)
            }
        }
    }
    // per destination rank: the buckets of its position shard, in order
    std::vector<unsigned> cur((size_t)be.nb * kCursorStride);
    fetch_small(c, cur.data(), be.cursor, sizeof(unsigned) * cur.size());
    std::vector<long long> off((size_t)be.nb);
    long long acc = 0;
    for (long long b = 0; b < be.nb; ++b) {
        off[(size_t)b] = acc;
        acc += cur[(size_t)b * kCursorStride];
    }
    for (int q = 0; q < world; ++q) {
        const long long b0 = (long long)q * be.nb / world, b1 = (long long)(q + 1) * be.nb / world;
        long long t = 0;
        for (long long b = b0; b < b1; ++b) t += cur[(size_t)b * kCursorStride];
        send_counts[q] = t;
    }
    uint2 *send = (uint2 *)buf(c, B_SEND, sizeof(uint2) * (size_t)(acc + 8));
    long long *d_off = (long long *)buf(c, B_I64D, sizeof(long long) * (size_t)be.nb);
    RS_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, c->stream));
    unsigned maxc = 0;
    for (long long b = 0; b < be.nb; ++b) maxc = std::max(maxc, cur[(size_t)b * kCursorStride]);
    if (acc > 0)
        RS_LAUNCH_B(c, 16.0 * acc, k_pack_send, dim3((maxc + 4095) / 4096, (unsigned)be.nb), 256, 0, be.stage,
                    be.cursor, be.shift, d_off, send);
    RS_CUDA(cudaStreamSynchronize(c->stream));  // the host-side offsets must outlive the copy
    c->dist.send_total = acc;
    c->dist.stage = 2;
    info[0] = 1;
    info[1] = acc;
}

void dist_apply(rs_ctx *c, long long n, int rank, int world, const void *recv, long long cnt, long long hcap,
                long long *info) {
    for (int i = 0; i < 16; ++i) info[i] = 0;
    if (c->dist.stage < 2) fail(RS_ESTATE, "rs_dist_update first");
    long long P0, P1;
    dist_shard(n, rank, world, &P0, &P1);
    hcap = (hcap + 3) & ~3ll;
    const long long R0 = P0 - hcap;  // rawbuf[i - R0] = raw[i], i >= P0 + 1 - hcap; R0 = 0 mod 4 (TMA alignment)
    const long long len = (P1 - P0) + hcap + 64;
    unsigned *rawbuf = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * (size_t)len);
    RS_CUDA(cudaMemsetAsync(rawbuf, 0, sizeof(unsigned) * (size_t)len, c->stream));
    unsigned *mx = (unsigned *)((unsigned long long *)buf(c, B_SMALL, 4096) + 14);
    RS_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned), c->stream));
    if (cnt > 0)
        RS_LAUNCH_B(c, 12.0 * cnt, k_apply_recv, (unsigned)((cnt + kARNT * kARIPT - 1) / (kARNT * kARIPT)), kARNT,
                    0, (const uint2 *)recv, cnt, R0, rawbuf, mx);
    unsigned maxraw = 0;
    fetch_small(c, &maxraw, mx, sizeof(maxraw));
    c->dist.P0 = P0;
    c->dist.P1 = P1;
    c->dist.R0 = R0;
    c->dist.hcap = hcap;
    c->dist.stage = 3;
    info[0] = 1;
    info[1] = P0;
    info[2] = P1;
    info[3] = maxraw;
    info[4] = R0;
}

bool query_range(rs_ctx *c, int mode, int path, const uint2 *d_e, long long count, const unsigned *d_raw,
                 long long kb, long long ke, int out_off, long long n_slots, long long min_lo);

void dist_scan(rs_ctx *c, long long n, int mode, long long halo, long long *total) {
    if (c->dist.stage < 3) fail(RS_ESTATE, "rs_dist_apply first");
    if (halo < 1 || halo + 4 > c->dist.hcap) fail(RS_ERANGE, "halo exceeds the raw shard's halo capacity");
    const long long P0 = c->dist.P0, P1 = c->dist.P1, cnt = P1 - P0;
    long long *o1 = (long long *)buf(c, B_OUT1, 8 * (size_t)(cnt + 2));
    buf(c, B_OUT0, 8 * (size_t)(cnt + 1));
    RS_CUDA(cudaMemsetAsync(o1, 0, 8, c->stream));
    c->total = 0;
    c->out_mode = mode;
    c->out_ref_layout = false;
    c->shard_lo = P0 + 1;
    c->shard_hi = P1 + 1;
    if (cnt > 0) {
        const unsigned *d_raw = (const unsigned *)c->bufs[B_RAW].p - c->dist.R0;
        // long repeats (a window beyond the fused kernel's shared stage): the
        // raw-path scan over the same shard + halo (same answers, Lemma 2)
        if (!query_range(c, mode, RS_PATH_COMPACT, nullptr, 0, d_raw, P0 + 1, P1, 0, cnt, P0 + 1 - halo))
            query_range(c, mode, RS_PATH_RAW, nullptr, 0, d_raw, P0 + 1, P1, 0, cnt, P0 + 1 - halo);
    }
    *total = mode == RS_MODE_ALL ? c->total : 0;
}

// B_ISA from the final SA when round 0 skipped it (rank for the API, Kasai).
void ensure_isa(rs_ctx *c) {
    if (!c->isa_lazy) return;
    const long long n = c->n;
    scatter_rank(c, (const unsigned *)c->bufs[B_SA].p, n, (unsigned *)c->bufs[B_ISA].p);
    c->isa_lazy = false;
}

}  // namespace rsb
