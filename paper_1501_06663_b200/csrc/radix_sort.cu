// radix_sort.cu -- hand-written LSD radix sort of (u64 key, u32 value) pairs.
//
// Used by the prefix-doubling suffix sort (suffix_array.cu), replacing the
// reference's np.argsort / np.lexsort (suffixes.py:34, :43).  B200 design:
//   * one histogram kernel reads the keys ONCE and builds the digit histograms
//     of every pass (8-bit digits);
//   * one "onesweep" kernel per pass: tile ranking with warp match_any, a
//     per-digit decoupled look-back across tiles for the global digit offsets,
//     and a shared-memory exchange so the scatter writes contiguous runs;
//   * passes whose digit is constant over all keys are skipped.
// HBM traffic per pass: read 12 B + write 12 B per pair.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace rsb {

namespace {

constexpr int kNT = 256;
constexpr int kIPT = 16;
constexpr int kTile = kNT * kIPT;  // 4096 pairs per tile
constexpr int kWarps = kNT / 32;
constexpr int kRadix = 256;

// hist_passes < passes: only the first hist_passes digit histograms are
// counted here (the rest follow from k_hist_shift).
template <bool TEXT, typename KeyT>
__global__ void __launch_bounds__(kNT) k_histograms(const KeyT *__restrict__ keys, long long count, int passes,
                                                    unsigned long long *__restrict__ hist /*[passes][256]*/,
                                                    TextKeys tk, int hist_passes) {
    __shared__ unsigned s_hist[8][kRadix];
    for (int i = threadIdx.x; i < 8 * kRadix; i += kNT) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    long long stride = (long long)gridDim.x * kNT;
    for (long long i = blockIdx.x * (long long)kNT + threadIdx.x; i < count; i += stride) {
        u64 k = TEXT ? text_key(tk, i) : (u64)keys[i];  // histograms need no particular order
        for (int p = 0; p < hist_passes; ++p) atomicAdd(&s_hist[p][(k >> (8 * p)) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += kNT) {
        unsigned v = (&s_hist[0][0])[i];
        if (v) atomicAdd(&hist[i], (unsigned long long)v);
    }
}

// Digit-0 histogram straight from the packed stream when digits hold whole
// symbols (B | 8): digit 0 of the key at i is the byte-wide window of symbols
// [i + K - 8/B, i + K); each thread takes whole 64-bit stream words and
// extracts every window starting in them (no per-key loads).
template <int B>
__global__ void __launch_bounds__(kNT) k_hist_digit0(TextKeys tk, unsigned long long *__restrict__ hist) {
    constexpr int cpw = 64 / B, cpd = 8 / B;
    __shared__ unsigned s_hist[kRadix];
    s_hist[threadIdx.x] = 0;
    __syncthreads();
    const long long j0 = tk.K - cpd, j1 = tk.n + tk.K - cpd;  // window start symbols [j0, j1)
    const long long w_first = j0 / cpw, w_last = (j1 - 1) / cpw;
    const long long stride = (long long)gridDim.x * kNT;
    for (long long w = w_first + blockIdx.x * (long long)kNT + threadIdx.x; w <= w_last; w += stride) {
        const u64 a = tk.stream[w], b = tk.stream[w + 1];
        const long long base = w * cpw;
        if (base >= j0 && base + cpw <= j1) {
#pragma unroll
            for (int q = 0; q < cpw; ++q) {
                const u64 x = q ? (a << (q * B)) | (b >> (64 - q * B)) : a;
                atomicAdd(&s_hist[x >> 56], 1u);
            }
        } else {
            for (int q = 0; q < cpw; ++q) {
                const long long j = base + q;
                if (j < j0 || j >= j1) continue;
                const u64 x = q ? (a << (q * B)) | (b >> (64 - q * B)) : a;
                atomicAdd(&s_hist[x >> 56], 1u);
            }
        }
    }
    __syncthreads();
    if (s_hist[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)s_hist[threadIdx.x]);
}

// Text keys whose 8-bit digits hold whole symbols (b | 8, 8 | b*K): digit p of
// the key at i is digit 0 of the key at i - p*cpd (cpd = 8/b symbols per
// digit), so hist_p = hist_0 - {digit 0 of keys at [n - p*cpd, n)} + {digit p
// of keys at [0, p*cpd)}: one counted histogram instead of `passes`.
__global__ void k_hist_shift(unsigned long long *hist, int passes, int cpd, TextKeys tk) {
    const int d = threadIdx.x;  // one thread per bin
    const long long n = tk.n;
    for (int p = 1; p < passes; ++p) {
        long long v = (long long)hist[d];
        const long long s = (long long)p * cpd;
        for (long long i = n - s; i < n; ++i) v -= (long long)((text_key(tk, i) & 0xff) == (u64)d);
        for (long long i = 0; i < s; ++i) v += (long long)(((text_key(tk, i) >> (8 * p)) & 0xff) == (u64)d);
        hist[(size_t)p * kRadix + d] = (unsigned long long)v;
    }
}

// Exclusive scan of each pass's 256 counts, in place (one block per pass).
__global__ void k_hist_scan(unsigned long long *hist) {
    __shared__ unsigned long long s[kRadix];
    unsigned long long *h = hist + blockIdx.x * kRadix;
    s[threadIdx.x] = h[threadIdx.x];
    __syncthreads();
    for (int o = 1; o < kRadix; o <<= 1) {
        unsigned long long v = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
        __syncthreads();
        s[threadIdx.x] += v;
        __syncthreads();
    }
    h[threadIdx.x] = s[threadIdx.x] - h[threadIdx.x];
}

// (key, suffix) pairs straight from the packed text, in sort input order.
template <typename KeyT>
__global__ void k_materialize(TextKeys tk, long long count, KeyT *__restrict__ keys, unsigned *__restrict__ vals) {
    long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= count) return;
    const long long pos = text_pos(tk, e);
    keys[e] = (KeyT)text_key(tk, pos);
    vals[e] = (unsigned)pos;
}

// peers & (lanes whose (x & bitmask) equals mine).  Written in PTX so ptxas
// keeps the predicate form (LOP3.P + VOTE + predicated NOT + LOP3): ~30% fewer
// issue slots than the shift/and/compare sequence it otherwise emits
// (tools/micro/match_bench.cu: 14.3 vs 20.6 SM-cycles per warp peer mask;
// MATCH.ANY costs 58.6 with ~30 distinct 8-bit digits per warp).
__device__ __forceinline__ unsigned peer_bit(unsigned peers, unsigned x, unsigned bitmask) {
    unsigned r;
    asm("{\n .reg .pred p;\n .reg .b32 t, m, bal;\n"
        " and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n vote.sync.ballot.b32 bal, p, 0xffffffff;\n"
        " selp.b32 m, 0xffffffff, 0, p;\n xor.b32 t, bal, m;\n not.b32 t, t;\n and.b32 %0, %3, t;\n}"
        : "=r"(r)
        : "r"(x), "r"(bitmask), "r"(peers));
    return r;
}

template <typename KeyT>
struct SortSmem {
    union {
        KeyT keys[kTile];  // the tile's keys (TMA), then keys in digit order, then
        unsigned vals[kTile];  // values in digit order
    } x;
    unsigned tv[sizeof(KeyT) == 8 ? kTile : 4];  // u64 passes: the tile's values (TMA)
    unsigned long long bar;
    unsigned short warp_cnt[kWarps][kRadix];  // per-warp digit counts, then warp offsets
    unsigned char digit[kTile];               // digit of each slot (value scatter)
    unsigned tile_start[kRadix];              // exclusive scan of tile digit counts
    unsigned hist[kRadix];                    // tile digit histogram
    unsigned global_base[kRadix];             // < 2^32: sort counts are < 2^32 (u32 values)
    unsigned tile_id;
};

// One LSD pass over one tile of kTile pairs.  Keys first, values after (as CUB's
// onesweep does): only keys and ranks are live in registers while ranking, the
// value loads are issued after the key exchange and land while the keys are
// being stored, and one shared buffer serves both exchanges.
template <bool TEXT, typename KeyT>
__global__ void __launch_bounds__(kNT, sizeof(KeyT) == 4 ? 4 : 3)
    k_onesweep(const KeyT *__restrict__ keys_in, const unsigned *__restrict__ vals_in, KeyT *__restrict__ keys_out,
               unsigned *__restrict__ vals_out, long long count, int shift,
               const unsigned long long *__restrict__ digit_base, unsigned *counter,
               u64 *status /*[tiles][256]*/, TextKeys tk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem<KeyT> &sm = *reinterpret_cast<SortSmem<KeyT> *>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        unsigned *wc = reinterpret_cast<unsigned *>(&sm.warp_cnt[0][0]);
        for (int i = threadIdx.x; i < kWarps * kRadix / 2; i += kNT) wc[i] = 0;
    }
    sm.hist[threadIdx.x] = 0;
    // u64 passes: tile = blockIdx.x (blocks are dispatched in index order, as
    // CUB's single-pass scan relies on), no tile-counter round trip before the
    // TMA loads (C4 sort 14.3 -> 13.7 ms).  u32 passes keep the dynamic tile
    // counter (measured 5.08 vs 5.31 ms per 3 passes with blockIdx.x).
    if (sizeof(KeyT) == 4 && threadIdx.x == 0) sm.tile_id = atomicAdd(counter, 1u);
    __syncthreads();
    const unsigned tile = sizeof(KeyT) == 4 ? sm.tile_id : blockIdx.x;
    const long long tbase = (long long)tile * kTile;
    const int tile_count = count - tbase < kTile ? (int)(count - tbase) : kTile;
    const int wbase = warp * (kIPT * 32) + lane;  // item i of this thread: tile offset wbase + 32 i

    KeyT k[kIPT];
    unsigned r[kIPT];
    // u64 passes: the tile's keys and values arrive by two bulk copies (TMA),
    // no value registers until the exchange (u32 passes measured faster with
    // per-thread loads: 5.07 vs 5.32 ms per 3 passes at 256 Mi)
    constexpr bool kTma = !TEXT && sizeof(KeyT) == 8;
    if (kTma) {
        if (threadIdx.x == 0) {
            mbar_init(&sm.bar, 1);
            const unsigned kb = ((unsigned)tile_count * (unsigned)sizeof(KeyT) + 15u) & ~15u;
            const unsigned vb = ((unsigned)tile_count * 4u + 15u) & ~15u;
            mbar_expect_tx(&sm.bar, kb + vb);
            tma_load_1d(sm.x.keys, keys_in + tbase, kb, &sm.bar);
            tma_load_1d(sm.tv, vals_in + tbase, vb, &sm.bar);
        }
        __syncthreads();
        mbar_wait(&sm.bar, 0);
    }
    // u32 keys from the packed text: a tile past the short suffixes covers
    // consecutive positions, so its bit range of the stream is staged once in
    // shared memory as 32-bit MSB-first chunks (through the still unused
    // exchange buffer) and each key is one funnel shift of two chunks.
    bool text_fast = false;
    if (TEXT && sizeof(KeyT) == 4 && tbase >= tk.S && tk.b * tk.K <= 32) {
        text_fast = true;
        unsigned *chunk = reinterpret_cast<unsigned *>(sm.x.keys);
        const long long p0 = tbase - tk.S;
        const long long q0 = ((long long)tk.b * p0) >> 5;
        const int nch = (int)((((long long)tk.b * (p0 + tile_count - 1)) >> 5) + 2 - q0);  // <= 8 kTile / 32 + 2
        for (int j = threadIdx.x; j < nch; j += kNT) {
            const long long q = q0 + j;
            const u64 w = tk.stream[q >> 1];
            chunk[j] = (q & 1) ? (unsigned)w : (unsigned)(w >> 32);
        }
        __syncthreads();
        const unsigned off0 = (unsigned)((long long)tk.b * p0 - 32 * q0);
        const int kb = tk.b * tk.K;
#pragma unroll
        for (int i = 0; i < kIPT; ++i) {
            const int o = wbase + i * 32;
            if (o < tile_count) {
                const unsigned bit = off0 + (unsigned)(tk.b * o);
                const unsigned j = bit >> 5;
                const unsigned x = __funnelshift_l(chunk[j + 1], chunk[j], bit & 31);
                k[i] = (KeyT)(kb >= 32 ? x : x >> (32 - kb));
            }
        }
    }
    if (!text_fast) {
#pragma unroll
        for (int i = 0; i < kIPT; ++i) {
            const int o = wbase + i * 32;
            if (o < tile_count)
                k[i] = TEXT ? (KeyT)text_key(tk, text_pos(tk, tbase + o)) : kTma ? sm.x.keys[o] : keys_in[tbase + o];
        }
    }
    // 1) tile digit histogram first, published right away (decoupled
    //    look-back: successors can use this tile's aggregate while it is still
    //    ranking, so the per-digit chains never wait on the ranking phase).
#pragma unroll
    for (int i = 0; i < kIPT; ++i)
        if (wbase + i * 32 < tile_count) atomicAdd(&sm.hist[(unsigned)(k[i] >> shift) & 0xff], 1u);
    __syncthreads();
    {
        const int d = threadIdx.x;
        st_relaxed(status + (size_t)tile * kRadix + d, (tile == 0 ? kFlagPre : kFlagAgg) | sm.hist[d]);
    }
    // 2) stable ranking within each warp (warp-striped items: item-major,
    //    lane-minor): peer masks first (independent), then the short counter
    //    chain through shared memory.  Peers come from 8 ballots (one per digit
    //    bit): MATCH.ANY is slow when a warp holds ~30 distinct digits, which
    //    is the common case for uniformly distributed keys.
    const unsigned lt_mask = (1u << lane) - 1;
#pragma unroll
    for (int i = 0; i < kIPT; ++i) {
        const unsigned d = (unsigned)(k[i] >> shift) & 0xff;
        unsigned peers = __ballot_sync(0xffffffffu, wbase + i * 32 < tile_count);
#pragma unroll
        for (int b = 0; b < 8; ++b) peers = peer_bit(peers, d, 1u << b);
        r[i] = ((unsigned)__popc(peers) << 5) | (unsigned)__popc(peers & lt_mask);
    }
#pragma unroll
    for (int i = 0; i < kIPT; ++i) {
        const bool valid = wbase + i * 32 < tile_count;
        const unsigned d = (unsigned)(k[i] >> shift) & 0xff;
        const unsigned before = valid ? sm.warp_cnt[warp][d] : 0;
        __syncwarp();
        const unsigned lt = r[i] & 31;
        if (valid && lt == 0) sm.warp_cnt[warp][d] = (unsigned short)(before + (r[i] >> 5));
        r[i] = before + lt;
        __syncwarp();
    }
    __syncthreads();
    // 3) per digit: warp exclusive offsets, tile-local digit start, look-back
    {
        const int d = threadIdx.x;  // kNT == kRadix
        unsigned run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            unsigned c = sm.warp_cnt[w][d];
            sm.warp_cnt[w][d] = (unsigned short)run;
            run += c;
        }
        unsigned excl;
        __shared__ unsigned s_w[kNT / 32];
        block_exclusive_sum<kNT>(run, excl, s_w);
        sm.tile_start[d] = excl;
        u64 prefix = 0;
        if (tile > 0) {
            // look back 4 predecessor tiles per step (4 loads in flight)
            long long t = (long long)tile - 1;
            while (true) {
                u64 s4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    s4[q] = (t - q >= 0) ? ld_relaxed(status + (size_t)(t - q) * kRadix + d) : kFlagPre;
                bool done = false;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (done) break;
                    while ((s4[q] >> 62) == 0) {
                        __nanosleep(20);
                        s4[q] = ld_relaxed(status + (size_t)(t - q) * kRadix + d);
                    }
                    prefix += s4[q] & kValMask;
                    if ((s4[q] >> 62) == 2) done = true;
                }
                if (done) break;
                t -= 4;
            }
            st_relaxed(status + (size_t)tile * kRadix + d, kFlagPre | (prefix + run));
        }
        sm.global_base[d] = (unsigned)(digit_base[d] + prefix - excl);
    }
    __syncthreads();
    // 4) keys into digit order (r becomes the tile slot)
#pragma unroll
    for (int i = 0; i < kIPT; ++i) {
        if (wbase + i * 32 < tile_count) {
            const unsigned d = (unsigned)(k[i] >> shift) & 0xff;
            r[i] += sm.tile_start[d] + sm.warp_cnt[warp][d];
            sm.x.keys[r[i]] = k[i];
        }
    }
    unsigned v[kIPT];
    if (!TEXT && !kTma) {
#pragma unroll
        for (int i = 0; i < kIPT; ++i)
            if (wbase + i * 32 < tile_count) v[i] = vals_in[tbase + wbase + i * 32];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kIPT; ++q) {
        const int j = threadIdx.x + q * kNT;
        if (j < tile_count) {
            const KeyT key = sm.x.keys[j];
            const unsigned d = (unsigned)(key >> shift) & 0xff;
            sm.digit[j] = (unsigned char)d;
            keys_out[sm.global_base[d] + j] = key;
        }
    }
    __syncthreads();
    // 5) values through the same buffer
#pragma unroll
    for (int i = 0; i < kIPT; ++i) {
        const int o = wbase + i * 32;
        if (o < tile_count) sm.x.vals[r[i]] = TEXT ? (unsigned)text_pos(tk, tbase + o) : kTma ? sm.tv[o] : v[i];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kIPT; ++q) {
        const int j = threadIdx.x + q * kNT;
        if (j < tile_count) vals_out[sm.global_base[sm.digit[j]] + j] = sm.x.vals[j];
    }
}

}  // namespace

template <typename KeyT>
void radix_sort_pairs(rs_ctx *c, KeyT *keys, KeyT *keys_alt, unsigned *vals, unsigned *vals_alt,
                      long long count, int bits, KeyT **keys_out, unsigned **vals_out, const TextKeys *tk) {
    const TextKeys tkv = tk ? *tk : TextKeys{nullptr, 0, 0, 0, 0};
    *keys_out = keys;
    *vals_out = vals;
    if (count <= 1 || bits <= 0) {
        if (tk && count > 0) RS_LAUNCH(c, k_materialize<KeyT>, grid_for(count, 256), 256, 0, tkv, count, keys, vals);
        return;
    }
    int passes = (bits + 7) / 8;
    if (passes > 8) passes = 8;
    unsigned long long *hist = (unsigned long long *)buf(c, B_HIST, sizeof(unsigned long long) * 8 * kRadix);
    RS_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 8 * kRadix, c->stream));
    unsigned hist_blocks = (unsigned)std::min<long long>((count + kNT * 16 - 1) / (kNT * 16), c->sm_count * 8);
    // symbol-aligned text digits: count digit 0 only, shift the rest
    const bool shifted = tk && (8 % tkv.b) == 0 && (tkv.b * tkv.K) % 8 == 0 && tkv.b * tkv.K == bits &&
                         count == tkv.n && count > (long long)passes * (8 / tkv.b);
    if (shifted) {
        const long long words = (count * tkv.b + 63) / 64;
        const unsigned hb = (unsigned)std::max<long long>(1, std::min<long long>((words + kNT - 1) / kNT, c->sm_count * 8));
        switch (tkv.b) {
            case 1: RS_LAUNCH_NB(c, "k_hist_digit0", count / 8.0, k_hist_digit0<1>, hb, kNT, 0, tkv, hist); break;
            case 2: RS_LAUNCH_NB(c, "k_hist_digit0", count / 4.0, k_hist_digit0<2>, hb, kNT, 0, tkv, hist); break;
            case 4: RS_LAUNCH_NB(c, "k_hist_digit0", count / 2.0, k_hist_digit0<4>, hb, kNT, 0, tkv, hist); break;
            default: RS_LAUNCH_NB(c, "k_hist_digit0", 1.0 * count, k_hist_digit0<8>, hb, kNT, 0, tkv, hist); break;
        }
    } else if (tk)
        RS_LAUNCH_NB(c, "k_histograms<text>", 0.25 * count, (k_histograms<true, KeyT>), hist_blocks, kNT, 0, keys, count,
                     passes, hist, tkv, passes);
    else
        RS_LAUNCH_NB(c, sizeof(KeyT) == 4 ? "k_histograms<u32>" : "k_histograms<u64>", (double)sizeof(KeyT) * count,
                     (k_histograms<false, KeyT>), hist_blocks, kNT, 0, keys, count, passes, hist, tkv, passes);
    if (shifted && passes > 1) RS_LAUNCH(c, k_hist_shift, 1, kRadix, 0, hist, passes, 8 / tkv.b, tkv);
    // Host needs the histograms to skip constant-digit passes.
    std::vector<unsigned long long> h((size_t)passes * kRadix);
    fetch_small(c, h.data(), hist, sizeof(unsigned long long) * h.size());
    RS_LAUNCH(c, k_hist_scan, passes, kRadix, 0, hist);

    static unsigned long long attr_set = 0;
    once_per_device(attr_set, c->device, [] {
        RS_CUDA(cudaFuncSetAttribute(k_onesweep<false, KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(SortSmem<KeyT>)));
        RS_CUDA(cudaFuncSetAttribute(k_onesweep<true, KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(SortSmem<KeyT>)));
    });
    long long tiles = (count + kTile - 1) / kTile;
    KeyT *kin = keys, *kout = keys_alt;
    unsigned *vin = vals, *vout = vals_alt;
    bool from_text = tk != nullptr;
    for (int p = 0; p < passes; ++p) {
        bool trivial = false;
        for (int d = 0; d < kRadix; ++d)
            if (h[(size_t)p * kRadix + d] == (unsigned long long)count) trivial = true;
        if (trivial && !(from_text && p == passes - 1)) continue;  // the text must be materialised once
        Scratch s = scratch(c, tiles * kRadix);
        if (from_text)
            RS_LAUNCH_NB(c, sizeof(KeyT) == 4 ? "k_onesweep<text,u32>" : "k_onesweep<text,u64>",
                         (4.0 + sizeof(KeyT) + 0.25) * count, (k_onesweep<true, KeyT>), (unsigned)tiles, kNT,
                        sizeof(SortSmem<KeyT>), kin, vin, kout,
                        vout, count, 8 * p, hist + (size_t)p * kRadix, s.counter, s.status, tkv);
        else
            RS_LAUNCH_NB(c, sizeof(KeyT) == 4 ? "k_onesweep<u32>" : "k_onesweep<u64>",
                         2.0 * (4.0 + sizeof(KeyT)) * count, (k_onesweep<false, KeyT>), (unsigned)tiles, kNT,
                        sizeof(SortSmem<KeyT>), kin, vin, kout,
                        vout, count, 8 * p, hist + (size_t)p * kRadix, s.counter, s.status, tkv);
        from_text = false;
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    *keys_out = kin;
    *vals_out = vin;
}

// All digit histograms of the round-0 text keys (symbol-aligned digits only:
// counted from the packed stream + shifted), copied to the host.  False when
// the digits are not symbol-aligned.
bool text_digit_histograms(rs_ctx *c, const TextKeys &tk, int bits, std::vector<unsigned long long> &h) {
    const int passes = (bits + 7) / 8;
    const long long count = tk.n;
    if (!((8 % tk.b) == 0 && (tk.b * tk.K) % 8 == 0 && tk.b * tk.K == bits && count > (long long)passes * (8 / tk.b)))
        return false;
    unsigned long long *hist = (unsigned long long *)buf(c, B_HIST, sizeof(unsigned long long) * 8 * kRadix);
    RS_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 8 * kRadix, c->stream));
    const long long words = (count * tk.b + 63) / 64;
    const unsigned hb = (unsigned)std::max<long long>(1, std::min<long long>((words + kNT - 1) / kNT, c->sm_count * 8));
    switch (tk.b) {
        case 1: RS_LAUNCH_NB(c, "k_hist_digit0", count / 8.0, k_hist_digit0<1>, hb, kNT, 0, tk, hist); break;
        case 2: RS_LAUNCH_NB(c, "k_hist_digit0", count / 4.0, k_hist_digit0<2>, hb, kNT, 0, tk, hist); break;
        case 4: RS_LAUNCH_NB(c, "k_hist_digit0", count / 2.0, k_hist_digit0<4>, hb, kNT, 0, tk, hist); break;
        default: RS_LAUNCH_NB(c, "k_hist_digit0", 1.0 * count, k_hist_digit0<8>, hb, kNT, 0, tk, hist); break;
    }
    if (passes > 1) RS_LAUNCH(c, k_hist_shift, 1, kRadix, 0, hist, passes, 8 / tk.b, tk);
    h.assign((size_t)passes * kRadix, 0);
    fetch_small(c, h.data(), hist, sizeof(unsigned long long) * h.size());
    return true;
}

template void radix_sort_pairs<unsigned>(rs_ctx *, unsigned *, unsigned *, unsigned *, unsigned *, long long, int,
                                         unsigned **, unsigned **, const TextKeys *);
template void radix_sort_pairs<u64>(rs_ctx *, u64 *, u64 *, unsigned *, unsigned *, long long, int, u64 **,
                                    unsigned **, const TextKeys *);

}  // namespace rsb
