// common.cuh -- shared runtime pieces of librepeatscan_b200 (sm_100a only).
//
// * rs_ctx: one per process per device; owns a stream, a grow-only device
//   buffer arena, CUDA events and the device-resident pipeline state.
// * RsError: internal exception; the C-ABI (capi.cu) maps it to a status code
//   plus rs_last_error().
// * Decoupled look-back (single-pass scan) primitives used by compaction,
//   the all-ties scan, the radix sort and the group-head scans.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/repeatscan_b200.h"

namespace rsb {

typedef unsigned long long u64;
typedef long long i64;

struct RsError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string &msg);
void check_cuda(cudaError_t e, const char *what, const char *file, int line);
#define RS_CUDA(x) ::rsb::check_cuda((x), #x, __FILE__, __LINE__)

enum BufId {
    B_TEXT = 0,
    B_SA,
    B_ISA,
    B_LCP,
    B_RAW,
    B_LLRC,      // uint2 (start, len) compact entries
    B_BOUNDS,    // per-grain (lo, hi) for the scan kernels
    B_OUT0,      // int64 answers: leftmost starts | all lengths
    B_OUT1,      // int64 answers: leftmost lengths | all offsets
    B_FLAT,      // int64 tie starts
    B_KEYS0,
    B_KEYS1,
    B_VALS0,
    B_VALS1,
    B_SCRATCH,   // look-back status words + counters
    B_HIST,      // radix histograms
    B_PHI,
    B_PLCP,
    B_T0,
    B_T1,
    B_T2,
    B_T3,
    B_I64A,      // staging for int64 API arrays
    B_I64B,
    B_I64C,
    B_I64D,
    B_SMALL,     // small device scalars (error flags, counts)
    B_CURSOR,    // bucketed-scatter fill counts
    B_T4,
    B_T5,
    B_PATCH,     // list of patched LCP slots
    B_PACKED,    // text packed as b-bit codes
    B_TSV,       // serialized TSV bytes
    B_H0,        // per-round unsorted group heads / suffixes (ping-pong)
    B_H1,
    B_V0,
    B_V1,
    B_SEND,      // distributed sort: (position, raw) entries bound for other ranks
    B_XFER,      // host_io.cu: two-slot device ring of 32-bit wire words
    B_XFER_ENDS, // host_io.cu: first / last value of every chunk
    B_WIRE,      // host_io.cu: byte-wide wire copy of the all-ties CSR
    B_COUNT
};

struct Buf {
    void *p = nullptr;
    size_t cap = 0;
};

constexpr int kMaxEvents = 64;

}  // namespace rsb

struct rs_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    std::string err;
    rsb::Buf bufs[rsb::B_COUNT];
    long long launches = 0;
    cudaEvent_t events[rsb::kMaxEvents] = {};
    void *small_host = nullptr;  // pinned scratch for scalar readbacks
    void *xfer_host[2] = {nullptr, nullptr};        // host_io.cu pinned pipeline slots
    void *nccl_comm = nullptr;                      // collectives.cu (ncclComm_t)
    int nccl_rank = 0, nccl_world = 1;
    cudaEvent_t xfer_ev[2] = {nullptr, nullptr};
    cudaStream_t xfer_side = nullptr;                // host_io.cu direct-DMA side stream
    cudaEvent_t xfer_side_ev = nullptr;
    long long h2d_bytes = 0, d2h_bytes = 0;         // host <-> device bytes copied (rs_transfer_bytes)
    // pipeline state
    long long n = -1;
    bool have_text = false;
    bool have_sa = false;   // SA + ISA on device
    bool have_lcp = false;  // SA-order LCP on device
    bool have_raw = false;
    bool have_compact = false;
    long long m = 0;
    int out_mode = -1;      // 0 leftmost, 1 all (what B_OUT* hold)
    long long total = 0;    // tie total of the last all-ties query
    int sa_rounds = 0;      // prefix-doubling rounds of the last SA build
    long long shard_lo = 0, shard_hi = 0;
    // distributed suffix sort state (one rank's segment; suffix_array.cu dist_*)
    struct {
        long long m = 0, S = 0, P0 = 0, P1 = 0, R0 = 0, hcap = 0, send_total = 0;
        unsigned *keys = nullptr, *vals = nullptr;
        unsigned long long first_key = 0, last_key = 0;
        unsigned first_pos = 0, last_pos = 0;
        int bits = 0, K = 0, stage = 0;  // stage: 1 sorted, 2 updated, 3 applied
    } dist;
    int sa_key_symbols = 0;                 // K of the round-0 keys
    int packed_bits = 0;                    // B_PACKED holds the current text at this many bits/symbol (0: none)
    bool isa_lazy = false;                  // B_ISA not built (device SA without later rounds): fill from SA on demand
    long long sa_unsorted_after_round0 = 0; // suffixes left in tied groups by round 0
    long long sa_final_depth = 0;          // sorted depth when prefix doubling stopped
    bool lcp_from_keys = false;             // B_LCP holds round-0 key LCPs (+ unknown marks)
    bool sa_device_built = false;           // SA/ISA/LCP built here (mutually consistent)
    bool sa_isa_consistent = false;         // caller sa/rank checked to be inverse permutations
    long long max_lcp = -1;                 // max of the resident LCP (-1: not computed)
    bool raw_from_round0 = false;           // B_RAW filled during the SA build (+ LCP patch fix-up)
    long long tsv_bytes = 0;
    long long patch_slots = 0;              // tied slots of round 0 kept in B_PATCH
    bool out_ref_layout = false;            // B_OUT* hold the reference 1-based layout
    // per-kernel profiling (CUDA events around every launch while enabled)
    bool profiling = false;
    struct ProfRec {
        const char *name;
        int ev0, ev1;
        double bytes;
    };
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> prof_events;
    struct ProfAgg {
        std::string name;
        long long launches;
        double ms, bytes;
    };
    std::vector<ProfAgg> prof_agg;
    double stage_ms[RS_NUM_STAGES] = {};
};

namespace rsb {

void *buf(rs_ctx *c, BufId id, size_t bytes);
void fetch_small(rs_ctx *c, void *host, const void *dev, size_t bytes);

// Counts one kernel launch, surfaces launch errors and, while profiling,
// brackets it with CUDA events.  `bytes` = algorithmic HBM bytes of the launch
// (the roofline numerator), 0 if not meaningful.
void before_launch(rs_ctx *c);
void after_launch(rs_ctx *c, const char *name, double bytes);
// Adds algorithmic bytes to the most recent launch (for outputs whose size is
// only known after the kernel ran, e.g. the tie total).
void add_bytes_last(rs_ctx *c, double bytes);
#define RS_LAUNCH_B(ctx, bytes, kernel, grid, block, smem, ...)                \
    do {                                                                       \
        ::rsb::before_launch(ctx);                                             \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);      \
        ::rsb::after_launch((ctx), #kernel, (double)(bytes));                  \
    } while (0)
// Same with an explicit profile name (template instantiations with type args).
#define RS_LAUNCH_NB(ctx, name, bytes, kernel, grid, block, smem, ...)        \
    do {                                                                       \
        ::rsb::before_launch(ctx);                                             \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);      \
        ::rsb::after_launch((ctx), (name), (double)(bytes));                   \
    } while (0)
#define RS_LAUNCH(ctx, kernel, grid, block, smem, ...) \
    RS_LAUNCH_B(ctx, 0, kernel, grid, block, smem, __VA_ARGS__)

// Kernel attributes (cudaFuncSetAttribute) are per device context: run `f`
// once per call site and device (a process may drive several devices).
template <typename F>
inline void once_per_device(unsigned long long &mask, int device, F &&f) {
    const unsigned long long bit = 1ull << (device & 63);
    if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit) return;
    f();
    __atomic_fetch_or(&mask, bit, __ATOMIC_RELEASE);
}

inline unsigned grid_for(long long items, int per_block) {
    long long g = (items + per_block - 1) / per_block;
    return (unsigned)(g < 1 ? 1 : g);
}

// ----------------------------------------------------------------------------
// Decoupled look-back.  Status word: bits 63..62 = flag (0 invalid,
// 1 aggregate, 2 inclusive prefix), bits 61..0 = value.
// ----------------------------------------------------------------------------
constexpr u64 kFlagAgg = 1ull << 62;
constexpr u64 kFlagPre = 2ull << 62;
constexpr u64 kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_relaxed(u64 *p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_relaxed(const u64 *p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

struct OpSum {
    __device__ __forceinline__ u64 operator()(u64 a, u64 b) const { return a + b; }
    static constexpr u64 identity = 0;
};
struct OpMax {
    __device__ __forceinline__ u64 operator()(u64 a, u64 b) const { return a > b ? a : b; }
    static constexpr u64 identity = 0;
};
// Two scans in one look-back: max over bits 61..31, sum over bits 30..0
// (both operands < 2^31, sums of n <= 2^31 - 2 items of 0/1 never carry).
struct OpMaxSum {
    __device__ __forceinline__ u64 operator()(u64 a, u64 b) const {
        const u64 m = (1ull << 31) - 1;
        u64 ha = a >> 31, hb = b >> 31;
        return ((ha > hb ? ha : hb) << 31) | (((a & m) + (b & m)) & m);
    }
    static constexpr u64 identity = 0;
};

template <typename Op>
__device__ __forceinline__ u64 warp_reduce(u64 v, Op op) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Called by ONE full warp of the tile.  Publishes `aggregate` for `tile`,
// looks back over predecessors and returns the exclusive prefix (identical
// in every lane).  status[] must be zeroed before the launch.
//
// Forward-progress assumption: a tile only waits on LOWER tile ids.  Kernels
// that take their tile id from an atomic counter (k_scan_i64, k_onesweep on
// u32 keys, k_compact_raw, ...) are safe under any block scheduling.  Two hot
// kernels (k_query_fused, k_onesweep on u64 keys) use tile = blockIdx.x to
// save the counter round trip before their TMA loads; that relies on the
// hardware dispatching a grid's blocks in increasing linear index, which it
// does for a whole GPU (measured: every launch in the parity suites and the
// fuzzers) but which is not a documented guarantee -- do not run those two
// under MPS / green-context SM partitioning without switching them back to
// the atomic tile counter.
// published = true: the caller already stored the tile's aggregate (or, for
// tile 0, its inclusive prefix) with lookback_publish, earlier, so that
// successors waiting on it are released before this tile starts waiting.
__device__ __forceinline__ void lookback_publish(u64 *status, long long tile, u64 aggregate) {
    st_relaxed(&status[tile], (tile == 0 ? kFlagPre : kFlagAgg) | (aggregate & kValMask));
}

template <typename Op>
__device__ u64 lookback_warp(u64 *status, long long tile, u64 aggregate, Op op, bool published = false) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0 && !published) st_relaxed(&status[0], kFlagPre | (aggregate & kValMask));
        return Op::identity;
    }
    if (lane == 0 && !published) st_relaxed(&status[tile], kFlagAgg | (aggregate & kValMask));
    u64 exclusive = Op::identity;
    long long base = tile - 1;
    while (true) {
        long long idx = base - lane;
        u64 s = idx >= 0 ? ld_relaxed(&status[idx]) : (kFlagPre | Op::identity);
        unsigned pre, ns = 32;
        int first;
        // wait only for the predecessors up to the nearest inclusive prefix:
        // tiles before it do not matter (waiting for all 32 lanes made a tile
        // spin ~170 times on neighbours it never needed)
        while (true) {
            pre = __ballot_sync(0xffffffffu, (s >> 62) == 2);
            first = pre ? __ffs(pre) - 1 : 32;
            const unsigned need = first == 32 ? 0xffffffffu : (2u << first) - 1u;
            const unsigned waiting = __ballot_sync(0xffffffffu, (s >> 62) == 0) & need;
            if (!waiting) break;
            __nanosleep(ns);  // exponential backoff: a waiting warp issues few instructions
            ns = ns < 512 ? 2 * ns : ns;
            if (waiting >> lane & 1) s = ld_relaxed(&status[idx]);
        }
        u64 v = (lane <= first) ? (s & kValMask) : Op::identity;
        v = warp_reduce(v, op);
        exclusive = op(exclusive, v);
        if (pre) break;
        base -= 32;
    }
    if (lane == 0) st_relaxed(&status[tile], kFlagPre | (op(exclusive, aggregate) & kValMask));
    return exclusive;
}

// Look-back for full 64-bit payloads (the int64 API scan, engine.py:77-110,
// whose values may be negative or exceed 2^62).  The flag lives in its own
// word and each tile has separate aggregate and inclusive slots, each written
// once before the flag that announces it (release / acquire), so a reader
// never pairs a flag with a value it does not describe.
// st layout: flag[tiles] | agg[tiles] | incl[tiles], zeroed before the launch.
__device__ __forceinline__ void st_release(u64 *p, u64 v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire(const u64 *p) {
    u64 v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __noinline__ static u64 lookback_warp_wide(u64 *st, long long tiles, long long tile, u64 aggregate) {
    const int lane = threadIdx.x & 31;
    u64 *flag = st, *agg = st + tiles, *incl = st + 2 * tiles;
    if (tile == 0) {
        if (lane == 0) {
            st_relaxed(&incl[0], aggregate);
            st_release(&flag[0], 2);
        }
        return 0;
    }
    if (lane == 0) {
        st_relaxed(&agg[tile], aggregate);
        st_release(&flag[tile], 1);
    }
    u64 exclusive = 0;
    long long base = tile - 1;
    while (true) {
        long long idx = base - lane;
        u64 f = idx >= 0 ? ld_acquire(&flag[idx]) : 2, v = 0;
        unsigned pre;
        int first;
        while (true) {  // wait only for the lanes up to the nearest inclusive prefix
            pre = __ballot_sync(0xffffffffu, f == 2);
            first = pre ? __ffs(pre) - 1 : 32;
            const unsigned need = first == 32 ? 0xffffffffu : (2u << first) - 1u;
            const unsigned waiting = __ballot_sync(0xffffffffu, f == 0) & need;
            if (!waiting) break;
            __nanosleep(20);
            if (waiting >> lane & 1) f = ld_acquire(&flag[idx]);
        }
        if (idx >= 0 && lane <= first) v = ld_relaxed(f == 2 ? &incl[idx] : &agg[idx]);
        v = warp_reduce(v, OpSum());
        exclusive += v;
        if (pre) break;
        base -= 32;
    }
    if (lane == 0) {
        st_relaxed(&incl[tile], exclusive + aggregate);
        st_release(&flag[tile], 2);
    }
    return exclusive;
}

// Block-wide exclusive sum of one u32 per thread; returns the block total.
// kTrailingSync = false: the caller never rewrites s_warp before its next
// __syncthreads (saves the closing barrier).
template <int NT, bool kTrailingSync = true>
__device__ __forceinline__ unsigned block_exclusive_sum(unsigned v, unsigned &excl,
                                                        unsigned *s_warp /*[NT/32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned w = (lane < NT / 32) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    unsigned warp_base = warp ? s_warp[warp - 1] : 0;
    excl = warp_base + x - v;
    unsigned total = s_warp[NT / 32 - 1];
    if (kTrailingSync) __syncthreads();
    return total;
}

// 64-bit variant.
template <int NT>
__device__ __forceinline__ u64 block_exclusive_sum64(u64 v, u64 &excl, u64 *s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u64 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        u64 w = (lane < NT / 32) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u64 y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) s_warp[lane] = w;
    }
    __syncthreads();
    u64 warp_base = warp ? s_warp[warp - 1] : 0;
    excl = warp_base + x - v;
    u64 total = s_warp[NT / 32 - 1];
    __syncthreads();
    return total;
}

// Block-wide inclusive max-scan of one u64 per thread.
template <int NT>
__device__ __forceinline__ u64 block_inclusive_max64(u64 v, u64 &incl, u64 *s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u64 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = x > y ? x : y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        u64 w = (lane < NT / 32) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u64 y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w = w > y ? w : y;
        }
        if (lane < NT / 32) s_warp[lane] = w;
    }
    __syncthreads();
    u64 wb = warp ? s_warp[warp - 1] : 0;
    incl = x > wb ? x : wb;
    u64 total = s_warp[NT / 32 - 1];
    __syncthreads();
    return total;
}

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

// Scratch layout for single-pass kernels: [counter (u64)] [status words ...].
struct Scratch {
    unsigned *counter;
    u64 *status;
};
// Zeroes and returns scratch for `tiles` look-back tiles (async on ctx stream).
Scratch scratch(rs_ctx *c, long long tiles, int slot = 0);

// ----------------------------------------------------------------------------
// Host-side stage entry points (defined in the .cu files).
// ----------------------------------------------------------------------------
// compact.cu
long long compact_from_raw(rs_ctx *c, long long n);                 // B_RAW -> B_LLRC, returns m
void raw_from_rank_lcp(rs_ctx *c, long long n);                     // B_ISA(rank-1), B_LCP -> B_RAW
void narrow_i64_to_u32(rs_ctx *c, const long long *d_in, unsigned *d_out, long long count,
                       long long lo, long long hi, long long add, const char *what);
void widen_u32_to_i64(rs_ctx *c, const unsigned *d_in, long long *d_out, long long count,
                      long long add);
// scan_query.cu
void query(rs_ctx *c, long long n, int mode, int path);  // -> B_OUT0/B_OUT1/B_FLAT
// suffix_array.cu
void build_suffix_array(rs_ctx *c, long long n);         // B_TEXT -> B_SA, B_ISA
void build_lcp(rs_ctx *c, long long n);                  // B_TEXT, B_SA, B_ISA -> B_LCP
// radix_sort.cu
// Sorts (keys, vals) pairs by the low `bits` bits of keys, stable.  Result
// lands in the returned buffers (ping-pong between the two given pairs).
// Round-0 keys generated on the fly from the text packed as a big-endian bit
// stream of b-bit symbol codes: key(p) = bits [b*p, b*p + b*K) of the stream,
// and the element order is the suffix-sort input order (short suffixes first).
struct TextKeys {
    const u64 *stream;   // packed codes, zero padded past the end
    long long n;         // text length
    int b, K;            // code bits, symbols per key
    long long S;         // number of short suffixes placed first
};
__device__ __forceinline__ u64 text_key(const TextKeys &tk, long long p) {
    const long long o = (long long)tk.b * p;
    const u64 *w = tk.stream + (o >> 6);
    const unsigned sh = (unsigned)(o & 63);
    u64 x = w[0];
    if (sh) x = (x << sh) | (w[1] >> (64 - sh));
    const int kb = tk.b * tk.K;
    return kb >= 64 ? x : (x >> (64 - kb));
}
__device__ __forceinline__ long long text_pos(const TextKeys &tk, long long e) {
    return e < tk.S ? tk.n - 1 - e : e - tk.S;
}
bool text_digit_histograms(rs_ctx *c, const TextKeys &tk, int bits, std::vector<unsigned long long> &h);

// Text prepared for the suffix sort (suffix_array.cu prepare_text).
struct TextPrep {
    u64 *stream;      // B_PACKED: b-bit codes, zero padded
    long long words;  // stream words incl. padding
    int bits, K, sigma;
};
TextPrep prepare_text(rs_ctx *c, long long n);

// Round-0 update over one rank's contiguous segment of the suffix array: the
// text length and the LCPs with the neighbouring segments' boundary suffixes
// (0 at the ends of the whole array).
struct SegBoundary {
    long long n_text;
    unsigned lcp_first, lcp_last;
    unsigned long long *group_count;  // optional: += number of still-tied groups (final pass)
};

// Sorts (keys, vals) pairs by the low `bits` bits of keys, stable.  With tk,
// the input pairs are generated from the packed text (keys/vals unread).
template <typename KeyT>
void radix_sort_pairs(rs_ctx *c, KeyT *keys, KeyT *keys_alt, unsigned *vals, unsigned *vals_alt,
                      long long count, int bits, KeyT **keys_out, unsigned **vals_out,
                      const TextKeys *tk = nullptr);

}  // namespace rsb
