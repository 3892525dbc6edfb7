// compact.cu -- raw LLR array and its compaction (north-star subsystem 2).
//
// Reference semantics:
//   raw[i]  = max(lcp[rank[i]], lcp[rank[i]+1])          _kernels_numba.py:33-38
//   flag[i] = raw[i] > 0 && raw[i] >= raw[i-1]            _kernels_numba.py:41-46
//   ps      = inclusive scan of flags                     engine.py:77-110
//   LLRc[ps[i]-1] = (i, raw[i]) if flag[i]                _kernels_numba.py:49-55
//
// B200 design: flag -> scan -> scatter is ONE single-pass kernel (block scan
// + decoupled look-back across tiles, dynamic tile ids), so raw is read once
// and LLRc written once: 4n + 8m algorithmic bytes.  The int64 kernels at the
// bottom serve the array-level API (compute_flags / prefix_sum /
// scatter_compact on caller arrays).
#include "common.cuh"

namespace rsb {

namespace {

constexpr int kNT = 256;
// 32 slots per thread: a decoupled look-back per 8192 slots (with 2048 the
// tiles mostly waited on their predecessors: 1.1 TB/s at 1 Gi slots)
constexpr int kIPT = 32;
constexpr int kTile = kNT * kIPT;  // 8192 raw slots per tile

// raw: u32[n+1] (slot 0 = 0 pad), padded so reads up to the last tile are safe.
__global__ void __launch_bounds__(kNT) k_compact_raw(const unsigned *__restrict__ raw, long long n,
                                                     uint2 *__restrict__ llrc, unsigned long long *m_out,
                                                     unsigned *counter, u64 *status, long long tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[kNT / 32];
    __shared__ u64 s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long idx0 = tile * kTile + (long long)threadIdx.x * kIPT;
    unsigned v[kIPT];
    {
        const uint4 *p = reinterpret_cast<const uint4 *>(raw + idx0);
#pragma unroll
        for (int q = 0; q < kIPT / 4; ++q) {
            const uint4 a = __ldg(p + q);
            v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
        }
    }
#pragma unroll
    for (int j = 0; j < kIPT; ++j)
        if (idx0 + j > n) v[j] = 0;
    unsigned prev = __shfl_up_sync(0xffffffffu, v[kIPT - 1], 1);
    if ((threadIdx.x & 31) == 0) prev = (idx0 > 0 && idx0 - 1 <= n) ? raw[idx0 - 1] : 0;
    unsigned flags = 0, cnt = 0;
#pragma unroll
    for (int j = 0; j < kIPT; ++j) {
        unsigned p = j ? v[j - 1] : prev;
        bool f = v[j] > 0 && v[j] >= p;
        flags |= (unsigned)f << j;
        cnt += f;
    }
    unsigned excl;
    unsigned total = block_exclusive_sum<kNT>(cnt, excl, s_warp);
    if (threadIdx.x < 32) {
        u64 base = lookback_warp(status, tile, (u64)total, OpSum());
        if (threadIdx.x == 0) {
            s_base = base;
            if (tile == tiles - 1) *m_out = base + total;
        }
    }
    __syncthreads();
    u64 o = s_base + excl;
#pragma unroll
    for (int j = 0; j < kIPT; ++j)
        if (flags >> j & 1) llrc[o++] = make_uint2((unsigned)(idx0 + j), v[j]);
}

// raw[i] = max(lcp_d[isa[i-1]], lcp_d[isa[i-1]+1]) for i in 1..n (1-based i),
// with isa 0-based ranks and lcp_d[r] = lcp(sa[r-1], sa[r]), lcp_d[0] = lcp_d[n] = 0.
// 8 consecutive slots per thread so 16 independent random loads are in flight.
__global__ void k_raw_from_isa_lcp(const unsigned *__restrict__ isa, const unsigned *__restrict__ lcp_d,
                                   long long n, unsigned *__restrict__ raw, long long first = 0) {
    const long long i0 = first + (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 8;  // raw slots i0..i0+7
    if (i0 > n) return;
    unsigned r[8], a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        long long i = i0 + j;
        r[j] = (i >= 1 && i <= n) ? __ldg(isa + i - 1) : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (r[j] != 0xffffffffu) {
            a[j] = __ldg(lcp_d + r[j]);
            b[j] = __ldg(lcp_d + r[j] + 1);
        } else {
            a[j] = b[j] = 0;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (i0 + j <= n) raw[i0 + j] = a[j] > b[j] ? a[j] : b[j];
}

// ---- int64 array-level kernels ------------------------------------------------

__global__ void k_raw_llr_i64(const long long *__restrict__ rank, const long long *__restrict__ lcp,
                              long long n, long long *__restrict__ out, unsigned *err) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == 0) {
        out[0] = 0;
        return;
    }
    long long r = rank[i];
    if (r < 1 || r > n) {
        atomicOr(err, 1u);
        out[i] = 0;
        return;
    }
    long long a = lcp[r], b = lcp[r + 1];
    out[i] = a > b ? a : b;
}

__global__ void k_flags_i64(const long long *__restrict__ raw, long long n, long long *__restrict__ out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == 0) {
        out[0] = 0;
        return;
    }
    long long len = raw[i];
    out[i] = (len > 0 && len >= raw[i - 1]) ? 1 : 0;
}

// Inclusive scan of `count` int64 values (single pass, look-back).
constexpr int kScanIPT = 8;
__global__ void __launch_bounds__(kNT) k_scan_i64(const long long *__restrict__ in, long long count,
                                                  long long *__restrict__ out, unsigned *counter,
                                                  u64 *status, long long tiles) {
    __shared__ unsigned s_tile;
    __shared__ u64 s_warp[kNT / 32];
    __shared__ u64 s_base;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long i0 = tile * (kNT * kScanIPT) + (long long)threadIdx.x * kScanIPT;
    long long v[kScanIPT];
    u64 s = 0;
#pragma unroll
    for (int j = 0; j < kScanIPT; ++j) {
        v[j] = (i0 + j < count) ? in[i0 + j] : 0;
        s += (u64)v[j];
    }
    u64 excl;
    u64 total = block_exclusive_sum64<kNT>(s, excl, s_warp);
    if (threadIdx.x < 32) {
        u64 base = lookback_warp_wide(status, tiles, tile, total);
        if (threadIdx.x == 0) s_base = base;
    }
    __syncthreads();
    u64 acc = s_base + excl;  // two's-complement wraparound, like np.cumsum on int64
#pragma unroll
    for (int j = 0; j < kScanIPT; ++j) {
        acc += (u64)v[j];
        if (i0 + j < count) out[i0 + j] = (long long)acc;
    }
}

__global__ void k_scatter_i64(const long long *__restrict__ raw, const long long *__restrict__ flags,
                              const long long *__restrict__ ps, long long n, long long m,
                              long long *__restrict__ starts, long long *__restrict__ lengths,
                              unsigned *err) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1;
    if (i > n) return;
    if (flags[i] == 1) {
        long long t = ps[i] - 1;
        if (t < 0 || t >= m) {
            atomicOr(err, 1u);
            return;
        }
        starts[t] = i;
        lengths[t] = raw[i];
    }
}

__global__ void k_narrow(const long long *__restrict__ in, unsigned *__restrict__ out, long long count,
                         long long lo, long long hi, long long add, unsigned *err) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= count) return;
    long long x = in[i];
    if (x < lo || x > hi) {
        atomicOr(err, 1u);
        x = lo;
    }
    out[i] = (unsigned)(x + add);
}

__global__ void k_widen(const unsigned *__restrict__ in, long long *__restrict__ out, long long count,
                        long long add) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= count) return;
    out[i] = (long long)in[i] + add;
}

__global__ void k_add_i64(long long *__restrict__ a, long long count, long long add) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < count) a[i] += add;
}

__global__ void k_split_llrc(const uint2 *__restrict__ llrc, long long m, long long *__restrict__ starts,
                             long long *__restrict__ lengths) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= m) return;
    uint2 e = llrc[t];
    starts[t] = e.x;
    lengths[t] = e.y;
}

__global__ void k_join_llrc(const long long *__restrict__ starts, const long long *__restrict__ lengths,
                            long long m, long long n, uint2 *__restrict__ llrc, unsigned *err) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= m) return;
    long long s = starts[t], l = lengths[t];
    // CompactLlr invariant (llr.py:31-37): strictly increasing
    // starts and ends, entries inside [1, n].
    bool ok = s >= 1 && l >= 1 && s + l - 1 <= n;
    if (ok && t > 0) {
        long long ps = starts[t - 1], pl = lengths[t - 1];
        ok = ps < s && ps + pl < s + l;
    }
    if (!ok) atomicOr(err, 1u);
    llrc[t] = make_uint2((unsigned)s, (unsigned)l);
}

// LLR end-monotonicity (Lemma 2 / test_llr.py:45-50): raw[i] <= raw[i+1] + 1.
// The windowed raw-path scan relies on it; the reference walk assumes it too.
__global__ void k_check_raw(const unsigned *__restrict__ raw, long long n, unsigned *err) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1;
    if (i >= n) return;
    if ((long long)raw[i] > (long long)raw[i + 1] + 1) atomicOr(err, 1u);
}

__global__ void k_check_llrc(const uint2 *__restrict__ e, long long m, long long n, unsigned *err) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= m) return;
    uint2 x = e[t];
    bool ok = x.x >= 1 && x.y >= 1 && (long long)x.x + x.y - 1 <= n;
    if (ok && t > 0) {
        uint2 p = e[t - 1];
        ok = p.x < x.x && (long long)p.x + p.y < (long long)x.x + x.y;
    }
    if (!ok) atomicOr(err, 1u);
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

long long compact_from_raw(rs_ctx *c, long long n) {
    long long tiles = (n + 1 + kTile - 1) / kTile;
    // B_RAW is allocated by the producer with >= tiles*kTile + 8 slots.
    const unsigned *raw = (const unsigned *)c->bufs[B_RAW].p;
    uint2 *llrc = (uint2 *)buf(c, B_LLRC, sizeof(uint2) * (size_t)(n + 8));
    unsigned long long *m_dev = (unsigned long long *)buf(c, B_SMALL, 4096);
    Scratch s = scratch(c, tiles);
    RS_LAUNCH_B(c, 4.0 * (n + 1), k_compact_raw, (unsigned)tiles, kNT, 0, raw, n, llrc, m_dev, s.counter,
                s.status, tiles);
    unsigned long long m = 0;
    fetch_small(c, &m, m_dev, sizeof(m));
    add_bytes_last(c, 8.0 * (double)m);
    // zero the two pad entries after the last one (TMA staging reads them)
    RS_CUDA(cudaMemsetAsync(llrc + m, 0, sizeof(uint2) * 4, c->stream));
    return (long long)m;
}

size_t raw_slots(long long n) {
    long long tiles = (n + 1 + kTile - 1) / kTile;
    return (size_t)(tiles * kTile + 16);
}

// raw slots [first, last] only (a position shard and its left halo)
void raw_from_rank_lcp_range(rs_ctx *c, long long n, long long first, long long last) {
    unsigned *raw = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots(n));
    const long long cnt = last - first + 1;
    if (cnt <= 0) return;
    RS_LAUNCH_B(c, 16.0 * cnt, k_raw_from_isa_lcp, grid_for((cnt + 7) / 8, 256), 256, 0,
                (const unsigned *)c->bufs[B_ISA].p, (const unsigned *)c->bufs[B_LCP].p, last, raw, first);
}

__global__ void k_max_u32(const unsigned *__restrict__ a, long long count, unsigned *out) {
    unsigned v = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
        v = max(v, a[i]);
    v = __reduce_max_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// max over the resident SA-order LCP (bounds every raw LLR value: a shard's halo)
long long max_lcp(rs_ctx *c, long long n) {
    unsigned *o = (unsigned *)((char *)buf(c, B_SMALL, 4096) + 320);
    RS_CUDA(cudaMemsetAsync(o, 0, sizeof(unsigned), c->stream));
    if (n > 0) RS_LAUNCH(c, k_max_u32, 4 * c->sm_count, 256, 0, (const unsigned *)c->bufs[B_LCP].p, n + 1, o);
    unsigned h = 0;
    fetch_small(c, &h, o, sizeof(h));
    return (long long)h;
}

void raw_from_rank_lcp(rs_ctx *c, long long n) {
    unsigned *raw = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots(n));
    RS_LAUNCH_B(c, 16.0 * n, k_raw_from_isa_lcp, grid_for((n + 8) / 8, 256), 256, 0, (const unsigned *)c->bufs[B_ISA].p,
              (const unsigned *)c->bufs[B_LCP].p, n, raw);
}

static unsigned *err_flag(rs_ctx *c) {
    unsigned *e = (unsigned *)((char *)buf(c, B_SMALL, 4096) + 64);
    RS_CUDA(cudaMemsetAsync(e, 0, sizeof(unsigned), c->stream));
    return e;
}

static void check_err_flag(rs_ctx *c, unsigned *e, int code, const std::string &what) {
    unsigned h = 0;
    fetch_small(c, &h, e, sizeof(h));
    if (h) fail(code, what);
}

void narrow_i64_to_u32(rs_ctx *c, const long long *d_in, unsigned *d_out, long long count,
                       long long lo, long long hi, long long add, const char *what) {
    if (count <= 0) return;
    unsigned *e = err_flag(c);
    RS_LAUNCH(c, k_narrow, grid_for(count, 256), 256, 0, d_in, d_out, count, lo, hi, add, e);
    check_err_flag(c, e, RS_EINVAL, std::string(what) + " has values out of range");
}

void widen_u32_to_i64(rs_ctx *c, const unsigned *d_in, long long *d_out, long long count, long long add) {
    if (count <= 0) return;
    RS_LAUNCH(c, k_widen, grid_for(count, 256), 256, 0, d_in, d_out, count, add);
}

void add_i64(rs_ctx *c, long long *d, long long count, long long add) {
    if (count <= 0 || add == 0) return;
    RS_LAUNCH(c, k_add_i64, grid_for(count, 256), 256, 0, d, count, add);
}

void split_llrc(rs_ctx *c, long long m, long long *d_starts, long long *d_lengths) {
    if (m <= 0) return;
    RS_LAUNCH(c, k_split_llrc, grid_for(m, 256), 256, 0, (const uint2 *)c->bufs[B_LLRC].p, m, d_starts,
              d_lengths);
}

void join_llrc(rs_ctx *c, const long long *d_starts, const long long *d_lengths, long long m,
               long long n) {
    uint2 *llrc = (uint2 *)buf(c, B_LLRC, sizeof(uint2) * (size_t)(m + 8));
    RS_CUDA(cudaMemsetAsync(llrc + m, 0, sizeof(uint2) * 4, c->stream));
    if (m <= 0) return;
    unsigned *e = err_flag(c);
    RS_LAUNCH(c, k_join_llrc, grid_for(m, 256), 256, 0, d_starts, d_lengths, m, n, llrc, e);
    check_err_flag(c, e, RS_EINVAL,
                   "compact LLR arrays must be 1-based, inside the text, with strictly increasing "
                   "starts and ends");
}

void check_raw(rs_ctx *c, long long n) {
    if (n < 2) return;
    unsigned *e = err_flag(c);
    RS_LAUNCH(c, k_check_raw, grid_for(n, 256), 256, 0, (const unsigned *)c->bufs[B_RAW].p, n, e);
    check_err_flag(c, e, RS_EINVAL,
                   "raw LLR array violates raw[i] <= raw[i+1] + 1 (not an LLR array of any text)");
}

void validate_llrc(rs_ctx *c, long long m, long long n) {
    if (m <= 0) return;
    unsigned *e = err_flag(c);
    RS_LAUNCH(c, k_check_llrc, grid_for(m, 256), 256, 0, (const uint2 *)c->bufs[B_LLRC].p, m, n, e);
    check_err_flag(c, e, RS_EINVAL,
                   "compact LLR entries must be 1-based, inside the text, with strictly increasing "
                   "starts and ends");
}

void raw_llr_i64(rs_ctx *c, const long long *d_rank, const long long *d_lcp, long long n,
                 long long *d_out) {
    unsigned *e = err_flag(c);
    RS_LAUNCH(c, k_raw_llr_i64, grid_for(n + 1, 256), 256, 0, d_rank, d_lcp, n, d_out, e);
    check_err_flag(c, e, RS_EINVAL, "rank values must lie in 1..n");
}

void flags_i64(rs_ctx *c, const long long *d_raw, long long n, long long *d_out) {
    RS_LAUNCH(c, k_flags_i64, grid_for(n + 1, 256), 256, 0, d_raw, n, d_out);
}

void scan_i64(rs_ctx *c, const long long *d_in, long long count, long long *d_out) {
    if (count <= 0) return;
    long long tiles = (count + kNT * kScanIPT - 1) / (kNT * kScanIPT);
    Scratch s = scratch(c, 3 * tiles);
    RS_LAUNCH(c, k_scan_i64, (unsigned)tiles, kNT, 0, d_in, count, d_out, s.counter, s.status, tiles);
}

void scatter_i64(rs_ctx *c, const long long *d_raw, const long long *d_flags, const long long *d_ps,
                 long long n, long long m, long long *d_starts, long long *d_lengths) {
    if (n <= 0) return;
    unsigned *e = err_flag(c);
    RS_LAUNCH(c, k_scatter_i64, grid_for(n, 256), 256, 0, d_raw, d_flags, d_ps, n, m, d_starts,
              d_lengths, e);
    check_err_flag(c, e, RS_EINVAL, "prefix sums do not match the flags");
}

}  // namespace rsb
