// host_io.cu -- host <-> device transfers of the reference's int64 arrays.
//
// The API hands back (and takes) int64 numpy arrays in the reference layout
// (query.py:130-168, suffixes.py:20-28): 8 bytes per value although every
// value fits 32 bits (positions, lengths and starts are < 2^31; CSR offsets
// are nondecreasing with small steps).  Measured on the B200 box
// (tools/exp_d2h.py): a plain cudaMemcpy into a fresh pageable numpy array
// runs at 4.1 GB/s, into pinned memory at 51 GB/s, and 16 host threads write
// touched memory at ~90 GB/s (fresh pages ~40 GB/s).  So large transfers go
// through a two-slot pipeline with 4 bytes per value on the wire:
//   D2H: narrow kernel (int64 -> u32 word) into a device ring slot -> DMA into
//        a pinned ring slot -> host threads widen into the caller's array,
//        while the next slot's DMA runs;
//   H2D: host threads narrow (range-checked) into a pinned slot -> DMA -> the
//        caller's device u32 array (or, for bytes, a plain staged copy).
// Offsets travel as their low 32 bits; each chunk's first value is fetched
// in full beforehand and the host adds the (mod 2^32) differences, exact as
// long as a chunk's span stays below 2^32 (checked; else plain int64 DMA).
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace rsb {

// host_widen.cpp: out[j] = f(w[j]) + add, streaming stores
void widen_words(const unsigned *w, long long *out, long long x, long long y, int mode, unsigned w0,
                 long long add);
void widen_bytes(const unsigned char *w, long long *out, long long x, long long y);
void prefix_bytes(const unsigned char *w, long long *out, long long x, long long y, long long start, bool is_signed);
void leftmost_pairs(const unsigned char *w, long long *starts, long long *lengths, long long x, long long y,
                    long long pos_x);
void decode_block(const unsigned char *w, int width, int mode, long long *out, long long count, long long start);
bool narrow_words(const long long *in, unsigned *w, long long x, long long y, long long lo, long long hi,
                  long long add);
int narrow_bytes(const long long *in, unsigned char *b, long long x, long long y, long long lo, long long hi);
void decode_left_block(const unsigned char *w, int width, long long count, long long pos0, long long *starts,
                       long long *lengths);

namespace {

void h2d(rs_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes) RS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += (long long)bytes;
}
void d2h(rs_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes) RS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += (long long)bytes;
}

// ---- host thread pool: run(f) calls f(t, T) on T threads and waits ----------
class Pool {
  public:
    static Pool &get() {
        static Pool p;
        return p;
    }
    int size() const { return (int)workers_.size() + 1; }
    void run(const std::function<void(int, int)> &f) {
        const int T = size();
        if (T == 1) {
            f(0, 1);
            return;
        }
        // one job at a time: contexts of different devices may transfer from
        // different host threads concurrently
        std::lock_guard<std::mutex> one(run_m_);
        {
            std::unique_lock<std::mutex> lk(m_);
            job_ = &f;
            pending_ = T - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0, T);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    Pool() {
        // threads we may actually run on (cgroup / taskset), not the host's core count
        cpu_set_t set;
        int T = sched_getaffinity(0, sizeof(set), &set) == 0 ? CPU_COUNT(&set)
                                                             : (int)std::thread::hardware_concurrency();
        if (const char *e = std::getenv("RS_HOST_THREADS")) T = std::atoi(e);
        T = std::max(1, std::min(T, 64));
        for (int i = 1; i < T; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    void loop(int id) {
        unsigned long long seen = 0;
        for (;;) {
            const std::function<void(int, int)> *f;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                f = job_;
            }
            (*f)(id, (int)workers_.size() + 1);
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::mutex run_m_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int, int)> *job_ = nullptr;
    int pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

inline void split(long long count, int t, int T, long long &a, long long &b) {
    const long long per = (count + T - 1) / T;
    a = std::min(count, per * t);
    b = std::min(count, a + per);
}

#ifndef RS_XFER_CHUNK
#define RS_XFER_CHUNK (16ll << 20)
#endif
constexpr long long kChunk = RS_XFER_CHUNK;     // values per pipeline slot (64 MiB of 32-bit words)
constexpr size_t kMinStaged = 8u << 20;         // smaller arrays: one plain copy

__global__ void k_narrow_words(const long long *__restrict__ src, unsigned *__restrict__ dst, long long count) {
    long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
    if (i + 3 < count) {
        const longlong2 a = *reinterpret_cast<const longlong2 *>(src + i);
        const longlong2 b = *reinterpret_cast<const longlong2 *>(src + i + 2);
        *reinterpret_cast<uint4 *>(dst + i) = make_uint4((unsigned)a.x, (unsigned)a.y, (unsigned)b.x, (unsigned)b.y);
    } else {
        for (; i < count; ++i) dst[i] = (unsigned)src[i];
    }
}

// every chunk's first and last value (offsets reconstruction / span check)
__global__ void k_chunk_ends(const long long *__restrict__ src, long long count, long long chunk, long long nch,
                             long long *__restrict__ out) {
    long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= nch) return;
    long long a = c * chunk, b = (a + chunk < count ? a + chunk : count) - 1;
    out[2 * c] = src[a];
    out[2 * c + 1] = src[b];
}

struct Stage {
    void **host;
    cudaEvent_t *ev;
};

// the context's two pinned slots + events (allocated on first use, freed by
// rs_destroy); waits until neither slot is still being copied
Stage stage(rs_ctx *c) {
    for (int i = 0; i < 2; ++i) {
        if (!c->xfer_host[i]) RS_CUDA(cudaHostAlloc(&c->xfer_host[i], 4 * (size_t)kChunk, cudaHostAllocDefault));
        if (!c->xfer_ev[i]) RS_CUDA(cudaEventCreateWithFlags(&c->xfer_ev[i], cudaEventDisableTiming));
        RS_CUDA(cudaEventSynchronize(c->xfer_ev[i]));
    }
    return Stage{c->xfer_host, c->xfer_ev};
}

}  // namespace

// Two-slot D2H pipeline: issue(a, len, slot) enqueues whatever produces the
// chunk's 32-bit words on the stream and returns their device address; the
// words are copied into the pinned slot, and widen(words, out, x, y, chunk)
// runs on the host threads over [x, y) of the chunk while the next chunk's
// copy is in flight.
template <typename Issue, typename Widen>
void pipeline_out(rs_ctx *c, long long count, Issue issue, Widen widen, long long *dst) {
    const long long nch = (count + kChunk - 1) / kChunk;
    Stage s = stage(c);
    auto start = [&](long long i) {
        const long long a = i * kChunk, len = std::min(kChunk, count - a);
        const void *d = issue(a, len, (int)(i & 1));
        RS_CUDA(cudaMemcpyAsync(s.host[i & 1], d, 4 * (size_t)len, cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += 4 * len;
        RS_CUDA(cudaEventRecord(s.ev[i & 1], c->stream));
    };
    start(0);
    if (nch > 1) start(1);
    Pool &pool = Pool::get();
    for (long long i = 0; i < nch; ++i) {
        RS_CUDA(cudaEventSynchronize(s.ev[i & 1]));
        const long long a = i * kChunk, len = std::min(kChunk, count - a);
        const unsigned *w = (const unsigned *)s.host[i & 1];
        long long *out = dst + a;
        pool.run([&](int t, int T) {
            long long x, y;
            split(len, t, T, x, y);
            if (y > x) widen(w, out, x, y, i);
        });
        if (i + 2 < nch) start(i + 2);
    }
}

static void fetch_i64_staged(rs_ctx *c, long long *dst, const long long *dsrc, long long count, int kind);

static bool page_locked(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// D2H of `count` int64 values.  kind: 0 = values in [0, 2^32), 1 = values in
// [-1, 2^31) (sign-extended), 2 = nondecreasing offsets.
// A page-locked destination lets both limits work at once: the leading part
// of the array is DMA'd as int64 straight into it on a side stream (PCIe
// bound) while the rest goes through the wire-word pipeline (bound by the
// host's memory bandwidth).  RS_DIRECT_FRAC (default 0: with streaming stores the pipeline alone is as fast, tools/exp_fetch.py) sets the split.
void fetch_i64(rs_ctx *c, long long *dst, const long long *dsrc, long long count, int kind) {
    if (count <= 0) return;
    if ((size_t)count * 8 < kMinStaged) {
        d2h(c, dst, dsrc, 8 * (size_t)count);
        RS_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    double frac = 0.0;
    if (const char *e = std::getenv("RS_DIRECT_FRAC")) frac = std::atof(e);
    long long direct = 0;
    if (count >= 4 * kChunk && frac > 0 && page_locked(dst))
        direct = std::min(count, (long long)(frac * (double)count) & ~1023ll);
    if (direct > 0) {
        if (!c->xfer_side) RS_CUDA(cudaStreamCreateWithFlags(&c->xfer_side, cudaStreamNonBlocking));
        if (!c->xfer_side_ev) RS_CUDA(cudaEventCreateWithFlags(&c->xfer_side_ev, cudaEventDisableTiming));
        RS_CUDA(cudaEventRecord(c->xfer_side_ev, c->stream));  // after the producing kernels
        RS_CUDA(cudaStreamWaitEvent(c->xfer_side, c->xfer_side_ev, 0));
        RS_CUDA(cudaMemcpyAsync(dst, dsrc, 8 * (size_t)direct, cudaMemcpyDeviceToHost, c->xfer_side));
        c->d2h_bytes += 8 * direct;
    }
    if (count > direct) fetch_i64_staged(c, dst + direct, dsrc + direct, count - direct, kind);
    if (direct > 0) RS_CUDA(cudaStreamSynchronize(c->xfer_side));
}

static void fetch_i64_staged(rs_ctx *c, long long *dst, const long long *dsrc, long long count, int kind) {
    if ((size_t)count * 8 < kMinStaged) {
        d2h(c, dst, dsrc, 8 * (size_t)count);
        RS_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    const long long nch = (count + kChunk - 1) / kChunk;
    std::vector<long long> ends;
    if (kind == 2) {
        long long *d_ends = (long long *)buf(c, B_XFER_ENDS, 16 * (size_t)nch);
        RS_LAUNCH(c, k_chunk_ends, grid_for(nch, 128), 128, 0, dsrc, count, kChunk, nch, d_ends);
        ends.resize(2 * nch);
        d2h(c, ends.data(), d_ends, 16 * (size_t)nch);
        RS_CUDA(cudaStreamSynchronize(c->stream));
        for (long long i = 0; i < nch; ++i)
            if ((unsigned long long)(ends[2 * i + 1] - ends[2 * i]) >= (1ull << 32)) {  // span too wide
                d2h(c, dst, dsrc, 8 * (size_t)count);
                RS_CUDA(cudaStreamSynchronize(c->stream));
                return;
            }
    }
    unsigned *ring = (unsigned *)buf(c, B_XFER, 2 * 4 * (size_t)kChunk);
    const long long *ends_p = ends.data();
    pipeline_out(
        c, count,
        [&](long long a, long long len, int slot) {  // wire words of chunk [a, a + len) -> device slot
            unsigned *d = ring + slot * kChunk;
            RS_LAUNCH(c, k_narrow_words, grid_for((len + 3) / 4, 256), 256, 0, dsrc + a, d, len);
            return (const void *)d;
        },
        [&](const unsigned *w, long long *out, long long x, long long y, long long chunk) {
            if (kind == 2) widen_words(w, out, x, y, 2, w[0], ends_p[2 * chunk]);
            else widen_words(w, out, x, y, kind, 0u, 0ll);
        },
        dst);
}

// D2H of a device u32 array as int64 values + add (structures, raw LLR):
// the 4-byte words go on the wire as they are.
void fetch_u32_as_i64(rs_ctx *c, long long *dst, const unsigned *dsrc, long long count, long long add) {
    if (count <= 0) return;
    pipeline_out(
        c, count, [&](long long a, long long, int) { return (const void *)(dsrc + a); },
        [&](const unsigned *w, long long *out, long long x, long long y, long long) {
            widen_words(w, out, x, y, 0, 0u, add);
        },
        dst);
}

// ---- byte wire for the all-ties CSR --------------------------------------
//
// With short repeats (every length, tie count and start-to-start step below
// 2^7 .. 2^8 -- i.i.d. DNA has max LLR ~ 28) the three CSR arrays travel as ONE
// byte per value: lengths as u8, offsets as u8 tie counts (offsets[k+1] -
// offsets[k]), tie starts as i8 differences of consecutive starts.  The host
// rebuilds offsets and starts with running sums, restarting every kSample
// values from an exact int64 sample taken on the device.  4.2 GB of 32-bit
// wire words become 1.05 GB on C3, and the host's memory traffic (DMA in,
// read, int64 out) drops from ~16.8 GB to ~10.5 GB.  If any value does not fit
// the caller falls back to the 32-bit wire.
constexpr long long kSample = 1ll << 16;

__global__ void k_wire_len_cnt(const long long *__restrict__ len, const long long *__restrict__ off, long long count,
                               unsigned char *__restrict__ len8, unsigned char *__restrict__ cnt8,
                               long long *__restrict__ osamp, unsigned *__restrict__ bad) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    bool b = false;
    if (k < count) {
        const long long L = len[k], o = off[k], C = off[k + 1] - o;
        b = (unsigned long long)L > 255ull || (unsigned long long)C > 255ull;
        len8[k] = (unsigned char)L;
        cnt8[k] = (unsigned char)C;
        if ((k & (kSample - 1)) == 0) osamp[k / kSample] = o;
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

__global__ void k_wire_flat(const long long *__restrict__ flat, long long T, unsigned char *__restrict__ d8,
                            long long *__restrict__ fsamp, unsigned *__restrict__ bad) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    bool b = false;
    if (t < T) {
        const long long v = flat[t];
        long long d = 0;
        if (t > 0) {
            d = v - flat[t - 1];
            b = d < -128 || d > 127;
        }
        d8[t] = (unsigned char)(signed char)d;
        if ((t & (kSample - 1)) == 0) fsamp[t / kSample] = v;
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// leftmost answers as byte pairs: w[2j] = length, w[2j+1] = position - start
// (slot j answers position pos0 + j; a zero length means start -1)
__global__ void k_wire_leftmost(const long long *__restrict__ starts, const long long *__restrict__ lengths,
                                long long count, long long pos0, unsigned char *__restrict__ w,
                                unsigned *__restrict__ bad) {
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    bool b = false;
    if (j < count) {
        const long long L = lengths[j], d = L ? pos0 + j - starts[j] : 0;
        b = (unsigned long long)L > 255ull || (unsigned long long)d > 255ull;
        w[2 * j] = (unsigned char)L;
        w[2 * j + 1] = (unsigned char)d;
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// D2H of `count` wire bytes through the two pinned slots; decode(w, a, x, y)
// rebuilds values [a + x, a + y) from the slot holding bytes [a, a + len),
// x a multiple of kSample, on the host threads while the next DMA runs.
template <typename Decode>
static void pipeline_bytes(rs_ctx *c, const unsigned char *dsrc, long long count, Decode decode) {
    const long long ch = 4 * kChunk;  // bytes per slot (a multiple of kSample)
    const long long nch = (count + ch - 1) / ch;
    Stage s = stage(c);
    auto start = [&](long long i) {
        const long long a = i * ch, len = std::min(ch, count - a);
        RS_CUDA(cudaMemcpyAsync(s.host[i & 1], dsrc + a, (size_t)len, cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += len;
        RS_CUDA(cudaEventRecord(s.ev[i & 1], c->stream));
    };
    start(0);
    if (nch > 1) start(1);
    Pool &pool = Pool::get();
    for (long long i = 0; i < nch; ++i) {
        RS_CUDA(cudaEventSynchronize(s.ev[i & 1]));
        const long long a = i * ch, len = std::min(ch, count - a);
        const unsigned char *w = (const unsigned char *)s.host[i & 1];
        const long long blocks = (len + kSample - 1) / kSample;
        pool.run([&](int t, int T) {
            long long bx, by;
            split(blocks, t, T, bx, by);
            const long long x = bx * kSample, y = std::min(len, by * kSample);
            if (y > x) decode(w, a, x, y);
        });
        if (i + 2 < nch) start(i + 2);
    }
}

// CSR answers (lengths[L], offsets[L + 1], flat[T]) from device int64 arrays
// over the byte wire; false (nothing written) when a value does not fit.
bool fetch_csr_bytes(rs_ctx *c, const long long *d_len, const long long *d_off, const long long *d_flat,
                     long long L, long long T, long long *lengths, long long *offsets, long long *flat) {
    if (L < (4ll << 20) || std::getenv("RS_WORD_WIRE")) return false;
    const long long ns = (L + kSample - 1) / kSample, ts = (T + kSample - 1) / kSample;
    unsigned char *w = (unsigned char *)buf(c, B_WIRE, (size_t)(2 * L + T) + 16 * (size_t)(ns + ts + 2) + 64);
    unsigned char *len8 = w, *cnt8 = w + L, *d8 = w + 2 * L;
    long long *osamp = (long long *)(((uintptr_t)(d8 + T) + 15) & ~(uintptr_t)15);
    long long *fsamp = osamp + ns;
    unsigned *bad = (unsigned *)(fsamp + ts + 1);
    RS_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), c->stream));
    RS_LAUNCH_B(c, 25.0 * (double)L, k_wire_len_cnt, grid_for(L, 256), 256, 0, d_len, d_off, L, len8, cnt8, osamp,
                bad);
    if (T > 0) RS_LAUNCH_B(c, 9.0 * (double)T, k_wire_flat, grid_for(T, 256), 256, 0, d_flat, T, d8, fsamp, bad);
    std::vector<long long> samp((size_t)(ns + ts));
    unsigned hbad = 0;
    d2h(c, &hbad, bad, sizeof(hbad));
    d2h(c, samp.data(), osamp, sizeof(long long) * (size_t)(ns + ts));
    RS_CUDA(cudaStreamSynchronize(c->stream));
    if (hbad) return false;
    const long long *os = samp.data(), *fs = samp.data() + ns;
    pipeline_bytes(c, len8, L, [&](const unsigned char *b, long long a, long long x, long long y) {
        widen_bytes(b, lengths + a, x, y);
    });
    offsets[0] = os[0];
    pipeline_bytes(c, cnt8, L, [&](const unsigned char *b, long long a, long long x, long long y) {
        prefix_bytes(b, offsets + 1 + a, x, y, os[(a + x) / kSample], false);
    });
    if (T > 0)
        pipeline_bytes(c, d8, T, [&](const unsigned char *b, long long a, long long x, long long y) {
            prefix_bytes(b, flat + a, x, y, fs[(a + x) / kSample] - (long long)(signed char)b[x], true);
        });
    return true;
}

// ---- mixed-width wire: 1, 2 or 4 bytes per value, chosen per 2^16 block ----
//
// When some value does not fit a byte (long repeats: C5's lengths reach
// 129453), the CSR still crosses PCIe as narrow as each block of kSample
// values allows instead of falling back to 4 bytes everywhere: a block's
// lengths, tie counts and start steps each take the width of that block's
// largest value (steps signed).  Blocks are laid out back to back; the host
// decodes each from its int64 sample.
__device__ __forceinline__ unsigned char width_of(unsigned long long maxv) {
    return maxv <= 0xffull ? 1 : (maxv <= 0xffffull ? 2 : 4);
}
__device__ __forceinline__ unsigned char swidth_of(long long lo, long long hi) {
    return (lo >= -128 && hi <= 127) ? 1 : ((lo >= -32768 && hi <= 32767) ? 2 : 4);
}
__device__ __forceinline__ void put_w(unsigned char *p, int w, unsigned long long v) {
    if (w == 1) *p = (unsigned char)v;
    else if (w == 2) *reinterpret_cast<unsigned short *>(p) = (unsigned short)v;
    else *reinterpret_cast<unsigned *>(p) = (unsigned)v;
}

// one CTA per block of positions: widths of its lengths and tie counts + sample
__global__ void k_widths_pos(const long long *__restrict__ len, const long long *__restrict__ off, long long L,
                             unsigned char *__restrict__ wl, unsigned char *__restrict__ wc,
                             long long *__restrict__ osamp) {
    const long long b = blockIdx.x, k0 = b * kSample, k1 = k0 + kSample < L ? k0 + kSample : L;
    unsigned long long ml = 0, mc = 0;
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const unsigned long long l = (unsigned long long)len[k], cn = (unsigned long long)(off[k + 1] - off[k]);
        ml = l > ml ? l : ml;
        mc = cn > mc ? cn : mc;
    }
    __shared__ unsigned long long s_l[8], s_c[8];
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, ml, o), c2 = __shfl_xor_sync(0xffffffffu, mc, o);
        ml = a > ml ? a : ml;
        mc = c2 > mc ? c2 : mc;
    }
    if ((threadIdx.x & 31) == 0) {
        s_l[threadIdx.x >> 5] = ml;
        s_c[threadIdx.x >> 5] = mc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            ml = s_l[i] > ml ? s_l[i] : ml;
            mc = s_c[i] > mc ? s_c[i] : mc;
        }
        wl[b] = width_of(ml);
        wc[b] = width_of(mc);
        osamp[b] = off[k0];
    }
}

// one CTA per block of ties: width of its start steps (the block's first step
// is not sent: the block starts from its sample) + sample
__global__ void k_widths_flat(const long long *__restrict__ flat, long long T, unsigned char *__restrict__ wf,
                              long long *__restrict__ fsamp) {
    const long long b = blockIdx.x, t0 = b * kSample, t1 = t0 + kSample < T ? t0 + kSample : T;
    long long lo = 0, hi = 0;
    for (long long t = t0 + 1 + threadIdx.x; t < t1; t += blockDim.x) {
        const long long d = flat[t] - flat[t - 1];
        lo = d < lo ? d : lo;
        hi = d > hi ? d : hi;
    }
    __shared__ long long s_lo[8], s_hi[8];
    for (int o = 16; o; o >>= 1) {
        const long long a = __shfl_xor_sync(0xffffffffu, lo, o), c2 = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = c2 > hi ? c2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            lo = s_lo[i] < lo ? s_lo[i] : lo;
            hi = s_hi[i] > hi ? s_hi[i] : hi;
        }
        wf[b] = swidth_of(lo, hi);
        fsamp[b] = flat[t0];
    }
}

__global__ void k_pack_pos(const long long *__restrict__ len, const long long *__restrict__ off, long long L,
                           const unsigned char *__restrict__ wl, const unsigned char *__restrict__ wc,
                           const long long *__restrict__ lbase, const long long *__restrict__ cbase,
                           unsigned char *__restrict__ lw, unsigned char *__restrict__ cw) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= L) return;
    const long long b = k / kSample, i = k - b * kSample;
    const int a = wl[b], c2 = wc[b];
    put_w(lw + lbase[b] + i * a, a, (unsigned long long)len[k]);
    put_w(cw + cbase[b] + i * c2, c2, (unsigned long long)(off[k + 1] - off[k]));
}

__global__ void k_pack_flat(const long long *__restrict__ flat, long long T, const unsigned char *__restrict__ wf,
                            const long long *__restrict__ fbase, unsigned char *__restrict__ fw) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const long long b = t / kSample, i = t - b * kSample;
    const int w = wf[b];
    const long long d = i ? flat[t] - flat[t - 1] : 0;
    put_w(fw + fbase[b] + i * w, w, (unsigned long long)d);
}

// D2H of a block-structured wire array (block b: bytes [base[b], base[b+1]),
// `values` of them) through the pinned slots; decode(b, bytes) on the host threads.
template <typename Decode>
static void pipeline_blocks(rs_ctx *c, const unsigned char *dsrc, const std::vector<long long> &base, Decode decode) {
    const long long nb = (long long)base.size() - 1, cap = 4 * kChunk;
    std::vector<long long> cb{0};  // chunk boundaries (block indices)
    for (long long b = 0; b < nb; ++b)
        if (base[b + 1] - base[cb.back()] > cap) cb.push_back(b);
    cb.push_back(nb);
    const long long nch = (long long)cb.size() - 1;
    Stage s = stage(c);
    auto start = [&](long long i) {
        const long long a = base[cb[i]], len = base[cb[i + 1]] - a;
        RS_CUDA(cudaMemcpyAsync(s.host[i & 1], dsrc + a, (size_t)len, cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += len;
        RS_CUDA(cudaEventRecord(s.ev[i & 1], c->stream));
    };
    start(0);
    if (nch > 1) start(1);
    Pool &pool = Pool::get();
    for (long long i = 0; i < nch; ++i) {
        RS_CUDA(cudaEventSynchronize(s.ev[i & 1]));
        const unsigned char *w = (const unsigned char *)s.host[i & 1];
        const long long b0 = cb[i], b1 = cb[i + 1], a = base[b0];
        pool.run([&](int t, int T) {
            long long x, y;
            split(b1 - b0, t, T, x, y);
            for (long long b = b0 + x; b < b0 + y; ++b) decode(b, w + (base[b] - a));
        });
        if (i + 2 < nch) start(i + 2);
    }
}

bool fetch_csr_mixed(rs_ctx *c, const long long *d_len, const long long *d_off, const long long *d_flat,
                     long long L, long long T, long long *lengths, long long *offsets, long long *flat) {
    if (L < (4ll << 20) || std::getenv("RS_WORD_WIRE")) return false;
    const long long nb = (L + kSample - 1) / kSample, tb = (T + kSample - 1) / kSample;
    // metadata: widths (3 arrays), samples, block byte bases (device copies)
    const size_t meta = 16 * (size_t)(nb + tb + 2) + 8 * (size_t)(2 * (nb + 1) + tb + 1) + 256;
    unsigned char *m = (unsigned char *)buf(c, B_XFER_ENDS, meta);
    long long *osamp = (long long *)m, *fsamp = osamp + nb;
    long long *lbase = fsamp + tb + 1, *cbase = lbase + nb + 1, *fbase = cbase + nb + 1;
    unsigned char *wl = (unsigned char *)(fbase + tb + 1), *wc = wl + nb, *wf = wc + nb;
    RS_LAUNCH(c, k_widths_pos, (unsigned)nb, 256, 0, d_len, d_off, L, wl, wc, osamp);
    if (T > 0) RS_LAUNCH(c, k_widths_flat, (unsigned)tb, 256, 0, d_flat, T, wf, fsamp);
    std::vector<unsigned char> w((size_t)(2 * nb + tb));
    std::vector<long long> samp((size_t)(nb + tb));
    d2h(c, w.data(), wl, w.size());
    d2h(c, samp.data(), osamp, sizeof(long long) * samp.size());
    RS_CUDA(cudaStreamSynchronize(c->stream));
    const unsigned char *hwl = w.data(), *hwc = hwl + nb, *hwf = hwc + nb;
    std::vector<long long> lb(nb + 1, 0), cbv(nb + 1, 0), fb(tb + 1, 0);
    for (long long b = 0; b < nb; ++b) {
        const long long cntb = std::min(kSample, L - b * kSample);
        lb[b + 1] = lb[b] + cntb * hwl[b];
        cbv[b + 1] = cbv[b] + cntb * hwc[b];
    }
    for (long long b = 0; b < tb; ++b) fb[b + 1] = fb[b] + std::min(kSample, T - b * kSample) * hwf[b];
    h2d(c, lbase, lb.data(), sizeof(long long) * lb.size());
    h2d(c, cbase, cbv.data(), sizeof(long long) * cbv.size());
    if (T > 0) h2d(c, fbase, fb.data(), sizeof(long long) * fb.size());
    auto r16 = [](long long v) { return (v + 15) & ~15ll; };  // 2- and 4-byte stores stay aligned
    unsigned char *wire = (unsigned char *)buf(c, B_WIRE, (size_t)(r16(lb[nb]) + r16(cbv[nb]) + fb[tb]) + 64);
    unsigned char *lw = wire, *cw = wire + r16(lb[nb]), *fw = cw + r16(cbv[nb]);
    RS_LAUNCH_B(c, 24.0 * (double)L, k_pack_pos, grid_for(L, 256), 256, 0, d_len, d_off, L, wl, wc, lbase, cbase, lw,
                cw);
    if (T > 0) RS_LAUNCH_B(c, 16.0 * (double)T, k_pack_flat, grid_for(T, 256), 256, 0, d_flat, T, wf, fbase, fw);
    const long long *os = samp.data(), *fs = samp.data() + nb;
    pipeline_blocks(c, lw, lb, [&](long long b, const unsigned char *p) {
        decode_block(p, hwl[b], 0, lengths + b * kSample, std::min(kSample, L - b * kSample), 0);
    });
    offsets[0] = os[0];
    pipeline_blocks(c, cw, cbv, [&](long long b, const unsigned char *p) {
        decode_block(p, hwc[b], 1, offsets + 1 + b * kSample, std::min(kSample, L - b * kSample), os[b]);
    });
    if (T > 0)
        pipeline_blocks(c, fw, fb, [&](long long b, const unsigned char *p) {
            decode_block(p, hwf[b], 2, flat + b * kSample, std::min(kSample, T - b * kSample), fs[b]);
        });
    return true;
}

// Leftmost answers over the mixed-width wire: per block of 2^16 slots one
// width (that of the block's longest answer; position - start is smaller),
// the block's lengths then its position - start values.
__global__ void k_widths_left(const long long *__restrict__ len, long long L, unsigned char *__restrict__ wl) {
    const long long b = blockIdx.x, k0 = b * kSample, k1 = k0 + kSample < L ? k0 + kSample : L;
    unsigned long long ml = 0;
    for (long long k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const unsigned long long l = (unsigned long long)len[k];
        ml = l > ml ? l : ml;
    }
    __shared__ unsigned long long s_l[8];
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, ml, o);
        ml = a > ml ? a : ml;
    }
    if ((threadIdx.x & 31) == 0) s_l[threadIdx.x >> 5] = ml;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) ml = s_l[i] > ml ? s_l[i] : ml;
        wl[b] = width_of(ml);
    }
}

__global__ void k_pack_left(const long long *__restrict__ starts, const long long *__restrict__ len, long long L,
                            long long pos0, const unsigned char *__restrict__ wl,
                            const long long *__restrict__ base, unsigned char *__restrict__ wire) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= L) return;
    const long long b = k / kSample, i = k - b * kSample, cntb = (L - b * kSample) < kSample ? L - b * kSample : kSample;
    const int w = wl[b];
    const long long l = len[k];
    put_w(wire + base[b] + i * w, w, (unsigned long long)l);
    put_w(wire + base[b] + (cntb + i) * w, w, (unsigned long long)(l ? pos0 + k - starts[k] : 0));
}

bool fetch_leftmost_mixed(rs_ctx *c, const long long *d_starts, const long long *d_len, long long L, long long pos0,
                          long long *starts, long long *lengths) {
    if (L < (4ll << 20) || std::getenv("RS_WORD_WIRE")) return false;
    const long long nb = (L + kSample - 1) / kSample;
    unsigned char *m = (unsigned char *)buf(c, B_XFER_ENDS, 8 * (size_t)(nb + 1) + (size_t)nb + 64);
    long long *base = (long long *)m;
    unsigned char *wl = (unsigned char *)(base + nb + 1);
    RS_LAUNCH(c, k_widths_left, (unsigned)nb, 256, 0, d_len, L, wl);
    std::vector<unsigned char> w((size_t)nb);
    d2h(c, w.data(), wl, w.size());
    RS_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<long long> bs(nb + 1, 0);
    for (long long b = 0; b < nb; ++b) bs[b + 1] = bs[b] + 2 * std::min(kSample, L - b * kSample) * w[b];
    h2d(c, base, bs.data(), sizeof(long long) * bs.size());
    unsigned char *wire = (unsigned char *)buf(c, B_WIRE, (size_t)bs[nb] + 64);
    RS_LAUNCH_B(c, 16.0 * (double)L, k_pack_left, grid_for(L, 256), 256, 0, d_starts, d_len, L, pos0, wl, base, wire);
    pipeline_blocks(c, wire, bs, [&](long long b, const unsigned char *p) {
        decode_left_block(p, w[b], std::min(kSample, L - b * kSample), pos0 + b * kSample, starts + b * kSample,
                          lengths + b * kSample);
    });
    return true;
}

// Leftmost answers (starts[L], lengths[L], slot j = position pos0 + j) over
// the byte wire (2 bytes per position instead of 8 + 8 in memory, 4 + 4 on the
// 32-bit wire); false (nothing written) when a value does not fit.
bool fetch_leftmost_bytes(rs_ctx *c, const long long *d_starts, const long long *d_len, long long L, long long pos0,
                          long long *starts, long long *lengths) {
    if (L < (4ll << 20) || std::getenv("RS_WORD_WIRE")) return false;
    unsigned char *w = (unsigned char *)buf(c, B_WIRE, (size_t)(2 * L) + 64);
    unsigned *bad = (unsigned *)(((uintptr_t)(w + 2 * L) + 15) & ~(uintptr_t)15);
    RS_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), c->stream));
    RS_LAUNCH_B(c, 18.0 * (double)L, k_wire_leftmost, grid_for(L, 256), 256, 0, d_starts, d_len, L, pos0, w, bad);
    unsigned hbad = 0;
    d2h(c, &hbad, bad, sizeof(hbad));
    RS_CUDA(cudaStreamSynchronize(c->stream));
    if (hbad) return false;
    pipeline_bytes(c, w, 2 * L, [&](const unsigned char *b, long long a, long long x, long long y) {
        // byte offsets [a + x, a + y) are slots [(a + x) / 2, (a + y) / 2)
        const long long j0 = (a + x) / 2;
        leftmost_pairs(b + x, starts + j0, lengths + j0, 0, (y - x) / 2, pos0 + j0);
    });
    return true;
}

// H2D of `count` int64 values into a device u32 array, each checked to lie in
// [lo, hi] and stored as value + add.  Returns false (nothing usable written)
// if a value is out of range.
__global__ void k_expand_bytes(const unsigned char *__restrict__ b, unsigned *__restrict__ out, long long count,
                               unsigned add) {
    const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
    if (i + 3 < count) {
        const uchar4 v = *reinterpret_cast<const uchar4 *>(b + i);
        out[i] = v.x + add;
        out[i + 1] = v.y + add;
        out[i + 2] = v.z + add;
        out[i + 3] = v.w + add;
    } else {
        for (long long j = i; j < count; ++j) out[j] = b[j] + add;
    }
}

// bytes: values of at most 255 (LCP of short-repeat texts) cross PCIe as one
// byte each and are widened on the device, chunk by chunk (a chunk with a
// larger value goes as 32-bit words)
bool put_i64_as_u32(rs_ctx *c, unsigned *ddst, const long long *src, long long count, long long lo, long long hi,
                    long long add, bool bytes) {
    if (count <= 0) return true;
    Stage s = stage(c);
    Pool &pool = Pool::get();
    const long long nch = (count + kChunk - 1) / kChunk;
    unsigned char *ring = bytes ? (unsigned char *)buf(c, B_XFER, 2 * 4 * (size_t)kChunk) : nullptr;
    std::atomic<int> bad{0};
    for (long long i = 0; i < nch; ++i) {
        const long long a = i * kChunk, len = std::min(kChunk, count - a);
        if (i >= 2) RS_CUDA(cudaEventSynchronize(s.ev[i & 1]));  // slot free again
        const long long *in = src + a;
        bool as_bytes = false;
        if (bytes) {
            unsigned char *b = (unsigned char *)s.host[i & 1];
            bad.store(0);
            pool.run([&](int t, int T) {
                long long x, y;
                split(len, t, T, x, y);
                const int r = narrow_bytes(in, b, x, y, lo, hi);
                if (r) bad.fetch_or(r, std::memory_order_relaxed);
            });
            if (bad.load() & 1) {
                RS_CUDA(cudaStreamSynchronize(c->stream));
                return false;
            }
            as_bytes = bad.load() == 0;
            if (as_bytes) {
                unsigned char *d = ring + (size_t)(i & 1) * 4 * kChunk;
                RS_CUDA(cudaMemcpyAsync(d, b, (size_t)len, cudaMemcpyHostToDevice, c->stream));
                c->h2d_bytes += len;
                RS_LAUNCH(c, k_expand_bytes, grid_for((len + 3) / 4, 256), 256, 0, d, ddst + a, len, (unsigned)add);
            }
        }
        if (!as_bytes) {
            unsigned *w = (unsigned *)s.host[i & 1];
            bad.store(0);
            pool.run([&](int t, int T) {
                long long x, y;
                split(len, t, T, x, y);
                if (!narrow_words(in, w, x, y, lo, hi, add)) bad.store(1, std::memory_order_relaxed);
            });
            if (bad.load()) {
                RS_CUDA(cudaStreamSynchronize(c->stream));
                return false;
            }
            RS_CUDA(cudaMemcpyAsync(ddst + a, w, 4 * (size_t)len, cudaMemcpyHostToDevice, c->stream));
            c->h2d_bytes += 4 * len;
        }
        RS_CUDA(cudaEventRecord(s.ev[i & 1], c->stream));
    }
    RS_CUDA(cudaStreamSynchronize(c->stream));
    return true;
}

// H2D of plain bytes (the text): host threads copy into the pinned slot, DMA
// overlaps the next slot's copy.  Small copies go straight through.
void put_bytes(rs_ctx *c, void *ddst, const void *src, size_t bytes) {
    if (bytes < kMinStaged) {
        h2d(c, ddst, src, bytes);
        return;
    }
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost) {
        h2d(c, ddst, src, bytes);  // already page-locked: direct DMA
        return;
    }
    cudaGetLastError();
    Stage s = stage(c);
    Pool &pool = Pool::get();
    const size_t ch = 4 * (size_t)kChunk;
    const size_t nch = (bytes + ch - 1) / ch;
    for (size_t i = 0; i < nch; ++i) {
        const size_t a = i * ch, len = std::min(ch, bytes - a);
        if (i >= 2) RS_CUDA(cudaEventSynchronize(s.ev[i & 1]));
        char *w = (char *)s.host[i & 1];
        const char *in = (const char *)src + a;
        pool.run([&](int t, int T) {
            long long x, y;
            split((long long)len, t, T, x, y);
            if (y > x) std::memcpy(w + x, in + x, (size_t)(y - x));
        });
        RS_CUDA(cudaMemcpyAsync((char *)ddst + a, w, len, cudaMemcpyHostToDevice, c->stream));
        c->h2d_bytes += (long long)len;
        RS_CUDA(cudaEventRecord(s.ev[i & 1], c->stream));
    }
}

}  // namespace rsb
