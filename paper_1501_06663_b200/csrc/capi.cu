// capi.cu -- runtime (context, arena, timing) and the extern "C" entry points
// declared in include/repeatscan_b200.h.
#include <cstdio>
#include <cstring>
#include <exception>
#include <algorithm>
#include <new>

#include "common.cuh"
#include "scatter.cuh"

namespace rsb {

// defined in compact.cu / scan_query.cu
size_t raw_slots(long long n);
void split_llrc(rs_ctx *c, long long m, long long *d_starts, long long *d_lengths);
void add_i64(rs_ctx *c, long long *d, long long count, long long add);
void join_llrc(rs_ctx *c, const long long *d_starts, const long long *d_lengths, long long m, long long n);
void validate_llrc(rs_ctx *c, long long m, long long n);
void check_raw(rs_ctx *c, long long n);
void raw_from_rank_lcp_range(rs_ctx *c, long long n, long long first, long long last);
long long max_lcp(rs_ctx *c, long long n);
void raw_llr_i64(rs_ctx *c, const long long *d_rank, const long long *d_lcp, long long n, long long *d_out);
void flags_i64(rs_ctx *c, const long long *d_raw, long long n, long long *d_out);
void scan_i64(rs_ctx *c, const long long *d_in, long long count, long long *d_out);
void scatter_i64(rs_ctx *c, const long long *d_raw, const long long *d_flags, const long long *d_ps,
                 long long n, long long m, long long *d_starts, long long *d_lengths);
long long check_answers(rs_ctx *c, const long long *d_cs, const long long *d_cl, long long m, long long n,
                        const long long *d_L, const long long *d_O, const long long *d_F, long long T,
                        const long long *d_ls, const long long *d_ll);
bool verify_structures(rs_ctx *c, const unsigned char *d_text, long long n, const long long *d_sa,
                       const long long *d_rank, const long long *d_lcp);
long long serialize_tsv(rs_ctx *c, int mode, long long lo, long long hi);
void walk_steps(rs_ctx *c, int path, long long n, long long *d_steps, unsigned long long *acc_host);
void summarize(rs_ctx *c, const long long *d_steps, long long count, unsigned long long *acc_host);
void ensure_isa(rs_ctx *c);
void dist_sort(rs_ctx *c, long long n, int rank, int world, long long *info);
void dist_update(rs_ctx *c, long long n, int rank, int world, const long long *nbr, long long *send_counts,
                 long long *info);
void dist_apply(rs_ctx *c, long long n, int rank, int world, const void *recv, long long cnt, long long hcap,
                long long *info);
void dist_scan(rs_ctx *c, long long n, int mode, long long halo, long long *total);
bool query_range(rs_ctx *c, int mode, int path, const uint2 *d_e, long long count, const unsigned *d_raw,
                 long long kb, long long ke, int out_off, long long n_slots, long long min_lo = 1);

void fetch_i64(rs_ctx *c, long long *dst, const long long *dsrc, long long count, int kind);
bool put_i64_as_u32(rs_ctx *c, unsigned *ddst, const long long *src, long long count, long long lo, long long hi,
                    long long add, bool bytes = false);
void put_bytes(rs_ctx *c, void *ddst, const void *src, size_t bytes);
void fetch_u32_as_i64(rs_ctx *c, long long *dst, const unsigned *dsrc, long long count, long long add);
bool fetch_csr_bytes(rs_ctx *c, const long long *d_len, const long long *d_off, const long long *d_flat,
                     long long L, long long T, long long *lengths, long long *offsets, long long *flat);
bool fetch_csr_mixed(rs_ctx *c, const long long *d_len, const long long *d_off, const long long *d_flat,
                     long long L, long long T, long long *lengths, long long *offsets, long long *flat);
bool fetch_leftmost_mixed(rs_ctx *c, const long long *d_starts, const long long *d_len, long long L, long long pos0,
                          long long *starts, long long *lengths);
bool fetch_leftmost_bytes(rs_ctx *c, const long long *d_starts, const long long *d_len, long long L, long long pos0,
                          long long *starts, long long *lengths);

void nccl_unique_id(unsigned char *out);
void nccl_init(rs_ctx *c, const unsigned char *id_bytes, int rank, int world);
void nccl_destroy(rs_ctx *c);
void nccl_broadcast_text(rs_ctx *c, long long n, int root);
void nccl_allgather_i64(rs_ctx *c, long long value, long long *out);

void fail(int code, const std::string &msg) { throw RsError{code, msg}; }

void check_cuda(cudaError_t e, const char *what, const char *file, int line) {
    if (e == cudaSuccess) return;
    char b[512];
    snprintf(b, sizeof(b), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file,
             line, what);
    throw RsError{e == cudaErrorMemoryAllocation ? RS_ENOMEM : RS_ECUDA, b};
}

void *buf(rs_ctx *c, BufId id, size_t bytes) {
    Buf &b = c->bufs[id];
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return b.p;
    if (b.p) {
        RS_CUDA(cudaStreamSynchronize(c->stream));
        RS_CUDA(cudaFree(b.p));
        b.p = nullptr;
        b.cap = 0;
    }
    size_t want = (bytes + 4095) & ~size_t(4095);
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        char m[160];
        snprintf(m, sizeof(m), "device allocation of %zu bytes failed (buffer %d)", want, (int)id);
        fail(RS_ENOMEM, m);
    }
    b.cap = want;
    return b.p;
}

void fetch_small(rs_ctx *c, void *host, const void *dev, size_t bytes) {
    if (bytes > 65536) fail(RS_EINVAL, "fetch_small too large");
    RS_CUDA(cudaMemcpyAsync(c->small_host, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += (long long)bytes;
    RS_CUDA(cudaStreamSynchronize(c->stream));
    memcpy(host, c->small_host, bytes);
}

static int prof_event(rs_ctx *c) {
    int idx = 0;
    for (const auto &r : c->prof) idx = std::max(idx, r.ev1 + 1);
    while ((int)c->prof_events.size() <= idx) {
        cudaEvent_t e;
        RS_CUDA(cudaEventCreate(&e));
        c->prof_events.push_back(e);
    }
    return idx;
}

void before_launch(rs_ctx *c) {
    if (!c->profiling) return;
    int e0 = prof_event(c);
    RS_CUDA(cudaEventRecord(c->prof_events[e0], c->stream));
    c->prof.push_back({nullptr, e0, e0 + 1, 0.0});
}

void after_launch(rs_ctx *c, const char *name, double bytes) {
    ++c->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char b[256];
        snprintf(b, sizeof(b), "launch of %s failed: %s", name, cudaGetErrorString(e));
        fail(RS_ECUDA, b);
    }
    if (c->profiling && !c->prof.empty() && c->prof.back().name == nullptr) {
        auto &r = c->prof.back();
        while ((int)c->prof_events.size() <= r.ev1) {
            cudaEvent_t ev;
            RS_CUDA(cudaEventCreate(&ev));
            c->prof_events.push_back(ev);
        }
        RS_CUDA(cudaEventRecord(c->prof_events[r.ev1], c->stream));
        r.name = name;
        r.bytes = bytes;
    }
}

void add_bytes_last(rs_ctx *c, double bytes) {
    if (c->profiling && !c->prof.empty()) c->prof.back().bytes += bytes;
}

Scratch scratch(rs_ctx *c, long long tiles, int slot) {
    (void)slot;
    size_t bytes = sizeof(u64) * (size_t)(tiles + 2);
    char *p = (char *)buf(c, B_SCRATCH, bytes);
    RS_CUDA(cudaMemsetAsync(p, 0, bytes, c->stream));
    return Scratch{(unsigned *)p, (u64 *)(p + 16)};
}

}  // namespace rsb

using namespace rsb;

namespace {

constexpr int kStageEv = 32;  // stage events use slots 32..(32+2*RS_NUM_STAGES)

template <typename F>
int guarded(rs_ctx *c, F &&f) {
    if (!c) return RS_EINVAL;
    try {
        RS_CUDA(cudaSetDevice(c->device));
        f();
        c->err.clear();
        return RS_OK;
    } catch (const RsError &e) {
        c->err = e.msg;
        if (e.code == RS_ECUDA) {
            // leave the context usable for the next call if the error is not sticky
            cudaGetLastError();
        }
        return e.code;
    } catch (const std::bad_alloc &) {
        c->err = "host allocation failed";
        return RS_ENOMEM;
    } catch (const std::exception &e) {
        c->err = e.what();
        return RS_ECUDA;
    }
}

struct Stage {
    rs_ctx *c;
    int s;
    Stage(rs_ctx *c_, int s_) : c(c_), s(s_) { RS_CUDA(cudaEventRecord(c->events[kStageEv + 2 * s], c->stream)); }
    ~Stage() { cudaEventRecord(c->events[kStageEv + 2 * s + 1], c->stream); }
};

void collect_stages(rs_ctx *c, const bool *used) {
    RS_CUDA(cudaStreamSynchronize(c->stream));
    for (int s = 0; s < RS_NUM_STAGES; ++s) {
        if (!used[s]) {
            c->stage_ms[s] = 0;
            continue;
        }
        float ms = 0;
        RS_CUDA(cudaEventElapsedTime(&ms, c->events[kStageEv + 2 * s], c->events[kStageEv + 2 * s + 1]));
        c->stage_ms[s] = ms;
    }
}

void check_n(long long n) {
    if (n < 0) fail(RS_EINVAL, "negative length");
    if (n > 2147483646ll) fail(RS_ERANGE, "n exceeds 2^31 - 2 (32-bit device indices)");
}

void h2d(rs_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes) RS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += (long long)bytes;
}
void d2h(rs_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes) RS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += (long long)bytes;
}

void invalidate(rs_ctx *c) {
    c->have_text = c->have_sa = c->have_lcp = c->have_raw = c->have_compact = false;
    c->sa_device_built = false;
    c->sa_isa_consistent = false;
    c->max_lcp = -1;
    c->raw_from_round0 = false;
    c->packed_bits = 0;
    c->isa_lazy = false;
    c->out_mode = -1;
    c->n = -1;
}

// Ensure the raw LLR array for the pipeline exists (B_RAW, u32, 1-based).
void ensure_raw(rs_ctx *c, bool *used) {
    if (c->have_raw) return;
    if (c->have_lcp && c->raw_from_round0) {  // produced during the SA/LCP build
        c->have_raw = true;
        return;
    }
    long long n = c->n;
    if (!c->have_lcp) {
        if (!c->have_sa) {
            if (!c->have_text) fail(RS_ESTATE, "no text, structures or raw array loaded");
            Stage st(c, RS_STAGE_SA);
            used[RS_STAGE_SA] = true;
            build_suffix_array(c, n);
            c->have_sa = true;
        }
        if (!c->have_text) fail(RS_ESTATE, "LCP needs the text");
        Stage st(c, RS_STAGE_LCP);
        used[RS_STAGE_LCP] = true;
        build_lcp(c, n);
        c->have_lcp = true;
        c->max_lcp = -1;
        if (c->raw_from_round0) {  // the SA/LCP build already produced raw
            c->have_raw = true;
            return;
        }
    }
    Stage st(c, RS_STAGE_RAW_LLR);
    used[RS_STAGE_RAW_LLR] = true;
    if (c->have_sa && (c->sa_device_built || c->sa_isa_consistent))
        raw_from_sa_lcp(c, n, raw_slots(n));  // SA order + bucketed scatter (consistent structures)
    else
        raw_from_rank_lcp(c, n);  // reference formula on caller-given rank/lcp
    c->have_raw = true;
}

void ensure_compact(rs_ctx *c, bool *used) {
    if (c->have_compact) return;
    ensure_raw(c, used);
    Stage st(c, RS_STAGE_COMPACT);
    used[RS_STAGE_COMPACT] = true;
    c->m = compact_from_raw(c, c->n);
    c->have_compact = true;
}

}  // namespace

extern "C" {

const char *rs_version(void) { return "repeatscan_b200 0.1.0 (sm_100a)"; }

int rs_device_count(int *count) {
    if (!count) return RS_EINVAL;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
    }
    return RS_OK;
}

int rs_create(int device, rs_ctx **out) {
    if (!out) return RS_EINVAL;
    *out = nullptr;
    rs_ctx *c = new (std::nothrow) rs_ctx();
    if (!c) return RS_ENOMEM;
    c->device = device;
    int rc = guarded(c, [&] {
        int ndev = 0;
        RS_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) fail(RS_EINVAL, "no such CUDA device");
        cudaDeviceProp prop;
        RS_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) fail(RS_ECUDA, std::string("librepeatscan_b200 is built for sm_100a; device is ") +
                                                 prop.name);
        c->sm_count = prop.multiProcessorCount;
        RS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        for (int i = 0; i < kMaxEvents; ++i) RS_CUDA(cudaEventCreate(&c->events[i]));
        RS_CUDA(cudaHostAlloc(&c->small_host, 65536, cudaHostAllocDefault));
    });
    if (rc != RS_OK) {
        fprintf(stderr, "rs_create: %s\n", c->err.c_str());
        rs_destroy(c);
        return rc;
    }
    *out = c;
    return RS_OK;
}

int rs_destroy(rs_ctx *c) {
    if (!c) return RS_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (int i = 0; i < B_COUNT; ++i)
        if (c->bufs[i].p) cudaFree(c->bufs[i].p);
    for (int i = 0; i < kMaxEvents; ++i)
        if (c->events[i]) cudaEventDestroy(c->events[i]);
    for (auto e : c->prof_events) cudaEventDestroy(e);
    if (c->nccl_comm) {
        try {
            nccl_destroy(c);
        } catch (...) {
        }
    }
    if (c->small_host) cudaFreeHost(c->small_host);
    for (int i = 0; i < 2; ++i) {
        if (c->xfer_host[i]) cudaFreeHost(c->xfer_host[i]);
        if (c->xfer_ev[i]) cudaEventDestroy(c->xfer_ev[i]);
    }
    if (c->xfer_side_ev) cudaEventDestroy(c->xfer_side_ev);
    if (c->xfer_side) cudaStreamDestroy(c->xfer_side);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return RS_OK;
}

const char *rs_last_error(const rs_ctx *c) { return c ? c->err.c_str() : "null context"; }

int rs_synchronize(rs_ctx *c) {
    return guarded(c, [&] { RS_CUDA(cudaStreamSynchronize(c->stream)); });
}

int rs_launch_count(const rs_ctx *c, int64_t *count) {
    if (!c || !count) return RS_EINVAL;
    *count = c->launches;
    return RS_OK;
}

int rs_transfer_bytes(const rs_ctx *c, int64_t *h2d_bytes, int64_t *d2h_bytes) {
    if (!c || !h2d_bytes || !d2h_bytes) return RS_EINVAL;
    *h2d_bytes = c->h2d_bytes;
    *d2h_bytes = c->d2h_bytes;
    return RS_OK;
}

int rs_stage_times(const rs_ctx *c, double *ms) {
    if (!c || !ms) return RS_EINVAL;
    for (int i = 0; i < RS_NUM_STAGES; ++i) ms[i] = c->stage_ms[i];
    return RS_OK;
}

int rs_record_event(rs_ctx *c, int slot) {
    return guarded(c, [&] {
        if (slot < 0 || slot >= kStageEv) fail(RS_EINVAL, "event slot must be 0..31");
        RS_CUDA(cudaEventRecord(c->events[slot], c->stream));
    });
}

int rs_elapsed_ms(rs_ctx *c, int a, int b, float *ms) {
    return guarded(c, [&] {
        if (a < 0 || a >= kStageEv || b < 0 || b >= kStageEv || !ms) fail(RS_EINVAL, "bad event slot");
        RS_CUDA(cudaEventSynchronize(c->events[b]));
        RS_CUDA(cudaEventElapsedTime(ms, c->events[a], c->events[b]));
    });
}

int rs_device_bytes(const rs_ctx *c, int64_t *bytes) {
    if (!c || !bytes) return RS_EINVAL;
    int64_t t = 0;
    for (int i = 0; i < B_COUNT; ++i) t += (int64_t)c->bufs[i].cap;
    *bytes = t;
    return RS_OK;
}

int rs_release(rs_ctx *c) {
    return guarded(c, [&] {
        RS_CUDA(cudaStreamSynchronize(c->stream));
        for (int i = 0; i < B_COUNT; ++i) {
            if (c->bufs[i].p) RS_CUDA(cudaFree(c->bufs[i].p));
            c->bufs[i] = Buf();
        }
        invalidate(c);
    });
}

int rs_host_alloc(int64_t bytes, void **out) {
    if (!out || bytes < 0) return RS_EINVAL;
    *out = nullptr;
    if (bytes == 0) bytes = 64;
    cudaError_t e = cudaHostAlloc(out, (size_t)bytes, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return RS_ENOMEM;
    }
    return RS_OK;
}

int rs_host_free(void *p) {
    if (p) cudaFreeHost(p);
    return RS_OK;
}

// ---- array-level operators -----------------------------------------------------

int rs_raw_llr(rs_ctx *c, const int64_t *rank, const int64_t *lcp, int64_t n, int64_t *raw) {
    return guarded(c, [&] {
        check_n(n);
        invalidate(c);
        long long *dr = (long long *)buf(c, B_I64A, 8 * (size_t)(n + 1));
        long long *dl = (long long *)buf(c, B_I64B, 8 * (size_t)(n + 2));
        long long *dout = (long long *)buf(c, B_I64C, 8 * (size_t)(n + 1));
        h2d(c, dr, rank, 8 * (size_t)(n + 1));
        h2d(c, dl, lcp, 8 * (size_t)(n + 2));
        raw_llr_i64(c, dr, dl, n, dout);
        d2h(c, raw, dout, 8 * (size_t)(n + 1));
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_flags(rs_ctx *c, const int64_t *raw, int64_t n, int64_t *flags) {
    return guarded(c, [&] {
        check_n(n);
        invalidate(c);
        long long *dr = (long long *)buf(c, B_I64A, 8 * (size_t)(n + 1));
        long long *dout = (long long *)buf(c, B_I64C, 8 * (size_t)(n + 1));
        h2d(c, dr, raw, 8 * (size_t)(n + 1));
        flags_i64(c, dr, n, dout);
        d2h(c, flags, dout, 8 * (size_t)(n + 1));
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_inclusive_scan(rs_ctx *c, const int64_t *values, int64_t count, int64_t *out) {
    return guarded(c, [&] {
        if (count < 0) fail(RS_EINVAL, "negative count");
        if (count == 0) return;
        invalidate(c);
        long long *din = (long long *)buf(c, B_I64A, 8 * (size_t)count);
        long long *dout = (long long *)buf(c, B_I64C, 8 * (size_t)count);
        h2d(c, din, values, 8 * (size_t)count);
        scan_i64(c, din, count, dout);
        d2h(c, out, dout, 8 * (size_t)count);
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_prefix_sum(rs_ctx *c, const int64_t *flags, int64_t n, int64_t *ps) {
    return guarded(c, [&] {
        check_n(n);
        ps[0] = 0;
        if (n == 0) return;
        invalidate(c);
        long long *din = (long long *)buf(c, B_I64A, 8 * (size_t)n);
        long long *dout = (long long *)buf(c, B_I64C, 8 * (size_t)n);
        h2d(c, din, flags + 1, 8 * (size_t)n);
        scan_i64(c, din, n, dout);
        d2h(c, ps + 1, dout, 8 * (size_t)n);
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_scatter_compact(rs_ctx *c, const int64_t *raw, const int64_t *flags, const int64_t *ps, int64_t n,
                       int64_t *starts, int64_t *lengths) {
    return guarded(c, [&] {
        check_n(n);
        long long m = n > 0 ? ps[n] : 0;
        if (m < 0 || m > n) fail(RS_EINVAL, "ps[n] out of range");
        if (n == 0 || m == 0) return;
        invalidate(c);
        long long *dr = (long long *)buf(c, B_I64A, 8 * (size_t)(n + 1));
        long long *df = (long long *)buf(c, B_I64B, 8 * (size_t)(n + 1));
        long long *dp = (long long *)buf(c, B_I64C, 8 * (size_t)(n + 1));
        long long *ds = (long long *)buf(c, B_I64D, 16 * (size_t)m);
        h2d(c, dr, raw, 8 * (size_t)(n + 1));
        h2d(c, df, flags, 8 * (size_t)(n + 1));
        h2d(c, dp, ps, 8 * (size_t)(n + 1));
        scatter_i64(c, dr, df, dp, n, m, ds, ds + m);
        d2h(c, starts, ds, 8 * (size_t)m);
        d2h(c, lengths, ds + m, 8 * (size_t)m);
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_set_raw(rs_ctx *c, const int64_t *raw, int64_t n) {
    return guarded(c, [&] {
        check_n(n);
        invalidate(c);
        long long *dr = (long long *)buf(c, B_I64A, 8 * (size_t)(n + 1));
        unsigned *r32 = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots(n));
        RS_CUDA(cudaMemsetAsync(r32, 0, sizeof(unsigned) * raw_slots(n), c->stream));
        h2d(c, dr, raw, 8 * (size_t)(n + 1));
        // slot 0 is a pad: the reference reads raw[0] only as the "previous"
        // length of position 1 (fill_flags), where any value <= 0 behaves as 0.
        if (n > 0) narrow_i64_to_u32(c, dr + 1, r32 + 1, n, 0, n, 0, "raw LLR array");
        check_raw(c, n);
        c->n = n;
        c->have_raw = true;
    });
}

int rs_compact(rs_ctx *c, const int64_t *raw, int64_t n, int64_t *starts, int64_t *lengths, int64_t *m) {
    return guarded(c, [&] {
        check_n(n);
        invalidate(c);
        *m = 0;
        if (n == 0) return;
        long long *dr = (long long *)buf(c, B_I64A, 8 * (size_t)(n + 1));
        unsigned *r32 = (unsigned *)buf(c, B_RAW, sizeof(unsigned) * raw_slots(n));
        RS_CUDA(cudaMemsetAsync(r32, 0, sizeof(unsigned) * raw_slots(n), c->stream));
        h2d(c, dr, raw, 8 * (size_t)(n + 1));
        narrow_i64_to_u32(c, dr + 1, r32 + 1, n, 0, n, 0, "raw LLR array");
        long long mm = compact_from_raw(c, n);
        long long *ds = (long long *)buf(c, B_I64D, 16 * (size_t)(mm + 1));
        split_llrc(c, mm, ds, ds + mm);
        d2h(c, starts, ds, 8 * (size_t)mm);
        d2h(c, lengths, ds + mm, 8 * (size_t)mm);
        RS_CUDA(cudaStreamSynchronize(c->stream));
        *m = mm;
    });
}

// ---- pipeline ----------------------------------------------------------------------

int rs_set_text(rs_ctx *c, const uint8_t *text, int64_t n) {
    return guarded(c, [&] {
        check_n(n);
        invalidate(c);
        bool used[RS_NUM_STAGES] = {};
        {
            Stage st(c, RS_STAGE_H2D);
            used[RS_STAGE_H2D] = true;
            unsigned char *d = (unsigned char *)buf(c, B_TEXT, (size_t)n + 128);
            RS_CUDA(cudaMemsetAsync(d + n, 0, 128, c->stream));
            put_bytes(c, d, text, (size_t)n);
        }
        collect_stages(c, used);
        c->n = n;
        c->have_text = true;
    });
}

int rs_set_structures(rs_ctx *c, const int64_t *sa, const int64_t *rank, const int64_t *lcp, int64_t n) {
    return guarded(c, [&] {
        check_n(n);
        if (!rank || !lcp) fail(RS_EINVAL, "rank and lcp are required");
        bool keep_text = c->have_text && c->n == n;
        invalidate(c);
        c->have_text = keep_text;
        unsigned *disa = (unsigned *)buf(c, B_ISA, sizeof(unsigned) * (size_t)(n + 4));
        unsigned *dlcp = (unsigned *)buf(c, B_LCP, sizeof(unsigned) * (size_t)(n + 4));
        RS_CUDA(cudaMemsetAsync(dlcp, 0, sizeof(unsigned) * (size_t)(n + 4), c->stream));
        if (n > 0) {  // narrowed (range-checked) on the host, 4 bytes per value on the wire
            if (sa) {
                unsigned *dsa = (unsigned *)buf(c, B_SA, sizeof(unsigned) * (size_t)(n + 4));
                if (!put_i64_as_u32(c, dsa, (const long long *)sa + 1, n, 1, n, -1))
                    fail(RS_EINVAL, "sa has values out of range");
            }
            if (!put_i64_as_u32(c, disa, (const long long *)rank + 1, n, 1, n, -1))
                fail(RS_EINVAL, "rank has values out of range");
            if (!put_i64_as_u32(c, dlcp, (const long long *)lcp + 1, n + 1, 0, n, 0, true))
                fail(RS_EINVAL, "lcp has values out of range");
        }
        // The reference computes raw LLR from rank and lcp (_kernels_numba.py:33-38).
        // When sa is given and is exactly the inverse of rank, the same values
        // come from SA order (lcp read sequentially + one bucketed scatter)
        // instead of two random lcp gathers per position; checked once here.
        if (sa && n > 0)
            c->sa_isa_consistent =
                check_rank_inverse(c, (const unsigned *)c->bufs[B_SA].p, disa, n);
        RS_CUDA(cudaStreamSynchronize(c->stream));
        c->n = n;
        c->have_sa = sa != nullptr;
        c->have_lcp = true;
        c->max_lcp = -1;
    });
}

int rs_verify_structures(rs_ctx *c, const uint8_t *text, int64_t n, const int64_t *sa, const int64_t *rank,
                         const int64_t *lcp, int64_t *ok) {
    return guarded(c, [&] {
        check_n(n);
        invalidate(c);
        *ok = 0;
        unsigned char *dt = (unsigned char *)buf(c, B_TEXT, (size_t)n + 128);
        RS_CUDA(cudaMemsetAsync(dt + n, 0, 128, c->stream));
        h2d(c, dt, text, (size_t)n);
        long long *dsa = (long long *)buf(c, B_I64A, 8 * (size_t)(n + 1));
        long long *drk = (long long *)buf(c, B_I64B, 8 * (size_t)(n + 1));
        long long *dlc = (long long *)buf(c, B_I64C, 8 * (size_t)(n + 2));
        h2d(c, dsa, sa, 8 * (size_t)(n + 1));
        h2d(c, drk, rank, 8 * (size_t)(n + 1));
        h2d(c, dlc, lcp, 8 * (size_t)(n + 2));
        *ok = verify_structures(c, dt, n, dsa, drk, dlc) ? 1 : 0;
    });
}

int rs_check_answers(rs_ctx *c, const int64_t *starts, const int64_t *lengths, int64_t m, int64_t n,
                     const int64_t *a_lengths, const int64_t *a_offsets, const int64_t *a_flat, int64_t total,
                     const int64_t *l_starts, const int64_t *l_lengths, int64_t *bad) {
    return guarded(c, [&] {
        check_n(n);
        if (m < 0 || m > n || total < 0) fail(RS_EINVAL, "bad entry count or tie total");
        invalidate(c);
        *bad = 0;
        long long *dcs = (long long *)buf(c, B_I64A, 8 * (size_t)(m + 1));
        long long *dcl = (long long *)buf(c, B_I64B, 8 * (size_t)(m + 1));
        h2d(c, dcs, starts, 8 * (size_t)m);
        h2d(c, dcl, lengths, 8 * (size_t)m);
        long long *dL = nullptr, *dO = nullptr, *dF = nullptr, *dls = nullptr, *dll = nullptr;
        if (a_lengths) {
            dL = (long long *)buf(c, B_I64C, 8 * (size_t)(n + 1));
            dO = (long long *)buf(c, B_I64D, 8 * (size_t)(n + 2));
            dF = (long long *)buf(c, B_T1, 8 * (size_t)(total + 1));
            h2d(c, dL, a_lengths, 8 * (size_t)(n + 1));
            h2d(c, dO, a_offsets, 8 * (size_t)(n + 2));
            h2d(c, dF, a_flat, 8 * (size_t)total);
        }
        if (l_starts) {
            dls = (long long *)buf(c, B_T2, 8 * (size_t)(n + 1));
            dll = (long long *)buf(c, B_T3, 8 * (size_t)(n + 1));
            h2d(c, dls, l_starts, 8 * (size_t)(n + 1));
            h2d(c, dll, l_lengths, 8 * (size_t)(n + 1));
        }
        *bad = check_answers(c, dcs, dcl, m, n, dL, dO, dF, total, dls, dll);
    });
}

int rs_build_structures(rs_ctx *c) {
    return guarded(c, [&] {
        if (!c->have_text) fail(RS_ESTATE, "rs_build_structures needs rs_set_text first");
        bool used[RS_NUM_STAGES] = {};
        long long n = c->n;
        c->have_raw = c->have_compact = false;
        {
            Stage st(c, RS_STAGE_SA);
            used[RS_STAGE_SA] = true;
            build_suffix_array(c, n);
        }
        c->have_sa = true;
        {
            Stage st(c, RS_STAGE_LCP);
            used[RS_STAGE_LCP] = true;
            build_lcp(c, n);
        }
        c->have_lcp = true;
        c->max_lcp = -1;
        collect_stages(c, used);
    });
}

int rs_get_structures(rs_ctx *c, int64_t *sa, int64_t *rank, int64_t *lcp) {
    return guarded(c, [&] {
        if (!c->have_sa || !c->have_lcp) fail(RS_ESTATE, "no structures on device");
        long long n = c->n;
        sa[0] = rank[0] = lcp[0] = 0;
        fetch_u32_as_i64(c, (long long *)sa + 1, (const unsigned *)c->bufs[B_SA].p, n, 1);
        ensure_isa(c);
        fetch_u32_as_i64(c, (long long *)rank + 1, (const unsigned *)c->bufs[B_ISA].p, n, 1);
        fetch_u32_as_i64(c, (long long *)lcp + 1, (const unsigned *)c->bufs[B_LCP].p, n + 1, 0);
        if (n == 0) lcp[1] = 0;
    });
}

int rs_set_compact(rs_ctx *c, const int64_t *starts, const int64_t *lengths, int64_t m, int64_t n) {
    return guarded(c, [&] {
        check_n(n);
        if (m < 0 || m > n) fail(RS_EINVAL, "compact size out of range");
        invalidate(c);
        long long *ds = (long long *)buf(c, B_I64D, 16 * (size_t)(m + 1));
        h2d(c, ds, starts, 8 * (size_t)m);
        h2d(c, ds + m, lengths, 8 * (size_t)m);
        join_llrc(c, ds, ds + m, m, n);
        c->n = n;
        c->m = m;
        c->have_compact = true;
    });
}

int rs_query(rs_ctx *c, int mode, int path, int64_t *total) {
    return guarded(c, [&] {
        if (mode != RS_MODE_LEFTMOST && mode != RS_MODE_ALL) fail(RS_EINVAL, "unknown mode");
        if (path != RS_PATH_RAW && path != RS_PATH_COMPACT) fail(RS_EINVAL, "unknown path");
        if (c->n < 0) fail(RS_ESTATE, "nothing loaded");
        long long n = c->n;
        bool used[RS_NUM_STAGES] = {};
        // compact path: unless LLRc already exists, compact inside the scan
        // tiles (k_query_fused); materialise LLRc only for long repeats
        bool fused = path == RS_PATH_COMPACT && !c->have_compact && n > 0;
        if (path == RS_PATH_RAW || fused) ensure_raw(c, used);
        else ensure_compact(c, used);
        if (fused) {
            Stage st(c, RS_STAGE_QUERY);
            used[RS_STAGE_QUERY] = true;
            c->out_ref_layout = true;
            if (!query_range(c, mode, path, nullptr, 0, (const unsigned *)c->bufs[B_RAW].p, 1, n, 1, n)) {
                fused = false;
                ensure_compact(c, used);
            }
        }
        if (!fused) {
            Stage st(c, RS_STAGE_QUERY);
            used[RS_STAGE_QUERY] = true;
            if (n == 0) {
                long long *o0 = (long long *)buf(c, B_OUT0, 16);
                long long *o1 = (long long *)buf(c, B_OUT1, 16);
                long long z[2] = {mode == RS_MODE_ALL ? 0 : -1, 0};
                h2d(c, o0, z, 8);
                h2d(c, o1, z + 1, 8);
                if (mode == RS_MODE_ALL) h2d(c, o1 + 1, z + 1, 8);
                c->total = 0;
                c->out_mode = mode;
                c->out_ref_layout = true;
            } else if (path == RS_PATH_RAW) {
                c->out_ref_layout = true;
                query_range(c, mode, path, nullptr, 0, (const unsigned *)c->bufs[B_RAW].p, 1, n, 1, n);
            } else {
                c->out_ref_layout = true;
                query_range(c, mode, path, (const uint2 *)c->bufs[B_LLRC].p, c->m, nullptr, 1, n, 1, n);
            }
        }
        collect_stages(c, used);
        if (total) *total = mode == RS_MODE_ALL ? c->total : 0;
    });
}

int rs_fetch_leftmost(rs_ctx *c, int64_t *starts, int64_t *lengths) {
    return guarded(c, [&] {
        if (c->out_mode != 0) fail(RS_ESTATE, "no leftmost results on device");
        long long n = c->n;
        if (fetch_leftmost_bytes(c, (const long long *)c->bufs[B_OUT0].p, (const long long *)c->bufs[B_OUT1].p,
                                 n + 1, 0, (long long *)starts, (long long *)lengths))
            return;
        if (fetch_leftmost_mixed(c, (const long long *)c->bufs[B_OUT0].p, (const long long *)c->bufs[B_OUT1].p,
                                 n + 1, 0, (long long *)starts, (long long *)lengths))
            return;
        fetch_i64(c, (long long *)starts, (const long long *)c->bufs[B_OUT0].p, n + 1, 1);
        fetch_i64(c, (long long *)lengths, (const long long *)c->bufs[B_OUT1].p, n + 1, 0);
    });
}

int rs_fetch_all(rs_ctx *c, int64_t *lengths, int64_t *offsets, int64_t *flat) {
    return guarded(c, [&] {
        if (c->out_mode != 1) fail(RS_ESTATE, "no all-ties results on device");
        long long n = c->n;
        if (fetch_csr_bytes(c, (const long long *)c->bufs[B_OUT0].p, (const long long *)c->bufs[B_OUT1].p,
                            (const long long *)c->bufs[B_FLAT].p, n + 1, c->total, (long long *)lengths,
                            (long long *)offsets, (long long *)flat))
            return;
        if (fetch_csr_mixed(c, (const long long *)c->bufs[B_OUT0].p, (const long long *)c->bufs[B_OUT1].p,
                            (const long long *)c->bufs[B_FLAT].p, n + 1, c->total, (long long *)lengths,
                            (long long *)offsets, (long long *)flat))
            return;
        fetch_i64(c, (long long *)lengths, (const long long *)c->bufs[B_OUT0].p, n + 1, 0);
        fetch_i64(c, (long long *)offsets, (const long long *)c->bufs[B_OUT1].p, n + 2, 2);
        fetch_i64(c, (long long *)flat, (const long long *)c->bufs[B_FLAT].p, c->total, 0);
    });
}

int rs_get_raw(rs_ctx *c, int64_t *raw) {
    return guarded(c, [&] {
        bool used[RS_NUM_STAGES] = {};
        ensure_raw(c, used);
        long long n = c->n;
        fetch_u32_as_i64(c, (long long *)raw, (const unsigned *)c->bufs[B_RAW].p, n + 1, 0);
        raw[0] = 0;
    });
}

int rs_get_compact_size(rs_ctx *c, int64_t *m) {
    return guarded(c, [&] {
        bool used[RS_NUM_STAGES] = {};
        ensure_compact(c, used);
        *m = c->m;
    });
}

int rs_get_compact(rs_ctx *c, int64_t *starts, int64_t *lengths) {
    return guarded(c, [&] {
        bool used[RS_NUM_STAGES] = {};
        ensure_compact(c, used);
        long long m = c->m;
        if (m == 0) return;
        long long *ds = (long long *)buf(c, B_I64D, 16 * (size_t)(m + 1));
        split_llrc(c, m, ds, ds + m);
        d2h(c, starts, ds, 8 * (size_t)m);
        d2h(c, lengths, ds + m, 8 * (size_t)m);
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_reset(rs_ctx *c) {
    return guarded(c, [&] { invalidate(c); });
}

int rs_clear_derived(rs_ctx *c) {
    return guarded(c, [&] {
        if (!c->have_text) fail(RS_ESTATE, "no text loaded");
        c->have_sa = c->have_lcp = c->have_raw = c->have_compact = false;
        c->max_lcp = -1;
        c->out_mode = -1;
    });
}

int rs_clear_llr(rs_ctx *c) {
    return guarded(c, [&] {
        if (!c->have_lcp) fail(RS_ESTATE, "no structures on device");
        c->have_raw = c->have_compact = false;
        c->raw_from_round0 = false;
        c->out_mode = -1;
    });
}

int rs_profile_begin(rs_ctx *c) {
    return guarded(c, [&] {
        c->prof.clear();
        c->prof_agg.clear();
        c->profiling = true;
    });
}

int rs_profile_end(rs_ctx *c, int *kinds) {
    return guarded(c, [&] {
        c->profiling = false;
        RS_CUDA(cudaStreamSynchronize(c->stream));
        c->prof_agg.clear();
        for (const auto &r : c->prof) {
            if (!r.name) continue;
            float ms = 0;
            RS_CUDA(cudaEventElapsedTime(&ms, c->prof_events[r.ev0], c->prof_events[r.ev1]));
            std::string nm(r.name);
            auto it = std::find_if(c->prof_agg.begin(), c->prof_agg.end(),
                                   [&](const rs_ctx::ProfAgg &a) { return a.name == nm; });
            if (it == c->prof_agg.end()) {
                c->prof_agg.push_back({nm, 0, 0.0, 0.0});
                it = c->prof_agg.end() - 1;
            }
            it->launches += 1;
            it->ms += ms;
            it->bytes += r.bytes;
        }
        c->prof.clear();
        if (kinds) *kinds = (int)c->prof_agg.size();
    });
}

int rs_profile_kernel(rs_ctx *c, int i, char *name, int cap, int64_t *launches, double *total_ms,
                      double *bytes) {
    return guarded(c, [&] {
        if (i < 0 || i >= (int)c->prof_agg.size()) fail(RS_ERANGE, "no such profiled kernel");
        const auto &a = c->prof_agg[i];
        if (name && cap > 0) {
            snprintf(name, (size_t)cap, "%s", a.name.c_str());
        }
        if (launches) *launches = a.launches;
        if (total_ms) *total_ms = a.ms;
        if (bytes) *bytes = a.bytes;
    });
}

int rs_sa_rounds(const rs_ctx *c, int *rounds) {
    if (!c || !rounds) return RS_EINVAL;
    *rounds = c->sa_rounds;
    return RS_OK;
}

int rs_suffix_structures(rs_ctx *c, const uint8_t *text, int64_t n, int64_t *sa, int64_t *rank, int64_t *lcp) {
    int rc = rs_set_text(c, text, n);
    if (rc) return rc;
    rc = rs_build_structures(c);
    if (rc) return rc;
    return rs_get_structures(c, sa, rank, lcp);
}

// ---- TSV ---------------------------------------------------------------------------

int rs_serialize(rs_ctx *c, int64_t lo, int64_t hi, int64_t *nbytes) {
    return guarded(c, [&] {
        if (c->out_mode != RS_MODE_LEFTMOST && c->out_mode != RS_MODE_ALL) fail(RS_ESTATE, "no query results");
        if (!c->out_ref_layout) fail(RS_ESTATE, "shard-local results are not serializable");
        if (lo < 1 || hi > c->n || (hi < lo && !(hi == lo - 1))) fail(RS_ERANGE, "range out of range");
        *nbytes = serialize_tsv(c, c->out_mode, lo, hi);
        if (hi < lo) c->tsv_bytes = 0;
    });
}

int rs_fetch_serialized(rs_ctx *c, uint8_t *out) {
    return guarded(c, [&] {
        if (c->tsv_bytes > 0) {
            d2h(c, out, c->bufs[B_TSV].p, (size_t)c->tsv_bytes);
            RS_CUDA(cudaStreamSynchronize(c->stream));
        }
    });
}

// ---- walk statistics ---------------------------------------------------------------

static void stats_out(const unsigned long long *acc, int64_t *stats) {
    stats[0] = acc[3] ? (int64_t)acc[0] : 0;
    stats[1] = (int64_t)acc[1];
    stats[2] = (int64_t)acc[2];
    stats[3] = (int64_t)acc[3];
}

int rs_walk_steps(rs_ctx *c, int path, int64_t *steps, int64_t *stats) {
    return guarded(c, [&] {
        if (path != RS_PATH_RAW && path != RS_PATH_COMPACT) fail(RS_EINVAL, "unknown path");
        if (!stats) fail(RS_EINVAL, "stats output required");
        if (c->n < 0) fail(RS_ESTATE, "nothing loaded");
        bool used[RS_NUM_STAGES] = {};
        if (path == RS_PATH_RAW) ensure_raw(c, used);
        else ensure_compact(c, used);
        long long n = c->n;
        long long *d = nullptr;
        if (steps) d = (long long *)buf(c, B_I64C, 8 * (size_t)(n + 1));
        unsigned long long acc[4];
        walk_steps(c, path, n, d, acc);
        if (steps) {
            d2h(c, steps, d, 8 * (size_t)(n + 1));
            RS_CUDA(cudaStreamSynchronize(c->stream));
        }
        stats_out(acc, stats);
    });
}

int rs_summarize_steps(rs_ctx *c, const int64_t *steps, int64_t count, int64_t *stats) {
    return guarded(c, [&] {
        if (count < 0 || !stats) fail(RS_EINVAL, "bad arguments");
        long long *d = (long long *)buf(c, B_I64C, 8 * (size_t)(count + 1));
        h2d(c, d, steps, 8 * (size_t)count);
        unsigned long long acc[4];
        summarize(c, d, count, acc);
        stats_out(acc, stats);
    });
}

// ---- sharded ---------------------------------------------------------------------

int rs_device_buffer(rs_ctx *c, int which, int64_t bytes, void **ptr) {
    return guarded(c, [&] {
        static const BufId ids[7] = {B_LLRC, B_OUT0, B_OUT1, B_FLAT, B_TEXT, B_SEND, B_RAW};
        if (which < 0 || which > 6 || bytes < 0 || !ptr) fail(RS_EINVAL, "bad buffer request");
        // exactly `bytes` (+ the text's zero pad): a request within the current
        // capacity never reallocates, so views of filled buffers stay valid
        *ptr = buf(c, ids[which], (size_t)bytes + (which == RS_BUF_TEXT ? 128 : 0));
    });
}

int rs_set_compact_device(rs_ctx *c, int64_t m, int64_t n) {
    return guarded(c, [&] {
        check_n(n);
        if (m < 0 || m > n) fail(RS_EINVAL, "compact size out of range");
        if (c->bufs[B_LLRC].cap < sizeof(uint2) * (size_t)(m + 4)) fail(RS_ESTATE, "LLRc buffer too small");
        invalidate(c);
        RS_CUDA(cudaMemsetAsync((uint2 *)c->bufs[B_LLRC].p + m, 0, sizeof(uint2) * 4, c->stream));
        validate_llrc(c, m, n);
        c->n = n;
        c->m = m;
        c->have_compact = true;
    });
}

int rs_stream(rs_ctx *c, void **stream) {
    if (!c || !stream) return RS_EINVAL;
    *stream = (void *)c->stream;
    return RS_OK;
}

int rs_query_shard(rs_ctx *c, int mode, int64_t lo, int64_t hi, int64_t *total) {
    return guarded(c, [&] {
        if (!c->have_compact) fail(RS_ESTATE, "no compact entries on device");
        if (mode != RS_MODE_LEFTMOST && mode != RS_MODE_ALL) fail(RS_EINVAL, "unknown mode");
        if (lo < 1 || hi < lo || hi > c->n + 1) fail(RS_ERANGE, "shard out of range");
        bool used[RS_NUM_STAGES] = {};
        {
            Stage st(c, RS_STAGE_QUERY);
            used[RS_STAGE_QUERY] = true;
            long long cnt = hi - lo;
            long long *o1 = (long long *)buf(c, B_OUT1, 8 * (size_t)(cnt + 2));
            buf(c, B_OUT0, 8 * (size_t)(cnt + 1));
            RS_CUDA(cudaMemsetAsync(o1, 0, 8, c->stream));
            c->total = 0;
            c->out_mode = mode;
            c->out_ref_layout = false;
            if (cnt > 0)
                query_range(c, mode, RS_PATH_COMPACT, (const uint2 *)c->bufs[B_LLRC].p, c->m, nullptr, lo, hi - 1,
                            0, cnt);
        }
        collect_stages(c, used);
        c->shard_lo = lo;
        c->shard_hi = hi;
        if (total) *total = mode == RS_MODE_ALL ? c->total : 0;
    });
}

int rs_query_structures_shard(rs_ctx *c, int mode, int64_t lo, int64_t hi, int64_t *total) {
    return guarded(c, [&] {
        if (!c->have_lcp) fail(RS_ESTATE, "no suffix structures on device");
        if (mode != RS_MODE_LEFTMOST && mode != RS_MODE_ALL) fail(RS_EINVAL, "unknown mode");
        if (lo < 1 || hi < lo || hi > c->n + 1) fail(RS_ERANGE, "shard out of range");
        const long long n = c->n;
        bool used[RS_NUM_STAGES] = {};
        if (c->isa_lazy) ensure_isa(c);
        if (c->max_lcp < 0) c->max_lcp = max_lcp(c, n);
        const long long cnt = hi - lo;
        // raw slots that can cover [lo, hi): a slot i < lo reaches lo only if
        // raw[i] > lo - i, and raw[i] <= max LCP (Lemma 1)
        const long long first = std::max(1ll, lo - c->max_lcp);
        {
            Stage st(c, RS_STAGE_RAW_LLR);
            used[RS_STAGE_RAW_LLR] = true;
            // SA order (one read of SA/LCP + a bucketed scatter of the shard's
            // slots) beats two random LCP gathers per slot once the shard is a
            // sizeable part of the text (measured at 256 Mi: ~0.45 ms + 2.8 ms x
            // shard fraction vs 5.8 ms x shard fraction)
            const long long span = hi - std::max(0ll, first - 1);
            const bool sa_order = c->have_sa && (c->sa_device_built || c->sa_isa_consistent) && 6 * span >= n;
            if (cnt > 0 && sa_order) {
                raw_from_sa_lcp_range(c, n, raw_slots(n), std::max(1ll, first - 1), hi - 1);
            } else if (cnt > 0) {
                raw_from_rank_lcp_range(c, n, std::max(0ll, first - 1), hi - 1);
            }
        }
        {
            Stage st(c, RS_STAGE_QUERY);
            used[RS_STAGE_QUERY] = true;
            long long *o1 = (long long *)buf(c, B_OUT1, 8 * (size_t)(cnt + 2));
            buf(c, B_OUT0, 8 * (size_t)(cnt + 1));
            RS_CUDA(cudaMemsetAsync(o1, 0, 8, c->stream));
            c->total = 0;
            c->out_ref_layout = false;
            const unsigned *raw = (const unsigned *)c->bufs[B_RAW].p;
            if (cnt > 0 && !query_range(c, mode, RS_PATH_COMPACT, nullptr, 0, raw, lo, hi - 1, 0, cnt, first))
                query_range(c, mode, RS_PATH_RAW, nullptr, 0, raw, lo, hi - 1, 0, cnt, first);
            c->out_mode = mode;
        }
        collect_stages(c, used);
        c->have_raw = c->have_compact = false;  // B_RAW holds only the shard's slots
        c->shard_lo = lo;
        c->shard_hi = hi;
        if (total) *total = mode == RS_MODE_ALL ? c->total : 0;
    });
}

int rs_shard_rebase(rs_ctx *c, int64_t base) {
    return guarded(c, [&] {
        if (c->out_mode != RS_MODE_ALL) fail(RS_ESTATE, "no all-ties shard results on device");
        long long cnt = c->shard_hi - c->shard_lo;
        add_i64(c, (long long *)c->bufs[B_OUT1].p, cnt + 1, base);
        RS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int rs_fetch_shard(rs_ctx *c, int mode, int64_t *a, int64_t *b, int64_t *flat) {
    return guarded(c, [&] {
        if (c->out_mode != mode) fail(RS_ESTATE, "no shard results of this mode on device");
        long long cnt = c->shard_hi - c->shard_lo;
        const long long *o0 = (const long long *)c->bufs[B_OUT0].p, *o1 = (const long long *)c->bufs[B_OUT1].p;
        if (mode == RS_MODE_ALL) {
            if (fetch_csr_bytes(c, o0, o1, (const long long *)c->bufs[B_FLAT].p, cnt, c->total, (long long *)a,
                                (long long *)b, (long long *)flat))
                return;
            if (fetch_csr_mixed(c, o0, o1, (const long long *)c->bufs[B_FLAT].p, cnt, c->total, (long long *)a,
                                (long long *)b, (long long *)flat))
                return;
            fetch_i64(c, (long long *)a, o0, cnt, 0);
            fetch_i64(c, (long long *)b, o1, cnt + 1, 2);
            fetch_i64(c, (long long *)flat, (const long long *)c->bufs[B_FLAT].p, c->total, 0);
        } else {
            if (fetch_leftmost_bytes(c, o0, o1, cnt, c->shard_lo, (long long *)a, (long long *)b)) return;
            if (fetch_leftmost_mixed(c, o0, o1, cnt, c->shard_lo, (long long *)a, (long long *)b)) return;
            fetch_i64(c, (long long *)a, o0, cnt, 1);
            fetch_i64(c, (long long *)b, o1, cnt, 0);
        }
    });
}

// ---- NCCL inside the library (collectives.cu) ---------------------------------------

int rs_nccl_unique_id(uint8_t *id) {
    if (!id) return RS_EINVAL;
    try {
        nccl_unique_id(id);
        return RS_OK;
    } catch (const RsError &e) {
        fprintf(stderr, "rs_nccl_unique_id: %s\n", e.msg.c_str());
        return e.code;
    }
}

int rs_nccl_init(rs_ctx *c, const uint8_t *id, int32_t rank, int32_t world) {
    return guarded(c, [&] {
        if (!id) fail(RS_EINVAL, "null NCCL id");
        nccl_init(c, id, rank, world);
    });
}

int rs_nccl_destroy(rs_ctx *c) {
    return guarded(c, [&] { nccl_destroy(c); });
}

int rs_nccl_broadcast_text(rs_ctx *c, int64_t n, int32_t root) {
    return guarded(c, [&] {
        check_n(n);
        nccl_broadcast_text(c, n, root);
        invalidate(c);
        c->n = n;
        c->have_text = true;
    });
}

int rs_nccl_allgather_i64(rs_ctx *c, int64_t value, int64_t *out) {
    return guarded(c, [&] { nccl_allgather_i64(c, value, (long long *)out); });
}

int rs_set_text_device(rs_ctx *c, int64_t n) {
    return guarded(c, [&] {
        check_n(n);
        if (c->bufs[B_TEXT].cap < (size_t)n + 128) fail(RS_ESTATE, "text buffer too small (rs_device_buffer(RS_BUF_TEXT))");
        unsigned char *d = (unsigned char *)c->bufs[B_TEXT].p;
        invalidate(c);
        RS_CUDA(cudaMemsetAsync(d + n, 0, 128, c->stream));
        RS_CUDA(cudaStreamSynchronize(c->stream));
        c->n = n;
        c->have_text = true;
    });
}

int rs_dist_sort(rs_ctx *c, int32_t rank, int32_t world, int64_t *info) {
    return guarded(c, [&] {
        if (!c->have_text) fail(RS_ESTATE, "no text loaded");
        if (!info) fail(RS_EINVAL, "info is required");
        long long tmp[16];
        dist_sort(c, c->n, rank, world, tmp);
        for (int i = 0; i < 16; ++i) info[i] = tmp[i];
    });
}

int rs_dist_update(rs_ctx *c, int32_t rank, int32_t world, const int64_t *nbr, int64_t *send_counts,
                   int64_t *info) {
    return guarded(c, [&] {
        if (!nbr || !send_counts || !info || world < 1) fail(RS_EINVAL, "bad arguments");
        long long nb[6], tmp[16];
        for (int i = 0; i < 6; ++i) nb[i] = nbr[i];
        std::vector<long long> sc((size_t)world, 0);
        dist_update(c, c->n, rank, world, nb, sc.data(), tmp);
        for (int q = 0; q < world; ++q) send_counts[q] = sc[(size_t)q];
        for (int i = 0; i < 16; ++i) info[i] = tmp[i];
    });
}

int rs_dist_apply(rs_ctx *c, int32_t rank, int32_t world, const void *recv, int64_t count, int64_t halo_cap,
                  int64_t *info) {
    return guarded(c, [&] {
        if ((count > 0 && !recv) || !info || count < 0 || halo_cap < 8) fail(RS_EINVAL, "bad arguments");
        long long tmp[16];
        dist_apply(c, c->n, rank, world, recv, count, halo_cap, tmp);
        for (int i = 0; i < 16; ++i) info[i] = tmp[i];
    });
}

int rs_dist_scan(rs_ctx *c, int mode, int64_t halo, int64_t *total) {
    return guarded(c, [&] {
        if (mode != RS_MODE_LEFTMOST && mode != RS_MODE_ALL) fail(RS_EINVAL, "unknown mode");
        if (!total) fail(RS_EINVAL, "total is required");
        bool used[RS_NUM_STAGES] = {};
        long long t = 0;
        {
            Stage st(c, RS_STAGE_QUERY);
            used[RS_STAGE_QUERY] = true;
            dist_scan(c, c->n, mode, halo, &t);
        }
        collect_stages(c, used);
        *total = t;
    });
}

}  // extern "C"
