// tsv.cu -- the reference CLI's TSV wire format produced on device.
//
// Reference (cli.py:62-93):
//   leftmost line  "k\tstart\tlength\n"                 (start = -1 when none)
//   all-ties line  "k\ts1,L;s2,L;...\n", or "k\t-1,0\n"  when no repeat covers k
// Byte-identical output (pinned by tests against the reference's serialized
// digests).  Three steps over the positions [lo, hi] of the last query held on
// device (B_OUT0 / B_OUT1 / B_FLAT): line lengths -> inclusive scan -> every
// position formats its line at its offset.  The text never exists on the host
// until the one D2H copy.
#include "common.cuh"

namespace rsb {

void scan_i64(rs_ctx *c, const long long *d_in, long long count, long long *d_out);

namespace {

__device__ __forceinline__ int ndigits(long long v) {  // v >= 0
    int d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}

__device__ __forceinline__ int num_len(long long v) { return v < 0 ? 1 + ndigits(-v) : ndigits(v); }

// writes v at p, returns the byte count
__device__ __forceinline__ int put_num(unsigned char *p, long long v) {
    int len = num_len(v);
    int i = len;
    long long u = v < 0 ? -v : v;
    do {
        p[--i] = (unsigned char)('0' + u % 10);
        u /= 10;
    } while (u);
    if (v < 0) p[0] = '-';
    return len;
}

// MODE 0 leftmost: a = starts, b = lengths.  MODE 1 all: a = lengths, b = offsets, flat.
template <int MODE>
__global__ void k_line_len(const long long *__restrict__ a, const long long *__restrict__ b,
                           long long lo, long long hi, long long *__restrict__ len) {
    long long k = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k > hi) return;
    long long L = num_len(k) + 2;  // "k\t" ... "\n"
    if (MODE == 0) {
        L += num_len(a[k]) + 1 + num_len(b[k]);
    } else {
        const long long length = a[k];
        if (length == 0) {
            L += 4;  // "-1,0"
        } else {
            const long long t = b[k + 1] - b[k];
            // per tie "s,L" plus ';' separators; starts are summed in the write pass,
            // here their digits are counted from the flat array
            L += t * (1 + num_len(length)) + (t - 1);
        }
    }
    len[k - lo] = L;
}

// all mode needs the digits of every tie start: added separately
__global__ void k_line_len_ties(const long long *__restrict__ lengths, const long long *__restrict__ offsets,
                                const long long *__restrict__ flat, long long lo, long long hi,
                                long long *__restrict__ len) {
    long long k = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k > hi) return;
    if (lengths[k] == 0) return;
    long long s = 0;
    for (long long j = offsets[k]; j < offsets[k + 1]; ++j) s += num_len(flat[j]);
    len[k - lo] += s;
}

template <int MODE>
__global__ void k_write_lines(const long long *__restrict__ a, const long long *__restrict__ b,
                              const long long *__restrict__ flat, long long lo, long long hi,
                              const long long *__restrict__ end_incl, unsigned char *__restrict__ out) {
    long long k = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k > hi) return;
    const long long i = k - lo;
    unsigned char *p = out + (i ? end_incl[i - 1] : 0);
    p += put_num(p, k);
    *p++ = '\t';
    if (MODE == 0) {
        p += put_num(p, a[k]);
        *p++ = '\t';
        p += put_num(p, b[k]);
    } else {
        const long long length = a[k];
        if (length == 0) {
            p[0] = '-';
            p[1] = '1';
            p[2] = ',';
            p[3] = '0';
            p += 4;
        } else {
            for (long long j = b[k]; j < b[k + 1]; ++j) {
                if (j > b[k]) *p++ = ';';
                p += put_num(p, flat[j]);
                *p++ = ',';
                p += put_num(p, length);
            }
        }
    }
    *p = '\n';
}

}  // namespace

// Serialize positions [lo, hi] of the last query into B_T3 (bytes); returns the size.
long long serialize_tsv(rs_ctx *c, int mode, long long lo, long long hi) {
    if (hi < lo) return 0;
    const long long cnt = hi - lo + 1;
    const long long *a = (const long long *)c->bufs[B_OUT0].p;
    const long long *b = (const long long *)c->bufs[B_OUT1].p;
    const long long *flat = (const long long *)c->bufs[B_FLAT].p;
    long long *len = (long long *)buf(c, B_I64A, sizeof(long long) * (size_t)cnt);
    long long *incl = (long long *)buf(c, B_I64B, sizeof(long long) * (size_t)cnt);
    if (mode == RS_MODE_LEFTMOST) {
        RS_LAUNCH(c, k_line_len<0>, grid_for(cnt, 256), 256, 0, a, b, lo, hi, len);
    } else {
        RS_LAUNCH(c, k_line_len<1>, grid_for(cnt, 256), 256, 0, a, b, lo, hi, len);
        RS_LAUNCH(c, k_line_len_ties, grid_for(cnt, 256), 256, 0, a, b, flat, lo, hi, len);
    }
    scan_i64(c, len, cnt, incl);
    long long total = 0;
    fetch_small(c, &total, incl + cnt - 1, sizeof(total));
    unsigned char *out = (unsigned char *)buf(c, B_TSV, (size_t)total + 16);
    if (mode == RS_MODE_LEFTMOST)
        RS_LAUNCH_B(c, 16.0 * cnt + total, k_write_lines<0>, grid_for(cnt, 256), 256, 0, a, b, flat, lo, hi, incl,
                    out);
    else
        RS_LAUNCH_B(c, 16.0 * cnt + total, k_write_lines<1>, grid_for(cnt, 256), 256, 0, a, b, flat, lo, hi, incl,
                    out);
    c->tsv_bytes = total;
    return total;
}

}  // namespace rsb
