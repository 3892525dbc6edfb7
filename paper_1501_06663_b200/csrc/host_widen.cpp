// host_widen.cpp -- the host side of csrc/host_io.cu's transfer pipeline:
// 32-bit wire words -> int64 output values, written with non-temporal
// (streaming) stores.
//
// The destination arrays are far larger than the caches and written once, so
// ordinary stores make every written line a read-for-ownership first: 8 more
// bytes of host memory traffic per value on top of the 4 read + 8 written.
// The transfer is bound by the host's memory bandwidth (tools/exp_fetch.py),
// so streaming stores (AVX2 _mm256_stream_si256, no RFO) cut its traffic by a
// third.  Portable scalar loop when the CPU lacks AVX2.
#include <immintrin.h>

#include <cstdint>
#include <cstring>

namespace rsb {

namespace {

// mode 0: zero-extend, 1: sign-extend, 2: zero-extend of (w - w0)
template <int MODE>
inline long long scalar_one(unsigned w, unsigned w0, long long add) {
    if (MODE == 1) return (long long)(int)w + add;
    if (MODE == 2) return (long long)(unsigned)(w - w0) + add;
    return (long long)w + add;
}

template <int MODE>
__attribute__((target("avx2"))) void widen_avx2(const unsigned *w, long long *out, long long x, long long y,
                                                  unsigned w0, long long add) {
    long long j = x;
    while (j < y && (reinterpret_cast<uintptr_t>(out + j) & 31)) {
        out[j] = scalar_one<MODE>(w[j], w0, add);
        ++j;
    }
    const __m256i vadd = _mm256_set1_epi64x(add);
    const __m128i vw0 = _mm_set1_epi32((int)w0);
    for (; j + 8 <= y; j += 8) {
        __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + j));
        __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + j + 4));
        if (MODE == 2) {
            a = _mm_sub_epi32(a, vw0);
            b = _mm_sub_epi32(b, vw0);
        }
        __m256i ea = MODE == 1 ? _mm256_cvtepi32_epi64(a) : _mm256_cvtepu32_epi64(a);
        __m256i eb = MODE == 1 ? _mm256_cvtepi32_epi64(b) : _mm256_cvtepu32_epi64(b);
        ea = _mm256_add_epi64(ea, vadd);
        eb = _mm256_add_epi64(eb, vadd);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j), ea);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j + 4), eb);
    }
    for (; j < y; ++j) out[j] = scalar_one<MODE>(w[j], w0, add);
    _mm_sfence();
}

template <int MODE>
void widen_scalar(const unsigned *w, long long *out, long long x, long long y, unsigned w0, long long add) {
    for (long long j = x; j < y; ++j) out[j] = scalar_one<MODE>(w[j], w0, add);
}

bool have_avx2() {
    static const bool ok = __builtin_cpu_supports("avx2");
    return ok;
}

}  // namespace

// out[j] = f(w[j]) + add for j in [x, y)
void widen_words(const unsigned *w, long long *out, long long x, long long y, int mode, unsigned w0,
                 long long add) {
    if (y <= x) return;
    if (have_avx2()) {
        if (mode == 1) widen_avx2<1>(w, out, x, y, w0, add);
        else if (mode == 2) widen_avx2<2>(w, out, x, y, w0, add);
        else widen_avx2<0>(w, out, x, y, w0, add);
        return;
    }
    if (mode == 1) widen_scalar<1>(w, out, x, y, w0, add);
    else if (mode == 2) widen_scalar<2>(w, out, x, y, w0, add);
    else widen_scalar<0>(w, out, x, y, w0, add);
}

// ---- byte wire decoders (host_io.cu fetch_all_bytes) ----------------------

// out[j] = w[j] for j in [x, y)
__attribute__((target("avx2"))) static void widen_u8_avx2(const unsigned char *w, long long *out, long long x,
                                                           long long y) {
    long long j = x;
    while (j < y && (reinterpret_cast<uintptr_t>(out + j) & 31)) {
        out[j] = w[j];
        ++j;
    }
    for (; j + 16 <= y; j += 16) {
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(w + j));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j), _mm256_cvtepu8_epi64(b));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j + 4), _mm256_cvtepu8_epi64(_mm_srli_si128(b, 4)));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j + 8), _mm256_cvtepu8_epi64(_mm_srli_si128(b, 8)));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j + 12), _mm256_cvtepu8_epi64(_mm_srli_si128(b, 12)));
    }
    for (; j < y; ++j) out[j] = w[j];
    _mm_sfence();
}

void widen_bytes(const unsigned char *w, long long *out, long long x, long long y) {
    if (y <= x) return;
    if (have_avx2()) {
        widen_u8_avx2(w, out, x, y);
        return;
    }
    for (long long j = x; j < y; ++j) out[j] = w[j];
}

// Running sums: out[j] = start + w[x] + ... + w[j] (SIGNED: w as int8).
// 8 values per step: an in-register prefix over 32-bit lanes (relative to the
// step's carry-in; a step adds at most 8 * 255), widened to int64 and stored
// with streaming stores.
template <bool SIGNED>
__attribute__((target("avx2"))) static void prefix_avx2(const unsigned char *w, long long *out, long long x,
                                                        long long y, long long run) {
    long long j = x;
    while (j < y && (reinterpret_cast<uintptr_t>(out + j) & 31)) {
        run += SIGNED ? (long long)(signed char)w[j] : (long long)w[j];
        out[j] = run;
        ++j;
    }
    for (; j + 8 <= y; j += 8) {
        const __m128i b = _mm_loadl_epi64(reinterpret_cast<const __m128i *>(w + j));
        __m256i v = SIGNED ? _mm256_cvtepi8_epi32(b) : _mm256_cvtepu8_epi32(b);
        v = _mm256_add_epi32(v, _mm256_slli_si256(v, 4));  // prefix within each 128-bit half
        v = _mm256_add_epi32(v, _mm256_slli_si256(v, 8));
        const __m256i lowtot = _mm256_permutevar8x32_epi32(v, _mm256_set1_epi32(3));
        v = _mm256_add_epi32(v, _mm256_blend_epi32(_mm256_setzero_si256(), lowtot, 0xF0));
        const __m256i base = _mm256_set1_epi64x(run);
        const __m256i lo = _mm256_add_epi64(base, _mm256_cvtepi32_epi64(_mm256_castsi256_si128(v)));
        const __m256i hi = _mm256_add_epi64(base, _mm256_cvtepi32_epi64(_mm256_extracti128_si256(v, 1)));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j), lo);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(out + j + 4), hi);
        run += (long long)_mm256_extract_epi32(v, 7);
    }
    for (; j < y; ++j) {
        run += SIGNED ? (long long)(signed char)w[j] : (long long)w[j];
        out[j] = run;
    }
    _mm_sfence();
}

void prefix_bytes(const unsigned char *w, long long *out, long long x, long long y, long long start, bool is_signed) {
    if (y <= x) return;
    if (have_avx2()) {
        if (is_signed) prefix_avx2<true>(w, out, x, y, start);
        else prefix_avx2<false>(w, out, x, y, start);
        return;
    }
    long long run = start;
    for (long long j = x; j < y; ++j) {
        run += is_signed ? (long long)(signed char)w[j] : (long long)w[j];
        out[j] = run;
    }
}

// Leftmost answers from (length, distance) byte pairs: lengths[j] = w[2j],
// starts[j] = pos_x + j - w[2j+1] (or -1 when the length is 0), j in [x, y).
__attribute__((target("avx2"))) static void leftmost_avx2(const unsigned char *w, long long *starts,
                                                          long long *lengths, long long x, long long y,
                                                          long long pos_x) {
    long long j = x;
    auto one = [&](long long i) {
        const unsigned L = w[2 * i], d = w[2 * i + 1];
        lengths[i] = L;
        starts[i] = L ? pos_x + (i - x) - (long long)d : -1ll;
    };
    while (j < y && ((reinterpret_cast<uintptr_t>(starts + j) | reinterpret_cast<uintptr_t>(lengths + j)) & 31)) one(j++);
    const __m256i step = _mm256_set_epi64x(3, 2, 1, 0), minus1 = _mm256_set1_epi64x(-1);
    const __m128i lo_mask = _mm_set1_epi16(0x00ff);
    for (; j + 4 <= y; j += 4) {
        const __m128i p = _mm_loadl_epi64(reinterpret_cast<const __m128i *>(w + 2 * j));  // 4 pairs
        const __m128i len16 = _mm_and_si128(p, lo_mask), d16 = _mm_srli_epi16(p, 8);
        const __m256i L = _mm256_cvtepu16_epi64(len16), D = _mm256_cvtepu16_epi64(d16);
        const __m256i pos = _mm256_add_epi64(_mm256_set1_epi64x(pos_x + (j - x)), step);
        const __m256i st = _mm256_sub_epi64(pos, D);
        const __m256i none = _mm256_cmpeq_epi64(L, _mm256_setzero_si256());
        _mm256_stream_si256(reinterpret_cast<__m256i *>(lengths + j), L);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(starts + j), _mm256_blendv_epi8(st, minus1, none));
    }
    for (; j < y; ++j) one(j);
    _mm_sfence();
}

void leftmost_pairs(const unsigned char *w, long long *starts, long long *lengths, long long x, long long y,
                    long long pos_x) {
    if (y <= x) return;
    if (have_avx2()) {
        leftmost_avx2(w, starts, lengths, x, y, pos_x);
        return;
    }
    for (long long j = x; j < y; ++j) {
        const unsigned L = w[2 * j], d = w[2 * j + 1];
        lengths[j] = L;
        starts[j] = L ? pos_x + (j - x) - (long long)d : -1ll;
    }
}

// One block of the mixed-width wire: `count` values of `width` bytes.
// mode 0: out[j] = w[j]; mode 1: out[j] = start + w[0] + ... + w[j];
// mode 2: the same with signed steps.
template <typename U, typename S>
static void decode_wide(const unsigned char *w, int mode, long long *out, long long count, long long start) {
    const U *u = reinterpret_cast<const U *>(w);
    long long run = start;
    for (long long j = 0; j < count; ++j) {
        U v;
        std::memcpy(&v, u + j, sizeof(U));
        long long x = mode == 2 ? (long long)(S)v : (long long)v;
        if (mode == 0) {
            _mm_stream_si64(reinterpret_cast<long long *>(out + j), x);
        } else {
            run += x;
            _mm_stream_si64(reinterpret_cast<long long *>(out + j), run);
        }
    }
    _mm_sfence();
}

void decode_block(const unsigned char *w, int width, int mode, long long *out, long long count, long long start) {
    if (count <= 0) return;
    if (width == 1) {
        if (mode == 0) widen_bytes(w, out, 0, count);
        else prefix_bytes(w, out, 0, count, start, mode == 2);
    } else if (width == 2) {
        decode_wide<unsigned short, short>(w, mode, out, count, start);
    } else {
        decode_wide<unsigned, int>(w, mode, out, count, start);
    }
}

// One leftmost block of the mixed-width wire: `count` lengths then `count`
// position - start values, `width` bytes each; slot j answers position pos0 + j.
template <typename U>
static void decode_left_wide(const unsigned char *w, long long count, long long pos0, long long *starts,
                             long long *lengths) {
    const U *l = reinterpret_cast<const U *>(w), *d = l + count;
    for (long long j = 0; j < count; ++j) {
        U lv, dv;
        std::memcpy(&lv, l + j, sizeof(U));
        std::memcpy(&dv, d + j, sizeof(U));
        _mm_stream_si64(reinterpret_cast<long long *>(lengths + j), (long long)lv);
        _mm_stream_si64(reinterpret_cast<long long *>(starts + j), lv ? pos0 + j - (long long)dv : -1ll);
    }
    _mm_sfence();
}

void decode_left_block(const unsigned char *w, int width, long long count, long long pos0, long long *starts,
                       long long *lengths) {
    if (count <= 0) return;
    if (width == 1) decode_left_wide<unsigned char>(w, count, pos0, starts, lengths);
    else if (width == 2) decode_left_wide<unsigned short>(w, count, pos0, starts, lengths);
    else decode_left_wide<unsigned>(w, count, pos0, starts, lengths);
}

// ---- H2D narrowing (host_io.cu put_i64_as_u32) ------------------------------

// w[j] = in[j] + add for j in [x, y); false if some in[j] lies outside [lo, hi]
__attribute__((target("avx2"))) static bool narrow_avx2(const long long *in, unsigned *w, long long x, long long y,
                                                        long long lo, long long hi, long long add) {
    long long j = x;
    bool ok = true;
    while (j < y && (reinterpret_cast<uintptr_t>(w + j) & 31)) {
        const long long v = in[j];
        ok &= (v >= lo) & (v <= hi);
        w[j] = (unsigned)(v + add);
        ++j;
    }
    const __m256i vlo = _mm256_set1_epi64x(lo), vhi = _mm256_set1_epi64x(hi), vadd = _mm256_set1_epi64x(add);
    const __m256i pick = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    __m256i badv = _mm256_setzero_si256();
    for (; j + 8 <= y; j += 8) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(in + j));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(in + j + 4));
        // lo > v or v > hi: out of range
        badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(vlo, a), _mm256_cmpgt_epi64(a, vhi)));
        badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(vlo, b), _mm256_cmpgt_epi64(b, vhi)));
        const __m256i pa = _mm256_permutevar8x32_epi32(_mm256_add_epi64(a, vadd), pick);  // low words in lanes 0-3
        const __m256i pb = _mm256_permutevar8x32_epi32(_mm256_add_epi64(b, vadd), pick);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(w + j), _mm256_permute2x128_si256(pa, pb, 0x20));
    }
    ok &= _mm256_testz_si256(badv, badv) != 0;
    for (; j < y; ++j) {
        const long long v = in[j];
        ok &= (v >= lo) & (v <= hi);
        w[j] = (unsigned)(v + add);
    }
    _mm_sfence();
    return ok;
}

bool narrow_words(const long long *in, unsigned *w, long long x, long long y, long long lo, long long hi,
                  long long add) {
    if (y <= x) return true;
    if (have_avx2()) return narrow_avx2(in, w, x, y, lo, hi, add);
    bool ok = true;
    for (long long j = x; j < y; ++j) {
        const long long v = in[j];
        ok &= (v >= lo) & (v <= hi);
        w[j] = (unsigned)(v + add);
    }
    return ok;
}

// b[j] = in[j] for j in [x, y) when every value lies in [0, 255]; returns
// 0 if so, 1 if some value is outside [lo, hi] (an error), 2 if all are in
// [lo, hi] but some exceeds a byte (send 32-bit words instead)
int narrow_bytes(const long long *in, unsigned char *b, long long x, long long y, long long lo, long long hi) {
    unsigned long long big = 0;
    bool ok = true;
    for (long long j = x; j < y; ++j) {
        const long long v = in[j];
        ok &= (v >= lo) & (v <= hi);
        big |= (unsigned long long)v;
        b[j] = (unsigned char)v;
    }
    if (!ok) return 1;
    return big > 255ull ? 2 : 0;
}

}  // namespace rsb
