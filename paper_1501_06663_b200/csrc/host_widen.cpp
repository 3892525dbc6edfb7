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

}  // namespace rsb
