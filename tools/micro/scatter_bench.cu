// Micro-benchmark: the apply phase of the bucketed permutation scatter
// (csrc/scatter.cu k_bucket_apply) against alternatives, on a random
// permutation of 2^28 u32 values (the C3 raw-LLR scatter size).
//
//   A<NT,IPT>  current scheme: 256 coarse buckets (2^20 slots, 4 MB of out),
//              each block stores 4096 staged (dest, val) pairs straight to out
//   S<FINE>    fine buckets of 2^FINE slots: a block loads one fine bucket's
//              pairs, scatters them into shared memory and writes the slot
//              range coalesced; needs a second partition pass (timed as P)
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_bench scatter_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int LOGN = 28;
constexpr long long N = 1ll << LOGN;

__device__ __forceinline__ unsigned perm(unsigned i) {  // bijection on [0, 2^28)
    const unsigned m = (1u << LOGN) - 1;
    i = (i * 2654435761u) & m;
    i ^= i >> 13;
    i = (i * 0x2545F491u) & m;
    i ^= i >> 11;
    return i & m;
}

// untimed setup: pairs grouped by bucket of 2^shift slots (counting sort)
__global__ void k_count(unsigned *cnt, int shift) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < N) atomicAdd(&cnt[perm((unsigned)i) >> shift], 1u);
}
__global__ void k_place(uint2 *stage, unsigned *cur, int shift) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= N) return;
    unsigned d = perm((unsigned)i);
    unsigned p = atomicAdd(&cur[d >> shift], 1u);
    stage[p] = make_uint2(d, (unsigned)i);
}

template <int NT, int IPT>
__global__ void __launch_bounds__(NT) k_apply(const uint2 *__restrict__ stage, unsigned *__restrict__ out) {
    const long long base = (long long)blockIdx.x * NT * IPT;
    uint2 v[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) v[j] = __ldcs(stage + base + j * NT + threadIdx.x);
#pragma unroll
    for (int j = 0; j < IPT; ++j) out[v[j].x] = v[j].y;
}

// one fine bucket (2^FINE slots, pairs stage[beg[b], beg[b+1])) per block
template <int FINE, int NT>
__global__ void __launch_bounds__(NT) k_apply_smem(const uint2 *__restrict__ stage, const unsigned *__restrict__ beg,
                                                   unsigned *__restrict__ out) {
    extern __shared__ unsigned s[];
    const unsigned b = blockIdx.x, a0 = beg[b], a1 = beg[b + 1];
    for (unsigned i = a0 + threadIdx.x; i < a1; i += NT) {
        const uint2 v = __ldcs(stage + i);
        s[v.x & ((1u << FINE) - 1)] = v.y;
    }
    __syncthreads();
    uint4 *o = reinterpret_cast<uint4 *>(out + ((long long)b << FINE));
    const uint4 *si = reinterpret_cast<const uint4 *>(s);
    for (int i = threadIdx.x; i < (1 << FINE) / 4; i += NT) __stcs(o + i, si[i]);
}

// the extra partition pass of the fine scheme: read 8 B + write 8 B per pair
__global__ void k_copy_pairs(const uint2 *__restrict__ a, uint2 *__restrict__ b) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < N) b[i] = __ldcs(a + i);
}

__global__ void k_check(const unsigned *out, unsigned long long *bad) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < N && perm(out[i]) != (unsigned)i) atomicAdd(bad, 1ull);
}

template <typename F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    uint2 *stage, *stage2;
    unsigned *out, *cnt;
    unsigned long long *bad;
    CK(cudaMalloc(&stage, 8 * N));
    CK(cudaMalloc(&stage2, 8 * N));
    CK(cudaMalloc(&out, 4 * N));
    CK(cudaMalloc(&cnt, 4 * ((1 << 16) + 1)));
    CK(cudaMalloc(&bad, 8));
    const int blocks = (int)(N / 256);
    auto check = [&](const char *name, float ms) {
        CK(cudaMemset(bad, 0, 8));
        k_check<<<blocks, 256>>>(out, bad);
        unsigned long long h;
        CK(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost));
        printf("%-28s %7.3f ms  %6.0f GB/s (12 B/pair)  %s\n", name, ms, 12.0 * N / ms / 1e6, h ? "WRONG" : "ok");
    };
    auto group = [&](int shift, std::vector<unsigned> &beg) {
        const int nb = (int)(N >> shift);
        CK(cudaMemset(cnt, 0, 4 * (nb + 1)));
        k_count<<<blocks, 256>>>(cnt, shift);
        std::vector<unsigned> h(nb);
        CK(cudaMemcpy(h.data(), cnt, 4 * nb, cudaMemcpyDeviceToHost));
        beg.assign(nb + 1, 0);
        for (int b = 0; b < nb; ++b) beg[b + 1] = beg[b] + h[b];
        CK(cudaMemcpy(cnt, beg.data(), 4 * nb, cudaMemcpyHostToDevice));
        k_place<<<blocks, 256>>>(stage, cnt, shift);
        CK(cudaDeviceSynchronize());
    };
    std::vector<unsigned> beg;
    group(20, beg);
    check("A<256,16> (current)", timeit([&] { k_apply<256, 16><<<(unsigned)(N / 4096), 256>>>(stage, out); }));
    check("A<256,8>", timeit([&] { k_apply<256, 8><<<(unsigned)(N / 2048), 256>>>(stage, out); }));
    check("A<256,4>", timeit([&] { k_apply<256, 4><<<(unsigned)(N / 1024), 256>>>(stage, out); }));
    check("A<512,8>", timeit([&] { k_apply<512, 8><<<(unsigned)(N / 4096), 512>>>(stage, out); }));
    check("A<128,16>", timeit([&] { k_apply<128, 16><<<(unsigned)(N / 2048), 128>>>(stage, out); }));
    check("A<256,32>", timeit([&] { k_apply<256, 32><<<(unsigned)(N / 8192), 256>>>(stage, out); }));
    float pcopy = timeit([&] { k_copy_pairs<<<blocks, 256>>>(stage, stage2); });
    printf("%-28s %7.3f ms  (partition-pass traffic stand-in)\n", "P copy pairs", pcopy);
    {
        group(14, beg);
        unsigned *dbeg;
        CK(cudaMalloc(&dbeg, 4 * beg.size()));
        CK(cudaMemcpy(dbeg, beg.data(), 4 * beg.size(), cudaMemcpyHostToDevice));
        CK(cudaFuncSetAttribute(k_apply_smem<14, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << 14));
        check("S<14> (64 KB smem, 512 thr)", timeit([&] {
                  k_apply_smem<14, 512><<<(unsigned)(N >> 14), 512, 4 << 14>>>(stage, dbeg, out);
              }));
        group(15, beg);
        CK(cudaMemcpy(dbeg, beg.data(), 4 * beg.size(), cudaMemcpyHostToDevice));
        CK(cudaFuncSetAttribute(k_apply_smem<15, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << 15));
        check("S<15> (128 KB smem, 1024 thr)", timeit([&] {
                  k_apply_smem<15, 1024><<<(unsigned)(N >> 15), 1024, 4 << 15>>>(stage, dbeg, out);
              }));
    }
    return 0;
}
