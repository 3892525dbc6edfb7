// Micro-benchmark: cost of warp peer-mask computation (MATCH.ANY vs ballots)
// as a function of the number of distinct values per warp.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned peer_bit(unsigned peers, unsigned x, unsigned bitmask) {
    unsigned r;
    asm("{\n .reg .pred p;\n .reg .b32 t, m, bal;\n"
        " and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n vote.sync.ballot.b32 bal, p, 0xffffffff;\n"
        " selp.b32 m, 0xffffffff, 0, p;\n xor.b32 t, bal, m;\n not.b32 t, t;\n and.b32 %0, %3, t;\n}"
        : "=r"(r) : "r"(x), "r"(bitmask), "r"(peers));
    return r;
}

template <int MODE>
__global__ void k(const unsigned *in, unsigned *out, int iters, unsigned mask) {
    unsigned lane = threadIdx.x & 31;
    unsigned d = in[(blockIdx.x * blockDim.x + threadIdx.x) & 1023] & mask;
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned x = (d + it * 0x9e3779b9u) & mask;  // new values each iteration, same #distinct
        unsigned peers;
        if (MODE == 0) {
            peers = __match_any_sync(0xffffffffu, x);
        } else if (MODE == 1) {
            peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                unsigned bal = __ballot_sync(0xffffffffu, (x >> b) & 1);
                peers &= bal ^ (((x >> b) & 1) - 1u);
            }
        } else if (MODE == 2) {
            peers = __match_any_sync(0xffffffffu, x & 15) & __match_any_sync(0xffffffffu, x >> 4);
        } else {
            peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; ++b) peers = peer_bit(peers, x, 1u << b);
        }
        acc += __popc(peers & ((1u << lane) - 1));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    unsigned *in, *out;
    cudaMalloc(&in, 1024 * 4);
    cudaMalloc(&out, 148 * 8 * 256 * 4);
    unsigned h[1024];
    unsigned s = 1;
    for (int i = 0; i < 1024; ++i) { s = s * 1664525u + 1013904223u; h[i] = s >> 8; }
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (unsigned mask : {0x0u, 0x3u, 0xfu, 0x3fu, 0xffu}) {
        for (int mode = 0; mode < 4; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) k<0><<<148 * 8, 256>>>(in, out, iters, mask);
                if (mode == 1) k<1><<<148 * 8, 256>>>(in, out, iters, mask);
                if (mode == 2) k<2><<<148 * 8, 256>>>(in, out, iters, mask);
                if (mode == 3) k<3><<<148 * 8, 256>>>(in, out, iters, mask);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                double per = ms * 1e-3 / (148.0 * 8 * 256 / 32 * iters) * 148 * 1.9e9;  // SM-cycles per warp-op
                if (rep) printf("mask %3x mode %d (%s): %.3f ms, %.2f SM-cycles per warp peer mask\n", mask, mode,
                                mode == 0 ? "match8" : mode == 1 ? "ballot8" : mode == 2 ? "match4x2" : "ballot8-lop3", ms, per);
            }
        }
    }
    return 0;
}
