// Dev microbenchmark: achievable HBM bandwidth for 256-byte warp stores in
// different address patterns (sequential / random / region-local) with and
// without a random 256-byte read stream.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE, bool READS>
__global__ void k(double* out, const double* in, int64_t nchunks, int64_t nin, int per_warp) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0;
    for (int64_t base = w * per_warp; base < nchunks; base += nw * per_warp) {
        for (int t = 0; t < per_warp; ++t) {
            int64_t c;
            if (MODE == 0) c = base + t;                                   // sequential
            else if (MODE == 1) c = hash32((uint32_t)(base + t)) % nchunks;   // random
            else c = (base & ~1023ll) + (hash32((uint32_t)(base + t)) & 1023);  // 256 KB windows
            if (c >= nchunks) c = nchunks - 1;
            if (READS && (t & 3) == 0) acc += __ldg(in + (int64_t)(hash32((uint32_t)(base * 7 + t)) % nin) * 32 + lane);
            __stcs(out + c * 32 + lane, acc + 1.0);
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    const int64_t bytes = 2283ll << 20, nchunks = bytes / 256;
    const int64_t nin = (300ll << 20) / 256;
    double *out, *in;
    cudaMalloc(&out, bytes);
    cudaMalloc(&in, nin * 256);
    cudaMemset(in, 0, nin * 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, const char* name) {
        for (int r = 0; r < 3; ++r) kern<<<148 * 8, 256>>>(out, in, nchunks, nin, 16);
        cudaEventRecord(a);
        kern<<<148 * 8, 256>>>(out, in, nchunks, nin, 16);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %.3f ms  %.0f GB/s (writes)\n", name, ms, bytes / ms / 1e6);
    };
    run(k<0, false>, "seq writes");
    run(k<1, false>, "random writes");
    run(k<2, false>, "window writes");
    run(k<0, true>, "seq writes + rand reads");
    run(k<1, true>, "random writes + rand reads");
    run(k<2, true>, "window writes + rand reads");
    return 0;
}
