// Micro test (dev tool): TMA tile::gather4 of 256-byte fp64 rows on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 gather4.cu -o gather4
// 1. correctness: gather 4 arbitrary rows of a [R x 32] fp64 tensor into
//    shared memory through one mbarrier, compare;
// 2. throughput: every warp gathers random row quads (double-buffered) and
//    reduces them, against the same with per-lane 16-byte cp.async.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__);     \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(m)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, int bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, int parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(su32(m)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* m, int r0,
                                        int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst)),
        "l"(tm), "r"(su32(m)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

__global__ void k_check(const __grid_constant__ CUtensorMap tm, const int* rows, double* out) {
    __shared__ __align__(1024) double buf[4 * 32];
    __shared__ uint64_t mb;
    if (threadIdx.x == 0) {
        mbar_init(&mb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect(&mb, 4 * 256);
        gather4(buf, &tm, &mb, rows[0], rows[1], rows[2], rows[3]);
    }
    mbar_wait(&mb, 0);
    for (int k = threadIdx.x; k < 128; k += blockDim.x) out[k] = buf[k];
}

// throughput: W warps per CTA, each loops over `iters` random quads
template <bool TMA>
__global__ void __launch_bounds__(768, 1) k_tput(const __grid_constant__ CUtensorMap tm,
                                                  const double* base, const int* rows, int nq,
                                                  double* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t mb[24][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* slot[2] = {reinterpret_cast<double*>(sm + warp * 2048),
                       reinterpret_cast<double*>(sm + warp * 2048 + 1024)};
    if (lane == 0) {
        mbar_init(&mb[warp][0], 1);
        mbar_init(&mb[warp][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int gw = blockIdx.x * 24 + warp, nw = gridDim.x * 24;
    double acc = 0.0;
    auto issue = [&](int q, int s) {
        if (TMA) {
            if (lane == 0) {
                const int4 r = reinterpret_cast<const int4*>(rows)[q];
                mbar_expect(&mb[warp][s], 1024);
                gather4(slot[s], &tm, &mb[warp][s], r.x, r.y, r.z, r.w);
            }
        } else {
            const int4 r = reinterpret_cast<const int4*>(rows)[q];
            const int half = lane >> 4, ch = lane & 15;
            for (int p = 0; p < 2; ++p) {
                const int rr = 2 * p + half;
                const int row = rr == 0 ? r.x : rr == 1 ? r.y : rr == 2 ? r.z : r.w;
                const uint32_t dst = su32(slot[s]) + rr * 256 + ch * 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                             "l"(base + (size_t)row * 32 + ch * 2)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
    int k = 0;
    issue(gw, 0);
    for (int q = gw; q < nq; q += nw, ++k) {
        const int s = k & 1;
        if (q + nw < nq) issue(q + nw, s ^ 1);
        else if (!TMA) asm volatile("cp.async.commit_group;" ::: "memory");
        if (TMA) mbar_wait(&mb[warp][s], (k >> 1) & 1);
        else asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        for (int rr = 0; rr < 4; ++rr) acc += slot[s][rr * 32 + lane];
        __syncwarp();
    }
    if (acc == 12345.678) sink[0] = acc;
}

int main() {
    const int R = 1 << 21;   // 512 MB
    double* d;
    CK(cudaMalloc(&d, (size_t)R * 256));
    std::vector<double> h((size_t)R * 32);
    for (size_t r = 0; r < (size_t)R; ++r)
        for (int c = 0; c < 32; ++c) h[r * 32 + c] = r * 100.0 + c;
    CK(cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {32, (cuuint64_t)R};
    cuuint64_t gstr[1] = {256};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, gdim, gstr, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)cr);
    if (cr) return 1;

    int hr[4] = {7, 1234567, 3, 2097151};
    int* dr;
    double* dout;
    CK(cudaMalloc(&dr, 64 << 20));
    CK(cudaMalloc(&dout, 128 * 8));
    CK(cudaMemcpy(dr, hr, 16, cudaMemcpyHostToDevice));
    k_check<<<1, 128>>>(tm, dr, dout);
    CK(cudaDeviceSynchronize());
    double ho[128];
    CK(cudaMemcpy(ho, dout, 128 * 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int rr = 0; rr < 4; ++rr)
        for (int c = 0; c < 32; ++c) bad += ho[rr * 32 + c] != hr[rr] * 100.0 + c;
    printf("gather4 check: %s\n", bad ? "FAIL" : "ok");

    const int nq = 4 << 20;   // quads
    std::vector<int> rows((size_t)nq * 4);
    srand(1);
    for (auto& x : rows) x = (int)(((unsigned)rand() * 2654435761u) % (unsigned)R);
    CK(cudaMemcpy(dr, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t smem = 24 * 2048;
    CK(cudaFuncSetAttribute(k_tput<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_tput<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep)
        for (int t = 0; t < 2; ++t) {
            cudaEventRecord(a);
            if (t) k_tput<true><<<sms, 768, smem>>>(tm, d, dr, nq, dout);
            else k_tput<false><<<sms, 768, smem>>>(tm, d, dr, nq, dout);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s: %.3f ms  %.0f GB/s\n", t ? "tma gather4" : "cp.async  ", ms,
                   (double)nq * 1024 / ms / 1e6);
        }
    return 0;
}
