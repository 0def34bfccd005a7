// Pipeline structure of the tensor-core tile kernel, isolated (no producers): one CTA per SM,
// one MMA thread, E epilogue warps draining NS TMEM stages of N columns each. Measures SM
// cycles per 128 x 256 candidates (one "tile") for
//   NS x N       : 2 x 256 (the kernel today), 4 x 128, 8 x 64
//   EPI          : 0 = packed 16-bit minimum tree (today), 1 = OR of the packed words (sign
//                  test after a threshold folded into the MMA), 2 = loads only
//   GROUPS       : epilogue warps per stage = E / GROUPS; warp group g drains stages s with
//                  s % GROUPS == g (GROUPS = 1: every warp takes a slice of every stage)
//   KT           : K = 32 KT int8 coordinates
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -I paper_2408_10743_b200/csrc -o tools/microbench/tc_pipe tools/microbench/tc_pipe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace sdb::tc;

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));    \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

constexpr int M = 128, NB = 256;  // B holds 256 rows; a stage uses N of them

__device__ __forceinline__ uint32_t idesc(int n) { return idesc_i8(M, n); }

template <int KT, int NS, int N, int E, int GROUPS, int EPI, int NA = 1, int NBT = 1>
__global__ void __launch_bounds__(32 * (1 + E), 1) pipe_bench(int T, long long *cycles, int *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[NS], empty[NS];
    __shared__ uint32_t tbase;
    constexpr int KB = 32 * KT;
    constexpr int WPS = E / GROUPS;          // warps per stage
    constexpr int QW = WPS / 4;              // warps per lane quarter and stage
    constexpr int COLS = N / QW;             // columns per warp and stage
    static_assert(COLS % 32 == 0, "a warp reads whole 32-column chunks");
    unsigned char *sA = sm, *sB = sm + NA * M * KB;  // NA A tiles, NBT B tiles (rotated like the kernel)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&tbase, 512);
    for (int i = threadIdx.x; i < (NA * M + NBT * NB) * KB; i += blockDim.x) sm[i] = (unsigned char)((i * 7 + 3) % 5 - 2);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], WPS);
        }
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    const int tiles = T * (NB / N);  // stages to run: T tiles of 128 x 256
    long long t0 = clock64();
    uint32_t acc = 0;
    if (warp == 0) {
        if (lane == 0) {
            const uint32_t id = idesc(N);
            for (int it = 0; it < tiles; it++) {
                const int s = it % NS;
                const uint32_t ph = (it / NS) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                fence_after();
                const int boff = (it % (NB / N)) * N;  // which N rows of B
                const int ta_ = (it / NBT) % NA, tb_ = it % NBT;  // like the kernel: a head tile meets NBT tail tiles
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    const uint64_t ad = sdesc(smem_u32(sA) + ta_ * M * KB + k * 2 * (M * 16), M * 16, 128);
                    const uint64_t bd = sdesc(smem_u32(sB) + tb_ * NB * KB + boff * 16 + k * 2 * (NB * 16), NB * 16, 128);
                    mma_i8(tb + s * N, ad, bd, id, k > 0);
                }
                commit(&full[s]);
            }
        }
    } else {
        const int e = warp - 1;
        const int grp = e / WPS, w = e % WPS;
        const int quarter = warp & 3;
        const int slice = w / 4;  // which column slice of the stage (warps e and e + 4 share a quarter)
        for (int it = grp; it < tiles; it += GROUPS) {
            const int s = it % NS;
            const uint32_t ph = (it / NS) & 1;
            mbar_wait(&full[s], ph);
            fence_after();
            const uint32_t ta = tb + ((uint32_t)(32 * quarter) << 16) + s * N + slice * COLS;
            uint32_t v[COLS / 2];
#pragma unroll
            for (int c = 0; c < COLS; c += 32) ld16_pack(ta + c, *reinterpret_cast<uint32_t(*)[16]>(v + c / 2));
            ld_wait();
            if (EPI == 0) {
                uint32_t m = v[0];
#pragma unroll
                for (int i = 1; i < COLS / 2; i++) m = __vmins2(m, v[i]);
                acc |= m;
            } else if (EPI == 1) {
                uint32_t o = 0;
#pragma unroll
                for (int i = 0; i < COLS / 2; i += 2) o = o | v[i] | v[i + 1];
                acc |= o & 0x80008000u;
            } else {
                acc ^= v[0];
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345u) out[blockIdx.x] = int(acc);
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

template <int KT, int NS, int N, int E, int GROUPS, int EPI, int NA = 1, int NBT = 1>
void run(int T, int nsm, long long *dcyc, int *dout) {
    constexpr int KB = 32 * KT;
    const size_t smem = size_t(NA * M + NBT * NB) * KB;
    auto kern = pipe_bench<KT, NS, N, E, GROUPS, EPI, NA, NBT>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<nsm, 32 * (1 + E), smem>>>(16, dcyc, dout);
    CK(cudaDeviceSynchronize());
    kern<<<nsm, 32 * (1 + E), smem>>>(T, dcyc, dout);
    CK(cudaDeviceSynchronize());
    std::vector<long long> cyc(nsm);
    CK(cudaMemcpy(cyc.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (long long c : cyc) avg += double(c);
    avg /= nsm;
    printf("NA=%d NBT=%d KT=%d NS=%d N=%3d E=%2d groups=%d epi=%-6s: %7.1f cyc per 128x256 tile, %6.1f cand/clk/SM (MMA floor %d)\n", NA, NBT, KT,
           NS, N, E, GROUPS, EPI == 0 ? "min16" : EPI == 1 ? "or16" : "ld", avg / T, double(M) * NB * T / avg, 128 * KT);
}

int main(int argc, char **argv) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int nsm = prop.multiProcessorCount;
    const int T = argc > 1 ? atoi(argv[1]) : 8000;
    long long *dcyc;
    int *dout;
    CK(cudaMalloc(&dcyc, nsm * 8));
    CK(cudaMalloc(&dout, nsm * 4));
    printf("device %s, %d SMs, T=%d tiles per SM\n", prop.name, nsm, T);
    run<2, 2, 256, 8, 1, 1>(T, nsm, dcyc, dout);
    run<2, 2, 256, 8, 1, 1, 4, 1>(T, nsm, dcyc, dout);
    run<2, 2, 256, 8, 1, 1, 1, 5>(T, nsm, dcyc, dout);
    run<2, 2, 256, 8, 1, 1, 4, 5>(T, nsm, dcyc, dout);
    run<2, 2, 256, 8, 1, 2, 4, 5>(T, nsm, dcyc, dout);
    run<3, 2, 256, 8, 1, 1, 1, 1>(T, nsm, dcyc, dout);
    run<3, 2, 256, 8, 1, 1, 4, 3>(T, nsm, dcyc, dout);
    printf("done\n");
    return 0;
}
