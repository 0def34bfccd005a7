// Gate for the tensor-core candidate path: can tcgen05.mma kind::i8 with
// TMEM accumulators plus a tcgen05.ld + min epilogue beat the POPC path's 15.6 candidates per
// clock per SM? One candidate = one int32 accumulator element (head row x tail column).
//
//   check : one 128x256 tile vs a host reference (descriptor / layout / idesc correctness),
//           plus what pack::16b returns for 32-bit accumulators
//   bench : persistent, one CTA per SM; warp 0 issues MMAs into two TMEM stages of 256
//           columns, E epilogue warps drain them (tcgen05.ld, VIMNMX3 running minimum)
//           modes: full, mma-only (epilogue only hands stages back), ld-only (no MMA waits)
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -I paper_2408_10743_b200/csrc -o tools/microbench/tc_i8 tools/microbench/tc_i8.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace sdb::tc;

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

constexpr int M = 128, NT = 256;

__global__ void check_kernel(const int8_t *A, const int8_t *B, int KB, int *D, uint32_t *P) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned char *sA = sm, *sB = sm + M * KB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&tbase, 256);
    for (int i = threadIdx.x; i < M * KB; i += blockDim.x) sA[kmajor_off(M, i / KB, i % KB)] = A[i];
    for (int i = threadIdx.x; i < NT * KB; i += blockDim.x) sB[kmajor_off(NT, i / KB, i % KB)] = B[i];
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_i8(M, NT);
        for (int s = 0; s < KB / 32; s++) {
            const uint64_t ad = sdesc(smem_u32(sA) + s * 2 * (M * 16), M * 16, 128);
            const uint64_t bd = sdesc(smem_u32(sB) + s * 2 * (NT * 16), NT * 16, 128);
            mma_i8(tb, ad, bd, id, s > 0);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    for (int c = 0; c < NT; c += 16) {
        uint32_t v[16];
        ld16(tb + ((uint32_t)(32 * warp) << 16) + c, v);
        ld_wait();
        for (int i = 0; i < 16; i++) D[(32 * warp + lane) * NT + c + i] = int(v[i]);
    }
    for (int c = 0; c < NT; c += 32) {
        uint32_t v[16];
        ld16_pack(tb + ((uint32_t)(32 * warp) << 16) + c, v);
        ld_wait();
        for (int i = 0; i < 16; i++) P[(32 * warp + lane) * (NT / 2) + c / 2 + i] = v[i];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 256);
}

// MODE 0 full, 1 mma-only, 2 ld-only, 3 full with pack::16b loads + VIMNMX.S16x2
template <int KT, int E, int MODE>
__global__ void __launch_bounds__(32 * (1 + E), 1) bench_kernel(const int8_t *A, const int8_t *B, int T,
                                                                   long long *cycles, int *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[2], empty[2];
    __shared__ uint32_t tbase;
    constexpr int KB = 32 * KT;
    unsigned char *sA = sm, *sB = sm + M * KB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&tbase, 512);
    for (int i = threadIdx.x; i < M * KB; i += blockDim.x) sA[kmajor_off(M, i / KB, i % KB)] = A[i];
    for (int i = threadIdx.x; i < NT * KB; i += blockDim.x) sB[kmajor_off(NT, i / KB, i % KB)] = B[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], E);
        }
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    long long t0 = clock64();
    int m = 0x7fffffff;
    if (warp == 0) {
        if (MODE != 2 && MODE != 4 && lane == 0) {
            const uint32_t id = idesc_i8(M, NT);
            for (int it = 0; it < T; it++) {
                const int s = it & 1;
                const uint32_t ph = (it >> 1) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                fence_after();
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    const uint64_t ad = sdesc(smem_u32(sA) + k * 2 * (M * 16), M * 16, 128);
                    const uint64_t bd = sdesc(smem_u32(sB) + k * 2 * (NT * 16), NT * 16, 128);
                    mma_i8(tb + s * 256, ad, bd, id, k > 0);
                }
                commit(&full[s]);
            }
        }
    } else {
        const int e = warp - 1;
        const int quarter = warp & 3;
        // 32-column chunks of a stage, dealt round-robin to the E/4 warps of each lane quarter
        constexpr int Q = E / 4;
        const int r = e / 4;
        for (int it = 0; it < T; it++) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            if (MODE != 2 && MODE != 4) mbar_wait(&full[s], ph);
            fence_after();
            const uint32_t ta = tb + ((uint32_t)(32 * quarter) << 16) + s * 256;
            if (MODE == 0 || MODE == 2) {
#pragma unroll
                for (int c = 32 * r; c < 256; c += 32 * Q) {
                    uint32_t v[32];
                    ld32(ta + c, v);
                    ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; i += 2) m = min3i(m, int(v[i]), int(v[i + 1]));
                }
            } else if (MODE == 3 || MODE == 4) {
#pragma unroll
                for (int c = 32 * r; c < 256; c += 32 * Q) {
                    uint32_t v[16];
                    ld16_pack(ta + c, v);
                    ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; i++) m = int(__vmins2(unsigned(m), v[i]));
                }
            } else if (MODE == 5 || MODE == 6) {
                // f16x2 minimum (HMNMX2) on the packed halves; MODE 6 alternates with VIMNMX.S16x2
                uint32_t m2 = 0x7bff7bffu;
#pragma unroll
                for (int c = 32 * r; c < 256; c += 32 * Q) {
                    uint32_t v[16];
                    ld16_pack(ta + c, v);
                    ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        if (MODE == 6 && (i & 1)) {
                            m = int(__vmins2(unsigned(m), v[i]));
                        } else {
                            asm("min.f16x2 %0, %0, %1;" : "+r"(m2) : "r"(v[i]));
                        }
                    }
                }
                m = min(m, int(m2));
            }
            fence_before();
            __syncwarp();
            if (MODE != 2 && MODE != 4 && lane == 0) mbar_arrive(&empty[s]);
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
    if (m == 12345) out[blockIdx.x] = m;  // keeps the reduction alive
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

// per-SM issue rate of VIMNMX.S16x2 (0), HMNMX2 (1), both interleaved (2), VIMNMX3 (3)
template <int OP>
__global__ void __launch_bounds__(512, 1) pipe_kernel(uint32_t seed, int iters, long long *cycles, uint32_t *out) {
    uint32_t a[8], b = seed * 3u + threadIdx.x;
    for (int i = 0; i < 8; i++) a[i] = seed + i * 77u + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0 || (OP == 2 && (i & 1))) {
                a[i] = __vmins2(a[i], b);
            } else if (OP == 1 || OP == 2) {
                asm volatile("min.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            } else {
                a[i] = uint32_t(min(min(int(a[i]), int(b)), int(a[(i + 1) & 7])));
            }
        }
        b += 0x00010001u;
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    uint32_t x = 0;
    for (int i = 0; i < 8; i++) x ^= a[i];
    if (x == 0x12345678u) out[blockIdx.x] = x;
}

template <int OP>
void run_pipe(int nsm, long long *dcyc, uint32_t *dout) {
    const int iters = 4096;
    pipe_kernel<OP><<<nsm, 512>>>(1u, iters, dcyc, dout);
    CK(cudaDeviceSynchronize());
    std::vector<long long> cyc(nsm);
    CK(cudaMemcpy(cyc.data(), dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    double avg = 0;
    for (long long c : cyc) avg += c;
    avg /= nsm;
    printf("pipe op=%s: %.1f lane-ops/clk/SM\n",
           OP == 0 ? "VIMNMX.S16x2" : OP == 1 ? "HMNMX2" : OP == 2 ? "both (1:1)" : "VIMNMX3", 512.0 * 8 * iters / avg);
}

template <int KT, int E, int MODE>
double run_bench(const int8_t *dA, const int8_t *dB, int T, int nsm, long long *dcyc, int *dout) {
    constexpr int KB = 32 * KT;
    const size_t smem = (size_t)(M + NT) * KB;
    auto kern = bench_kernel<KT, E, MODE>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nsm, 32 * (1 + E), smem>>>(dA, dB, 8, dcyc, dout);  // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<nsm, 32 * (1 + E), smem>>>(dA, dB, T, dcyc, dout);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> cyc(nsm);
    CK(cudaMemcpy(cyc.data(), dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    double avg = 0;
    for (long long c : cyc) {
        mx = c > mx ? c : mx;
        avg += c;
    }
    avg /= nsm;
    const double cand = (double)T * M * NT;
    const double per_clk = cand / avg;
    printf("KT=%d (K=%3d) E=%d mode=%-8s T=%6d: %8.2f ms, %7.1f cyc/tile, %6.1f cand/clk/SM, chip %.3e cand/s (%.0f MHz eff)\n",
           KT, KB, E, MODE == 0 ? "full" : MODE == 1 ? "mma-only" : MODE == 2 ? "ld-only" : MODE == 3 ? "full-pk16" : MODE == 4 ? "ld-pk16" : MODE == 5 ? "full-hmnmx2" : "full-mixed", T, ms,
           avg / T, per_clk, cand * nsm / (ms * 1e-3), avg / (ms * 1e3));
    return per_clk;
}

int main(int argc, char **argv) {
    int dev = 0;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    const int nsm = prop.multiProcessorCount;
    printf("device %s, %d SMs\n", prop.name, nsm);
    const int KBmax = 128;
    std::vector<int8_t> hA(M * KBmax), hB(NT * KBmax);
    unsigned s = 12345;
    auto rnd = [&]() {
        s = s * 1103515245u + 12345u;
        return int((s >> 16) % 5) - 2;
    };
    for (auto &x : hA) x = (int8_t)rnd();
    for (auto &x : hB) x = (int8_t)rnd();
    int8_t *dA, *dB;
    int *dD, *dout;
    uint32_t *dP;
    long long *dcyc;
    CK(cudaMalloc(&dA, hA.size()));
    CK(cudaMalloc(&dB, hB.size()));
    CK(cudaMalloc(&dD, M * NT * 4));
    CK(cudaMalloc(&dP, M * NT * 2));
    CK(cudaMalloc(&dout, nsm * 4));
    CK(cudaMalloc(&dcyc, nsm * 8));
    int bad_total = 0;
    for (int KB : {32, 64, 96, 128}) {
        // A, B as row-major [R][KB] slices of the random pools
        std::vector<int8_t> a(M * KB), b(NT * KB);
        for (int r = 0; r < M; r++)
            for (int k = 0; k < KB; k++) a[r * KB + k] = hA[r * KBmax + k];
        for (int r = 0; r < NT; r++)
            for (int k = 0; k < KB; k++) b[r * KB + k] = hB[r * KBmax + k];
        CK(cudaMemcpy(dA, a.data(), a.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, b.data(), b.size(), cudaMemcpyHostToDevice));
        const size_t smem = (size_t)(M + NT) * KB;
        CK(cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        check_kernel<<<1, 128, smem>>>(dA, dB, KB, dD, dP);
        CK(cudaDeviceSynchronize());
        std::vector<int> D(M * NT);
        std::vector<uint32_t> P(M * NT / 2);
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(P.data(), dP, P.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0, badp = 0;
        for (int i = 0; i < M; i++)
            for (int j = 0; j < NT; j++) {
                int ref = 0;
                for (int k = 0; k < KB; k++) ref += a[i * KB + k] * b[j * KB + k];
                if (D[i * NT + j] != ref && bad++ < 5)
                    printf("  KB=%d D[%d][%d] = %d, want %d\n", KB, i, j, D[i * NT + j], ref);
                if (j % 2 == 0) {
                    int ref2 = 0;
                    for (int k = 0; k < KB; k++) ref2 += a[i * KB + k] * b[(j + 1) * KB + k];
                    const uint32_t want = (uint32_t(ref) & 0xffffu) | (uint32_t(ref2) << 16);
                    if (P[i * (NT / 2) + j / 2] != want && badp++ < 3)
                        printf("  KB=%d pack16 [%d][%d] = %08x, want %08x\n", KB, i, j, P[i * (NT / 2) + j / 2], want);
                }
            }
        printf("check KB=%d: %d mismatches (32-bit), %d (pack::16b as low halves of adjacent columns)\n", KB, bad, badp);
        bad_total += bad;
    }
    if (bad_total) {
        printf("CHECK FAILED\n");
        return 1;
    }
    CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
    const int T = argc > 1 ? atoi(argv[1]) : 20000;
    run_pipe<0>(nsm, dcyc, (uint32_t *)dout);
    run_pipe<1>(nsm, dcyc, (uint32_t *)dout);
    run_pipe<2>(nsm, dcyc, (uint32_t *)dout);
    run_pipe<3>(nsm, dcyc, (uint32_t *)dout);
    run_bench<2, 8, 4>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 12, 4>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 16, 4>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 12, 3>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 16, 3>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 8, 5>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 8, 6>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 12, 6>(dA, dB, T, nsm, dcyc, dout);
    run_bench<3, 12, 6>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 4, 1>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 4, 2>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 8, 2>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 4, 0>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 8, 0>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 8, 3>(dA, dB, T, nsm, dcyc, dout);
    run_bench<2, 4, 3>(dA, dB, T, nsm, dcyc, dout);
    run_bench<3, 4, 1>(dA, dB, T, nsm, dcyc, dout);
    run_bench<3, 8, 0>(dA, dB, T, nsm, dcyc, dout);
    run_bench<3, 8, 3>(dA, dB, T, nsm, dcyc, dout);
    run_bench<4, 4, 1>(dA, dB, T, nsm, dcyc, dout);
    run_bench<4, 8, 0>(dA, dB, T, nsm, dcyc, dout);
    run_bench<4, 8, 3>(dA, dB, T, nsm, dcyc, dout);
    run_bench<1, 4, 1>(dA, dB, T, nsm, dcyc, dout);
    run_bench<1, 8, 0>(dA, dB, T, nsm, dcyc, dout);
    printf("done\n");
    return 0;
}
