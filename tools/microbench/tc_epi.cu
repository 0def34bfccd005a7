// Epilogue floor of the tensor-core tile kernel, isolated: how fast can 8 (or 16) warps drain
// 128 x 256 s32 accumulators from TMEM with pack::16b loads, with and without the MMA and the
// stage barriers?
//   mode 0 : loads only, no barriers, no MMA (TMEM read throughput per load shape)
//   mode 1 : the two-stage pipeline of the kernel: MMA warp (KT = 0 skips the MMAs: barriers
//            only) + E epilogue warps; ARR = 0 lane 0 arrives after __syncwarp, 1 every lane
//            arrives, 2 lane 0 arrives without __syncwarp
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -I paper_2408_10743_b200/csrc -o tools/microbench/tc_epi tools/microbench/tc_epi.cu
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

constexpr int M = 128, N = 256;

__device__ __forceinline__ void ld32_pack(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// OR of n packed words as a tree of 3-input ORs
template <int n>
__device__ __forceinline__ uint32_t or_tree(const uint32_t *v) {
    if constexpr (n == 1) return v[0];
    else if constexpr (n == 2) return v[0] | v[1];
    else {
        constexpr int m = (n + 2) / 3;
        uint32_t r[m];
#pragma unroll
        for (int i = 0; i < m; i++) {
            if (3 * i + 2 < n) r[i] = or3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
            else if (3 * i + 1 < n) r[i] = v[3 * i] | v[3 * i + 1];
            else r[i] = v[3 * i];
        }
        return or_tree<m>(r);
    }
}

// LD: 0 = one x64 pack (128 columns), 1 = two x32 pack (64 + 64), 2 = one x64 plain (64 columns),
//     3 = one x32 pack (64 columns: for E = 16)
template <int LD>
__device__ __forceinline__ uint32_t drain(uint32_t ta, uint32_t early_bar = 0) {
    if constexpr (LD == 0) {
        uint32_t v[64];
        ld64_pack(ta, v);
        ld_wait();
        if (early_bar) {
            fence_before();
            if ((threadIdx.x & 31) == 0) mbar_arrive_a(early_bar);
        }
        return or_tree<64>(v);
    } else if constexpr (LD == 1) {
        uint32_t v[32], w[32];
        ld32_pack(ta, v);
        ld32_pack(ta + 64, w);
        ld_wait();
        return or_tree<32>(v) | or_tree<32>(w);
    } else if constexpr (LD == 2) {
        uint32_t v[32], w[32];
        ld32(ta, v);
        ld32(ta + 32, w);
        ld_wait();
        return or_tree<32>(v) | or_tree<32>(w);
    } else {
        uint32_t v[32];
        ld32_pack(ta, v);
        ld_wait();
        return or_tree<32>(v);
    }
}

// WAIT: 0 = try_wait with the suspend-time hint (the kernel's mbar_wait_a), 1 = try_wait without a
// hint, 2 = test_wait spin
template <int WAIT>
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t parity) {
    if constexpr (WAIT == 0) {
        mbar_wait_a(bar, parity);
    } else if constexpr (WAIT == 1) {
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
            "r"(parity)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "WAIT_%=:\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
            "r"(parity)
            : "memory");
    }
}

template <int MODE, int KT, int E, int LD, int ARR, int WAIT = 0, int TL = 0>
__global__ void __launch_bounds__(32 * (1 + E), 1) epi_bench(int T, long long *cycles, int *out) {
    __shared__ volatile long long ts_commit[2], ts_arrive[2];
    long long lat1 = 0, lat2 = 0, wt = 0, work = 0;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[2], empty[2];
    __shared__ uint32_t tbase;
    constexpr int KB = 32 * (KT > 0 ? KT : 1);
    unsigned char *sA = sm, *sB = sm + M * KB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&tbase, 512);
    for (int i = threadIdx.x; i < (M + N) * KB; i += blockDim.x) sm[i] = (unsigned char)((i * 7 + 3) % 5 - 2);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ARR == 1 ? 32 * E : E);
        }
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    long long t0 = clock64();
    uint32_t acc = 0;
    if (warp == 0) {
        if (MODE == 1) {
            const uint32_t id = idesc_i8(M, N);
            const uint32_t f0 = smem_u32(&full[0]), e0 = smem_u32(&empty[0]);
            for (int it = 0; it < T; it++) {
                const int s = it & 1;
                const uint32_t ph = (it >> 1) & 1;
                long long w0 = 0;
                if (TL) w0 = clock64();
                wait_bar<WAIT>(e0 + 8 * s, ph ^ 1);
                if (TL) {
                    const long long now = clock64();
                    wt += now - w0;
                    if (it >= 2) lat2 += now - ts_arrive[s];
                }
                fence_after();
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    const uint64_t ad = sdesc(smem_u32(sA) + k * 2 * (M * 16), M * 16, 128);
                    const uint64_t bd = sdesc(smem_u32(sB) + k * 2 * (N * 16), N * 16, 128);
                    mma_i8_elect(tb + s * N, ad, bd, id, k > 0);
                }
                if (TL && lane == 0) ts_commit[s] = clock64();
                commit_elect_a(f0 + 8 * s);
            }
            if (TL && lane == 0 && blockIdx.x == 0)
                printf("  mma warp: tempty wait %.1f per stage, arrive->seen %.1f\n", double(wt) / T, double(lat2) / (T - 2));
        }
    } else {
        const int e = warp - 1;
        const int quarter = warp & 3;
        constexpr int COLS = N / (E / 4);
        const int slice = e / 4;
        const uint32_t f0 = smem_u32(&full[0]), e0 = smem_u32(&empty[0]);
        for (int it = 0; it < T; it++) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            long long w0 = 0, w1 = 0;
            if (MODE == 1) {
                if (TL) w0 = clock64();
                wait_bar<WAIT>(f0 + 8 * s, ph);
                if (TL) {
                    w1 = clock64();
                    wt += w1 - w0;
                    lat1 += w1 - ts_commit[s];
                }
                fence_after();
            }
            const uint32_t ta = tb + ((uint32_t)(32 * quarter) << 16) + s * N + slice * COLS;
            const uint32_t o = drain<LD>(ta, (MODE == 1 && ARR == 3) ? e0 + 8 * s : 0u);
            if (__any_sync(0xffffffffu, o & 0x80008000u)) acc += o;
            if (MODE == 1) {
                fence_before();
                if (ARR == 1) {
                    mbar_arrive_a(e0 + 8 * s);
                } else if (ARR == 3) {
                } else {
                    if (ARR == 0) __syncwarp();
                    if (TL && e == E - 1 && lane == 0) ts_arrive[s] = clock64();
                    if (lane == 0) mbar_arrive_a(e0 + 8 * s);
                }
                if (TL) work += clock64() - w1;
            }
        }
        if (TL && (e == 0 || e == E - 1) && lane == 0 && blockIdx.x == 0)
            printf("  epi warp %d: tfull wait %.1f per stage, commit->seen %.1f, ld+or+arrive %.1f\n", e, double(wt) / T,
                   double(lat1) / T, double(work) / T);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345u) out[blockIdx.x] = int(acc);
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

// MMA issue rate alone: one warp issues T MMAs of M = 128 x NN x K = 32 back to back (a commit
// every 8), waits for the last; cycles per MMA
template <int NN>
__global__ void __launch_bounds__(32, 1) mma_only(int T, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    tmem_alloc(&tbase, 512);
    for (int i = threadIdx.x; i < (M + N) * 32; i += 32) sm[i] = (unsigned char)((i * 7 + 3) % 5 - 2);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    fence_async_smem();
    fence_before();
    __syncwarp();
    fence_after();
    const uint32_t tb = tbase;
    const uint32_t id = idesc_i8(M, NN);
    const uint64_t ad = sdesc(smem_u32(sm), M * 16, 128), bd = sdesc(smem_u32(sm + M * 32), N * 16, 128);
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < T; it += 8) {
#pragma unroll
        for (int k = 0; k < 8; k++) mma_i8_elect(tb + ((it / 8) & 1) * 256, ad, bd, id, k > 0);
        commit_elect_a(smem_u32(&bar));
        if ((it / 8) & 1) {  // every 16 MMAs: drain (keeps the issue queue bounded)
            mbar_wait_a(smem_u32(&bar), ph);
            ph ^= 1;
            mbar_wait_a(smem_u32(&bar), ph);
            ph ^= 1;
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    fence_before();
    __syncwarp();
    tmem_dealloc(tb, 512);
}
template <int NN>
void run_mma(int nsm, long long *dcyc) {
    const int T = 16 * 2000;
    CK(cudaFuncSetAttribute(mma_only<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, int((M + N) * 32)));
    mma_only<NN><<<nsm, 32, (M + N) * 32>>>(T, dcyc);
    CK(cudaDeviceSynchronize());
    std::vector<long long> cyc(nsm);
    CK(cudaMemcpy(cyc.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (long long c : cyc) avg += double(c);
    printf("mma only M=128 N=%3d K=32 i8: %6.1f cycles per MMA\n", NN, avg / nsm / T);
}

template <int MODE, int KT, int E, int LD, int ARR, int WAIT = 0, int TL = 0>
void run(int T, int nsm, long long *dcyc, int *dout) {
    constexpr int KB = 32 * (KT > 0 ? KT : 1);
    const size_t smem = size_t(M + N) * KB;
    auto kern = epi_bench<MODE, KT, E, LD, ARR, WAIT, TL>;
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
    static const char *ldn[] = {"x64pack", "2x32pack", "2x32plain", "x32pack"};
    static const char *arn[] = {"lane0+sync", "all-lane", "lane0", "early"};
    static const char *wn[] = {"try+hint", "try", "test"};
    printf("mode=%d KT=%d E=%2d ld=%-9s arrive=%-10s wait=%-8s: %7.1f cyc per stage (MMA floor %d)\n", MODE, KT, E,
           ldn[LD], arn[ARR], wn[WAIT], avg / T, 128 * KT);
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
    printf("device %s, %d SMs, T=%d stages per SM\n", prop.name, nsm, T);
    run_mma<256>(nsm, dcyc);
    run_mma<128>(nsm, dcyc);
    run_mma<64>(nsm, dcyc);
    run_mma<192>(nsm, dcyc);
    // TMEM read throughput alone
    run<0, 0, 8, 0, 0>(T, nsm, dcyc, dout);
    run<0, 0, 8, 1, 0>(T, nsm, dcyc, dout);
    run<0, 0, 8, 2, 0>(T, nsm, dcyc, dout);   // 64 plain columns per warp: half a stage
    run<0, 0, 16, 3, 0>(T, nsm, dcyc, dout);
    // barriers only (no MMA): the sync chain
    run<1, 0, 8, 0, 0>(T, nsm, dcyc, dout);
    run<1, 0, 8, 0, 1>(T, nsm, dcyc, dout);
    run<1, 0, 8, 0, 2>(T, nsm, dcyc, dout);
    run<1, 0, 16, 3, 2>(T, nsm, dcyc, dout);
    // with the MMA at K = 32, 64
    run<1, 1, 8, 0, 0>(T, nsm, dcyc, dout);
    run<1, 1, 8, 0, 1>(T, nsm, dcyc, dout);
    run<1, 1, 8, 0, 2>(T, nsm, dcyc, dout);
    run<1, 1, 8, 1, 2>(T, nsm, dcyc, dout);
    run<1, 1, 16, 3, 2>(T, nsm, dcyc, dout);
    run<1, 2, 8, 0, 0>(T, nsm, dcyc, dout);
    run<1, 2, 8, 0, 1>(T, nsm, dcyc, dout);
    run<1, 2, 8, 0, 2>(T, nsm, dcyc, dout);
    run<1, 2, 16, 3, 2>(T, nsm, dcyc, dout);
    // the wait flavour
    run<1, 0, 8, 0, 2, 1>(T, nsm, dcyc, dout);
    run<1, 0, 8, 0, 2, 2>(T, nsm, dcyc, dout);
    run<1, 1, 8, 0, 2, 1>(T, nsm, dcyc, dout);
    run<1, 1, 8, 0, 2, 2>(T, nsm, dcyc, dout);
    run<1, 2, 8, 0, 2, 1>(T, nsm, dcyc, dout);
    run<1, 2, 8, 0, 2, 2>(T, nsm, dcyc, dout);
    run<1, 3, 8, 0, 2, 0>(T, nsm, dcyc, dout);
    run<1, 3, 8, 0, 2, 2>(T, nsm, dcyc, dout);
    // release right after the load
    run<1, 0, 8, 0, 3>(T, nsm, dcyc, dout);
    run<1, 1, 8, 0, 3>(T, nsm, dcyc, dout);
    run<1, 2, 8, 0, 3>(T, nsm, dcyc, dout);
    run<1, 3, 8, 0, 3>(T, nsm, dcyc, dout);
    printf("done\n");
    return 0;
}
