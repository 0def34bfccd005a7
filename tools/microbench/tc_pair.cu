// CTA-pair (tcgen05 cta_group::2) gate for the tensor-core tile kernel: one MMA instruction
// computes a 256 x 256 x 32 int8 tile across two SMs. Checks the operand / accumulator
// layout against a host reference, then times the pair pipeline (leader MMA thread, 8
// epilogue warps per CTA with the OR-reduce epilogue, TMEM stages handed back across the
// pair through the leader's mbarriers).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -I paper_2408_10743_b200/csrc -o tools/microbench/tc_pair tools/microbench/tc_pair.cu
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

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the peer CTA's address of a local shared-memory word
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t *dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}
__device__ __forceinline__ void mma2_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     bar),
                 "h"((unsigned short)3)
                 : "memory");
}

constexpr int R = 128;  // rows of A and of B each CTA holds

// A[c][r][k] and B[c][r][k]: small ints
__host__ __device__ inline int8_t aval(int c, int r, int k) { return int8_t(((c * 7 + r * 3 + k * 5) % 5) - 2); }
__host__ __device__ inline int8_t bval(int c, int r, int k) { return int8_t(((c * 11 + r * 5 + k * 3) % 7) - 3); }

template <int KT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) check_pair(int *D) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    constexpr int KB = 32 * KT;
    unsigned char *sA = sm, *sB = sm + R * KB;
    const uint32_t c = cta_rank();
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < R * KB; i += blockDim.x) {
        sA[kmajor_off(R, i / KB, i % KB)] = (unsigned char)aval(int(c), i / KB, i % KB);
        sB[kmajor_off(R, i / KB, i % KB)] = (unsigned char)bval(int(c), i / KB, i % KB);
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (warp == 0) tmem_alloc2(&tbase, 256);
    fence_async_smem();
    fence_before();
    cluster_sync();
    fence_after();
    const uint32_t tb = tbase;
    if (c == 0 && threadIdx.x == 0) {
        const uint32_t id = idesc_i8(256, 256);
        for (int k = 0; k < KT; k++) {
            const uint64_t ad = sdesc(smem_u32(sA) + k * 2 * (R * 16), R * 16, 128);
            const uint64_t bd = sdesc(smem_u32(sB) + k * 2 * (R * 16), R * 16, 128);
            mma2_i8(tb, ad, bd, id, k > 0);
        }
        commit2(smem_u32(&bar));
    }
    mbar_wait(&bar, 0);
    fence_after();
    for (int col = 0; col < 256; col += 16) {
        uint32_t v[16];
        ld16(tb + ((uint32_t)(32 * warp) << 16) + col, v);
        ld_wait();
        for (int i = 0; i < 16; i++) D[(c * 128 + 32 * warp + (threadIdx.x & 31)) * 256 + col + i] = int(v[i]);
    }
    fence_before();
    cluster_sync();
    if (warp == 0) tmem_dealloc2(tb, 256);
}

// Pipeline timing: leader lane issues KT MMAs per stage into NS=2 stages of 256 columns;
// each CTA's 8 epilogue warps read their 128 lanes x 128 columns (x64 pack16), OR-reduce,
// and arrive on the leader's tempty barrier (remote for the peer).
template <int KT, int LOCAL_ONLY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(288, 1) pipe_pair(int T, long long *cycles, int *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t tfull[2], tempty[2];
    __shared__ uint32_t tbase;
    constexpr int KB = 32 * KT;
    constexpr int NA = 4, NBT = 5;
    unsigned char *sA = sm, *sB = sm + NA * R * KB;
    const uint32_t c = cta_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (NA + NBT) * R * KB; i += blockDim.x) sm[i] = (unsigned char)((i * 7 + 3) % 5 - 2);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; s++) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], (LOCAL_ONLY ? 1 : 2) * 8 * 32);  // every epilogue thread of both CTAs
        }
        mbar_fence_init();
    }
    if (warp == 0) tmem_alloc2(&tbase, 512);
    fence_async_smem();
    fence_before();
    cluster_sync();
    fence_after();
    const uint32_t tb = tbase;
    long long t0 = clock64();
    uint32_t acc = 0;
    if (warp == 0) {
        if (c == 0) {
            const uint32_t id = idesc_i8(256, 256);
            uint32_t st = 0, par = 0;
            const uint64_t aD = sdesc(smem_u32(sA), R * 16, 128), bD = sdesc(smem_u32(sB), R * 16, 128);
            for (int it = 0; it < T; it++) {
                mbar_wait(&tempty[st], par ^ 1);
                fence_after();
                const uint64_t aT = aD + uint64_t(((it / NBT) % NA) * R * KB / 16);
                const uint64_t bT = bD + uint64_t((it % NBT) * R * KB / 16);
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    const uint32_t acc_ = k > 0;
                    asm volatile(
                        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tb + st * 256),
                        "l"(aT + uint64_t(k * 2 * R)), "l"(bT + uint64_t(k * 2 * R)), "r"(id), "r"(acc_));
                }
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
                        smem_u32(&tfull[st])),
                    "h"((unsigned short)3)
                    : "memory");
                st ^= 1;
                par ^= st == 0;
            }
        }
    } else {
        const int q = warp & 3, half = (warp - 1) >> 2;
        const uint32_t ta0 = tb + (uint32_t(32 * q) << 16) + uint32_t(half * 128);
        uint32_t st = 0, par = 0;
        const uint32_t te_leader0 = mapa(smem_u32(&tempty[0]), 0), te_leader1 = mapa(smem_u32(&tempty[1]), 0);
        for (int it = 0; it < T; it++) {
            mbar_wait(&tfull[st], par);
            fence_after();
            uint32_t v[64];
            ld64_pack(ta0 + st * 256, v);
            ld_wait();
            uint32_t o = 0;
#pragma unroll
            for (int i = 0; i < 64; i += 3) o |= or3(v[i], v[i + 1 < 64 ? i + 1 : 63], v[i + 2 < 64 ? i + 2 : 63]);
            acc |= o & 0x80008000u;
            fence_before();
            if (!LOCAL_ONLY || c == 0) arrive_cluster(st ? te_leader1 : te_leader0);
            st ^= 1;
            par ^= st == 0;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345u) out[blockIdx.x] = int(acc);
    fence_before();
    cluster_sync();
    if (warp == 0) tmem_dealloc2(tb, 512);
}

int main(int argc, char **argv) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int nsm = prop.multiProcessorCount;
    printf("device %s, %d SMs\n", prop.name, nsm);
    // ---- layout check
    {
        constexpr int KT = 2, KB = 64;
        int *dD;
        CK(cudaMalloc(&dD, 256 * 256 * 4));
        const size_t smem = 2 * R * KB;
        CK(cudaFuncSetAttribute(check_pair<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        check_pair<KT><<<2, 128, smem>>>(dD);
        CK(cudaDeviceSynchronize());
        std::vector<int> D(256 * 256);
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        // hypothesis: A rows 0..127 from CTA 0, 128..255 from CTA 1; B rows (= D columns) likewise
        int bad = 0, bad_rep = 0;
        for (int m = 0; m < 256; m++)
            for (int n = 0; n < 256; n++) {
                int ref = 0, ref_rep = 0;
                for (int k = 0; k < KB; k++) {
                    ref += int(aval(m / 128, m % 128, k)) * int(bval(n / 128, n % 128, k));
                    ref_rep += int(aval(m / 128, m % 128, k)) * int(bval(0, n % 128, k));
                }
                if (D[m * 256 + n] != ref && bad++ < 4) printf("  D[%d][%d] = %d, split-B hypothesis %d\n", m, n, D[m * 256 + n], ref);
                bad_rep += D[m * 256 + n] != ref_rep;
            }
        printf("pair layout check: %d mismatches (A and B split across the pair), %d (B from CTA 0 only)\n", bad, bad_rep);
        if (bad) return 1;
    }
    // ---- pipeline timing
    {
        const int T = argc > 1 ? atoi(argv[1]) : 6000;
        long long *dc;
        int *dout;
        CK(cudaMalloc(&dc, nsm * 8));
        CK(cudaMalloc(&dout, nsm * 4));
        for (int v = 0; v < 4; v++) {
            const int kt = 2 + (v & 1), lo = v >> 1;
            const size_t smem = size_t(4 + 5) * R * 32 * kt;
            auto kern = v == 0 ? pipe_pair<2, 0> : v == 1 ? pipe_pair<3, 0> : v == 2 ? pipe_pair<2, 1> : pipe_pair<3, 1>;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            const int grid = nsm - nsm % 2;
            kern<<<grid, 288, smem>>>(16, dc, dout);
            CK(cudaDeviceSynchronize());
            kern<<<grid, 288, smem>>>(T, dc, dout);
            CK(cudaDeviceSynchronize());
            std::vector<long long> cyc(grid);
            CK(cudaMemcpy(cyc.data(), dc, grid * 8, cudaMemcpyDeviceToHost));
            double avg = 0;
            for (long long x : cyc) avg += double(x);
            avg /= grid;
            printf("pair KT=%d%s: %.1f cycles per stage (256 x 256 per pair = 128 x 256 per SM; 1-CTA MMA floor %d)\n", kt, lo ? " (leader's epilogue only)" : "",
                   avg / T, 128 * kt);
        }
    }
    printf("done\n");
    return 0;
}
