// sm_100a tensor-core plumbing for the tensor-core tile kernel (kernels.cu, tc_tile_kernel) and
// its microbenchmark (tools/microbench/tc_i8.cu): shared-memory matrix descriptors,
// tcgen05.mma kind::i8, TMEM allocation, tcgen05.ld, mbarriers. Inline PTX only; no CUTLASS.
#pragma once
#include <cstdint>

namespace sdb {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major operand, no swizzle ("interleaved" canonical layout): 8-row x 16-byte core
// matrices of 128 contiguous bytes. lbo = byte distance between the two 16-byte K chunks of
// one MMA step, sbo = byte distance between consecutive 8-row groups.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;  // descriptor version 1 (sm_100)
    return d;                // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

// instruction descriptor: kind::i8, s8 x s8 -> s32, both operands K-major, dense
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4)                       // D format s32
           | (1u << 7) | (1u << 10)        // A, B signed 8-bit
           | (uint32_t(N >> 3) << 17)      // N / 8
           | (uint32_t(M >> 4) << 24);     // M / 16
}

// byte offset of element (row, k) of an R-row K-major operand in the layout sdesc() describes
// with sbo = 128 and lbo = R * 16
__host__ __device__ constexpr uint32_t kmajor_off(int R, int row, int k) {
    return uint32_t((k >> 4) * (R * 16) + (row >> 3) * 128 + (row & 7) * 16 + (k & 15));
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// the same from a converged warp: one elected lane issues it (the descriptors are warp-uniform)
__device__ __forceinline__ void mma_i8_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// arrive on an mbarrier once every tcgen05.mma this thread issued so far has completed
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// from a converged warp: the elected lane commits (one arrival)
__device__ __forceinline__ void commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core's async proxy
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// whole warp: allocate `cols` TMEM columns, base address written to *dst (shared memory)
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Waits for the phase with the given parity to complete. The suspend-time hint lets the
// hardware park the warp until the phase flips (instead of re-issuing the test), so waiting
// warps leave the issue slots to the working ones.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef SDB_TC_NO_SUSPEND_HINT  // A/B experiments
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// the same on precomputed shared-window addresses (one cvta for the kernel, not one per call)
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
        "r"(parity), "r"(0x989680)
        : "memory");
}
// The same wait from a converged warp, with a warp-uniform exit (vote.all over the lanes'
// try_wait results): ptxas then sees uniform control flow around the wait and keeps the
// caller's warp-uniform state (descriptors, barrier addresses, counters) in uniform registers.
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity), "r"(0x989680)
            : "memory");
    } while (!__all_sync(0xffffffffu, ok));
}
__device__ __forceinline__ void commit_elect_a(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
        : "memory");
}

// One TMEM stage of the MMA warp as a single block, from a converged warp: wait for the stage's
// tempty phase (and, when `bwait`, for the tail tile's bfull phase), then the elected lane issues
// the KT MMAs of the stage (K = 32 each; the operand descriptors advance by a_step / b_step per
// K step), commits them to `tfull` and, when `release`, to the tail slot's `bempty`. Everything
// the MMAs need is an input of the block, so it is computed before the wait and the path from
// the barrier flip to the first UTCIMMA holds no address arithmetic.
#define SDB_MMA_STAGE_HEAD                                                       \
    "{\n\t"                                                                      \
    ".reg .pred p, e, bw, rel, pf, pt;\n\t"                                      \
    ".reg .b64 a1, a2, a3, b1, b2, b3, as, bs;\n\t"                              \
    "setp.ne.b32 bw, %4, 0;\n\t"                                                 \
    "setp.ne.b32 rel, %13, 0;\n\t"                                               \
    "setp.ne.b32 pf, 0, 0;\n\t"                                                  \
    "setp.eq.b32 pt, 0, 0;\n\t"                                                  \
    "cvt.u64.u32 as, %8;\n\t"                                                    \
    "cvt.u64.u32 bs, %9;\n\t"                                                    \
    "add.u64 a1, %6, as;\n\t"                                                    \
    "add.u64 b1, %7, bs;\n\t"                                                    \
    "add.u64 a2, a1, as;\n\t"                                                    \
    "add.u64 b2, b1, bs;\n\t"                                                    \
    "add.u64 a3, a2, as;\n\t"                                                    \
    "add.u64 b3, b2, bs;\n\t"                                                    \
    "elect.sync _|e, 0xffffffff;\n\t"                                            \
    "and.pred rel, rel, e;\n"                                                    \
    "WT_%=:\n\t"                                                                 \
    "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %14;\n\t"             \
    "@!p bra WT_%=;\n\t"                                                         \
    "@!bw bra GO_%=;\n"                                                          \
    "WB_%=:\n\t"                                                                 \
    "mbarrier.try_wait.parity.shared::cta.b64 p, [%2], %3, %14;\n\t"             \
    "@!p bra WB_%=;\n"                                                           \
    "GO_%=:\n\t"                                                                 \
    "tcgen05.fence::after_thread_sync;\n\t"                                      \
    "@e tcgen05.mma.cta_group::1.kind::i8 [%5], %6, %7, %10, pf;\n\t"
#define SDB_MMA_STAGE_K(a, b) "@e tcgen05.mma.cta_group::1.kind::i8 [%5], " a ", " b ", %10, pt;\n\t"
#define SDB_MMA_STAGE_TAIL                                                                        \
    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%11];\n\t"         \
    "@rel tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%12];\n\t"       \
    "}\n"
#define SDB_MMA_STAGE_OPS                                                                                         \
    ::"r"(tempty), "r"(tpar), "r"(bfull), "r"(bpar), "r"(uint32_t(bwait)), "r"(d_tmem), "l"(adesc), "l"(bdesc),     \
        "r"(a_step), "r"(b_step), "r"(idesc), "r"(tfull), "r"(bempty), "r"(uint32_t(release)), "r"(0x989680)        \
        : "memory"
template <int KT>
__device__ __forceinline__ void mma_stage(uint32_t tempty, uint32_t tpar, uint32_t bfull, uint32_t bpar, bool bwait,
                                          uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t a_step,
                                          uint32_t b_step, uint32_t idesc, uint32_t tfull, uint32_t bempty,
                                          bool release) {
    static_assert(KT >= 1 && KT <= 4, "K steps per stage");
    if constexpr (KT == 1) {
        asm volatile(SDB_MMA_STAGE_HEAD SDB_MMA_STAGE_TAIL SDB_MMA_STAGE_OPS);
    } else if constexpr (KT == 2) {
        asm volatile(SDB_MMA_STAGE_HEAD SDB_MMA_STAGE_K("a1", "b1") SDB_MMA_STAGE_TAIL SDB_MMA_STAGE_OPS);
    } else if constexpr (KT == 3) {
        asm volatile(SDB_MMA_STAGE_HEAD SDB_MMA_STAGE_K("a1", "b1") SDB_MMA_STAGE_K("a2", "b2")
                         SDB_MMA_STAGE_TAIL SDB_MMA_STAGE_OPS);
    } else {
        asm volatile(SDB_MMA_STAGE_HEAD SDB_MMA_STAGE_K("a1", "b1") SDB_MMA_STAGE_K("a2", "b2")
                         SDB_MMA_STAGE_K("a3", "b3") SDB_MMA_STAGE_TAIL SDB_MMA_STAGE_OPS);
    }
}
#undef SDB_MMA_STAGE_HEAD
#undef SDB_MMA_STAGE_K
#undef SDB_MMA_STAGE_TAIL
#undef SDB_MMA_STAGE_OPS

__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 16 consecutive 32-bit columns: thread t gets lane (taddr.lane + t), columns
// taddr.col .. +15
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// as ld16, with pack::16b: the low halves of two adjacent columns per register (32 columns)
__device__ __forceinline__ void ld16_pack(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// 32 lanes x 128 columns with pack::16b: 64 registers, the low halves of adjacent columns
__device__ __forceinline__ void ld64_pack(uint32_t taddr, uint32_t (&v)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
        : "r"(taddr));
}

__device__ __forceinline__ int min3i(int a, int b, int c) { return min(min(a, b), c); }

// a | b | c as one LOP3 that ptxas keeps where it stands (no re-association into chains)
__device__ __forceinline__ uint32_t or3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xFE;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

}  // namespace tc
}  // namespace sdb
