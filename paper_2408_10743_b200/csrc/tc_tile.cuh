// Tensor-core tile kernel (device.hpp: TcPlan). Included by kernels.cu inside its anonymous
// namespace: it shares binom_at, tile_exact, TileUnit, run_done and start_threshold with the
// POPC tile kernel.
//
// Warp roles, one CTA per SM (kTcThreads = 576):
//   warp 0        TMEM owner (512 columns: two 128 x 256 s32 stages) and MMA issuer: a converged
//                 warp, one PTX block per stage (tc::mma_stage: wait, elected MMAs, commits)
//   warps 1..8    epilogue: one tcgen05.ld x64 pack::16b per stage, the stage handed back right
//                 after the load, an OR tree over the packed words, a per-row bitmask of the
//                 stages whose sign bits came out set; once per head tile a vote, and for the
//                 flagged (row, stage) pairs the exact path on recomputed pairs (tc_rare_rows)
//   warp 9        unit warp: claims units and publishes their descriptors, one unit ahead
//   warps 10..17  producers, two groups of four: group g writes the head tiles c with
//                 c % 2 == g (A, a ring of four; thread r of the group writes row r), and all
//                 256 threads write the chunk's tail tiles (B, a ring of nbt + 1 slots) —
//                 int8 coordinates in the canonical K-major no-swizzle layout (8-row x 16-byte
//                 core matrices)
// Pipelines (mbarriers): unit queue full/empty, A slot full/empty, B slot full/empty, TMEM
// stage full/empty. No CTA-wide barrier after the start: every warp signals its own part, so
// warps drift freely within the rings.
//
// A unit is (Gamma j, boundary b, up to 128 * kTcUnitTiles heads, up to 256 nbt tails): its na
// head tiles each meet all of its nbt tail tiles. Head row r of the unit's tiles walks na
// consecutive colex ranks (successor steps); a producer thread's nbt tails are consecutive
// ranks too. Element lists stay in registers: the producer routines are compiled per element
// count (h, t - 1 <= kTcMaxPart) and per sign words per row (KW).
//
// Variant builds (tools/build_variant.sh): SDB_TC_TRACE (clock-stamped timeline of block 0,
// tools/tc_trace.py), SDB_TC_LAT (signalling latencies), SDB_TC_GAPS / SDB_TC_PROF (MMA-warp
// gaps and waits), SDB_TC_NOPROD / SDB_TC_NOMMA (pipeline bisection), SDB_TC_COUNT_RARE.
#pragma once

#include "tc_ptx.cuh"

#ifdef SDB_TC_PROF
#define TCP_DECL unsigned long long tcp_t0 = 0, tcp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define TCP_BEGIN tcp_t0 = clock64();
#define TCP_END(i) tcp_acc[i] += clock64() - tcp_t0;
#else
#define TCP_DECL
#define TCP_BEGIN
#define TCP_END(i)
#endif

// 4 coordinates (bytes) of a head: sign bit set -> +1, clear -> -1 (the head carries -s)
__device__ __forceinline__ uint32_t tc_head_word(uint32_t s, int jj) {
    return 0xFFFFFFFFu - ((s >> jj) & 0x01010101u) * 0xFEu;
}
// ... of a tail: clear -> +v, set -> -v (v = 1 or 2)
__device__ __forceinline__ uint32_t tc_tail_word(uint32_t s, int jj, bool v2) {
    const uint32_t b = (s >> jj) & 0x01010101u;
    return v2 ? 0x02020202u + b * 0xFCu : 0x01010101u + b * 0xFEu;
}

// the 32 coordinates of sign word `s` (block blk) of operand row `row` (R rows per tile)
template <bool HEAD>
__device__ __forceinline__ void tc_store_block(unsigned char *tile, int R, int row, int blk, uint32_t s, int W1) {
    uint32_t o[8];
#pragma unroll
    for (int jj = 0; jj < 8; jj++) o[jj] = HEAD ? tc_head_word(s, jj) : tc_tail_word(s, jj, blk * 8 + jj < W1);
    unsigned char *d = tile + tc::kmajor_off(R, row, 32 * blk);
    *reinterpret_cast<uint4 *>(d) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4 *>(d + R * 16) = make_uint4(o[4], o[5], o[6], o[7]);
}

// colex unrank of rho into an M-subset of [0, lim), ascending, in registers (the estimate of
// unrank_colex_est, loops unrolled)
template <int M>
__device__ __forceinline__ void tc_unrank(unsigned long long rho, int lim, const unsigned long long *binom, int BK,
                                          int (&e)[kTcMaxPart]) {
    int c = lim - 1;
#pragma unroll
    for (int i = M; i >= 1; i--) {
        int cc;
        if (i == 1) {
            cc = int(min(rho, (unsigned long long)c));
        } else {
            const float lx = (__log2f(float(rho) + 1.0f) + c_log2fact[i]) * c_inv[i];
            const float est = exp2f(lx) + 0.5f * float(i - 1);
            cc = max(est >= float(c) ? c : int(est), i - 1);
            while (binom_at(binom, BK, cc, i) > rho) cc--;
            while (cc < c && binom_at(binom, BK, cc + 1, i) <= rho) cc++;
        }
        e[i - 1] = cc;
        rho -= binom_at(binom, BK, cc, i);
        c = cc - 1;
    }
}

// colex successor of the ascending M-subset e, in registers
template <int M>
__device__ __forceinline__ void tc_succ(int (&e)[kTcMaxPart]) {
    int q = M - 1;
#pragma unroll
    for (int k = M - 2; k >= 0; k--)
        if (e[k] + 1 != e[k + 1]) q = k;
#pragma unroll
    for (int k = 0; k < M; k++) {
        if (k < q) e[k] = k;
        else if (k == q) e[k]++;
    }
}

// sign words and mask count of rows off + e[k] (k < M), plus row `first` when FIRST
template <int M, int KW, bool FIRST>
__device__ __forceinline__ void tc_gather(const uint32_t *sg, const short *mk, int off, int first,
                                          const int (&e)[kTcMaxPart], uint32_t (&sw)[KW], int &cnt) {
#pragma unroll
    for (int w = 0; w < KW; w++) sw[w] = FIRST ? sg[first * KW + w] : 0u;
    cnt = FIRST ? int(mk[first] >= 0) : 0;
#pragma unroll
    for (int k = 0; k < M; k++) {
        const int rr = off + e[k];
        cnt += mk[rr] >= 0;
#pragma unroll
        for (int w = 0; w < KW; w++) sw[w] ^= sg[rr * KW + w];
    }
}

// slot of the c-th head tile of the kernel, and its phase parity
__device__ __forceinline__ int tc_slot(int c) { return c % kTcSlots; }
__device__ __forceinline__ uint32_t tc_slot_par(int c) { return (c / kTcSlots) & 1; }

#ifdef SDB_TC_TRACE
// Timeline of block 0 (variant builds): SM clock stamps per stage / head tile of the MMA warp
// (actor 0), the epilogue warps (1..8) and one producer warp per group (9, 10); printed by the
// last launch's block 0 at exit, analysed offline (tools/tc_trace.py).
constexpr int kTrN = 192, kTrS0 = 3000, kTrC0 = 300;
__device__ long long g_tct[12][4][kTrN];
#define TCT(actor, ev, idx, base)                                                         \
    do {                                                                                  \
        if (blockIdx.x == 0 && unsigned((idx) - (base)) < unsigned(kTrN) && (threadIdx.x & 31) == 0) \
            g_tct[actor][ev][(idx) - (base)] = clock64();                                 \
    } while (0)
#define TCT_V(actor, ev, idx, base, val)                                                  \
    do {                                                                                  \
        if (blockIdx.x == 0 && unsigned((idx) - (base)) < unsigned(kTrN) && (threadIdx.x & 31) == 0) \
            g_tct[actor][ev][(idx) - (base)] = (val);                                     \
    } while (0)
#else
#define TCT(actor, ev, idx, base)
#define TCT_V(actor, ev, idx, base, val)
#endif
#ifdef SDB_TC_LAT
// signalling latencies between the MMA warp and the epilogue (variant builds): SM clock stamps
// through shared memory; block 0 prints the averages
__device__ unsigned long long g_tc_lat[8];
#endif
// Unroll factor of the epilogue's stage loop. Inside an unrolled body ptxas hoists the next
// stage's tfull wait into the current stage's OR tree; the best factor follows the tail tiles per
// chunk, which follow the row bytes (measured on the g = 9 levels: K = 64, nbt = 10: 4.51 ms with
// 5, 4.64 with 3 or 4, 4.73 with 8, 4.90 with 2, 4.85 with 1; K = 96, nbt = 5: 126.8 ms with 2 or 3, 129.9 with 5,
// 132.2 with 1, 139.9 with 4).
#ifdef SDB_TC_EPI_UNROLL
template <int KW> constexpr int kTcEpiUnroll = SDB_TC_EPI_UNROLL;
#else
template <int KW> constexpr int kTcEpiUnroll = KW <= 2 ? 5 : 2;
#endif
#ifndef SDB_TC_RUN
#define SDB_TC_RUN 8  // units claimed per dispenser atomic (measured g = 9: 4.51 / 4.48 / 4.53 ms with 4 / 8 / 16)
#endif
struct TcShared {
#ifdef SDB_TC_LAT
    volatile long long lat_commit[kTcStages], lat_arrive[kTcStages], lat_acc[8];
#endif
    uint64_t uqfull[kTcUnitQ], uqempty[kTcUnitQ], afull[kTcSlots], aempty[kTcSlots], bfull[kTcMaxBSlots],
        bempty[kTcMaxBSlots],
        tfull[kTcStages], tempty[kTcStages];
};
// shared-window addresses of the mbarrier arrays (bar i of an array at base + 8 i), computed
// once per thread
struct TcBars {
    uint32_t uqfull, uqempty, afull, aempty, bfull, bempty, tfull, tempty;
    __device__ explicit TcBars(TcShared &sh) {
        const uint32_t b = tc::smem_u32(&sh);
        uqfull = b + uint32_t(offsetof(TcShared, uqfull));
        uqempty = b + uint32_t(offsetof(TcShared, uqempty));
        afull = b + uint32_t(offsetof(TcShared, afull));
        aempty = b + uint32_t(offsetof(TcShared, aempty));
        bfull = b + uint32_t(offsetof(TcShared, bfull));
        bempty = b + uint32_t(offsetof(TcShared, bempty));
        tfull = b + uint32_t(offsetof(TcShared, tfull));
        tempty = b + uint32_t(offsetof(TcShared, tempty));
    }
};
__device__ __forceinline__ uint32_t bar_at(uint32_t base, int i) { return base + 8u * uint32_t(i); }

// Producer thread pq (0..255): this unit's tails pq * nbt .. + nbt - 1, tail pq * nbt + r into
// row pq of the chunk's tile r. Tile r is ring fill Fc + r: slot (Fc + r) % nsb, written once
// the MMA released that slot's previous fill (sempty), announced with sfull per tile.
template <int T1, int KW>
__device__ void tc_write_tails(const TcUnitDesc &d, const TcGammaDev &gm, int pq, int lane, int N, int kmax,
                               const uint32_t *sg, const short *mk, const unsigned long long *binom, int BKs,
                               unsigned char *sB, unsigned long long Fc, int nsb, const TcBars &bars) {
    const int b = d.b, R = d.nbt, i0 = pq * R;
    int e[kTcMaxPart];
    tc_unrank<T1>(d.t0 + min(i0, d.ntails - 1), N - 1 - b, binom, BKs, e);
    int slot = int(Fc % unsigned(nsb));
    uint32_t epar = uint32_t((Fc / unsigned(nsb)) & 1u) ^ 1u;  // parity of the release a fill waits for
    const size_t tile_bytes = size_t(kTcTileN) * kmax;
    for (int r = 0; r < R; r++) {
        if (r > 0 && i0 + r < d.ntails) tc_succ<T1>(e);
        uint32_t sw[KW];
        int cnt;
        tc_gather<T1, KW, true>(sg, mk, b + 1, b, e, sw, cnt);
        SDB_CHECK(slot >= 0 && slot < nsb && (T1 > 0 ? b + 1 + e[T1 - 1] : b) < N);
        if (lane == 0) tc::mbar_wait_a(bar_at(bars.bempty, slot), epar);
        __syncwarp();
        unsigned char *tile = sB + size_t(slot) * tile_bytes;
        const int trow = pq;
#pragma unroll
        for (int w = 0; w < KW; w++)
            if (w < gm.K / 32) tc_store_block<false>(tile, kTcTileN, trow, w, sw[w], gm.W1);
        if (mk[b] >= 0) tile[tc::kmajor_off(kTcTileN, trow, mk[b])] = 0;
#pragma unroll
        for (int k = 0; k < T1; k++) {
            const int cc = mk[b + 1 + e[k]];
            if (cc >= 0) tile[tc::kmajor_off(kTcTileN, trow, cc)] = 0;
        }
        tile[tc::kmajor_off(kTcTileN, trow, gm.kc)] = (unsigned char)(-(gm.alpha * cnt));
        tile[tc::kmajor_off(kTcTileN, trow, gm.kt)] = 1;
        tile[tc::kmajor_off(kTcTileN, trow, gm.kt + 1)] = 16;
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(bar_at(bars.bfull, slot));
        if (++slot == nsb) {
            slot = 0;
            epar ^= 1u;
        }
    }
}

// Producer group g, thread pt (0..127): row pt of the unit's head tiles a with (c0 + a) % 2 == g
// (c0 = the kernel-wide index of the unit's first tile); returns the tiles this group wrote.
template <int H, int KW>
__device__ int tc_write_heads(const TcUnitDesc &d, const TcGammaDev &gm, int g, int pt, int lane, int c0, int kmax,
                              const uint32_t *sg, const short *mk, const unsigned long long *binom, int BKs,
                              unsigned char *sA, const TcBars &bars, const unsigned *s_thr,
                              unsigned sshift, int a_from, int a_to) {
    const int r0 = pt * d.na;
    int e[kTcMaxPart];
    int a = a_from + ((g - c0 - a_from) & 1);  // this group's first tile in [a_from, a_to)
    a_to = min(a_to, d.na);
    if (a >= a_to) return 0;
    tc_unrank<H>(d.hbase0 + min(r0 + a, d.nheads - 1), d.b, binom, BKs, e);
    const size_t a_slot = size_t(kTcHeads) * kmax;
    int wrote = 0;
    for (; a < a_to; a += 2) {
        if (wrote > 0) {
            if (r0 + a - 1 < d.nheads) tc_succ<H>(e);
            if (r0 + a < d.nheads) tc_succ<H>(e);
        }
        uint32_t sw[KW];
        int cnt;
        tc_gather<H, KW, false>(sg, mk, 0, 0, e, sw, cnt);
        const int c = c0 + a, s = tc_slot(c);
        SDB_CHECK(s >= 0 && s < kTcSlots && (H == 0 || e[H - 1] < d.b) && pt < kTcHeads);
        if (pt < 32) TCT(9 + g, 0, c, kTrC0);
        if (lane == 0) tc::mbar_wait_a(bar_at(bars.aempty, s), tc_slot_par(c) ^ 1);
        __syncwarp();
        if (pt < 32) TCT(9 + g, 1, c, kTrC0);
        unsigned char *tile = sA + size_t(s) * a_slot;
#pragma unroll
        for (int w = 0; w < KW; w++)
            if (w < gm.K / 32) tc_store_block<true>(tile, kTcHeads, pt, w, sw[w], 0);
#pragma unroll
        for (int k = 0; k < H; k++) {
            const int cc = mk[e[k]];
            if (cc >= 0) tile[tc::kmajor_off(kTcHeads, pt, cc)] = 0;
        }
        // the threshold, folded into the MMA: the accumulator of a pair is val - T - 1 (T from
        // the CTA's current bound; rows past the unit's heads never pass)
        const int chv = gm.alpha * cnt;
        const int T = r0 + a < d.nheads ? gm.S * int(*(volatile const unsigned *)s_thr >> sshift) - gm.C0 - chv
                                        : -32768;
        int tr = 0, tq = 0;
        tc_threshold_bytes(T, tr, tq);
        tile[tc::kmajor_off(kTcHeads, pt, gm.kt)] = (unsigned char)tr;
        tile[tc::kmajor_off(kTcHeads, pt, gm.kt + 1)] = (unsigned char)tq;
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_a(bar_at(bars.afull, s));
        if (pt < 32) TCT(9 + g, 2, c, kTrC0);
        wrote++;
    }
    return wrote;
}

#ifdef SDB_TC_PROF
#define TCP_ARGS , tcp_t0, tcp_acc
#define TCP_PARAMS , unsigned long long &tcp_t0, unsigned long long (&tcp_acc)[8]
#else
#define TCP_ARGS
#define TCP_PARAMS
#endif

// The MMA thread's inner loop: one head tile (descriptor aT) against the unit's nbt tail tiles,
// one TMEM stage each. Kept lean: the tensor pipe takes about one MMA ahead, so every cycle
// the issuer spends between MMAs is a bubble.
// a relaxed (not .sys) load of a word other CTAs update with atomics
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#ifdef SDB_TC_GAPS
// stage-to-stage issue gaps of the MMA warp, by boundary kind: 0 inside a head tile, 1 first
// stage of a head tile, 2 first stage of a unit (block 0 prints them)
struct TcGaps {
    unsigned long long last = 0, sum[3] = {0, 0, 0}, n[3] = {0, 0, 0}, wait[3] = {0, 0, 0}, afw = 0, uqw = 0;
};
#define TCG_PARAMS , TcGaps &gp, int kind0
#define TCG_ARGS(k) , gaps, (k)
#define TCGU_PARAMS , TcGaps &gaps
#define TCGU_ARGS , gaps
#else
#define TCG_PARAMS
#define TCG_ARGS(k)
#define TCGU_PARAMS
#define TCGU_ARGS
#endif

// The MMA warp's inner loop: one head tile (descriptor aT) against the chunk's nbt tail tiles,
// one TMEM stage each. Tail tile nb is ring fill Fc + nb (slot bslot0 + nb mod nsb); `release`
// (the chunk's last head tile) hands each slot back (sempty) as soon as its stage's MMAs finish.
// Kept lean: every operand is warp-uniform by construction (kernel parameters, loop counters
// and the unit's packed word taken through redux.sync), so ptxas keeps descriptors, barrier
// addresses and loop state in uniform registers and the path from a stage's tempty wait to its
// UTCIMMA is a handful of instructions; the tensor pipe takes about one MMA ahead, so every
// cycle the issuer spends between MMAs is a bubble.
template <int KT>
__device__ __forceinline__ void tc_mma_stages(uint64_t aT, uint64_t bD, uint32_t b_tile16, int nbt, int bslot0,
                                              uint32_t bpar0, int nsb, bool bwait, bool release, uint32_t tbase,
                                              uint32_t idesc, uint32_t &st, uint32_t &tpar,
                                              const TcBars &bars TCP_PARAMS TCG_PARAMS, int &sidx, int ctile) {
    int slot = bslot0;
    uint32_t bpar = bpar0;
    for (int nb = 0; nb < nbt; nb++) {
#ifdef SDB_TC_GAPS
        const unsigned long long w0 = clock64();
#endif
        // this stage's operands, ready before the wait (tc::mma_stage)
        const uint32_t dT = tbase + st * kTcTileN;
        const uint64_t bT = bD + uint64_t(uint32_t(slot) * b_tile16);
#if defined(SDB_TC_GAPS) || defined(SDB_TC_PROF) || defined(SDB_TC_NOMMA)
        TCP_BEGIN
        tc::mbar_wait_u(bar_at(bars.tempty, st), tpar ^ 1);
        TCP_END(3)
        if (bwait) tc::mbar_wait_u(bar_at(bars.bfull, slot), bpar);  // a chunk's first head tile only
#ifdef SDB_TC_GAPS
        {
            const unsigned long long now = clock64();
            const int kind = nb == 0 ? kind0 : 0;
            if (gp.last) {
                gp.sum[kind] += now - gp.last;
                gp.wait[kind] += now - w0;
                gp.n[kind]++;
            }
            gp.last = now;
        }
#endif
        TCP_BEGIN
        tc::fence_after();
#ifndef SDB_TC_NOMMA  // pipeline experiments: the MMAs skipped
#pragma unroll
        for (int k = 0; k < KT; k++)
            tc::mma_i8_elect(dT, aT + uint64_t(k * 2 * kTcHeads), bT + uint64_t(k * 2 * kTcTileN), idesc, k > 0);
#endif
        tc::commit_elect_a(bar_at(bars.tfull, st));
        if (release) tc::commit_elect_a(bar_at(bars.bempty, slot));
        TCP_END(4)
#else
        TCT(0, 0, sidx, kTrS0);
        TCT_V(11, 0, sidx, kTrS0, ctile);
        tc::mma_stage<KT>(bar_at(bars.tempty, st), tpar ^ 1, bar_at(bars.bfull, slot), bpar, bwait, dT, aT, bT,
                          2 * kTcHeads, 2 * kTcTileN, idesc, bar_at(bars.tfull, st), bar_at(bars.bempty, slot), release);
        TCT(0, 1, sidx, kTrS0);
        sidx++;
#ifdef SDB_TC_LAT
        if ((threadIdx.x & 31) == 0) {
            const long long now = clock64();
            TcShared *shp = reinterpret_cast<TcShared *>(__cvta_shared_to_generic(bars.uqfull - offsetof(TcShared, uqfull)));
            if (shp->lat_arrive[st] && !bwait) {
                shp->lat_acc[0] += now - shp->lat_arrive[st];  // arrive -> next commit issue
                shp->lat_acc[1] += 1;
            }
            shp->lat_commit[st] = now;
        }
#endif
#endif
        st ^= 1u;
        tpar ^= st ^ 1u;  // flips after stage 1
        if (++slot == nsb) {
            slot = 0;
            bpar ^= 1u;
        }
    }
}

// All head tiles of one unit (KT fixed per Gamma: one dispatch per unit, not per tile).
template <int KT>
__device__ __forceinline__ void tc_mma_unit(int na, int nbt, bool restage, bool chunk_last, int &c, uint64_t aD,
                                            uint32_t a_slot16, uint64_t bD, uint32_t b_tile16, int bslot0,
                                            uint32_t bpar0, int nsb, uint32_t tbase, uint32_t idesc, uint32_t &st,
                                            uint32_t &tpar, const TcBars &bars TCP_PARAMS TCGU_PARAMS, int &sidx) {
    for (int a = 0; a < na; a++, c++) {
        const int s = tc_slot(c);
        const uint64_t aT = aD + uint64_t(uint32_t(s) * a_slot16);
        TCT(0, 2, sidx, kTrS0);
#ifndef SDB_TC_MMA_NOAFULL
#ifdef SDB_TC_GAPS
        const unsigned long long aw0 = clock64();
#endif
        TCP_BEGIN
        tc::mbar_wait_u(bar_at(bars.afull, s), tc_slot_par(c));
        TCP_END(2)
#ifdef SDB_TC_GAPS
        gaps.afw += clock64() - aw0;
#endif
#endif
        // the tail tiles were written for the chunk's first head tile; its last frees the slots
        tc_mma_stages<KT>(aT, bD, b_tile16, nbt, bslot0, bpar0, nsb, restage && a == 0, chunk_last && a == na - 1,
                          tbase, idesc, st, tpar, bars TCP_ARGS TCG_ARGS(a == 0 ? 2 : 1), sidx, c);
        tc::commit_elect_a(bar_at(bars.aempty, s));
    }
}

#ifdef SDB_TC_COUNT_RARE
__device__ unsigned long long g_tc_rare[4];  // calls, flagged rows, flagged (row, stage) pairs (variant builds)
#endif
// Rare path of the epilogue, once per head tile and out of line (its registers stay out of the
// stage loop): some head row of the warp met a pair below the folded threshold in the stages of
// `stage_hits`. The TMEM stages are long released, so the warp recomputes: for each flagged
// (row, stage) its lanes take the stage's 128 columns of this warp's half through the exact
// path (exact weight against the current bound, syndromes, key). Returns the warp's new bound.
template <int W>
__device__ __noinline__ unsigned tc_rare_rows(const ProblemDev p, const TilePlan tl, const uint32_t *s_rows,
                                              const unsigned long long *s_binom, int BKs, const TileUnit *un,
                                              unsigned stage_hits, int hoff, int half, int nbt, int ntails, int nheads,
                                              unsigned thrH) {
    const int lane = threadIdx.x & 31;
    unsigned rows_hit = __ballot_sync(0xffffffffu, stage_hits != 0);
#ifdef SDB_TC_COUNT_RARE
    if (lane == 0) {
        atomicAdd(&g_tc_rare[0], 1ull);
        atomicAdd(&g_tc_rare[1], (unsigned long long)__popc(rows_hit));
    }
    atomicAdd(&g_tc_rare[2], (unsigned long long)__popc(stage_hits));
#endif
    while (rows_hit) {
        const int L = __ffs(rows_hit) - 1;
        rows_hit &= rows_hit - 1;
        unsigned stL = __shfl_sync(0xffffffffu, stage_hits, L);
        const int hoffL = __shfl_sync(0xffffffffu, hoff, L);
        while (stL) {
            const int nb = __ffs(stL) - 1;
            stL &= stL - 1;
#pragma unroll 1
            for (int i = lane; i < 128; i += 32) {
                const int y = nb * kTcTileN + half * 128 + i;  // B row of the unit
                const int tix = min((y % (kTcProdWarps * 32)) * nbt + y / (kTcProdWarps * 32), ntails - 1);
                SDB_CHECK(tix >= 0 && tix < ntails && hoffL >= 0 && hoffL < nheads);
                thrH = tile_exact<W>(p, tl, s_rows, s_binom, BKs, un, hoffL, tix, thrH);
            }
        }
    }
    return __reduce_min_sync(0xffffffffu, thrH);  // the bound is global
}

template <int W, int KW>
__global__ void __launch_bounds__(kTcThreads, 1) tc_tile_kernel(ProblemDev p, TcPlan tp) {
    if (run_done(p)) return;
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    __shared__ TcShared sh;
    __shared__ uint32_t s_tbase;
    __shared__ unsigned long long s_visited;
    __shared__ unsigned s_thr;  // the CTA's bound (scaled weight units): producers fold it into head rows
    const TilePlan &tl = tp.tile;
    const int G = p.G, N = p.N, kmax = tp.kmax;
    const int BKs = min(p.BK, tl.g + 2);
    const TcSmem lay = tc_smem_layout(G, N, W, kmax, KW, tp.nbt, BKs);
    unsigned char *smem = tc_smem;
    unsigned char *sA = smem + lay.a, *sB = smem + lay.b;
    uint32_t *s_sign = reinterpret_cast<uint32_t *>(smem + lay.sign);
    short *s_mask = reinterpret_cast<short *>(smem + lay.mask);
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem + lay.rows);
    unsigned long long *s_binom = reinterpret_cast<unsigned long long *>(smem + lay.binom);
    TcUnitDesc *s_uq = reinterpret_cast<TcUnitDesc *>(smem + lay.uq);
    TcGammaDev *s_gam = reinterpret_cast<TcGammaDev *>(smem + lay.gam);
    unsigned long long *s_cum = reinterpret_cast<unsigned long long *>(smem + lay.cum);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    for (int i = threadIdx.x; i < G * N * 2 * W; i += blockDim.x) s_rows[i] = p.rows[i];
    for (int i = threadIdx.x; i < G * N * KW; i += blockDim.x) s_sign[i] = tp.sign[i];
    for (int i = threadIdx.x; i < G * N; i += blockDim.x) s_mask[i] = tp.mask[i];
    for (int i = threadIdx.x; i < (N + 1) * BKs; i += blockDim.x) s_binom[i] = p.binom[(i / BKs) * p.BK + i % BKs];
    for (int i = threadIdx.x; i < G; i += blockDim.x) s_gam[i] = tp.gam[i];
    for (int i = threadIdx.x; i <= G * tl.nb; i += blockDim.x) s_cum[i] = tl.cum[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcUnitQ; s++) {
            tc::mbar_init(&sh.uqfull[s], 1);
            tc::mbar_init(&sh.uqempty[s], kTcProdWarps + 1 + kTcEpiWarps);  // producers, MMA thread, epilogue
        }
        for (int s = 0; s < kTcSlots; s++) {
            tc::mbar_init(&sh.afull[s], kTcProdWarps / 2);   // the four warps of the writing group
            tc::mbar_init(&sh.aempty[s], 1);                 // the MMA commit after the tile's last stage
        }
        for (int s = 0; s < kTcMaxBSlots; s++) {
            tc::mbar_init(&sh.bfull[s], kTcProdWarps);
            tc::mbar_init(&sh.bempty[s], 1);
        }
        for (int s = 0; s < kTcStages; s++) {
            tc::mbar_init(&sh.tfull[s], 1);
            tc::mbar_init(&sh.tempty[s], 32 * kTcEpiWarps);  // every epilogue thread (no lane test, no warp sync)
        }
        tc::mbar_fence_init();
        s_visited = 0;
        s_thr = start_threshold(p, tl.thr0);
#ifdef SDB_TC_LAT
        for (int i = 0; i < kTcStages; i++) sh.lat_commit[i] = sh.lat_arrive[i] = 0;
        for (int i = 0; i < 8; i++) sh.lat_acc[i] = 0;
#endif
    }
    if (warp == 0) tc::tmem_alloc(&s_tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = s_tbase;
    const TcBars bars(sh);
    const size_t a_slot = size_t(kTcHeads) * kmax;           // bytes per head tile
    const int nsb = tp.nbt + 1;                              // B ring slots (tail tiles)

    if (warp == 0) {
        // ------------------------------------------------------------ MMA issuer: the whole
        // warp runs the loop converged (warp-uniform values stay in uniform registers); one
        // elected lane issues each tcgen05.mma / commit (tc::mma_i8_elect, tc::commit_elect)
        {
            const uint32_t idesc = tc::idesc_i8(kTcHeads, kTcTileN);
            // operand descriptors; an offset of x bytes is + (x >> 4) on the start-address field
            const uint64_t aD = tc::sdesc(tc::smem_u32(sA), kTcHeads * 16, 128);
            const uint64_t bD = tc::sdesc(tc::smem_u32(sB), kTcTileN * 16, 128);
            const uint32_t a_slot16 = uint32_t(a_slot >> 4);
            const uint32_t b_tile16 = uint32_t((size_t(kTcTileN) * kmax) >> 4);
            const uint32_t tb_u = __reduce_or_sync(0xffffffffu, tbase);  // the same value, known warp-uniform
            int ts = 0;
            // B ring: slot and phase parity of the current chunk's first fill and of the next free fill
            int bslot_c = 0, bslot_n = 0;
            uint32_t bpar_c = 0, bpar_n = 0;
            uint32_t st = 0, tpar = 0;  // next TMEM stage and the parity its tempty wait expects
#ifdef SDB_TC_GAPS
            TcGaps gaps;
#endif
            int c = 0;
            int sidx = 0;
            TCP_DECL
            const unsigned long long tcp_start = clock64();
            for (int u = 0;; u++) {
                TCP_BEGIN
                tc::mbar_wait_u(bar_at(bars.uqfull, u % kTcUnitQ), (u / kTcUnitQ) & 1);
                TCP_END(0)
                // the unit's packed word (tc_unit_word), made warp-uniform for the compiler
                const unsigned mw = __reduce_or_sync(0xffffffffu, unsigned(s_uq[u % kTcUnitQ].pad));
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_a(bar_at(bars.uqempty, u % kTcUnitQ));
                if (mw & kTcWordEnd) {
#ifdef SDB_TC_GAPS
                    if (blockIdx.x == 0 && lane == 0)
                        printf("[tcgaps] afull wait avg %.1f per tile | in-tile %llu stages avg %.1f (wait %.1f) | tile start %llu avg %.1f (wait %.1f) | unit start %llu avg %.1f (wait %.1f)\n",
                               double(gaps.afw) / max(1ull, gaps.n[1] + gaps.n[2]),
                               gaps.n[0], double(gaps.sum[0]) / max(1ull, gaps.n[0]), double(gaps.wait[0]) / max(1ull, gaps.n[0]),
                               gaps.n[1], double(gaps.sum[1]) / max(1ull, gaps.n[1]), double(gaps.wait[1]) / max(1ull, gaps.n[1]),
                               gaps.n[2], double(gaps.sum[2]) / max(1ull, gaps.n[2]), double(gaps.wait[2]) / max(1ull, gaps.n[2]));
#endif
#ifdef SDB_TC_PROF
                    if (blockIdx.x == 0 && lane == 0) printf("[tcprof] mma: total %llu wait_uq %llu wait_bfull %llu wait_afull %llu wait_tempty %llu issue %llu stages %d\n", clock64() - tcp_start, tcp_acc[0], tcp_acc[1], tcp_acc[2], tcp_acc[3], tcp_acc[4], ts);
#endif
                    break;
                }
                const int na = int(mw & 0xffu), nbt = int((mw >> 8) & 0xffu), KT = int((mw >> 16) & 0xfu);
                const bool restage = (mw & kTcWordRestage) != 0, chunk_last = (mw & kTcWordChunkLast) != 0;
                if (restage) {
                    bslot_c = bslot_n;
                    bpar_c = bpar_n;
                    bslot_n += nbt;  // nbt < nsb: at most one wrap
                    if (bslot_n >= nsb) {
                        bslot_n -= nsb;
                        bpar_n ^= 1u;
                    }
                }
                switch (KT) {
#define SDB_TC_UNIT(k)                                                                                       \
    case k:                                                                                                  \
        tc_mma_unit<k>(na, nbt, restage, chunk_last, c, aD, a_slot16, bD, b_tile16, bslot_c, bpar_c, nsb, tb_u, \
                       idesc, st, tpar, bars TCP_ARGS TCGU_ARGS, sidx);                                      \
        break;
                    SDB_TC_UNIT(1) SDB_TC_UNIT(2) SDB_TC_UNIT(3)
                    default: tc_mma_unit<4>(na, nbt, restage, chunk_last, c, aD, a_slot16, bD, b_tile16, bslot_c, bpar_c,
                                            nsb, tb_u, idesc, st, tpar, bars TCP_ARGS TCGU_ARGS, sidx);
                        break;
#undef SDB_TC_UNIT
                }
                ts += na * nbt;
            }
        }
    } else if (warp <= kTcEpiWarps) {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;             // TMEM lane quarter this warp may read
        const int half = (warp - 1) >> 2;   // which 128 columns of a stage
        const int row = 32 * q + lane;      // head row of the tile = TMEM lane
        const uint32_t ta0 = tbase + (uint32_t(32 * q) << 16) + uint32_t(half * 128);  // + st * 256
        unsigned thrH = start_threshold(p, tl.thr0);
        unsigned s_thr_seen = thrH;  // this warp's last bound published to s_thr
        unsigned wmin_next = thrH;   // the level minimum as loaded at the previous head tile
        // the current TMEM stage's full/empty barriers and columns, flipped per stage with XOR
        // masks (keeps the per-stage loop free of index arithmetic)
        uint32_t st_e = 0, tpar_e = 0;
        uint32_t tf_st = bar_at(bars.tfull, 0), te_st = bar_at(bars.tempty, 0), ta_st = ta0;
        const uint32_t tf_x = tf_st ^ bar_at(bars.tfull, 1), te_x = te_st ^ bar_at(bars.tempty, 1),
                       ta_x = ta0 ^ (ta0 + uint32_t(kTcTileN));
        int c = 0;  // head tiles consumed
        int sidx = 0;
#ifdef SDB_TC_LAT
        long long lat_r[4] = {0, 0, 0, 0};
#endif
        TCP_DECL
        const unsigned long long tcp_start = clock64();
        for (int u = 0;; u++) {
            TCP_BEGIN
            tc::mbar_wait_a(bar_at(bars.uqfull, u % kTcUnitQ), (u / kTcUnitQ) & 1);
            TCP_END(0)
            const TcUnitDesc d = s_uq[u % kTcUnitQ];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_a(bar_at(bars.uqempty, u % kTcUnitQ));
            if (d.end) {
#ifdef SDB_TC_LAT
                if (blockIdx.x == 0 && lane == 0 && (warp == 1 || warp == 8) && lat_r[3] > 5000)
                    printf("[tclat] epi warp %d: commit issue->seen %.1f | waiting %.1f | seen->release %.1f | stages %lld | mma: arrive(w8)->commit issue %.1f\n",
                           warp, double(lat_r[0]) / lat_r[3], double(lat_r[1]) / lat_r[3], double(lat_r[2]) / lat_r[3], lat_r[3],
                           double(sh.lat_acc[0]) / double(max(1ll, (long long)sh.lat_acc[1])));
#endif
#ifdef SDB_TC_PROF
                if (blockIdx.x == 0 && lane == 0 && (warp == 1 || warp == 5)) printf("[tcprof] epi warp %d: total %llu wait_uq %llu wait_afull %llu wait_tfull %llu work %llu\n", warp, clock64() - tcp_start, tcp_acc[0], tcp_acc[1], tcp_acc[2], tcp_acc[3]);
#endif
                break;
            }
            TileUnit un;
            un.j = d.j;
            un.b = d.b;
            un.t0 = d.t0;
            un.hbase0 = d.hbase0;
            un.tcount = d.ntails;
            un.pad = d.nheads;
            for (int a = 0; a < d.na; a++, c++) {
                const int hoff = row * d.na + a;  // this row's head: rank hbase0 + hoff
                // other CTAs' finds: the value loaded one head tile ago (its L2 latency hidden
                // behind that tile's stages) tightens the bound now; load the next one
                thrH = min(thrH, wmin_next);
                wmin_next = ld_relaxed_u32(&p.state->wmin);
                unsigned stage_hits = 0;  // bit nb: this row has a pair below the folded threshold in stage nb
#pragma unroll kTcEpiUnroll<KW>
                for (int nb = 0; nb < d.nbt; nb++) {
                    TCP_BEGIN
#ifdef SDB_TC_LAT
                    const long long lat_enter = clock64();
#endif
                    TCT(warp, 0, sidx, kTrS0);
                    tc::mbar_wait_a(tf_st, tpar_e);
                    TCT(warp, 1, sidx, kTrS0);
                    TCP_END(2)
#ifdef SDB_TC_LAT
                    const long long lat_seen = clock64();
                    lat_r[0] += lat_seen - sh.lat_commit[st_e];  // commit issue -> seen
                    lat_r[1] += lat_seen - lat_enter;             // spent waiting
                    lat_r[3] += 1;
#endif
                    TCP_BEGIN
                    tc::fence_after();
                    uint32_t v[64];
                    tc::ld64_pack(ta_st, v);
                    tc::ld_wait();
#ifdef SDB_TC_LAT
                    {
                        const long long now = clock64();
                        lat_r[2] += now - lat_seen;  // seen -> release
                        if (warp == 8 && lane == 0) sh.lat_arrive[st_e] = now;
                    }
#endif
                    // the accumulators are in registers: hand the TMEM stage back to the MMA
                    // warp before looking at them (the stage's release is on the kernel's
                    // critical path, the sign test is not)
                    tc::fence_before();
                    tc::mbar_arrive_a(te_st);
                    TCT(warp, 2, sidx, kTrS0);
                    // a pair passes the folded threshold iff its 16-bit accumulator is negative:
                    // OR the packed words as a tree of 3-input ORs (depth 4; ptxas turns a plain OR
                    // reduction into one 32-deep dependent LOP3 chain) and note, per head row, the
                    // stages whose two sign bits come out set. No vote and no branch here: the
                    // rows are looked at once per head tile.
                    uint32_t r[22];
#pragma unroll
                    for (int i = 0; i < 21; i++) r[i] = tc::or3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
                    r[21] = v[63];
                    uint32_t r2[8];
#pragma unroll
                    for (int i = 0; i < 7; i++) r2[i] = tc::or3(r[3 * i], r[3 * i + 1], r[3 * i + 2]);
                    r2[7] = r[21];
                    uint32_t o = tc::or3(tc::or3(r2[0], r2[1], r2[2]), tc::or3(r2[3], r2[4], r2[5]), r2[6] | r2[7]);
#if defined(SDB_TC_NOMMA) || defined(SDB_TC_NOPROD)
                    o = 0;  // TMEM / the operands hold no real data
#endif
                    if (o & 0x80008000u) stage_hits |= 1u << nb;
                    // next stage: flip the TMEM stage (and the phase parity after stage 1)
                    tf_st ^= tf_x;
                    te_st ^= te_x;
                    ta_st ^= ta_x;
                    tpar_e ^= st_e;
                    st_e ^= 1u;
                    TCT(warp, 3, sidx, kTrS0);
                    sidx++;
                    TCP_END(3)
                }
                if (hoff >= d.nheads) stage_hits = 0;  // rows past the unit's heads never pass
                if (__any_sync(0xffffffffu, stage_hits != 0))
                    thrH = tc_rare_rows<W>(p, tl, s_rows, s_binom, BKs, &un, stage_hits, hoff, half, d.nbt, d.ntails,
                                           d.nheads, thrH);
                // hand a tighter bound to the producers' next head tiles (s_thr_seen is
                // warp-uniform; the loop above is too, so the whole warp gets here)
                if (__any_sync(0xffffffffu, thrH < s_thr_seen)) {
                    const unsigned m = __reduce_min_sync(0xffffffffu, thrH);
                    if (lane == 0) atomicMin(&s_thr, m);
                    s_thr_seen = m;
                }
            }
        }
    } else if (warp == kTcEpiWarps + 1) {
        // ------------------------------------------------------------ unit warp (lane 0)
        if (lane == 0) {
            const unsigned long long local_units =
                (tl.unit_total + tl.shard_world - 1 - tl.shard_rank) / tl.shard_world;
            constexpr int kHB = kTcHeads * kTcUnitTiles;  // heads per unit
            int sj = -1, sb = -1;
            unsigned long long st0 = 0, claim = 0, claim_end = 0, seen = 0, visited = 0, skipped = 0;
            int lo = 0;  // (Gamma, b) index of the previous unit: units of a run mostly share it
            // the next unit in dispensing order (skipping what the early exit leaves out)
            auto next_unit = [&](TcUnitDesc &d) {
                for (;;) {
                    d = TcUnitDesc{};
                    if (claim == claim_end) {
                        // consecutive units mostly share their tail chunk: longer runs restage less
                        // often; single units near the end keep the SMs level
                        constexpr unsigned long long kRun = SDB_TC_RUN;
                        const unsigned long long run = seen + kRun * 4 * gridDim.x < local_units ? kRun : 1ull;
                        claim = atomicAdd(tl.counter, run);
                        claim_end = claim + run;
                        seen = claim_end;
                    }
                    const unsigned long long unit = (claim++) * tl.shard_world + tl.shard_rank;
                    d.end = unit >= tl.unit_total;
                    if (d.end) return;
                    if (!(s_cum[lo] <= unit && unit < s_cum[lo + 1])) {
                        int l = 0, hi = G * tl.nb - 1;
                        while (l < hi) {
                            const int mid = (l + hi + 1) >> 1;
                            if (s_cum[mid] <= unit) l = mid; else hi = mid - 1;
                        }
                        lo = l;
                    }
                    SDB_CHECK(lo >= 0 && lo < G * tl.nb && s_cum[lo] <= unit && unit < s_cum[lo + 1]);
                    const int b = tl.h + lo % tl.nb;
                    const unsigned long long uu = unit - s_cum[lo];
                    const unsigned long long Hb = binom_at(s_binom, BKs, b, tl.h);
                    const unsigned long long Tb = binom_at(s_binom, BKs, N - 1 - b, tl.t - 1);
                    const unsigned long long nH = (Hb + kHB - 1) / kHB;
                    const unsigned long long tcn = uu / nH, hc = uu % nH;
                    d.j = lo / tl.nb;
                    d.b = b;
                    d.t0 = tcn * tl.tchunk;
                    d.ntails = int(min((unsigned long long)tl.tchunk, Tb - d.t0));
                    d.nbt = (d.ntails + kTcTileN - 1) / kTcTileN;
                    d.hbase0 = hc * kHB;
                    d.nheads = int(min((unsigned long long)kHB, Hb - d.hbase0));
                    d.na = (d.nheads + kTcHeads - 1) / kTcHeads;
                    if ((unsigned long long)d.j > (early_key(p, tl.lprev) >> kKeyRankBits)) {
                        // mid-level early exit: a later Gamma's keys all exceed the best one
                        skipped += (unsigned long long)d.nheads * (unsigned long long)d.ntails;
                        continue;
                    }
                    d.restage = d.j != sj || b != sb || d.t0 != st0;
                    sj = d.j;
                    sb = b;
                    st0 = d.t0;
                    visited += (unsigned long long)d.nheads * (unsigned long long)d.ntails;
                    return;
                }
            };
            // one unit of lookahead: a unit is published once the next one is known, so it can
            // say whether its tail chunk ends with it (the MMA then frees the B ring slots tile by
            // tile during the unit's last head tile)
            TcUnitDesc pend;
            next_unit(pend);
            for (int u = 0;; u++) {
                TcUnitDesc nd{};
                if (pend.end) nd.end = 1; else next_unit(nd);
                pend.chunk_last = nd.end || nd.restage;
                pend.pad = int(tc_unit_word(pend, pend.end ? 0 : s_gam[pend.j].K / 32));
                tc::mbar_wait_a(bar_at(bars.uqempty, u % kTcUnitQ), ((u / kTcUnitQ) & 1) ^ 1);
                s_uq[u % kTcUnitQ] = pend;
                tc::mbar_arrive_a(bar_at(bars.uqfull, u % kTcUnitQ));
                if (pend.end) break;
                pend = nd;
            }
            s_visited = visited;
            if (skipped) atomicAdd(&p.state->skipped, skipped);
        }
    } else {
        // ------------------------------------------------------------ producers
        const unsigned sshift = p.scale == 2 ? 1u : 0u;
        const int pw = warp - (kTcEpiWarps + 2);   // 0..7
        const int g = pw >> 2;                     // group: head tiles c with c % 2 == g
        const int pt = 32 * (pw & 3) + lane;       // head row
        const int pq = 32 * pw + lane;             // tail thread index (0..255)
        int c0 = 0;                                // kernel-wide index of the unit's first head tile
        unsigned long long Fc = 0, Fn = 0;         // B ring: the current chunk's first fill, the next free fill
        for (int u = 0;; u++) {
            tc::mbar_wait_a(bar_at(bars.uqfull, u % kTcUnitQ), (u / kTcUnitQ) & 1);
            const TcUnitDesc d = s_uq[u % kTcUnitQ];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_a(bar_at(bars.uqempty, u % kTcUnitQ));
            if (d.end) break;
            const TcGammaDev gm = s_gam[d.j];
            const uint32_t *sg = s_sign + size_t(d.j) * N * KW;
            const short *mk = s_mask + d.j * N;
            if (d.restage) {
                Fc = Fn;
                Fn += unsigned(d.nbt);
            }
#ifdef SDB_TC_NOPROD
            if (d.restage)
                for (int r = 0; r < d.nbt; r++) {
                    const unsigned long long F = Fc + unsigned(r);
                    const int slot = int(F % unsigned(nsb));
                    if (lane == 0) tc::mbar_wait_a(bar_at(bars.bempty, slot), uint32_t((F / unsigned(nsb)) & 1u) ^ 1u);
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_a(bar_at(bars.bfull, slot));
                }
            for (int a = (g - c0) & 1; a < d.na; a += 2) {
                const int s = tc_slot(c0 + a);
                if (lane == 0) tc::mbar_wait_a(bar_at(bars.aempty, s), tc_slot_par(c0 + a) ^ 1);
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_a(bar_at(bars.afull, s));
            }
#else
#define SDB_TC_HEADS(from, to)                                                                                \
    switch (tl.h) {                                                                                           \
        SDB_TC_HEADS_CASE(1, from, to) SDB_TC_HEADS_CASE(2, from, to) SDB_TC_HEADS_CASE(3, from, to)            \
        SDB_TC_HEADS_CASE(4, from, to) SDB_TC_HEADS_CASE(5, from, to) SDB_TC_HEADS_CASE(6, from, to)            \
        SDB_TC_HEADS_CASE(7, from, to) SDB_TC_HEADS_CASE(8, from, to)                                           \
    }
#define SDB_TC_HEADS_CASE(m, from, to)                                                                        \
    case m:                                                                                                   \
        tc_write_heads<m, KW>(d, gm, g, pt, lane, c0, kmax, sg, mk, s_binom, BKs, sA, bars, &s_thr, sshift, \
                              from, to);                                                                      \
        break;
            int a_from = 0;
            if (d.restage) {
                // the new chunk's first head tiles go first (the MMA needs them and tail tile 0 to
                // start); tail tiles follow, each as soon as the ring slot it takes is released
                SDB_TC_HEADS(0, 2)
                a_from = 2;
                switch (tl.t - 1) {
#define SDB_TC_TAILS(m) \
    case m: tc_write_tails<m, KW>(d, gm, pq, lane, N, kmax, sg, mk, s_binom, BKs, sB, Fc, nsb, bars); break;
                    SDB_TC_TAILS(0) SDB_TC_TAILS(1) SDB_TC_TAILS(2) SDB_TC_TAILS(3) SDB_TC_TAILS(4)
                    SDB_TC_TAILS(5) SDB_TC_TAILS(6) SDB_TC_TAILS(7) SDB_TC_TAILS(8)
#undef SDB_TC_TAILS
                }
            }
            SDB_TC_HEADS(a_from, d.na)
#undef SDB_TC_HEADS
#undef SDB_TC_HEADS_CASE
#endif
            c0 += d.na;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
#ifdef SDB_TC_COUNT_RARE
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("[tcrare] cumulative: calls %llu rows %llu (row, stage) pairs %llu\n", g_tc_rare[0], g_tc_rare[1], g_tc_rare[2]);
#endif
#ifdef SDB_TC_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_tct[0][0][kTrN - 1] != 0) {
        const long long t0 = g_tct[0][0][0];
        for (int a = 0; a < 12; a++)
            for (int e = 0; e < 4; e++)
                for (int i = 0; i < kTrN; i += 8) {
                    const long long *v = &g_tct[a][e][i];
                    const long long b = a == 11 ? 0 : t0;
                    printf("[tct] %d %d %d %lld %lld %lld %lld %lld %lld %lld %lld\n", a, e, i, v[0] ? v[0] - b : -1,
                           v[1] ? v[1] - b : -1, v[2] ? v[2] - b : -1, v[3] ? v[3] - b : -1, v[4] ? v[4] - b : -1,
                           v[5] ? v[5] - b : -1, v[6] ? v[6] - b : -1, v[7] ? v[7] - b : -1);
                }
        for (int a = 0; a < 12; a++)
            for (int e = 0; e < 4; e++)
                for (int i = 0; i < kTrN; i++) g_tct[a][e][i] = 0;
    }
#endif
    if (threadIdx.x == 0 && s_visited) atomicAdd(&p.state->visited, s_visited);
}

template <int W, int KW>
int launch_tc_impl(const ProblemDev &p, const TcPlan &tp, cudaStream_t st, int num_sms) {
    const size_t smem = tc_smem_layout(p.G, p.N, W, tp.kmax, KW, tp.nbt, min(p.BK, tp.tile.g + 2)).total;
    if (smem > kTcSmemMax) return -1;
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(done.load() & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(tc_tile_kernel<W, KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmemMax));
        done.fetch_or(1ull << (dev & 63));
    }
    const unsigned long long units = (tp.tile.unit_total + tp.tile.shard_world - 1 - tp.tile.shard_rank) / tp.tile.shard_world;
    unsigned long long blocks = (unsigned long long)num_sms;
    if (blocks > units) blocks = units;
    if (blocks == 0) return 0;
    tc_tile_kernel<W, KW><<<unsigned(blocks), kTcThreads, smem, st>>>(p, tp);
    return 1;
}

template <int W>
int launch_tc_w(const ProblemDev &p, const TcPlan &tp, cudaStream_t st, int num_sms) {
    switch (tp.kw) {
        case 1: return launch_tc_impl<W, 1>(p, tp, st, num_sms);
        case 2: return launch_tc_impl<W, 2>(p, tp, st, num_sms);
        case 3: return launch_tc_impl<W, 3>(p, tp, st, num_sms);
        case 4: return launch_tc_impl<W, 4>(p, tp, st, num_sms);
    }
    return -1;
}
