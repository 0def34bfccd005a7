// Tensor-core tile kernel (device.hpp: TcPlan). Included by kernels.cu inside its anonymous
// namespace: it shares binom_at, tile_exact, TileUnit, run_done and start_threshold with the
// POPC tile kernel.
//
// Warp roles, one CTA per SM (kTcThreads = 416):
//   warp 0        TMEM owner (512 columns: two 128 x 256 s32 stages); lane 0 issues the MMAs
//   warps 1..8    epilogue: tcgen05.ld pack::16b -> packed 16-bit minimum -> threshold test
//   warps 9..12   producers: claim units, write the tail tiles (B, double-buffered) and the
//                 head tiles (A, kTcSlots-deep ring) as int8 coordinates in the canonical
//                 K-major no-swizzle layout (8-row x 16-byte core matrices)
// Pipelines (mbarriers): A slot full/empty, B buffer full/empty, TMEM stage full/empty.
//
// A unit is (Gamma j, boundary b, up to 1024 heads, up to 256 nbt tails): its na <= 8 head
// tiles each meet all of its nbt tail tiles. Producer thread r owns head row r of every tile
// of the unit — na consecutive colex ranks, one successor step per tile — and 2 nbt
// consecutive tails of the unit's chunk, so the element lists stay in registers and no
// thread unranks more than twice per unit.
#pragma once

#include "tc_ptx.cuh"

struct TcUnitInfo {
    unsigned long long hbase0, t0;
    int j, b, nheads, ntails, nbt, na, restage, end;
};

__device__ __forceinline__ void tc_prod_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcProdWarps) : "memory"); }

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

// colex unrank of rho into an m-subset of [0, lim) (m <= kTcMaxPart), ascending, in registers:
// the estimate of unrank_colex_est with its loops unrolled over the compile-time bound
__device__ __forceinline__ void tc_unrank(unsigned long long rho, int m, int lim, const unsigned long long *binom, int BK,
                                          int (&e)[kTcMaxPart]) {
    int c = lim - 1;
#pragma unroll
    for (int i = kTcMaxPart; i >= 1; i--) {
        if (i <= m) {
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
}

// colex successor of the ascending m-subset e (1 <= m <= kTcMaxPart), in registers
__device__ __forceinline__ void tc_succ(int m, int (&e)[kTcMaxPart]) {
    int q = m - 1;
#pragma unroll
    for (int k = kTcMaxPart - 2; k >= 0; k--)
        if (k < m - 1 && e[k] + 1 != e[k + 1]) q = k;
#pragma unroll
    for (int k = 0; k < kTcMaxPart; k++) {
        if (k < q) e[k] = k;
        else if (k == q) e[k]++;
    }
}

template <int W>
__global__ void __launch_bounds__(kTcThreads, 1) tc_tile_kernel(ProblemDev p, TcPlan tp) {
    if (run_done(p)) return;
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    __shared__ uint64_t bar_afull[kTcSlots], bar_aempty[kTcSlots], bar_bfull[2], bar_bempty[2], bar_tfull[2],
        bar_tempty[2];
    __shared__ uint32_t s_tbase;
    __shared__ unsigned long long s_claim, s_claim_end, s_visited;
    __shared__ int s_staged_j, s_staged_b;
    __shared__ unsigned long long s_staged_t0;
    __shared__ TcUnitInfo s_pu;
    const TilePlan &tl = tp.tile;
    const int G = p.G, N = p.N, kmax = tp.kmax, kw = tp.kw;
    const int BKs = min(p.BK, tl.g + 2);
    const TcSmem lay = tc_smem_layout(G, N, W, kmax, kw, tp.nbt, BKs);
    unsigned char *smem = tc_smem;
    unsigned char *sA = smem + lay.a, *sB = smem + lay.b;
    uint32_t *s_sign = reinterpret_cast<uint32_t *>(smem + lay.sign);
    short *s_mask = reinterpret_cast<short *>(smem + lay.mask);
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem + lay.rows);
    unsigned long long *s_binom = reinterpret_cast<unsigned long long *>(smem + lay.binom);
    TcMeta *s_meta = reinterpret_cast<TcMeta *>(smem + lay.meta);
    TcGammaDev *s_gam = reinterpret_cast<TcGammaDev *>(smem + lay.gam);
    unsigned long long *s_cum = reinterpret_cast<unsigned long long *>(smem + lay.cum);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    for (int i = threadIdx.x; i < G * N * 2 * W; i += blockDim.x) s_rows[i] = p.rows[i];
    for (int i = threadIdx.x; i < G * N * kw; i += blockDim.x) s_sign[i] = tp.sign[i];
    for (int i = threadIdx.x; i < G * N; i += blockDim.x) s_mask[i] = tp.mask[i];
    for (int i = threadIdx.x; i < (N + 1) * BKs; i += blockDim.x) s_binom[i] = p.binom[(i / BKs) * p.BK + i % BKs];
    for (int i = threadIdx.x; i < G; i += blockDim.x) s_gam[i] = tp.gam[i];
    for (int i = threadIdx.x; i <= G * tl.nb; i += blockDim.x) s_cum[i] = tl.cum[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcSlots; s++) {
            tc::mbar_init(&bar_afull[s], 1);
            tc::mbar_init(&bar_aempty[s], 1 + kTcEpiWarps);
        }
        for (int s = 0; s < 2; s++) {
            tc::mbar_init(&bar_bfull[s], 1);
            tc::mbar_init(&bar_bempty[s], 1);
            tc::mbar_init(&bar_tfull[s], 1);
            tc::mbar_init(&bar_tempty[s], kTcEpiWarps);
        }
        tc::mbar_fence_init();
        s_claim = s_claim_end = 0;
        s_visited = 0;
        s_staged_j = -1;
        s_staged_b = -1;
        s_staged_t0 = 0;
    }
    if (warp == 0) tc::tmem_alloc(&s_tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = s_tbase;
    const size_t a_slot = size_t(kTcHeads) * kmax;                // bytes per head tile
    const size_t b_buf = size_t(tp.nbt) * kTcTileN * kmax;        // bytes per tail buffer

    if (warp == 0) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_i8(kTcHeads, kTcTileN);
            const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
            int ts = 0, cur_bb = -1;
            int uses[2] = {0, 0};
            for (int it = 0;; it++) {
                const int s = it % kTcSlots;
                tc::mbar_wait(&bar_afull[s], (it / kTcSlots) & 1);
                const TcMeta &m = s_meta[s];
                if (m.end) break;
                if (m.restage) {
                    if (cur_bb >= 0) tc::commit(&bar_bempty[cur_bb]);  // old buffer free once its MMAs finish
                    cur_bb = m.bb;
                    tc::mbar_wait(&bar_bfull[cur_bb], uses[cur_bb] & 1);
                    uses[cur_bb]++;
                }
                const int KT = s_gam[m.j].K / 32, nbt = m.nbt;
                tc::fence_after();
                const uint32_t a0 = aBase + uint32_t(s * a_slot);
                for (int nb = 0; nb < nbt; nb++, ts++) {
                    const int st = ts & 1;
                    tc::mbar_wait(&bar_tempty[st], ((ts >> 1) & 1) ^ 1);
                    tc::fence_after();
                    const uint32_t b0 = bBase + uint32_t(cur_bb * b_buf + size_t(nb) * kTcTileN * kmax);
                    for (int k = 0; k < KT; k++) {
                        const uint64_t ad = tc::sdesc(a0 + k * 2 * (kTcHeads * 16), kTcHeads * 16, 128);
                        const uint64_t bd = tc::sdesc(b0 + k * 2 * (kTcTileN * 16), kTcTileN * 16, 128);
                        tc::mma_i8(tbase + st * kTcTileN, ad, bd, idesc, k > 0);
                    }
                    tc::commit(&bar_tfull[st]);
                }
                tc::commit(&bar_aempty[s]);
            }
        }
    } else if (warp <= kTcEpiWarps) {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;             // TMEM lane quarter this warp may read
        const int half = (warp - 1) >> 2;   // which 128 columns of a stage
        const int row = 32 * q + lane;      // head row of the tile = TMEM lane
        const unsigned sshift = p.scale == 2 ? 1u : 0u;
        unsigned thrH = start_threshold(p, tl.thr0);
        int ts = 0;
        for (int it = 0;; it++) {
            const int s = it % kTcSlots;
            tc::mbar_wait(&bar_afull[s], (it / kTcSlots) & 1);
            const TcMeta &m = s_meta[s];
            const int end = m.end;
            TileUnit un;
            un.j = m.j;
            un.b = m.b;
            un.t0 = m.t0;
            un.hbase0 = m.hbase0;
            un.tcount = m.ntails;
            un.pad = m.nheads;
            const int nbt = m.nbt;
            const int hoff = row * m.na + m.a;  // this row's head: rank hbase0 + hoff
            const int ch = m.ch[row];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar_aempty[s]);
            if (end) break;
            const TcGammaDev gm = s_gam[un.j];
            // other CTAs' finds tighten the threshold from the next tile on (the load's latency
            // overlaps this tile's stages)
            const unsigned wmin_seen = *(volatile unsigned int *)&p.state->wmin;
            int T = hoff < un.pad ? gm.S * int(thrH >> sshift) - gm.C0 - ch : -32768;
            for (int nb = 0; nb < nbt; nb++, ts++) {
                const int st = ts & 1;
                tc::mbar_wait(&bar_tfull[st], (ts >> 1) & 1);
                tc::fence_after();
                const uint32_t ta = tbase + (uint32_t(32 * q) << 16) + uint32_t(st * kTcTileN + half * 128);
                uint32_t v0[16], v1[16], v2[16], v3[16];
                tc::ld16_pack(ta, v0);
                tc::ld16_pack(ta + 32, v1);
                tc::ld16_pack(ta + 64, v2);
                tc::ld16_pack(ta + 96, v3);
                tc::ld_wait();
                uint32_t mn = v0[0];
#pragma unroll
                for (int i = 1; i < 16; i++) mn = __vmins2(mn, v0[i]);
#pragma unroll
                for (int i = 0; i < 16; i++) mn = __vmins2(__vmins2(mn, v1[i]), __vmins2(v2[i], v3[i]));
                const int lo = int(short(mn & 0xFFFFu)), hi = int(short(mn >> 16));
                if (min(lo, hi) <= T) {
                    // rare: the exact path for every pair at or below the threshold
                    uint32_t all[64];
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        all[i] = v0[i];
                        all[16 + i] = v1[i];
                        all[32 + i] = v2[i];
                        all[48 + i] = v3[i];
                    }
                    const int R = 2 * nbt;
                    for (int x = 0; x < 128; x++) {
                        const int val = int(short(all[x >> 1] >> (16 * (x & 1))));
                        if (val > T) continue;
                        const int y = nb * kTcTileN + half * 128 + x;  // B row -> tail rank offset
                        const int tix = min((y & 127) * R + (y >> 7), un.tcount - 1);
                        thrH = tile_exact<W>(p, tl, s_rows, s_binom, BKs, &un, hoff, tix, thrH);
                        T = gm.S * int(thrH >> sshift) - gm.C0 - ch;
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar_tempty[st]);
            }
            thrH = min(thrH, wmin_seen);
        }
    } else {
        // ------------------------------------------------------------ producers
        const int pt = threadIdx.x - 32 * (1 + kTcEpiWarps);
        const unsigned long long local_units = (tl.unit_total + tl.shard_world - 1 - tl.shard_rank) / tl.shard_world;
        constexpr int kHB = kTcHeads * kTcUnitTiles;  // heads per unit
        int cur_bb = -1;
        int fills[2] = {0, 0};
        int lo = 0;  // (Gamma, b) index of the previous unit (pt == 0): units of a run share it mostly
        unsigned long long seen = 0;
        int it = 0;  // head tiles produced
        for (;;) {
            if (pt == 0) {
                TcUnitInfo u{};
                if (s_claim == s_claim_end) {
                    const unsigned long long run = seen + 4ull * 4 * gridDim.x < local_units ? 4ull : 1ull;
                    s_claim = atomicAdd(tl.counter, run);
                    s_claim_end = s_claim + run;
                    seen = s_claim + run;
                }
                const unsigned long long unit = (s_claim++) * tl.shard_world + tl.shard_rank;
                u.end = unit >= tl.unit_total;
                if (!u.end) {
                    if (!(s_cum[lo] <= unit && unit < s_cum[lo + 1])) {
                        int l = 0, hi = G * tl.nb - 1;
                        while (l < hi) {
                            const int mid = (l + hi + 1) >> 1;
                            if (s_cum[mid] <= unit) l = mid; else hi = mid - 1;
                        }
                        lo = l;
                    }
                    const int b = tl.h + lo % tl.nb;
                    const unsigned long long uu = unit - s_cum[lo];
                    const unsigned long long Hb = binom_at(s_binom, BKs, b, tl.h);
                    const unsigned long long Tb = binom_at(s_binom, BKs, N - 1 - b, tl.t - 1);
                    const unsigned long long nH = (Hb + kHB - 1) / kHB;
                    const unsigned long long tc = uu / nH, hc = uu % nH;
                    u.j = lo / tl.nb;
                    u.b = b;
                    u.t0 = tc * tl.tchunk;
                    u.ntails = int(min((unsigned long long)tl.tchunk, Tb - u.t0));
                    u.nbt = (u.ntails + kTcTileN - 1) / kTcTileN;
                    u.hbase0 = hc * kHB;
                    u.nheads = int(min((unsigned long long)kHB, Hb - u.hbase0));
                    u.na = (u.nheads + kTcHeads - 1) / kTcHeads;
                    u.restage = u.j != s_staged_j || b != s_staged_b || u.t0 != s_staged_t0;
                    s_staged_j = u.j;
                    s_staged_b = b;
                    s_staged_t0 = u.t0;
                    s_visited += (unsigned long long)u.nheads * (unsigned long long)u.ntails;
                }
                s_pu = u;
            }
            tc_prod_sync();
            const TcUnitInfo u = s_pu;
            tc_prod_sync();
            if (u.end) {
                if (pt == 0) {
                    const int s = it % kTcSlots;
                    tc::mbar_wait(&bar_aempty[s], ((it / kTcSlots) & 1) ^ 1);
                    s_meta[s].end = 1;
                    tc::mbar_arrive(&bar_afull[s]);
                }
                break;
            }
            const TcGammaDev gm = s_gam[u.j];
            const int KT = gm.K / 32;
            const uint32_t *sg = s_sign + size_t(u.j) * N * kw;
            const short *mk = s_mask + u.j * N;
            if (u.restage) {
                const int bb = cur_bb < 0 ? 0 : cur_bb ^ 1;
                tc::mbar_wait(&bar_bempty[bb], (fills[bb] & 1) ^ 1);
                fills[bb]++;
                cur_bb = bb;
                // tails {b} + colex (t-1)-subsets of (b, N): this thread takes the R = 2 nbt
                // consecutive ranks t0 + pt R .. and writes rank pt R + r to row r * 128 + pt;
                // ranks past ntails repeat the last tail (their candidates are duplicates)
                unsigned char *buf = sB + size_t(bb) * b_buf;
                const int t = tl.t, b = u.b;
                const int R = 2 * u.nbt;
                const int i0 = pt * R;
                int e[kTcMaxPart];
                tc_unrank(u.t0 + min(i0, u.ntails - 1), t - 1, N - 1 - b, s_binom, BKs, e);
                for (int r = 0; r < R; r++) {
                    if (r > 0 && i0 + r < u.ntails) tc_succ(t - 1, e);
                    uint32_t sw[kTcMaxK / 32];
                    int cnt = mk[b] >= 0;
#pragma unroll
                    for (int w = 0; w < kTcMaxK / 32; w++) sw[w] = w < kw ? sg[b * kw + w] : 0u;
#pragma unroll
                    for (int k = 0; k < kTcMaxPart; k++)
                        if (k < t - 1) {
                            const int rr = b + 1 + e[k];
                            cnt += mk[rr] >= 0;
#pragma unroll
                            for (int w = 0; w < kTcMaxK / 32; w++)
                                if (w < kw) sw[w] ^= sg[rr * kw + w];
                        }
                    const int y = r * kTcHeads + pt;  // B row
                    unsigned char *tile = buf + size_t(y / kTcTileN) * kTcTileN * kmax;
                    const int trow = y % kTcTileN;
#pragma unroll
                    for (int w = 0; w < kTcMaxK / 32; w++)
                        if (w < KT) tc_store_block<false>(tile, kTcTileN, trow, w, sw[w], gm.W1);
                    if (mk[b] >= 0) tile[tc::kmajor_off(kTcTileN, trow, mk[b])] = 0;
#pragma unroll
                    for (int k = 0; k < kTcMaxPart; k++)
                        if (k < t - 1) {
                            const int c = mk[b + 1 + e[k]];
                            if (c >= 0) tile[tc::kmajor_off(kTcTileN, trow, c)] = 0;
                        }
                    tile[tc::kmajor_off(kTcTileN, trow, gm.kc)] = (unsigned char)(-(gm.alpha * cnt));
                }
                tc::fence_async_smem();
                tc_prod_sync();
                if (pt == 0) tc::mbar_arrive(&bar_bfull[bb]);
            }
            // the unit's head tiles: row pt of tile a is head rank hbase0 + pt * na + a (rows past
            // nheads repeat the last head; the epilogue ignores them)
            const int h = tl.h;
            const int r0 = pt * u.na;
            int e[kTcMaxPart];
            tc_unrank(u.hbase0 + min(r0, u.nheads - 1), h, u.b, s_binom, BKs, e);
            for (int a = 0; a < u.na; a++, it++) {
                if (a > 0 && r0 + a < u.nheads) tc_succ(h, e);
                const int s = it % kTcSlots;
                uint32_t sw[kTcMaxK / 32];
#pragma unroll
                for (int w = 0; w < kTcMaxK / 32; w++) sw[w] = 0;
                int cnt = 0;
#pragma unroll
                for (int k = 0; k < kTcMaxPart; k++)
                    if (k < h) {
                        cnt += mk[e[k]] >= 0;
#pragma unroll
                        for (int w = 0; w < kTcMaxK / 32; w++)
                            if (w < kw) sw[w] ^= sg[e[k] * kw + w];
                    }
                if (pt == 0) tc::mbar_wait(&bar_aempty[s], ((it / kTcSlots) & 1) ^ 1);
                tc_prod_sync();
                unsigned char *tile = sA + size_t(s) * a_slot;
#pragma unroll
                for (int w = 0; w < kTcMaxK / 32; w++)
                    if (w < KT) tc_store_block<true>(tile, kTcHeads, pt, w, sw[w], 0);
#pragma unroll
                for (int k = 0; k < kTcMaxPart; k++)
                    if (k < h) {
                        const int c = mk[e[k]];
                        if (c >= 0) tile[tc::kmajor_off(kTcHeads, pt, c)] = 0;
                    }
                TcMeta &m = s_meta[s];
                m.ch[pt] = short(gm.alpha * cnt);
                if (pt == 0) {
                    m.hbase0 = u.hbase0;
                    m.t0 = u.t0;
                    m.j = u.j;
                    m.b = u.b;
                    m.nheads = u.nheads;
                    m.ntails = u.ntails;
                    m.nbt = u.nbt;
                    m.bb = cur_bb;
                    m.restage = a == 0 ? u.restage : 0;
                    m.end = 0;
                    m.a = a;
                    m.na = u.na;
                }
                tc::fence_async_smem();
                tc_prod_sync();
                if (pt == 0) tc::mbar_arrive(&bar_afull[s]);
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
    if (threadIdx.x == 0 && s_visited) atomicAdd(&p.state->visited, s_visited);
}

template <int W>
int launch_tc_impl(const ProblemDev &p, const TcPlan &tp, cudaStream_t st, int num_sms) {
    const size_t smem = tc_smem_layout(p.G, p.N, W, tp.kmax, tp.kw, tp.nbt, min(p.BK, tp.tile.g + 2)).total;
    if (smem > kTcSmemMax) return -1;
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(done.load() & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(tc_tile_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTcSmemMax));
        done.fetch_or(1ull << (dev & 63));
    }
    const unsigned long long units = (tp.tile.unit_total + tp.tile.shard_world - 1 - tp.tile.shard_rank) / tp.tile.shard_world;
    unsigned long long blocks = (unsigned long long)num_sms;
    if (blocks > units) blocks = units;
    if (blocks == 0) return 0;
    tc_tile_kernel<W><<<unsigned(blocks), kTcThreads, smem, st>>>(p, tp);
    return 1;
}
