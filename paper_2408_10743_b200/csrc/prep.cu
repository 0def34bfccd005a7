// Batch prep on the device (BASELINE config 3): one warp per code
// runs the host prep of the isometry route — validate_normalizer (distance.cpp:71-93),
// isometry_transform (prep.cpp:299-315), information_sets (prep.cpp:317-364) and the
// admissibility syndromes (engine.cpp:14-29) — and writes the batch kernel's inputs.
//
// Rows live in registers, two per lane (row i: lane i % 32, slot i / 32). Every elimination
// step is warp-uniform: a ballot finds the pivot row (first row >= r with a 1 in column c,
// exactly the host's and the reference's rule), shuffles broadcast it, and each lane XORs it
// into its own rows. So the Gamma_j — and the bound trace — are the host's bit for bit.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.hpp"

namespace sdb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// word i of a register array without dynamic indexing (which would put the array in local
// memory)
template <int NW>
__device__ __forceinline__ unsigned long long word_at(const unsigned long long (&w)[NW], int i) {
    unsigned long long x = w[0];
#pragma unroll
    for (int k = 1; k < NW; k++)
        if (i == k) x = w[k];
    return x;
}

template <int NW>
__device__ __forceinline__ void or_at(unsigned long long (&w)[NW], int i, unsigned long long v) {
#pragma unroll
    for (int k = 0; k < NW; k++)
        if (i == k) w[k] |= v;
}

// image rows: 3n <= 192 columns -> 3 words; normalizer rows: 2n <= 128 -> 2 words
template <int S, int NW>
struct WarpRows {
    unsigned long long v[2][NW];  // rows lane and lane + 32 (slot 1 only when S == 2)

    __device__ __forceinline__ bool bit(int slot, int c) const { return (word_at(v[slot], c >> 6) >> (c & 63)) & 1ull; }

    // row i broadcast to every lane (i warp-uniform)
    __device__ __forceinline__ void fetch(int i, unsigned long long (&out)[NW]) const {
        const int slot = i >> 5, src = i & 31;
#pragma unroll
        for (int w = 0; w < NW; w++) out[w] = __shfl_sync(kFull, (S == 2 && slot) ? v[1][w] : v[0][w], src);
    }

    // one step of the reference's elimination (bitvec.cpp:213-233 / prep.cpp:330-346): the
    // first row sel >= r with a 1 in column c becomes row r and is XORed into every other
    // row with a 1 there. Returns false when no row qualifies.
    __device__ __forceinline__ bool pivot(int c, int r, int rows) {
        const int lane = threadIdx.x & 31;
        const unsigned b0 = __ballot_sync(kFull, lane < rows && lane >= r && bit(0, c));
        const unsigned b1 = S == 2 ? __ballot_sync(kFull, lane + 32 < rows && lane + 32 >= r && bit(1, c)) : 0u;
        if (!(b0 | b1)) return false;
        const int sel = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
        unsigned long long prow[NW], rrow[NW];
        fetch(sel, prow);
        fetch(r, rrow);
        if (sel != r) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                const int i = lane + 32 * s;
                if (i == r)
#pragma unroll
                    for (int w = 0; w < NW; w++) v[s][w] = prow[w];
                else if (i == sel)
#pragma unroll
                    for (int w = 0; w < NW; w++) v[s][w] = rrow[w];
            }
        }
#pragma unroll
        for (int s = 0; s < S; s++) {
            const int i = lane + 32 * s;
            if (i < rows && i != r && bit(s, c))
#pragma unroll
                for (int w = 0; w < NW; w++) v[s][w] ^= prow[w];
        }
        return true;
    }
};

// columns [from, from + len) of a packed NW-word row, len <= 64
template <int NW>
__device__ __forceinline__ unsigned long long bits_at(const unsigned long long (&w)[NW], int from, int len) {
    const int wi = from >> 6, sh = from & 63;
    unsigned long long x = 0;
#pragma unroll
    for (int i = 0; i < NW; i++)
        if (i == wi) x = w[i] >> sh;
    if (sh)
#pragma unroll
        for (int i = 1; i < NW; i++)
            if (i == wi + 1) x |= w[i] << (64 - sh);
    return len == 64 ? x : (x & ((1ull << len) - 1));
}

template <int S>
__global__ void __launch_bounds__(128) batch_prep_kernel(BatchPrepDev d) {
    const int lane = threadIdx.x & 31;
    const int code = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (code >= d.codes) return;
    const int N = d.N, n = d.n;
    __shared__ unsigned char s_piv[4][3 * kPrepMaxN];
    unsigned char *piv = s_piv[threadIdx.x >> 5];

    // ---- load the normalizer (a|b): row i of this code
    WarpRows<S, 2> A;
#pragma unroll
    for (int s = 0; s < S; s++) {
        const int i = lane + 32 * s;
#pragma unroll
        for (int w = 0; w < 2; w++)
            A.v[s][w] = (i < N && w < d.in_words) ? d.normalizers[((size_t)code * N + i) * d.in_words + w] : 0ull;
    }
    // mask padding bits beyond 2n
#pragma unroll
    for (int s = 0; s < S; s++)
#pragma unroll
        for (int w = 0; w < 2; w++) {
            const int lo = 64 * w, hi = min(2 * n, 64 * w + 64);
            if (hi <= lo) A.v[s][w] = 0;
            else if (hi - lo < 64) A.v[s][w] &= (1ull << (hi - lo)) - 1;
        }
    int status = 0;

    // ---- validate_normalizer (distance.cpp:71-93); shape checks are done on the host
    if (d.validate) {
        WarpRows<S, 2> E = A;  // echelon form of A (rank, in_rowspace)
        int r = 0;
        for (int c = 0; c < 2 * n && r < N; c++)
            if (E.pivot(c, r, N)) piv[r++] = (unsigned char)c;
        const int rankA = r;
        if (rankA != N) {
            status = 2;
        } else {
            // symplectic dual = Euclidean kernel of the half-swapped rows (bitvec.cpp:261-274)
            WarpRows<S, 2> Sd;
#pragma unroll
            for (int s = 0; s < S; s++) {
                const unsigned long long a = bits_at(A.v[s], 0, n), b = bits_at(A.v[s], n, n);
                // (b | a) packed at columns [0, n) and [n, 2n)
                unsigned long long lo = b, hi = 0;
                if (n < 64) {
                    lo |= a << n;
                    hi = n == 0 ? 0 : (a >> (64 - n));
                } else {
                    hi = a;
                }
                Sd.v[s][0] = lo;
                Sd.v[s][1] = 2 * n > 64 ? hi : 0;
            }
            __shared__ unsigned char s_spiv[4][2 * kPrepMaxN];
            unsigned char *spiv = s_spiv[threadIdx.x >> 5];
            int rs = 0;
            for (int c = 0; c < 2 * n && rs < N; c++)
                if (Sd.pivot(c, rs, N)) spiv[rs++] = (unsigned char)c;
            // free columns in ascending order; dual vector f: e_f + sum_r S[r][f] e_{spiv[r]}
            // two free columns per lane (n - k <= 64)
            unsigned long long dv[2][2] = {{0, 0}, {0, 0}};
            int fcol[2] = {-1, -1};
            {
                int nf = 0, pi = 0;
                for (int c = 0; c < 2 * n; c++) {
                    if (pi < rs && spiv[pi] == c) { pi++; continue; }
                    if ((nf & 31) == lane) {
                        if (nf >> 5) fcol[1] = c;
                        else fcol[0] = c;
                    }
                    nf++;
                }
            }
#pragma unroll
            for (int s = 0; s < S; s++)
                if (fcol[s] >= 0) or_at(dv[s], fcol[s] >> 6, 1ull << (fcol[s] & 63));
            for (int q = 0; q < rs; q++) {
                unsigned long long row[2];
                Sd.fetch(q, row);
#pragma unroll
                for (int s = 0; s < S; s++)
                    if (fcol[s] >= 0 && ((word_at(row, fcol[s] >> 6) >> (fcol[s] & 63)) & 1ull))
                        or_at(dv[s], spiv[q] >> 6, 1ull << (spiv[q] & 63));
            }
            // in_rowspace(A, v): reduce by the echelon rows of A
            for (int q = 0; q < rankA; q++) {
                unsigned long long row[2];
                E.fetch(q, row);
                const int pc = piv[q];
#pragma unroll
                for (int s = 0; s < S; s++)
                    if ((word_at(dv[s], pc >> 6) >> (pc & 63)) & 1ull) {
                        dv[s][0] ^= row[0];
                        dv[s][1] ^= row[1];
                    }
            }
            const bool bad = (dv[0][0] | dv[0][1] | dv[1][0] | dv[1][1]) != 0;
            if (__any_sync(kFull, bad)) status = 2;
        }
    }

    // ---- isometry_transform: (a | b | a^b) in 3n <= 192 columns
    WarpRows<S, 3> cur;
#pragma unroll
    for (int s = 0; s < S; s++) {
        const unsigned long long a = bits_at(A.v[s], 0, n), b = bits_at(A.v[s], n, n), c = a ^ b;
        unsigned long long out[3] = {0, 0, 0};
        // place a at 0, b at n, c at 2n
        const unsigned long long parts[3] = {a, b, c};
#pragma unroll
        for (int p = 0; p < 3; p++) {
            const int from = p * n, wi = from >> 6, sh = from & 63;
            out[wi] |= parts[p] << sh;
            if (sh && wi + 1 < 3 && n > 64 - sh) out[wi + 1] |= parts[p] >> (64 - sh);
        }
#pragma unroll
        for (int w = 0; w < 3; w++) cur.v[s][w] = out[w];
    }

    // ---- information_sets (prep.cpp:317-364): greedy elimination on unused columns, cur
    // carried over between matrices, rank_deficit = rows - pivots
    unsigned long long used[3] = {0, 0, 0};
    unsigned long long gx[kPrepGammaSlots][2], gz[kPrepGammaSlots][2];
#pragma unroll
    for (int j = 0; j < kPrepGammaSlots; j++) gx[j][0] = gx[j][1] = gz[j][0] = gz[j][1] = 0;
    int G = 0;
    const int W = d.W, rowlen = 2 * d.W;
    for (; status == 0;) {
        int r = 0;
        for (int c = 0; c < 3 * n && r < N; c++) {
            if ((word_at(used, c >> 6) >> (c & 63)) & 1ull) continue;
            if (cur.pivot(c, r, N)) piv[r++] = (unsigned char)c;
        }
        if (r == 0) break;
        if (G == 0 && r != N) {  // information_sets: rows are linearly dependent
            status = 2;
            break;
        }
        if (G < d.Gs) {
            // rows of Gamma_G: x = columns [0, n), z = columns [n, 2n) of the image
#pragma unroll
            for (int s = 0; s < S; s++) {
                const unsigned long long x = bits_at(cur.v[s], 0, n), z = bits_at(cur.v[s], n, n);
#pragma unroll
                for (int j = 0; j < kPrepGammaSlots; j++)
                    if (j == G) {
                        gx[j][s] = x;
                        gz[j][s] = z;
                    }
                const int i = lane + 32 * s;
                if (i >= N) continue;
                uint32_t *dst = d.rows + (((size_t)code * d.Gs + G) * N + i) * rowlen;
                for (int w = 0; w < W; w++) {
                    dst[w] = uint32_t(x >> (32 * w));
                    dst[W + w] = uint32_t(z >> (32 * w));
                }
            }
            if (lane == 0) d.deficits[(size_t)code * d.Gs + G] = N - r;
        }
        for (int q = 0; q < r; q++) or_at(used, piv[q] >> 6, 1ull << (piv[q] & 63));
        G++;
    }

    // ---- admissibility syndromes: bit f of row i = <first 2n columns of row i, A_f>_s;
    // N <= 64 so the raw syndrome is one word (zero iff the compressed one is zero)
    if (status == 0 && d.filter) {
        unsigned long long syn[kPrepGammaSlots][2];
#pragma unroll
        for (int j = 0; j < kPrepGammaSlots; j++) syn[j][0] = syn[j][1] = 0;
        for (int f = 0; f < N; f++) {
            unsigned long long arow[2];
            A.fetch(f, arow);
            const unsigned long long fa = bits_at(arow, 0, n), fb = bits_at(arow, n, n);
#pragma unroll
            for (int j = 0; j < kPrepGammaSlots; j++)
#pragma unroll
                for (int s = 0; s < S; s++)
                    syn[j][s] |= (unsigned long long)((__popcll(gx[j][s] & fb) + __popcll(gz[j][s] & fa)) & 1) << f;
        }
        const int gs = min(G, d.Gs);
#pragma unroll
        for (int j = 0; j < kPrepGammaSlots; j++)
#pragma unroll
            for (int s = 0; s < S; s++) {
                const int i = lane + 32 * s;
                if (j < gs && i < N) d.syn[((size_t)code * d.Gs + j) * N + i] = syn[j][s];
            }
    }
    // pad unused slots with Gamma_0 and a deficit that never reaches L (duplicates cannot
    // lower the minimum)
    if (status == 0 && G > 0)
        for (int j = G; j < d.Gs; j++) {
            for (int i = lane; i < N; i += 32) {
                const uint32_t *src = d.rows + (((size_t)code * d.Gs) * N + i) * rowlen;
                uint32_t *dst = d.rows + (((size_t)code * d.Gs + j) * N + i) * rowlen;
                for (int w = 0; w < rowlen; w++) dst[w] = src[w];
                if (d.filter) d.syn[((size_t)code * d.Gs + j) * N + i] = d.syn[((size_t)code * d.Gs) * N + i];
            }
            if (lane == 0) d.deficits[(size_t)code * d.Gs + j] = 1 << 20;
        }
    if (lane == 0) {
        d.status[code] = status;
        d.n_gammas[code] = G;
    }
}

// ---- small codes (n + k <= 32 rows, n <= 32): column-major elimination
//
// Lane c holds column c of the isometry image (slot s: column 32 s + c) as a 32-bit mask over
// the rows. A pivot step of information_sets — the first row sel >= r with a 1 in column c
// becomes row r, then row r is XORed into every other row with a 1 there — is then one shuffle
// (the pivot column) and a few lane-local bit operations on each held column: swap bits r and
// sel, and XOR the pivot column (minus bit r) into every column with bit r set. Same rule,
// same Gamma_j as the row-major kernel above and the host.
//
// validate_normalizer's dual test uses rank(A) = N (checked by the first information set) and
// rank(A Omega A^T) = 2k: the symplectic dual V^perp of the N-dimensional rowspace V lies in V
// iff dim(V cap V^perp) = N - rank(A Omega A^T) equals dim V^perp = 2n - N.
__device__ __forceinline__ unsigned swap_bits(unsigned x, int r, int sel) {
    const unsigned t = ((x >> r) ^ (x >> sel)) & 1u;
    return x ^ ((t << r) | (t << sel));
}

__global__ void __launch_bounds__(128) batch_prep_small_kernel(BatchPrepDev d) {
    const int lane = threadIdx.x & 31;
    const int code = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (code >= d.codes) return;
    const int N = d.N, n = d.n;
    const unsigned nmask = n == 32 ? ~0u : ((1u << n) - 1u);

    // row `lane` of the normalizer: a (columns [0, n)) and b (columns [n, 2n))
    unsigned a = 0, b = 0;
    if (lane < N) {
        const unsigned long long w0 = d.normalizers[((size_t)code * N + lane) * d.in_words];
        const unsigned long long w1 = d.in_words > 1 ? d.normalizers[((size_t)code * N + lane) * d.in_words + 1] : 0ull;
        a = unsigned(w0) & nmask;
        b = unsigned(n == 32 ? w1 : (w0 >> n)) & nmask;
    }
    int status = 0;

    if (d.validate) {
        // Gram row: bit j = <row lane, row j>_s
        unsigned gram = 0;
        for (int j = 0; j < N; j++) {
            const unsigned aj = __shfl_sync(kFull, a, j), bj = __shfl_sync(kFull, b, j);
            gram |= ((__popc(a & bj) ^ __popc(b & aj)) & 1u) << j;
        }
        if (lane >= N) gram = 0;
        int rank = 0;
        bool done = false;
        for (int c = 0; c < N; c++) {
            const unsigned cand = __ballot_sync(kFull, !done && ((gram >> c) & 1u));
            if (!cand) continue;
            const int p = __ffs(cand) - 1;
            const unsigned prow = __shfl_sync(kFull, gram, p);
            if (lane == p) done = true;
            else if ((gram >> c) & 1u) gram ^= prow;
            rank++;
        }
        if (rank != 2 * (N - n)) status = 2;
    }

    // image columns (a | b | a^b): column c in lane c & 31, slot c >> 5
    unsigned col[3] = {0u, 0u, 0u};
    const unsigned ab = a ^ b;
    for (int c = 0; c < 3 * n; c++) {
        const int part = c < n ? 0 : (c < 2 * n ? 1 : 2), bit = c - part * n;
        const unsigned src = part == 0 ? a : (part == 1 ? b : ab);
        const unsigned v = __ballot_sync(kFull, lane < N && ((src >> bit) & 1u));
        if (lane == (c & 31)) {
#pragma unroll
            for (int s = 0; s < 3; s++)
                if (s == (c >> 5)) col[s] = v;
        }
    }

    // information_sets (prep.cpp:317-364): greedy elimination on unused columns, carried over
    unsigned used[3] = {0u, 0u, 0u};  // warp-uniform: bit c & 31 of word c >> 5
    unsigned gx[kPrepGammaSlots], gz[kPrepGammaSlots];
#pragma unroll
    for (int j = 0; j < kPrepGammaSlots; j++) gx[j] = gz[j] = 0u;
    int G = 0;
    const int rowlen = 2;  // W = 1
    for (; status == 0;) {
        int r = 0;
        unsigned piv[3] = {0u, 0u, 0u};  // pivot columns of this round
        for (int c = 0; c < 3 * n && r < N; c++) {
            const int sc = c >> 5, lc = c & 31;
            unsigned us = used[0], cs = col[0];
#pragma unroll
            for (int s = 1; s < 3; s++)
                if (s == sc) {
                    us = used[s];
                    cs = col[s];
                }
            if ((us >> lc) & 1u) continue;
            const unsigned pcol = __shfl_sync(kFull, cs, lc);
            const unsigned cand = pcol & (~0u << r);
            if (!cand) continue;
            const int sel = __ffs(cand) - 1;
            const unsigned pc = swap_bits(pcol, r, sel), m = pc & ~(1u << r);
#pragma unroll
            for (int s = 0; s < 3; s++) {
                unsigned x = swap_bits(col[s], r, sel);
                if ((x >> r) & 1u) x ^= m;
                col[s] = x;
            }
#pragma unroll
            for (int s = 0; s < 3; s++)
                if (s == sc) piv[s] |= 1u << lc;
            r++;
        }
        if (r == 0) break;
        if (G == 0 && r != N) {  // information_sets: rows are linearly dependent
            status = 2;
            break;
        }
        if (G < d.Gs) {
            // rows of Gamma_G: row i = bit i of every column; x = columns [0, n), z = [n, 2n)
            unsigned long long lo = 0ull;  // this lane's row, columns [0, 64)
            for (int i = 0; i < N; i++) {
                const unsigned w0 = __ballot_sync(kFull, (col[0] >> i) & 1u);
                const unsigned w1 = __ballot_sync(kFull, (col[1] >> i) & 1u);
                if (lane == i) lo = (unsigned long long)w0 | ((unsigned long long)w1 << 32);
            }
            const unsigned x = unsigned(lo) & nmask, z = unsigned(lo >> n) & nmask;
#pragma unroll
            for (int j = 0; j < kPrepGammaSlots; j++)
                if (j == G) {
                    gx[j] = x;
                    gz[j] = z;
                }
            if (lane < N) {
                uint32_t *dst = d.rows + (((size_t)code * d.Gs + G) * N + lane) * rowlen;
                dst[0] = x;
                dst[1] = z;
            }
            if (lane == 0) d.deficits[(size_t)code * d.Gs + G] = N - r;
        }
#pragma unroll
        for (int s = 0; s < 3; s++) used[s] |= piv[s];
        G++;
    }

    // admissibility syndromes: bit f of row i = <first 2n columns of row i, A_f>_s
    if (status == 0 && d.filter) {
        unsigned long long syn[kPrepGammaSlots];
#pragma unroll
        for (int j = 0; j < kPrepGammaSlots; j++) syn[j] = 0ull;
        for (int f = 0; f < N; f++) {
            const unsigned fa = __shfl_sync(kFull, a, f), fb = __shfl_sync(kFull, b, f);
#pragma unroll
            for (int j = 0; j < kPrepGammaSlots; j++)
                syn[j] |= (unsigned long long)((__popc(gx[j] & fb) ^ __popc(gz[j] & fa)) & 1) << f;
        }
        const int gs = min(G, d.Gs);
#pragma unroll
        for (int j = 0; j < kPrepGammaSlots; j++)
            if (j < gs && lane < N) d.syn[((size_t)code * d.Gs + j) * N + lane] = syn[j];
    }
    if (lane == 0) {
        d.status[code] = status;
        d.n_gammas[code] = G;
    }
}

}  // namespace

int launch_batch_prep(const BatchPrepDev &d, void *stream) {
    if (d.codes <= 0) return 0;
    const int warps = 4;
    const unsigned grid = unsigned((d.codes + warps - 1) / warps);
    // column-major elimination when rows and columns fit a lane's word; else one row per lane
    // (two when the normalizer has more than 32 rows)
    if (d.N <= 32 && d.n <= 32 && d.W == 1 && !d.force_rows)
        batch_prep_small_kernel<<<grid, 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(d);
    else if (d.N <= 32)
        batch_prep_kernel<1><<<grid, 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(d);
    else
        batch_prep_kernel<2><<<grid, 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(d);
    return 1;
}

}  // namespace sdb
