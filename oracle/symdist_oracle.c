/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the symdist-b200 hot path.
 *
 * Plain-C restatement of the reference's Saved_isometry route
 * (/root/reference/proj, C++20). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * (paper_2408_10743_b200/) never links or calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle_pins.py):
 *   - against the reference library itself, compiled from its own sources into
 *     oracle/_ref/ by oracle/Makefile (ref_shim.cpp), on random instances;
 *   - against the JSON fixtures in tests/golden/, frozen from that reference build by
 *     tests/golden/make_golden.py.
 *
 * Restated functions (reference file:line they follow):
 *   orc_generate          BASELINE.md §2 / SURVEY.md §8(d) config generator
 *                         (xorshift64* transvections; not a reference function)
 *   orc_isometry          isometry_transform      proj/src/prep.cpp:299-315
 *   orc_information_sets  information_sets        proj/src/prep.cpp:317-364
 *   orc_lower_bound       lower_bound (hamming)   proj/src/engine.cpp:31-39
 *   orc_run_levels        run_bz + enumerate_generation + Worker::{run,descend,leaves}
 *                         + offer/admissible      proj/src/engine.cpp:14-29,125-241,303-343
 *                         with saved_isometry's   proj/src/distance.cpp:135-149
 *   orc_brute_force       brute_force_distance    proj/src/distance.cpp:151-224
 *   orc_rank / orc_validate  rank, validate_normalizer proj/src/bitvec.cpp:213-288,
 *                         proj/src/distance.cpp:71-93
 *
 * Matrices cross the boundary as row-major 0/1 bytes.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_GAMMAS 64

/* ---------- config generator ---------- */

static uint64_t xs64star(uint64_t *s) {
    uint64_t x = *s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    *s = x;
    return x * 0x2545F4914F6CDD1DULL;
}

/* Rows Z_1..Z_{n-k}, X_{n-k+1}..X_n, Z_{n-k+1}..Z_n in (x|z) column order, then
 * `transvections` maps u -> u + <u,v>_s v with v uniform nonzero in GF(2)^{2n}. */
int orc_generate(int n, int k, uint64_t seed, int transvections, uint8_t *out) {
    if (n <= 0 || k < 0 || k > n || seed == 0) return 5;
    const int rows = n + k, cols = 2 * n, words = (cols + 63) / 64;
    memset(out, 0, (size_t)rows * cols);
    int r = 0;
    for (int i = 0; i < n - k; i++, r++) out[(size_t)r * cols + n + i] = 1;
    for (int i = n - k; i < n; i++, r++) out[(size_t)r * cols + i] = 1;
    for (int i = n - k; i < n; i++, r++) out[(size_t)r * cols + n + i] = 1;
    uint8_t *v = (uint8_t *)malloc((size_t)cols);
    uint64_t s = seed;
    for (int t = 0; t < transvections; t++) {
        int nz;
        do {
            nz = 0;
            for (int w = 0; w < words; w++) {
                uint64_t o = xs64star(&s);
                for (int b = 0; b < 64; b++) {
                    int c = 64 * w + b;
                    if (c < cols) {
                        v[c] = (uint8_t)((o >> b) & 1u);
                        nz |= v[c];
                    }
                }
            }
        } while (!nz);
        for (int i = 0; i < rows; i++) {
            uint8_t *u = out + (size_t)i * cols;
            int ip = 0;
            for (int c = 0; c < n; c++) ip ^= (u[c] & v[n + c]) ^ (u[n + c] & v[c]);
            if (ip)
                for (int c = 0; c < cols; c++) u[c] ^= v[c];
        }
    }
    free(v);
    return 0;
}

/* ---------- GF(2) helpers on byte matrices ---------- */

static int echelon_bytes(uint8_t *m, int rows, int cols, int *pivots) {
    int r = 0;
    for (int c = 0; c < cols && r < rows; c++) {
        int sel = -1;
        for (int i = r; i < rows; i++)
            if (m[(size_t)i * cols + c]) { sel = i; break; }
        if (sel < 0) continue;
        if (sel != r)
            for (int x = 0; x < cols; x++) {
                uint8_t t = m[(size_t)r * cols + x];
                m[(size_t)r * cols + x] = m[(size_t)sel * cols + x];
                m[(size_t)sel * cols + x] = t;
            }
        for (int i = 0; i < rows; i++)
            if (i != r && m[(size_t)i * cols + c])
                for (int x = 0; x < cols; x++) m[(size_t)i * cols + x] ^= m[(size_t)r * cols + x];
        if (pivots) pivots[r] = c;
        r++;
    }
    return r;
}

int orc_rank(const uint8_t *bits, int rows, int cols) {
    uint8_t *m = (uint8_t *)malloc((size_t)rows * cols + 1);
    memcpy(m, bits, (size_t)rows * cols);
    int rk = echelon_bytes(m, rows, cols, NULL);
    free(m);
    return rk;
}

/* validate_normalizer: shape, full rank, symplectic dual inside the rowspace.
 * Returns 0 ok; 1 no rows; 2 k<0; 3 rows>cols; 4 dependent; 5 not a normalizer. */
int orc_validate(const uint8_t *bits, int rows, int cols) {
    const int n = cols / 2, k = rows - n;
    if (rows == 0) return 1;
    if (k < 0) return 2;
    if (rows > cols) return 3;
    if (orc_rank(bits, rows, cols) != rows) return 4;
    /* dual = kernel of the half-swapped matrix */
    uint8_t *sw = (uint8_t *)malloc((size_t)rows * cols);
    for (int i = 0; i < rows; i++)
        for (int c = 0; c < n; c++) {
            sw[(size_t)i * cols + c] = bits[(size_t)i * cols + n + c];
            sw[(size_t)i * cols + n + c] = bits[(size_t)i * cols + c];
        }
    int *piv = (int *)malloc(sizeof(int) * (size_t)rows);
    int rk = echelon_bytes(sw, rows, cols, piv);
    uint8_t *ispiv = (uint8_t *)calloc((size_t)cols, 1);
    for (int r = 0; r < rk; r++) ispiv[piv[r]] = 1;
    uint8_t *ech = (uint8_t *)malloc((size_t)rows * cols);
    memcpy(ech, bits, (size_t)rows * cols);
    int *piv2 = (int *)malloc(sizeof(int) * (size_t)rows);
    int rk2 = echelon_bytes(ech, rows, cols, piv2);
    uint8_t *v = (uint8_t *)malloc((size_t)cols);
    int bad = 0;
    for (int f = 0; f < cols && !bad; f++) {
        if (ispiv[f]) continue;
        memset(v, 0, (size_t)cols);
        v[f] = 1;
        for (int r = 0; r < rk; r++)
            if (sw[(size_t)r * cols + f]) v[piv[r]] = 1;
        for (int r = 0; r < rk2; r++)
            if (v[piv2[r]])
                for (int x = 0; x < cols; x++) v[x] ^= ech[(size_t)r * cols + x];
        for (int x = 0; x < cols; x++)
            if (v[x]) { bad = 1; break; }
    }
    free(sw); free(piv); free(ispiv); free(ech); free(piv2); free(v);
    return bad ? 5 : 0;
}

/* ---------- prep (proj/src/prep.cpp:299-364) ---------- */

int orc_isometry(const uint8_t *bits, int rows, int cols, uint8_t *out) {
    if (cols % 2) return 5;
    const int n = cols / 2;
    for (int r = 0; r < rows; r++)
        for (int i = 0; i < n; i++) {
            uint8_t a = bits[(size_t)r * cols + i], b = bits[(size_t)r * cols + n + i];
            out[(size_t)r * 3 * n + i] = a;
            out[(size_t)r * 3 * n + n + i] = b;
            out[(size_t)r * 3 * n + 2 * n + i] = a ^ b;
        }
    return 0;
}

/* Greedy systematic forms on disjoint unused columns; `cur` carries over between
 * matrices. out: up to max_gammas blocks of rows x cols bytes. */
int orc_information_sets(const uint8_t *b, int rows, int cols, int max_gammas, uint8_t *out,
                         int *deficits, int *pivots, int *n_gammas) {
    if (orc_rank(b, rows, cols) != rows) return 2;
    uint8_t *cur = (uint8_t *)malloc((size_t)rows * cols);
    uint8_t *used = (uint8_t *)calloc((size_t)cols, 1);
    int *pc = (int *)malloc(sizeof(int) * (size_t)(rows + 1));
    memcpy(cur, b, (size_t)rows * cols);
    *n_gammas = 0;
    for (;;) {
        int r = 0;
        for (int c = 0; c < cols && r < rows; c++) {
            if (used[c]) continue;
            int sel = -1;
            for (int i = r; i < rows; i++)
                if (cur[(size_t)i * cols + c]) { sel = i; break; }
            if (sel < 0) continue;
            if (sel != r)
                for (int x = 0; x < cols; x++) {
                    uint8_t t = cur[(size_t)r * cols + x];
                    cur[(size_t)r * cols + x] = cur[(size_t)sel * cols + x];
                    cur[(size_t)sel * cols + x] = t;
                }
            for (int i = 0; i < rows; i++)
                if (i != r && cur[(size_t)i * cols + c])
                    for (int x = 0; x < cols; x++) cur[(size_t)i * cols + x] ^= cur[(size_t)r * cols + x];
            pc[r++] = c;
        }
        if (r == 0) break;
        if (*n_gammas < max_gammas) {
            memcpy(out + (size_t)(*n_gammas) * rows * cols, cur, (size_t)rows * cols);
            deficits[*n_gammas] = rows - r;
            for (int i = 0; i < rows; i++) pivots[*n_gammas * rows + i] = i < r ? pc[i] : -1;
        }
        (*n_gammas)++;
        for (int i = 0; i < r; i++) used[pc[i]] = 1;
    }
    free(cur); free(used); free(pc);
    return 0;
}

/* lower_bound, hamming mode (proj/src/engine.cpp:33-39) */
long orc_lower_bound(int g, const int *deficits, int n_gammas) {
    long s = 0;
    for (int j = 0; j < n_gammas; j++) {
        long t = (long)g + 1 - deficits[j];
        s += t > 0 ? t : 0;
    }
    return s;
}

/* ---------- enumeration (proj/src/engine.cpp:125-271) ---------- */

typedef struct {
    int rows, stride;        /* stride: u64 words per packed row */
    const uint64_t *row;     /* rows x stride */
    const uint64_t *syn;     /* rows x syn_words: admissibility syndromes */
    int syn_words;
    int filter_on;
} orc_gamma;

typedef struct {
    const orc_gamma *gm;
    int g;
    int next_i1;             /* dispenser (protected by mu) */
    pthread_mutex_t mu;
    long upper;              /* level-local running min of admissible weights < upper_in */
    uint64_t best_rank;      /* lexicographic rank of the first minimal candidate */
    long best_w;
    const uint64_t *binom;   /* (rows+1) x (g+1) */
    int bstride;
} orc_level;

static uint64_t binom_at(const orc_level *L, int a, int b) {
    if (b < 0 || a < 0 || b > a) return 0;
    return L->binom[(size_t)a * L->bstride + b];
}

typedef struct {
    orc_level *L;
    uint64_t *stack;     /* (g+1) x stride */
    uint64_t *sstack;    /* (g+1) x syn_words */
    int *idx;
    long local_upper;
} orc_worker;

static void offer(orc_worker *W, long w, uint64_t rank) {
    orc_level *L = W->L;
    pthread_mutex_lock(&L->mu);
    if (w < L->best_w || (w == L->best_w && rank < L->best_rank)) {
        L->best_w = w;
        L->best_rank = rank;
    }
    W->local_upper = L->best_w;
    pthread_mutex_unlock(&L->mu);
}

/* depth-first lexicographic walk; prefix at stack[depth]; `rank` is the lexicographic
 * rank of the first leaf under this node. */
static void descend(orc_worker *W, int depth, int first, uint64_t rank) {
    orc_level *L = W->L;
    const orc_gamma *G = L->gm;
    const int np = G->rows, g = L->g, st = G->stride, sw = G->syn_words;
    const uint64_t *pre = W->stack + (size_t)depth * st;
    const uint64_t *spre = W->sstack + (size_t)depth * sw;
    const int remaining = g - depth;
    for (int p = first; p <= np - remaining; p++) {
        const uint64_t *row = G->row + (size_t)p * st;
        if (remaining == 1) {
            long w = 0;
            for (int i = 0; i < st; i++) w += __builtin_popcountll(pre[i] ^ row[i]);
            /* ties kept so the minimal lexicographic rank is found */
            if (w <= W->local_upper) {
                int adm = 1;
                if (G->filter_on) {
                    adm = 0;
                    for (int i = 0; i < sw; i++)
                        if (spre[i] ^ G->syn[(size_t)p * sw + i]) adm = 1;
                }
                if (adm) offer(W, w, rank);
            }
            rank++;
        } else {
            uint64_t *nx = W->stack + (size_t)(depth + 1) * st;
            uint64_t *snx = W->sstack + (size_t)(depth + 1) * sw;
            for (int i = 0; i < st; i++) nx[i] = pre[i] ^ row[i];
            for (int i = 0; i < sw; i++) snx[i] = spre[i] ^ G->syn[(size_t)p * sw + i];
            descend(W, depth + 1, p + 1, rank);
            rank += binom_at(L, np - 1 - p, remaining - 1);
        }
    }
}

static void *worker_main(void *arg) {
    orc_worker *W = (orc_worker *)arg;
    orc_level *L = W->L;
    const orc_gamma *G = L->gm;
    const int np = G->rows, g = L->g;
    for (;;) {
        pthread_mutex_lock(&L->mu);
        int i1 = L->next_i1++;
        W->local_upper = L->best_w;
        pthread_mutex_unlock(&L->mu);
        if (i1 > np - g) break;
        uint64_t rank = 0;
        for (int p = 0; p < i1; p++) rank += binom_at(L, np - 1 - p, g - 1);
        /* depth 0 prefix is zero; place row i1 as the depth-1 prefix (or leaf when g=1) */
        if (g == 1) {
            memset(W->stack, 0, sizeof(uint64_t) * (size_t)G->stride);
            memset(W->sstack, 0, sizeof(uint64_t) * (size_t)(G->syn_words ? G->syn_words : 1));
            /* emulate descend(0, i1, ...) restricted to p == i1 */
            const uint64_t *row = G->row + (size_t)i1 * G->stride;
            long w = 0;
            for (int i = 0; i < G->stride; i++) w += __builtin_popcountll(row[i]);
            if (w <= W->local_upper) {
                int adm = 1;
                if (G->filter_on) {
                    adm = 0;
                    for (int i = 0; i < G->syn_words; i++)
                        if (G->syn[(size_t)i1 * G->syn_words + i]) adm = 1;
                }
                if (adm) offer(W, w, rank);
            }
        } else {
            uint64_t *nx = W->stack + (size_t)G->stride;
            uint64_t *snx = W->sstack + (size_t)G->syn_words;
            memcpy(nx, G->row + (size_t)i1 * G->stride, sizeof(uint64_t) * (size_t)G->stride);
            if (G->syn_words) memcpy(snx, G->syn + (size_t)i1 * G->syn_words, sizeof(uint64_t) * (size_t)G->syn_words);
            descend(W, 1, i1 + 1, rank);
        }
    }
    return NULL;
}

/* One generation on one matrix. Returns the level minimum (or `upper_in` when nothing
 * admissible is <= upper_in - 1) and its lexicographic rank. */
static void enumerate_level(const orc_gamma *G, int g, long upper_in, int threads, const uint64_t *binom,
                            int bstride, long *w_out, uint64_t *rank_out) {
    orc_level L;
    memset(&L, 0, sizeof L);
    L.gm = G;
    L.g = g;
    L.best_w = upper_in - 1; /* improving candidates only: w < upper_in */
    L.best_rank = UINT64_MAX;
    L.binom = binom;
    L.bstride = bstride;
    pthread_mutex_init(&L.mu, NULL);
    if (threads < 1) threads = 1;
    orc_worker *ws = (orc_worker *)calloc((size_t)threads, sizeof(orc_worker));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; t++) {
        ws[t].L = &L;
        ws[t].stack = (uint64_t *)calloc((size_t)(g + 1) * G->stride, sizeof(uint64_t));
        ws[t].sstack = (uint64_t *)calloc((size_t)(g + 1) * (G->syn_words ? G->syn_words : 1), sizeof(uint64_t));
    }
    if (threads == 1) {
        worker_main(&ws[0]);
    } else {
        for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, worker_main, &ws[t]);
        for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    }
    for (int t = 0; t < threads; t++) { free(ws[t].stack); free(ws[t].sstack); }
    free(ws); free(th);
    pthread_mutex_destroy(&L.mu);
    if (L.best_rank == UINT64_MAX) {
        *w_out = upper_in;
        *rank_out = UINT64_MAX;
    } else {
        *w_out = L.best_w;
        *rank_out = L.best_rank;
    }
}

static uint64_t pack_row(const uint8_t *r, int cols, uint64_t *dst) {
    const int words = (cols + 63) / 64;
    memset(dst, 0, sizeof(uint64_t) * (size_t)words);
    for (int c = 0; c < cols; c++)
        if (r[c]) dst[c / 64] |= 1ULL << (c % 64);
    return 0;
}

/*
 * saved_isometry through run_bz's generation loop (proj/src/distance.cpp:135-149,
 * proj/src/engine.cpp:303-343), stopped after g_max levels when g_max > 0.
 * trace: n_levels x {g, L, U}; best_*: per-level (Gamma index, lexicographic rank)
 * of the first candidate reaching the level's new minimum, or -1 when U did not move.
 * Returns 0 ok, 2 validation error, 3 internal error (no admissible codeword), 5 bad args.
 */
int orc_run_levels(const uint8_t *bits, int rows, int cols, int validate, int dual_filter, int g_max,
                   int threads, int *trace_g, long *trace_l, long *trace_u, int *best_gamma,
                   uint64_t *best_rank, int trace_cap, int *n_levels, long *upper_out) {
    if (cols % 2 || rows <= 0) return 5;
    if (validate && orc_validate(bits, rows, cols) != 0) return 2;
    const int n = cols / 2, k = rows - n, icols = 3 * n;
    uint8_t *img = (uint8_t *)malloc((size_t)rows * icols);
    orc_isometry(bits, rows, cols, img);
    uint8_t *gam = (uint8_t *)malloc((size_t)ORC_MAX_GAMMAS * rows * icols);
    int defs[ORC_MAX_GAMMAS], ng = 0;
    int *piv = (int *)malloc(sizeof(int) * (size_t)ORC_MAX_GAMMAS * rows);
    int rc = orc_information_sets(img, rows, icols, ORC_MAX_GAMMAS, gam, defs, piv, &ng);
    if (rc) { free(img); free(gam); free(piv); return rc; }
    if (ng > ORC_MAX_GAMMAS) ng = ORC_MAX_GAMMAS;
    const int stride = (icols + 63) / 64;
    /* filter: enabled iff dual_filter and k >= 1 (proj/src/engine.cpp:16-21);
     * syndrome bit r of a Gamma row = <first 2n columns, A_r>_s */
    const int filter_on = dual_filter && k >= 1;
    const int sw = filter_on ? (rows + 63) / 64 : 0;
    orc_gamma G[ORC_MAX_GAMMAS];
    uint64_t *rowbuf = (uint64_t *)calloc((size_t)ng * rows * stride, sizeof(uint64_t));
    uint64_t *synbuf = (uint64_t *)calloc((size_t)ng * rows * (sw ? sw : 1), sizeof(uint64_t));
    for (int j = 0; j < ng; j++) {
        for (int r = 0; r < rows; r++) {
            const uint8_t *gr = gam + ((size_t)j * rows + r) * icols;
            pack_row(gr, icols, rowbuf + ((size_t)j * rows + r) * stride);
            for (int a = 0; filter_on && a < rows; a++) {
                const uint8_t *ar = bits + (size_t)a * cols;
                int ip = 0;
                for (int c = 0; c < n; c++) ip ^= (gr[c] & ar[n + c]) ^ (gr[n + c] & ar[c]);
                if (ip) synbuf[((size_t)j * rows + r) * sw + a / 64] |= 1ULL << (a % 64);
            }
        }
        G[j].rows = rows;
        G[j].stride = stride;
        G[j].row = rowbuf + (size_t)j * rows * stride;
        G[j].syn = synbuf + (size_t)j * rows * (sw ? sw : 1);
        G[j].syn_words = sw;
        G[j].filter_on = filter_on;
    }
    int g_limit = rows; /* every information-set matrix has one singleton package per row */
    if (g_max > 0 && g_max < g_limit) g_limit = g_max;
    const int bstride = g_limit + 2;
    uint64_t *binom = (uint64_t *)calloc((size_t)(rows + 1) * bstride, sizeof(uint64_t));
    for (int a = 0; a <= rows; a++)
        for (int b = 0; b < bstride && b <= a; b++)
            binom[(size_t)a * bstride + b] = (b == 0 || b == a) ? 1 : binom[(size_t)(a - 1) * bstride + b - 1] + binom[(size_t)(a - 1) * bstride + b];
    long U = (long)icols + 1, Lb = 1;
    *n_levels = 0;
    for (int g = 1; g <= g_limit; g++) {
        int bg = -1;
        uint64_t br = 0;
        for (int j = 0; j < ng; j++) {
            long w;
            uint64_t rk;
            enumerate_level(&G[j], g, U, threads, binom, bstride, &w, &rk);
            if (w < U) { U = w; bg = j; br = rk; }
        }
        Lb = orc_lower_bound(g, defs, ng);
        if (*n_levels < trace_cap) {
            trace_g[*n_levels] = g;
            trace_l[*n_levels] = Lb;
            trace_u[*n_levels] = U;
            best_gamma[*n_levels] = bg;
            best_rank[*n_levels] = br;
        }
        (*n_levels)++;
        if (Lb >= U) break;
    }
    *upper_out = U;
    free(img); free(gam); free(piv); free(rowbuf); free(synbuf); free(binom);
    if (g_max <= 0 && U >= (long)icols + 1) return 3;
    return 0;
}

/* brute_force_distance (proj/src/distance.cpp:151-224): Gray walk over all 2^rows - 1
 * combinations; symplectic weight; filtered by the accumulated syndrome. */
int orc_brute_force(const uint8_t *bits, int rows, int cols, int dual_filter, int *distance) {
    if (rows > 28 || rows == 0 || cols % 2) return 5;
    const int n = cols / 2, k = rows - n, wpb = (n + 63) / 64;
    const int filter_on = dual_filter && k >= 1;
    uint64_t *ra = (uint64_t *)calloc((size_t)rows * wpb, 8), *rb = (uint64_t *)calloc((size_t)rows * wpb, 8);
    uint64_t *syn = (uint64_t *)calloc((size_t)rows, 8);
    for (int r = 0; r < rows; r++)
        for (int c = 0; c < n; c++) {
            if (bits[(size_t)r * cols + c]) ra[r * wpb + c / 64] |= 1ULL << (c % 64);
            if (bits[(size_t)r * cols + n + c]) rb[r * wpb + c / 64] |= 1ULL << (c % 64);
        }
    for (int i = 0; filter_on && i < rows; i++)
        for (int j = 0; j < rows; j++) {
            int ip = 0;
            for (int c = 0; c < n; c++)
                ip ^= (bits[(size_t)i * cols + c] & bits[(size_t)j * cols + n + c]) ^
                      (bits[(size_t)i * cols + n + c] & bits[(size_t)j * cols + c]);
            if (ip) syn[i] |= 1ULL << j;
        }
    uint64_t acca[8] = {0}, accb[8] = {0}, accs = 0;
    long best = -1;
    const uint64_t total = (1ULL << rows) - 1;
    for (uint64_t m = 1; m <= total; m++) {
        const int f = __builtin_ctzll(m);
        for (int w = 0; w < wpb; w++) { acca[w] ^= ra[f * wpb + w]; accb[w] ^= rb[f * wpb + w]; }
        accs ^= syn[f];
        if (filter_on && accs == 0) continue;
        long wt = 0;
        for (int w = 0; w < wpb; w++) wt += __builtin_popcountll(acca[w] | accb[w]);
        if (best < 0 || wt < best) best = wt;
    }
    free(ra); free(rb); free(syn);
    if (best < 0) return 3;
    *distance = (int)best;
    return 0;
}
