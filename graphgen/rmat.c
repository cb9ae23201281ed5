/*
 * graphgen/rmat.c -- seeded synthetic input generator (test + bench infrastructure).
 *
 * This module produces INPUTS only: a forward CSR graph and per-edge Q1.31 weights.
 * It holds none of the method's arithmetic (no coins, no traversal, no reverse CSR,
 * no selection) and is shared by the CPU oracle and the CUDA path alike
 * (DESIGN.md "Input recipe").
 *
 * Graph: Graph500-style R-MAT / Kronecker generator, initiator (A,B,C,D) =
 * (0.57, 0.19, 0.19, 0.05) [SURVEY §8(d)], scale S = ceil(log2 n).
 *   - draw i (i = 0,1,2,...) picks S quadrants from a counter-based hash keyed by
 *     (graph_seed, i), so the output is independent of thread count;
 *   - endpoints >= n are rejected, self-loops dropped, duplicate (u,v) collapsed;
 *   - the FIRST m unique edges in draw order are kept;
 *   - a seeded random permutation relabels the vertices (Graph500 practice);
 *   - forward CSR rows are emitted with destinations sorted ascending.
 * Weights: Q1.31 thresholds (p = thr / 2^31), drawn as integers from the same
 * counter-based hash keyed by (weight_seed, forward edge position).
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC (done by __graft_entry__.build()).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

/* ---- counter-based hash (SplitMix64 finalizer, applied twice) ------------------ */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t ghash(uint64_t seed, uint64_t stream, uint64_t idx) {
    uint64_t x = mix64(seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL);
    return mix64(x ^ (idx * 0x9E3779B97F4A7C15ULL + 0x2545F4914F6CDD1DULL));
}

enum { STREAM_EDGE = 1, STREAM_PERM = 2, STREAM_W_IC = 3, STREAM_W_LT = 4 };

/* R-MAT quadrant thresholds on a 16-bit uniform: A=0.57, A+B=0.76, A+B+C=0.95 */
#define T_A   37355u   /* floor(0.57*65536) */
#define T_AB  49807u   /* floor(0.76*65536) */
#define T_ABC 62259u   /* floor(0.95*65536) */

static int scale_of(uint64_t n) { int s = 0; while ((1ULL << s) < n) s++; return s < 1 ? 1 : s; }

/* one R-MAT draw; returns packed key (u<<S)|v or UINT64_MAX if rejected */
static inline uint64_t draw_edge(uint64_t seed, uint64_t i, int S, uint64_t n) {
    uint64_t u = 0, v = 0, h = 0;
    for (int l = 0; l < S; l++) {
        if ((l & 3) == 0) h = ghash(seed, STREAM_EDGE, i * 16 + (uint64_t)(l >> 2));
        uint32_t r = (uint32_t)(h & 0xffff); h >>= 16;
        uint32_t bu, bv;
        if (r < T_A) { bu = 0; bv = 0; }
        else if (r < T_AB) { bu = 0; bv = 1; }
        else if (r < T_ABC) { bu = 1; bv = 0; }
        else { bu = 1; bv = 1; }
        u = (u << 1) | bu; v = (v << 1) | bv;
    }
    if (u >= n || v >= n || u == v) return UINT64_MAX;
    return (u << S) | v;
}

/* stable LSD radix sort of (key, idx) by key, 11-bit digits, OpenMP-parallel per pass */
static void radix_sort_pairs(uint64_t* key, uint32_t* idx, uint64_t* tk, uint32_t* ti, uint64_t K, int key_bits) {
    const int D = 11, R = 1 << D;
    int passes = (key_bits + D - 1) / D;
    int T = omp_get_max_threads();
    uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)T * R);
    for (int p = 0; p < passes; p++) {
        int sh = p * D;
        memset(hist, 0, sizeof(uint64_t) * (size_t)T * R);
        #pragma omp parallel num_threads(T)
        {
            int t = omp_get_thread_num();
            uint64_t lo = K * (uint64_t)t / T, hi = K * (uint64_t)(t + 1) / T;
            uint64_t* h = hist + (size_t)t * R;
            for (uint64_t i = lo; i < hi; i++) h[(key[i] >> sh) & (R - 1)]++;
        }
        /* exclusive scan in (digit, thread) order -> stable */
        uint64_t run = 0;
        for (int d = 0; d < R; d++)
            for (int t = 0; t < T; t++) { uint64_t c = hist[(size_t)t * R + d]; hist[(size_t)t * R + d] = run; run += c; }
        #pragma omp parallel num_threads(T)
        {
            int t = omp_get_thread_num();
            uint64_t lo = K * (uint64_t)t / T, hi = K * (uint64_t)(t + 1) / T;
            uint64_t* h = hist + (size_t)t * R;
            for (uint64_t i = lo; i < hi; i++) {
                uint64_t pos = h[(key[i] >> sh) & (R - 1)]++;
                tk[pos] = key[i]; ti[pos] = idx[i];
            }
        }
        memcpy(key, tk, K * sizeof(uint64_t)); memcpy(idx, ti, K * sizeof(uint32_t));
    }
    free(hist);
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b; return (x > y) - (x < y);
}

/*
 * gg_rmat: n vertices, m unique directed edges. out_row_ptr[n+1] (u64), out_col[m] (u32).
 * Returns 0 on success, -1 bad args, -2 out of memory, -3 could not find m unique edges.
 */
int gg_rmat(uint64_t n, uint64_t m, uint64_t seed, uint64_t* out_row_ptr, uint32_t* out_col) {
    if (n < 2 || m == 0 || n > 0xFFFFFFFFull || m >= 0xFFFFFFFFull) return -1;
    int S = scale_of(n);
    if (2 * S > 62) return -1;
    uint64_t K = m + m / 4 + 1024;
    for (int attempt = 0; attempt < 8; attempt++) {
        if (K >= 0xFFFFFFFFull) return -3;
        uint64_t* orig = (uint64_t*)malloc(K * sizeof(uint64_t));
        uint64_t* key = (uint64_t*)malloc(K * sizeof(uint64_t));
        uint32_t* idx = (uint32_t*)malloc(K * sizeof(uint32_t));
        uint64_t* tk = (uint64_t*)malloc(K * sizeof(uint64_t));
        uint32_t* ti = (uint32_t*)malloc(K * sizeof(uint32_t));
        if (!orig || !key || !idx || !tk || !ti) { free(orig); free(key); free(idx); free(tk); free(ti); return -2; }
        #pragma omp parallel for schedule(static)
        for (uint64_t i = 0; i < K; i++) { orig[i] = key[i] = draw_edge(seed, i, S, n); idx[i] = (uint32_t)i; }
        radix_sort_pairs(key, idx, tk, ti, K, 2 * S + 1 > 64 ? 64 : 2 * S + 1);
        free(tk); free(ti);
        /* keep[i] = 1 iff draw i is the first occurrence of its key (stable sort => run head) */
        uint8_t* keep = (uint8_t*)calloc(K, 1);
        if (!keep) { free(orig); free(key); free(idx); return -2; }
        #pragma omp parallel for schedule(static)
        for (uint64_t j = 0; j < K; j++)
            if (key[j] != UINT64_MAX && (j == 0 || key[j] != key[j - 1])) keep[idx[j]] = 1;
        free(key); free(idx);
        /* first m unique draws in draw order: chunked parallel compaction */
        int T = omp_get_max_threads();
        uint64_t* cnt = (uint64_t*)calloc((size_t)T + 1, sizeof(uint64_t));
        #pragma omp parallel num_threads(T)
        {
            int t = omp_get_thread_num();
            uint64_t lo = K * (uint64_t)t / T, hi = K * (uint64_t)(t + 1) / T, c = 0;
            for (uint64_t i = lo; i < hi; i++) c += keep[i];
            cnt[t + 1] = c;
        }
        for (int t = 0; t < T; t++) cnt[t + 1] += cnt[t];
        uint64_t got = cnt[T];
        if (got < m) {
            free(cnt); free(keep); free(orig);
            K = (uint64_t)((double)K * ((double)m / (double)(got ? got : 1)) * 1.05) + 1024;
            continue;
        }
        uint64_t* sel = (uint64_t*)malloc(m * sizeof(uint64_t));
        if (!sel) { free(cnt); free(keep); free(orig); return -2; }
        #pragma omp parallel num_threads(T)
        {
            int t = omp_get_thread_num();
            uint64_t lo = K * (uint64_t)t / T, hi = K * (uint64_t)(t + 1) / T, o = cnt[t];
            for (uint64_t i = lo; i < hi && o < m; i++) if (keep[i]) sel[o++] = orig[i];
        }
        free(cnt); free(keep); free(orig);
        /* seeded label permutation (Fisher-Yates, sequential) */
        uint32_t* perm = (uint32_t*)malloc(n * sizeof(uint32_t));
        if (!perm) { free(sel); return -2; }
        for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
        for (uint64_t i = n - 1; i > 0; i--) {
            uint64_t j = (uint64_t)(((__uint128_t)ghash(seed, STREAM_PERM, i) * (i + 1)) >> 64);
            uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
        }
        uint64_t vmask = (1ULL << S) - 1;
        /* forward CSR: count, scan, scatter, sort rows */
        /* (parallel with atomics; the order inside a row is fixed by the row sort below) */
        memset(out_row_ptr, 0, (n + 1) * sizeof(uint64_t));
        #pragma omp parallel for schedule(static)
        for (uint64_t e = 0; e < m; e++) __atomic_fetch_add(&out_row_ptr[perm[sel[e] >> S] + 1], 1, __ATOMIC_RELAXED);
        for (uint64_t v = 0; v < n; v++) out_row_ptr[v + 1] += out_row_ptr[v];
        uint64_t* cur = (uint64_t*)malloc(n * sizeof(uint64_t));
        if (!cur) { free(perm); free(sel); return -2; }
        memcpy(cur, out_row_ptr, n * sizeof(uint64_t));
        #pragma omp parallel for schedule(static)
        for (uint64_t e = 0; e < m; e++) {
            uint32_t u = perm[sel[e] >> S], v = perm[sel[e] & vmask];
            out_col[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
        }
        #pragma omp parallel for schedule(dynamic, 1024)
        for (uint64_t u = 0; u < n; u++) {
            uint64_t a = out_row_ptr[u], b = out_row_ptr[u + 1];
            if (b - a > 1) qsort(out_col + a, b - a, sizeof(uint32_t), cmp_u32);
        }
        free(cur); free(perm); free(sel);
        return 0;
    }
    return -3;
}

/* IC weights: thr[e] uniform in [0, 2^31) (p uniform in [0,1)), keyed by forward position e */
void gg_weights_uniform(uint64_t m, uint64_t seed, uint32_t* thr) {
    #pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < m; e++) thr[e] = (uint32_t)(ghash(seed, STREAM_W_IC, e) >> 33);
}

/*
 * LT weights: per destination v, raw_j uniform in [0,2^31) for each in-edge j, then
 * thr_j = floor(raw_j * 2^31 / sum_raw(v)) so that sum_j thr_j <= 2^31 (SURVEY C-6).
 * Edges are indexed by forward position; col gives the destination.
 */
int gg_weights_lt(uint64_t n, uint64_t m, const uint32_t* col, uint64_t seed, uint32_t* thr) {
    uint64_t* sum = (uint64_t*)calloc(n, sizeof(uint64_t));
    if (!sum) return -2;
    for (uint64_t e = 0; e < m; e++) sum[col[e]] += ghash(seed, STREAM_W_LT, e) >> 33;
    #pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < m; e++) {
        uint64_t raw = ghash(seed, STREAM_W_LT, e) >> 33, s = sum[col[e]];
        thr[e] = s ? (uint32_t)(((__uint128_t)raw << 31) / s) : 0u;
    }
    free(sum);
    return 0;
}
