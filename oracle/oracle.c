/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the fused-BPT hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2311_10201_b200, libbpt.so) never links, imports or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n;
 * C-k = reading k of SURVEY.md §8(c), restated in DESIGN.md "Readings"):
 *   - RRR sets one BPT at a time, UNFUSED (Def. 2; "RRR sets can be
 *     equivalently computed as the visited array of a Probabilistic Breadth-First
 *     Traversal"). IC: queue BFS over the reverse graph, each edge live with
 *     probability p(e). LT: reverse live-edge walk (reading C-6).
 *   - Work counters: E_logical (unfused edge reads) and E_phys (edge reads of a
 *     level-synchronous fused group, "fusing occurs only if BPTs within the
 *     same group visit a vertex in the same traversal step"), Theorem 1.
 *   - Greedy max-k-cover over the RRR sets, naive and lazy, sigma_hat.
 *
 * Parity status of each function: see the "pins" list in DESIGN.md §Oracle.
 * Threads: samples are claimed from a shared atomic counter (the paper's host-side
 * work counter); each sample is computed independently, so results do not
 * depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>

/* ------------------------------------------------------------------------------------
 * Philox2x32-10 (reading C-1: Salmon et al. SC'11, Random123 constants).
 * One round: (hi, lo) = M * x0; x0' = hi ^ key ^ x1; x1' = lo. The key is bumped by
 * W before every round but the first. Pinned by the Random123 known-answer vectors.
 * ---------------------------------------------------------------------------------- */
#define PHILOX_M 0xD256D193u
#define PHILOX_W 0x9E3779B9u

void or_philox2x32_10(uint32_t x0, uint32_t x1, uint32_t key, uint32_t out[2]) {
    for (int round = 0; round < 10; round++) {
        if (round > 0) key += PHILOX_W;
        uint64_t prod = (uint64_t)PHILOX_M * (uint64_t)x0;
        uint32_t hi = (uint32_t)(prod >> 32), lo = (uint32_t)prod;
        uint32_t n0 = hi ^ key ^ x1;
        uint32_t n1 = lo;
        x0 = n0; x1 = n1;
    }
    out[0] = x0; out[1] = x1;
}

/* stream tags (reading C-1) */
#define TAG_IC    0x49430001u
#define TAG_LT    0x4C540001u
#define TAG_START 0x53540001u

/* k_tag = Philox2x32_10(ctr = {lo32(seed), hi32(seed)}, key = TAG)[0]   (reading C-1) */
uint32_t or_stream_key(uint64_t seed, uint32_t tag) {
    uint32_t out[2];
    or_philox2x32_10((uint32_t)seed, (uint32_t)(seed >> 32), tag, out);
    return out[0];
}

/* start(s): r64 = (w1 << 32) | w0 from Philox(ctr={lo32(s), hi32(s)}, key=k_START);
 * start = floor(r64 * n / 2^64)  -- "selected uniformly at random from V", C-3 */
uint32_t or_start_vertex(uint64_t s, uint32_t n, uint32_t k_start) {
    uint32_t w[2];
    or_philox2x32_10((uint32_t)s, (uint32_t)(s >> 32), k_start, w);
    uint64_t r64 = ((uint64_t)w[1] << 32) | (uint64_t)w[0];
    return (uint32_t)(((unsigned __int128)r64 * (unsigned __int128)n) >> 64);
}

/* IC coin for sample s on reverse-CSR edge e: live iff (r >> 1) < thr(e)   (C-1, C-2)
 * Listing 1 line 13 keeps a colour with probability e.prob. */
int or_ic_edge_live(uint64_t s, uint32_t e, uint32_t thr, uint32_t k_ic) {
    uint32_t r[2];
    or_philox2x32_10(e, (uint32_t)s, k_ic, r);
    return (r[0] >> 1) < thr;
}

/* LT draw at vertex v for sample s: r = coinLT(s, v) >> 1 in [0, 2^31)   (C-6) */
uint32_t or_lt_draw(uint64_t s, uint32_t v, uint32_t k_lt) {
    uint32_t r[2];
    or_philox2x32_10(v, (uint32_t)s, k_lt, r);
    return r[0] >> 1;
}

/* Q1.31 threshold from a probability in [0,1]: floor(p * 2^31)   (reading C-5) */
uint32_t or_q31_from_f32(float p) {
    return (uint32_t)floor((double)p * 2147483648.0);
}

/* SplitMix64 output function of v + golden gamma (digest mix) */
uint64_t or_digest_mix(uint64_t v) {
    uint64_t z = v + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------------------
 * Graph: the reverse CSR ("transpose") the BPTs traverse (Def. 2: u reaches v in G
 * iff v reaches u in the transpose; Listing 1's mate(e,v) is the other endpoint of
 * the transposed edge, reading C-8).
 * Canonical order (reading C-4): rows by destination v; within a row, entries in
 * forward-CSR position order (a stable counting sort of the forward edge list).
 * The edge id e used by the coins is the position in this reverse CSR.
 * ---------------------------------------------------------------------------------- */
typedef struct {
    uint32_t n;
    uint64_t m;
    int model;              /* 0 = IC, 1 = LT */
    uint64_t* roff;         /* [n+1] */
    uint32_t* src;          /* [m] source u of reverse entry e (original edge u -> v) */
    uint32_t* thr;          /* [m] Q1.31 threshold of entry e */
    uint64_t* cum;          /* [m] LT: inclusive prefix of thr within the row */
} or_graph;

void or_graph_free(or_graph* g) {
    if (!g) return;
    free(g->roff); free(g->src); free(g->thr); free(g->cum); free(g);
}

/*
 * Build from a forward CSR. Exactly one of w_f32 / w_q31 is non-NULL.
 * Returns NULL on invalid input (the oracle does not diagnose; tests pass valid input).
 */
or_graph* or_graph_new(uint32_t n, uint64_t m, const uint64_t* row_ptr, const uint32_t* col,
                       const float* w_f32, const uint32_t* w_q31, int model) {
    if (n == 0 || row_ptr[0] != 0 || row_ptr[n] != m) return NULL;
    or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
    g->n = n; g->m = m; g->model = model;
    g->roff = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    g->src = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
    g->thr = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
    g->cum = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
    /* in-degree histogram */
    for (uint64_t e = 0; e < m; e++) g->roff[col[e] + 1]++;
    for (uint32_t v = 0; v < n; v++) g->roff[v + 1] += g->roff[v];
    uint64_t* cursor = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
    memcpy(cursor, g->roff, ((size_t)n + 1) * sizeof(uint64_t));
    /* stable scatter in forward order: u ascending, then forward position */
    for (uint32_t u = 0; u < n; u++) {
        for (uint64_t ef = row_ptr[u]; ef < row_ptr[u + 1]; ef++) {
            uint32_t v = col[ef];
            uint64_t e = cursor[v]++;
            g->src[e] = u;
            g->thr[e] = w_q31 ? w_q31[ef] : or_q31_from_f32(w_f32[ef]);
        }
    }
    free(cursor);
    /* LT: cum[j] = sum of thr over the row up to and including j   (reading C-6) */
    for (uint32_t v = 0; v < n; v++) {
        uint64_t run = 0;
        for (uint64_t e = g->roff[v]; e < g->roff[v + 1]; e++) { run += g->thr[e]; g->cum[e] = run; }
    }
    return g;
}

void or_graph_export(const or_graph* g, uint64_t* roff, uint32_t* src, uint32_t* thr) {
    memcpy(roff, g->roff, ((size_t)g->n + 1) * sizeof(uint64_t));
    memcpy(src, g->src, g->m * sizeof(uint32_t));
    memcpy(thr, g->thr, g->m * sizeof(uint32_t));
}

/* ------------------------------------------------------------------------------------
 * One BPT (one sample s), unfused.
 * Per-thread scratch keeps a stamp per vertex so "visited" needs no clearing.
 * ---------------------------------------------------------------------------------- */
typedef struct {
    uint32_t* stamp;        /* stamp[v] == cur  <=>  v visited in the current sample */
    uint32_t* level;        /* BFS level of v in the current sample (valid if visited) */
    uint32_t* queue;        /* visit order; queue[0] = start */
    uint32_t cur;
} or_scratch;

static void scratch_init(or_scratch* w, uint32_t n) {
    w->stamp = (uint32_t*)calloc(n, sizeof(uint32_t));
    w->level = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    w->queue = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    w->cur = 0;
}
static void scratch_free(or_scratch* w) { free(w->stamp); free(w->level); free(w->queue); }

typedef struct {
    uint32_t k_ic, k_lt, k_start;
} or_keys;

static or_keys keys_of(uint64_t seed) {
    or_keys k;
    k.k_ic = or_stream_key(seed, TAG_IC);
    k.k_lt = or_stream_key(seed, TAG_LT);
    k.k_start = or_stream_key(seed, TAG_START);
    return k;
}

/*
 * Runs sample s; on return w->queue[0..size) holds RR_s in visit order with levels in
 * w->level[]. *elog = E_logical contribution (IC: sum of in-degrees of the dequeued
 * vertices, i.e. the unfused BPT's edge reads; LT: |RR_s|).
 */
static uint32_t run_sample(const or_graph* g, const or_keys* k, uint64_t s, or_scratch* w, uint64_t* elog) {
    if (++w->cur == 0) { memset(w->stamp, 0, (size_t)g->n * sizeof(uint32_t)); w->cur = 1; }
    const uint32_t cur = w->cur;
    uint32_t start = or_start_vertex(s, g->n, k->k_start);
    uint32_t head = 0, tail = 0;
    w->queue[tail++] = start; w->stamp[start] = cur; w->level[start] = 0;
    uint64_t reads = 0;
    if (g->model == 0) {
        /* IC: BPT over the reverse graph; edge e is live for s iff its coin passes */
        while (head < tail) {
            uint32_t v = w->queue[head++];
            for (uint64_t e = g->roff[v]; e < g->roff[v + 1]; e++) {
                reads++;
                uint32_t u = g->src[e];
                if (w->stamp[u] == cur) continue;
                if (or_ic_edge_live(s, (uint32_t)e, g->thr[e], k->k_ic)) {
                    w->stamp[u] = cur; w->level[u] = w->level[v] + 1; w->queue[tail++] = u;
                }
            }
        }
    } else {
        /* LT: at v keep in-edge j iff cum[j-1] <= r < cum[j] (none if r >= row sum);
         * walk continues only to an unvisited vertex (reading C-6) */
        uint32_t v = start;
        for (;;) {
            uint32_t r = or_lt_draw(s, v, k->k_lt);
            uint64_t chosen = UINT64_MAX, lo = 0;
            for (uint64_t e = g->roff[v]; e < g->roff[v + 1]; e++) {
                if (lo <= r && (uint64_t)r < g->cum[e]) { chosen = e; break; }
                lo = g->cum[e];
            }
            if (chosen == UINT64_MAX) break;
            uint32_t u = g->src[chosen];
            if (w->stamp[u] == cur) break;
            w->stamp[u] = cur; w->level[u] = w->level[v] + 1; w->queue[tail++] = u;
            v = u;
        }
        reads = tail;
    }
    *elog = reads;
    return tail;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b; return (x > y) - (x < y);
}
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b; return (x > y) - (x < y);
}

/* Single sample, members sorted ascending (C-10). levels[i] = level of members[i] (optional). */
uint32_t or_sample_one(const or_graph* g, uint64_t seed, uint64_t s, uint32_t* members, uint32_t* levels,
                       uint64_t* elog) {
    or_keys k = keys_of(seed);
    or_scratch w; scratch_init(&w, g->n);
    uint32_t size = run_sample(g, &k, s, &w, elog);
    memcpy(members, w.queue, (size_t)size * sizeof(uint32_t));
    qsort(members, size, sizeof(uint32_t), cmp_u32);
    if (levels) for (uint32_t i = 0; i < size; i++) levels[i] = w.level[members[i]];
    scratch_free(&w);
    return size;
}

/* ------------------------------------------------------------------------------------
 * Many samples, multi-threaded. For each ids[i]: sizes[i], digests[i], elog[i].
 * If offsets != NULL (two-pass use: first call with members == NULL to get sizes),
 * members[offsets[i] .. offsets[i+1]) receives the sorted list.
 * ---------------------------------------------------------------------------------- */
typedef struct {
    const or_graph* g; or_keys k; const uint64_t* ids; uint64_t count;
    uint32_t* sizes; uint64_t* digests; uint64_t* elog;
    const uint64_t* offsets; uint32_t* members;
    atomic_ulong next;
} many_job;

static void* many_worker(void* arg) {
    many_job* J = (many_job*)arg;
    or_scratch w; scratch_init(&w, J->g->n);
    for (;;) {
        uint64_t i = atomic_fetch_add(&J->next, 1);   /* claim one sample */
        if (i >= J->count) break;
        uint64_t el = 0;
        uint32_t size = run_sample(J->g, &J->k, J->ids[i], &w, &el);
        uint64_t d = 0;
        for (uint32_t j = 0; j < size; j++) d += or_digest_mix(w.queue[j]);
        if (J->sizes) J->sizes[i] = size;
        if (J->digests) J->digests[i] = d;
        if (J->elog) J->elog[i] = el;
        if (J->members) {
            uint32_t* out = J->members + J->offsets[i];
            memcpy(out, w.queue, (size_t)size * sizeof(uint32_t));
            qsort(out, size, sizeof(uint32_t), cmp_u32);
        }
    }
    scratch_free(&w);
    return NULL;
}

int or_sample_many(const or_graph* g, uint64_t seed, const uint64_t* ids, uint64_t count, int nthreads,
                   uint32_t* sizes, uint64_t* digests, uint64_t* elog,
                   const uint64_t* offsets, uint32_t* members) {
    many_job J;
    J.g = g; J.k = keys_of(seed); J.ids = ids; J.count = count;
    J.sizes = sizes; J.digests = digests; J.elog = elog; J.offsets = offsets; J.members = members;
    atomic_init(&J.next, 0);
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, many_worker, &J);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Fused-group work (Theorem 1). For the traversal group of
 * samples [s0, s1): a level-synchronous fused traversal processes vertex v at level L
 * once iff some colour of the group first reaches v at level L, reading all indeg(v)
 * entries of its row. So
 *     E_phys(group) = sum over distinct pairs (v, L) with L = d_s(v), s in group, of indeg(v)
 *     frontier[L]   = number of distinct v with some d_s(v) = L.
 * (SURVEY §8(c) "Proof that fused frontiers equal the oracle's level sets".)
 * For LT, E_phys := sum_s |RR_s| (number of vertex-colour expansions).
 * Outputs: *e_phys, *e_logical (sum of the unfused reads), *levels (number of non-empty
 * levels), frontier[0..levels) (if frontier != NULL and levels <= cap).
 * ---------------------------------------------------------------------------------- */
/* The same for a traversal group of arbitrary sample ids (slots sorted by
 * start vertex form groups of non-consecutive samples; the definition is unchanged). */
int or_group_work_ids(const or_graph* g, uint64_t seed, const uint64_t* ids, uint64_t count,
                      uint64_t* e_phys, uint64_t* e_logical, uint32_t* levels, uint64_t* frontier, uint32_t cap);

int or_group_work(const or_graph* g, uint64_t seed, uint64_t s0, uint64_t s1,
                  uint64_t* e_phys, uint64_t* e_logical, uint32_t* levels, uint64_t* frontier, uint32_t cap) {
    uint64_t* ids = (uint64_t*)malloc((s1 > s0 ? s1 - s0 : 1) * sizeof(uint64_t));
    for (uint64_t s = s0; s < s1; s++) ids[s - s0] = s;
    int r = or_group_work_ids(g, seed, ids, s1 > s0 ? s1 - s0 : 0, e_phys, e_logical, levels, frontier, cap);
    free(ids);
    return r;
}

int or_group_work_ids(const or_graph* g, uint64_t seed, const uint64_t* ids, uint64_t count,
                      uint64_t* e_phys, uint64_t* e_logical, uint32_t* levels, uint64_t* frontier, uint32_t cap) {
    or_keys k = keys_of(seed);
    or_scratch w; scratch_init(&w, g->n);
    uint64_t npairs = 0, cap_pairs = 1024;
    uint64_t* pairs = (uint64_t*)malloc(cap_pairs * sizeof(uint64_t));
    uint64_t elog_total = 0, lt_total = 0;
    for (uint64_t i = 0; i < count; i++) {
        uint64_t s = ids[i];
        uint64_t el = 0;
        uint32_t size = run_sample(g, &k, s, &w, &el);
        elog_total += el; lt_total += size;
        if (npairs + size > cap_pairs) {
            while (npairs + size > cap_pairs) cap_pairs *= 2;
            pairs = (uint64_t*)realloc(pairs, cap_pairs * sizeof(uint64_t));
        }
        for (uint32_t j = 0; j < size; j++) {
            uint32_t v = w.queue[j];
            pairs[npairs++] = ((uint64_t)w.level[v] << 32) | v;   /* sorted by (level, v) */
        }
    }
    qsort(pairs, npairs, sizeof(uint64_t), cmp_u64);
    uint64_t ep = 0; uint32_t nlev = 0;
    for (uint64_t i = 0; i < npairs; i++) {
        if (i > 0 && pairs[i] == pairs[i - 1]) continue;
        uint32_t v = (uint32_t)pairs[i], L = (uint32_t)(pairs[i] >> 32);
        ep += g->roff[v + 1] - g->roff[v];
        if (L + 1 > nlev) nlev = L + 1;
        if (frontier && L < cap) frontier[L]++;
    }
    *e_phys = g->model == 0 ? ep : lt_total;
    *e_logical = elog_total;
    *levels = nlev;
    free(pairs);
    scratch_free(&w);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Greedy max-k-cover over RRR sets ("greedy hill climbing ... 1-1/e";
 * P:95 "the problem of selecting the k seeds in S reduces to computing a
 * maximum-k-cover over the collection of RRR sets").
 * Sets given as CSR: set i = members[set_off[i] .. set_off[i+1]).
 * Tie-break (reading C-11): max gain, then smallest vertex id; once every set is
 * covered, the smallest unselected ids (gain 0).
 * lazy = 0: naive (recount every round). lazy = 1: CELF with exact re-evaluation.
 * gains[r] = number of sets newly covered in round r.
 * ---------------------------------------------------------------------------------- */
static void build_vertex_index(uint32_t n, uint64_t nsets, const uint64_t* set_off, const uint32_t* members,
                               uint64_t** voff_out, uint64_t** vsets_out) {
    uint64_t total = set_off[nsets];
    uint64_t* voff = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    uint64_t* vsets = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < total; i++) voff[members[i] + 1]++;
    for (uint32_t v = 0; v < n; v++) voff[v + 1] += voff[v];
    uint64_t* cur = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
    memcpy(cur, voff, ((size_t)n + 1) * sizeof(uint64_t));
    for (uint64_t si = 0; si < nsets; si++)
        for (uint64_t j = set_off[si]; j < set_off[si + 1]; j++) vsets[cur[members[j]]++] = si;
    free(cur);
    *voff_out = voff; *vsets_out = vsets;
}

static uint64_t true_gain(uint32_t v, const uint64_t* voff, const uint64_t* vsets, const uint8_t* covered) {
    uint64_t gsum = 0;
    for (uint64_t j = voff[v]; j < voff[v + 1]; j++) gsum += !covered[vsets[j]];
    return gsum;
}

int or_greedy(uint32_t n, uint64_t nsets, const uint64_t* set_off, const uint32_t* members,
              uint32_t k, int lazy, uint32_t* seeds, uint64_t* gains) {
    if (k == 0 || k > n) return -1;
    uint64_t *voff, *vsets;
    build_vertex_index(n, nsets, set_off, members, &voff, &vsets);
    uint8_t* covered = (uint8_t*)calloc(nsets ? nsets : 1, 1);
    uint8_t* selected = (uint8_t*)calloc(n, 1);
    if (!lazy) {
        for (uint32_t r = 0; r < k; r++) {
            uint64_t best_gain = 0; int64_t best = -1;
            for (uint32_t v = 0; v < n; v++) {
                if (selected[v]) continue;
                uint64_t gv = true_gain(v, voff, vsets, covered);
                if (best < 0 || gv > best_gain) { best = v; best_gain = gv; }  /* strict: smallest id wins ties */
            }
            uint32_t b = (uint32_t)best;
            selected[b] = 1; seeds[r] = b; gains[r] = best_gain;
            for (uint64_t j = voff[b]; j < voff[b + 1]; j++) covered[vsets[j]] = 1;
        }
    } else {
        /* CELF: max-heap of (stale gain, vertex) ordered by gain desc, id asc */
        uint64_t* hg = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
        uint32_t* hv = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
        uint32_t hn = 0;
#define BETTER(ga, va, gb, vb) ((ga) > (gb) || ((ga) == (gb) && (va) < (vb)))
        for (uint32_t v = 0; v < n; v++) {
            uint64_t gv = voff[v + 1] - voff[v];
            uint32_t i = hn++;
            hg[i] = gv; hv[i] = v;
            while (i > 0) {
                uint32_t p = (i - 1) / 2;
                if (!BETTER(hg[i], hv[i], hg[p], hv[p])) break;
                uint64_t tg = hg[i]; hg[i] = hg[p]; hg[p] = tg;
                uint32_t tv = hv[i]; hv[i] = hv[p]; hv[p] = tv;
                i = p;
            }
        }
        for (uint32_t r = 0; r < k; r++) {
            for (;;) {
                /* pop top */
                uint32_t v = hv[0];
                hn--; hg[0] = hg[hn]; hv[0] = hv[hn];
                uint32_t i = 0;
                for (;;) {
                    uint32_t l = 2 * i + 1, rr = l + 1, b = i;
                    if (l < hn && BETTER(hg[l], hv[l], hg[b], hv[b])) b = l;
                    if (rr < hn && BETTER(hg[rr], hv[rr], hg[b], hv[b])) b = rr;
                    if (b == i) break;
                    uint64_t tg = hg[i]; hg[i] = hg[b]; hg[b] = tg;
                    uint32_t tv = hv[i]; hv[i] = hv[b]; hv[b] = tv;
                    i = b;
                }
                uint64_t gv = true_gain(v, voff, vsets, covered);
                /* stale gains are upper bounds (submodularity), so v wins if it still
                 * beats the best remaining stale key */
                if (hn == 0 || BETTER(gv, v, hg[0], hv[0])) {
                    selected[v] = 1; seeds[r] = v; gains[r] = gv;
                    for (uint64_t j = voff[v]; j < voff[v + 1]; j++) covered[vsets[j]] = 1;
                    break;
                }
                /* re-insert with its fresh gain */
                uint32_t q = hn++;
                hg[q] = gv; hv[q] = v;
                while (q > 0) {
                    uint32_t p = (q - 1) / 2;
                    if (!BETTER(hg[q], hv[q], hg[p], hv[p])) break;
                    uint64_t tg = hg[q]; hg[q] = hg[p]; hg[p] = tg;
                    uint32_t tv = hv[q]; hv[q] = hv[p]; hv[p] = tv;
                    q = p;
                }
            }
        }
#undef BETTER
        free(hg); free(hv);
    }
    free(covered); free(selected); free(voff); free(vsets);
    return 0;
}

/* sigma_hat = n * covered / theta   (reading C-12; RIS estimate) */
double or_sigma_hat(uint32_t n, uint64_t covered, uint64_t theta) {
    return (double)n * (double)covered / (double)theta;
}

/* ------------------------------------------------------------------------------------
 * RRR store of a sample range (SURVEY §8(c) oracle step 3): every sample kept as a
 * sorted u32 member list if |RR_s| <= list_max (default n/32), else as an n-bit
 * bitset (bit v of word v/64 set iff v in RR_s). Built group by group (traversal
 * group = `colors` consecutive samples, reading C-9): for each group the distinct
 * (v, L) pairs reached by its samples (L = BFS level d_s(v) < 64) give
 *     E_phys(group)      = sum over distinct (v, L) of indeg(v)
 *     frontier(group)[L] = number of distinct v with some d_s(v) = L
 * -- the definitions or_group_work uses, counted with a per-vertex level mask instead
 * of a sort (levels >= 64 make the call fail; IC levels are ~10).
 * Greedy on the store: max-k-cover (reading C-11) with the occurrence count
 * of every vertex kept current: a newly covered sample leaves the count of each of
 * its members (the gain of v = number of uncovered samples containing v).
 * ---------------------------------------------------------------------------------- */
typedef struct {
    uint32_t n, colors;
    uint64_t s0, count, ngroups;
    const uint64_t* ids;   /* sample ids in traversal order (NULL: s0, s0 + 1, ...) */
    int keep;              /* keep the sets (lists / bitsets); 0: sizes, digests and group work only */
    uint32_t list_max;
    uint32_t* size;        /* [count] */
    uint64_t* digest;      /* [count] */
    uint32_t** list;       /* [count] sorted members, or NULL */
    uint64_t** bits;       /* [count] n-bit set, or NULL */
    uint64_t* e_phys;      /* [ngroups] */
    uint32_t* levels;      /* [ngroups] */
    uint64_t* frontier;    /* [ngroups][64] */
    uint64_t e_logical;
} or_store;

typedef struct {
    const or_graph* g; or_keys k; or_store* S; atomic_ulong next; atomic_int fail;
    pthread_mutex_t mu;
} store_job;

static void* store_worker(void* arg) {
    store_job* J = (store_job*)arg;
    or_store* S = J->S;
    const or_graph* g = J->g;
    or_scratch w; scratch_init(&w, g->n);
    uint64_t* lvmask = (uint64_t*)calloc(g->n, sizeof(uint64_t));
    uint32_t* touched = (uint32_t*)malloc((size_t)g->n * sizeof(uint32_t));
    uint64_t el_sum = 0;
    for (;;) {
        uint64_t grp = atomic_fetch_add(&J->next, 1);   /* claim one traversal group */
        if (grp >= S->ngroups) break;
        uint64_t a = grp * S->colors, b = a + S->colors;
        if (b > S->count) b = S->count;
        uint32_t ntouched = 0;
        for (uint64_t i = a; i < b; i++) {
            uint64_t el = 0;
            uint32_t size = run_sample(g, &J->k, S->ids ? S->ids[i] : S->s0 + i, &w, &el);
            el_sum += el;
            uint64_t d = 0;
            for (uint32_t j = 0; j < size; j++) {
                uint32_t v = w.queue[j], L = w.level[v];
                d += or_digest_mix(v);
                if (L >= 64) { atomic_store(&J->fail, 1); continue; }
                if (!lvmask[v]) touched[ntouched++] = v;
                lvmask[v] |= 1ULL << L;
            }
            S->size[i] = size; S->digest[i] = d;
            if (!S->keep) continue;
            if (size <= S->list_max) {
                uint32_t* l = (uint32_t*)malloc((size ? size : 1) * sizeof(uint32_t));
                memcpy(l, w.queue, (size_t)size * sizeof(uint32_t));
                qsort(l, size, sizeof(uint32_t), cmp_u32);
                S->list[i] = l;
            } else {
                uint64_t* bs = (uint64_t*)calloc(((size_t)S->n + 63) / 64, sizeof(uint64_t));
                for (uint32_t j = 0; j < size; j++) bs[w.queue[j] >> 6] |= 1ULL << (w.queue[j] & 63);
                S->bits[i] = bs;
            }
        }
        uint64_t ep = 0; uint32_t nlev = 0;
        uint64_t* fr = S->frontier + grp * 64;
        for (uint32_t t = 0; t < ntouched; t++) {
            uint32_t v = touched[t];
            uint64_t m = lvmask[v];
            ep += (g->roff[v + 1] - g->roff[v]) * (uint64_t)__builtin_popcountll(m);
            for (uint32_t L = 0; L < 64; L++)
                if (m >> L & 1) { fr[L]++; if (L + 1 > nlev) nlev = L + 1; }
            lvmask[v] = 0;
        }
        S->e_phys[grp] = ep; S->levels[grp] = nlev;
    }
    pthread_mutex_lock(&J->mu);
    S->e_logical += el_sum;
    pthread_mutex_unlock(&J->mu);
    free(lvmask); free(touched);
    scratch_free(&w);
    return NULL;
}

void or_store_free(or_store* S) {
    if (!S) return;
    for (uint64_t i = 0; i < S->count; i++) { free(S->list[i]); free(S->bits[i]); }
    free(S->list); free(S->bits); free(S->size); free(S->digest);
    free(S->e_phys); free(S->levels); free(S->frontier); free(S);
}

/* samples [s0, s0 + count) -- or ids[0 .. count) in that order if ids != NULL --, traversal groups
 * of `colors` consecutive entries; list_max = 0 selects n/32; keep = 0 keeps no sets */
or_store* or_store_build_ids(const or_graph* g, uint64_t seed, uint64_t s0, const uint64_t* ids, uint64_t count,
                             uint32_t colors, int nthreads, uint32_t list_max, int keep) {
    if (colors == 0 || g->model != 0) return NULL;
    or_store* S = (or_store*)calloc(1, sizeof(or_store));
    S->n = g->n; S->colors = colors; S->s0 = s0; S->count = count; S->ids = ids; S->keep = keep;
    S->ngroups = (count + colors - 1) / colors;
    S->list_max = list_max ? list_max : g->n / 32;
    S->size = (uint32_t*)calloc(count ? count : 1, sizeof(uint32_t));
    S->digest = (uint64_t*)calloc(count ? count : 1, sizeof(uint64_t));
    S->list = (uint32_t**)calloc(count ? count : 1, sizeof(uint32_t*));
    S->bits = (uint64_t**)calloc(count ? count : 1, sizeof(uint64_t*));
    S->e_phys = (uint64_t*)calloc(S->ngroups ? S->ngroups : 1, sizeof(uint64_t));
    S->levels = (uint32_t*)calloc(S->ngroups ? S->ngroups : 1, sizeof(uint32_t));
    S->frontier = (uint64_t*)calloc((S->ngroups ? S->ngroups : 1) * 64, sizeof(uint64_t));
    store_job J;
    J.g = g; J.k = keys_of(seed); J.S = S;
    atomic_init(&J.next, 0); atomic_init(&J.fail, 0);
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, store_worker, &J);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    if (atomic_load(&J.fail)) { or_store_free(S); return NULL; }
    S->ids = NULL;  /* not retained */
    return S;
}

or_store* or_store_build(const or_graph* g, uint64_t seed, uint64_t s0, uint64_t count, uint32_t colors,
                         int nthreads, uint32_t list_max) {
    return or_store_build_ids(g, seed, s0, NULL, count, colors, nthreads, list_max, 1);
}

void or_store_info(const or_store* S, uint32_t* sizes, uint64_t* digests, uint64_t* e_phys, uint32_t* levels,
                   uint64_t* frontier, uint64_t* e_logical) {
    if (sizes) memcpy(sizes, S->size, S->count * sizeof(uint32_t));
    if (digests) memcpy(digests, S->digest, S->count * sizeof(uint64_t));
    if (e_phys) memcpy(e_phys, S->e_phys, S->ngroups * sizeof(uint64_t));
    if (levels) memcpy(levels, S->levels, S->ngroups * sizeof(uint32_t));
    if (frontier) memcpy(frontier, S->frontier, S->ngroups * 64 * sizeof(uint64_t));
    if (e_logical) *e_logical = S->e_logical;
}

/* members of sample s0 + i, ascending; returns the size */
uint32_t or_store_members(const or_store* S, uint64_t i, uint32_t* out) {
    if (S->list[i]) { memcpy(out, S->list[i], (size_t)S->size[i] * sizeof(uint32_t)); return S->size[i]; }
    uint32_t c = 0;
    for (uint32_t wd = 0; wd < (S->n + 63) / 64; wd++)
        for (uint64_t m = S->bits[i][wd]; m; m &= m - 1) out[c++] = wd * 64 + (uint32_t)__builtin_ctzll(m);
    return c;
}

static int store_contains(const or_store* S, uint64_t i, uint32_t v) {
    if (S->bits[i]) return (int)(S->bits[i][v >> 6] >> (v & 63) & 1);
    uint32_t lo = 0, hi = S->size[i];
    const uint32_t* l = S->list[i];
    while (lo < hi) { uint32_t mid = (lo + hi) / 2; if (l[mid] < v) lo = mid + 1; else hi = mid; }
    return lo < S->size[i] && l[lo] == v;
}

static void store_leave(const or_store* S, uint64_t i, uint64_t* cnt) {
    if (S->list[i]) { for (uint32_t j = 0; j < S->size[i]; j++) cnt[S->list[i][j]]--; return; }
    for (uint32_t wd = 0; wd < (S->n + 63) / 64; wd++)
        for (uint64_t m = S->bits[i][wd]; m; m &= m - 1) cnt[wd * 64 + (uint32_t)__builtin_ctzll(m)]--;
}

int or_store_greedy(const or_store* S, uint32_t k, uint32_t* seeds, uint64_t* gains) {
    if (k == 0 || k > S->n) return -1;
    uint64_t* cnt = (uint64_t*)calloc(S->n, sizeof(uint64_t));
    uint8_t* covered = (uint8_t*)calloc(S->count ? S->count : 1, 1);
    uint8_t* selected = (uint8_t*)calloc(S->n, 1);
    for (uint64_t i = 0; i < S->count; i++) {   /* occurrence counts: gain of every vertex */
        if (S->list[i]) { for (uint32_t j = 0; j < S->size[i]; j++) cnt[S->list[i][j]]++; continue; }
        for (uint32_t wd = 0; wd < (S->n + 63) / 64; wd++)
            for (uint64_t m = S->bits[i][wd]; m; m &= m - 1) cnt[wd * 64 + (uint32_t)__builtin_ctzll(m)]++;
    }
    for (uint32_t r = 0; r < k; r++) {
        int64_t best = -1; uint64_t bg = 0;
        for (uint32_t v = 0; v < S->n; v++) {
            if (selected[v]) continue;
            if (best < 0 || cnt[v] > bg) { best = v; bg = cnt[v]; }   /* strict: smallest id wins ties */
        }
        uint32_t b = (uint32_t)best;
        selected[b] = 1; seeds[r] = b; gains[r] = bg;
        for (uint64_t i = 0; i < S->count; i++) {
            if (covered[i] || !store_contains(S, i, b)) continue;
            covered[i] = 1;
            store_leave(S, i, cnt);
        }
    }
    free(cnt); free(covered); free(selected);
    return 0;
}
