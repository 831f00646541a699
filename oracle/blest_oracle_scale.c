/* TEST INFRASTRUCTURE ONLY — full-scale half of the CPU oracle (see blest_oracle.h).
 * Never linked into the product library; only tests/, __graft_entry__.smoke() and
 * bench.py's validation / cpu_baseline / reference legs load it, as the checker.
 *
 * The functions here produce exactly what the single-threaded restatements in
 * blest_oracle.c (and the reference, "R:" = /root/reference/proj/) produce, with work
 * split over host threads and without materialising the mirrored arc list, so a
 * Kronecker scale-27 graph (4.3 G arcs) fits a GPU box's host memory:
 *
 *   orc_gen_csr            generator twin -> relabel -> Graph::from_edges (R:src/graph.cpp:33-55)
 *   orc_permute_csr        apply_permutation (R:src/graph.cpp:126-134)
 *   orc_transpose_csr      in-view (R:src/graph.cpp:52-53, build_csr of the reversed arcs)
 *   orc_symmetrise_csr     symmetrised_adjacency (R:src/ordering.cpp:171-182)
 *   orc_jaccard_windows    jaccard_with_windows (R:src/ordering.cpp:139-166, WindowClusterer :65-135)
 *   orc_rcm                rcm (R:src/ordering.cpp:190-266)
 *   orc_bvss_count_mt/fill_mt  build_bvss (R:src/bvss.cpp:19-101)
 *
 * Each is pinned against the reference (tests/test_oracle_scale_cpu.py).
 */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "blest_oracle.h"

#define INF32 0xFFFFFFFFu

/* ---------------------------------------------------------------------------------
 * A tiny fork/join parallel-for: chunks of [0, count) handed out from a counter.
 * --------------------------------------------------------------------------------- */
typedef void (*RangeFn)(void* ctx, uint64_t lo, uint64_t hi, int tid);
typedef struct {
    RangeFn fn;
    void* ctx;
    uint64_t count, chunk, next;
    int tid_next;
} ParFor;

static void* parfor_worker(void* arg) {
    ParFor* p = (ParFor*)arg;
    const int tid = __atomic_fetch_add(&p->tid_next, 1, __ATOMIC_RELAXED);
    for (;;) {
        const uint64_t lo = __atomic_fetch_add(&p->next, p->chunk, __ATOMIC_RELAXED);
        if (lo >= p->count) return NULL;
        const uint64_t hi = lo + p->chunk < p->count ? lo + p->chunk : p->count;
        p->fn(p->ctx, lo, hi, tid);
    }
}

static void parallel_for(int threads, uint64_t count, uint64_t chunk, RangeFn fn, void* ctx) {
    if (threads < 1) threads = 1;
    if (chunk < 1) chunk = 1;
    ParFor p = {fn, ctx, count, chunk, 0, 0};
    pthread_t* t = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 1; i < threads; ++i) pthread_create(&t[i], NULL, parfor_worker, &p);
    parfor_worker(&p);
    for (int i = 1; i < threads; ++i) pthread_join(t[i], NULL);
    free(t);
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

static void sort_u32(uint32_t* a, uint64_t len) {
    if (len <= 24) { /* insertion sort */
        for (uint64_t i = 1; i < len; ++i) {
            const uint32_t x = a[i];
            uint64_t j = i;
            while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
            a[j] = x;
        }
    } else {
        qsort(a, len, sizeof(uint32_t), cmp_u32);
    }
}

void orc_free(void* p) { free(p); }

/* ---------------------------------------------------------------------------------
 * Generated graphs. Edge e of RMAT / urand and the grid's per-vertex edges are the same
 * pure functions as orc_gen_rmat / orc_gen_urand / orc_gen_grid (blest_oracle.c), so the
 * arc multiset equals the one those lists feed to orc_from_edges.
 * --------------------------------------------------------------------------------- */
typedef struct {
    int kind; /* 0 rmat, 1 urand, 2 grid */
    uint32_t a, b, n;
    uint64_t k, seed;
    uint64_t ab, abc, words;
    uint32_t t0;
    const uint32_t* fwd; /* relabel (forward map) or NULL */
    /* bucketed build: items are cut into `chunks` chunks of `per` items; every arc key
     * (src << 32 | dst) goes to bucket src / vpb */
    uint64_t items, per, chunks;
    uint32_t buckets, vpb;
    uint64_t* keys;      /* chunk c's keys at [c * 2 * per * ipk, ...) */
    uint32_t ipk;        /* max edges per item (grid: 2) */
    uint64_t* nkeys;     /* keys per chunk */
    uint64_t* hist;      /* [chunk][bucket] counts, then scatter cursors */
    uint64_t* bstart;    /* bucket start in `sorted` (buckets + 1) */
    uint64_t* sorted;    /* keys grouped by bucket */
    uint32_t* deg;       /* deduplicated degree per vertex */
    uint64_t* off;
    uint32_t* tgt;
} GenCtx;

/* Edges of item i (edge index, or grid vertex): returns the count (0..2). */
static inline int gen_item(const GenCtx* c, uint64_t i, uint32_t* u, uint32_t* v) {
    if (c->kind == 0) {
        uint32_t x = 0, y = 0;
        uint64_t w = 0;
        for (uint32_t lvl = 0; lvl < c->a; ++lvl) {
            if ((lvl & 1) == 0) w = orc_hash64(c->seed, i * c->words + lvl / 2);
            const uint64_t r = (lvl & 1) ? (w >> 32) : (w & 0xFFFFFFFFull);
            uint32_t bu, bv;
            if (r < c->t0) { bu = 0; bv = 0; }
            else if (r < c->ab) { bu = 0; bv = 1; }
            else if (r < c->abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            x = (x << 1) | bu;
            y = (y << 1) | bv;
        }
        u[0] = x;
        v[0] = y;
        return 1;
    }
    if (c->kind == 1) {
        u[0] = (uint32_t)(((unsigned __int128)orc_hash64(c->seed, 2 * i) * c->n) >> 64);
        v[0] = (uint32_t)(((unsigned __int128)orc_hash64(c->seed, 2 * i + 1) * c->n) >> 64);
        return 1;
    }
    const uint32_t rows = c->a, cols = c->b;
    const uint32_t r = (uint32_t)(i / cols), col = (uint32_t)(i % cols), x = (uint32_t)i;
    int k = 0;
    if (col + 1 < cols) { u[k] = x; v[k] = x + 1; ++k; }
    if (r + 1 < rows) { u[k] = x; v[k] = x + cols; ++k; }
    return k;
}

/* Phase A: each chunk generates its arc keys (mirrored, self-loops dropped, relabelled;
 * R:src/graph.cpp:35-44) into its own region and counts them per bucket. */
static void gen_chunks(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    GenCtx* c = (GenCtx*)ctx;
    for (uint64_t ch = lo; ch < hi; ++ch) {
        uint64_t* out = c->keys + ch * 2 * c->per * c->ipk;
        uint64_t* h = c->hist + ch * c->buckets;
        const uint64_t b = ch * c->per, e = b + c->per < c->items ? b + c->per : c->items;
        uint64_t nk = 0;
        for (uint64_t i = b; i < e; ++i) {
            uint32_t u[2], v[2];
            const int k = gen_item(c, i, u, v);
            for (int j = 0; j < k; ++j) {
                uint32_t x = u[j], y = v[j];
                if (x == y) continue;
                if (c->fwd) { x = c->fwd[x]; y = c->fwd[y]; }
                out[nk++] = (uint64_t)x << 32 | y;
                out[nk++] = (uint64_t)y << 32 | x;
                ++h[x / c->vpb];
                ++h[y / c->vpb];
            }
        }
        c->nkeys[ch] = nk;
    }
}

/* Phase C: scatter each chunk's keys to its (bucket, chunk) slots — stable, no atomics. */
static void gen_scatter(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    GenCtx* c = (GenCtx*)ctx;
    for (uint64_t ch = lo; ch < hi; ++ch) {
        const uint64_t* in = c->keys + ch * 2 * c->per * c->ipk;
        uint64_t* cur = c->hist + ch * c->buckets;
        for (uint64_t i = 0; i < c->nkeys[ch]; ++i) {
            const uint64_t key = in[i];
            c->sorted[cur[(key >> 32) / c->vpb]++] = key;
        }
    }
}

/* Phase D: per bucket, counting sort by source, then sort + unique every list
 * (R:src/graph.cpp:45-46); the deduplicated targets are written back as u32 over the
 * start of the bucket's own key range. */
static void gen_buckets(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    GenCtx* c = (GenCtx*)ctx;
    for (uint64_t bk = lo; bk < hi; ++bk) {
        const uint64_t s = c->bstart[bk], e = c->bstart[bk + 1], len = e - s;
        const uint32_t v0 = (uint32_t)(bk * c->vpb);
        const uint32_t v1 = (uint64_t)v0 + c->vpb < c->n ? v0 + c->vpb : c->n;
        const uint32_t nv = v1 - v0;
        uint64_t* cnt = (uint64_t*)calloc((size_t)nv + 1, sizeof(uint64_t));
        uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (len ? len : 1));
        for (uint64_t i = s; i < e; ++i) ++cnt[(uint32_t)(c->sorted[i] >> 32) - v0 + 1];
        for (uint32_t x = 0; x < nv; ++x) cnt[x + 1] += cnt[x];
        for (uint64_t i = s; i < e; ++i) {
            const uint64_t key = c->sorted[i];
            tmp[cnt[(uint32_t)(key >> 32) - v0]++] = (uint32_t)key;
        }
        uint32_t* dst = (uint32_t*)(c->sorted + s);
        uint64_t w = 0, b = 0;
        for (uint32_t x = 0; x < nv; ++x) { /* cnt[x] is now the end of x's list */
            uint32_t* a = tmp + b;
            const uint64_t l = cnt[x] - b;
            sort_u32(a, l);
            uint64_t d = 0;
            for (uint64_t i = 0; i < l; ++i)
                if (i == 0 || a[i] != a[i - 1]) dst[w + d++] = a[i];
            c->deg[v0 + x] = (uint32_t)d;
            w += d;
            b = cnt[x];
        }
        free(tmp);
        free(cnt);
    }
}

static void gen_compact(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    GenCtx* c = (GenCtx*)ctx;
    for (uint64_t bk = lo; bk < hi; ++bk) {
        const uint32_t v0 = (uint32_t)(bk * c->vpb);
        const uint32_t v1 = (uint64_t)v0 + c->vpb < c->n ? v0 + c->vpb : c->n;
        if (v0 >= v1) continue;
        const uint32_t* src = (const uint32_t*)(c->sorted + c->bstart[bk]);
        memcpy(c->tgt + c->off[v0], src, sizeof(uint32_t) * (c->off[v1] - c->off[v0]));
    }
}

uint64_t orc_gen_csr(int kind, uint32_t a, uint32_t b, uint64_t k, uint64_t seed, uint32_t t0,
                     uint32_t t1, uint32_t t2, const uint32_t* forward, int threads,
                     uint64_t** off_out, uint32_t** tgt_out) {
    GenCtx c;
    memset(&c, 0, sizeof c);
    if (threads < 1) threads = 1;
    c.kind = kind;
    c.a = a;
    c.b = b;
    c.k = k;
    c.seed = seed;
    c.t0 = t0;
    c.ab = (uint64_t)t0 + t1;
    c.abc = c.ab + t2;
    c.words = ((uint64_t)a + 1) / 2;
    c.fwd = forward;
    const uint64_t n64 = kind == 0 ? (1ull << a) : (kind == 1 ? a : (uint64_t)a * b);
    const uint32_t n = (uint32_t)n64;
    c.n = n;
    c.items = kind == 2 ? n64 : k;
    c.ipk = kind == 2 ? 2 : 1;
    c.chunks = (uint64_t)threads * 16;
    c.per = (c.items + c.chunks - 1) / c.chunks;
    if (c.per == 0) c.per = 1;
    c.chunks = (c.items + c.per - 1) / c.per;
    c.buckets = n < 4096 ? (n ? n : 1) : 4096;
    c.vpb = (uint32_t)((n64 + c.buckets - 1) / c.buckets);
    if (c.vpb == 0) c.vpb = 1;
    c.buckets = (uint32_t)((n64 + c.vpb - 1) / c.vpb);  /* every bucket starts below n */
    if (c.buckets == 0) c.buckets = 1;
    c.keys = (uint64_t*)malloc(sizeof(uint64_t) * (c.chunks * 2 * c.per * c.ipk + 1));
    c.nkeys = (uint64_t*)calloc(c.chunks + 1, sizeof(uint64_t));
    c.hist = (uint64_t*)calloc(c.chunks * c.buckets + 1, sizeof(uint64_t));
    parallel_for(threads, c.chunks, 1, gen_chunks, &c);
    /* Phase B: bucket-major, chunk-minor exclusive scan -> scatter cursors */
    c.bstart = (uint64_t*)malloc(sizeof(uint64_t) * ((uint64_t)c.buckets + 1));
    uint64_t run = 0;
    for (uint32_t bk = 0; bk < c.buckets; ++bk) {
        c.bstart[bk] = run;
        for (uint64_t ch = 0; ch < c.chunks; ++ch) {
            const uint64_t x = c.hist[ch * c.buckets + bk];
            c.hist[ch * c.buckets + bk] = run;
            run += x;
        }
    }
    c.bstart[c.buckets] = run;
    c.sorted = (uint64_t*)malloc(sizeof(uint64_t) * (run ? run : 1));
    parallel_for(threads, c.chunks, 1, gen_scatter, &c);
    free(c.keys);
    free(c.hist);
    free(c.nkeys);
    c.deg = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    parallel_for(threads, c.buckets, 1, gen_buckets, &c);
    c.off = (uint64_t*)malloc(sizeof(uint64_t) * ((uint64_t)n + 1));
    c.off[0] = 0;
    for (uint32_t u = 0; u < n; ++u) c.off[u + 1] = c.off[u] + c.deg[u];
    c.tgt = (uint32_t*)malloc(sizeof(uint32_t) * (c.off[n] ? c.off[n] : 1));
    parallel_for(threads, c.buckets, 1, gen_compact, &c);
    free(c.sorted);
    free(c.bstart);
    free(c.deg);
    *off_out = c.off;
    *tgt_out = c.tgt;
    return c.off[n];
}

/* Seeded relabel, multi-threaded: forward[i] = rank of (hash64(seed, i), i) — the same
 * map as orc_random_relabel. Chunks sorted in parallel, then one k-way merge. */
typedef struct { uint64_t key; uint32_t idx; } KI;
static int cmp_ki(const void* x, const void* y) {
    const KI* a = (const KI*)x;
    const KI* b = (const KI*)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}
typedef struct { KI* k; uint64_t n, per; uint64_t seed; } RelCtx;
static void rel_fill_sort(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    RelCtx* c = (RelCtx*)ctx;
    for (uint64_t ch = lo; ch < hi; ++ch) {
        const uint64_t b = ch * c->per, e = b + c->per < c->n ? b + c->per : c->n;
        for (uint64_t i = b; i < e; ++i) { c->k[i].key = orc_hash64(c->seed, i); c->k[i].idx = (uint32_t)i; }
        qsort(c->k + b, e - b, sizeof(KI), cmp_ki);
    }
}
void orc_random_relabel_mt(uint32_t n, uint64_t seed, int threads, uint32_t* forward) {
    if (threads < 1) threads = 1;
    const uint64_t chunks = (uint64_t)threads * 4;
    RelCtx c = {(KI*)malloc(sizeof(KI) * (n ? n : 1)), n, (n + chunks - 1) / chunks, seed};
    if (c.per == 0) c.per = 1;
    const uint64_t nch = (n + c.per - 1) / c.per;
    parallel_for(threads, nch, 1, rel_fill_sort, &c);
    uint64_t* head = (uint64_t*)malloc(sizeof(uint64_t) * (nch ? nch : 1));
    for (uint64_t ch = 0; ch < nch; ++ch) head[ch] = ch * c.per;
    for (uint32_t p = 0; p < n; ++p) { /* merge: the smallest head (nch is small) */
        uint64_t best = UINT64_MAX;
        for (uint64_t ch = 0; ch < nch; ++ch) {
            const uint64_t e = (ch + 1) * c.per < n ? (ch + 1) * c.per : n;
            if (head[ch] < e && (best == UINT64_MAX || cmp_ki(&c.k[head[ch]], &c.k[head[best]]) < 0)) best = ch;
        }
        forward[c.k[head[best]].idx] = p;
        ++head[best];
    }
    free(head);
    free(c.k);
}

/* ---------------------------------------------------------------------------------
 * apply_permutation (R:src/graph.cpp:126-134) on a CSR: arc (u, v) -> (f[u], f[v]).
 * The arc set stays duplicate-free, so only the new lists need sorting.
 * --------------------------------------------------------------------------------- */
typedef struct {
    const uint64_t* off;
    const uint32_t* tgt;
    const uint32_t* fwd;
    uint64_t* off2;
    uint32_t* tgt2;
} PermCtx;
static void perm_lists(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    PermCtx* c = (PermCtx*)ctx;
    for (uint64_t u = lo; u < hi; ++u) {
        uint32_t* d = c->tgt2 + c->off2[c->fwd[u]];
        const uint64_t b = c->off[u], len = c->off[u + 1] - b;
        for (uint64_t i = 0; i < len; ++i) d[i] = c->fwd[c->tgt[b + i]];
        sort_u32(d, len);
    }
}
uint64_t orc_permute_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint32_t* forward,
                         int threads, uint64_t* off_out, uint32_t* tgt_out) {
    memset(off_out, 0, sizeof(uint64_t) * ((uint64_t)n + 1));
    for (uint32_t u = 0; u < n; ++u) off_out[forward[u] + 1] = off[u + 1] - off[u];
    for (uint32_t u = 0; u < n; ++u) off_out[u + 1] += off_out[u];
    PermCtx c = {off, tgt, forward, off_out, tgt_out};
    parallel_for(threads, n, 1 << 12, perm_lists, &c);
    return off_out[n];
}

/* In-view (sources of each vertex's in-arcs, ascending): a stable scatter by source. */
uint64_t orc_transpose_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint64_t* ioff,
                           uint32_t* isrc) {
    memset(ioff, 0, sizeof(uint64_t) * ((uint64_t)n + 1));
    const uint64_t m = off[n];
    for (uint64_t i = 0; i < m; ++i) ++ioff[tgt[i] + 1];
    for (uint32_t u = 0; u < n; ++u) ioff[u + 1] += ioff[u];
    uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    memcpy(cur, ioff, sizeof(uint64_t) * n);
    for (uint32_t u = 0; u < n; ++u)
        for (uint64_t i = off[u]; i < off[u + 1]; ++i) isrc[cur[tgt[i]]++] = u;
    free(cur);
    return m;
}

/* symmetrised_adjacency (R:src/ordering.cpp:171-182): sorted-unique out ∪ in per vertex.
 * Two calls: with aoff only (counts -> offsets, returns the total), then with atgt. */
uint64_t orc_symmetrise_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint64_t* ioff,
                            const uint32_t* isrc, uint64_t* aoff, uint32_t* atgt) {
    if (!atgt) aoff[0] = 0;
    for (uint32_t u = 0; u < n; ++u) {
        uint64_t i = off[u], j = ioff[u], k = atgt ? aoff[u] : 0;
        const uint64_t ie = off[u + 1], je = ioff[u + 1];
        uint32_t last = INF32;
        int have = 0;
        while (i < ie || j < je) {
            uint32_t x;
            if (j >= je || (i < ie && tgt[i] <= isrc[j])) x = tgt[i++];
            else x = isrc[j++];
            if (have && x == last) continue;
            last = x;
            have = 1;
            if (atgt) atgt[k] = x;
            ++k;
        }
        if (!atgt) aoff[u + 1] = aoff[u] + k;
    }
    return aoff[n];
}

/* ---------------------------------------------------------------------------------
 * jaccard_with_windows (R:src/ordering.cpp:139-166; WindowClusterer :65-135), windows
 * split over threads like the reference's workers (:152). Per cluster: seed = smallest
 * unpicked id (:79-80); then sigma-1 greedy picks maximising
 * J = inter / (deg + |U| - inter) in double, ties to the smallest id (:111-126).
 * inter is maintained incrementally as in take() (:92-109). Data-structure changes that
 * do not change the result: "x already in U" is a binary search in the <= 7 earlier
 * members' sorted out-lists (instead of an n-sized epoch array); the argmax scans only
 * the candidates (unpicked ids with inter > 0 this cluster — every one of them scores
 * > 0 and so beats any non-candidate); with no candidate the smallest unpicked id wins,
 * exactly as the reference's strict '>' scan from -1.0 resolves it.
 * --------------------------------------------------------------------------------- */
typedef struct {
    const uint64_t* off;
    const uint32_t* tgt;
    const uint64_t* ioff;
    const uint32_t* isrc;
    uint32_t n, sigma, w;
    uint32_t* forward;
    /* per-thread scratch, w entries each */
    uint32_t** inter;
    uint32_t** stamp;
    uint32_t** cand;
    unsigned char** picked;
    uint32_t* epoch;
} JacCtx;

static int bsearch_in(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t x) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] == x) return 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return 0;
}

static void jac_windows(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    JacCtx* c = (JacCtx*)ctx;
    uint32_t* inter = c->inter[tid];
    uint32_t* stamp = c->stamp[tid];
    uint32_t* cand = c->cand[tid];
    unsigned char* picked = c->picked[tid];
    for (uint64_t win = lo; win < hi; ++win) {
        const uint32_t begin = (uint32_t)(win * c->w);
        const uint32_t end = (uint64_t)begin + c->w < c->n ? begin + c->w : c->n;
        const uint32_t len = end - begin;
        memset(picked, 0, len);
        uint32_t first_unpicked = 0, pos = 0;
        while (pos < len) {
            const uint32_t ep = ++c->epoch[tid];
            uint32_t union_size = 0, cc = 0, nmem = 0;
            uint32_t members[8];
            while (picked[first_unpicked]) ++first_unpicked;
            uint32_t best = begin + first_unpicked;
            for (uint32_t r = 0; r < c->sigma && pos < len; ++r) {
                if (r > 0) { /* argmax (:111-126) over the candidates */
                    double bs = -1.0;
                    uint32_t bj = INF32;
                    const double us = (double)union_size;
                    for (uint32_t i = 0; i < cc; ++i) {
                        const uint32_t j = cand[i];
                        if (picked[j - begin]) continue;
                        const uint32_t it = inter[j - begin];
                        const double denom = ((double)(c->off[j + 1] - c->off[j]) + us) - (double)it;
                        const double score = denom > 0 ? (double)it / denom : 0.0;
                        if (score > bs || (score == bs && j < bj)) { bs = score; bj = j; }
                    }
                    if (bj == INF32) {
                        while (picked[first_unpicked]) ++first_unpicked;
                        bj = begin + first_unpicked;
                    }
                    best = bj;
                }
                /* take(best) (:92-109) */
                const uint32_t v = best;
                picked[v - begin] = 1;
                c->forward[v] = begin + pos++;
                for (uint64_t i = c->off[v]; i < c->off[v + 1]; ++i) {
                    const uint32_t x = c->tgt[i];
                    int fresh = 1;
                    for (uint32_t q = 0; q < nmem && fresh; ++q)
                        if (bsearch_in(c->tgt, c->off[members[q]], c->off[members[q] + 1], x)) fresh = 0;
                    if (!fresh) continue;
                    ++union_size;
                    uint64_t t = c->ioff[x], te = c->ioff[x + 1];
                    { /* lower_bound(begin) */
                        uint64_t l = t, h = te;
                        while (l < h) {
                            const uint64_t mid = (l + h) >> 1;
                            if (c->isrc[mid] < begin) l = mid + 1;
                            else h = mid;
                        }
                        t = l;
                    }
                    for (; t < te; ++t) {
                        const uint32_t j = c->isrc[t];
                        if (j >= end) break;
                        if (picked[j - begin]) continue;
                        if (stamp[j - begin] != ep) {
                            stamp[j - begin] = ep;
                            inter[j - begin] = 0;
                            cand[cc++] = j;
                        }
                        ++inter[j - begin];
                    }
                }
                members[nmem++] = v;
            }
        }
    }
}

int orc_jaccard_windows(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint64_t* ioff,
                        const uint32_t* isrc, uint32_t sigma, uint32_t w, int threads, uint32_t* forward) {
    if (sigma == 0 || sigma > 8 || w == 0 || w % sigma != 0) return -1;
    if (n == 0) return 0;
    if (threads < 1) threads = 1;
    const uint64_t num_windows = ((uint64_t)n + w - 1) / w;
    JacCtx c = {off, tgt, ioff, isrc, n, sigma, w, forward, NULL, NULL, NULL, NULL, NULL};
    c.inter = (uint32_t**)malloc(sizeof(void*) * threads);
    c.stamp = (uint32_t**)malloc(sizeof(void*) * threads);
    c.cand = (uint32_t**)malloc(sizeof(void*) * threads);
    c.picked = (unsigned char**)malloc(sizeof(void*) * threads);
    c.epoch = (uint32_t*)calloc(threads, sizeof(uint32_t));
    for (int t = 0; t < threads; ++t) {
        c.inter[t] = (uint32_t*)malloc(sizeof(uint32_t) * w);
        c.stamp[t] = (uint32_t*)calloc(w, sizeof(uint32_t));
        c.cand[t] = (uint32_t*)malloc(sizeof(uint32_t) * w);
        c.picked[t] = (unsigned char*)malloc(w);
    }
    parallel_for(threads, num_windows, 1, jac_windows, &c);
    for (int t = 0; t < threads; ++t) {
        free(c.inter[t]);
        free(c.stamp[t]);
        free(c.cand[t]);
        free(c.picked[t]);
    }
    free(c.inter);
    free(c.stamp);
    free(c.cand);
    free(c.picked);
    free(c.epoch);
    return 0;
}

/* ---------------------------------------------------------------------------------
 * rcm (R:src/ordering.cpp:246-266) over the symmetrised adjacency (aoff, atgt):
 * per unplaced vertex v (ascending), pseudo_peripheral(v) (:220-242) by repeated
 * sym_bfs (:190-218) — the smallest (degree, id) vertex of the last level, until the
 * eccentricity stops growing — then sym_bfs from it with children sorted by
 * (degree, id); the concatenated visit orders reversed give the inverse map.
 * Levels are reset only over the visited vertices (same result, O(n + m) per pass
 * instead of the reference's n-sized arrays per component).
 * --------------------------------------------------------------------------------- */
static const uint32_t* g_rcm_deg; /* qsort comparator context (orc_rcm is not reentrant) */
static int cmp_deg_id(const void* x, const void* y) {
    const uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    if (g_rcm_deg[a] != g_rcm_deg[b]) return g_rcm_deg[a] < g_rcm_deg[b] ? -1 : 1;
    return (a > b) - (a < b);
}

static uint32_t rcm_bfs(const uint64_t* aoff, const uint32_t* atgt, uint32_t* level, uint32_t start,
                        int sort_children, uint32_t* out, uint64_t* out_len) {
    uint64_t len = 0;
    level[start] = 0;
    out[len++] = start;
    uint32_t ecc = 0;
    for (uint64_t head = 0; head < len; ++head) {
        const uint32_t u = out[head];
        const uint64_t first = len;
        for (uint64_t i = aoff[u]; i < aoff[u + 1]; ++i) {
            const uint32_t v = atgt[i];
            if (level[v] == INF32) {
                level[v] = level[u] + 1;
                if (level[v] > ecc) ecc = level[v];
                out[len++] = v;
            }
        }
        if (sort_children && len - first > 1) qsort(out + first, len - first, sizeof(uint32_t), cmp_deg_id);
    }
    *out_len = len;
    return ecc;
}

void orc_rcm(uint32_t n, const uint64_t* aoff, const uint32_t* atgt, uint32_t* forward) {
    uint32_t* deg = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint32_t u = 0; u < n; ++u) deg[u] = (uint32_t)(aoff[u + 1] - aoff[u]);
    g_rcm_deg = deg;
    uint32_t* level = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint32_t u = 0; u < n; ++u) level[u] = INF32;
    uint32_t* visit = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    unsigned char* placed = (unsigned char*)calloc(n ? n : 1, 1);
    uint64_t placed_n = 0, len = 0;
    for (uint32_t v = 0; v < n; ++v) {
        if (placed[v]) continue;
        uint32_t current = v, best_ecc = 0;
        for (;;) {
            const uint32_t ecc = rcm_bfs(aoff, atgt, level, current, 0, visit, &len);
            const int stop = (ecc <= best_ecc && current != v) || ecc == 0;
            uint32_t next = current, bk0 = INF32, bk1 = INF32;
            if (!stop)
                for (uint64_t i = 0; i < len; ++i) {
                    const uint32_t x = visit[i];
                    if (level[x] == ecc && (deg[x] < bk0 || (deg[x] == bk0 && x < bk1))) {
                        bk0 = deg[x];
                        bk1 = x;
                        next = x;
                    }
                }
            for (uint64_t i = 0; i < len; ++i) level[visit[i]] = INF32;
            if (stop || ecc <= best_ecc) break;
            best_ecc = ecc;
            current = next;
        }
        rcm_bfs(aoff, atgt, level, current, 1, visit, &len);
        for (uint64_t i = 0; i < len; ++i) {
            level[visit[i]] = INF32;
            placed[visit[i]] = 1;
            order[placed_n++] = visit[i];
        }
    }
    for (uint64_t i = 0; i < placed_n; ++i) forward[order[placed_n - 1 - i]] = (uint32_t)i;
    free(deg);
    free(level);
    free(visit);
    free(order);
    free(placed);
}

/* ---------------------------------------------------------------------------------
 * build_bvss (R:src/bvss.cpp:19-101) with slice sets split over threads. Pass 1 counts the
 * distinct rows of each set's <= 8 sorted out-lists by merging them (same count as the
 * reference's mark array, :35-46); pass 2 is orc_bvss_fill's merge + column-major
 * placement (:71-97, 64-bit slot math) writing each set's own VSS range, padding
 * (mask 0, row n, :60-61) included.
 * --------------------------------------------------------------------------------- */
typedef struct {
    uint32_t n;
    const uint64_t* off;
    const uint32_t* tgt;
    uint32_t* counts; /* pass 1 */
    const uint32_t* rp;
    uint32_t* v2r;
    uint32_t* rows;
    uint32_t* masks;
} BvCtx;

static inline uint32_t set_merge(const BvCtx* c, uint32_t s, uint32_t* row_out, uint32_t* mask_out,
                                 uint64_t base_vss) {
    const uint32_t lo = s * 8, width = (uint64_t)lo + 8 < c->n ? 8 : c->n - lo;
    uint64_t cur[8], end[8];
    for (uint32_t j = 0; j < width; ++j) { cur[j] = c->off[lo + j]; end[j] = c->off[lo + j + 1]; }
    uint64_t k = 0;
    for (;;) {
        uint32_t next = INF32;
        for (uint32_t j = 0; j < width; ++j)
            if (cur[j] < end[j] && c->tgt[cur[j]] < next) next = c->tgt[cur[j]];
        if (next == INF32) break;
        uint32_t mask = 0;
        for (uint32_t j = 0; j < width; ++j)
            if (cur[j] < end[j] && c->tgt[cur[j]] == next) { mask |= 1u << j; ++cur[j]; }
        if (row_out) {
            const uint64_t v = base_vss + k / 128;
            const uint32_t slot = (uint32_t)(k % 128), lane = slot % 32, column = slot / 32;
            mask_out[32 * v + lane] |= mask << (8 * column);
            row_out[4 * (32 * v + lane) + column] = next;
        }
        ++k;
    }
    return (uint32_t)k;
}

static void bv_count(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    BvCtx* c = (BvCtx*)ctx;
    for (uint64_t s = lo; s < hi; ++s) c->counts[s] = set_merge(c, (uint32_t)s, NULL, NULL, 0);
}

static void bv_fill(void* ctx, uint64_t lo, uint64_t hi, int tid) {
    (void)tid;
    BvCtx* c = (BvCtx*)ctx;
    for (uint64_t s = lo; s < hi; ++s) {
        const uint64_t vb = c->rp[s], ve = c->rp[s + 1];
        if (vb == ve) continue;
        for (uint64_t v = vb; v < ve; ++v) c->v2r[v] = (uint32_t)s;
        for (uint64_t i = 128 * vb; i < 128 * ve; ++i) c->rows[i] = c->n;
        memset(c->masks + 32 * vb, 0, sizeof(uint32_t) * 32 * (ve - vb));
        set_merge(c, (uint32_t)s, c->rows, c->masks, vb);
    }
}

uint64_t orc_bvss_count_mt(uint32_t n, const uint64_t* off, const uint32_t* tgt, int threads,
                           uint32_t* real_ptrs, uint64_t* num_unpadded) {
    const uint32_t sets = (uint32_t)(((uint64_t)n + 7) / 8);
    BvCtx c;
    memset(&c, 0, sizeof c);
    c.n = n;
    c.off = off;
    c.tgt = tgt;
    c.counts = (uint32_t*)malloc(sizeof(uint32_t) * (sets ? sets : 1));
    parallel_for(threads, sets, 1 << 10, bv_count, &c);
    uint64_t unp = 0;
    real_ptrs[0] = 0;
    for (uint32_t s = 0; s < sets; ++s) {
        real_ptrs[s + 1] = real_ptrs[s] + (c.counts[s] + 127) / 128; /* :48-53 */
        unp += c.counts[s];
    }
    free(c.counts);
    *num_unpadded = unp;
    return real_ptrs[sets];
}

void orc_bvss_fill_mt(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint32_t* real_ptrs,
                      int threads, uint32_t* v2r, uint32_t* row_ids, uint32_t* masks) {
    const uint32_t sets = (uint32_t)(((uint64_t)n + 7) / 8);
    BvCtx c;
    memset(&c, 0, sizeof c);
    c.n = n;
    c.off = off;
    c.tgt = tgt;
    c.rp = real_ptrs;
    c.v2r = v2r;
    c.rows = row_ids;
    c.masks = masks;
    parallel_for(threads, sets, 1 << 10, bv_fill, &c);
}

/* ---------------------------------------------------------------------------------
 * Traversed undirected edges of a level array (the GTEPS numerator):
 * 1/2 * sum of out-degrees of the reached vertices.
 * --------------------------------------------------------------------------------- */
uint64_t orc_traversed_edges(uint32_t n, const uint64_t* off, const uint32_t* levels) {
    uint64_t s = 0;
    for (uint32_t v = 0; v < n; ++v)
        if (levels[v] != INF32) s += off[v + 1] - off[v];
    return s / 2;
}
