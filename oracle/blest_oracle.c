/* TEST INFRASTRUCTURE ONLY — CPU oracle (see blest_oracle.h). Never linked into the
 * product library; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg load it, as the checker.
 *
 * Each function restates the reference function cited in its comment
 * ("R:" = /root/reference/proj/). Compiled with -ffp-contract=off so the two
 * floating-point statistics round exactly like the reference's x86-64 build.
 */
#include "blest_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define INF32 0xFFFFFFFFu

/* ---------------------------------------------------------------------------------
 * Synthetic inputs. The reference ships no Kronecker/urand generator;
 * these are the harness definitions shared bit-for-bit with the device generators
 * (paper_2512_21967_b200/csrc/generators.cu): a counter-based splitmix64 hash, so the
 * i-th edge is a pure function of (seed, i) on CPU and GPU alike.
 * --------------------------------------------------------------------------------- */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_hash64(uint64_t seed, uint64_t i) { return mix64(mix64(seed) ^ i); }

/* Graph500-style RMAT: per level one 32-bit draw r against integer thresholds
 * a, a+b, a+b+c (probabilities scaled by 2^32) picks the quadrant. */
void orc_gen_rmat(uint32_t scale, uint64_t num_edges, uint64_t seed, uint32_t a, uint32_t b,
                  uint32_t c, uint32_t* src, uint32_t* dst) {
    const uint64_t ab = (uint64_t)a + b, abc = ab + c;
    const uint64_t words = (scale + 1) / 2;
    for (int64_t e = 0; e < (int64_t)num_edges; ++e) {
        uint32_t u = 0, v = 0;
        uint64_t w = 0;
        for (uint32_t k = 0; k < scale; ++k) {
            if ((k & 1) == 0) w = orc_hash64(seed, (uint64_t)e * words + k / 2);
            const uint64_t r = (k & 1) ? (w >> 32) : (w & 0xFFFFFFFFull);
            uint32_t bu, bv;
            if (r < a) { bu = 0; bv = 0; }
            else if (r < ab) { bu = 0; bv = 1; }
            else if (r < abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        src[e] = u;
        dst[e] = v;
    }
}

static inline uint32_t mulhi_n(uint64_t h, uint32_t n) {
    return (uint32_t)(((unsigned __int128)h * n) >> 64);
}

void orc_gen_urand(uint32_t n, uint64_t num_edges, uint64_t seed, uint32_t* src, uint32_t* dst) {
    for (int64_t e = 0; e < (int64_t)num_edges; ++e) {
        src[e] = mulhi_n(orc_hash64(seed, 2 * (uint64_t)e), n);
        dst[e] = mulhi_n(orc_hash64(seed, 2 * (uint64_t)e + 1), n);
    }
}

/* grid_graph (R:tests/support/generators.cpp:41-50): row-major, right then down. */
uint64_t orc_gen_grid(uint32_t rows, uint32_t cols, uint32_t* src, uint32_t* dst) {
    uint64_t k = 0;
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t c = 0; c < cols; ++c) {
            const uint32_t v = r * cols + c;
            if (c + 1 < cols) { if (src) { src[k] = v; dst[k] = v + 1; } ++k; }
            if (r + 1 < rows) { if (src) { src[k] = v; dst[k] = v + cols; } ++k; }
        }
    return k;
}

typedef struct { uint64_t key; uint32_t idx; } KeyIdx;
static int cmp_keyidx(const void* a, const void* b) {
    const KeyIdx* x = (const KeyIdx*)a;
    const KeyIdx* y = (const KeyIdx*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Seeded relabel: new id of i = rank of (hash64(seed, i), i). */
void orc_random_relabel(uint32_t n, uint64_t seed, uint32_t* forward) {
    KeyIdx* k = (KeyIdx*)malloc(sizeof(KeyIdx) * (n ? n : 1));
    for (uint32_t i = 0; i < n; ++i) { k[i].key = orc_hash64(seed, i); k[i].idx = i; }
    qsort(k, n, sizeof(KeyIdx), cmp_keyidx);
    for (uint32_t p = 0; p < n; ++p) forward[k[p].idx] = p;
    free(k);
}

/* ---------------------------------------------------------------------------------
 * Graph construction.
 * --------------------------------------------------------------------------------- */
static void radix_sort_u64(uint64_t* a, uint64_t* tmp, uint64_t k) {
    uint64_t* cnt = (uint64_t*)malloc(sizeof(uint64_t) * 65536);
    for (int pass = 0; pass < 4; ++pass) {
        const int sh = 16 * pass;
        memset(cnt, 0, sizeof(uint64_t) * 65536);
        for (uint64_t i = 0; i < k; ++i) ++cnt[(a[i] >> sh) & 0xFFFF];
        uint64_t nonzero = 0;
        for (int d = 0; d < 65536; ++d) nonzero += cnt[d] != 0;
        if (nonzero <= 1) continue; /* digit constant: pass is the identity */
        uint64_t run = 0;
        for (int d = 0; d < 65536; ++d) { const uint64_t c = cnt[d]; cnt[d] = run; run += c; }
        for (uint64_t i = 0; i < k; ++i) tmp[cnt[(a[i] >> sh) & 0xFFFF]++] = a[i];
        memcpy(a, tmp, sizeof(uint64_t) * k);
    }
    free(cnt);
}

/* Graph::from_edges (R:src/graph.cpp:33-55): mirror when undirected (:35-39), range check
 * (:40-43), drop self-loops (:44), sort + unique (:45-46), CSR by source (:52, build_csr
 * :15-29 — targets end up sorted because the arc list is sorted). */
uint64_t orc_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k,
                        int directed, uint64_t* offsets, uint32_t* targets) {
    const uint64_t total = directed ? k : 2 * k;
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (total ? total : 1));
    uint64_t m = 0;
    for (uint64_t i = 0; i < k; ++i) {
        if (src[i] >= n || dst[i] >= n) { free(keys); return UINT64_MAX; }
        if (src[i] == dst[i]) continue;
        keys[m++] = ((uint64_t)src[i] << 32) | dst[i];
        if (!directed) keys[m++] = ((uint64_t)dst[i] << 32) | src[i];
    }
    uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
    radix_sort_u64(keys, tmp, m);
    free(tmp);
    uint64_t u = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) keys[u++] = keys[i];
    memset(offsets, 0, sizeof(uint64_t) * ((uint64_t)n + 1));
    for (uint64_t i = 0; i < u; ++i) {
        ++offsets[(keys[i] >> 32) + 1];
        targets[i] = (uint32_t)keys[i];
    }
    for (uint32_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
    free(keys);
    return u;
}

/* apply_permutation (R:src/graph.cpp:126-134): relabel every arc and rebuild. The input
 * is already mirrored, so it is rebuilt as directed (the arc set stays symmetric). */
uint64_t orc_apply_permutation(uint32_t n, const uint64_t* off, const uint32_t* tgt,
                               const uint32_t* forward, uint64_t* off_out, uint32_t* tgt_out) {
    const uint64_t m = off[n];
    uint32_t* s = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
    uint32_t* d = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
    for (uint32_t u = 0; u < n; ++u)
        for (uint64_t i = off[u]; i < off[u + 1]; ++i) { s[i] = forward[u]; d[i] = forward[tgt[i]]; }
    const uint64_t r = orc_from_edges(n, s, d, m, 1, off_out, tgt_out);
    free(s);
    free(d);
    return r;
}

/* reference_bfs (R:src/graph.cpp:144-167): FIFO queue over out-edges. */
uint32_t orc_reference_bfs(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint32_t src,
                           uint32_t* levels, uint32_t* num_levels) {
    for (uint32_t v = 0; v < n; ++v) levels[v] = INF32;
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint64_t head = 0, tail = 0;
    levels[src] = 0;
    q[tail++] = src;
    uint32_t visited = 1, max_level = 0;
    while (head < tail) {
        const uint32_t u = q[head++];
        for (uint64_t i = off[u]; i < off[u + 1]; ++i) {
            const uint32_t v = tgt[i];
            if (levels[v] == INF32) {
                levels[v] = levels[u] + 1;
                if (levels[v] > max_level) max_level = levels[v];
                ++visited;
                q[tail++] = v;
            }
        }
    }
    free(q);
    *num_levels = max_level + 1;
    return visited;
}

typedef struct {
    uint32_t n;
    const uint64_t* off;
    const uint32_t* tgt;
    const uint32_t* srcs;
    uint32_t count;
    uint32_t* levels;
    uint32_t* visited;
    uint32_t next; /* work counter */
    pthread_mutex_t mu;
} ManyJob;

static void* many_worker(void* arg) {
    ManyJob* j = (ManyJob*)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        const uint32_t i = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->count) return NULL;
        uint32_t nl;
        j->visited[i] = orc_reference_bfs(j->n, j->off, j->tgt, j->srcs[i],
                                          j->levels + (uint64_t)i * j->n, &nl);
    }
}

void orc_reference_bfs_many(uint32_t n, const uint64_t* off, const uint32_t* tgt,
                            const uint32_t* srcs, uint32_t count, uint32_t* levels,
                            uint32_t* visited, int threads) {
    ManyJob j = {n, off, tgt, srcs, count, levels, visited, 0, PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = 1;
    pthread_t* t = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 1; i < threads; ++i) pthread_create(&t[i], NULL, many_worker, &j);
    many_worker(&j);
    for (int i = 1; i < threads; ++i) pthread_join(t[i], NULL);
    free(t);
}

uint64_t orc_validate_levels(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint32_t src,
                             const uint32_t* L) {
    if (L[src] != 0) return 1 + (uint64_t)src;
    unsigned char* has_parent = (unsigned char*)calloc(n ? n : 1, 1);
    uint64_t bad = 0;
    for (uint32_t u = 0; u < n && !bad; ++u) {
        if (L[u] == INF32) continue;
        for (uint64_t i = off[u]; i < off[u + 1]; ++i) {
            const uint32_t v = tgt[i];
            if (L[v] == INF32 || L[v] > L[u] + 1) { bad = 1 + (uint64_t)v; break; }
            if (L[v] == L[u] + 1) has_parent[v] = 1;
        }
    }
    for (uint32_t v = 0; v < n && !bad; ++v)
        if (L[v] != INF32 && v != src && !has_parent[v]) bad = 1 + (uint64_t)v;
    free(has_parent);
    return bad;
}

/* ---------------------------------------------------------------------------------
 * BVSS (R:src/bvss.cpp:19-101). sigma = 8, tau = 128, lane = slot % 32,
 * column = slot / 32, masks[32v+lane] byte `column`, row_ids[4(32v+lane)+column].
 * --------------------------------------------------------------------------------- */
uint64_t orc_bvss_count(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint32_t* real_ptrs,
                        uint64_t* num_unpadded) {
    const uint32_t sets = (uint32_t)(((uint64_t)n + 7) / 8);
    uint32_t* mark = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint32_t v = 0; v < n; ++v) mark[v] = INF32;
    uint64_t unpadded = 0;
    real_ptrs[0] = 0;
    for (uint32_t s = 0; s < sets; ++s) { /* pass 1, R:src/bvss.cpp:35-46 */
        const uint32_t lo = s * 8;
        const uint32_t hi = (uint64_t)lo + 8 < n ? lo + 8 : n;
        uint32_t count = 0;
        for (uint32_t col = lo; col < hi; ++col)
            for (uint64_t i = off[col]; i < off[col + 1]; ++i)
                if (mark[tgt[i]] != s) { mark[tgt[i]] = s; ++count; }
        real_ptrs[s + 1] = real_ptrs[s] + (count + 127) / 128; /* :48-53 */
        unpadded += count;
    }
    free(mark);
    *num_unpadded = unpadded;
    return real_ptrs[sets];
}

void orc_bvss_fill(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint32_t* real_ptrs,
                   uint64_t num_vss, uint32_t* v2r, uint32_t* row_ids, uint32_t* masks) {
    const uint32_t sets = (uint32_t)(((uint64_t)n + 7) / 8);
    for (uint32_t s = 0; s < sets; ++s) /* :55-58 */
        for (uint32_t v = real_ptrs[s]; v < real_ptrs[s + 1]; ++v) v2r[v] = s;
    for (uint64_t i = 0; i < num_vss * 128; ++i) row_ids[i] = n; /* :60 sentinel */
    memset(masks, 0, sizeof(uint32_t) * num_vss * 32);           /* :61 */
    for (uint32_t s = 0; s < sets; ++s) {                          /* pass 2, :65-98 */
        const uint32_t lo = s * 8;
        const uint32_t width = (uint64_t)lo + 8 < n ? 8 : n - lo;
        uint64_t cur[8];
        for (uint32_t j = 0; j < width; ++j) cur[j] = off[lo + j];
        uint64_t k = 0;
        for (;;) { /* merge the <=8 sorted out-lists by ascending row (:75-88) */
            uint32_t next = n;
            for (uint32_t j = 0; j < width; ++j)
                if (cur[j] < off[lo + j + 1] && tgt[cur[j]] < next) next = tgt[cur[j]];
            if (next == n) break;
            uint32_t mask = 0;
            for (uint32_t j = 0; j < width; ++j)
                if (cur[j] < off[lo + j + 1] && tgt[cur[j]] == next) { mask |= 1u << j; ++cur[j]; }
            const uint64_t v = real_ptrs[s] + k / 128; /* :89-97, 64-bit slot math */
            const uint32_t slot = (uint32_t)(k % 128), lane = slot % 32, column = slot / 32;
            masks[32 * v + lane] |= mask << (8 * column);
            row_ids[4 * (32 * v + lane) + column] = next;
            ++k;
        }
    }
}

double orc_compression_ratio(uint64_t m, uint64_t num_unpadded) { /* :103-107 */
    if (num_unpadded == 0) return 0.0;
    return (double)m / ((double)num_unpadded * 8);
}

double orc_update_divergence(uint32_t n, uint64_t num_vss, const uint32_t* row_ids) { /* :109-141 */
    double sum = 0;
    uint64_t counted = 0;
    for (uint64_t v = 0; v < num_vss; ++v) {
        double col_sum = 0;
        unsigned nonempty = 0;
        for (unsigned c = 0; c < 4; ++c) {
            double mean = 0;
            unsigned count = 0;
            for (unsigned lane = 0; lane < 32; ++lane) {
                const uint32_t r = row_ids[4 * (32 * v + lane) + c];
                if (r != n) { mean += r; ++count; }
            }
            if (count == 0) continue;
            mean /= count;
            double var = 0;
            for (unsigned lane = 0; lane < 32; ++lane) {
                const uint32_t r = row_ids[4 * (32 * v + lane) + c];
                if (r != n) var += (r - mean) * (r - mean);
            }
            col_sum += sqrt(var / count);
            ++nonempty;
        }
        if (nonempty) { sum += col_sum / nonempty; ++counted; }
    }
    return counted ? sum / (double)counted : 0.0;
}

/* ---------------------------------------------------------------------------------
 * Tile (R:src/tc_emu.cpp): FragA word (i,q) = lane 4i+q's 16-bit round field
 * (pack_fragA_round :31-38); FragB word (r,2r) = alpha, (r,2r+1) = alpha<<8
 * (build_fragB :22-29); C[i][j] = sum_q popc(A(i,q) & B(q,j)) (mma_m8n8k128 :9-20).
 * --------------------------------------------------------------------------------- */
void orc_tile_pull(const uint32_t* mask_words, uint8_t alpha, unsigned round, uint32_t* c64) {
    uint32_t A[32], B[32];
    const unsigned sh = round ? 16 : 0;
    for (unsigned lane = 0; lane < 32; ++lane) A[lane] = (mask_words[lane] >> sh) & 0xFFFFu;
    memset(B, 0, sizeof B);
    for (unsigned r = 0; r < 4; ++r) {
        B[8 * r + 2 * r] = alpha;
        B[8 * r + 2 * r + 1] = (uint32_t)alpha << 8;
    }
    for (unsigned i = 0; i < 8; ++i)
        for (unsigned j = 0; j < 8; ++j) {
            uint32_t acc = 0;
            for (unsigned q = 0; q < 4; ++q) acc += __builtin_popcount(A[4 * i + q] & B[8 * q + j]);
            c64[8 * i + j] = acc;
        }
}

/* ---------------------------------------------------------------------------------
 * Engines (R:src/bfs_engine.cpp), single worker. Per dequeued VSS the lane's two
 * popcounts per round are popc(mask_byte & alpha) (lane_dot_products :40-45, the
 * per-lane locality of the tile; pinned against orc_tile_pull in the tests).
 * --------------------------------------------------------------------------------- */
typedef struct {
    uint32_t* items;
    uint64_t len, cap;
} Queue;

static void q_push_range(Queue* q, uint32_t b, uint32_t e) {
    if (q->len + (e - b) > q->cap) {
        q->cap = (q->len + (e - b)) * 2 + 16;
        q->items = (uint32_t*)realloc(q->items, sizeof(uint32_t) * q->cap);
    }
    for (uint32_t x = b; x < e; ++x) q->items[q->len++] = x;
}

static inline uint8_t frontier_byte(const uint32_t* f, uint32_t ss) { /* :148-151 */
    return (uint8_t)(f[ss / 4] >> (8 * (ss % 4)));
}

int64_t orc_run_engine(uint32_t n, const uint32_t* real_ptrs, uint64_t num_vss, const uint32_t* v2r,
                       const uint32_t* row_ids, const uint32_t* masks, uint32_t src, int lazy,
                       uint32_t num_warps, uint32_t max_levels, uint32_t* L,
                       uint64_t* trace, uint64_t trace_cap) {
    (void)num_vss;
    if (src >= n || num_warps < 1) return -4;
    const uint64_t words = ((uint64_t)n + 31) / 32;
    const uint32_t cap = max_levels ? max_levels : n + 1; /* level_cap :68-70 */
    uint32_t* f_curr = (uint32_t*)calloc(words ? words : 1, 4);
    uint32_t* f_next = (uint32_t*)calloc(words ? words : 1, 4);
    uint32_t* v_curr = (uint32_t*)calloc(words ? words : 1, 4);
    uint32_t* v_next = (uint32_t*)calloc(words ? words : 1, 4);
    uint32_t* stamp = (uint32_t*)calloc(words ? words : 1, 4);
    /* init_state :30-49 */
    for (uint32_t v = 0; v < n; ++v) L[v] = INF32;
    L[src] = 0;
    f_curr[src / 32] |= 1u << (src % 32);
    v_curr[src / 32] |= 1u << (src % 32);
    v_next[src / 32] |= 1u << (src % 32);
    Queue qc = {0, 0, 0}, qn = {0, 0, 0};
    q_push_range(&qc, real_ptrs[src / 8], real_ptrs[src / 8 + 1]);

    int64_t status = 0;
    uint32_t level = 0;
    const uint64_t threads = (uint64_t)num_warps * 32;
    while (qc.len) {
        if (++level > cap) { status = -1; break; } /* runaway :72-75 */
        if ((uint64_t)level > trace_cap) { status = -2; break; }
        uint64_t* row = trace + 8 * (uint64_t)(level - 1);
        memset(row, 0, 8 * sizeof(uint64_t));
        row[0] = level;
        row[1] = qc.len;
        uint64_t pop = 0;
        for (uint64_t i = 0; i < words; ++i)
            if (!lazy || stamp[i] == level - 1) pop += __builtin_popcount(f_curr[i]);
        row[2] = pop;
        qn.len = 0;
        for (uint64_t p = 0; p < qc.len; ++p) {
            const uint32_t vss = qc.items[p];
            const uint32_t ss = v2r[vss];
            if (lazy && stamp[ss / 4] != level - 1) { status = -3; goto done; } /* :279-280 */
            const uint8_t alpha = frontier_byte(f_curr, ss);
            if (alpha == 0) { status = -3; goto done; } /* :194-195, :283-284 */
            for (unsigned round = 0; round < 2; ++round) /* pull_vss :131-146 */
                for (unsigned lane = 0; lane < 32; ++lane) {
                    const uint32_t m = masks[32 * (uint64_t)vss + lane];
                    for (unsigned h = 0; h < 2; ++h) {
                        const unsigned col = 2 * round + h;
                        if (!__builtin_popcount((m >> (8 * col)) & alpha)) continue;
                        const uint32_t u = row_ids[4 * (32 * (uint64_t)vss + lane) + col];
                        if (lazy) { /* stage-1 sink :286-289 */
                            v_next[u / 32] |= 1u << (u % 32);
                            ++row[6];
                            continue;
                        }
                        if (level >= L[u]) continue; /* eager sink :198-211 */
                        L[u] = level;
                        const uint32_t old = f_next[u / 32];
                        f_next[u / 32] |= 1u << (u % 32);
                        ++row[4];
                        if (((old >> (8 * ((u / 8) % 4))) & 0xFFu) == 0) {
                            ++row[4];
                            q_push_range(&qn, real_ptrs[u / 8], real_ptrs[u / 8 + 1]);
                            row[7] += real_ptrs[u / 8 + 1] - real_ptrs[u / 8];
                        }
                    }
                }
        }
        if (!lazy) {
            row[5] = row[4];
            uint64_t disc = 0;
            for (uint64_t i = 0; i < words; ++i) disc += __builtin_popcount(f_next[i]);
            row[3] = disc;
            uint32_t* t = f_curr; f_curr = f_next; f_next = t; /* :226-229 */
            memset(f_next, 0, words * 4);
        } else { /* stage 2 :296-338, thread t owns words t, t+threads, ... */
            for (uint32_t w = 0; w < num_warps; ++w)
                for (uint64_t base = 32 * (uint64_t)w; base < words; base += threads) {
                    const uint64_t end = base + 32 < words ? base + 32 : words;
                    uint64_t pending = 0;
                    for (uint64_t idx = base; idx < end; ++idx) {
                        const uint32_t diff = v_curr[idx] ^ v_next[idx];
                        if (!diff) continue;
                        v_curr[idx] = v_next[idx];
                        f_curr[idx] = diff;
                        stamp[idx] = level;
                        row[3] += __builtin_popcount(diff);
                        for (unsigned set = 0; set < 4; ++set) {
                            uint32_t field = (diff >> (8 * set)) & 0xFFu;
                            if (!field) continue;
                            while (field) {
                                const unsigned bit = __builtin_ctz(field);
                                field &= field - 1;
                                L[32 * idx + 8 * set + bit] = level;
                            }
                            const uint64_t ss = 4 * idx + set;
                            q_push_range(&qn, real_ptrs[ss], real_ptrs[ss + 1]);
                            pending += real_ptrs[ss + 1] - real_ptrs[ss];
                        }
                    }
                    if (pending) { ++row[4]; row[7] += pending; }
                }
        }
        Queue t = qc; qc = qn; qn = t;
    }
done:
    free(f_curr); free(f_next); free(v_curr); free(v_next); free(stamp);
    free(qc.items); free(qn.items);
    return status < 0 ? status : (int64_t)level;
}
