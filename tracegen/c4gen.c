/*
 * c4gen.c — C4 workload (BASELINE.json configs[3]): "global-memory graph
 * BFS/histogram on a 2^24-vertex power-law graph, cross-block atomics and
 * contended hot addresses".  INPUT ONLY: builds the graph and lays out the
 * recorded access streams of the traced kernels; no race-check arithmetic.
 *
 * Graph: RMAT (a, b, c, d) = (.57, .19, .19, .05) (Graph500-style), 2^lv
 * vertices, avg out-degree `deg`, counter-based splitmix64 draws (16-bit
 * fixed-point quadrant choice per level).  Vertices are relabelled by
 * descending out-degree (ties by id) so that each warp's 32 threads carry
 * similar degrees (thread v handles vertex v).  CSR keeps edge order.
 *
 * Traced kernels (one per BFS level L from source 0, then one histogram):
 *   level L, thread v:  access level[v]                  (R racy / A race-free)
 *     if level(v) == L: for each out-neighbour x, in CSR order:
 *        racy:      R level[x]; W level[x] if x is first reached at L+1
 *        race-free: A level[x]                            (atomicMin)
 *   histogram, thread v: bin = min(outdeg(v), 1023)
 *        racy: R hist[bin], W hist[bin];  race-free: A hist[bin]
 * level[] = words [0, 2^lv), hist[] = words [2^lv, 2^lv + 1024).
 * Rows per warp = 1 + K * (max out-degree over the warp's frontier lanes),
 * K = 2 racy / 1 race-free; lanes with fewer neighbours get NOPs.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NOPR (3ull << 62)
#define REC(op, w) (((uint64_t)(op) << 62) | (uint64_t)(w))

static inline uint64_t mix(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

typedef struct {
    uint32_t lv, n;
    uint64_t m;
    uint64_t *rp;      /* n + 1 */
    uint32_t *col;     /* m */
    int32_t *level;    /* n, -1 = unreached */
    uint32_t n_levels; /* BFS kernels = levels with a non-empty frontier */
} c4_graph;


void *c4_build(uint64_t seed, uint32_t lv, uint32_t deg)
{
    c4_graph *g = (c4_graph *)calloc(1, sizeof *g);
    g->lv = lv;
    g->n = 1u << lv;
    g->m = (uint64_t)g->n * deg;
    uint32_t n = g->n;
    uint64_t m = g->m;
    uint32_t *src = (uint32_t *)malloc(m * 4), *dst = (uint32_t *)malloc(m * 4);
    /* RMAT thresholds in 1/65536: a = .57, a+b = .76, a+b+c = .95 */
    const uint32_t ta = 37355, tab = 49807, tabc = 62259;
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < m; e++) {
        uint32_t u = 0, v = 0;
        uint64_t h = 0;
        for (uint32_t i = 0; i < lv; i++) {
            if ((i & 3) == 0) h = mix(seed * 0xD1B54A32D192ED03ull + e * 8 + (i >> 2));
            uint32_t r = (uint32_t)(h & 0xffff);
            h >>= 16;
            uint32_t q = r < ta ? 0 : r < tab ? 1 : r < tabc ? 2 : 3;
            u = (u << 1) | (q >> 1);
            v = (v << 1) | (q & 1);
        }
        src[e] = u;
        dst[e] = v;
    }
    /* relabel by descending out-degree (counting sort, stable by id) */
    uint32_t *odeg = (uint32_t *)calloc(n, 4);
    uint32_t maxd = 0;
    for (uint64_t e = 0; e < m; e++) odeg[src[e]]++;
    for (uint32_t v = 0; v < n; v++) if (odeg[v] > maxd) maxd = odeg[v];
    uint64_t *bucket = (uint64_t *)calloc((size_t)maxd + 2, 8);
    for (uint32_t v = 0; v < n; v++) bucket[maxd - odeg[v]]++;
    uint64_t acc = 0;
    for (uint32_t d = 0; d <= maxd + 1; d++) { uint64_t t = bucket[d]; bucket[d] = acc; acc += t; }
    uint32_t *newid = (uint32_t *)malloc((size_t)n * 4);
    for (uint32_t v = 0; v < n; v++) newid[v] = (uint32_t)(bucket[maxd - odeg[v]]++);
    free(bucket);
    /* CSR over new ids, edges in generation order */
    g->rp = (uint64_t *)calloc((size_t)n + 1, 8);
    for (uint32_t v = 0; v < n; v++) g->rp[newid[v] + 1] = odeg[v];
    for (uint32_t v = 0; v < n; v++) g->rp[v + 1] += g->rp[v];
    uint64_t *fill = (uint64_t *)malloc((size_t)n * 8);
    memcpy(fill, g->rp, (size_t)n * 8);
    g->col = (uint32_t *)malloc(m * 4);
    for (uint64_t e = 0; e < m; e++) {
        uint32_t u = newid[src[e]];
        g->col[fill[u]++] = newid[dst[e]];
    }
    free(fill); free(src); free(dst); free(odeg); free(newid);
    /* BFS from vertex 0 */
    g->level = (int32_t *)malloc((size_t)n * 4);
    for (uint32_t v = 0; v < n; v++) g->level[v] = -1;
    uint32_t *q = (uint32_t *)malloc((size_t)n * 4);
    uint64_t qh = 0, qt = 0;
    g->level[0] = 0;
    q[qt++] = 0;
    int32_t maxl = 0;
    while (qh < qt) {
        uint32_t u = q[qh++];
        for (uint64_t k = g->rp[u]; k < g->rp[u + 1]; k++) {
            uint32_t x = g->col[k];
            if (g->level[x] < 0) { g->level[x] = g->level[u] + 1; if (g->level[x] > maxl) maxl = g->level[x]; q[qt++] = x; }
        }
    }
    free(q);
    g->n_levels = (uint32_t)maxl + 1;
    return g;
}

void c4_free(void *h)
{
    c4_graph *g = (c4_graph *)h;
    free(g->rp); free(g->col); free(g->level); free(g);
}

void c4_stats(void *h, uint64_t *out /* n, m, n_levels, reached, maxdeg */)
{
    c4_graph *g = (c4_graph *)h;
    uint64_t reached = 0, maxd = 0;
    for (uint32_t v = 0; v < g->n; v++) {
        if (g->level[v] >= 0) reached++;
        uint64_t d = g->rp[v + 1] - g->rp[v];
        if (d > maxd) maxd = d;
    }
    out[0] = g->n; out[1] = g->m; out[2] = g->n_levels; out[3] = reached; out[4] = maxd;
}

static uint64_t warp_rows(c4_graph *g, uint32_t kern, uint64_t w, int racy)
{
    if (kern == g->n_levels) return racy ? 2 : 1;                     /* histogram */
    uint64_t md = 0;
    for (uint32_t l = 0; l < 32; l++) {
        uint32_t v = (uint32_t)(w * 32 + l);
        if (g->level[v] == (int32_t)kern) {
            uint64_t d = g->rp[v + 1] - g->rp[v];
            if (d > md) md = d;
        }
    }
    return 1 + (racy ? 2 : 1) * md;
}

/* sizes: kernels = n_levels + 1; warp offsets = kernels * (n/32 + 1) */
void c4_sizes(void *h, int racy, uint64_t *n_rows, uint32_t *n_kernels, uint64_t *n_woff)
{
    c4_graph *g = (c4_graph *)h;
    uint64_t nw = g->n / 32, rows = 0;
    for (uint32_t k = 0; k <= g->n_levels; k++)
        for (uint64_t w = 0; w < nw; w++) rows += warp_rows(g, k, w, racy);
    *n_rows = rows;
    *n_kernels = g->n_levels + 1;
    *n_woff = (uint64_t)(g->n_levels + 1) * (nw + 1);
}

void c4_fill(void *h, int racy, uint64_t *rec, uint64_t *kdesc, uint64_t *woff)
{
    c4_graph *g = (c4_graph *)h;
    const uint64_t nw = g->n / 32, hist = g->n;
    uint64_t row = 0, wo = 0;
    for (uint32_t k = 0; k <= g->n_levels; k++) {
        uint64_t *kd = kdesc + 8 * k;
        memset(kd, 0, 64);
        kd[0] = g->n / 256; kd[1] = 8; kd[2] = 32; kd[3] = 0; kd[4] = wo; kd[5] = kd[6] = kd[7] = 0;
        for (uint64_t w = 0; w < nw; w++) {
            woff[wo++] = row;
            uint64_t nr = warp_rows(g, k, w, racy);
            uint64_t *r = rec + row * 32;
            for (uint64_t i = 0; i < nr * 32; i++) r[i] = NOPR;
            for (uint32_t l = 0; l < 32; l++) {
                uint32_t v = (uint32_t)(w * 32 + l);
                uint64_t d = g->rp[v + 1] - g->rp[v];
                if (k == g->n_levels) {                                   /* histogram */
                    uint64_t bin = hist + (d < 1023 ? d : 1023);
                    if (racy) { r[l] = REC(0, bin); r[32 + l] = REC(1, bin); }
                    else r[l] = REC(2, bin);
                    continue;
                }
                r[l] = REC(racy ? 0 : 2, v);
                if (g->level[v] != (int32_t)k) continue;
                for (uint64_t j = 0; j < d; j++) {
                    uint32_t x = g->col[g->rp[v] + j];
                    if (racy) {
                        r[(1 + 2 * j) * 32 + l] = REC(0, x);
                        if (g->level[x] == (int32_t)k + 1) r[(2 + 2 * j) * 32 + l] = REC(1, x);
                    } else {
                        r[(1 + j) * 32 + l] = REC(2, x);
                    }
                }
            }
            row += nr;
        }
        woff[wo++] = row;
    }
}

/* CSR and final BFS levels, for the online-instrumented kernels */
void c4_export(void *h, uint64_t *rp, uint32_t *col, int32_t *level)
{
    c4_graph *g = (c4_graph *)h;
    if (rp) memcpy(rp, g->rp, ((size_t)g->n + 1) * 8);
    if (col) memcpy(col, g->col, g->m * 4);
    if (level) memcpy(level, g->level, (size_t)g->n * 4);
}
