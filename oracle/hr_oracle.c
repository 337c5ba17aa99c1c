/*
 * hr_oracle.c — plain, slow, single-threaded CPU oracle for the racy-address
 * set of an access trace.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code with the CUDA path (paper_2401_04701_b200/): it decodes the trace
 * records itself and never looks at an FSM.
 *
 * What it computes (the plain definition, §II-A "Data Races"):
 *   "A parallel program has a data race if multiple threads access the same
 *    memory location, at least one of the accesses is a write, and the
 *    accesses are concurrent (more precisely, are not ordered by some
 *    happens-before relation)."
 * with the happens-before relation of CUDA barriers (PAPER.md:261-264,
 * §II-B: __syncthreads orders a block, __syncwarp orders a warp) and kernel
 * boundaries.  Atomics are "a third class of memory action"
 * (PAPER.md:565); reading R1 in DESIGN.md: atomic–atomic pairs do not
 * conflict, atomic–read and atomic–write pairs do, atomics create no
 * happens-before edges.
 *
 * Per access a we derive (SPEC.md:69-77 materialize_threads):
 *   kernel, space, address block (shared memory: one instance per block),
 *   word, thread (block, warp, lane), bc = #__syncthreads before a in its
 *   thread, wc = #__syncwarp before a in its thread, kind.
 * Two accesses a, b of distinct threads in the same kernel are UNORDERED iff
 *   block(a) != block(b), or
 *   block equal ∧ bc equal ∧ (warp differs ∨ wc equal)
 * (SPEC.md:410 static_hb_races: ordered by block-epoch order — same block,
 *  different bc — or by warp-epoch order — same warp, different wc).
 * A RACE PAIR is: same address ∧ distinct threads ∧ conflict ∧ unordered.
 * Output 1: the sorted set of racy addresses (kernel, space, block, word).
 * Output 2: scope per racy address — GRID if some race pair has its two
 *   threads in different blocks, BLOCK otherwise (reading R4 in DESIGN.md).
 * Output 3: race classes per racy address — the set of kind pairs among its
 *   race pairs: bit0 W–W, bit1 R–W, bit2 A–W, bit3 A–R.
 *
 * Two modes:
 *   HRO_PAIRWISE  — the literal O(n^2) loop over pairs of each address.
 *   HRO_BUCKETED  — the same predicate evaluated per group of the sort key
 *                   (block, bc, warp, wc, lane) with kind-set counts; needed
 *                   for hub addresses with 10^5..10^6 accesses.
 *   tests/test_oracle_pins.py checks both modes equal on random traces.
 *
 * Control records (readings R8 and R12 in DESIGN.md): 1 = __syncthreads, 2 =
 * __syncwarp; a __syncwarp only some active lanes of a warp row hold is a
 * sub-warp __syncwarp(mask) and any other code is undefined —
 * both flag a model violation and order nothing (no clock moves).
 *
 * Clock overflow (PAPER.md:540 footnote: "race detection is discontinued with
 * a warning if a clock overflows (after reporting any previously identified
 * races)"): reading R6 — a thread whose bc (wc) would exceed bc_max (wc_max)
 * latches HRO_F_CLOCK_OVERFLOW and its later accesses are not checked.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HRO_PAIRWISE 0
#define HRO_BUCKETED 1

#define HRO_F_CLOCK_OVERFLOW 1u
#define HRO_F_MODEL_VIOLATION 4u
#define HRO_F_BARRIER_DIVERGENCE 8u

#define K_READ 0
#define K_WRITE 1
#define K_ATOMIC 2

#define GLOBAL_BLOCK 0xFFFFFFFFu

typedef struct {
    uint64_t word;
    uint32_t kernel;
    uint32_t ablock;   /* address instance: simulated block for shared, GLOBAL_BLOCK for global */
    uint32_t tblock;   /* accessing thread: block, warp, lane */
    uint32_t bc;       /* __syncthreads crossed by the thread before this access */
    uint32_t wc;       /* __syncwarp crossed by the thread before this access */
    uint16_t twarp;
    uint8_t tlane;
    uint8_t space;
    uint8_t kind;
    uint8_t pad[3];
} acc_t;

typedef struct {
    uint64_t word;
    uint32_t kernel;
    uint32_t block;
    uint8_t space;
    uint8_t scope;   /* 1 = BLOCK, 2 = GRID */
    uint8_t classes; /* bit0 WW, bit1 RW, bit2 AW, bit3 AR */
    uint8_t pad[5];
} hro_race;

static unsigned pair_class(int k1, int k2)
{
    if (k1 == K_WRITE && k2 == K_WRITE) return 1u;
    if ((k1 == K_READ && k2 == K_WRITE) || (k1 == K_WRITE && k2 == K_READ)) return 2u;
    if ((k1 == K_ATOMIC && k2 == K_WRITE) || (k1 == K_WRITE && k2 == K_ATOMIC)) return 4u;
    if ((k1 == K_ATOMIC && k2 == K_READ) || (k1 == K_READ && k2 == K_ATOMIC)) return 8u;
    return 0u;   /* R-R, A-A: not a conflict */
}

/* ---- step 1: materialise per-access (thread, bc, wc) from the records ---- */

static int materialize(const uint64_t *rec, const uint64_t *kdesc, uint64_t n_kernels,
                       const uint64_t *warp_off, uint32_t bc_max, uint32_t wc_max,
                       acc_t **out, uint64_t *n_out, uint32_t *flags)
{
    uint64_t cap = 1024, n = 0;
    acc_t *a = (acc_t *)malloc(cap * sizeof(acc_t));
    if (!a) return -2;
    for (uint64_t k = 0; k < n_kernels; k++) {
        const uint64_t *kd = kdesc + 8 * k;
        uint64_t blocks = kd[0], warps = kd[1], lanes = kd[2], woi = kd[4];
        /* kdesc[5]: the kernel's warp tile, log2 of its lanes (0 = whole warps).  With
         * tiles of T lanes, an aligned __syncwarp(tile mask) orders exactly the tile's
         * lanes (reading R8 in DESIGN.md), so a tile plays the role of a
         * warp: threads are (block, tile = warp*32/T + lane/T, lane%T) below */
        const uint64_t tl = kd[5];
        if (lanes < 1 || lanes > 32 || tl > 4) { free(a); return -1; }
        const uint64_t T = tl ? (1ull << tl) : 32;
        for (uint64_t b = 0; b < blocks; b++) {
            int64_t block_sync_count = -1;
            for (uint64_t w = 0; w < warps; w++) {
                uint64_t gw = b * warps + w;
                uint64_t r0 = warp_off[woi + gw], r1 = warp_off[woi + gw + 1];
                uint32_t bc[32], wc[32];
                int dead[32];
                memset(bc, 0, sizeof bc); memset(wc, 0, sizeof wc); memset(dead, 0, sizeof dead);
                for (uint64_t r = r0; r < r1; r++) {
                    const uint64_t *row = rec + r * 32;
                    /* barrier uniformity within the warp */
                    int nbar = 0, same = 1;
                    uint64_t first_bar = 0;
                    for (uint64_t l = 0; l < lanes; l++) {
                        uint64_t x = row[l];
                        if ((x >> 62) == 3 && (x & ((1ull << 61) - 1)) != 0) {
                            if (nbar == 0) first_bar = x; else if (x != first_bar) same = 0;
                            nbar++;
                        }
                    }
                    /* a __syncwarp that only some active lanes hold is __syncwarp(mask) with a
                     * sub-warp mask ("takes a mask argument"): reading R8 —
                     * model violation, and conservatively NO happens-before edge (no clock
                     * moves), so every race the masked barrier would hide is still reported */
                    int partial_ws = nbar != 0 && nbar != (int)lanes && same &&
                                     (first_bar & ((1ull << 61) - 1)) == 2;
                    /* tile kernels: a __syncwarp held by whole tiles (every active lane of
                     * each tile it touches) is one tile barrier per such tile: exact */
                    int tile_ws = 0;
                    if (partial_ws && tl) {
                        tile_ws = 1;
                        for (uint64_t t0 = 0; t0 < lanes; t0 += T) {
                            int held = 0, n_in = 0;
                            for (uint64_t l = t0; l < t0 + T && l < lanes; l++) {
                                n_in++;
                                held += (row[l] & ~(1ull << 61)) == ((3ull << 62) | 2);
                            }
                            if (held != 0 && held != n_in) tile_ws = 0;
                        }
                        if (tile_ws) partial_ws = 0;
                    }
                    if (partial_ws) *flags |= HRO_F_MODEL_VIOLATION;
                    else if (!tile_ws && nbar != 0 && (nbar != (int)lanes || !same))
                        *flags |= HRO_F_BARRIER_DIVERGENCE;
                    for (uint64_t l = 0; l < lanes; l++) {
                        uint64_t x = row[l];
                        uint32_t op = (uint32_t)(x >> 62);
                        uint32_t space = (uint32_t)((x >> 61) & 1);
                        uint64_t word = x & ((1ull << 61) - 1);
                        if (op == 3) {
                            if (partial_ws) continue;   /* sub-warp __syncwarp: no edge (above) */
                            (void)tile_ws;              /* tile barrier: advances its lanes' wc below */
                            if (word == 1) {            /* __syncthreads: bc + 1 */
                                if (bc[l] + 1 > bc_max) { dead[l] = 1; *flags |= HRO_F_CLOCK_OVERFLOW; }
                                else bc[l]++;
                            } else if (word == 2) {     /* __syncwarp: wc + 1 */
                                if (wc[l] + 1 > wc_max) { dead[l] = 1; *flags |= HRO_F_CLOCK_OVERFLOW; }
                                else wc[l]++;
                            } else if (word != 0) {
                                *flags |= HRO_F_MODEL_VIOLATION;
                            }
                            continue;
                        }
                        if (dead[l]) continue;
                        if (n == cap) {
                            cap *= 2;
                            acc_t *t = (acc_t *)realloc(a, cap * sizeof(acc_t));
                            if (!t) { free(a); return -2; }
                            a = t;
                        }
                        acc_t *e = &a[n++];
                        memset(e, 0, sizeof *e);
                        e->word = word;
                        e->kernel = (uint32_t)k;
                        e->space = (uint8_t)space;
                        e->ablock = space ? (uint32_t)b : GLOBAL_BLOCK;
                        e->tblock = (uint32_t)b;
                        e->twarp = (uint16_t)(w * (32 / T) + l / T);   /* the tile (= the warp without tiles) */
                        e->tlane = (uint8_t)(l % T);
                        e->bc = bc[l];
                        e->wc = wc[l];
                        e->kind = (uint8_t)op;
                    }
                }
                /* every thread of a block crosses the same number of __syncthreads */
                for (uint64_t l = 0; l < lanes; l++) {
                    if (dead[l]) continue;
                    if (block_sync_count < 0) block_sync_count = bc[l];
                    else if ((int64_t)bc[l] != block_sync_count) *flags |= HRO_F_BARRIER_DIVERGENCE;
                }
            }
        }
    }
    *out = a;
    *n_out = n;
    return 0;
}

/* ---- the race predicate, written out ---- */

static int conflict(int k1, int k2)
{
    /* at least one write; atomics conflict with plain accesses but not with
     * each other (reading R1) */
    if (k1 == K_READ && k2 == K_READ) return 0;
    if (k1 == K_ATOMIC && k2 == K_ATOMIC) return 0;
    return 1;
}

static int same_thread(const acc_t *a, const acc_t *b)
{
    return a->tblock == b->tblock && a->twarp == b->twarp && a->tlane == b->tlane;
}

static int unordered(const acc_t *a, const acc_t *b)
{
    if (a->tblock != b->tblock) return 1;      /* no inter-block barrier */
    if (a->bc != b->bc) return 0;              /* a __syncthreads separates them */
    if (a->twarp != b->twarp) return 1;        /* same block epoch, different warps */
    return a->wc == b->wc;                     /* same warp: ordered iff a __syncwarp separates */
}

static int cmp_addr(const void *x, const void *y)
{
    const acc_t *a = (const acc_t *)x, *b = (const acc_t *)y;
#define C(f) if (a->f != b->f) return a->f < b->f ? -1 : 1;
    C(kernel) C(space) C(ablock) C(word)
    C(tblock) C(bc) C(twarp) C(wc) C(tlane)
#undef C
    return 0;
}

static int same_addr(const acc_t *a, const acc_t *b)
{
    return a->kernel == b->kernel && a->space == b->space && a->ablock == b->ablock && a->word == b->word;
}

/* pairwise: returns 0 (race-free), 1 (BLOCK), 2 (GRID) for one address group;
 * *classes receives the kind pairs of all race pairs */
static int group_pairwise(const acc_t *g, uint64_t n, unsigned *classes)
{
    int scope = 0;
    *classes = 0;
    for (uint64_t i = 0; i < n; i++)
        for (uint64_t j = i + 1; j < n; j++) {
            const acc_t *a = &g[i], *b = &g[j];
            if (same_thread(a, b)) continue;
            if (!conflict(a->kind, b->kind)) continue;
            if (!unordered(a, b)) continue;
            *classes |= pair_class(a->kind, b->kind);
            scope = (a->tblock != b->tblock) ? 2 : (scope ? scope : 1);
        }
    return scope;
}

/* Kind-set test over distinct sub-groups (distinct sub-groups of one level
 * are pairwise unordered; inside a sub-group the next level decides). For
 * kinds x != y the number of ordered (x in group i, y in group j, i != j)
 * choices is n_x * n_y - n_xy; for W-W, at least two groups with a write. */
static unsigned kc_classes(uint64_t nW, uint64_t nR, uint64_t nA, uint64_t nRW, uint64_t nAW, uint64_t nRA)
{
    unsigned m = 0;
    if (nW >= 2) m |= 1u;
    if (nR * nW - nRW > 0) m |= 2u;
    if (nA * nW - nAW > 0) m |= 4u;
    if (nA * nR - nRA > 0) m |= 8u;
    return m;
}

/* per-sub-group kind-mask accumulator for the class test */
typedef struct { uint64_t n, nW, nR, nA, nRW, nAW, nRA; } kc2;

static void kc2_add(kc2 *c, unsigned m)
{
    const int r = (m >> K_READ) & 1, w = (m >> K_WRITE) & 1, a = (m >> K_ATOMIC) & 1;
    c->n++;
    c->nW += w; c->nR += r; c->nA += a;
    c->nRW += r && w; c->nAW += a && w; c->nRA += r && a;
}

static unsigned kc2_classes(const kc2 *c)
{
    return kc_classes(c->nW, c->nR, c->nA, c->nRW, c->nAW, c->nRA);
}

/* bucketed: same predicate; g is sorted by (tblock, bc, twarp, wc, tlane).
 * Returns the scope; *classes receives the classes of all race pairs. */
static int group_bucketed(const acc_t *g, uint64_t n, unsigned *classes)
{
    /* cross-block pairs are always unordered */
    kc2 blocks = {0};
    unsigned cls = 0;
    uint64_t i = 0;
    while (i < n) {
        uint64_t jb = i;
        unsigned mb = 0;
        while (jb < n && g[jb].tblock == g[i].tblock) { mb |= 1u << g[jb].kind; jb++; }
        kc2_add(&blocks, mb);
        /* inside block: pairs with equal bc, different warps are unordered */
        uint64_t e = i;
        while (e < jb) {
            uint64_t je = e;
            while (je < jb && g[je].bc == g[e].bc) je++;
            kc2 warps = {0};
            uint64_t w = e;
            while (w < je) {
                uint64_t jw = w;
                unsigned mw = 0;
                while (jw < je && g[jw].twarp == g[w].twarp) { mw |= 1u << g[jw].kind; jw++; }
                kc2_add(&warps, mw);
                /* inside warp: equal wc, different lanes are unordered */
                uint64_t c = w;
                while (c < jw) {
                    uint64_t jc = c;
                    while (jc < jw && g[jc].wc == g[c].wc) jc++;
                    kc2 lanes = {0};
                    uint64_t t = c;
                    while (t < jc) {
                        uint64_t jt = t;
                        unsigned mt = 0;
                        while (jt < jc && g[jt].tlane == g[t].tlane) { mt |= 1u << g[jt].kind; jt++; }
                        kc2_add(&lanes, mt);
                        t = jt;
                    }
                    cls |= kc2_classes(&lanes);
                    c = jc;
                }
                w = jw;
            }
            cls |= kc2_classes(&warps);
            e = je;
        }
        i = jb;
    }
    const unsigned cross = kc2_classes(&blocks);
    *classes = cls | cross;
    if (cross) return 2;
    return cls ? 1 : 0;
}

/* Entry point.  Returns 0 on success, -1 bad trace, -2 out of memory,
 * -3 output capacity too small (n_out then holds the needed count). */
int hro_check(const uint64_t *rec, const uint64_t *kdesc, uint64_t n_kernels,
              const uint64_t *warp_off, int mode, uint32_t bc_max, uint32_t wc_max,
              hro_race *out, uint64_t cap, uint64_t *n_out, uint32_t *flags_out,
              uint64_t *n_accesses_out)
{
    acc_t *a = NULL;
    uint64_t n = 0;
    uint32_t flags = 0;
    int rc = materialize(rec, kdesc, n_kernels, warp_off, bc_max, wc_max, &a, &n, &flags);
    if (rc) return rc;
    if (n_accesses_out) *n_accesses_out = n;
    qsort(a, n, sizeof(acc_t), cmp_addr);   /* library sort: groups each address */
    uint64_t nr = 0;
    uint64_t i = 0;
    while (i < n) {
        uint64_t j = i + 1;
        while (j < n && same_addr(&a[i], &a[j])) j++;
        unsigned cls = 0;
        int s = mode == HRO_PAIRWISE ? group_pairwise(a + i, j - i, &cls) : group_bucketed(a + i, j - i, &cls);
        if (s) {
            if (nr < cap) {
                hro_race *r = &out[nr];
                memset(r, 0, sizeof *r);
                r->word = a[i].word;
                r->kernel = a[i].kernel;
                r->block = a[i].ablock;
                r->space = a[i].space;
                r->scope = (uint8_t)s;
                r->classes = (uint8_t)cls;
            }
            nr++;
        }
        i = j;
    }
    free(a);
    *n_out = nr;
    *flags_out = flags;
    return nr > cap ? -3 : 0;
}

uint64_t hro_sizeof_race(void) { return sizeof(hro_race); }
