/*
 * c5gen.h — counter-based generator of the C5 workload (BASELINE.json
 * configs[4]: "2^32-access global trace over 16 GB address space,
 * address-sharded across 1/2/4/8 B200"), INPUT ONLY: no race-check
 * arithmetic.  Compiled twice from this one header: by gcc into the CPU
 * generator (c5gen.c, used by tests and the oracle's sampled check) and by
 * nvcc into the GPU generator (c5gen.cu, used by bench.py to build the
 * 32 GiB trace in HBM).  Both produce bit-identical rows.
 *
 * Shape, with B = 2^lb blocks of 256 threads (8 warps x 32
 * lanes), 256 accesses per thread, a __syncthreads after every 32 accesses:
 *   owned  [0, B*2^15):       block b owns words b*2^15 + 256*row + ltid
 *                             (thread-private; a warp's 32 lanes on one row
 *                             hit 32 consecutive words)
 *   read-only [B*2^15, T-H):  uniform random reads (T = B*2^16 words)
 *   hot  [T-H, T), H = B*16:  atomics, log-uniform rank ~ Zipf(1)
 * Per (warp, access j) one category drawn for the whole warp: 50% own-row
 * (each lane R 60% / W 40%), 40% random read gather, 10% hot atomic.
 * Planted races: per block b one owned word pw_b gets two conflicting writes
 * replacing regular accesses — two threads of block b (warps 0-3 and 4-5) in
 * the same epoch (BLOCK scope), or one thread of b and one of block b+1
 * (warps 6-7) (GRID scope).  No other access can race, so the racy set is
 * exactly {pw_b} with those scopes (closed form, tests/test_c5.py).
 *
 * Row layout per warp: 8 epochs x (32 access rows, 1 __syncthreads row) = 264
 * rows.  Sharded variant (rank r of N = 2^log2n): a lane keeps only records
 * whose shadow granule (word >> glog2; default 3 = 64 B of shadow) is owned by r (hr_shard_owner), kept
 * records are compacted per lane inside each epoch, epoch segments are padded
 * with NOPs to the warp's longest lane, barrier rows are kept.
 */
#ifndef C5GEN_H_
#define C5GEN_H_

#include <stdint.h>

#ifdef __CUDACC__
#define C5_HD __host__ __device__ __forceinline__
#else
#define C5_HD static inline
#endif

#define C5_WARPS 8
#define C5_LANES 32
#define C5_ACC 256
#define C5_EPOCH 32
#define C5_EPOCHS (C5_ACC / C5_EPOCH)
#define C5_ROWS (C5_ACC + C5_EPOCHS)
#define C5_NOP (3ull << 62)
#define C5_SYNC ((3ull << 62) | 1ull)

#define C5_TAG_WS 0x1ull
#define C5_TAG_LANE 0x2ull
#define C5_TAG_PLANT 0x3ull

typedef struct {
    uint64_t seed;
    uint32_t lb;      /* log2 blocks, 1..16 */
} c5_params;

C5_HD uint64_t c5_mix(uint64_t x)
{
    /* splitmix64 finaliser */
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

C5_HD uint64_t c5_hash(uint64_t seed, uint64_t tag, uint64_t ctr)
{
    return c5_mix(seed * 0xD1B54A32D192ED03ull + (tag << 58) + ctr);
}

C5_HD uint64_t c5_total_words(uint32_t lb) { return 1ull << (lb + 16); }
C5_HD uint64_t c5_owned_words(uint32_t lb) { return 1ull << (lb + 15); }
C5_HD uint32_t c5_hot_log2(uint32_t lb) { return lb + 4; }

typedef struct {
    uint64_t word;
    uint32_t t1, t2, j1, j2, b2, grid;
} c5_plant;

C5_HD c5_plant c5_plant_of(const c5_params *p, uint64_t b)
{
    uint64_t h = c5_hash(p->seed, C5_TAG_PLANT, b);
    c5_plant r;
    uint64_t prow = h & 127, pt = (h >> 7) & 255;
    r.word = (b << 15) | (prow << 8) | pt;
    r.grid = (uint32_t)((h >> 15) & 1);
    uint32_t e = (uint32_t)((h >> 16) & 7);
    r.j1 = e * 32 + (uint32_t)((h >> 19) & 31);
    r.j2 = e * 32 + (uint32_t)((h >> 24) & 31);
    r.t1 = (uint32_t)((h >> 29) & 127);
    r.t2 = (r.grid ? 192u : 128u) + (uint32_t)((h >> 36) & 63);
    uint64_t nb = 1ull << p->lb;
    r.b2 = (uint32_t)(r.grid ? ((b + 1) & (nb - 1)) : b);
    return r;
}

/* The record of thread (b, ltid) at access j (0 <= j < 256). */
C5_HD uint64_t c5_record(const c5_params *p, uint64_t b, uint32_t t, uint32_t j)
{
    const uint64_t nb = 1ull << p->lb;
    /* planted writes replace regular accesses */
    if (t < 128) {
        c5_plant q = c5_plant_of(p, b);
        if (t == q.t1 && j == q.j1) return (1ull << 62) | q.word;
    } else if (t < 192) {
        c5_plant q = c5_plant_of(p, b);
        if (!q.grid && t == q.t2 && j == q.j2) return (1ull << 62) | q.word;
    } else {
        uint64_t pb = (b + nb - 1) & (nb - 1);
        c5_plant q = c5_plant_of(p, pb);
        if (q.grid && t == q.t2 && j == q.j2) return (1ull << 62) | q.word;
    }
    const uint32_t w = t >> 5;
    const uint64_t u = c5_hash(p->seed, C5_TAG_WS, (((b << 3) | w) << 8) | j);
    const uint64_t v = c5_hash(p->seed, C5_TAG_LANE, (((b << 8) | t) << 8) | j);
    const uint32_t cat = (uint32_t)((u & 0xffff) % 10);
    const uint64_t owned = c5_owned_words(p->lb);
    const uint64_t total = c5_total_words(p->lb);
    const uint32_t hl = c5_hot_log2(p->lb);
    if (cat < 5) {
        uint64_t row = (u >> 16) & 127;
        uint64_t word = (b << 15) | (row << 8) | t;
        uint64_t kind = (v % 5) < 3 ? 0 : 1;
        return (kind << 62) | word;
    }
    if (cat < 9) {
        uint64_t ro = total - (1ull << hl) - owned;
        uint64_t word = owned + (((v >> 32) * ro) >> 32);
        return word;                                   /* read */
    }
    uint32_t e = (uint32_t)((v >> 8) % hl);
    uint64_t rank = ((1ull << e) - 1) + ((v >> 32) & ((1ull << e) - 1));
    return (2ull << 62) | (total - (1ull << hl) + rank);   /* atomic */
}

/* shard owner of a record's granule: include/hr.h hr_shard_owner (stripes of
 * 2^log2n granules, rotated per stripe by a multiplicative hash) */
C5_HD int c5_owned_by(uint64_t rec, uint32_t rank, uint32_t log2n, uint32_t glog2)
{
    const uint64_t gran = (rec & ((1ull << 61) - 1)) >> glog2;
    const uint64_t stripe = gran >> log2n;
    const uint32_t rot = log2n ? ((uint32_t)(stripe ^ (stripe >> 32)) * 0x9E3779B1u) >> (32u - log2n) : 0u;
    return (((uint32_t)gran + rot) & ((1u << log2n) - 1u)) == rank;
}

#endif /* C5GEN_H_ */
