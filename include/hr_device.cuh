/*
 * hr_device.cuh — header-only, device-inlined HiRace per-access check for
 * sm_100a (B200).  Citations: PAPER.md:n = /root/reference/PAPER.md line n.
 *
 * Algorithm 1 "UpdateShadow", per access:
 *   repeat
 *     oShadow <- atomicRead(sAddr)                         (a4)
 *     <oState, oTid, oBC, oWC> <- UnpackShadow(oShadow)
 *     tRel <- compareTids(tid, oTid);  sRel <- checkSync   (a5)
 *     nState <- table[oState, access, sRel, tRel]          (a6)
 *     nShadow <- PackShadow(nState, tid, bc, wc)
 *   until atomicCAS(sAddr, oShadow, nShadow)              (a8)
 *
 * B200-first changes, none of which changes the result:
 *   a3  lanes of a warp hitting the same word are grouped with
 *       __match_any_sync (MATCH.ANY.U64); the lowest lane folds the group's
 *       accesses in lane order (they are unordered: same warp, same epochs,
 *       so any order is happens-before consistent) and commits ONE CAS.
 *   a7  fast exits without a write: nShadow == oShadow, or the state is in a
 *       label-insensitive closure (GREAD, GATOMIC, RACE_GRID: the stored
 *       tid/clocks are dead), or block-only (RACE_BLOCK) with a non-Global
 *       relation.  Linearisable at the load.
 *   a9  race reports go to an append-only ring with one warp-aggregated
 *       atomicAdd per warp.
 * Global shadow: 1:1 word-granular 8-byte words in HBM, loaded with
 * ld.relaxed.gpu (L2, never a stale L1 line) and ATOMG.E.CAS.64.  Shared
 * shadow: per-block instance staged in SMEM, ATOMS.CAS.64.
 *
 * Entry points for online instrumentation:
 *   hr_thread_begin, hr_check_read / _write / _atomic, hr_syncthreads, hr_syncwarp.
 * The replay kernel (csrc/hr_replay.cu) calls the same hr_check_lanes core.
 */
#ifndef HR_DEVICE_CUH_
#define HR_DEVICE_CUH_

#include <stdint.h>

#include "hr.h"

#define HR_FSM_BYTES 2048
/* table + per-state flags + a 16-byte block scratch (zero in the global copy):
 * [HR_FSM_DROP_OFF] counts this block's shared-space race records the full
 * ring dropped (a9 overflow; hr_thread_end spills the instance when non-zero) */
#define HR_FSM_DROP_OFF (HR_FSM_BYTES + 32)
#define HR_FSM_SMEM_BYTES (HR_FSM_BYTES + 48)
/* a NOP C32 record in the global table copy (word 0 at +0, op byte 3 at +4):
 * the row loop points lanes beyond the grid at it instead of testing them */
#define HR_FSM_NOP_OFF (HR_FSM_BYTES + 40)
#define HR_STATE_SHIFT 59
#define HR_TID_SHIFT 32
#define HR_RACE_BLOCK 30u
#define HR_RACE_GRID 31u
#define HR_FLAG_RACE 1u
#define HR_FLAG_INSENSITIVE 2u
#define HR_FLAG_BLOCK_ONLY 4u
#define HR_WORD_MASK ((1ull << 61) - 1)

/* By-value kernel argument: everything the check needs (owned by hr_ctx). */
struct hr_dev {
    unsigned long long *gshadow;  /* local global-shadow slice (this shard's granules) */
    uint64_t gbase;               /* first monitored global word */
    uint64_t gwords;              /* monitored global words (whole region, all shards) */
    hr_race *ring;
    unsigned int *ring_tail;
    unsigned int *flags;          /* = ring_tail + 1 */
    hr_race *spill;               /* a9 overflow store (right after the ring: ring + ring_cap) */
    unsigned int *ovf;            /* = ring_tail + 2: [0] spill tail [1] shared drops not yet spilled [2] global drop:
                                     kernel id + 1 of a kernel whose global race record the full ring
                                     dropped (0 = none) [3] spill-scan completion counter */
    uint32_t spill_cap;
    unsigned long long *counters; /* [0] checks [1] CAS retries [2] fast exits */
    const unsigned char *fsm;     /* HR_FSM_SMEM_BYTES in global memory */
    uint32_t ring_cap;
    uint32_t kernel_id;
    uint32_t shard_rank, shard_log2; /* owner(granule) = hr_shard_owner(granule, shard_log2) (hr.h) */
    uint32_t gran_log2;           /* shard granule = 2^gran_log2 words (default 3: 64 B of shadow) */
    uint32_t wc_bits;             /* bc occupies [31:wc_bits], wc [wc_bits-1:0] */
    uint32_t bc_max, wc_max;
    uint32_t options;             /* HR_OPT_* */
    uint32_t block_base;          /* simulated block of blockIdx 0 (chunked replay launches) */
    uint32_t rep_bstride, rep_wstride; /* representative threads (hr_set_representatives): only
                                          blocks % rep_bstride == 0 and warps % rep_wstride == 0
                                          are checked; 1 = all */
    uint32_t owned_only;          /* the replayed trace is HR_TRACE_F_SHARD_OWNED: no owner test */
    uint32_t wc_lsh;              /* 32 - wc_bits (shifts the wc field to the top) */
    uint32_t tile_log2;           /* warp-level barriers order tiles of 2^tile_log2 lanes (5 = whole
                                     warps): the "Warp" relation is "same tile" (reading R8) */
    uint32_t epoch_tag;           /* HR_OPT_LAZY_RESET: kernel epoch tag 1..15 in bits [31:28] of the
                                     shadow's clock word; a global word with another tag is INIT.
                                     0 = off (the shadow is zeroed at every kernel boundary) */
    /* hybrid binned replay (HR_OPT_BINNED, csrc/hr_hybrid.cuh): the row replay appends
     * the global accesses of the shadow buckets set in hy_map as entries (run of
     * (bucket, block) at hy_off[bucket * hy_nb + block]) instead of checking them */
    const uint32_t *hy_map;       /* bitmap over 2^HR_HY_BITS-word buckets; nullptr = off */
    const unsigned long long *hy_off;
    unsigned long long *hy_ent;
    uint32_t hy_nb, hy_nbk;       /* blocks of the launch, buckets */
    uint32_t hy_sa_off;           /* per-bucket write positions (u64) at this offset past the FSM copy */
    uint64_t glocal_words;        /* words of the local global shadow (gshadow[0, glocal_words)) */
};

/* hybrid entry: [63:42] word offset in the bucket | [41:40] kind | [39:13] packed tid
 * | [12:6] bc | [5:0] wc */
#ifdef HR_HY_BITS_OVERRIDE
#define HR_HY_BITS HR_HY_BITS_OVERRIDE
#else
#define HR_HY_BITS 22u
#endif
#define HR_HY_BC_MAX 127u
#define HR_HY_WC_MAX 63u

/* Per-thread registers. */
struct hr_thr {
    /* tid<<32 | bc<<wc_bits | wc: the packed tid (block:17 | warp:5 | lane:5) and
     * the thread-private block / warp scalar clocks, kept in the
     * shadow word's own layout so a barrier is one add (no separate registers) */
    unsigned long long meta;
    uint32_t sshadow;             /* shared-space address of this block's shadow instance */
    uint32_t swords;
    uint32_t fsm;                 /* shared-space address of the FSM table copy */
    uint32_t off;                 /* bit 0: detection disabled (clock overflow); bit 1: this block's
                                     shared instance belongs to another shard (set once) */
    __device__ __forceinline__ uint32_t tid() const { return (uint32_t)(meta >> HR_TID_SHIFT) & 0x7ffffffu; }
};

/* ---------------- schedule fuzzing (tests only) ----------------
 * Built with -DHR_FUZZ (libhirace_fuzz.so, tests/test_gpu_fuzz.py): a
 * pseudo-random __nanosleep before a quarter of the shadow CASes, same-word
 * groups folded in descending lane order, and the replay grid's CUDA blocks
 * mapped to simulated blocks in reverse.  Each changes the commit order of
 * some words; the racy set must not change (schedule independence). */
#ifdef HR_FUZZ
__device__ __forceinline__ void hr__jitter()
{
    uint32_t x = (uint32_t)clock64() * 2654435761u ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
    x ^= x >> 15;
    x *= 0x2C1B3C6Du;
    x ^= x >> 12;
    if ((x & 3u) == 0u) __nanosleep(x >> 22);
}
#define HR_JITTER() hr__jitter()
#else
#define HR_JITTER()
#endif

/* ---------------- memory primitives ---------------- */

__device__ __forceinline__ unsigned long long hr__ld_g(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long hr__cas_g(unsigned long long *p, unsigned long long cmp,
                                                        unsigned long long val)
{
    HR_JITTER();
    return atomicCAS(p, cmp, val);
}

__device__ __forceinline__ unsigned long long hr__ld_s(uint32_t a)
{
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long hr__cas_s(uint32_t a, unsigned long long cmp,
                                                        unsigned long long val)
{
    unsigned long long r;
    HR_JITTER();
    asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(r) : "r"(a), "l"(cmp), "l"(val) : "memory");
    return r;
}

/* HR_OPT_SMEM32 shared-shadow words: state 5 | warp 5 | lane 5 | bc 9 | wc 8;
 * the block is implicit (one instance per block).  Converted to and from the
 * 64-bit layout at the SMEM boundary, so Algorithm 1 itself is unchanged;
 * exact while bc <= 511 and wc <= 255 (make_dev caps the clocks there). */
#define HR_S32_STATE_SHIFT 27
__device__ __forceinline__ uint32_t hr__s32_pack(unsigned long long w, uint32_t wc_bits)
{
    const uint32_t lo = (uint32_t)w;
    return ((uint32_t)(w >> HR_STATE_SHIFT) << HR_S32_STATE_SHIFT) | (((uint32_t)(w >> HR_TID_SHIFT) & 1023u) << 17) |
           (((lo >> wc_bits) & 511u) << 8) | (lo & 255u);
}

/* `tag_hi` = the epoch-tag bits of the current kernel (shared words are always
 * of this kernel: the instance is zeroed at block start) */
__device__ __forceinline__ unsigned long long hr__s32_unpack(uint32_t v, uint32_t own_tid, uint32_t wc_bits,
                                                             uint32_t tag_hi)
{
    if (v == 0u) return 0ull;                                           /* INIT */
    const uint32_t tid = (own_tid & ~1023u) | ((v >> 17) & 1023u);
    return ((unsigned long long)(v >> HR_S32_STATE_SHIFT) << HR_STATE_SHIFT) |
           ((unsigned long long)tid << HR_TID_SHIFT) | (tag_hi | (((v >> 8) & 511u) << wc_bits) | (v & 255u));
}

__device__ __forceinline__ uint32_t hr__lds_u8(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t hr__laneid()
{
    uint32_t l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

/* Diagnostic counters (only in builds with -DHR_COUNTERS; hr_counters):
 * [0] checked accesses [1] failed CAS (Algorithm 1 retries) [2] a7 fast exits
 * [3] committed CAS.  Slices per SM (HR_CNT_BASE + slice * 4 + i) keep the
 * atomics of a diagnostic run from serialising on one word. */
#define HR_CNT_BASE 32u
#define HR_CNT_SLICES 32u
#ifdef HR_COUNTERS
__device__ __forceinline__ uint32_t hr__smid()
{
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}
#define HR_COUNT(d, i) atomicAdd(&(d).counters[HR_CNT_BASE + ((hr__smid() % HR_CNT_SLICES) << 2) + (i)], 1ull)
#else
#define HR_COUNT(d, i) ((void)0)
#endif

/* Control rows (replay: the trace format's warp-aligned barriers,
 * tracegen/format.py): do the lanes holding a control record disagree on it? */
__device__ __forceinline__ bool hr__ctrl_mixed(uint64_t x, unsigned ctrl)
{
    const bool is_ctrl = (x >> 62) == 3u && (x & HR_WORD_MASK) != 0u;
    const unsigned same = __match_any_sync(0xffffffffu, is_ctrl ? x : 0ull);
    return __any_sync(0xffffffffu, is_ctrl && same != ctrl);
}

/* Divergent control row, except a sub-warp __syncwarp (every control lane holds
 * the same __syncwarp record, but not every active lane): that one is
 * __syncwarp(mask), see hr__barrier_row. */
__device__ __forceinline__ bool hr__ctrl_divergent(uint64_t x, unsigned ctrl, unsigned lane_mask)
{
    return ctrl != lane_mask || hr__ctrl_mixed(x, ctrl);
}

/* ---------------- labels ---------------- */

/* compareTids: Self 0, Warp 1, Block 2, Global 3 from the packed-tid XOR.  With
 * warp tiles of 2^tl lanes the packed tid block:17 | warp:5 | lane:5 is also
 * block:17 | tile:(10-tl) | lane-in-tile:tl, and "Warp" means "same tile" (the
 * unit a warp-level barrier orders); tl = 5: whole warps. */
__device__ __forceinline__ uint32_t hr__rel(uint32_t tid, uint32_t otid, uint32_t tl = 5u)
{
    uint32_t x = tid ^ otid;
    return (x != 0u) + (x >= (1u << tl)) + (x >= 1024u);
}

/* checkSync: Bs 2 if same block and bc advanced; else Ws 1 if same warp and wc
 * advanced; else Us 0 (Bs dominates Ws). */
__device__ __forceinline__ uint32_t hr__sync(uint32_t rel, uint32_t lo, uint32_t olo, uint32_t wc_bits)
{
    uint32_t bc = lo >> wc_bits, obc = olo >> wc_bits;
    uint32_t wmask = (1u << wc_bits) - 1u;   /* 1 <= wc_bits <= 31 */
    uint32_t wc = lo & wmask, owc = olo & wmask;
    if (rel != 3u && bc > obc) return 2u;
    if (rel <= 1u && wc > owc) return 1u;
    return 0u;
}

__device__ __forceinline__ void hr__set_flag(const hr_dev &d, unsigned int f)
{
    if ((*(volatile unsigned int *)d.flags & f) != f) atomicOr(d.flags, f);
}

/* ---------------- the check core ---------------- */

/* Ablation options (HR_OPT_NO_COALESCE / NO_FASTEXIT / SPECULATE) are read
 * only when ABL: the default replay kernels are instantiated with ABL = false
 * and carry no option tests on the per-access path. */
template <bool ABL>
__device__ __forceinline__ bool hr__opt(const hr_dev &d, uint32_t bit)
{
    return ABL && (d.options & bit);
}

/* L1-cacheable probe (weak load): only used to take the insensitive-closure exit,
 * which is valid for any value observed during this kernel (a7). */
__device__ __forceinline__ unsigned long long hr__ld_g_l1(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

/* emit-info word (one register instead of a 24-byte record):
 * [31] emit  [30:26] racing lane  [25:24] its kind  [23:19] prev state  [0] grid */
#define HR_EI_EMIT 0x80000000u
/* first-attempt provenance of `old`: guess (INIT), weak L1 probe, coherent */
#define HR_OLD_GUESS 0u
#define HR_OLD_PROBE 1u
#define HR_OLD_FRESH 2u

/* a11 with HR_OPT_LAZY_RESET: the value Algorithm 1 sees.  A word written
 * under another kernel's epoch tag belongs to an earlier kernel, and a kernel
 * boundary orders everything, so it is INIT (the CAS still compares against
 * the raw word).  hr_kernel_begin zeroes the shadow for real before a tag is
 * reused (every 15 kernels). */
__device__ __forceinline__ unsigned long long hr__live(const hr_dev &d, unsigned long long old)
{
    return (d.epoch_tag && old != 0ull && (((uint32_t)old >> 28) & 15u) != d.epoch_tag) ? 0ull : old;
}

/* Shared shadow word of this block's instance: load / CAS in the 64-bit layout. */
template <bool ABL>
__device__ __forceinline__ uint32_t hr__saddr(const hr_dev &d, const hr_thr &t, uint64_t local)
{
    return t.sshadow + ((uint32_t)local << (hr__opt<ABL>(d, HR_OPT_SMEM32) ? 2 : 3));
}

/* HR_OPT_SMEM32 is read only by the ABL (all options at run time) kernels; the
 * host routes a ctx with SMEM32 to them */
template <bool ABL>
__device__ __forceinline__ unsigned long long hr__ld_sh(const hr_dev &d, const hr_thr &t, uint32_t a)
{
    if (hr__opt<ABL>(d, HR_OPT_SMEM32)) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return hr__s32_unpack(v, t.tid(), d.wc_bits, d.epoch_tag << 28);
    }
    return hr__ld_s(a);
}

template <bool ABL>
__device__ __forceinline__ unsigned long long hr__cas_sh(const hr_dev &d, const hr_thr &t, uint32_t a,
                                                         unsigned long long cmp, unsigned long long val)
{
    if (hr__opt<ABL>(d, HR_OPT_SMEM32)) {
        const uint32_t c = hr__s32_pack(cmp, d.wc_bits), v = hr__s32_pack(val, d.wc_bits);
        uint32_t r;
        HR_JITTER();
        asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(r) : "r"(a), "r"(c), "r"(v) : "memory");
        return r == c ? cmp : hr__s32_unpack(r, t.tid(), d.wc_bits, d.epoch_tag << 28);
    }
    return hr__cas_s(a, cmp, val);
}

/* t.off of a thread of simulated block `block`, warp `warp`: bit 1 = its block's
 * shared instance belongs to another address shard, bit 0 = not a representative
 * thread ("tracking only representative threads for user-defined
 * symmetric work groups"), so its accesses are not checked. */
__device__ __forceinline__ uint32_t hr__thread_off(const hr_dev &d, uint32_t block, uint32_t warp)
{
    const uint32_t sh = ((block & ((1u << d.shard_log2) - 1u)) == d.shard_rank) ? 0u : 2u;
    const bool rep = (d.rep_bstride <= 1u || block % d.rep_bstride == 0u) &&
                     (d.rep_wstride <= 1u || warp % d.rep_wstride == 0u);
    return sh | (rep ? 0u : 1u);
}

/* a2: shard-local shadow index; false if this ctx does not check the access. */
__device__ __forceinline__ bool hr__locate(const hr_dev &d, const hr_thr &t, uint32_t space, uint64_t word,
                                           uint64_t &local)
{
    if (space != 0u) {
        if (word >= t.swords) { hr__set_flag(d, HR_F_UNMONITORED); return false; }
        local = word;
        return !(t.off & 2u);
    }
    const uint64_t g = word - d.gbase;
    if (word < d.gbase || g >= d.gwords) { hr__set_flag(d, HR_F_UNMONITORED); return false; }
    const uint64_t gran = g >> d.gran_log2;
    local = ((gran >> d.shard_log2) << d.gran_log2) | (g & ((1ull << d.gran_log2) - 1u));
    return d.owned_only || hr_shard_owner(gran, d.shard_log2) == d.shard_rank;
}

/* a5 + a6 (+ a3 fold): the state after this lane's access from `old`, then the
 * accesses of the other lanes of `peers` (kinds in kb0/kb1) in lane order with
 * label (kind_j, Us, Warp).  rinfo receives the first RACE entry, rel the
 * relation of the first label. */
__device__ __forceinline__ uint32_t hr__transition(const hr_dev &d, const hr_thr &t, unsigned long long old,
                                                   uint32_t kind, uint32_t lane, unsigned peers, unsigned kb0,
                                                   unsigned kb1, uint32_t &rinfo, uint32_t &rel)
{
    const uint32_t os = (uint32_t)(old >> HR_STATE_SHIFT);
#ifdef HR_FUZZ
    /* descending lane order: the highest peer's access is labelled against `old` */
    {
        const uint32_t f = 31u - __clz(peers);
        kind = ((kb0 >> f) & 1u) | (((kb1 >> f) & 1u) << 1);
        lane = f;
    }
    const uint32_t ftid = (t.tid() & ~31u) | lane;
#else
    const uint32_t ftid = t.tid();
#endif
    rel = hr__rel(ftid, (uint32_t)(old >> HR_TID_SHIFT) & 0x7ffffffu, d.tile_log2);
    const uint32_t sync = hr__sync(rel, (uint32_t)t.meta, (uint32_t)old, d.wc_bits);
    uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | (kind << 4) | (sync << 2) | rel));
    rinfo = (cur >= HR_RACE_BLOCK && cur != os) ? (HR_EI_EMIT | (lane << 26) | (kind << 24) | (os << 19)) : 0u;
    unsigned r = peers & ~(1u << lane);
    uint32_t prev = lane;
    while (r) {
#ifdef HR_FUZZ
        const uint32_t j = 31u - __clz(r);
        r &= ~(1u << j);
#else
        const uint32_t j = __ffs(r) - 1;
        r &= r - 1;
#endif
        const uint32_t kj = ((kb0 >> j) & 1u) | (((kb1 >> j) & 1u) << 1);
        /* lanes of one row: same epochs (Us); Warp inside a tile, Block across tiles */
        const uint32_t rj = ((j ^ prev) >> d.tile_log2) ? 2u : 1u;
        prev = j;
        const uint32_t nx = hr__lds_u8(t.fsm + ((cur << 6) | (kj << 4) | rj));
        if (nx >= HR_RACE_BLOCK && cur < HR_RACE_BLOCK && !rinfo)
            rinfo = HR_EI_EMIT | (j << 26) | (kj << 24) | (cur << 19);
        cur = nx;
    }
    return cur;
}

__device__ __forceinline__ unsigned long long hr__nmeta(const hr_thr &t, unsigned peers)
{
#ifdef HR_FUZZ
    const uint32_t last_lane = __ffs(peers) - 1;                 /* descending fold ends at the lowest */
#else
    const uint32_t last_lane = 31u - __clz(peers);
#endif
    return (t.meta & ~(0x1full << HR_TID_SHIFT)) | ((unsigned long long)last_lane << HR_TID_SHIFT);
}

/* Fold-free variant for the common case of a lane alone on its word: one
 * label, the lane's own meta, no group bookkeeping. */
template <bool ABL>
__device__ __forceinline__ uint32_t hr__commit_single(const hr_dev &d, const hr_thr &t, bool is_shared,
                                                      uint32_t sh_addr, unsigned long long *gp,
                                                      unsigned long long old, uint32_t fresh, uint32_t kind)
{
    const bool fastexit = !hr__opt<ABL>(d, HR_OPT_NO_FASTEXIT);
    const uint32_t kcol = kind << 4;
    while (true) {
        const unsigned long long lv = is_shared ? old : hr__live(d, old);   /* shared words are this kernel's */
        const uint32_t os = (uint32_t)(lv >> HR_STATE_SHIFT);
        const uint32_t rel = hr__rel(t.tid(), (uint32_t)(lv >> HR_TID_SHIFT) & 0x7ffffffu, d.tile_log2);
        const uint32_t sync = hr__sync(rel, (uint32_t)t.meta, (uint32_t)lv, d.wc_bits);
        const uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | kcol | (sync << 2) | rel));
        const unsigned long long nw = ((unsigned long long)cur << HR_STATE_SHIFT) | t.meta;
        if (cur == os && fresh != HR_OLD_GUESS && fastexit) {
            const uint32_t f = hr__lds_u8(t.fsm + HR_FSM_BYTES + os);
            if ((f & HR_FLAG_INSENSITIVE) || ((f & HR_FLAG_BLOCK_ONLY) && rel != 3u && fresh == HR_OLD_FRESH)) {
                HR_COUNT(d, 2);
                return 0u;                                                /* a7 (ii), (iii) */
            }
        }
        if (nw == old) {
            if (fresh == HR_OLD_FRESH) { HR_COUNT(d, 2); return 0u; }     /* a7 (i) */
            if (fresh == HR_OLD_PROBE) { old = hr__ld_g(gp); fresh = HR_OLD_FRESH; continue; }
        }
        const unsigned long long prev = is_shared ? hr__cas_sh<ABL>(d, t, sh_addr, old, nw) : hr__cas_g(gp, old, nw);
        if (prev == old) {                                                /* a8 committed */
            HR_COUNT(d, 3);
            if (cur >= HR_RACE_BLOCK && cur != os)
                return HR_EI_EMIT | (hr__laneid() << 26) | (kind << 24) | (os << 19) | (cur == HR_RACE_GRID);
            return 0u;
        }
        HR_COUNT(d, 1);
        old = prev;
        fresh = HR_OLD_FRESH;
    }
}

/* a7 + a8: Algorithm 1's repeat/until loop from a first value `old` of the
 * given provenance; returns the emit info of the committed transition (0 if
 * none or a fast exit). */
template <bool ABL>
__device__ __forceinline__ uint32_t hr__commit(const hr_dev &d, const hr_thr &t, bool is_shared, uint32_t sh_addr,
                                               unsigned long long *gp, unsigned long long old, uint32_t fresh,
                                               uint32_t kind, uint32_t lane, unsigned peers, unsigned kb0,
                                               unsigned kb1)
{
    const bool fastexit = !hr__opt<ABL>(d, HR_OPT_NO_FASTEXIT);
    const unsigned long long nmeta = hr__nmeta(t, peers);
    while (true) {
        const unsigned long long lv = is_shared ? old : hr__live(d, old);   /* shared words are this kernel's */
        const uint32_t os = (uint32_t)(lv >> HR_STATE_SHIFT);
        uint32_t rinfo, rel;
        const uint32_t cur = hr__transition(d, t, lv, kind, lane, peers, kb0, kb1, rinfo, rel);
        const unsigned long long nw = ((unsigned long long)cur << HR_STATE_SHIFT) | nmeta;
        if (fastexit && cur == os && fresh != HR_OLD_GUESS) {
            const uint32_t f = hr__lds_u8(t.fsm + HR_FSM_BYTES + os);
            if ((f & HR_FLAG_INSENSITIVE) || ((f & HR_FLAG_BLOCK_ONLY) && rel != 3u && fresh == HR_OLD_FRESH)) {
                HR_COUNT(d, 2);
                return 0u;                                                /* a7 (ii), (iii) */
            }
        }
        if (nw == old) {
            if (fresh == HR_OLD_FRESH) { HR_COUNT(d, 2); return 0u; }     /* a7 (i) */
            if (fresh == HR_OLD_PROBE) { old = hr__ld_g(gp); fresh = HR_OLD_FRESH; continue; }
        }
        const unsigned long long prev = is_shared ? hr__cas_sh<ABL>(d, t, sh_addr, old, nw) : hr__cas_g(gp, old, nw);
        if (prev == old) {                                                /* a8 committed */
            HR_COUNT(d, 3);
            return rinfo ? (rinfo | (cur == HR_RACE_GRID ? 1u : 0u)) : 0u;
        }
        HR_COUNT(d, 1);
        old = prev;
        fresh = HR_OLD_FRESH;
    }
}

/* First value of Algorithm 1's loop (a4): SMEM load; L1 probe for global
 * atomics; a coherent L2 load (ld.relaxed.gpu) for global reads/writes, or
 * with HR_OPT_SPECULATE an INIT guess (the CAS then doubles as the atomic read). */
template <bool ABL>
__device__ __forceinline__ unsigned long long hr__first(const hr_dev &d, const hr_thr &t, bool is_shared,
                                                        uint32_t sh_addr, const unsigned long long *gp, uint32_t kind,
                                                        uint32_t &fresh)
{
    if (is_shared) { fresh = HR_OLD_FRESH; return hr__ld_sh<ABL>(d, t, sh_addr); }
    if (kind == HR_ATOMIC && !hr__opt<ABL>(d, HR_OPT_NO_FASTEXIT)) { fresh = HR_OLD_PROBE; return hr__ld_g_l1(gp); }
    if (hr__opt<ABL>(d, HR_OPT_SPECULATE)) { fresh = HR_OLD_GUESS; return 0ull; }
    fresh = HR_OLD_FRESH;
    return hr__ld_g(gp);
}

/* a9 overflow: the ring is full and this race record is dropped.  Every drop
 * is recovered exactly ("ring overflow"):
 *   global: the kernel's id is latched in ovf[2]; hr_spill_scan_kernel, which
 *     the host enqueues after the kernel (before its shadow is reset), copies
 *     every RACE word of that kernel's global shadow into the spill;
 *   shared: the block's drop count (shared address `drop_sa`) and ovf[1] are raised;
 *     hr_thread_end spills every RACE word of the block's instance and lowers
 *     ovf[1] again.  ovf[1] != 0 at report time = a block that never spilled.
 * The finite-history baseline has no FSM shadow to scan: its drops are lost. */
/* (scalar arguments: a rare path kept out of line without copying hr_dev to the
 * stack; flags and ovf are found from the ring tail: make_dev lays them out as
 * tail[1] and tail[2..5], so the hot loop keeps no extra constants live) */
static __device__ __noinline__ void hr__ring_drop_x(unsigned int *tail, bool fh, uint32_t kernel_id, uint32_t drop_sa,
                                                   uint32_t space)
{
    unsigned int *flags = tail + 1, *ovf = tail + 2;
    if ((*(volatile unsigned int *)flags & HR_F_RING_OVERFLOW) == 0u) atomicOr(flags, HR_F_RING_OVERFLOW);
    if (fh) {
        atomicAdd(&ovf[1], 1u);
    } else if (space) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(drop_sa) : "memory");
        atomicAdd(&ovf[1], 1u);
    } else if (*(volatile unsigned int *)&ovf[2] != kernel_id + 1u) {
        *(volatile unsigned int *)&ovf[2] = kernel_id + 1u;
    }
}

template <bool FH = false>
__device__ __forceinline__ void hr__ring_drop(const hr_dev &d, uint32_t drop_sa, uint32_t space)
{
    hr__ring_drop_x(d.ring_tail, FH, d.kernel_id, drop_sa, space);
}

/* Append one record to the spill (warp-aggregated over the lanes of `mask`
 * with want = true); past spill_cap the set is incomplete (HR_F_INCOMPLETE). */
__device__ __forceinline__ void hr__spill_put(hr_race *spill, unsigned int *ovf, uint32_t spill_cap,
                                              unsigned int *flags, unsigned mask, bool want, const hr_race &r)
{
    const unsigned m = __ballot_sync(mask, want);
    if (!m) return;
    const uint32_t lane = hr__laneid(), leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&ovf[0], (unsigned)__popc(m));
    base = __shfl_sync(mask, base, leader);
    if (want) {
        const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
        if (slot < spill_cap) spill[slot] = r;
        else atomicOr(flags, HR_F_INCOMPLETE);
    }
}

/* The RACE words of one shared instance (`words` words at shared address
 * `sa`, 64-bit or HR_OPT_SMEM32 layout) into the spill, by the `nthr` threads
 * of the caller (ltid = 0..nthr-1: whole warps, or nthr < 32 lanes of one). */
static __device__ __noinline__ void hr__spill_instance_x(hr_race *spill, unsigned int *ovf, uint32_t spill_cap,
                                                         unsigned int *flags, uint32_t options, uint32_t kernel_id,
                                                         uint32_t sa, uint32_t words, uint32_t block, uint32_t ltid,
                                                         uint32_t nthr)
{
    const bool s32 = (options & HR_OPT_SMEM32) != 0u;
    const unsigned mask = nthr >= 32u ? 0xffffffffu : ((1u << nthr) - 1u);
    for (uint32_t i0 = ltid & ~31u; i0 < words; i0 += nthr) {
        const uint32_t i = i0 + (ltid & 31u);
        uint32_t st = 0, tid = 0;
        if (i < words) {
            if (s32) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sa + 4u * i) : "memory");
                st = v >> HR_S32_STATE_SHIFT;
                tid = (block << 10) | ((v >> 17) & 1023u);
            } else {
                const unsigned long long v = hr__ld_s(sa + 8u * i);
                st = (uint32_t)(v >> HR_STATE_SHIFT);
                tid = (uint32_t)(v >> HR_TID_SHIFT) & 0x7ffffffu;
            }
        }
        hr_race r;
        r.word = i;
        r.block = block;
        r.kernel = kernel_id;
        r.first_tid = tid;
        r.space = HR_SHARED;
        r.scope = (uint8_t)(st == HR_RACE_GRID ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
        r.first_kind = 0xff;                      /* witness unknown: diagnostic fields only */
        r.prev_state = 0xff;
        hr__spill_put(spill, ovf, spill_cap, flags, mask, i < words && st >= HR_RACE_BLOCK, r);
    }
}

__device__ __forceinline__ void hr__spill_instance(const hr_dev &d, uint32_t sa, uint32_t words, uint32_t block,
                                                   uint32_t ltid, uint32_t nthr)
{
    hr__spill_instance_x(d.spill, d.ovf, d.spill_cap, d.flags, d.options, d.kernel_id, sa, words, block, ltid, nthr);
}

template <bool FH = false>
__device__ __forceinline__ void hr__write_race(const hr_dev &d, const hr_thr &t, uint32_t slot, uint32_t space,
                                               uint64_t word, uint32_t ei)
{
    if (slot < d.ring_cap) {
        hr_race rr;
        rr.word = word;
        rr.block = space ? (t.tid() >> 10) : 0xffffffffu;
        rr.kernel = d.kernel_id;
        rr.first_tid = (t.tid() & ~31u) | ((ei >> 26) & 31u);
        rr.space = (uint8_t)space;
        rr.scope = (uint8_t)((ei & 1u) ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
        rr.first_kind = (uint8_t)((ei >> 24) & 3u);
        rr.prev_state = (uint8_t)((ei >> 19) & 31u);
        d.ring[slot] = rr;
    } else {
        hr__ring_drop<FH>(d, t.fsm + HR_FSM_DROP_OFF, space);
    }
}

/* a3 grouping of one row: peers (lanes with the same key, lowest = leader) and
 * the kind bits for the fold.  Pre-test: strictly increasing keys over the full
 * warp means all distinct, and MATCH is skipped. */
template <bool ONLINE, bool ABL>
__device__ __forceinline__ unsigned hr__group(const hr_dev &d, const hr_thr &t, unsigned mask, uint32_t lane,
                                              uint64_t key, uint32_t kind, unsigned &kb0, unsigned &kb1)
{
    unsigned peers = 1u << lane;
    kb0 = kb1 = 0;
    if (hr__opt<ABL>(d, HR_OPT_NO_COALESCE)) return peers;
    if (mask == 0xffffffffu) {
        const unsigned long long prev = __shfl_up_sync(mask, key, 1);
        if (__all_sync(mask, lane == 0 || key > prev)) return peers;
    }
    peers = __match_any_sync(mask, key);
    if ((ONLINE || d.tile_log2 < 5u) && __any_sync(mask, peers != (1u << lane))) {
        /* a fold needs one epoch: true in any program with uniform barriers (one SHFL +
         * VOTE to confirm); otherwise (online code, or warp tiles whose barriers move
         * the tiles' clocks apart) split the groups by epoch with a second MATCH */
        const uint32_t lo = (uint32_t)t.meta;
        if (!__all_sync(mask, lo == __shfl_sync(mask, lo, __ffs(mask) - 1))) {
            const unsigned same_epoch = __match_any_sync(mask, (unsigned long long)lo);
            if (peers & ~same_epoch) peers = 1u << lane;
        }
    }
    kb0 = __ballot_sync(mask, kind & 1u);
    kb1 = __ballot_sync(mask, (kind >> 1) & 1u);
    return peers;
}

/*
 * hr_check_lanes: every lane of `mask` calls it (convergent), `valid` says
 * whether this lane has an access.  `space` (0 global / 1 shared), `word` the
 * monitored word (global: absolute word; shared: index in the block's
 * instance), `kind` hr_kind.  Lanes of one call share bc/wc (uniform barriers);
 * ONLINE=true re-checks that with a second MATCH.  Returns after every lane's
 * access is committed (the final ballot is the warp's convergence point), so a
 * lane never runs ahead of an access folded into another lane (program order).
 */
/* Hybrid binned replay: an access to a binned bucket becomes one entry of its
 * (bucket, block) run, in this thread's program order and epoch order (the
 * position counter is the block's, in shared memory, and the row replay's real
 * barriers separate the epochs), checked later by hr_hy_replay_kernel. */
__device__ __forceinline__ bool hr__hy_append(const hr_dev &d, const hr_thr &t, uint64_t local, uint32_t kind)
{
    const uint32_t bk = (uint32_t)(local >> HR_HY_BITS);
    if (!((__ldg(d.hy_map + (bk >> 5)) >> (bk & 31u)) & 1u)) return false;
    const uint32_t lo = (uint32_t)t.meta & 0x0fffffffu;
    const uint32_t bc = lo >> d.wc_bits, wc = lo & ((1u << d.wc_bits) - 1u);
    const uint64_t e = ((local & ((1ull << HR_HY_BITS) - 1u)) << 42) | ((uint64_t)kind << 40) |
                       ((uint64_t)t.tid() << 13) | ((uint64_t)bc << 6) | (uint64_t)wc;
    unsigned long long slot;
    asm volatile("atom.shared.add.u64 %0, [%1], 1;" : "=l"(slot) : "r"(t.fsm + d.hy_sa_off + 8u * bk) : "memory");
    __stcs(reinterpret_cast<unsigned long long *>(d.hy_ent) + slot, (unsigned long long)e);
    return true;
}

__device__ __forceinline__ void hr__check_shared_row(const hr_dev &d, const hr_thr &t, uint32_t word, uint32_t kind);
__device__ __forceinline__ bool hr__shared_row_ok(const hr_thr &t, uint32_t op, uint32_t space, uint64_t word);

template <bool ONLINE, bool ABL = true>
__device__ __forceinline__ void hr_check_lanes(const hr_dev &d, const hr_thr &t, unsigned mask, bool valid,
                                               uint32_t space, uint64_t word, uint32_t kind)
{
    /* online, full warp of distinct shared words (a stencil / tile access): the specialised
     * shared row (no grouping needed, clocks per lane) */
    if (ONLINE && !ABL && mask == 0xffffffffu && hr__shared_row_ok(t, valid ? kind : 3u, space, word)) {
        hr__check_shared_row(d, t, (uint32_t)word, kind);
        return;
    }
    const uint32_t lane = hr__laneid();
    const bool is_shared = space != 0u;
    uint64_t local = 0;
    valid = valid && !(t.off & 1u) && hr__locate(d, t, space, word, local);
    if (!ONLINE && d.hy_map != nullptr) {
        if (valid && !is_shared) valid = !hr__hy_append(d, t, local, kind);
        if (!__any_sync(mask, valid)) return;                       /* a row of binned accesses only */
    }
    if (valid) HR_COUNT(d, 0);
    /* match key: 0 = no access on this lane (filtered lanes must not alias owned words) */
    const uint64_t key = valid ? ((local << 2) | (is_shared ? 2u : 0u) | 1u) : 0ull;
    unsigned kb0, kb1;
    const unsigned peers = hr__group<ONLINE, ABL>(d, t, mask, lane, key, kind, kb0, kb1);

    uint32_t ei = 0;
    if (valid && (__ffs(peers) - 1) == (int)lane) {
        const uint32_t sh_addr = hr__saddr<ABL>(d, t, local);
        unsigned long long *gp = d.gshadow + local;
        uint32_t fresh;
        const unsigned long long old = hr__first<ABL>(d, t, is_shared, sh_addr, gp, kind, fresh);
        ei = (peers == (1u << lane)) ? hr__commit_single<ABL>(d, t, is_shared, sh_addr, gp, old, fresh, kind)
                                     : hr__commit<ABL>(d, t, is_shared, sh_addr, gp, old, fresh, kind, lane, peers, kb0, kb1);
    }

    /* a9: warp-aggregated ring append; also the warp's convergence point */
    const unsigned em = __ballot_sync(mask, ei != 0u);
    if (em) {
        const uint32_t leader = __ffs(em) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(d.ring_tail, (unsigned)__popc(em));
        base = __shfl_sync(mask, base, leader);
        if (ei) hr__write_race(d, t, base + __popc(em & ((1u << lane) - 1u)), space, word, ei);
    }
}

/*
 * Shared-space row (a2-a9 specialised): every lane of the warp holds a
 * shared-space access to its own word (the caller checked: 32 valid lanes,
 * strictly increasing words < swords, t.off clear, a kernel without run-time
 * options).  Algorithm 1 exactly as in hr__commit_single, with what the
 * shared space fixes folded in (DESIGN.md §5 "shared row"):
 *   - the instance is this block's: the relation is never Global, so it is
 *     the XOR of the low 10 tid bits (Self / Warp / Block), and Bs needs only
 *     bc > oBC (an INIT word ignores relation and sync, any value indexes
 *     the same table row);
 *   - no epoch tag (the instance is zeroed at block start), no probe;
 *   - a7 is left out: its exits only save a write.  (ii)'s insensitive states
 *     (GREAD, GATOMIC, RACE_GRID) need another block and never occur; (iii),
 *     RACE_BLOCK under a non-Global relation, maps to itself for every label
 *     in the generated table, so committing it rewrites only the diagnostic
 *     tid and clocks; the unchanged word (i) rewrites the same value.  One
 *     CAS per access, no exit test on the common path.
 */
/* The racy lanes of a shared row that arrive together share one ring
 * reservation (warp-aggregated over __activemask); a full ring drops the
 * record into the block's shared spill count (hr__ring_drop_x).  Out of line:
 * the common path keeps no ring constants live. */
static __device__ __noinline__ void hr__emit_shared_x(hr_race *ring, unsigned int *tail, uint32_t ring_cap,
                                                      uint32_t kernel_id, uint32_t fsm_sa, uint32_t tid,
                                                      uint32_t word, uint32_t ei)
{
    const unsigned m = __activemask();
    const uint32_t lane = hr__laneid(), leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(tail, (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
    if (slot < ring_cap) {
        hr_race rr;
        rr.word = word;
        rr.block = tid >> 10;
        rr.kernel = kernel_id;
        rr.first_tid = tid;
        rr.space = (uint8_t)HR_SHARED;
        rr.scope = (uint8_t)((ei & 1u) ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
        rr.first_kind = (uint8_t)((ei >> 24) & 3u);
        rr.prev_state = (uint8_t)((ei >> 19) & 31u);
        ring[slot] = rr;
    } else {
        hr__ring_drop_x(tail, false, kernel_id, fsm_sa + HR_FSM_DROP_OFF, 1u);
    }
}

/* min(v, 1) as one VIMNMX (inline PTX: the compiler would otherwise turn it into a
 * compare and a select/add pair per term) */
__device__ __forceinline__ uint32_t hr__min1(uint32_t v)
{
    uint32_t r;
    asm("min.u32 %0, %1, 1;" : "=r"(r) : "r"(v));
    return r;
}

/* (wcb, wsh, tl) = d.wc_bits, d.wc_lsh, d.tile_log2, passed in so that a row loop
 * can keep them in registers instead of reloading them per row */
__device__ __forceinline__ void hr__check_shared_row_k(const hr_dev &d, const hr_thr &t, uint32_t word, uint32_t kind,
                                                       uint32_t wcb, uint32_t wsh, uint32_t tl)
{
    const uint32_t sa = t.sshadow + (word << 3);
    const uint32_t lo = (uint32_t)t.meta, tid_lo = (uint32_t)(t.meta >> HR_TID_SHIFT) & 1023u;
    const uint32_t kcol = t.fsm + (kind << 4);
    unsigned long long old = hr__ld_s(sa);
    uint32_t os, cur;
    bool done;
    HR_COUNT(d, 0);
    do {
        const uint32_t ohi = (uint32_t)(old >> 32);
        os = ohi >> (HR_STATE_SHIFT - 32);
        const uint32_t x = (tid_lo ^ ohi) & 1023u;
        /* checkSync by XOR: in a happens-before consistent commit order the stored
         * access of this block is never in a later block epoch (oBC <= BC), nor, in
         * this warp and block epoch, in a later warp epoch (oWC <= WC), so "advanced"
         * is "differs".  The two sync bits are set independently (bit 1: bc differs,
         * bit 0: wc differs); the table maps index 3 to Bs and Ws under a Block
         * relation to Us (fsm/generate.py), and an INIT word ignores the label.
         * Each 0/1 term as a min (one VIMNMX) so the index folds into LEA/IADD3. */
        const uint32_t dlo = (uint32_t)old ^ lo;
        const uint32_t idx = (os << 6) + (hr__min1(dlo >> wcb) << 3) + (hr__min1(dlo << wsh) << 2) +
                             hr__min1(x) + hr__min1(x >> tl);                 /* + rel: Self / Warp / Block */
        cur = hr__lds_u8(kcol + idx);
        /* no a7 exit: every access commits its word with one CAS.  Inside one block's
         * instance the relation is never Global, so a RACE_BLOCK word stays RACE_BLOCK
         * and rewriting it only refreshes the diagnostic tid and clocks (no second
         * record: the emit test below needs a state change) */
        const unsigned long long prev = hr__cas_s(sa, old, ((unsigned long long)cur << HR_STATE_SHIFT) | t.meta);
        done = prev == old;                                               /* a8 committed */
        if (!done) HR_COUNT(d, 1);
        old = prev;
    } while (!done);
    HR_COUNT(d, 3);
    /* a9: rare here, so no warp vote on the common path and the emit out of line */
    if (cur >= HR_RACE_BLOCK && cur != os)
        hr__emit_shared_x(d.ring, d.ring_tail, d.ring_cap, d.kernel_id, t.fsm, t.tid(), word,
                          HR_EI_EMIT | (kind << 24) | (os << 19) | (cur == HR_RACE_GRID ? 1u : 0u));
}

__device__ __forceinline__ void hr__check_shared_row(const hr_dev &d, const hr_thr &t, uint32_t word, uint32_t kind)
{
    hr__check_shared_row_k(d, t, word, kind, d.wc_bits, d.wc_lsh, d.tile_log2);
}

/* The test for hr__check_shared_row (warp-uniform result). */
__device__ __forceinline__ bool hr__shared_row_ok(const hr_thr &t, uint32_t op, uint32_t space, uint64_t word)
{
    const uint32_t w32 = (uint32_t)word, prevw = __shfl_up_sync(0xffffffffu, w32, 1);   /* word < swords < 2^32 */
    return __all_sync(0xffffffffu, op != 3u && space != 0u && word < t.swords && !(t.off & 3u) &&
                                       (hr__laneid() == 0u || w32 > prevw));
}

/* ---------------- online instrumentation API ---------------- */

/* Copy the FSM table into `smem_fsm` (HR_FSM_SMEM_BYTES, 16-B aligned), zero the
 * block's shared shadow instance, and __syncthreads.  Every thread of the block
 * must call it. */
__device__ __forceinline__ hr_thr hr_thread_begin(const hr_dev &d, unsigned char *smem_fsm,
                                                  unsigned long long *smem_shadow, uint32_t smem_words)
{
    const uint32_t nthr = blockDim.x * blockDim.y * blockDim.z;
    const uint32_t ltid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const uint4 *src = reinterpret_cast<const uint4 *>(d.fsm);
    uint4 *dst = reinterpret_cast<uint4 *>(smem_fsm);
    for (uint32_t i = ltid; i < HR_FSM_SMEM_BYTES / 16; i += nthr) dst[i] = src[i];
    const uint32_t n64 = (d.options & HR_OPT_SMEM32) ? (smem_words + 1u) / 2u : smem_words;
    for (uint32_t i = ltid; i < n64; i += nthr) smem_shadow[i] = 0ull;
    __syncthreads();
    hr_thr t;
    uint32_t block = d.block_base + blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const uint32_t tid = (block << 10) | ((ltid >> 5) << 5) | (ltid & 31u);
    t.meta = ((unsigned long long)tid << HR_TID_SHIFT) | ((unsigned long long)d.epoch_tag << 28);
    /* the two shared-space bases pass through a SHFL, which ptxas does not
     * rematerialise: they stay in registers instead of an S2R SR_CgaCtaId + LEA
     * chain before every check (every thread of the block is here) */
    const unsigned am = __activemask();
    t.sshadow = __shfl_sync(am, (uint32_t)__cvta_generic_to_shared(smem_shadow), __ffs(am) - 1);
    t.swords = smem_words;
    t.fsm = __shfl_sync(am, (uint32_t)__cvta_generic_to_shared(smem_fsm), __ffs(am) - 1);
    t.off = hr__thread_off(d, block, ltid >> 5);
    return t;
}

/* End of a block: if the full ring dropped a race record of
 * this block's shared instance, copy every RACE word of the instance into the
 * spill before the instance dies with the block (a9 overflow recovery).  Every
 * thread of the block must call it (it holds a __syncthreads) after its last
 * check; a kernel that cannot (an early return) must keep the ring large
 * enough, else hr_report returns HR_E_INCOMPLETE. */
__device__ __forceinline__ void hr_thread_end(const hr_dev &d, const hr_thr &t)
{
    if (t.swords == 0u) return;                   /* block-uniform */
    __syncthreads();
    uint32_t drops;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(drops) : "r"(t.fsm + HR_FSM_DROP_OFF) : "memory");
    if (drops == 0u) return;                      /* block-uniform: read after the barrier */
    const uint32_t nthr = blockDim.x * blockDim.y * blockDim.z;
    const uint32_t ltid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const uint32_t nscan = (nthr & 31u) ? min(nthr, 32u) : nthr;   /* whole warps, or one (partial) warp */
    if (ltid < nscan) hr__spill_instance(d, t.sshadow, t.swords, t.tid() >> 10, ltid, nscan);
    if (ltid == 0u) atomicSub(&d.ovf[1], drops);
}

/* OPTS = true reads the ablation options and HR_OPT_SMEM32 at run time; a
 * kernel instantiated with OPTS = false must only run on a ctx without them. */
template <bool OPTS = true>
__device__ __forceinline__ void hr_check_read(const hr_dev &d, hr_thr &t, hr_space space, uint64_t word)
{
    hr_check_lanes<true, OPTS>(d, t, __activemask(), true, (uint32_t)space, word, HR_READ);
}

template <bool OPTS = true>
__device__ __forceinline__ void hr_check_write(const hr_dev &d, hr_thr &t, hr_space space, uint64_t word)
{
    hr_check_lanes<true, OPTS>(d, t, __activemask(), true, (uint32_t)space, word, HR_WRITE);
}

template <bool OPTS = true>
__device__ __forceinline__ void hr_check_atomic(const hr_dev &d, hr_thr &t, hr_space space, uint64_t word)
{
    hr_check_lanes<true, OPTS>(d, t, __activemask(), true, (uint32_t)space, word, HR_ATOMIC);
}

/* __syncthreads(); ++bc.  Overflow: saturate,
 * latch HR_F_CLOCK_OVERFLOW, stop checking this thread's accesses. */
__device__ __forceinline__ void hr_syncthreads(const hr_dev &d, hr_thr &t)
{
    __syncthreads();
    /* the clock word's bits [31:28] hold the epoch tag under HR_OPT_LAZY_RESET */
    const uint32_t lo = d.epoch_tag ? ((uint32_t)t.meta & 0x0fffffffu) : (uint32_t)t.meta;
    if ((lo >> d.wc_bits) >= d.bc_max) { t.off |= 1u; hr__set_flag(d, HR_F_CLOCK_OVERFLOW); }
    else t.meta += 1ull << d.wc_bits;
}

/* Do the lanes of `held` (a __syncwarp record on those lanes of a row) form whole
 * warp tiles of 2^tl lanes within the active `lane_mask`?  Convergent call. */
__device__ __forceinline__ bool hr__tile_aligned(unsigned held, unsigned lane_mask, uint32_t tl)
{
    const uint32_t T = 1u << tl, lane = hr__laneid();
    const unsigned tm = (T >= 32u ? 0xffffffffu : (((1u << T) - 1u) << (lane & ~(T - 1u)))) & lane_mask;
    const unsigned h = held & tm;
    return __all_sync(0xffffffffu, h == 0u || h == tm);
}

/* __syncwarp(mask) for a sub-warp mask ("takes a mask argument";
 * PAPER.md:1054 lists sub-warp support as future work).  A thread's scalar warp
 * clock cannot say that only some lanes synchronised, so (reading R8 in
 * DESIGN.md, the same rule as the replay and the oracle) the call synchronises
 * the lanes for real but adds NO happens-before edge: no clock moves and
 * HR_F_MODEL_VIOLATION is latched.  Races the masked barrier would order are
 * therefore still reported (sound, not precise).  A full mask is hr_syncwarp. */
__device__ __forceinline__ void hr_syncwarp_mask(const hr_dev &d, hr_thr &t, unsigned mask);

/* __syncwarp(); ++wc (full warp; see hr_syncwarp_mask for sub-warp masks). */
__device__ __forceinline__ void hr_syncwarp(const hr_dev &d, hr_thr &t)
{
    __syncwarp();
    if (((uint32_t)t.meta & d.wc_max) >= d.wc_max) { t.off |= 1u; hr__set_flag(d, HR_F_CLOCK_OVERFLOW); }
    else t.meta += 1ull;
}

__device__ __forceinline__ void hr_syncwarp_mask(const hr_dev &d, hr_thr &t, unsigned mask)
{
    if (mask == 0xffffffffu && d.tile_log2 >= 5u) { hr_syncwarp(d, t); return; }
    __syncwarp(mask);
    /* a kernel with warp tiles (hr_set_warp_tile): a mask of whole tiles holding this
     * lane is that tile's barrier: this lane's warp-tile clock advances (exact) */
    bool whole = d.tile_log2 < 5u;
    if (whole) {
        const uint32_t T = 1u << d.tile_log2, lane = hr__laneid();
        const unsigned tm = T >= 32u ? 0xffffffffu : (((1u << T) - 1u) << (lane & ~(T - 1u)));
        whole = (mask & tm) == tm;
    }
    if (whole) {
        if (((uint32_t)t.meta & d.wc_max) >= d.wc_max) { t.off |= 1u; hr__set_flag(d, HR_F_CLOCK_OVERFLOW); }
        else t.meta += 1ull;
    } else if (hr__laneid() == (uint32_t)(__ffs(mask) - 1)) {
        hr__set_flag(d, HR_F_MODEL_VIOLATION);
    }
}

/* The lanes of `held` take a warp-tile barrier (replay of a tile row): a real
 * __syncwarp for the converged warp, and each holding lane's clock advances. */
__device__ __forceinline__ void hr_syncwarp_lanes(const hr_dev &d, hr_thr &t, unsigned held)
{
    __syncwarp();
    if (!((held >> hr__laneid()) & 1u)) return;
    if (((uint32_t)t.meta & d.wc_max) >= d.wc_max) { t.off |= 1u; hr__set_flag(d, HR_F_CLOCK_OVERFLOW); }
    else t.meta += 1ull;
}

#endif /* HR_DEVICE_CUH_ */
