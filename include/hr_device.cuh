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
#define HR_FSM_SMEM_BYTES (HR_FSM_BYTES + 32)   /* table + per-state flags */
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
    unsigned int *flags;
    unsigned long long *counters; /* [0] checks [1] CAS retries [2] fast exits */
    const unsigned char *fsm;     /* HR_FSM_SMEM_BYTES in global memory */
    uint32_t ring_cap;
    uint32_t kernel_id;
    uint32_t shard_rank, shard_log2; /* owner(granule) = granule & (2^log2 - 1) */
    uint32_t wc_bits;             /* bc occupies [31:wc_bits], wc [wc_bits-1:0] */
    uint32_t bc_max, wc_max;
    uint32_t options;             /* HR_OPT_* */
};

/* Per-thread registers. */
struct hr_thr {
    uint32_t tid;                 /* block:17 | warp:5 | lane:5 */
    uint32_t bc, wc;              /* thread-private block / warp scalar clocks */
    unsigned long long meta;      /* tid<<32 | bc<<wc_bits | wc, refreshed at barriers */
    uint32_t sshadow;             /* shared-space address of this block's shadow instance */
    uint32_t swords;
    uint32_t fsm;                 /* shared-space address of the FSM table copy */
    uint32_t off;                 /* detection disabled (clock overflow) */
};

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
    asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(r) : "r"(a), "l"(cmp), "l"(val) : "memory");
    return r;
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

/* ---------------- labels ---------------- */

/* compareTids: Self 0, Warp 1, Block 2, Global 3 from the packed-tid XOR. */
__device__ __forceinline__ uint32_t hr__rel(uint32_t tid, uint32_t otid)
{
    uint32_t x = tid ^ otid;
    return (x != 0u) + (x >= 32u) + (x >= 1024u);
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

/* L1-cacheable probe (weak load): only used to take the insensitive-closure exit,
 * which is valid for any value observed during this kernel (a7). */
__device__ __forceinline__ unsigned long long hr__ld_g_l1(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

/* emit-info word (one register instead of a 24-byte record) */
#define HR_EI_EMIT 0x80000000u

/*
 * hr_check_lanes: every lane of `mask` calls it (convergent), `valid` says
 * whether this lane has an access.  `space` (0 global / 1 shared), `word` the
 * monitored word (global: absolute word; shared: index in the block's
 * instance), `kind` hr_kind.  Lanes of one call share bc/wc (uniform barriers);
 * ONLINE=true re-checks that with a second MATCH.  Returns after every lane's
 * access is committed (the final ballot is the warp's convergence point), so a
 * lane never runs ahead of an access folded into another lane (program order).
 *
 * First attempt (a4): global reads/writes speculate INIT and issue the CAS
 * directly (one round trip for a first touch; a failed CAS returns the current
 * word, which is the atomic read of Algorithm 1); atomics probe L1 first (hot
 * GATOMIC words exit without L2 traffic); shared words are read with ld.shared.
 */
template <bool ONLINE>
__device__ __forceinline__ void hr_check_lanes(const hr_dev &d, const hr_thr &t, unsigned mask, bool valid,
                                               uint32_t space, uint64_t word, uint32_t kind)
{
    const uint32_t lane = hr__laneid();
    valid = valid && !t.off;

    /* a2: shadow address (local index inside the shard) */
    const bool is_shared = space != 0u;
    uint64_t local = 0;
    if (valid) {
        if (is_shared) {
            if (word >= t.swords) { hr__set_flag(d, HR_F_UNMONITORED); valid = false; }
            if (((t.tid >> 10) & ((1u << d.shard_log2) - 1u)) != d.shard_rank) valid = false;
            local = word;
        } else {
            const uint64_t g = word - d.gbase;
            if (word < d.gbase || g >= d.gwords) { hr__set_flag(d, HR_F_UNMONITORED); valid = false; }
            const uint64_t gran = g >> 9;
            if (((uint32_t)gran & ((1u << d.shard_log2) - 1u)) != d.shard_rank) valid = false;
            local = ((gran >> d.shard_log2) << 9) | (g & 511u);
        }
    }
    /* match key: 0 = no access on this lane (filtered lanes must not alias owned words) */
    const uint64_t key = valid ? ((local << 2) | (is_shared ? 2u : 0u) | 1u) : 0ull;

    /* a3: same-address coalescing (skipped when the warp's words are consecutive) */
    unsigned peers = 1u << lane;
    unsigned kb0 = 0, kb1 = 0;
    if (!(d.options & HR_OPT_NO_COALESCE)) {
        const uint32_t first = __ffs(mask) - 1;
        const unsigned long long k0 = __shfl_sync(mask, key, first);
        const bool seq = !valid || key == k0 + ((unsigned long long)(lane - first) << 2);
        if (!__all_sync(mask, seq)) {
            peers = __match_any_sync(mask, key);
            if (ONLINE) {
                const unsigned same_epoch = __match_any_sync(mask, (unsigned long long)(uint32_t)t.meta);
                if (peers & ~same_epoch) peers = 1u << lane;
            }
            kb0 = __ballot_sync(mask, kind & 1u);
            kb1 = __ballot_sync(mask, (kind >> 1) & 1u);
        }
    }

    uint32_t ei = 0;   /* [31] emit [30:26] racing lane [25:24] its kind [23:19] prev state [0] grid */
    if (valid && (__ffs(peers) - 1) == (int)lane) {
        const uint32_t sh_addr = t.sshadow + (uint32_t)(local << 3);
        unsigned long long *gp = d.gshadow + local;
        const bool fastexit = !(d.options & HR_OPT_NO_FASTEXIT);
        const uint32_t last_lane = 31u - __clz(peers);
        const unsigned long long nmeta = (t.meta & ~(0x1full << HR_TID_SHIFT)) |
                                         ((unsigned long long)last_lane << HR_TID_SHIFT);
        /* 0: value is a guess (INIT); 1: weak L1 probe; 2: coherent (L2/SMEM or CAS return) */
        uint32_t fresh;
        unsigned long long old;
        if (is_shared) { old = hr__ld_s(sh_addr); fresh = 2; }
        else if (kind == HR_ATOMIC && fastexit) { old = hr__ld_g_l1(gp); fresh = 1; }
        else if (d.options & HR_OPT_NO_SPECULATE) { old = hr__ld_g(gp); fresh = 2; }
        else { old = 0ull; fresh = 0; }
        while (true) {
            const uint32_t os = (uint32_t)(old >> HR_STATE_SHIFT);
            const uint32_t rel = hr__rel(t.tid, (uint32_t)(old >> HR_TID_SHIFT) & 0x7ffffffu);
            const uint32_t sync = hr__sync(rel, (uint32_t)t.meta, (uint32_t)old, d.wc_bits);
            uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | (kind << 4) | (sync << 2) | rel));
            uint32_t rinfo = (cur >= HR_RACE_BLOCK && cur != os)
                                 ? (HR_EI_EMIT | (lane << 26) | (kind << 24) | (os << 19)) : 0u;
            /* fold the rest of the group: (kind_j, Us, Warp) in lane order */
            unsigned r = peers & ~(1u << lane);
            while (r) {
                const uint32_t j = __ffs(r) - 1;
                r &= r - 1;
                const uint32_t kj = ((kb0 >> j) & 1u) | (((kb1 >> j) & 1u) << 1);
                const uint32_t nx = hr__lds_u8(t.fsm + ((cur << 6) | (kj << 4) | 1u));
                if (nx >= HR_RACE_BLOCK && cur < HR_RACE_BLOCK && !rinfo)
                    rinfo = HR_EI_EMIT | (j << 26) | (kj << 24) | (cur << 19);
                cur = nx;
            }
            const unsigned long long nw = ((unsigned long long)cur << HR_STATE_SHIFT) | nmeta;
            if (fastexit && cur == os && fresh) {
                const uint32_t f = hr__lds_u8(t.fsm + HR_FSM_BYTES + os);
                if ((f & HR_FLAG_INSENSITIVE) || ((f & HR_FLAG_BLOCK_ONLY) && rel != 3u && fresh == 2))
                    break;                                                /* a7 (ii), (iii) */
            }
            if (nw == old && fresh == 2) break;                           /* a7 (i) */
            if (fresh == 1 && nw == old) { old = hr__ld_g(gp); fresh = 2; continue; }
            const unsigned long long prev = is_shared ? hr__cas_s(sh_addr, old, nw) : hr__cas_g(gp, old, nw);
            if (prev == old) {                                            /* a8 committed */
                if (rinfo) ei = rinfo | (cur == HR_RACE_GRID ? 1u : 0u);
                break;
            }
            old = prev;
            fresh = 2;
#ifdef HR_COUNTERS
            atomicAdd(&d.counters[1], 1ull);
#endif
        }
    }

    /* a9: warp-aggregated ring append; also the warp's convergence point */
    const unsigned em = __ballot_sync(mask, ei != 0u);
    if (em) {
        const uint32_t leader = __ffs(em) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(d.ring_tail, (unsigned)__popc(em));
        base = __shfl_sync(mask, base, leader);
        if (ei) {
            const uint32_t slot = base + __popc(em & ((1u << lane) - 1u));
            if (slot < d.ring_cap) {
                hr_race rr;
                rr.word = word;
                rr.block = is_shared ? (t.tid >> 10) : 0xffffffffu;
                rr.kernel = d.kernel_id;
                rr.first_tid = (t.tid & ~31u) | ((ei >> 26) & 31u);
                rr.space = (uint8_t)space;
                rr.scope = (uint8_t)((ei & 1u) ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
                rr.first_kind = (uint8_t)((ei >> 24) & 3u);
                rr.prev_state = (uint8_t)((ei >> 19) & 31u);
                d.ring[slot] = rr;
            } else {
                hr__set_flag(d, HR_F_RING_OVERFLOW);
            }
        }
    }
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
    for (uint32_t i = ltid; i < smem_words; i += nthr) smem_shadow[i] = 0ull;
    __syncthreads();
    hr_thr t;
    uint32_t block = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    t.tid = (block << 10) | ((ltid >> 5) << 5) | (ltid & 31u);
    t.bc = 0;
    t.wc = 0;
    t.meta = (unsigned long long)t.tid << HR_TID_SHIFT;
    t.sshadow = (uint32_t)__cvta_generic_to_shared(smem_shadow);
    t.swords = smem_words;
    t.fsm = (uint32_t)__cvta_generic_to_shared(smem_fsm);
    t.off = 0;
    return t;
}

__device__ __forceinline__ void hr__refresh_meta(const hr_dev &d, hr_thr &t)
{
    t.meta = ((unsigned long long)t.tid << HR_TID_SHIFT) |
             ((unsigned long long)t.bc << d.wc_bits) | (unsigned long long)t.wc;
}

__device__ __forceinline__ void hr_check_read(const hr_dev &d, hr_thr &t, hr_space space, uint64_t word)
{
    hr_check_lanes<true>(d, t, __activemask(), true, (uint32_t)space, word, HR_READ);
}

__device__ __forceinline__ void hr_check_write(const hr_dev &d, hr_thr &t, hr_space space, uint64_t word)
{
    hr_check_lanes<true>(d, t, __activemask(), true, (uint32_t)space, word, HR_WRITE);
}

__device__ __forceinline__ void hr_check_atomic(const hr_dev &d, hr_thr &t, hr_space space, uint64_t word)
{
    hr_check_lanes<true>(d, t, __activemask(), true, (uint32_t)space, word, HR_ATOMIC);
}

/* __syncthreads(); ++bc.  Overflow: saturate,
 * latch HR_F_CLOCK_OVERFLOW, stop checking this thread's accesses. */
__device__ __forceinline__ void hr_syncthreads(const hr_dev &d, hr_thr &t)
{
    __syncthreads();
    if (t.bc >= d.bc_max) { t.off = 1; hr__set_flag(d, HR_F_CLOCK_OVERFLOW); }
    else { t.bc++; hr__refresh_meta(d, t); }
}

/* __syncwarp(); ++wc (full warp only; sub-warp masks are future work). */
__device__ __forceinline__ void hr_syncwarp(const hr_dev &d, hr_thr &t)
{
    __syncwarp();
    if (t.wc >= d.wc_max) { t.off = 1; hr__set_flag(d, HR_F_CLOCK_OVERFLOW); }
    else { t.wc++; hr__refresh_meta(d, t); }
}

#endif /* HR_DEVICE_CUH_ */
