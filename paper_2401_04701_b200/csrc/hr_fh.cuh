/*
 * hr_fh.cuh — finite-history BASELINE detector, not the method.
 *
 * The design HiRace is compared against: FastTrack-style access records with a
 * bounded history.  "iGUARD is only able to store a single prior accessor"
 * (PAPER.md:277); it "relies on a single prior reader and a single writer"
 * in "16 bytes of metadata per monitored word".
 * Per word: one writer record (last write or atomic) and one reader record
 * (last read), 64 bits each = 16 bytes, updated with ATOMG/ATOMS.CAS.128.
 *
 *   record = valid:1 | kind:2 | tid:27 | bc:16 | wc:16        (62 bits used)
 *   lo = writer, hi = reader; bit 63 of hi = "already reported" (one report per word)
 *
 * Access N races with a held record P iff distinct threads, conflicting kinds
 * and P, N unordered (the same happens-before predicate as the oracle,
 * evaluated only against what the two slots still hold).  A read replaces the
 * reader record, a write/atomic the writer record: an earlier reader evicted
 * by a later one is forgotten, which is how Listing 4's race is missed
 * (PAPER.md:960-966).  Sound (every report is a real racing pair), incomplete.
 *
 * Replayed row by row with the same barrier handling as hr_replay_kernel.
 */
#ifndef HR_FH_CUH_
#define HR_FH_CUH_

#include "hr_device.cuh"
#include "hr_records.cuh"

typedef unsigned __int128 hr_u128;

#define HR_FH_VALID (1ull << 61)
#define HR_FH_REPORTED (1ull << 63)

__device__ __forceinline__ uint64_t hr_fh__rec(uint32_t kind, uint32_t tid, unsigned long long meta_lo)
{
    return HR_FH_VALID | ((uint64_t)kind << 59) | ((uint64_t)(tid & 0x7ffffffu) << 32) | (meta_lo & 0xffffffffull);
}

__device__ __forceinline__ bool hr_fh__conflict(uint32_t a, uint32_t b)
{
    return !((a == HR_READ && b == HR_READ) || (a == HR_ATOMIC && b == HR_ATOMIC));
}

/* unordered (and distinct threads): 0 = ordered/same thread, 1 = same block, 2 = other block */
__device__ __forceinline__ uint32_t hr_fh__unordered(uint64_t p, uint32_t tid, uint32_t lo, uint32_t wc_bits,
                                                     uint32_t tl)
{
    const uint32_t ptid = (uint32_t)(p >> 32) & 0x7ffffffu;
    if (ptid == tid) return 0;
    if ((ptid >> 10) != (tid >> 10)) return 2;
    const uint32_t plo = (uint32_t)p;
    if ((plo >> wc_bits) != (lo >> wc_bits)) return 0;                 /* a __syncthreads separates */
    if (((ptid ^ tid) & 1023u) >> tl) return 1;                        /* same block epoch, other warp (tile) */
    const uint32_t m = (1u << wc_bits) - 1u;
    return (plo & m) == (lo & m) ? 1u : 0u;                           /* same warp: warp epoch */
}

__device__ __forceinline__ hr_u128 hr_fh__cas(hr_u128 *p, hr_u128 cmp, hr_u128 val)
{
    return atomicCAS(p, cmp, val);
}

/* one access; returns the race scope to report (0 none, 1 block, 2 grid) */
__device__ __forceinline__ uint32_t hr_fh__access(const hr_dev &d, const hr_thr &t, hr_u128 *p, uint32_t kind)
{
    const uint32_t lo = (uint32_t)t.meta;
    const uint64_t mine = hr_fh__rec(kind, t.tid(), t.meta);
    hr_u128 old = *(volatile hr_u128 *)p;
    while (true) {
        const uint64_t wr = (uint64_t)old, rd = (uint64_t)(old >> 64);
        uint32_t scope = 0;
        if (!(rd & HR_FH_REPORTED)) {
            if ((wr & HR_FH_VALID) && hr_fh__conflict(kind, (uint32_t)(wr >> 59) & 3u)) {
                const uint32_t u = hr_fh__unordered(wr, t.tid(), lo, d.wc_bits, d.tile_log2);
                scope = u > scope ? u : scope;
            }
            if ((rd & HR_FH_VALID) && kind != HR_READ) {
                const uint32_t u = hr_fh__unordered(rd, t.tid(), lo, d.wc_bits, d.tile_log2);
                scope = u > scope ? u : scope;
            }
        }
        uint64_t nwr = wr, nrd = rd;
        if (kind == HR_READ) nrd = (rd & HR_FH_REPORTED) | mine;
        else nwr = mine;
        if (scope) nrd |= HR_FH_REPORTED;
        const hr_u128 nw = ((hr_u128)nrd << 64) | nwr;
        if (nw == old) return 0;
        const hr_u128 prev = hr_fh__cas(p, old, nw);
        if (prev == old) return scope;
        old = prev;
    }
}

template <typename SRC>
__global__ void __launch_bounds__(1024, 1) hr_fh_replay_kernel(hr_dev d, SRC src, const uint64_t *__restrict__ woff,
                                                               uint32_t warps, uint32_t lanes, uint32_t smem_words)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    hr_u128 *sshadow = reinterpret_cast<hr_u128 *>(hr_smem + HR_FSM_SMEM_BYTES);
    /* hr_thread_begin zero-fills 8-byte words: pass twice the count for 16-byte records */
    hr_thr t = hr_thread_begin(d, hr_smem, reinterpret_cast<unsigned long long *>(sshadow), 2 * smem_words);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * warps + warp;
    const uint64_t r0 = woff[gw], r1 = woff[gw + 1], n = r1 - r0;
    const unsigned lane_mask = lanes >= 32u ? 0xffffffffu : ((1u << lanes) - 1u);
    const bool active = lane < lanes;
    hr_u128 *gsh = reinterpret_cast<hr_u128 *>(d.gshadow);
    for (uint64_t i = 0; i < n; i++) {
        const uint64_t x = active ? src.row(r0 + i, lane) : HR_NOP_REC;
        const uint32_t op = (uint32_t)(x >> 62);
        const uint64_t w = x & HR_WORD_MASK;
        const unsigned ctrl = __ballot_sync(0xffffffffu, op == 3u && w != 0u);
        if (ctrl) {
            const unsigned bst = __ballot_sync(0xffffffffu, op == 3u && w == 1u);
            const unsigned bsw = __ballot_sync(0xffffffffu, op == 3u && w == 2u);
            const bool mixed = hr__ctrl_mixed(x, ctrl);
            bool partial_ws = bsw != 0u && bsw == ctrl && ctrl != lane_mask && !mixed;
            const bool tile_ws = partial_ws && d.tile_log2 < 5u && hr__tile_aligned(bsw, lane_mask, d.tile_log2);
            partial_ws = partial_ws && !tile_ws;
            if (lane == 0) {
                if (partial_ws) hr__set_flag(d, HR_F_MODEL_VIOLATION);           /* sub-warp mask: no edge */
                else if (!tile_ws && (ctrl != lane_mask || mixed)) hr__set_flag(d, HR_F_BARRIER_DIVERGENCE);
                if ((bst | bsw) != ctrl) hr__set_flag(d, HR_F_MODEL_VIOLATION);
            }
            if (partial_ws) continue;
            if (tile_ws) { hr_syncwarp_lanes(d, t, bsw); continue; }
            if (bst) hr_syncthreads(d, t);
            else if (bsw) hr_syncwarp(d, t);
            continue;
        }
        const uint32_t space = (uint32_t)(x >> 61) & 1u;
        uint64_t local = 0;
        uint32_t scope = 0;
        if (op != 3u && !(t.off & 1u) && hr__locate(d, t, space, w, local))
            scope = space ? hr_fh__access(d, t, sshadow + local, op) : hr_fh__access(d, t, gsh + local, op);
        const unsigned em = __ballot_sync(0xffffffffu, scope != 0u);
        if (em) {
            const uint32_t leader = __ffs(em) - 1;
            uint32_t b = 0;
            if (lane == leader) b = atomicAdd(d.ring_tail, (unsigned)__popc(em));
            b = __shfl_sync(0xffffffffu, b, leader);
            if (scope)
                hr__write_race<true>(d, t, b + __popc(em & ((1u << lane) - 1u)), space, w,
                               HR_EI_EMIT | (lane << 26) | (op << 24) | (scope == 2u ? 1u : 0u));
        }
    }
}

#endif /* HR_FH_CUH_ */
