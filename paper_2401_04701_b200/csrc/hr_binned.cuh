/*
 * hr_binned.cuh — address-binned replay (DESIGN.md §5 "binned replay").  Not a
 * step of the paper's method: a schedule of the replay for kernels whose
 * global accesses scatter over a shadow far larger than L2 (C5: 40% uniform
 * random reads over 16 GiB), where the per-access random DRAM read-modify-
 * write, not the check, sets the time.
 *
 * The check itself is unchanged: Algorithm 1 per access, one atomicCAS on the
 * packed 64-bit shadow word.  What changes is WHEN each
 * access is checked.  Words are independent FSMs, so only
 * the per-word commit order must stay a linear extension of happens-before.
 *
 *   walk    one CUDA warp per simulated block walks the block epoch by epoch
 *           (the block-serial order of hr_bserial.cuh: every warp's rows up to
 *           the next __syncthreads, then the next epoch; __syncwarp rows
 *           advance that warp's clock) and appends each global access, with
 *           its thread and (bc, wc), to stream (bucket, block), bucket = the
 *           shadow address >> HR_BN_BITS (64 MB of shadow).  Walk order is a
 *           linear extension of happens-before inside the block (epochs in
 *           order, a warp's rows in program order; rows of one warp epoch are
 *           unordered), and blocks are unordered, so every stream is in HB
 *           order.  A count pass sizes the streams, a CUB scan places them
 *           bucket-major, a write pass fills them.
 *   replay  a persistent grid takes the streams in bucket-major order, so the
 *           SMs work on one or two buckets at a time and their 64 MB of
 *           shadow stays in the 126 MB L2: the random RMWs hit L2 instead of
 *           DRAM.  A warp checks 32 consecutive entries of its streams as one
 *           pool; same-word entries are folded in entry order with their own
 *           (tid, bc, wc) labels (hr__bn_check) and committed with one CAS.
 *           Streams of different blocks are unordered, so a pool may join the
 *           tail of one stream and the head of the next.
 *
 * Entry (u64): [63:41] word - bucket base (23 bits) | [40:39] kind |
 * [38:34] warp | [33:29] lane | [28:17] bc | [16:5] wc | [4:0] 0.
 * Used only for kernels without shared shadow and with bc, wc < 4096 (the
 * walk reports otherwise and the host falls back to the row replay).
 */
#ifndef HR_BINNED_CUH_
#define HR_BINNED_CUH_

#include "hr_device.cuh"
#include "hr_records.cuh"
#include "hr_replay.cuh"

#define HR_BN_BITS 23u                /* bucket = 2^23 shadow words = 64 MB */
#define HR_BN_MAXBK 2048u             /* buckets per launch (SMEM counters of the walk) */
#define HR_BN_WALK_WARPS 4u
#define HR_BN_CLOCK_MAX 4095u
#define HR_BN_ST_CANCEL 1u            /* status: clocks too wide for an entry: fall back */

__device__ __forceinline__ uint64_t hr__bn_entry(uint32_t off, uint32_t kind, uint32_t warp, uint32_t lane,
                                                 uint32_t bc, uint32_t wc)
{
    return ((uint64_t)off << 41) | ((uint64_t)kind << 39) | ((uint64_t)warp << 34) | ((uint64_t)lane << 29) |
           ((uint64_t)bc << 17) | ((uint64_t)wc << 5);
}

/* The block-serial walk (count pass: WRITE = false; write pass: WRITE = true).
 * cnt / off are indexed [bucket * n_blocks + block]. */
template <bool WRITE, typename SRC>
__global__ void __launch_bounds__(HR_BN_WALK_WARPS * 32) hr_bn_walk_kernel(
    hr_dev d, SRC src, const uint64_t *__restrict__ woff, uint32_t n_blocks, uint32_t warps, uint32_t lanes,
    uint32_t nbk, uint64_t *__restrict__ cnt, const uint64_t *__restrict__ off, uint64_t *__restrict__ out,
    unsigned int *__restrict__ status)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    const uint32_t hw = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t sb = blockIdx.x * HR_BN_WALK_WARPS + hw;    /* simulated block (launch-relative) */
    /* per CUDA warp: stream positions [nbk] (u64), then wc[32] and cur[32] of its simulated warps */
    uint64_t *pos = reinterpret_cast<uint64_t *>(hr_smem) + (size_t)hw * (nbk + 32u);
    uint32_t *wcs = reinterpret_cast<uint32_t *>(pos + nbk), *cur = wcs + 32;
    if (sb >= n_blocks) return;                                  /* warp-uniform */
    for (uint32_t b = lane; b < nbk; b += 32u) pos[b] = WRITE ? off[(uint64_t)b * n_blocks + sb] : 0ull;
    wcs[lane] = 0u;
    cur[lane] = 0u;
    __syncwarp();
    const uint32_t blk = d.block_base + sb;
    const uint64_t *wo = woff + (uint64_t)sb * warps;
    const bool active = lane < lanes;
    const unsigned lane_mask = lanes >= 32u ? 0xffffffffu : ((1u << lanes) - 1u);
    const uint32_t off_b = hr__thread_off(d, blk, 0u) & 2u;     /* shared instance shard bit (unused: no smem) */
    (void)off_b;
    uint32_t bc = 0, dead = 0;                                   /* dead: simulated warps past a clock limit */
    bool more = true;
    while (more) {
        more = false;
        for (uint32_t sw = 0; sw < warps; sw++) {
            const uint64_t r0 = wo[sw];
            const uint32_t n = (uint32_t)(wo[sw + 1] - r0);
            uint32_t p = cur[sw];
            if (p >= n) continue;
            const bool rep = !(hr__thread_off(d, blk, sw) & 1u);
            while (p < n) {
                const uint64_t x = active ? src.row(r0 + p, lane) : HR_NOP_REC;
                p++;
                const uint32_t op = (uint32_t)(x >> 62);
                const uint64_t w = x & HR_WORD_MASK;
                const unsigned ctrl = __ballot_sync(0xffffffffu, op == 3u && w != 0u);
                if (ctrl) {
                    /* as hr__barrier_row: flags, sub-warp and undefined codes are no barrier */
                    const unsigned bst = __ballot_sync(0xffffffffu, op == 3u && w == 1u);
                    const unsigned bsw = __ballot_sync(0xffffffffu, op == 3u && w == 2u);
                    const bool mixed = hr__ctrl_mixed(x, ctrl);
                    const bool partial_ws = bsw != 0u && bsw == ctrl && ctrl != lane_mask && !mixed;
                    if (!WRITE && lane == 0) {
                        if (partial_ws) hr__set_flag(d, HR_F_MODEL_VIOLATION);
                        else if (ctrl != lane_mask || mixed) hr__set_flag(d, HR_F_BARRIER_DIVERGENCE);
                        if ((bst | bsw) != ctrl) hr__set_flag(d, HR_F_MODEL_VIOLATION);
                    }
                    if (partial_ws) continue;
                    if (bst) break;                                    /* this warp's block epoch ends */
                    if (!bsw) continue;
                    /* __syncwarp of simulated warp sw (hr_syncwarp: saturate, stop, flag) */
                    const uint32_t wcv = wcs[sw];
                    __syncwarp();
                    if (wcv >= d.wc_max) {
                        dead |= 1u << sw;
                        if (!WRITE && lane == 0) hr__set_flag(d, HR_F_CLOCK_OVERFLOW);
                    } else {
                        if (wcv + 1u > HR_BN_CLOCK_MAX && !WRITE && lane == 0) atomicOr(status, HR_BN_ST_CANCEL);
                        if (lane == 0) wcs[sw] = wcv + 1u;
                    }
                    __syncwarp();
                    continue;
                }
                /* a12-a2: global accesses of checked threads this shard owns; shared ones
                 * have no instance (smem_words == 0): unmonitored, as hr__locate */
                const uint32_t wcv = wcs[sw];
                const bool live = rep && !((dead >> sw) & 1u);
                bool v = op != 3u && live;
                uint64_t local = 0;
                if (v) {
                    if ((x >> 61) & 1u) {
                        if (!WRITE) hr__set_flag(d, HR_F_UNMONITORED);
                        v = false;
                    } else {
                        const uint64_t g = w - d.gbase;
                        if (w < d.gbase || g >= d.gwords) {
                            if (!WRITE) hr__set_flag(d, HR_F_UNMONITORED);
                            v = false;
                        } else {
                            const uint64_t gran = g >> d.gran_log2;
                            local = ((gran >> d.shard_log2) << d.gran_log2) | (g & ((1ull << d.gran_log2) - 1u));
                            v = d.owned_only || hr_shard_owner(gran, d.shard_log2) == d.shard_rank;
                        }
                    }
                }
                const uint32_t bk = (uint32_t)(local >> HR_BN_BITS);
                const unsigned grp = __match_any_sync(0xffffffffu, v ? bk : 0xffffffffu);
                const uint32_t leader = __ffs(grp) - 1;
                uint64_t base = 0;
                if (v && lane == leader) {
                    base = pos[bk];
                    pos[bk] = base + __popc(grp);
                }
                base = __shfl_sync(0xffffffffu, base, leader);
                if (WRITE && v)
                    out[base + __popc(grp & ((1u << lane) - 1u))] =
                        hr__bn_entry((uint32_t)(local & ((1ull << HR_BN_BITS) - 1u)), op, sw, lane, bc, wcv);
                __syncwarp();
            }
            if (lane == 0) cur[sw] = p;
            __syncwarp();
            if (p < n) more = true;
        }
        if (more) {                                                    /* the block barrier (hr_syncthreads) */
            if (bc >= d.bc_max) {
                if (dead != 0xffffffffu && !WRITE && lane == 0) hr__set_flag(d, HR_F_CLOCK_OVERFLOW);
                dead = 0xffffffffu;                                     /* later checks skipped */
            } else {
                bc++;
                if (bc > HR_BN_CLOCK_MAX && !WRITE && lane == 0) atomicOr(status, HR_BN_ST_CANCEL);
            }
        }
    }
    if (!WRITE)
        for (uint32_t b = lane; b < nbk; b += 32u) cnt[(uint64_t)b * n_blocks + sb] = pos[b];
}

/* One pool of up to 32 entries (lane i: entry i) of the streams in
 * [e0, e0 + n): a3 grouping by word, the leader folds its group in entry order
 * with each member's own (tid, bc, wc) label, a7/a8 as hr__commit, a9. */
__device__ __forceinline__ void hr__bn_decode(uint64_t e, uint32_t blk, uint32_t tag_hi, uint32_t wc_bits,
                                              uint32_t &tid, uint32_t &lo, uint32_t &kind)
{
    kind = (uint32_t)(e >> 39) & 3u;
    tid = (blk << 10) | ((uint32_t)(e >> 29) & 1023u);
    lo = tag_hi | (((uint32_t)(e >> 17) & 4095u) << wc_bits) | ((uint32_t)(e >> 5) & 4095u);
}

/* pool_sa: this warp's 32 x (u64 entry, u32 block) staging in SMEM */
template <bool ABL>
__device__ __forceinline__ void hr__bn_check(const hr_dev &d, const hr_thr &t, uint64_t e, bool valid, uint32_t blk,
                                             uint64_t local_base, uint32_t pool_sa)
{
    const uint32_t lane = hr__laneid();
    const uint32_t tag_hi = d.epoch_tag << 28;
    uint32_t tid, lo, kind;
    hr__bn_decode(e, blk, tag_hi, d.wc_bits, tid, lo, kind);
    const uint64_t local = local_base + (e >> 41);
    const unsigned long long key = valid ? ((local << 1) | 1u) : 0ull;
    unsigned peers = 1u << lane;
    if (!hr__opt<ABL>(d, HR_OPT_NO_COALESCE)) {
        const unsigned long long prevk = __shfl_up_sync(0xffffffffu, key, 1);
        if (!__all_sync(0xffffffffu, lane == 0 || key > prevk)) {
            peers = __match_any_sync(0xffffffffu, key);
            /* stage the pool: the group leaders fold their members from SMEM */
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(pool_sa + 8u * lane), "l"(e) : "memory");
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(pool_sa + 256u + 4u * lane), "r"(blk) : "memory");
            __syncwarp();
        }
    }
    uint32_t ei = 0;
    if (valid && (__ffs(peers) - 1) == (int)lane) {
        unsigned long long *gp = d.gshadow + local;
        const bool fastexit = !hr__opt<ABL>(d, HR_OPT_NO_FASTEXIT);
        uint32_t tid_l = tid, lo_l = lo;
        if (peers != (1u << lane)) {
            const uint32_t last = 31u - __clz(peers);
            uint32_t kl;
            uint64_t el;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(el) : "r"(pool_sa + 8u * last) : "memory");
            hr__bn_decode(el, hr__lds_u32(pool_sa + 256u + 4u * last), tag_hi, d.wc_bits, tid_l, lo_l, kl);
        }
        const unsigned long long nmeta = ((unsigned long long)tid_l << HR_TID_SHIFT) | lo_l;
        uint32_t fresh;
        unsigned long long old = hr__first<ABL>(d, t, false, 0u, gp, kind, fresh);
        while (true) {
            const unsigned long long lv = hr__live(d, old);
            const uint32_t os = (uint32_t)(lv >> HR_STATE_SHIFT);
            const uint32_t rel = hr__rel(tid, (uint32_t)(lv >> HR_TID_SHIFT) & 0x7ffffffu, d.tile_log2);
            const uint32_t sync = hr__sync(rel, lo, (uint32_t)lv, d.wc_bits);
            uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | (kind << 4) | (sync << 2) | rel));
            uint32_t rinfo = (cur >= HR_RACE_BLOCK && cur != os) ? (HR_EI_EMIT | (lane << 26) | (kind << 24) | (os << 19))
                                                                 : 0u;
            uint32_t ptid = tid, plo = lo;
            bool anyg = rel == 3u;                /* a Global label anywhere in the fold */
            unsigned r = peers & ~(1u << lane);
            while (r) {
                const uint32_t j = __ffs(r) - 1;
                r &= r - 1;
                uint64_t ej;
                uint32_t tj, lj, kj;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ej) : "r"(pool_sa + 8u * j) : "memory");
                hr__bn_decode(ej, hr__lds_u32(pool_sa + 256u + 4u * j), tag_hi, d.wc_bits, tj, lj, kj);
                const uint32_t rj = hr__rel(tj, ptid, d.tile_log2);
                anyg = anyg || rj == 3u;
                const uint32_t sj = hr__sync(rj, lj, plo, d.wc_bits);
                const uint32_t nx = hr__lds_u8(t.fsm + ((cur << 6) | (kj << 4) | (sj << 2) | rj));
                /* entering RACE, or (a member from another block) RACE_BLOCK -> RACE_GRID */
                if (nx >= HR_RACE_BLOCK && nx != cur && !rinfo)
                    rinfo = HR_EI_EMIT | (j << 26) | (kj << 24) | (cur << 19);
                cur = nx;
                ptid = tj;
                plo = lj;
            }
            const unsigned long long nw = ((unsigned long long)cur << HR_STATE_SHIFT) | nmeta;
            if (fastexit && cur == os && fresh != HR_OLD_GUESS) {
                const uint32_t f = hr__lds_u8(t.fsm + HR_FSM_BYTES + os);
                /* (iii) needs every label of the fold non-Global: members of a pool can
                 * come from other blocks (a RACE_BLOCK word they touch becomes RACE_GRID) */
                if ((f & HR_FLAG_INSENSITIVE) || ((f & HR_FLAG_BLOCK_ONLY) && !anyg && fresh == HR_OLD_FRESH))
                    break;
            }
            if (nw == old) {
                if (fresh == HR_OLD_FRESH) break;
                if (fresh == HR_OLD_PROBE) { old = hr__ld_g(gp); fresh = HR_OLD_FRESH; continue; }
            }
            const unsigned long long prv = hr__cas_g(gp, old, nw);
            if (prv == old) {
                if (rinfo) ei = rinfo | (cur == HR_RACE_GRID ? 1u : 0u);
                break;
            }
            old = prv;
            fresh = HR_OLD_FRESH;
        }
    }
    const unsigned em = __ballot_sync(0xffffffffu, ei != 0u);
    if (em) {
        /* the racing access's lane holds its own entry: its tid and word */
        const uint32_t src = (ei >> 26) & 31u;
        const uint32_t rtid = __shfl_sync(0xffffffffu, tid, src);
        const unsigned long long rw = __shfl_sync(0xffffffffu, (unsigned long long)local, src);
        const uint32_t leader = __ffs(em) - 1;
        uint32_t b = 0;
        if (lane == leader) b = atomicAdd(d.ring_tail, (unsigned)__popc(em));
        b = __shfl_sync(0xffffffffu, b, leader);
        if (ei) {
            const uint32_t slot = b + __popc(em & ((1u << lane) - 1u));
            /* global word of the shard-local index (the inverse of hr__locate) */
            const uint64_t gran_local = rw >> d.gran_log2;
            const uint64_t gw = d.gbase + ((hr_shard_granule(gran_local, d.shard_rank, d.shard_log2) << d.gran_log2) |
                                           (rw & ((1ull << d.gran_log2) - 1u)));
            if (slot < d.ring_cap) {
                hr_race rr;
                rr.word = gw;
                rr.block = 0xffffffffu;
                rr.kernel = d.kernel_id;
                rr.first_tid = rtid;
                rr.space = HR_GLOBAL;
                rr.scope = (uint8_t)((ei & 1u) ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
                rr.first_kind = (uint8_t)((ei >> 24) & 3u);
                rr.prev_state = (uint8_t)((ei >> 19) & 31u);
                d.ring[slot] = rr;
            } else {
                hr__ring_drop(d, t.fsm + HR_FSM_DROP_OFF, 0u);
            }
        }
    }
}

/* Persistent replay of the streams, bucket-major: a warp takes the next
 * HR_BN_GRAB streams (whole streams, so no stream is split between warps)
 * and checks their concatenated entries 32 at a time. */
#define HR_BN_WARPS 16u
#define HR_BN_GRAB 4u
template <bool ABL>
__global__ void __launch_bounds__(HR_BN_WARPS * 32, 2) hr_bn_replay_kernel(
    hr_dev d, const uint64_t *__restrict__ ent, const uint64_t *__restrict__ off, uint32_t n_blocks, uint64_t nstreams,
    unsigned long long *__restrict__ next)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    for (uint32_t i = threadIdx.x; i < HR_FSM_SMEM_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(hr_smem)[i] = reinterpret_cast<const uint4 *>(d.fsm)[i];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    hr_thr t;
    t.meta = 0;
    t.sshadow = 0;
    t.swords = 0;
    t.fsm = (uint32_t)__cvta_generic_to_shared(hr_smem);
    t.off = 0;
    const uint32_t pool_sa = t.fsm + ((HR_FSM_SMEM_BYTES + 15u) & ~15u) + (threadIdx.x >> 5) * 384u;
    while (true) {
        unsigned long long s0 = 0;
        if (lane == 0) s0 = atomicAdd(next, (unsigned long long)HR_BN_GRAB);
        s0 = __shfl_sync(0xffffffffu, s0, 0);
        if (s0 >= nstreams) break;
        const uint32_t ns = (uint32_t)((nstreams - s0) < (uint64_t)HR_BN_GRAB ? (nstreams - s0) : (uint64_t)HR_BN_GRAB);
        /* streams [s0, s0 + ns): entries [off[s0], off[s0 + ns]); stream s = bucket * n_blocks + block */
        uint64_t bnd[HR_BN_GRAB + 1];
#pragma unroll
        for (uint32_t k = 0; k <= HR_BN_GRAB; k++) bnd[k] = off[s0 + min(k, ns)];
        const uint32_t blk0 = (uint32_t)(s0 % n_blocks), bk0 = (uint32_t)(s0 / n_blocks);
        for (uint64_t e0 = bnd[0]; e0 < bnd[ns]; e0 += 32u) {
            const uint64_t e = e0 + lane;
            const bool valid = e < bnd[ns];
            const uint64_t x = valid ? __ldcs(reinterpret_cast<const unsigned long long *>(ent + e)) : 0ull;
            uint32_t k = 0;                                     /* this lane's stream within the grab */
#pragma unroll
            for (uint32_t q = 1; q < HR_BN_GRAB; q++) k += (q < ns && e >= bnd[q]) ? 1u : 0u;
            uint32_t blk = blk0 + k, bk = bk0;
            if (blk >= n_blocks) { blk -= n_blocks; bk++; }
            hr__bn_check<ABL>(d, t, x, valid, d.block_base + blk, (uint64_t)bk << HR_BN_BITS, pool_sa);
        }
    }
}

__host__ __forceinline__ size_t hr_bn_replay_smem()
{
    return ((HR_FSM_SMEM_BYTES + 15u) & ~15u) + HR_BN_WARPS * 384u;
}

__host__ __forceinline__ size_t hr_bn_walk_smem(uint32_t nbk)
{
    return (size_t)HR_BN_WALK_WARPS * (nbk + 32u) * 8u;
}

#endif /* HR_BINNED_CUH_ */
