/*
 * hr_hybrid.cuh — hybrid binned replay (HR_OPT_BINNED; DESIGN.md §5 "hybrid
 * binned replay").  Not a step of the paper's method: a schedule of the replay
 * for kernels whose global accesses scatter over a shadow far larger than L2
 * (C5: 40% uniform random reads over 16 GiB), where random DRAM read-modify-
 * writes, not the check, set the time.
 *
 * The check is unchanged: Algorithm 1 per access, one atomicCAS on the packed
 * 64-bit shadow word.  Only WHEN an access is checked
 * changes.  Words are independent FSMs, so each word's
 * commit order only has to stay a linear extension of happens-before.
 *
 *   choose  a sample of the blocks (1 in 64) counts, per 2^HR_HY_BITS-word
 *           shadow bucket, the accesses and how many arrive scattered (at
 *           most 4 lanes of a row in the bucket).  A bucket whose accesses
 *           are mostly scattered and numerous is BINNED; the others
 *           (coalesced own-row rows, hot sets that live in L2) stay with the
 *           row replay.  Every word belongs to one bucket, so each word is
 *           checked by exactly one of the two.
 *   count   one CTA per simulated block counts its accesses to each binned
 *           bucket: the length of its (bucket, block) run.
 *   row     the normal row replay, with real barriers; an access to a binned
 *           bucket becomes an entry of its (bucket, block) run (hr__hy_append)
 *           at the block's next position: a thread's entries follow its
 *           program order, and epochs are separated by the barriers, so each
 *           run is in happens-before order.
 *   replay  a persistent grid checks the runs bucket by bucket (the SMs work
 *           in one or two 32 MB buckets at a time, whose shadow is streamed
 *           into L2 ahead), each run by one warp in order, 32 entries per
 *           pool; same-word entries of a pool are folded in entry order with
 *           their own (tid, bc, wc) labels.  Runs of different blocks are
 *           unordered.
 *
 * Used only when the count is exact (no clock can overflow, no warp tiles)
 * and the clocks fit an entry (bc <= 127, wc <= 63); otherwise the host
 * replays the kernel row by row.
 */
#ifndef HR_HYBRID_CUH_
#define HR_HYBRID_CUH_

#include "hr_device.cuh"
#include "hr_records.cuh"

#define HR_HY_MAXBK 1024u
#define HR_HY_ROWS 8u                 /* rows loaded per batch by the count walk (ILP) */

/* The count walk, one CTA per simulated block (SAMPLE: every stride-th block).
 * SAMPLE: per bucket, accesses and scattered accesses (at most 4 lanes of a row
 * in the bucket) into stat [2 * nbk] — the binning decision is a heuristic, so
 * a sample suffices.  Otherwise: the block's accesses to each binned bucket (map)
 * into counts [nbk * nb + 1] (u64, bucket-major: run (bk, b) at bk * nb + b;
 * exact: the row replay appends exactly these), and clk [2] = the most
 * __syncthreads / __syncwarp rows of a warp. */
template <bool SAMPLE, typename SRC>
__global__ void hr_hy_count_kernel(hr_dev d, SRC src, const uint64_t *__restrict__ woff, uint32_t warps, uint32_t lanes,
                                   uint32_t nbk, uint32_t nb, uint32_t stride, const uint32_t *__restrict__ map,
                                   unsigned long long *__restrict__ cnt, unsigned long long *__restrict__ stat,
                                   unsigned int *__restrict__ clk)
{
    extern __shared__ uint32_t hy_sm[];                           /* [nbk] accesses, [nbk] scattered */
    for (uint32_t i = threadIdx.x; i < (SAMPLE ? 2u : 1u) * nbk; i += blockDim.x) hy_sm[i] = 0u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5, cta = SAMPLE ? blockIdx.x * stride : blockIdx.x;
    const uint32_t block = d.block_base + cta;
    const bool rep = !(hr__thread_off(d, block, w) & 1u);
    const bool active = lane < lanes;
    const uint64_t r0 = woff[(uint64_t)cta * warps + w], r1 = woff[(uint64_t)cta * warps + w + 1];
    uint32_t nbar = 0, nws = 0;
    for (uint64_t r = r0; r < r1; r += HR_HY_ROWS) {
        uint64_t xs[HR_HY_ROWS];
#pragma unroll
        for (uint32_t j = 0; j < HR_HY_ROWS; j++) xs[j] = (active && r + j < r1) ? src.row(r + j, lane) : HR_NOP_REC;
#pragma unroll
        for (uint32_t j = 0; j < HR_HY_ROWS; j++) {
            const uint64_t x = xs[j];
            const uint32_t op = (uint32_t)(x >> 62);
            const uint64_t wd = x & HR_WORD_MASK;
            /* a row holding any control record is a barrier row: the row replay checks
             * none of its accesses (hr__barrier_row) */
            if (__any_sync(0xffffffffu, op == 3u && wd != 0u)) {
                if (!SAMPLE) {
                    nbar += __any_sync(0xffffffffu, op == 3u && wd == 1u) ? 1u : 0u;
                    nws += __any_sync(0xffffffffu, op == 3u && wd == 2u) ? 1u : 0u;
                }
                continue;
            }
            bool v = rep && op != 3u && !((x >> 61) & 1u);
            uint32_t bk = 0;
            if (v) {
                const uint64_t g = wd - d.gbase;
                v = wd >= d.gbase && g < d.gwords;
                if (v) {
                    const uint64_t gran = g >> d.gran_log2;
                    const uint64_t local = ((gran >> d.shard_log2) << d.gran_log2) | (g & ((1ull << d.gran_log2) - 1u));
                    v = d.owned_only || hr_shard_owner(gran, d.shard_log2) == d.shard_rank;
                    bk = (uint32_t)(local >> HR_HY_BITS);
                    if (!SAMPLE) v = v && ((__ldg(map + (bk >> 5)) >> (bk & 31u)) & 1u);
                }
            }
            if (SAMPLE) {
                const unsigned grp = __match_any_sync(0xffffffffu, v ? bk : 0xffffffffu);
                if (v && (__ffs(grp) - 1) == (int)lane) {
                    const uint32_t n = __popc(grp);
                    atomicAdd(&hy_sm[bk], n);
                    if (n <= 4u) atomicAdd(&hy_sm[nbk + bk], n);
                }
            } else if (v) {
                atomicAdd(&hy_sm[bk], 1u);
            }
        }
    }
    if (!SAMPLE && lane == 0) {
        atomicMax(&clk[0], nbar);
        atomicMax(&clk[1], nws);
    }
    __syncthreads();
    for (uint32_t bk = threadIdx.x; bk < nbk; bk += blockDim.x) {
        const uint32_t n = hy_sm[bk];
        if (SAMPLE) {
            if (n) {
                atomicAdd(&stat[2u * bk], (unsigned long long)n);
                atomicAdd(&stat[2u * bk + 1u], (unsigned long long)hy_sm[nbk + bk]);
            }
        } else {
            cnt[(uint64_t)bk * nb + cta] = n;
        }
    }
}

/* binned buckets: at least min_acc accesses, at least half of them scattered */
__global__ void hr_hy_decide_kernel(const unsigned long long *__restrict__ stat, uint32_t nbk, uint32_t *__restrict__ map,
                                    unsigned long long min_acc)
{
    const uint32_t bk = blockIdx.x * blockDim.x + threadIdx.x;
    const bool binned = bk < nbk && stat[2u * bk] >= min_acc && 2ull * stat[2u * bk + 1u] >= stat[2u * bk];
    const unsigned m = __ballot_sync(0xffffffffu, binned);
    if ((threadIdx.x & 31u) == 0u && bk < nbk) map[bk >> 5] = m;
}

/* One pool of up to 32 entries: a3 grouping by word, the leader folds its
 * group in entry order with each member's own (tid, bc, wc) label, a7/a8 as
 * hr__commit, a9.  pool_sa: this warp's 32 x (tid u32, lo u32, kind u32) staging. */
__device__ __forceinline__ void hr__hy_check(const hr_dev &d, const hr_thr &t, bool valid, uint64_t local, uint32_t tid,
                                             uint32_t lo, uint32_t kind, uint32_t pool_sa)
{
    const uint32_t lane = hr__laneid();
    const unsigned long long key = valid ? ((local << 1) | 1u) : 0ull;
    unsigned peers = 1u << lane;
    const unsigned long long prevk = __shfl_up_sync(0xffffffffu, key, 1);
    if (!__all_sync(0xffffffffu, lane == 0 || key > prevk)) {
        peers = __match_any_sync(0xffffffffu, key);
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(pool_sa + 8u * lane), "r"(tid), "r"(lo) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(pool_sa + 256u + 4u * lane), "r"(kind) : "memory");
        __syncwarp();
    }
    uint32_t ei = 0;
    if (valid && (__ffs(peers) - 1) == (int)lane) {
        unsigned long long *gp = d.gshadow + local;
        uint32_t tid_l = tid, lo_l = lo;
        if (peers != (1u << lane)) {
            const uint32_t last = 31u - __clz(peers);
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(tid_l), "=r"(lo_l) : "r"(pool_sa + 8u * last) : "memory");
        }
        const unsigned long long nmeta = ((unsigned long long)tid_l << HR_TID_SHIFT) | lo_l;
        uint32_t fresh;
        unsigned long long old = hr__first<false>(d, t, false, 0u, gp, kind, fresh);
        while (true) {
            const unsigned long long lv = hr__live(d, old);
            const uint32_t os = (uint32_t)(lv >> HR_STATE_SHIFT);
            const uint32_t rel = hr__rel(tid, (uint32_t)(lv >> HR_TID_SHIFT) & 0x7ffffffu, d.tile_log2);
            const uint32_t sync = hr__sync(rel, lo, (uint32_t)lv, d.wc_bits);
            uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | (kind << 4) | (sync << 2) | rel));
            uint32_t rinfo =
                (cur >= HR_RACE_BLOCK && cur != os) ? (HR_EI_EMIT | (lane << 26) | (kind << 24) | (os << 19)) : 0u;
            uint32_t ptid = tid, plo = lo;
            bool anyg = rel == 3u;                /* a Global label anywhere in the fold */
            unsigned r = peers & ~(1u << lane);
            while (r) {
                const uint32_t j = __ffs(r) - 1;
                r &= r - 1;
                uint32_t tj, lj;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(tj), "=r"(lj) : "r"(pool_sa + 8u * j) : "memory");
                const uint32_t kj = hr__lds_u32(pool_sa + 256u + 4u * j);
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
            if (cur == os && fresh != HR_OLD_GUESS) {
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

/* Stream one bucket's shadow (2^HR_HY_BITS words = 32 MB) into L2: the warp's
 * lanes issue 64 KB bulk prefetches (cp.async.bulk.prefetch.L2), clipped to the
 * shadow's end. */
__device__ __forceinline__ void hr__hy_prefetch(const unsigned long long *p, const unsigned long long *end, uint32_t lane)
{
    const char *b = reinterpret_cast<const char *>(p), *e = reinterpret_cast<const char *>(end);
    for (uint32_t i = lane; i < ((8u << HR_HY_BITS) >> 16); i += 32u) {
        const char *a = b + ((size_t)i << 16);
        if (a >= e) break;
        const uint32_t n = (uint32_t)min((size_t)(e - a), (size_t)65536) & ~15u;
        if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    }
}

/* Persistent replay of the runs, bucket-major over the binned buckets only.  A
 * warp takes HR_HY_GRAB consecutive runs (runs are never split, so each is
 * checked by one warp in order) and checks their concatenated entries 32 at a
 * time.  The warp that takes a bucket's first runs streams the next
 * binned bucket's shadow into L2. */
#define HR_HY_WARPS 16u
#define HR_HY_GRAB 32u
#ifndef HR_HY_MINB
#define HR_HY_MINB 3
#endif
__global__ void __launch_bounds__(HR_HY_WARPS * 32, HR_HY_MINB) hr_hy_replay_kernel(
    hr_dev d, const unsigned long long *__restrict__ ent, const unsigned long long *__restrict__ off, uint32_t nb,
    uint32_t nbk, unsigned long long *__restrict__ next)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    for (uint32_t i = threadIdx.x; i < HR_FSM_SMEM_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(hr_smem)[i] = reinterpret_cast<const uint4 *>(d.fsm)[i];
    /* the binned buckets in order (from the map), and how many */
    uint16_t *bins = reinterpret_cast<uint16_t *>(hr_smem + ((HR_FSM_SMEM_BYTES + 15u) & ~15u));
    __shared__ uint32_t nbin_s;
    if (threadIdx.x < 32u) {
        uint32_t n = 0;
        for (uint32_t w0 = 0; w0 < nbk; w0 += 32u) {
            const uint32_t bk = w0 + threadIdx.x;
            const bool on = bk < nbk && ((d.hy_map[bk >> 5] >> (bk & 31u)) & 1u);
            const unsigned m = __ballot_sync(0xffffffffu, on);
            if (on) bins[n + __popc(m & ((1u << threadIdx.x) - 1u))] = (uint16_t)bk;
            n += __popc(m);
        }
        if (threadIdx.x == 0) nbin_s = n;
    }
    __syncthreads();
    const uint32_t nbin = nbin_s;
    /* virtual runs (binned bucket i, block b) at i * nbp + b, each bucket padded to whole
     * grabs so that a grab never crosses a bucket */
    const uint32_t nbp = (nb + HR_HY_GRAB - 1u) / HR_HY_GRAB * HR_HY_GRAB;
    const uint64_t nv = (uint64_t)nbin * nbp;
    const uint32_t lane = threadIdx.x & 31u;
    hr_thr t;
    t.meta = 0;
    t.sshadow = 0;
    t.swords = 0;
    t.fsm = (uint32_t)__cvta_generic_to_shared(hr_smem);
    t.off = 0;
    const uint32_t pool_sa = t.fsm + ((HR_FSM_SMEM_BYTES + 15u) & ~15u) + 2048u + (threadIdx.x >> 5) * 384u;
    const uint32_t tag_hi = d.epoch_tag << 28;
    /* grabs from one counter, in bucket order (measured: dealing them round-robin
     * over the warps was slower at 2^32 accesses, 128 vs 94.6 ms per step) */
    while (true) {
        unsigned long long v0 = 0;
        if (lane == 0) v0 = atomicAdd(next, (unsigned long long)HR_HY_GRAB);
        v0 = __shfl_sync(0xffffffffu, v0, 0);
        if (v0 >= nv) break;
        const uint32_t bi = (uint32_t)(v0 / nbp), b0 = (uint32_t)(v0 % nbp);
        if (b0 >= nb) continue;                                    /* padding */
        const uint32_t bk = bins[bi];
        /* runs [b0, b0 + n) of bucket bk */
        const uint32_t n = min(HR_HY_GRAB, nb - b0);
        const uint64_t sr = (uint64_t)bk * nb + b0;
        const uint64_t e0 = off[sr], e1 = off[sr + n];
        if (b0 == 0 && bi + 1u < nbin)
            hr__hy_prefetch(d.gshadow + ((uint64_t)bins[bi + 1u] << HR_HY_BITS), d.gshadow + d.glocal_words, lane);
        const uint64_t lbase = (uint64_t)bk << HR_HY_BITS;
        uint64_t xn = e0 + lane < e1 ? __ldcs(ent + e0 + lane) : 0ull;   /* next pool's entry, loaded ahead */
        for (uint64_t p = e0; p < e1; p += 32u) {
            const uint64_t e = p + lane;
            const bool valid = e < e1;
            const uint64_t x = xn;
            xn = e + 32u < e1 ? __ldcs(ent + e + 32u) : 0ull;
            const uint64_t local = lbase | (x >> 42);
            const uint32_t kind = (uint32_t)(x >> 40) & 3u;
            const uint32_t tid = (uint32_t)(x >> 13) & 0x7ffffffu;
            const uint32_t lo = tag_hi | ((((uint32_t)x >> 6) & 127u) << d.wc_bits) | ((uint32_t)x & 63u);
            hr__hy_check(d, t, valid, local, tid, lo, kind, pool_sa);
        }
    }
}

__host__ __forceinline__ size_t hr_hy_replay_smem(uint32_t nbk)
{
    (void)nbk;
    return ((HR_FSM_SMEM_BYTES + 15u) & ~15u) + 2048u + HR_HY_WARPS * 384u;
}

#endif /* HR_HYBRID_CUH_ */
