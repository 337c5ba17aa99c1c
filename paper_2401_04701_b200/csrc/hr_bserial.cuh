/*
 * hr_bserial.cuh — block-serial pooled replay for sparse traces (address
 * shards).  Not a step of the paper's method: a schedule of the replay.
 *
 * One CUDA warp replays a whole simulated block, epoch by epoch: for each
 * block epoch (the rows between two __syncthreads records) it walks the rows
 * of simulated warp 0, then warp 1, ..., pooling the accesses it owns, and
 * only then advances the block clock.  Within one block epoch, accesses of
 * different simulated warps are unordered by happens-before (they share bc,
 * and only __syncthreads orders warps), and one simulated warp's accesses
 * stay in program order, so the record order of every pool is a linear
 * extension of happens-before restricted to the pool.  A
 * __syncwarp record closes the pool and advances that warp's clock, so a
 * pool never spans a warp epoch either.  The same-word fold labels
 * consecutive members Self / Warp / Block with sync Us; the first member is
 * labelled against the stored word with its own tid and clocks (Algorithm 1,
 * PAPER.md:694-711).
 *
 * What it buys on an address shard: no __syncthreads between CUDA warps (the
 * block's barriers are implicit in the walk), and a pool collects the owned
 * accesses of all the block's warps, so it is full instead of flushed per
 * warp at every barrier.
 */
#ifndef HR_BSERIAL_CUH_
#define HR_BSERIAL_CUH_

#include "hr_device.cuh"
#include "hr_records.cuh"
#include "hr_replay.cuh"

#define HR_BS_WARPS 8u                 /* simulated blocks (CUDA warps) per CTA */

/* per CUDA warp: pool (32 records + 32 u16 tags), warp clocks and row cursors
 * of up to 32 simulated warps */
struct hr_bs_smem {
    uint64_t rec[32];
    uint16_t tag[32];                  /* simulated warp << 5 | lane */
    uint32_t wc[32];
    uint32_t cur[32];
    uint32_t drops;                    /* shared race records of this block the full ring dropped */
    uint32_t pad[3];
};

__device__ __forceinline__ uint32_t hr__lds_u32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t hr__lds_u16(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

/* emit word of this kernel: [31] emit [30:21] tag [20:19] kind [18:14] prev state [0] grid */
template <bool ABL>
__device__ __forceinline__ void hr__check_bpool(const hr_dev &d, const hr_thr &t, uint32_t ps, uint32_t n,
                                                uint32_t blk, uint32_t lo_base)
{
    const uint32_t rec_sa = ps, tag_sa = ps + 256u, wc_sa = ps + 320u;
    const uint32_t lane = hr__laneid();
    uint64_t x = HR_NOP_REC;
    if (lane < n) asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x) : "r"(rec_sa + 8u * lane) : "memory");
    const uint32_t space = (uint32_t)(x >> 61) & 1u;
    const uint32_t kind = (uint32_t)(x >> 62);
    const uint64_t word = x & HR_WORD_MASK;
    uint64_t local = 0;
    const bool valid = lane < n && hr__locate(d, t, space, word, local);
    const uint64_t key = valid ? ((local << 2) | (space << 1) | 1u) : 0ull;
    unsigned kb0, kb1;
    const unsigned peers = hr__group<false, ABL>(d, t, 0xffffffffu, lane, key, kind, kb0, kb1);
    uint32_t ei = 0;
    if (valid && (__ffs(peers) - 1) == (int)lane) {
        const bool sh = space != 0u;
        const uint32_t sa = hr__saddr<ABL>(d, t, local);
        unsigned long long *gp = d.gshadow + local;
        const bool fastexit = !hr__opt<ABL>(d, HR_OPT_NO_FASTEXIT);
        const uint32_t base = blk << 10;
        const uint32_t tag0 = hr__lds_u16(tag_sa + 2u * lane);
        const uint32_t lo0 = lo_base | hr__lds_u32(wc_sa + 4u * (tag0 >> 5));
        const uint32_t last = 31u - __clz(peers);
        const uint32_t tagl = hr__lds_u16(tag_sa + 2u * last);
        const unsigned long long nmeta = ((unsigned long long)(base | tagl) << HR_TID_SHIFT) |
                                         (lo_base | hr__lds_u32(wc_sa + 4u * (tagl >> 5)));
        uint32_t fresh;
        unsigned long long old = hr__first<ABL>(d, t, sh, sa, gp, kind, fresh);
        while (true) {
            const unsigned long long lv = sh ? old : hr__live(d, old);
            const uint32_t os = (uint32_t)(lv >> HR_STATE_SHIFT);
            const uint32_t rel = hr__rel(base | tag0, (uint32_t)(lv >> HR_TID_SHIFT) & 0x7ffffffu, d.tile_log2);
            const uint32_t sync = hr__sync(rel, lo0, (uint32_t)lv, d.wc_bits);
            uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | (kind << 4) | (sync << 2) | rel));
            uint32_t rinfo = (cur >= HR_RACE_BLOCK && cur != os)
                                 ? (HR_EI_EMIT | (tag0 << 21) | (kind << 19) | (os << 14)) : 0u;
            uint32_t prev = tag0;
            unsigned r = peers & ~(1u << lane);
            while (r) {
                const uint32_t j = __ffs(r) - 1;
                r &= r - 1;
                uint64_t xj;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(xj) : "r"(rec_sa + 8u * j) : "memory");
                const uint32_t tj = hr__lds_u16(tag_sa + 2u * j);
                const uint32_t kj = (uint32_t)(xj >> 62);
                const uint32_t rj = hr__rel(tj, prev, d.tile_log2); /* Self / Warp / Block, same epochs: Us */
                const uint32_t nx = hr__lds_u8(t.fsm + ((cur << 6) | (kj << 4) | rj));
                if (nx >= HR_RACE_BLOCK && cur < HR_RACE_BLOCK && !rinfo)
                    rinfo = HR_EI_EMIT | (tj << 21) | (kj << 19) | (cur << 14);
                cur = nx;
                prev = tj;
            }
            const unsigned long long nw = ((unsigned long long)cur << HR_STATE_SHIFT) | nmeta;
            if (fastexit && cur == os && fresh != HR_OLD_GUESS) {
                const uint32_t f = hr__lds_u8(t.fsm + HR_FSM_BYTES + os);
                if ((f & HR_FLAG_INSENSITIVE) || ((f & HR_FLAG_BLOCK_ONLY) && rel != 3u && fresh == HR_OLD_FRESH))
                    break;
            }
            if (nw == old) {
                if (fresh == HR_OLD_FRESH) break;
                if (fresh == HR_OLD_PROBE) { old = hr__ld_g(gp); fresh = HR_OLD_FRESH; continue; }
            }
            const unsigned long long prv = sh ? hr__cas_sh<ABL>(d, t, sa, old, nw) : hr__cas_g(gp, old, nw);
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
        const uint32_t leader = __ffs(em) - 1;
        uint32_t b = 0;
        if (lane == leader) b = atomicAdd(d.ring_tail, (unsigned)__popc(em));
        b = __shfl_sync(0xffffffffu, b, leader);
        if (ei) {
            const uint32_t slot = b + __popc(em & ((1u << lane) - 1u));
            if (slot < d.ring_cap) {
                hr_race rr;
                rr.word = word;
                rr.block = space ? blk : 0xffffffffu;
                rr.kernel = d.kernel_id;
                rr.first_tid = (blk << 10) | ((ei >> 21) & 1023u);
                rr.space = (uint8_t)space;
                rr.scope = (uint8_t)((ei & 1u) ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
                rr.first_kind = (uint8_t)((ei >> 19) & 3u);
                rr.prev_state = (uint8_t)((ei >> 14) & 31u);
                d.ring[slot] = rr;
            } else {
                hr__ring_drop(d, ps + (uint32_t)offsetof(hr_bs_smem, drops), space);
            }
        }
    }
}

/* grid: ceil(blocks / HR_BS_WARPS) CTAs of HR_BS_WARPS warps; dynamic smem:
 * FSM table, HR_BS_WARPS hr_bs_smem, HR_BS_WARPS shared-shadow instances */
template <bool ABL>
__global__ void __launch_bounds__(HR_BS_WARPS * 32, 64 / HR_BS_WARPS) hr_replay_bserial_kernel(
    hr_dev d, const uint64_t *__restrict__ rec, const uint64_t *__restrict__ woff, uint32_t n_blocks, uint32_t warps,
    uint32_t lanes, uint32_t smem_words)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    const uint32_t hw = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(hr_smem);
    /* FSM table for the CTA; this warp's pool / clocks / cursors and shared instance */
    for (uint32_t i = threadIdx.x; i < HR_FSM_SMEM_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(hr_smem)[i] = reinterpret_cast<const uint4 *>(d.fsm)[i];
    const uint32_t ps = smem0 + HR_FSM_SMEM_BYTES + hw * (uint32_t)sizeof(hr_bs_smem);
    const uint32_t sw_bytes = (d.options & HR_OPT_SMEM32) ? ((smem_words * 4u + 7u) & ~7u) : smem_words * 8u;
    const uint32_t sh0 = HR_FSM_SMEM_BYTES + HR_BS_WARPS * (uint32_t)sizeof(hr_bs_smem) + hw * sw_bytes;
    unsigned long long *sshadow = reinterpret_cast<unsigned long long *>(hr_smem + sh0);
    for (uint32_t i = lane; i < sw_bytes / 8u; i += 32u) sshadow[i] = 0ull;
    hr_bs_smem *me = reinterpret_cast<hr_bs_smem *>(hr_smem + HR_FSM_SMEM_BYTES + hw * sizeof(hr_bs_smem));
    me->wc[lane] = 0u;
    me->cur[lane] = 0u;
    if (lane == 0) me->drops = 0u;
    __syncthreads();                                   /* the only CTA barrier: setup */
    const uint32_t sb = blockIdx.x * HR_BS_WARPS + hw; /* simulated block of this warp (launch-relative) */
    if (sb >= n_blocks) return;
    const uint32_t blk = d.block_base + sb;
    hr_thr t;
    t.meta = (unsigned long long)(blk << 10) << HR_TID_SHIFT;
    t.sshadow = smem0 + sh0;
    t.swords = smem_words;
    t.fsm = smem0;
    t.off = hr__thread_off(d, blk, 0u) & 2u;   /* representatives: per simulated warp below */
    const uint64_t *wo = woff + (uint64_t)sb * warps;
    const uint32_t tag_hi = d.epoch_tag << 28;
    const bool active = lane < lanes;
    const unsigned lane_mask = lanes >= 32u ? 0xffffffffu : ((1u << lanes) - 1u);
    uint32_t bc = 0, wc_off = 0;                       /* wc_off: simulated warps stopped by wc overflow */
    bool bc_off = false;
    uint32_t cnt = 0;
    auto flush = [&]() {
        if (cnt) {
            __syncwarp();
            hr__check_bpool<ABL>(d, t, ps, cnt, blk, tag_hi | (bc << d.wc_bits));
            __syncwarp();
            cnt = 0;
        }
    };
    bool more = true;
    while (more) {
        more = false;
        for (uint32_t sw = 0; sw < warps; sw++) {
            const uint64_t r0 = wo[sw];
            const uint32_t n = (uint32_t)(wo[sw + 1] - r0);
            uint32_t pos = me->cur[sw];
            if (pos >= n) continue;
            const uint64_t *rp = rec + r0 * 32u + lane;
            uint64_t nxt = active ? __ldcs(reinterpret_cast<const unsigned long long *>(rp + (uint64_t)pos * 32u))
                                  : HR_NOP_REC;
            while (pos < n) {
                const uint64_t x = nxt;
                pos++;
                if (pos < n)
                    nxt = active ? __ldcs(reinterpret_cast<const unsigned long long *>(rp + (uint64_t)pos * 32u))
                                 : HR_NOP_REC;
                const uint32_t op = (uint32_t)(x >> 62);
                const uint64_t w = x & HR_WORD_MASK;
                const unsigned ctrl = __ballot_sync(0xffffffffu, op == 3u && w != 0u);
                if (ctrl) {
                    /* as hr__barrier_row: divergence and mixed barrier kinds are flagged */
                    const unsigned bst = __ballot_sync(0xffffffffu, op == 3u && w == 1u);
                    const unsigned bsw = __ballot_sync(0xffffffffu, op == 3u && w == 2u);
                    const bool mixed = hr__ctrl_mixed(x, ctrl);
                    const bool partial_ws = bsw != 0u && bsw == ctrl && ctrl != lane_mask && !mixed;
                    if (lane == 0) {
                        if (partial_ws) hr__set_flag(d, HR_F_MODEL_VIOLATION);   /* sub-warp mask: no edge */
                        else if (ctrl != lane_mask || mixed) hr__set_flag(d, HR_F_BARRIER_DIVERGENCE);
                        if ((bst | bsw) != ctrl) hr__set_flag(d, HR_F_MODEL_VIOLATION);
                    }
                    if (partial_ws) continue;
                    if (bst) break;                              /* this warp's block epoch ends */
                    if (!bsw) continue;                          /* undefined control code: no barrier */
                    /* __syncwarp of simulated warp sw: close the pool, advance its clock */
                    flush();
                    const uint32_t wc = me->wc[sw];
                    if (wc >= d.wc_max) {
                        wc_off |= 1u << sw;
                        if (lane == 0) hr__set_flag(d, HR_F_CLOCK_OVERFLOW);
                    } else if (lane == 0) {
                        me->wc[sw] = wc + 1u;
                    }
                    __syncwarp();
                    continue;
                }
                const bool v = !bc_off && !((wc_off >> sw) & 1u) && !(hr__thread_off(d, blk, sw) & 1u) &&
                               hr__pool_owned(d, t, x, 0u, 0u);
                const unsigned vm = __ballot_sync(0xffffffffu, v);
                const uint32_t k = __popc(vm);
                if (!k) continue;
                const uint32_t slot = cnt + __popc(vm & ((1u << lane) - 1u));
                const uint32_t tag = (sw << 5) | lane;
                if (v && slot < 32u) {
                    asm volatile("st.shared.u64 [%0], %1;" ::"r"(ps + 8u * slot), "l"(x) : "memory");
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(ps + 256u + 2u * slot), "h"((unsigned short)tag)
                                 : "memory");
                }
                if (cnt + k >= 32u) {
                    __syncwarp();
                    hr__check_bpool<ABL>(d, t, ps, 32u, blk, tag_hi | (bc << d.wc_bits));
                    __syncwarp();
                    if (v && slot >= 32u) {
                        asm volatile("st.shared.u64 [%0], %1;" ::"r"(ps + 8u * (slot - 32u)), "l"(x) : "memory");
                        asm volatile("st.shared.u16 [%0], %1;" ::"r"(ps + 256u + 2u * (slot - 32u)),
                                     "h"((unsigned short)tag)
                                     : "memory");
                    }
                    cnt = cnt + k - 32u;
                } else {
                    cnt += k;
                }
            }
            if (lane == 0) me->cur[sw] = pos;
            __syncwarp();
            if (pos < n) more = true;
        }
        /* block barrier: every warp of the block reached it (or ran out) */
        flush();
        if (more) {
            if (bc >= d.bc_max) {
                bc_off = true;
                if (lane == 0) hr__set_flag(d, HR_F_CLOCK_OVERFLOW);
            } else {
                bc++;
            }
        }
    }
    /* a12 + a9: the block's shared instance dies here; spill it if the ring dropped one of its races */
    __syncwarp();
    const uint32_t drops = *(volatile uint32_t *)&me->drops;
    if (drops) {
        hr__spill_instance(d, t.sshadow, smem_words, blk, lane, 32u);
        if (lane == 0) atomicSub(&d.ovf[1], drops);
    }
}

__host__ __forceinline__ size_t hr_bserial_smem(uint32_t smem_words, bool smem32)
{
    const size_t sw_bytes = smem32 ? ((smem_words * 4u + 7u) & ~7u) : (size_t)smem_words * 8u;
    return HR_FSM_SMEM_BYTES + HR_BS_WARPS * (sizeof(hr_bs_smem) + sw_bytes);
}

#endif /* HR_BSERIAL_CUH_ */
