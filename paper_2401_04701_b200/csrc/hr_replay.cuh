/*
 * hr_replay.cuh — trace replay kernel (SURVEY §8(a) a1, §3 call stack 3).
 *
 * One CUDA block per simulated block, one CUDA warp per simulated warp, lane l
 * of a row = simulated lane l.  Each thread walks its simulated thread's
 * records in program order and runs the device check (hr_device.cuh) on each
 * access; __syncthreads / __syncwarp records execute REAL barriers and advance
 * BC / WC, so every per-word commit order is consistent with the trace's
 * happens-before order (program order, block and warp epochs; kernels are
 * separate launches).  Replaying is therefore the paper's online check
 * driven by a synthetic access stream instead of a user
 * kernel's own loads and stores.
 *
 * Record rows are streamed with ld.global.cs (read once, evict-first) and
 * prefetched two rows ahead so the record latency is off the shadow-update
 * critical path.
 */
#ifndef HR_REPLAY_CUH_
#define HR_REPLAY_CUH_

#include "hr_device.cuh"

#define HR_NOP_REC (3ull << 62)

__device__ __forceinline__ uint64_t hr__ld_rec(const uint64_t *p)
{
    return __ldcs(reinterpret_cast<const unsigned long long *>(p));
}

/* minBlocks = 2 at 1024 threads caps registers at 32: 64 resident warps per SM
 * whatever the simulated block size (occupancy is the latency-hiding lever). */
#ifndef HR_MIN_BLOCKS
#define HR_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(1024, HR_MIN_BLOCKS) hr_replay_kernel(hr_dev d, const uint64_t *__restrict__ rec,
                                                            const uint64_t *__restrict__ woff, uint32_t warps,
                                                            uint32_t lanes, uint32_t smem_words)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    unsigned long long *sshadow = reinterpret_cast<unsigned long long *>(hr_smem + HR_FSM_SMEM_BYTES);
    hr_thr t = hr_thread_begin(d, hr_smem, sshadow, smem_words);

    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * warps + warp;
    const uint64_t r0 = woff[gw], r1 = woff[gw + 1];
    const unsigned lane_mask = lanes >= 32u ? 0xffffffffu : ((1u << lanes) - 1u);
    const bool active = lane < lanes;
    const uint64_t *p = rec + r0 * 32 + lane;
    const uint64_t n = r1 - r0;

    /* two-deep record prefetch (shift register, body not unrolled) */
    uint64_t x1 = (active && n > 0) ? hr__ld_rec(p) : HR_NOP_REC;
    uint64_t x2 = (active && n > 1) ? hr__ld_rec(p + 32) : HR_NOP_REC;
    for (uint64_t i = 0; i < n; i++) {
        const uint64_t x = x1;
        x1 = x2;
        x2 = (active && i + 2 < n) ? hr__ld_rec(p + 32 * (i + 2)) : HR_NOP_REC;
        const uint32_t op = (uint32_t)(x >> 62);
        const uint64_t w = x & HR_WORD_MASK;
        const unsigned ctrl = __ballot_sync(0xffffffffu, op == 3u && w != 0u);
        if (ctrl) {                                               /* warp-uniform */
            const unsigned bst = __ballot_sync(0xffffffffu, op == 3u && w == 1u);
            if ((bst && bst != lane_mask) || (ctrl != lane_mask))
                if (lane == 0) hr__set_flag(d, HR_F_BARRIER_DIVERGENCE);
            if (bst) hr_syncthreads(d, t);
            else hr_syncwarp(d, t);
            if (ctrl & ~bst) {
                const unsigned bsw = __ballot_sync(0xffffffffu, op == 3u && w == 2u);
                if (bsw != ctrl && lane == 0) hr__set_flag(d, HR_F_MODEL_VIOLATION);
            }
            continue;
        }
        hr_check_lanes<false>(d, t, 0xffffffffu, op != 3u, (uint32_t)(x >> 61) & 1u, w, op);
    }
}

/* Overflow fallback / cross-check: every RACE word of the (local) global
 * shadow becomes one record in `out` (a9 "end-of-kernel shadow scan"). */
__global__ void hr_scan_kernel(const unsigned long long *__restrict__ sh, uint64_t n_local, uint64_t gbase,
                               uint32_t shard_rank, uint32_t shard_log2, uint32_t kernel_id, hr_race *out,
                               unsigned int *count, uint32_t cap)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local;
         i += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long v = sh[i];
        uint32_t st = (uint32_t)(v >> HR_STATE_SHIFT);
        if (st >= HR_RACE_BLOCK) {
            uint32_t slot = atomicAdd(count, 1u);
            if (slot < cap) {
                uint64_t gran_local = i >> 9;
                uint64_t g = (((gran_local << shard_log2) | shard_rank) << 9) | (i & 511u);
                hr_race r;
                r.word = gbase + g;
                r.block = 0xffffffffu;
                r.kernel = kernel_id;
                r.first_tid = (uint32_t)(v >> HR_TID_SHIFT) & 0x7ffffffu;
                r.space = HR_GLOBAL;
                r.scope = (uint8_t)(st == HR_RACE_GRID ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
                r.first_kind = 0xff;
                r.prev_state = 0xff;
                out[slot] = r;
            }
        }
    }
}

#endif /* HR_REPLAY_CUH_ */
