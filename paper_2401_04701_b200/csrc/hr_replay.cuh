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
 * Record rows reach each warp through a per-warp ring of TMA bulk copies
 * (cp.async.bulk on an mbarrier, hr_records.cuh) issued NB chunks ahead, so the
 * record latency is off the shadow-update critical path.
 */
#ifndef HR_REPLAY_CUH_
#define HR_REPLAY_CUH_

#include "hr_device.cuh"
#include "hr_records.cuh"


/*
 * Pooled replay (default).  A warp compacts the valid accesses of consecutive
 * non-barrier rows (NOP records skipped) into a 32-slot pool, one access per
 * lane, each tagged with its simulated lane, and checks the pool with one
 * collective step.  Record order inside a pool is happens-before consistent:
 * the rows share one epoch (barrier rows flush the pool), and for each
 * simulated thread record order is program order.  So each same-word group is
 * folded in record order — Algorithm 1 applied access by access, labels
 * computed between consecutive members — and committed with one CAS.  Dense
 * rows (32 valid accesses) are a pool by themselves; sparse rows (one active
 * lane walking a hub's adjacency list, shard-filtered rows) are packed 32 per
 * step instead of one.
 */
template <bool B> struct hr_bool { static constexpr bool value = B; };

/* a warp-uniform value the compiler keeps in a vector register (a SHFL result is
 * not provably uniform, so it is not re-read from the parameter bank in a loop) */
__device__ __forceinline__ uint32_t hr__reg(uint32_t v)
{
    return __shfl_sync(0xffffffffu, v, 0);
}

struct hr_pool_smem {
    uint64_t rec[32];       /* pooled records */
    uint8_t src[32];        /* simulated lane of each pooled record */
};

/* A pool as seen by the check: 32 record slots and their simulated lanes, as
 * shared-space addresses (a hr_pool_smem, or a staged row of a compacted
 * stream); 32-bit addresses keep the generic->shared conversion out of the loop. */
struct hr_entries {
    uint32_t rec;               /* 32 x u64 */
    uint32_t src;               /* 32 x u8 */
    __device__ __forceinline__ hr_entries(uint32_t r, uint32_t s) : rec(r), src(s) {}
    __device__ __forceinline__ uint64_t rec_at(uint32_t i) const
    {
        uint64_t v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(rec + 8u * i) : "memory");
        return v;
    }
    __device__ __forceinline__ uint32_t src_at(uint32_t i) const { return hr__lds_u8(src + i); }
    __device__ __forceinline__ void put(uint32_t i, uint64_t x, uint32_t lane) const
    {
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(rec + 8u * i), "l"(x) : "memory");
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(src + i), "r"(lane) : "memory");
    }
};

__device__ __forceinline__ hr_entries hr__pool_at(uint32_t pool_sa)
{
    return hr_entries(pool_sa, pool_sa + 32u * 8u);
}

/* fold + commit of one pooled access group (leader side) */
__device__ __forceinline__ uint32_t hr__pool_transition(const hr_dev &d, const hr_thr &t, unsigned long long old,
                                                        const hr_entries ps, uint32_t lane, unsigned peers,
                                                        uint32_t &rinfo, uint32_t &rel)
{
    const uint32_t base = t.tid() & ~31u;
    const uint32_t os = (uint32_t)(old >> HR_STATE_SHIFT);
    const uint32_t src0 = ps.src_at(lane);
    const uint32_t kind0 = (uint32_t)(ps.rec_at(lane) >> 62);
    rel = hr__rel(base | src0, (uint32_t)(old >> HR_TID_SHIFT) & 0x7ffffffu, d.tile_log2);
    const uint32_t sync = hr__sync(rel, (uint32_t)t.meta, (uint32_t)old, d.wc_bits);
    uint32_t cur = hr__lds_u8(t.fsm + ((os << 6) | (kind0 << 4) | (sync << 2) | rel));
    rinfo = (cur >= HR_RACE_BLOCK && cur != os) ? (HR_EI_EMIT | (src0 << 26) | (kind0 << 24) | (os << 19)) : 0u;
    uint32_t prev_src = src0;
    unsigned r = peers & ~(1u << lane);
    while (r) {
        const uint32_t j = __ffs(r) - 1;
        r &= r - 1;
        const uint32_t sj = ps.src_at(j);
        const uint32_t kj = (uint32_t)(ps.rec_at(j) >> 62);
        /* Self / Warp (same tile) / Block (another tile), same epochs: Us */
        const uint32_t rj = sj == prev_src ? 0u : (((sj ^ prev_src) >> d.tile_log2) ? 2u : 1u);
        const uint32_t nx = hr__lds_u8(t.fsm + ((cur << 6) | (kj << 4) | rj));
        if (nx >= HR_RACE_BLOCK && cur < HR_RACE_BLOCK && !rinfo)
            rinfo = HR_EI_EMIT | (sj << 26) | (kj << 24) | (cur << 19);
        cur = nx;
        prev_src = sj;
    }
    return cur;
}

/* Check the pool: lanes < n hold one access each (ps.rec[lane], ps.src[lane]). */
template <bool ABL>
__device__ __forceinline__ void hr__check_pool(const hr_dev &d, const hr_thr &t, const hr_entries ps, uint32_t n)
{
    const uint32_t lane = hr__laneid();
    const uint64_t x = lane < n ? ps.rec_at(lane) : HR_NOP_REC;
    const uint32_t space = (uint32_t)(x >> 61) & 1u;
    const uint32_t kind = (uint32_t)(x >> 62);
    const uint64_t word = x & HR_WORD_MASK;
    uint64_t local = 0;
    /* pooled entries passed only the cheap owner test (hr__pool_owned): the
     * region check (HR_F_UNMONITORED) and the shard-local index happen here */
    const bool valid = lane < n && hr__locate(d, t, space, word, local);
    if (valid) HR_COUNT(d, 0);
    const uint64_t key = valid ? ((local << 2) | (space << 1) | 1u) : 0ull;
    unsigned kb0, kb1;
    const unsigned peers = hr__group<false, ABL>(d, t, 0xffffffffu, lane, key, kind, kb0, kb1);
    uint32_t ei = 0;
    if (valid && (__ffs(peers) - 1) == (int)lane) {
        const bool sh = space != 0u;
        const uint32_t sa = hr__saddr<ABL>(d, t, local);
        unsigned long long *gp = d.gshadow + local;
        const bool fastexit = !hr__opt<ABL>(d, HR_OPT_NO_FASTEXIT);
        const uint32_t last = 31u - __clz(peers);
        const unsigned long long nmeta = (t.meta & ~(0x1full << HR_TID_SHIFT)) |
                                         ((unsigned long long)ps.src_at(last) << HR_TID_SHIFT);
        uint32_t fresh;
        unsigned long long old = hr__first<ABL>(d, t, sh, sa, gp, kind, fresh);
        while (true) {
            const unsigned long long lv = sh ? old : hr__live(d, old);
            const uint32_t os = (uint32_t)(lv >> HR_STATE_SHIFT);
            uint32_t rinfo, rel;
            const uint32_t cur = hr__pool_transition(d, t, lv, ps, lane, peers, rinfo, rel);
            const unsigned long long nw = ((unsigned long long)cur << HR_STATE_SHIFT) | nmeta;
            if (fastexit && cur == os && fresh != HR_OLD_GUESS) {
                const uint32_t f = hr__lds_u8(t.fsm + HR_FSM_BYTES + os);
                if ((f & HR_FLAG_INSENSITIVE) || ((f & HR_FLAG_BLOCK_ONLY) && rel != 3u && fresh == HR_OLD_FRESH)) {
                    HR_COUNT(d, 2);
                    break;
                }
            }
            if (nw == old) {
                if (fresh == HR_OLD_FRESH) { HR_COUNT(d, 2); break; }
                if (fresh == HR_OLD_PROBE) { old = hr__ld_g(gp); fresh = HR_OLD_FRESH; continue; }
            }
            const unsigned long long prv = sh ? hr__cas_sh<ABL>(d, t, sa, old, nw) : hr__cas_g(gp, old, nw);
            if (prv == old) {
                HR_COUNT(d, 3);
                if (rinfo) ei = rinfo | (cur == HR_RACE_GRID ? 1u : 0u);
                break;
            }
            HR_COUNT(d, 1);
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
        if (ei) hr__write_race(d, t, b + __popc(em & ((1u << lane) - 1u)), space, word, ei);
    }
}

/* A row holding control records (a10).  Uniform rows: __syncthreads advances
 * bc, __syncwarp wc; a control code the trace format does not define (word > 2)
 * is no barrier at all — HR_F_MODEL_VIOLATION, no clock moves (as the oracle,
 * oracle/hr_oracle.c materialize).  A __syncwarp record held by only some of
 * the warp's lanes is __syncwarp(mask) with a sub-warp mask:
 * HR_F_MODEL_VIOLATION and, conservatively, no happens-before edge (reading
 * R8: the races it would order are still reported).  Any other disagreement
 * is HR_F_BARRIER_DIVERGENCE (undefined in CUDA; racy set unspecified). */
__device__ __forceinline__ void hr__barrier_row(const hr_dev &d, hr_thr &t, uint64_t x, unsigned lane_mask)
{
    const uint32_t op = (uint32_t)(x >> 62);
    const uint64_t w = x & HR_WORD_MASK;
    /* the common row: every active lane holds a __syncthreads (inactive lanes hold
     * NOP), so nothing is mixed, divergent or undefined */
    const unsigned bst = __ballot_sync(0xffffffffu, op == 3u && w == 1u);
    if (bst == lane_mask) { hr_syncthreads(d, t); return; }
    const unsigned ctrl = __ballot_sync(0xffffffffu, op == 3u && w != 0u);
    const unsigned bsw = __ballot_sync(0xffffffffu, op == 3u && w == 2u);
    const bool mixed = hr__ctrl_mixed(x, ctrl);
    bool partial_ws = bsw != 0u && bsw == ctrl && ctrl != lane_mask && !mixed;
    /* a tile kernel: a __syncwarp row held by whole tiles is one barrier per tile (exact) */
    const bool tile_ws = partial_ws && d.tile_log2 < 5u && hr__tile_aligned(bsw, lane_mask, d.tile_log2);
    partial_ws = partial_ws && !tile_ws;
    const bool div = !tile_ws && (ctrl != lane_mask || mixed);
    if ((threadIdx.x & 31u) == 0) {
        if (partial_ws) hr__set_flag(d, HR_F_MODEL_VIOLATION);
        else if (div) hr__set_flag(d, HR_F_BARRIER_DIVERGENCE);
        if ((bst | bsw) != ctrl) hr__set_flag(d, HR_F_MODEL_VIOLATION);
    }
    if (partial_ws) return;
    if (bst) hr_syncthreads(d, t);
    else if (tile_ws) hr_syncwarp_lanes(d, t, bsw);
    else if (bsw) hr_syncwarp(d, t);
}

/* Helper warp of a word when a simulated warp is split over 2^split_log2 CUDA
 * warps (multiplicative hash of the trace word: adjacent and strided words
 * spread evenly; any fixed function of the word keeps each word on one helper). */
__device__ __forceinline__ uint32_t hr__helper_of(uint64_t word, uint32_t split_log2)
{
    return ((uint32_t)(word ^ (word >> 29)) * 0x9E3779B1u) >> (32u - split_log2);
}

/* Cheap pre-pool test of a record: an access of an enabled thread whose word
 * belongs to this shard and (split) this helper.  Region bounds and the
 * shard-local index are left to hr__check_pool's hr__locate, so a record in a
 * pool may still turn out unmonitored (flagged there, not checked). */
__device__ __forceinline__ bool hr__pool_owned(const hr_dev &d, const hr_thr &t, uint64_t x, uint32_t split_log2,
                                               uint32_t helper)
{
    const uint32_t op = (uint32_t)(x >> 62);
    const uint32_t sp = (uint32_t)(x >> 61) & 1u;
    const uint64_t w = x & HR_WORD_MASK;
    bool v = op != 3u && !(t.off & 1u);
    if (sp) v = v && !(t.off & 2u);
    else if (d.shard_log2 && !d.owned_only) {
        /* words outside the region go on to hr__locate on every shard, which flags them */
        const uint64_t g = w - d.gbase;
        const bool in = w >= d.gbase && g < d.gwords;
        v = v && (!in || hr_shard_owner(g >> d.gran_log2, d.shard_log2) == d.shard_rank);
    }
    if (split_log2) v = v && hr__helper_of(w, split_log2) == helper;
    return v;
}

/* Per-warp TMA staging ring of the replay kernels: NB chunk buffers of CH
 * rows.  The 32-register kernels run 64 warps/SM, so 2 x 4 rows (2 KiB of u64
 * rows per warp); the 64-register kernels run at most 32: 2 x 8 rows (the
 * depth measured indifferent on C4; longer chunks halve the per-chunk work). */
#ifndef HR_STAGE_NB_WIDE
#define HR_STAGE_NB_WIDE 2u
#endif
#ifndef HR_STAGE_NB_ROW
#define HR_STAGE_NB_ROW 2u
#endif
#ifndef HR_WIDE_C32_CH
/* C3 (wide kernel, C32): 16-row chunks at 64 registers 0.226 ms; 8-row chunks at
 * 64 / 48 / 40 registers (more CTAs per SM) 0.244 / 0.252 / 0.254 ms */
#define HR_WIDE_C32_CH 16u
#endif
template <bool WIDE, bool POOL = false, uint32_t ROW_BYTES = 256u> struct hr_stage_cfg {
    static constexpr uint32_t NB = WIDE ? HR_STAGE_NB_WIDE : HR_STAGE_NB_ROW;
    /* the 64-register row kernel on C32 rows (160 B): 16-row chunks, which halve the
     * per-chunk refill work of the issue-bound shared-shadow traces (C3) */
    static constexpr uint32_t CH = WIDE ? ((!POOL && ROW_BYTES == 160u) ? HR_WIDE_C32_CH : 8u) : 4u;
};

/* Dynamic shared memory of a replay launch: FSM table, warp pools, the shared
 * shadow instance, then (16-byte aligned) the staging buffers and mbarriers. */
__host__ __device__ __forceinline__ uint32_t hr_stage_offset(bool pool, uint32_t warps, uint32_t smem_words)
{
    const uint32_t o = HR_FSM_SMEM_BYTES + (pool ? warps * (uint32_t)sizeof(hr_pool_smem) : 0u) + smem_words * 8u;
    return (o + 15u) & ~15u;
}

__host__ __device__ __forceinline__ uint32_t hr_stage_bytes(uint32_t warps, uint32_t nb, uint32_t ch, uint32_t row_bytes)
{
    return warps * nb * (ch * row_bytes + 8u);
}

/* POOL = false, WIDE = false: row-by-row at 48 registers, 40 warps/SM (dense
 *   global traces: occupancy hides the random-DRAM latency).
 * POOL = false, WIDE = true: row-by-row at up to 64 registers (shared-shadow
 *   heavy or small grids: issue and latency bound, spills cost more than warps).
 * POOL = true, WIDE = false: pooled at 32 registers (sparse, evenly spread
 *   traces, e.g. address shards).
 * POOL = true, WIDE = true: pooled at up to 64 registers, no spills (a few
 *   very long warps, e.g. power-law BFS hubs: per-warp latency decides).
 * Rows reach the warp through its TMA staging ring (hr_records.cuh). */
#ifndef HR_ROW_WIDE_REGS
#define HR_ROW_WIDE_REGS 64
#endif
#ifdef HR_ROW_REGS
/* register-cap experiments: the narrow kernels get __maxnreg__(HR_ROW_REGS) instead */
#define HR_REPLAY_BOUNDS(POOL, WIDE) __maxnreg__((WIDE) ? HR_ROW_WIDE_REGS : HR_ROW_REGS)
#else
/* narrow row kernel at 48 registers: on C5 (dense, random-DRAM bound) it beats both the
 * 64-register kernel (fewer warps) and the 32-register one (spills): 88.6 vs 90.2 ms,
 * round 2; the narrow pooled kernel stays at 32 (C5 shards: 32 < 40 < 48) */
#ifndef HR_ROW_NARROW_REGS
#define HR_ROW_NARROW_REGS 48
#endif
#ifndef HR_POOL_NARROW_REGS
#define HR_POOL_NARROW_REGS 32
#endif
#define HR_REPLAY_BOUNDS(POOL, WIDE) __maxnreg__((WIDE) ? HR_ROW_WIDE_REGS : ((POOL) ? HR_POOL_NARROW_REGS : HR_ROW_NARROW_REGS))
#endif
template <bool POOL, bool WIDE, bool ABL, typename SRC>
__global__ void HR_REPLAY_BOUNDS(POOL, WIDE) hr_replay_kernel(hr_dev d, SRC src,
                                                                       const uint64_t *__restrict__ woff,
                                                                       uint32_t warps, uint32_t lanes,
                                                                       uint32_t smem_words, uint32_t stage_off,
                                                                       uint32_t split_log2)
{
    /* split_log2 > 0 (pooled kernels only): each simulated warp is replayed by
     * 2^split_log2 CUDA warps of the block ("helpers"); helper h checks only the
     * accesses whose word hashes to h.  Every helper walks every row (barriers
     * and clocks stay identical), each word is still committed by one warp in
     * record order, so the per-word commit orders stay happens-before
     * consistent.  Parallelises the long warps of power-law traces. */
    const uint32_t nhw = warps << split_log2;                       /* CUDA warps in the block */
    extern __shared__ __align__(16) unsigned char hr_smem[];
    unsigned long long *sshadow = reinterpret_cast<unsigned long long *>(
        hr_smem + HR_FSM_SMEM_BYTES + (POOL ? nhw * sizeof(hr_pool_smem) : 0));
    hr_thr t = hr_thread_begin(d, hr_smem, sshadow, smem_words);
#ifdef HR_FUZZ
    const uint32_t cta = gridDim.x - 1u - blockIdx.x;               /* reversed block mapping */
    t.meta = ((unsigned long long)(((d.block_base + cta) << 10) | (t.tid() & 1023u)) << HR_TID_SHIFT) | (uint32_t)t.meta;
    t.off = hr__thread_off(d, d.block_base + cta, (t.tid() >> 5) & 31u);
#else
    const uint32_t cta = blockIdx.x;
#endif

    if (!POOL && d.hy_map != nullptr) {
        /* hybrid binned replay: this block's write position in each (bucket, block) run */
        unsigned long long *pos = reinterpret_cast<unsigned long long *>(hr_smem + d.hy_sa_off);
        for (uint32_t i = threadIdx.x; i < d.hy_nbk; i += blockDim.x) pos[i] = d.hy_off[(uint64_t)i * d.hy_nb + cta];
        __syncthreads();
    }
    constexpr uint32_t NB = hr_stage_cfg<WIDE, POOL, SRC::ROW_BYTES>::NB;
    constexpr uint32_t CH = hr_stage_cfg<WIDE, POOL, SRC::ROW_BYTES>::CH;
    constexpr uint32_t CHB = CH * SRC::ROW_BYTES;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t hw = threadIdx.x >> 5;                            /* CUDA warp */
    const uint32_t warp = POOL && split_log2 ? hw % warps : hw;      /* simulated warp */
    const uint32_t helper = POOL && split_log2 ? hw / warps : 0u;
    if (POOL && split_log2)
        t.meta = ((unsigned long long)(((d.block_base + cta) << 10) | (warp << 5) | lane) << HR_TID_SHIFT) |
                 (uint32_t)t.meta;
    if (POOL && split_log2) t.off = hr__thread_off(d, d.block_base + cta, warp);
    const uint64_t gw = (uint64_t)cta * warps + warp;
    const uint64_t r0 = woff[gw];
    const unsigned lane_mask = lanes >= 32u ? 0xffffffffu : ((1u << lanes) - 1u);
    const bool active = lane < lanes;
    /* rows per warp < 2^32 (180 GB of HBM holds < 2^30 rows) */
    const uint32_t n = (uint32_t)(woff[gw + 1] - r0);
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(hr_smem);
    const uint32_t stage = smem0 + stage_off;                       /* = hr_stage_offset() */
    const uint32_t buf0 = stage + hw * NB * CHB;
    const uint32_t bar0 = stage + nhw * NB * CHB + hw * NB * 8u;
    /* this warp's pool (shared-space address) */
    const hr_entries ps = hr__pool_at(smem0 + HR_FSM_SMEM_BYTES + hw * (uint32_t)sizeof(hr_pool_smem));
    if (lane == 0) {
#pragma unroll
        for (uint32_t b = 0; b < NB; b++) hr__mbar_init(bar0 + 8u * b, 1u);
        hr__mbar_init_fence();
#pragma unroll
        for (uint32_t b = 0; b < NB; b++)
            if (b * CH < n) {
                const uint32_t rows = min(CH, n - b * CH);
                hr__mbar_expect_tx(bar0 + 8u * b, rows * SRC::ROW_BYTES);
                src.bulk(buf0 + b * CHB, r0 + b * CH, rows, CH, bar0 + 8u * b);
            }
    }
    __syncwarp();

    /* Pool fill (warp-uniform cnt).  A row's owned accesses go to the pool in
     * lane order; when they overflow it, the first 32 - cnt are checked with the
     * pool and the rest start the next one.  Lanes of one row are unordered
     * (same warp, same epochs), so splitting a row between two consecutive pools
     * keeps every pool in record order: pools stay full except at barriers. */
    uint32_t cnt = 0;
    auto insert = [&](bool v, uint64_t x) {
        const unsigned vm = __ballot_sync(0xffffffffu, v);
        const uint32_t k = __popc(vm);
        const uint32_t slot = cnt + __popc(vm & ((1u << lane) - 1u));
        if (v && slot < 32u) ps.put(slot, x, lane);
        if (cnt + k >= 32u) {
            __syncwarp();
            hr__check_pool<ABL>(d, t, ps, 32u);
            __syncwarp();
            if (v && slot >= 32u) ps.put(slot - 32u, x, lane);
            cnt = cnt + k - 32u;
        } else {
            cnt += k;
        }
    };
    for (uint32_t c = 0; c * CH < n; c++) {
        const uint32_t b = c % NB;
        const uint32_t buf = buf0 + b * CHB;
        hr__mbar_wait(bar0 + 8u * b, (c / NB) & 1u);
        const uint32_t rows = min(CH, n - c * CH);
        uint32_t j0 = 0;
        if (POOL && WIDE) {
            /* whole chunk at once (ILP for the few long warps this kernel runs):
             * CH independent loads and validity tests, then the pool insertion;
             * a chunk holding a barrier row goes row by row below */
            uint64_t xs[CH];
            bool bar = false;
#pragma unroll
            for (uint32_t j = 0; j < CH; j++) {
                xs[j] = (active && j < rows) ? SRC::sld(buf, j, lane, CH) : HR_NOP_REC;
                bar |= (xs[j] >> 62) == 3u && (xs[j] & HR_WORD_MASK) != 0u;
            }
            if (!__any_sync(0xffffffffu, bar)) {
                bool vs[CH];
#pragma unroll
                for (uint32_t j = 0; j < CH; j++) vs[j] = hr__pool_owned(d, t, xs[j], split_log2, helper);
#pragma unroll
                for (uint32_t j = 0; j < CH; j++) insert(vs[j], xs[j]);
                j0 = rows;
            }
        }
        if (POOL && !WIDE && !ABL && SRC::C32 && split_log2 == 0u && (d.shard_log2 == 0u || d.owned_only)) {
            /* C32 rows into the pool, nothing to filter but the thread's enables (no
             * helper split, no owner hash: the trace is this shard's alone): the raw
             * (word, op | space << 2) pair of each lane, one barrier vote, one insert.
             * Lanes beyond the grid read the NOP record of the table copy. */
            uint32_t pw = active ? buf + lane * 4u : t.fsm + HR_FSM_NOP_OFF;
            uint32_t pb = active ? buf + CH * 128u + lane : t.fsm + HR_FSM_NOP_OFF + 4u;
            const uint32_t dw = active ? 128u : 0u, db = active ? 32u : 0u;
            /* bit s: accesses of space s are checked (t.off changes only at barriers) */
            uint32_t en = (t.off & 1u) ? 0u : ((t.off & 2u) ? 1u : 3u);
            for (uint32_t j = 0; j < rows; j++, pw += dw, pb += db) {
                uint32_t w32, ob;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w32) : "r"(pw) : "memory");
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(ob) : "r"(pb) : "memory");
                const bool ctl = (ob & 3u) == 3u;
                const uint64_t x = ((uint64_t)(ob & 3u) << 62) | ((uint64_t)((ob >> 2) & 1u) << 61) | w32;
                if (__any_sync(0xffffffffu, ctl && w32 != 0u)) {
                    if (cnt) { __syncwarp(); hr__check_pool<ABL>(d, t, ps, cnt); cnt = 0; __syncwarp(); }
                    hr__barrier_row(d, t, x, lane_mask);
                    en = (t.off & 1u) ? 0u : ((t.off & 2u) ? 1u : 3u);
                    continue;
                }
                insert(!ctl && ((en >> ((ob >> 2) & 1u)) & 1u), x);
            }
            j0 = rows;
        }
        if (!POOL && !ABL && SRC::C32) {
            /* C32 rows read undecoded: barrier test, then the shared-row fast path
             * (hr__check_shared_row) on the raw (word, op | space << 2) pair.  FULL (wide
             * kernel): every lane is in the grid (constant row strides); otherwise lanes
             * beyond the grid read the NOP record of the table copy (HR_FSM_NOP_OFF) on
             * every row. */
            auto c32_rows = [&](auto full) {
                constexpr bool FULL = decltype(full)::value;
                /* the shared-row word limit: 0 while this lane is off (t.off changes only at barriers) */
                uint32_t swl = (t.off & 3u) ? 0u : t.swords;
                const bool in = FULL || active;
                uint32_t pw = in ? buf + lane * 4u : t.fsm + HR_FSM_NOP_OFF;
                uint32_t pb = in ? buf + CH * 128u + lane : t.fsm + HR_FSM_NOP_OFF + 4u;
                const uint32_t dw = FULL ? 128u : (active ? 128u : 0u), db = FULL ? 32u : (active ? 32u : 0u);
                const uint32_t l0 = lane == 0u ? 1u : 0u;
                /* kept in registers (an opaque copy: not re-read from the parameter bank per row) */
                const uint32_t wcb = WIDE ? hr__reg(d.wc_bits) : d.wc_bits, wsh = WIDE ? hr__reg(d.wc_lsh) : d.wc_lsh,
                               tl = WIDE ? hr__reg(d.tile_log2) : d.tile_log2;
                for (uint32_t j = 0; j < rows; j++, pw += dw, pb += db) {
                    uint32_t w32, ob;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w32) : "r"(pw) : "memory");
                    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(ob) : "r"(pb) : "memory");
                    const bool ctl = (ob & 3u) == 3u;
                    /* one vote classifies a shared row: every lane a shared-space access
                     * (op | space << 2 in 4..6; a byte with other bits set takes the general
                     * path, which masks them) to strictly increasing in-range words (lane 0
                     * compares with itself: + 1) */
                    const uint32_t wprev = __shfl_up_sync(0xffffffffu, w32, 1);
                    if (__all_sync(0xffffffffu, (ob - 4u < 3u) & (w32 < swl) & (w32 + l0 > wprev))) {
                        hr__check_shared_row_k(d, t, w32, ob & 3u, wcb, wsh, tl);
                        continue;
                    }
                    if (__any_sync(0xffffffffu, ctl && w32 != 0u)) {
                        hr__barrier_row(d, t, ((uint64_t)(ob & 3u) << 62) | ((uint64_t)((ob >> 2) & 1u) << 61) | w32,
                                        lane_mask);
                        swl = (t.off & 3u) ? 0u : t.swords;
                        continue;
                    }
                    hr_check_lanes<false, ABL>(d, t, 0xffffffffu, !ctl, (ob >> 2) & 1u, w32, ob & 3u);
                }
            };
            /* (the 48-register kernel keeps one copy: the dense global traces it runs
             * rarely take the shared-row path, and a second copy costs it registers) */
            if (WIDE && lanes >= 32u) c32_rows(hr_bool<true>{});
            else c32_rows(hr_bool<false>{});
            j0 = rows;
        }
        for (uint32_t j = j0; j < rows; j++) {
            const uint64_t x = active ? SRC::sld(buf, j, lane, CH) : HR_NOP_REC;
            const uint32_t op = (uint32_t)(x >> 62);
            const uint64_t w = x & HR_WORD_MASK;
            if (__any_sync(0xffffffffu, op == 3u && w != 0u)) {      /* barrier row: flush, then sync */
                if (POOL && cnt) { __syncwarp(); hr__check_pool<ABL>(d, t, ps, cnt); cnt = 0; __syncwarp(); }
                hr__barrier_row(d, t, x, lane_mask);
                continue;
            }
            if (!POOL) {
                const uint32_t space = (uint32_t)(x >> 61) & 1u;
                if (!ABL && hr__shared_row_ok(t, op, space, w)) hr__check_shared_row(d, t, (uint32_t)w, op);
                else hr_check_lanes<false, ABL>(d, t, 0xffffffffu, op != 3u, space, w, op);
                continue;
            }
            insert(hr__pool_owned(d, t, x, split_log2, helper), x);
        }
        __syncwarp();                                                /* buffer b fully read: refill it */
        if (lane == 0 && (c + NB) * CH < n) {
            const uint32_t rows2 = min(CH, n - (c + NB) * CH);
            hr__mbar_expect_tx(bar0 + 8u * b, rows2 * SRC::ROW_BYTES);
            src.bulk(buf, r0 + (c + NB) * CH, rows2, CH, bar0 + 8u * b);
        }
    }
    if (POOL && cnt) { __syncwarp(); hr__check_pool<ABL>(d, t, ps, cnt); __syncwarp(); }
    if (!POOL && d.hy_map != nullptr) {
        /* hybrid: every run must end exactly where the count put the next one; a
         * mismatch (a count that disagrees with the appends) would corrupt a
         * neighbouring run, so it marks the result incomplete */
        __syncthreads();
        const unsigned long long *pos = reinterpret_cast<const unsigned long long *>(hr_smem + d.hy_sa_off);
        bool bad = false;
        for (uint32_t i = threadIdx.x; i < d.hy_nbk; i += blockDim.x)
            bad = bad || pos[i] != d.hy_off[(uint64_t)i * d.hy_nb + cta + 1u];
        if (bad) hr__set_flag(d, HR_F_INCOMPLETE);
    }
    hr_thread_end(d, t);                                             /* a9: spill a dropped shared race */
}

/* Probe for the kernel choice (one block): out[0..1] = access records / records
 * of the non-barrier rows among up to `samples` rows spread over [0, n_rows); out[2..3] = max / sum of
 * the warp lengths (rows) over the warp-offset array; out[4] = shared-space
 * access records among the samples. */
template <typename SRC>
__global__ void hr_density_kernel(SRC src, uint64_t n_rows, uint32_t samples, const uint64_t *woff, uint64_t n_woff,
                                  unsigned long long *out)
{
    __shared__ unsigned long long acc[5];
    if (threadIdx.x < 5) acc[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long mx = 0, sm = 0;
    for (uint64_t i = threadIdx.x; i + 1 < n_woff; i += blockDim.x) {
        const unsigned long long len = woff[i + 1] >= woff[i] ? woff[i + 1] - woff[i] : 0;
        mx = len > mx ? len : mx;
        sm += len;
    }
    atomicMax(&acc[2], mx);
    atomicAdd(&acc[3], sm);
    unsigned long long a = 0, tot = 0, sh = 0;
    for (uint32_t s = threadIdx.x >> 5; s < samples; s += blockDim.x >> 5) {
        /* one sample per stride, jittered by the golden-ratio sequence: a plain
         * stride aliases with the warp layout (C3: every sample on row 0) */
        const double u = ((double)s + fmod((double)s * 0.6180339887498949, 1.0)) / (double)samples;
        const uint64_t row = (uint64_t)(u * (double)n_rows);
        if (row >= n_rows) break;
        const uint64_t x = src.row(row, threadIdx.x & 31u);
        /* barrier rows are replayed by every kernel alike: density counts the
         * NOP lanes of access rows only (what pooling can skip) */
        if (__any_sync(0xffffffffu, (x >> 62) == 3u && (x & HR_WORD_MASK) != 0u)) continue;
        a += (x >> 62) != 3u;
        sh += (x >> 62) != 3u && ((x >> 61) & 1u);
        tot++;
    }
    atomicAdd(&acc[0], a);
    atomicAdd(&acc[1], tot);
    atomicAdd(&acc[4], sh);
    __syncthreads();
    if (threadIdx.x < 5) out[threadIdx.x] = acc[threadIdx.x];
}

/* a9 overflow recovery, global space (enqueued by the host after every kernel,
 * before its shadow is reset, and before a report): if the kernel latched a
 * dropped global race record in ovf[2] (hr__ring_drop), every RACE word of its
 * epoch in the (local) global shadow becomes one spill record — a superset of
 * the dropped ones, exact because the shadow word of a racy address stays in
 * RACE_* for the rest of the kernel.  Otherwise each CTA only reads one word.
 * The last CTA to finish clears ovf[2] (all CTAs read it before counting). */
__global__ void __launch_bounds__(256) hr_spill_scan_kernel(hr_dev d, const unsigned long long *__restrict__ sh,
                                                            uint64_t n_local, uint32_t epoch_tag)
{
    __shared__ uint32_t kid1;
    if (threadIdx.x == 0) kid1 = *(volatile unsigned int *)&d.ovf[2];
    __syncthreads();
    if (kid1) {
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
        for (uint64_t i0 = first; i0 < n_local; i0 += stride) {       /* warp-uniform trip count */
            const uint64_t i = i0 + (threadIdx.x & 31u);
            const unsigned long long v = i < n_local ? sh[i] : 0ull;
            const uint32_t st = (uint32_t)(v >> HR_STATE_SHIFT);
            /* lazy reset: a word of another epoch tag belongs to an earlier kernel */
            const bool mine = !epoch_tag || (((uint32_t)v >> 28) & 15u) == epoch_tag;
            const uint64_t gran = i >> d.gran_log2;
            hr_race r;
            r.word = d.gbase + ((hr_shard_granule(gran, d.shard_rank, d.shard_log2) << d.gran_log2) |
                                (i & ((1ull << d.gran_log2) - 1u)));
            r.block = 0xffffffffu;
            r.kernel = kid1 - 1u;
            r.first_tid = (uint32_t)(v >> HR_TID_SHIFT) & 0x7ffffffu;
            r.space = HR_GLOBAL;
            r.scope = (uint8_t)(st == HR_RACE_GRID ? HR_SCOPE_GRID : HR_SCOPE_BLOCK);
            r.first_kind = 0xff;
            r.prev_state = 0xff;
            hr__spill_put(d.spill, d.ovf, d.spill_cap, d.flags, 0xffffffffu, i < n_local && mine && st >= HR_RACE_BLOCK, r);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&d.ovf[3], 1u) == gridDim.x - 1u) {
            *(volatile unsigned int *)&d.ovf[2] = 0u;
            *(volatile unsigned int *)&d.ovf[3] = 0u;
            __threadfence();
        }
    }
}

#endif /* HR_REPLAY_CUH_ */
