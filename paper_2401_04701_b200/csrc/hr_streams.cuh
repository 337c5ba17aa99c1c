/*
 * hr_streams.cuh — stream-scheduled replay of barrier-free long-tailed
 * kernels (DESIGN.md §5 "hub fan-out").  Not a step of the paper's method: a
 * schedule of the replay.
 *
 * A thread-per-vertex BFS level on a power-law graph (C4) leaves a few hub
 * threads walking 10^5..10^6 adjacency records while the rest of the GPU
 * idles.  When a kernel has NO barrier records (no __syncthreads, no
 * __syncwarp) and no shared shadow, happens-before inside it is program order
 * only (barriers are the only intra-kernel ordering besides
 * program order; atomics order nothing, reading R1).  Words are independent
 * FSMs.  So the accesses of one simulated warp can be cut
 * by word hash into H "helper" streams, each kept in record order, and every
 * (warp, helper) stream can be replayed by ANY CUDA warp of ANY CTA, in any
 * order relative to the other streams: each word's accesses from one thread
 * stay in program order, and accesses of different threads are unordered.
 *
 * Plan (per launch over nw simulated warps):
 *   H_w = helpers of warp w: 1, or the power of two covering len_w / L rows
 *         (L from the launch's total rows, so the longest stream is short);
 *   a "unit" = (warp w, segment of HR_ST_SEG rows), walked by one CUDA warp:
 *   count pass  per (w, h, seg) the accesses helper h of w owns in the segment;
 *   write pass  the same walk writes them (record + simulated lane tag) into
 *               stream (w, h) at its position: streams start on 32-entry
 *               rows, segments follow each other without padding, the last
 *               row of a stream is NOP-padded;
 *   replay      a persistent grid whose warps take streams longest-first from
 *               an atomic counter and check each 32-entry row as one pool
 *               (hr__check_pool: same-word entries folded in record order).
 * A barrier record found by the count pass cancels the plan (the host falls
 * back to the per-block compacted replay, hr_compact.cuh).
 */
#ifndef HR_STREAMS_CUH_
#define HR_STREAMS_CUH_

#include "hr_compact.cuh"
#include "hr_device.cuh"
#include "hr_records.cuh"
#include "hr_replay.cuh"

#define HR_ST_SEG 1024u               /* rows per walk unit */
#define HR_ST_HMAX_LOG2 8u            /* at most 256 helper streams per simulated warp */
#define HR_ST_TARGET 8192u            /* aim: total rows / L >= this many streams of length <= L */
#define HR_ST_WALK_WARPS 8u
#ifndef HR_ST_PF
#define HR_ST_PF 1u                   /* rows a walk warp loads ahead (C4 2^24: 1 -> 24.8 ms, 4 -> 24.7, 8 -> 26.7: the
                                         unrolled body costs more than the overlap gains) */
#endif

__device__ __forceinline__ uint32_t hr__st_hlog2(uint64_t len, uint64_t L)
{
    uint32_t k = 0;
    while (k < HR_ST_HMAX_LOG2 && (L << k) < len) k++;
    return k;
}

/* per simulated warp: units, helper log2 and count slots; L = max(SEG, total / TARGET) */
__global__ void hr_st_plan_kernel(const uint64_t *__restrict__ woff, uint64_t nw, uint64_t *__restrict__ nunit,
                                  uint64_t *__restrict__ nstream, uint64_t *__restrict__ nslot,
                                  uint8_t *__restrict__ hlog2)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > nw) return;
    if (i == nw) { nunit[i] = nstream[i] = nslot[i] = 0; return; }
    const uint64_t total = woff[nw] - woff[0];
    const uint64_t L = max((uint64_t)HR_ST_SEG, (total + HR_ST_TARGET - 1) / HR_ST_TARGET);
    const uint64_t len = woff[i + 1] - woff[i];
    const uint32_t k = hr__st_hlog2(len, L);
    const uint64_t ns = (len + HR_ST_SEG - 1) / HR_ST_SEG;
    hlog2[i] = (uint8_t)k;
    nunit[i] = ns;
    nstream[i] = 1ull << k;
    nslot[i] = ns << k;
}

__device__ __forceinline__ uint64_t hr__st_find(const uint64_t *__restrict__ off, uint64_t n, uint64_t x)
{
    uint64_t lo = 0, hi = n;                              /* last i with off[i] <= x */
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (off[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

/* Walk one unit (w, seg).  Count pass: cnt[slotoff[w] + h * nseg_w + seg] =
 * accesses of helper h in the segment; sets *barrier on a barrier row.
 * Write pass: rec/tag at pos(w, h, seg) = sbase[streamoff[w] + h] + eoff[slot]
 * - eoff[slot of (w, h, 0)], in record order (lanes of one row: lane order). */
template <bool WRITE, typename SRC>
__global__ void __launch_bounds__(HR_ST_WALK_WARPS * 32) hr_st_walk_kernel(
    hr_dev d, SRC src, const uint64_t *__restrict__ woff, uint64_t nw, const uint64_t *__restrict__ unitoff,
    const uint64_t *__restrict__ slotoff, const uint64_t *__restrict__ streamoff, const uint8_t *__restrict__ hlog2,
    uint32_t lanes, uint64_t *__restrict__ cnt, const uint64_t *__restrict__ eoff, const uint64_t *__restrict__ sbase,
    uint64_t *__restrict__ out_rec, uint8_t *__restrict__ out_tag, unsigned int *__restrict__ barrier)
{
    __shared__ uint64_t pos_s[HR_ST_WALK_WARPS][1u << HR_ST_HMAX_LOG2];
    const uint32_t lane = threadIdx.x & 31u, hw = threadIdx.x >> 5;
    const uint64_t u = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= unitoff[nw]) return;                          /* warp-uniform */
    const uint64_t w = hr__st_find(unitoff, nw, u);
    const uint64_t nseg = unitoff[w + 1] - unitoff[w];
    const uint64_t seg = u - unitoff[w];
    const uint32_t k = hlog2[w], H = 1u << k;
    const uint64_t r0 = woff[w] + seg * HR_ST_SEG, r1 = min(woff[w + 1], r0 + HR_ST_SEG);
    uint64_t *pos = pos_s[hw];
    for (uint32_t h = lane; h < H; h += 32u) {
        uint64_t p = 0;
        if (WRITE) {
            const uint64_t s0 = slotoff[w] + (uint64_t)h * nseg;
            p = sbase[streamoff[w] + h] + (eoff[s0 + seg] - eoff[s0]);
        }
        pos[h] = p;
    }
    __syncwarp();
    const bool active = lane < lanes;
    for (uint64_t rb = r0; rb < r1; rb += HR_ST_PF) {
      /* HR_ST_PF rows loaded ahead: the walk is a chain of dependent row steps,
       * so independent loads are what keeps it off the latency floor */
      uint64_t xs[HR_ST_PF];
#pragma unroll
      for (uint32_t q = 0; q < HR_ST_PF; q++) xs[q] = (active && rb + q < r1) ? src.row(rb + q, lane) : HR_NOP_REC;
#pragma unroll
      for (uint32_t q = 0; q < HR_ST_PF; q++) {
        if (rb + q >= r1) break;
        const uint64_t x = xs[q];
        const uint32_t op = (uint32_t)(x >> 62);
        const uint64_t wd = x & HR_WORD_MASK;
        if (__any_sync(0xffffffffu, op == 3u && wd != 0u)) {
            if (!WRITE && lane == 0) atomicOr(barrier, 1u);
            return;                                           /* the plan is discarded */
        }
        bool v = op != 3u;
        if (v && !((x >> 61) & 1u) && d.shard_log2 && !d.owned_only) {
            const uint64_t g = wd - d.gbase;
            const bool in = wd >= d.gbase && g < d.gwords;
            v = !in || hr_shard_owner(g >> d.gran_log2, d.shard_log2) == d.shard_rank;
        }
        const uint32_t h = (v && k) ? hr__helper_of(wd, k) : 0u;
        const unsigned grp = __match_any_sync(0xffffffffu, v ? h : 0xffffffffu);
        const uint32_t leader = __ffs(grp) - 1;
        uint64_t base = 0;
        if (v && lane == leader) {
            base = pos[h];
            pos[h] = base + __popc(grp);
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        if (WRITE && v) {
            const uint64_t o = base + __popc(grp & ((1u << lane) - 1u));
            out_rec[o] = x;
            out_tag[o] = (uint8_t)lane;
        }
        __syncwarp();
      }
    }
    if (!WRITE)
        for (uint32_t h = lane; h < H; h += 32u) cnt[slotoff[w] + (uint64_t)h * nseg + seg] = pos[h];
}

/* per stream s = (w, h): entries T, padded length P (a multiple of 32), warp;
 * key = rows descending (for the longest-first order) */
__global__ void hr_st_stream_kernel(const uint64_t *__restrict__ streamoff, const uint64_t *__restrict__ unitoff,
                                    const uint64_t *__restrict__ slotoff, uint64_t nw, uint64_t ns,
                                    const uint64_t *__restrict__ eoff, uint64_t *__restrict__ plen,
                                    uint32_t *__restrict__ swarp, uint32_t *__restrict__ skey,
                                    uint32_t *__restrict__ sid, uint32_t *__restrict__ stot)
{
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s > ns) return;
    if (s == ns) { plen[s] = 0; return; }
    const uint64_t w = hr__st_find(streamoff, nw, s);
    const uint64_t h = s - streamoff[w];
    const uint64_t nseg = unitoff[w + 1] - unitoff[w];
    const uint64_t s0 = slotoff[w] + h * nseg;
    const uint64_t T = eoff[s0 + nseg] - eoff[s0];
    const uint64_t P = (T + 31u) & ~31ull;
    plen[s] = P;
    swarp[s] = (uint32_t)w;
    stot[s] = (uint32_t)T;
    skey[s] = 0xffffffffu - (uint32_t)((P >> 5) < 0xffffffffull ? (P >> 5) : 0xffffffffull);
    sid[s] = (uint32_t)s;
}

/* NOP-pad the last row of every stream */
__global__ void hr_st_pad_kernel(const uint64_t *__restrict__ sbase, const uint32_t *__restrict__ stot, uint64_t ns,
                                 uint64_t *__restrict__ out_rec, uint8_t *__restrict__ out_tag)
{
    const uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (s >= ns) return;
    const uint64_t e = sbase[s] + stot[s];
    if (e < sbase[s + 1] && (e & ~31ull) + lane >= e) {
        const uint64_t o = (e & ~31ull) + lane;
        out_rec[o] = HR_NOP_REC;
        out_tag[o] = (uint8_t)lane;
    }
}

/* Persistent replay of the streams: each CUDA warp takes the next stream
 * (longest first) from *next and checks its rows as pools, rows staged in
 * SMEM by TMA bulk copies (NB x CH rows per warp, phases continuing across
 * streams).  No shared shadow and no clocks (barrier-free kernel). */
#define HR_ST_WARPS 16u
#ifndef HR_ST_CTAS
#define HR_ST_CTAS 3u                 /* CTAs per SM (<= 42 registers, 48 warps/SM) */
#endif
template <bool ABL>
__global__ void __launch_bounds__(HR_ST_WARPS * 32, HR_ST_CTAS) hr_replay_streams_kernel(
    hr_dev d, hr_src_cmp src, const uint64_t *__restrict__ sbase, const uint32_t *__restrict__ order,
    const uint32_t *__restrict__ swarp, uint32_t ns, uint32_t warps, unsigned int *__restrict__ next)
{
    constexpr uint32_t NB = 2u, CH = 8u, CHB = CH * hr_src_cmp::ROW_BYTES;   /* NB = 2: parities ph0 / ph1 */
    extern __shared__ __align__(16) unsigned char hr_smem[];
    for (uint32_t i = threadIdx.x; i < HR_FSM_SMEM_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(hr_smem)[i] = reinterpret_cast<const uint4 *>(d.fsm)[i];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, hw = threadIdx.x >> 5;
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(hr_smem);
    const uint32_t stage = smem0 + ((HR_FSM_SMEM_BYTES + 15u) & ~15u);
    const uint32_t buf0 = stage + hw * NB * CHB;
    const uint32_t bar0 = stage + HR_ST_WARPS * NB * CHB + hw * NB * 8u;
    if (lane == 0) {
#pragma unroll
        for (uint32_t b = 0; b < NB; b++) hr__mbar_init(bar0 + 8u * b, 1u);
        hr__mbar_init_fence();
    }
    __syncwarp();
    hr_thr t;
    t.sshadow = 0;
    t.swords = 0;
    t.fsm = smem0;
    uint32_t ph0 = 0u, ph1 = 0u;                         /* phases completed per buffer (mbarrier parity) */
    while (true) {
        uint32_t i = 0;
        if (lane == 0) i = atomicAdd(next, 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= ns) break;
        const uint32_t s = order[i];
        const uint32_t w = swarp[s];
        const uint32_t block = d.block_base + w / warps, wib = w % warps;
        t.meta = ((unsigned long long)((block << 10) | (wib << 5)) << HR_TID_SHIFT) |
                 ((unsigned long long)d.epoch_tag << 28);
        t.off = hr__thread_off(d, block, wib);
        if (t.off & 1u) continue;                          /* not a representative thread */
        const uint64_t row0 = sbase[s] >> 5;
        const uint32_t n = (uint32_t)((sbase[s + 1] >> 5) - row0);
        if (lane == 0) {
#pragma unroll
            for (uint32_t b = 0; b < NB; b++)
                if (b * CH < n) {
                    const uint32_t rows = min(CH, n - b * CH);
                    hr__mbar_expect_tx(bar0 + 8u * b, rows * hr_src_cmp::ROW_BYTES);
                    src.bulk(buf0 + b * CHB, row0 + b * CH, rows, CH, bar0 + 8u * b);
                }
        }
        __syncwarp();
        for (uint32_t c = 0; c * CH < n; c++) {
            const uint32_t b = c % NB;
            const uint32_t buf = buf0 + b * CHB;
            hr__mbar_wait(bar0 + 8u * b, (b ? ph1 : ph0) & 1u);
            if (b) ph1++; else ph0++;
            const uint32_t rows = min(CH, n - c * CH);
            for (uint32_t j = 0; j < rows; j++) {
                const hr_entries row(buf + j * 256u, buf + CH * 256u + j * 32u);
                const uint64_t x = row.rec_at(lane);
                const uint32_t k = __popc(__ballot_sync(0xffffffffu, (x >> 62) != 3u));
                if (k) hr__check_pool<ABL>(d, t, row, k);
            }
            __syncwarp();
            if (lane == 0 && (c + NB) * CH < n) {
                const uint32_t rows2 = min(CH, n - (c + NB) * CH);
                hr__mbar_expect_tx(bar0 + 8u * b, rows2 * hr_src_cmp::ROW_BYTES);
                src.bulk(buf, row0 + (c + NB) * CH, rows2, CH, bar0 + 8u * b);
            }
        }
    }
}

__host__ __forceinline__ size_t hr_streams_smem()
{
    return ((HR_FSM_SMEM_BYTES + 15u) & ~15u) + HR_ST_WARPS * 2u * (8u * hr_src_cmp::ROW_BYTES + 8u);
}

#endif /* HR_STREAMS_CUH_ */
