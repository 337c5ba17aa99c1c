/*
 * hr_compact.cuh — compacted replay of long-tailed grids (DESIGN.md §5 item 8).
 *
 * Not a step of the paper's method: a re-layout of the replay input.  In a
 * power-law trace a few simulated warps are very long and sparse (a BFS hub's
 * thread walks its whole adjacency list, one active lane per row), and a U64
 * row costs a full 32-lane step however few lanes it carries.  A parallel
 * pre-pass therefore packs each long warp's accesses into dense rows, per
 * helper (the address-hash split of hr_replay_kernel), and the replay checks
 * each packed row as one pool.
 *
 * Packed stream of (simulated warp w, helper h): for each 256-row segment of
 * w, in row order, the accesses h owns are packed 32 per row in record order
 * (row-major, lanes ascending) with their simulated lane in a tag byte; a
 * barrier row ends the current piece (its last packed row is NOP-padded) and
 * is copied verbatim (tags = lanes); a segment end also closes the piece.  So
 * a packed row holds accesses of one epoch in record order: exactly the
 * invariant of a warp pool (hr_replay.cuh), and the per-word commit order is
 * the same as in the unpacked replay.  Records are packed unconditionally
 * except for NOP / inactive lanes and the shard and helper filters; the region
 * check, clock overflow and the shared-instance shard test stay in the replay.
 *
 * Layout: segoff[w] = first segment of warp w (exclusive scan of
 * ceil(rows_w / HR_CMP_SEG)); stream (w, h) owns packed rows
 * [rowoff[S*segoff[w] + h*nseg_w], rowoff[S*segoff[w] + (h+1)*nseg_w]) where
 * rowoff is the exclusive scan of the per-(w, h, segment) row counts.
 */
#ifndef HR_COMPACT_CUH_
#define HR_COMPACT_CUH_

#include "hr_device.cuh"
#include "hr_records.cuh"
#include "hr_replay.cuh"

#define HR_CMP_SEG 256u

/* nseg[i] = segments of warp i (i < nw), nseg[nw] = 0 */
__global__ void hr_cmp_nseg_kernel(const uint64_t *__restrict__ woff, uint64_t nw, uint64_t *__restrict__ nseg)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > nw) return;
    if (i == nw) { nseg[i] = 0; return; }
    const uint64_t n = woff[i + 1] - woff[i];
    nseg[i] = (n + HR_CMP_SEG - 1) / HR_CMP_SEG;
}

/* packed-stream source for the TMA staging: rows of 32 records + 32 tag bytes */
struct hr_src_cmp {
    typedef uint64_t raw_t;
    const uint64_t *rec;
    const uint8_t *tag;
    static constexpr uint32_t ROW_BYTES = 288;
    __device__ __forceinline__ void bulk(uint32_t dst, uint64_t row, uint32_t nrows, uint32_t ch, uint32_t bar) const
    {
        hr__bulk_g2s(dst, rec + row * 32, nrows * 256u, bar);
        hr__bulk_g2s(dst + ch * 256u, tag + row * 32, nrows * 32u, bar);
    }
    __host__ bool aligned_ok() const { return (((uintptr_t)rec | (uintptr_t)tag) & 15u) == 0; }
    static constexpr bool C32 = false;
    __device__ __forceinline__ static void sld2(uint32_t, uint32_t, uint32_t, uint32_t, uint32_t &, uint32_t &) {}
};

/* Walk one (warp, segment) unit: count (WRITE = false) or write the packed rows
 * of every helper.  One CUDA warp per unit; `cnt` / `rowoff` indexed
 * S*segoff[w] + h*nseg_w + seg. */
template <bool WRITE, typename SRC>
__global__ void __launch_bounds__(256) hr_cmp_walk_kernel(hr_dev d, SRC src, const uint64_t *__restrict__ woff,
                                                          const uint64_t *__restrict__ segoff, uint64_t nw,
                                                          uint32_t lanes, uint32_t split_log2,
                                                          uint64_t *__restrict__ cnt, uint64_t *__restrict__ out_rec,
                                                          uint8_t *__restrict__ out_tag)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gs = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gs >= segoff[nw]) return;
    /* warp of this segment: last w with segoff[w] <= gs */
    uint64_t lo = 0, hi = nw;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (segoff[mid] <= gs) lo = mid; else hi = mid;
    }
    const uint64_t w = lo;
    const uint64_t nsg = segoff[w + 1] - segoff[w];
    const uint64_t seg = gs - segoff[w];
    const uint64_t r0 = woff[w] + seg * HR_CMP_SEG;
    const uint64_t r1 = min(woff[w + 1], r0 + HR_CMP_SEG);
    const uint32_t S = 1u << split_log2;
    const bool active = lane < lanes;
    const uint64_t base_idx = (segoff[w] << split_log2) + seg;
    uint64_t orow[4];            /* next free packed row of each helper (WRITE) or rows counted */
    uint32_t acc[4];             /* entries of the open piece */
#pragma unroll
    for (uint32_t h = 0; h < 4; h++) {
        acc[h] = 0;
        orow[h] = (WRITE && h < S) ? cnt[base_idx + h * nsg] : 0;
    }
    for (uint64_t r = r0; r < r1; r++) {
        const uint64_t x = active ? src.row(r, lane) : HR_NOP_REC;
        const uint32_t op = (uint32_t)(x >> 62);
        const uint64_t wd = x & HR_WORD_MASK;
        const bool bar = __any_sync(0xffffffffu, op == 3u && wd != 0u);
        if (bar) {
#pragma unroll
            for (uint32_t h = 0; h < 4; h++) {
                if (h >= S) break;
                const uint32_t rem = acc[h] & 31u;
                if (WRITE && rem && lane >= rem) out_rec[(orow[h] + (acc[h] >> 5)) * 32 + lane] = HR_NOP_REC;
                orow[h] += (acc[h] + 31u) >> 5;
                acc[h] = 0;
                if (WRITE) {
                    out_rec[orow[h] * 32 + lane] = x;
                    out_tag[orow[h] * 32 + lane] = (uint8_t)lane;
                }
                orow[h] += 1;
            }
            continue;
        }
        bool v = op != 3u;
        if (v && !((x >> 61) & 1u) && d.shard_log2 && !d.owned_only) {
            const uint64_t g = wd - d.gbase;
            const bool in = wd >= d.gbase && g < d.gwords;
            v = !in || hr_shard_owner(g >> d.gran_log2, d.shard_log2) == d.shard_rank;
        }
        const uint32_t mine = split_log2 ? hr__helper_of(wd, split_log2) : 0u;
#pragma unroll
        for (uint32_t h = 0; h < 4; h++) {
            if (h >= S) break;
            const bool vh = v && mine == h;
            const unsigned m = __ballot_sync(0xffffffffu, vh);
            if (WRITE && vh) {
                const uint32_t e = acc[h] + __popc(m & ((1u << lane) - 1u));
                const uint64_t o = (orow[h] + (e >> 5)) * 32 + (e & 31u);
                out_rec[o] = x;
                out_tag[o] = (uint8_t)lane;
            }
            acc[h] += __popc(m);
        }
    }
#pragma unroll
    for (uint32_t h = 0; h < 4; h++) {
        if (h >= S) break;
        const uint32_t rem = acc[h] & 31u;
        if (WRITE && rem && lane >= rem) out_rec[(orow[h] + (acc[h] >> 5)) * 32 + lane] = HR_NOP_REC;
        orow[h] += (acc[h] + 31u) >> 5;
        if (!WRITE && lane == 0) cnt[base_idx + h * nsg] = orow[h];
    }
}

/* Replay of packed streams: one CUDA block per simulated block, warps << split
 * CUDA warps; CUDA warp hw replays stream (hw % warps, hw / warps).  Each
 * packed row is either a verbatim barrier row or one pool of up to 32 accesses
 * in record order (NOP-padded at the end). */
#ifndef HR_CMP_MINB
#define HR_CMP_MINB 1
#endif
/* NARROW = true: at most 32 registers (64 warps/SM: memory-level parallelism for
 * random-DRAM-bound pooled shards), else up to 64 */
template <bool ABL, bool NARROW = false>
__global__ void __launch_bounds__(1024, NARROW ? 2 : HR_CMP_MINB) hr_replay_compact_kernel(hr_dev d, hr_src_cmp src,
                                                                    const uint64_t *__restrict__ segoff,
                                                                    const uint64_t *__restrict__ rowoff,
                                                                    uint32_t warps, uint32_t lanes,
                                                                    uint32_t smem_words, uint32_t stage_off,
                                                                    uint32_t split_log2)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    unsigned long long *sshadow = reinterpret_cast<unsigned long long *>(hr_smem + HR_FSM_SMEM_BYTES);
    hr_thr t = hr_thread_begin(d, hr_smem, sshadow, smem_words);
#ifdef HR_FUZZ
    const uint32_t cta = gridDim.x - 1u - blockIdx.x;
    t.off = hr__thread_off(d, d.block_base + cta, 0u);
#else
    const uint32_t cta = blockIdx.x;
#endif
    constexpr uint32_t NB = 2u, CH = 8u, CHB = CH * hr_src_cmp::ROW_BYTES;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t hw = threadIdx.x >> 5;
    const uint32_t warp = hw % warps, helper = hw / warps;
    const uint32_t nhw = warps << split_log2;
    t.meta = ((unsigned long long)(((d.block_base + cta) << 10) | (warp << 5) | lane) << HR_TID_SHIFT) | (uint32_t)t.meta;
    t.off = hr__thread_off(d, d.block_base + cta, warp);
    const unsigned lane_mask = lanes >= 32u ? 0xffffffffu : ((1u << lanes) - 1u);
    const uint64_t w = (uint64_t)cta * warps + warp;
    /* segoff == NULL: one stream per warp with rows [rowoff[w], rowoff[w+1]) (HR_TRACE_POOLED) */
    const uint64_t nsg = segoff ? segoff[w + 1] - segoff[w] : 1u;
    const uint64_t bi = (segoff ? segoff[w] : w) << split_log2;
    const uint64_t c0 = rowoff[bi + helper * nsg], c1 = rowoff[bi + (helper + 1) * nsg];
    const uint32_t n = (uint32_t)(c1 - c0);
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(hr_smem);
    const uint32_t buf0 = smem0 + stage_off + hw * NB * CHB;
    const uint32_t bar0 = smem0 + stage_off + nhw * NB * CHB + hw * NB * 8u;
    if (lane == 0) {
#pragma unroll
        for (uint32_t b = 0; b < NB; b++) hr__mbar_init(bar0 + 8u * b, 1u);
        hr__mbar_init_fence();
#pragma unroll
        for (uint32_t b = 0; b < NB; b++)
            if (b * CH < n) {
                const uint32_t rows = min(CH, n - b * CH);
                hr__mbar_expect_tx(bar0 + 8u * b, rows * hr_src_cmp::ROW_BYTES);
                src.bulk(buf0 + b * CHB, c0 + b * CH, rows, CH, bar0 + 8u * b);
            }
    }
    __syncwarp();
    for (uint32_t c = 0; c * CH < n; c++) {
        const uint32_t b = c % NB;
        const uint32_t buf = buf0 + b * CHB;
        hr__mbar_wait(bar0 + 8u * b, (c / NB) & 1u);
        const uint32_t rows = min(CH, n - c * CH);
        for (uint32_t j = 0; j < rows; j++) {
            const hr_entries row(buf + j * 256u, buf + CH * 256u + j * 32u);
            const uint64_t x = row.rec_at(lane);
            const uint32_t op = (uint32_t)(x >> 62);
            const uint64_t wd = x & HR_WORD_MASK;
            if (__any_sync(0xffffffffu, op == 3u && wd != 0u)) {
                hr__barrier_row(d, t, x, lane_mask);
                continue;
            }
            if (t.off & 1u) continue;                              /* clock overflow (warp uniform) */
            const uint32_t k = __popc(__ballot_sync(0xffffffffu, op != 3u));
            if (k) hr__check_pool<ABL>(d, t, row, k);
        }
        __syncwarp();
        if (lane == 0 && (c + NB) * CH < n) {
            const uint32_t rows2 = min(CH, n - (c + NB) * CH);
            hr__mbar_expect_tx(bar0 + 8u * b, rows2 * hr_src_cmp::ROW_BYTES);
            src.bulk(buf, c0 + (c + NB) * CH, rows2, CH, bar0 + 8u * b);
        }
    }
    hr_thread_end(d, t);                                             /* a9: spill a dropped shared race */
}

#endif /* HR_COMPACT_CUH_ */
