/*
 * hr_pack.cuh — HR_TRACE_PACKED encoder and decoder (format in include/hr.h).
 *
 * Not part of the paper's method: a lossless transfer encoding of the replay
 * records so that hr_replay_trace_host moves fewer PCIe bytes.
 * Frame-of-reference per warp-row: a nibble per lane (op | space or control
 * word), one base word, and either word = base + lane (a coalesced row),
 * word = base (a broadcast), or k-bit deltas; a coalesced row of reads and
 * writes of one space keeps one bit per lane instead of a nibble.  C5's own-row
 * rows shrink from 160 B (C32) to 9 B, its random gathers to 133 B (a base
 * below 2^32 takes 4 bytes).
 *
 * Both directions run one CUDA warp per segment (one trace warp's rows).
 * The decoder writes U64 rows that the unchanged replay kernels then read.
 */
#ifndef HR_PACK_CUH_
#define HR_PACK_CUH_

#include <stdint.h>

#define HR_PACK_RAW 62u
#define HR_PACK_NOWORD 63u
#define HR_PACK_AFFINE 64u
#define HR_PACK_UNIFORM 128u
#define HR_PACK_SLACK 16u
#define HR_PACK_WORD_MASK ((1ull << 61) - 1)

/* An affine row whose lanes are all reads or writes of one space: the nibbles
 * are one u32 bit mask (bit l = lane l writes), k = 1 + space (affine rows have
 * no deltas, so these k values are otherwise unused); the uniform bit (a mask
 * row is never uniform) marks a base below 2^32 stored in one u32. */
__host__ __device__ __forceinline__ bool hr_pack_is_rwmask(uint32_t h)
{
    const uint32_t k = h & 63u;
    return (h & HR_PACK_AFFINE) && (k == 1u || k == 2u);
}

/* A delta row (k >= 3 bits) whose base fits 32 bits stores it in one u32; the
 * affine bit marks it (affine rows carry no deltas, so affine with k >= 3 is
 * otherwise unused; k = 62 / 63 keep their meaning). */
__host__ __device__ __forceinline__ bool hr_pack_is_short(uint32_t h)
{
    const uint32_t k = h & 63u;
    return (h & HR_PACK_AFFINE) && k >= 3u && k < HR_PACK_RAW;
}

/* Body bytes of a row with header byte h. */
__host__ __device__ __forceinline__ uint32_t hr_pack_body_bytes(uint32_t h)
{
    const uint32_t k = h & 63u;
    if (k == HR_PACK_RAW) return 256u;
    if (hr_pack_is_rwmask(h)) return (h & HR_PACK_UNIFORM) ? 8u : 12u;
    uint32_t b = (h & HR_PACK_UNIFORM) ? 4u : 16u;
    if (hr_pack_is_short(h)) return b + 4u + 4u * k;
    if (k != HR_PACK_NOWORD) b += 8u + ((h & HR_PACK_AFFINE) ? 0u : 4u * k);
    return b;
}

__device__ __forceinline__ uint64_t hr__shfl64(uint64_t v, int src)
{
    return ((uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src) << 32) |
           __shfl_sync(0xffffffffu, (uint32_t)v, src);
}

__device__ __forceinline__ uint64_t hr__xor64(uint64_t v, int m)
{
    return ((uint64_t)__shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m) << 32) |
           __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
}

/* Encoding decisions for one row; every lane holds its record x.  Returns the
 * header byte (identical in all lanes); nib/base/delta are this lane's. */
struct hr_pack_row {
    uint32_t h, nib;
    uint64_t base, delta;
};

__device__ __forceinline__ hr_pack_row hr__pack_decide(uint64_t x, uint32_t lane)
{
    hr_pack_row r;
    const uint32_t op = (uint32_t)(x >> 62), sp = (uint32_t)(x >> 61) & 1u;
    const uint64_t w = x & HR_PACK_WORD_MASK;
    const bool acc = op != 3u;
    const bool rep = acc || (sp == 0u && w <= 2u);
    r.nib = acc ? (op | (sp << 2)) : (3u | ((uint32_t)w << 2));
    r.base = 0;
    r.delta = 0;
    if (!__all_sync(0xffffffffu, rep)) {
        r.h = HR_PACK_RAW;
        return r;
    }
    const bool uniform = __all_sync(0xffffffffu, r.nib == (uint32_t)__shfl_sync(0xffffffffu, (int)r.nib, 0));
    const uint32_t amask = __ballot_sync(0xffffffffu, acc);
    uint32_t h = uniform ? HR_PACK_UNIFORM : 0u;
    if (!amask) {
        r.h = h | HR_PACK_NOWORD;
        return r;
    }
    const int l0 = __ffs((int)amask) - 1;
    const uint64_t base_a = hr__shfl64(w, l0) - (uint64_t)l0;
    if (__all_sync(0xffffffffu, !acc || w == base_a + lane)) {
        r.base = base_a;
        /* every lane a read or write of one space, not all the same op: a bit mask */
        const uint32_t sp0 = (uint32_t)__shfl_sync(0xffffffffu, (int)sp, 0);
        if (!uniform && amask == 0xffffffffu && __all_sync(0xffffffffu, op <= 1u && sp == sp0)) {
            r.h = HR_PACK_AFFINE | (1u + sp0) | (base_a < (1ull << 32) ? HR_PACK_UNIFORM : 0u);
            return r;
        }
        r.h = h | HR_PACK_AFFINE;
        return r;
    }
    uint64_t mn = acc ? w : ~0ull;
#pragma unroll
    for (int m = 16; m; m >>= 1) {
        const uint64_t o = hr__xor64(mn, m);
        mn = o < mn ? o : mn;
    }
    uint64_t mx = acc ? w - mn : 0ull;
#pragma unroll
    for (int m = 16; m; m >>= 1) {
        const uint64_t o = hr__xor64(mx, m);
        mx = o > mx ? o : mx;
    }
    r.base = mn;
    r.delta = acc ? w - mn : 0ull;
    const uint32_t k = mx ? (uint32_t)(64 - __clzll((long long)mx)) : 0u;
    r.h = h | k;
    if (k >= 3u && mn < (1ull << 32)) r.h |= HR_PACK_AFFINE;      /* 4-byte base */
    return r;
}

/* Pass 1: bytes of segment i -> seg_bytes[i] (0 for the last entry). */
__global__ void hr_pack_size_kernel(const uint64_t *__restrict__ rec, const uint64_t *__restrict__ woff,
                                    uint64_t n_woff, uint64_t *__restrict__ seg_bytes, unsigned int *err)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n_woff) return;
    if (i + 1 == n_woff) {
        if (lane == 0) seg_bytes[i] = 0;
        return;
    }
    const uint64_t r0 = woff[i], r1 = woff[i + 1];
    if (r1 < r0) {
        if (lane == 0) { seg_bytes[i] = 0; atomicOr(err, 1u); }
        return;
    }
    uint64_t bytes = (r1 - r0 + 3) & ~3ull;
    for (uint64_t r = r0; r < r1; r++) {
        const hr_pack_row pr = hr__pack_decide(rec[r * 32 + lane], lane);
        bytes += hr_pack_body_bytes(pr.h);
    }
    if (lane == 0) seg_bytes[i] = bytes;
}

/* Pass 2: write segment i at out + pack_off[i]. */
__global__ void __launch_bounds__(256) hr_pack_write_kernel(const uint64_t *__restrict__ rec,
                                                            const uint64_t *__restrict__ woff, uint64_t n_woff,
                                                            const uint64_t *__restrict__ pack_off,
                                                            uint8_t *__restrict__ out)
{
    __shared__ uint32_t bits[8][64];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i + 1 >= n_woff) return;
    const uint64_t r0 = woff[i], r1 = woff[i + 1];
    if (r1 < r0) return;
    const uint64_t n = r1 - r0;
    uint8_t *seg = out + pack_off[i];
    uint32_t *body = reinterpret_cast<uint32_t *>(seg + ((n + 3) & ~3ull));
    for (uint64_t j = lane; j < ((n + 3) & ~3ull); j += 32)
        if (j >= n) seg[j] = 0;
    uint32_t *sb = bits[wib];
    for (uint64_t j = 0; j < n; j++) {
        const uint64_t x = rec[(r0 + j) * 32 + lane];
        const hr_pack_row pr = hr__pack_decide(x, lane);
        const uint32_t h = pr.h, k = h & 63u;
        if (lane == 0) seg[j] = (uint8_t)h;
        if (k == HR_PACK_RAW) {
            body[2 * lane] = (uint32_t)x;
            body[2 * lane + 1] = (uint32_t)(x >> 32);
            body += 64;
            continue;
        }
        uint32_t nw;
        if (hr_pack_is_rwmask(h)) {
            const unsigned m = __ballot_sync(0xffffffffu, ((x >> 62) & 1u) != 0u);
            if (lane == 0) {
                body[0] = m;
                body[1] = (uint32_t)pr.base;
                if (!(h & HR_PACK_UNIFORM)) body[2] = (uint32_t)(pr.base >> 32);
            }
            body += (h & HR_PACK_UNIFORM) ? 2 : 3;
            continue;
        } else if (h & HR_PACK_UNIFORM) {
            if (lane == 0) body[0] = pr.nib;
            nw = 1;
        } else {
            uint32_t v = pr.nib << (4u * (lane & 7u));
            v |= __shfl_xor_sync(0xffffffffu, v, 1);
            v |= __shfl_xor_sync(0xffffffffu, v, 2);
            v |= __shfl_xor_sync(0xffffffffu, v, 4);
            if ((lane & 7u) == 0) body[lane >> 3] = v;
            nw = 4;
        }
        body += nw;
        if (k == HR_PACK_NOWORD) continue;
        const bool shb = hr_pack_is_short(h);
        if (lane == 0) {
            body[0] = (uint32_t)pr.base;
            if (!shb) body[1] = (uint32_t)(pr.base >> 32);
        }
        body += shb ? 1 : 2;
        if (((h & HR_PACK_AFFINE) && !shb) || k == 0) continue;
        sb[lane] = 0;
        sb[lane + 32] = 0;
        __syncwarp();
        if (pr.delta) {
            const uint32_t p = lane * k, q = p >> 5, s = p & 31u;
            atomicOr(&sb[q], (uint32_t)(pr.delta << s));
            if (s + k > 32) atomicOr(&sb[q + 1], (uint32_t)(pr.delta >> (32 - s)));
            if (s + k > 64) atomicOr(&sb[q + 2], (uint32_t)(pr.delta >> (64 - s)));
        }
        __syncwarp();
        for (uint32_t m = lane; m < k; m += 32) body[m] = sb[m];
        __syncwarp();
        body += k;
    }
}

/* This lane's record of the row at `body` with header h. */
__device__ __forceinline__ uint64_t hr__unpack_lane(const uint32_t *__restrict__ body, uint32_t h, uint32_t lane)
{
    const uint32_t k = h & 63u;
    if (k == HR_PACK_RAW) return (uint64_t)body[2 * lane] | ((uint64_t)body[2 * lane + 1] << 32);
    if (hr_pack_is_rwmask(h)) {
        const uint64_t base = (uint64_t)body[1] | ((h & HR_PACK_UNIFORM) ? 0ull : ((uint64_t)body[2] << 32));
        return ((uint64_t)((body[0] >> lane) & 1u) << 62) | ((uint64_t)(k - 1u) << 61) |
               ((base + lane) & HR_PACK_WORD_MASK);
    }
    uint32_t nib;
    uint32_t nw;
    if (h & HR_PACK_UNIFORM) {
        nib = body[0] & 15u;
        nw = 1;
    } else {
        nib = (body[lane >> 3] >> (4u * (lane & 7u))) & 15u;
        nw = 4;
    }
    const uint64_t op = nib & 3u, x2 = nib >> 2;
    if (op == 3u) return (3ull << 62) | x2;
    const bool shb = hr_pack_is_short(h);
    const uint64_t base = shb ? (uint64_t)body[nw] : ((uint64_t)body[nw] | ((uint64_t)body[nw + 1] << 32));
    uint64_t d;
    if ((h & HR_PACK_AFFINE) && !shb) {
        d = lane;
    } else if (k == 0) {
        d = 0;
    } else {
        const uint32_t *dw = body + nw + (shb ? 1u : 2u);
        const uint32_t p = lane * k, q = p >> 5, s = p & 31u;
        uint64_t lo = dw[q];
        if (s + k > 32) lo |= (uint64_t)dw[q + 1] << 32;
        d = lo >> s;
        if (s + k > 64) d |= (uint64_t)dw[q + 2] << (64 - s);
        d &= (1ull << k) - 1ull;
    }
    return (op << 62) | (x2 << 61) | ((base + d) & HR_PACK_WORD_MASK);
}

/* Decode segments [s0, s1) into U64 rows: row r goes to out[(r - rbase)*32 + lane]. */
__global__ void __launch_bounds__(256) hr_unpack_kernel(const uint8_t *__restrict__ packed,
                                                        const uint64_t *__restrict__ pack_off,
                                                        const uint64_t *__restrict__ woff, uint64_t s0, uint64_t s1,
                                                        uint64_t rbase, uint64_t *__restrict__ out)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t i = s0 + (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (i >= s1) return;
    const uint64_t r0 = woff[i], r1 = woff[i + 1];
    if (r1 <= r0) return;
    const uint64_t n = r1 - r0;
    const uint8_t *seg = packed + pack_off[i];
    const uint8_t *bodies = seg + ((n + 3) & ~3ull);
    uint64_t run = 0;
    uint64_t *dst = out + (r0 - rbase) * 32 + lane;
    for (uint64_t j0 = 0; j0 < n; j0 += 32) {
        const uint64_t j = j0 + lane;
        const uint32_t h = j < n ? seg[j] : 0u;
        const uint32_t sz = j < n ? hr_pack_body_bytes(h) : 0u;
        uint32_t inc = sz;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, m);
            if ((int)lane >= m) inc += o;
        }
        const uint64_t off = run + inc - sz;
        run += __shfl_sync(0xffffffffu, inc, 31);
        const uint32_t cnt = n - j0 < 32 ? (uint32_t)(n - j0) : 32u;
        for (uint32_t jj = 0; jj < cnt; jj++) {
            const uint32_t hh = __shfl_sync(0xffffffffu, h, jj);
            const uint64_t oo = hr__shfl64(off, jj);
            const uint32_t *body = reinterpret_cast<const uint32_t *>(bodies + oo);
            dst[(j0 + jj) * 32] = hr__unpack_lane(body, hh, lane);
        }
    }
}

#endif /* HR_PACK_CUH_ */
