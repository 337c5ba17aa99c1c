/*
 * hr_records.cuh — record sources of the replay kernels: row r of a warp for
 * one lane, decoded to the u64 record of tracegen/format.py (HR_TRACE_U64
 * stored as is; HR_TRACE_C32 split into a u32 word and a byte op | space<<2).
 * Streamed with ld.global.cs (read once).
 */
#ifndef HR_RECORDS_CUH_
#define HR_RECORDS_CUH_

#include <stdint.h>

#define HR_NOP_REC (3ull << 62)

__device__ __forceinline__ uint64_t hr__ld_rec(const uint64_t *p)
{
    return __ldcs(reinterpret_cast<const unsigned long long *>(p));
}

/* Record sources.  raw_t is what the prefetch buffer holds (loads stay in
 * flight until use); decode() turns it into the u64 record. */
struct hr_src_u64 {
    typedef uint64_t raw_t;
    const uint64_t *rec;
    __device__ __forceinline__ raw_t load(uint64_t r, uint32_t lane) const { return hr__ld_rec(rec + r * 32 + lane); }
    __device__ __forceinline__ static raw_t nop() { return HR_NOP_REC; }
    __device__ __forceinline__ static uint64_t decode(raw_t x) { return x; }
    __device__ __forceinline__ uint64_t row(uint64_t r, uint32_t lane) const { return load(r, lane); }
};

/* HR_TRACE_C32: u32 word + one byte (op | space << 2) per record, 160 B per row */
struct hr_src_c32 {
    struct raw_t { uint32_t w; uint32_t b; };
    const uint32_t *rec32;
    const uint8_t *recop;
    __device__ __forceinline__ raw_t load(uint64_t r, uint32_t lane) const
    {
        raw_t x;
        x.w = __ldcs(rec32 + r * 32 + lane);
        x.b = __ldcs(reinterpret_cast<const unsigned char *>(recop) + r * 32 + lane);
        return x;
    }
    __device__ __forceinline__ static raw_t nop() { raw_t x; x.w = 0; x.b = 3; return x; }
    __device__ __forceinline__ static uint64_t decode(raw_t x)
    {
        return ((uint64_t)(x.b & 3u) << 62) | ((uint64_t)((x.b >> 2) & 1u) << 61) | x.w;
    }
    __device__ __forceinline__ uint64_t row(uint64_t r, uint32_t lane) const { return decode(load(r, lane)); }
};

#endif /* HR_RECORDS_CUH_ */
