/*
 * hr_records.cuh — record sources of the replay kernels: row r of a warp for
 * one lane, decoded to the u64 record of tracegen/format.py (HR_TRACE_U64
 * stored as is; HR_TRACE_C32 split into a u32 word, a per-row u64 of 2-bit ops
 * and a per-row u32 space mask).  Streamed with ld.global.cs (read once).
 */
#ifndef HR_RECORDS_CUH_
#define HR_RECORDS_CUH_

#include <stdint.h>

#define HR_NOP_REC (3ull << 62)

__device__ __forceinline__ uint64_t hr__ld_rec(const uint64_t *p)
{
    return __ldcs(reinterpret_cast<const unsigned long long *>(p));
}

/* Record sources: row i of this warp for this lane, as a u64 record. */
struct hr_src_u64 {
    const uint64_t *rec;
    __device__ __forceinline__ uint64_t row(uint64_t r, uint32_t lane) const { return hr__ld_rec(rec + r * 32 + lane); }
};

struct hr_src_c32 {
    const uint32_t *rec32;
    const uint64_t *ops;
    const uint32_t *spc;
    __device__ __forceinline__ uint64_t row(uint64_t r, uint32_t lane) const
    {
        const uint64_t w = __ldcs(rec32 + r * 32 + lane);
        const uint64_t o = __ldcs(reinterpret_cast<const unsigned long long *>(ops + r));
        const uint32_t sp = __ldcs(spc + r);
        return (((o >> (2u * lane)) & 3ull) << 62) | ((uint64_t)((sp >> lane) & 1u) << 61) | w;
    }
};

#endif /* HR_RECORDS_CUH_ */
