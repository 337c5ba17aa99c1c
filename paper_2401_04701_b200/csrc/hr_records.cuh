/*
 * hr_records.cuh — record sources of the replay kernels: row r of a warp for
 * one lane, decoded to the u64 record of tracegen/format.py (HR_TRACE_U64
 * stored as is; HR_TRACE_C32 split into a u32 word and a byte op | space<<2).
 * The replay kernels stage rows in shared memory with TMA bulk copies (below);
 * the probes and the block-serial replay read them with ld.global.cs.
 */
#ifndef HR_RECORDS_CUH_
#define HR_RECORDS_CUH_

#include <stdint.h>

#define HR_NOP_REC (3ull << 62)

__device__ __forceinline__ uint64_t hr__ld_rec(const uint64_t *p)
{
    return __ldcs(reinterpret_cast<const unsigned long long *>(p));
}

/* ---------------- TMA staging (replay kernels) ----------------
 * A warp's rows are contiguous, so the replay kernels stage them in shared
 * memory with bulk copies (cp.async.bulk, SASS UBLKCP) completed on an
 * mbarrier: one lane arms the barrier with the byte count and issues the copy,
 * all lanes wait on the phase parity and read their record with ld.shared.
 * The prefetch then costs no registers and can run several rows ahead. */
__device__ __forceinline__ void hr__mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void hr__mbar_init_fence()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void hr__mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void hr__bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void hr__mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "HR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra HR_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

/* Record sources.  raw_t is what the prefetch buffer holds (loads stay in
 * flight until use); decode() turns it into the u64 record.  For the staged
 * replay: ROW_BYTES per row in global and shared memory, bulk() copies rows
 * [row, row + nrows) into a chunk buffer of capacity ch rows, sld() reads one
 * lane's record of row j of that buffer. */
struct hr_src_u64 {
    typedef uint64_t raw_t;
    const uint64_t *rec;
    __device__ __forceinline__ raw_t load(uint64_t r, uint32_t lane) const { return hr__ld_rec(rec + r * 32 + lane); }
    /* record at element index e = row * 32 + lane */
    __device__ __forceinline__ raw_t ld(uint64_t e) const { return hr__ld_rec(rec + e); }
    __device__ __forceinline__ static raw_t nop() { return HR_NOP_REC; }
    static constexpr uint32_t ROW_BYTES = 256;
    __device__ __forceinline__ void bulk(uint32_t dst, uint64_t row, uint32_t nrows, uint32_t ch, uint32_t bar) const
    {
        (void)ch;
        hr__bulk_g2s(dst, rec + row * 32, nrows * 256u, bar);
    }
    __device__ __forceinline__ static uint64_t sld(uint32_t buf, uint32_t j, uint32_t lane, uint32_t ch)
    {
        (void)ch;
        uint64_t v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(buf + (j * 32u + lane) * 8u) : "memory");
        return v;
    }
    __host__ bool aligned_ok() const { return ((uintptr_t)rec & 15u) == 0; }
    static constexpr bool C32 = false;
    __device__ __forceinline__ static void sld2(uint32_t, uint32_t, uint32_t, uint32_t, uint32_t &, uint32_t &) {}
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
    __device__ __forceinline__ raw_t ld(uint64_t e) const
    {
        raw_t x;
        x.w = __ldcs(rec32 + e);
        x.b = __ldcs(reinterpret_cast<const unsigned char *>(recop) + e);
        return x;
    }
    __device__ __forceinline__ static raw_t nop() { raw_t x; x.w = 0; x.b = 3; return x; }
    static constexpr uint32_t ROW_BYTES = 160;
    /* chunk buffer: ch rows of 32 u32 words, then ch rows of 32 op bytes */
    __device__ __forceinline__ void bulk(uint32_t dst, uint64_t row, uint32_t nrows, uint32_t ch, uint32_t bar) const
    {
        hr__bulk_g2s(dst, rec32 + row * 32, nrows * 128u, bar);
        hr__bulk_g2s(dst + ch * 128u, recop + row * 32, nrows * 32u, bar);
    }
    __device__ __forceinline__ static uint64_t sld(uint32_t buf, uint32_t j, uint32_t lane, uint32_t ch)
    {
        uint32_t w, b;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(buf + (j * 32u + lane) * 4u) : "memory");
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(buf + ch * 128u + j * 32u + lane) : "memory");
        raw_t x;
        x.w = w;
        x.b = b;
        return decode(x);
    }
    __host__ bool aligned_ok() const { return (((uintptr_t)rec32 | (uintptr_t)recop) & 15u) == 0; }
    /* the staged (word, op byte) pair undecoded (the row kernel's shared-row test) */
    static constexpr bool C32 = true;
    __device__ __forceinline__ static void sld2(uint32_t buf, uint32_t j, uint32_t lane, uint32_t ch, uint32_t &w,
                                                uint32_t &b)
    {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(buf + (j * 32u + lane) * 4u) : "memory");
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(buf + ch * 128u + j * 32u + lane) : "memory");
    }
    __device__ __forceinline__ static uint64_t decode(raw_t x)
    {
        return ((uint64_t)(x.b & 3u) << 62) | ((uint64_t)((x.b >> 2) & 1u) << 61) | x.w;
    }
    __device__ __forceinline__ uint64_t row(uint64_t r, uint32_t lane) const { return decode(load(r, lane)); }
};

#endif /* HR_RECORDS_CUH_ */
