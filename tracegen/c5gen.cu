/* c5gen.cu — GPU build of the C5 generator (c5gen.h).  INPUT ONLY: writes the
 * synthetic trace into HBM for bench.py; the race check never calls it. */
#include <cuda_runtime.h>
#include <stdint.h>

#include "c5gen.h"

/* one CUDA warp per simulated warp; pass 0 counts rows, pass 1 writes them:
 * u64 records to `out`, or (compact) the u32 word to out32 and op | space<<2
 * to the byte array outb (the HR_TRACE_C32 encoding). */
__device__ __forceinline__ void c5_put(uint64_t *out, uint32_t *out32, uint8_t *outb, uint64_t i, uint64_t x)
{
    if (out) { __stcs((unsigned long long *)&out[i], (unsigned long long)x); return; }
    out32[i] = (uint32_t)(x & 0xffffffffull);
    outb[i] = (uint8_t)((x >> 62) | (((x >> 61) & 1ull) << 2));
}

__global__ void c5_gen_kernel(c5_params p, uint32_t rank, uint32_t log2n, uint32_t glog2, uint64_t n_warps, int pass,
                              uint64_t *rows_out, const uint64_t *row_off, uint64_t *out, uint32_t *out32,
                              uint8_t *outb)
{
    uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t l = threadIdx.x & 31;
    if (gw >= n_warps) return;
    uint64_t b = gw >> 3;
    uint32_t w = (uint32_t)(gw & 7);
    uint64_t row = pass ? row_off[gw] : 0;
    for (uint32_t e = 0; e < C5_EPOCHS; e++) {
        uint32_t k = 0;
        for (uint32_t i = 0; i < C5_EPOCH; i++) {
            uint64_t x = c5_record(&p, b, w * 32 + l, e * C5_EPOCH + i);
            if (log2n == 0 || c5_owned_by(x, rank, log2n, glog2)) {
                if (pass) c5_put(out, out32, outb, (row + k) * 32 + l, x);
                k++;
            }
        }
        uint32_t maxk = __reduce_max_sync(0xffffffffu, k);
        if (pass) {
            for (uint32_t kk = k; kk < maxk; kk++) c5_put(out, out32, outb, (row + kk) * 32 + l, C5_NOP);
            c5_put(out, out32, outb, (row + maxk) * 32 + l, C5_SYNC);
        }
        row += maxk + 1;
    }
    if (!pass && l == 0) rows_out[gw] = row;
}

extern "C" int c5_gen_gpu(uint64_t seed, uint32_t lb, uint32_t rank, uint32_t log2n, uint32_t glog2, int pass,
                          uint64_t *rows_out, const uint64_t *row_off, uint64_t *out, uint32_t *out32,
                          uint8_t *outb, void *stream)
{
    c5_params p;
    p.seed = seed;
    p.lb = lb;
    uint64_t n_warps = (1ull << lb) * C5_WARPS;
    uint64_t threads = n_warps * 32;
    unsigned blocks = (unsigned)((threads + 255) / 256);
    c5_gen_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(p, rank, log2n, glog2, n_warps, pass, rows_out, row_off, out,
                                                              out32, outb);
    return (int)cudaGetLastError();
}
