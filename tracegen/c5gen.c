/* c5gen.c — CPU build of the C5 generator (c5gen.h).  INPUT ONLY. */
#include <stdint.h>
#include <string.h>

#include "c5gen.h"

/* rows warp gw occupies in shard (rank of 2^log2n) */
uint64_t c5_warp_rows(const c5_params *p, uint32_t rank, uint32_t log2n, uint32_t glog2, uint64_t gw)
{
    uint64_t b = gw >> 3;
    uint32_t w = (uint32_t)(gw & 7);
    if (log2n == 0) return C5_ROWS;
    uint64_t rows = 0;
    for (uint32_t e = 0; e < C5_EPOCHS; e++) {
        uint32_t maxk = 0;
        for (uint32_t l = 0; l < C5_LANES; l++) {
            uint32_t k = 0;
            for (uint32_t i = 0; i < C5_EPOCH; i++)
                if (c5_owned_by(c5_record(p, b, w * 32 + l, e * C5_EPOCH + i), rank, log2n, glog2)) k++;
            if (k > maxk) maxk = k;
        }
        rows += maxk + 1;
    }
    return rows;
}

/* write warps [w0, w1) at rows row_off[gw - w0] (relative to out) */
void c5_gen_cpu(const c5_params *p, uint32_t rank, uint32_t log2n, uint32_t glog2, uint64_t w0, uint64_t w1,
                const uint64_t *row_off, uint64_t *out)
{
    for (uint64_t gw = w0; gw < w1; gw++) {
        uint64_t b = gw >> 3;
        uint32_t w = (uint32_t)(gw & 7);
        uint64_t row = row_off[gw - w0];
        for (uint32_t e = 0; e < C5_EPOCHS; e++) {
            uint32_t ks[C5_LANES], maxk = 0;
            for (uint32_t l = 0; l < C5_LANES; l++) {
                uint32_t k = 0;
                for (uint32_t i = 0; i < C5_EPOCH; i++) {
                    uint64_t x = c5_record(p, b, w * 32 + l, e * C5_EPOCH + i);
                    if (log2n == 0 || c5_owned_by(x, rank, log2n, glog2)) {
                        out[(row + k) * 32 + l] = x;
                        k++;
                    }
                }
                ks[l] = k;
                if (k > maxk) maxk = k;
            }
            for (uint32_t l = 0; l < C5_LANES; l++)
                for (uint32_t k = ks[l]; k < maxk; k++) out[(row + k) * 32 + l] = C5_NOP;
            row += maxk;
            for (uint32_t l = 0; l < C5_LANES; l++) out[row * 32 + l] = C5_SYNC;
            row++;
        }
    }
}

/* planted racy words and scopes (1 BLOCK, 2 GRID), one per block */
void c5_planted(const c5_params *p, uint64_t *words, uint8_t *scopes)
{
    uint64_t nb = 1ull << p->lb;
    for (uint64_t b = 0; b < nb; b++) {
        c5_plant q = c5_plant_of(p, b);
        words[b] = q.word;
        scopes[b] = q.grid ? 2 : 1;
    }
}

uint64_t c5_record_at(const c5_params *p, uint64_t b, uint32_t t, uint32_t j) { return c5_record(p, b, t, j); }
