/*
 * hr_host.cu — implementation of the C ABI in include/hr.h.
 *
 * Owns the device state of one checker context: the FSM table (generated,
 * fsm_table.inc), the global shadow slice, the report ring + tail counter, the
 * sticky flags word and the replay staging buffers.  All allocation happens
 * in hr_init / hr_shadow_alloc / the first hr_replay_trace_host; the check
 * path allocates nothing.
 */
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <new>
#include <vector>

#include "hr.h"
#include "hr_device.cuh"
#include "hr_replay.cuh"
#include "hr_fh.cuh"
#include "hr_classes.cuh"
#include "hr_pack.cuh"
#include "hr_compact.cuh"
#include "hr_bserial.cuh"
#include "hr_streams.cuh"
#include "hr_binned.cuh"
#include "hr_hybrid.cuh"
#include "fsm_table.inc"
#include "fsm_classes.inc"

struct hr_ctx {
    int device = 0;
    hr_config cfg{};
    uint32_t shard_rank = 0, shard_count = 1, shard_log2 = 0, gran_log2 = 3;
    unsigned long long *gshadow = nullptr;       /* current buffer */
    unsigned long long *gbuf[2] = {nullptr, nullptr};
    int gcur = 0;
    bool double_shadow = false;
    bool dirty[2] = {false, false};              /* buffer used by a kernel since its last reset */
    cudaStream_t side = nullptr;                 /* deferred resets (double shadow) */
    cudaEvent_t used_done[2] = {nullptr, nullptr}, reset_done[2] = {nullptr, nullptr};
    uint64_t gbase = 0, gwords = 0, glocal = 0;
    uint64_t launches = 0;
    uint32_t epoch_tag = 0;                      /* HR_OPT_LAZY_RESET: tag of the current kernel (1..15) */
    uint32_t sort_tmp_n = 0;                     /* cached CUB temp size of the report sort */
    uint32_t rep_bstride = 1, rep_wstride = 1;   /* hr_set_representatives */
    bool cur_owned_only = false;                 /* the trace being replayed is HR_TRACE_F_SHARD_OWNED */
    uint32_t online_tile_log2 = 5;               /* hr_set_warp_tile: warp tile of online kernels */
    size_t sort_tmp_bytes = 0;                       /* kernels launched (1 per CUB call), hr_launch_count */
    uint32_t shadow_bytes = 8;                   /* per word: 8 (HiRace) or 16 (finite-history baseline) */
    uint32_t smem_words_max = 0;
    hr_race *ring = nullptr;                     /* ring_capacity records, then spill_cap spill records */
    uint32_t spill_cap = 0;
    bool scan_pending = false;                   /* a kernel used the current global shadow since its
                                                    end-of-kernel spill scan was enqueued */
    bool online_used = false;                    /* hr_device_view since the last hr_reset_report: ring
                                                    records may carry any kernel id / shared word */
    unsigned int *tail = nullptr;     /* [0] ring tail, [1] flags, [2..5] hr_dev.ovf (spill tail,
                                         unspilled shared drops, global drop kernel + 1, scan counter) */
    unsigned long long *counters = nullptr;
    unsigned char *fsm = nullptr;
    uint32_t last_kernel = 0;
    uint32_t max_kernel = 0;                     /* largest kernel id replayed on this ctx (report sort range) */
    bool have_kernel = false;
    int last_kind = 0;                           /* HR_K_* of the last replay */
    /* kernel choice of the last probed device trace (a performance hint only:
     * every kernel gives the same result, so a stale hint is harmless) */
    struct { const void *rec; uint64_t n_rows; const void *woff; uint64_t n_woff; uint32_t format, options; int kind; }
        choice_cache = {nullptr, 0, nullptr, 0, 0, 0, -1};
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;                 /* host-trace staging copies */
    /* staging: 0 warp_off, 1 rec|rec32|packed, 2 recop|decoded chunk, 3 pack_off,
     * 4 hr_pack_trace segment sizes + error word, 5 scan temporaries,
     * compacted replay: 6 segment counts, 7 segment offsets, 8 row counts,
     * 9 row offsets, 10 packed records, 11 packed tags,
     * stream-scheduled replay (hr_streams.cuh): 12 per-warp units/streams/slots (3 x nw+1),
     * 13 their scans (3 x nw+1), 14 helper log2, 15 slot counts, 16 slot offsets, 17 stream
     * lengths / bases, 18 stream warp / key / id / total, 19 sorted keys / order, 20 counters,
     * binned replay (hr_binned.cuh): 21 entries, 22 per-(bucket, block) counts, 23 their offsets */
    void *stage[24] = {};
    size_t stage_cap[24] = {};
    hr_race *rep_host = nullptr;                 /* pinned staging of the sorted report (D2H) */
    size_t rep_cap = 0;
    std::vector<hr_race> rep;                    /* report scratch, kept across calls */
    /* hr_report_async: device scratch, pinned mapped result (ring_capacity
     * records + a 4-word header: unique count, flags, raw count), completion event */
    void *arep_scratch = nullptr;
    size_t arep_scratch_bytes = 0, arep_tmp_bytes = 0;
    hr_race *arep_host = nullptr, *arep_dev = nullptr;
    uint32_t *arep_hdr_host = nullptr, *arep_hdr_dev = nullptr;
    cudaEvent_t arep_ev = nullptr;
    bool arep_pending = false;
    /* the report as one CUDA graph: the one-CTA small-set kernel, then an IF node
     * (set by that kernel) around the full-capacity CUB path; rebuilt when its
     * arguments change.  arep_big: kernels the IF body launched (hr_launch_count). */
    struct arep_key_t { const void *out, *hdr, *scratch, *ring; uint32_t out_cap, cap; int lo_bits, hi_bits; };
    /* two cached graphs (hr_report_async into the ctx's pinned buffer and
     * hr_report_async_to into a caller's may alternate); slot arep_lru is replaced next */
    struct { cudaGraph_t graph; cudaGraphExec_t exec; arep_key_t key; } arep_g[2] = {};
    int arep_lru = 0;
    cudaGraphExec_t arep_exec = nullptr;          /* the graph of the current call */
    cudaStream_t arep_cap = nullptr;              /* capture stream of the IF body */
    unsigned long long *arep_big = nullptr;
    bool arep_no_graph = false;                   /* graph build failed once: direct launches */
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_reset, ev_kernel;
    char err[512] = {0};
};

static cudaEvent_t get_event(hr_ctx *c)
{
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

static hr_status fail(hr_ctx *c, hr_status s, const char *fmt, ...)
{
    if (c) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(c->err, sizeof c->err, fmt, ap);
        va_end(ap);
    }
    return s;
}

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(c, HR_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                            \
    } while (0)

/* shared-shadow size of a replay block in 8-byte units (hr_stage_offset) */
static uint32_t smem_u64(const hr_ctx *c, uint64_t smem_words)
{
    return (c->cfg.options & HR_OPT_SMEM32) ? (uint32_t)((smem_words + 1) / 2) : (uint32_t)smem_words;
}

/* spill store: automatic capacity (hr.h, hr_config) and the tail words */
#define HR_SPILL_MIN (1u << 16)
#define HR_SPILL_AUTO_MAX (1u << 24)
#define HR_TAIL_WORDS 8

static hr_dev make_dev(hr_ctx *c, uint32_t kernel_id);

/* the device view for replaying kernel k of t: kdesc[5] is its warp tile */
static hr_dev make_kdev(hr_ctx *c, const hr_trace *t, uint32_t k)
{
    hr_dev d = make_dev(c, t->kernel_base + k);
    const uint64_t tl = t->kdesc[8ull * k + 5];
    d.tile_log2 = tl ? (uint32_t)tl : 5u;
    return d;
}

static hr_dev make_dev(hr_ctx *c, uint32_t kernel_id)
{
    hr_dev d;
    memset(&d, 0, sizeof d);
    d.gshadow = c->gshadow;
    d.gbase = c->gbase;
    d.gwords = c->gwords;
    d.glocal_words = c->glocal;
    d.ring = c->ring;
    d.ring_tail = c->tail;
    d.flags = c->tail + 1;
    d.spill = c->ring + c->cfg.ring_capacity;
    d.ovf = c->tail + 2;
    d.spill_cap = c->spill_cap;
    d.counters = c->counters;
    d.fsm = c->fsm;
    d.ring_cap = c->cfg.ring_capacity;
    d.kernel_id = kernel_id;
    d.shard_rank = c->shard_rank;
    d.shard_log2 = c->shard_log2;
    d.gran_log2 = c->gran_log2;
    d.wc_bits = c->cfg.wc_bits;
    d.wc_lsh = 32u - c->cfg.wc_bits;
    d.bc_max = (1u << c->cfg.bc_bits) - 1u;
    d.wc_max = (1u << c->cfg.wc_bits) - 1u;
    d.options = c->cfg.options;
    d.rep_bstride = c->rep_bstride;
    d.owned_only = c->cur_owned_only ? 1u : 0u;
    d.tile_log2 = c->online_tile_log2;
    d.rep_wstride = c->rep_wstride;
    if (d.options & HR_OPT_SMEM32) {            /* the 32-bit shared word holds bc:9, wc:8 */
        d.bc_max = std::min(d.bc_max, 511u);
        d.wc_max = std::min(d.wc_max, 255u);
    }
    if (d.options & HR_OPT_LAZY_RESET) {        /* the epoch tag takes bits [31:28] of the clock word */
        d.epoch_tag = c->epoch_tag;
        d.bc_max = std::min(d.bc_max, (1u << (28 - c->cfg.wc_bits)) - 1u);
    }
    return d;
}

extern "C" hr_status hr_init(const hr_config *cfg, hr_ctx **out)
{
    if (!out) return HR_E_ARG;
    *out = nullptr;
    hr_config def;
    def.state_bits = 5;
    def.tid_bits = 27;
    def.bc_bits = 16;
    def.wc_bits = 16;
    def.ring_capacity = 1u << 20;
    def.device = 0;
    def.options = 0;
    def.spill_capacity = 0;
    const hr_config &k = cfg ? *cfg : def;
    if (k.state_bits != 5 || k.tid_bits != 27 || k.bc_bits < 1 || k.wc_bits < 1 ||
        k.bc_bits + k.wc_bits != 32 || k.ring_capacity < 1 ||
        ((k.options & HR_OPT_SMEM32) && (k.options & HR_OPT_FINITE_HISTORY)) ||
        ((k.options & HR_OPT_LAZY_RESET) &&
         ((k.options & (HR_OPT_FINITE_HISTORY | HR_OPT_DOUBLE_SHADOW)) || k.wc_bits > 24)))
        return HR_E_ARG;
    hr_ctx *c = new (std::nothrow) hr_ctx;
    if (!c) return HR_E_NOMEM;
    c->cfg = k;
    c->device = k.device;
    hr_status st = HR_OK;
    do {
        cudaError_t e = cudaSetDevice(c->device);
        if (e != cudaSuccess) { st = fail(c, HR_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e)); break; }
        c->spill_cap = k.spill_capacity ? k.spill_capacity : HR_SPILL_MIN;
        if (cudaMalloc(&c->fsm, HR_FSM_SMEM_BYTES) != cudaSuccess ||
            cudaMalloc(&c->ring, sizeof(hr_race) * ((size_t)k.ring_capacity + c->spill_cap)) != cudaSuccess ||
            cudaMalloc(&c->tail, HR_TAIL_WORDS * sizeof(unsigned int)) != cudaSuccess ||
            cudaMalloc(&c->counters, 256 * sizeof(unsigned long long)) != cudaSuccess) {
            st = fail(c, HR_E_NOMEM, "device allocation failed in hr_init");
            break;
        }
        unsigned char host[HR_FSM_SMEM_BYTES];
        memset(host, 0, sizeof host);                /* the block scratch (HR_FSM_DROP_OFF) starts at 0 */
        host[HR_FSM_NOP_OFF + 4] = 3;                /* the NOP C32 record: word 0, op byte 3 */
        memcpy(host, hr_fsm_table_init, HR_FSM_BYTES);
        memcpy(host + HR_FSM_BYTES, hr_fsm_flags_init, 32);
        if (cudaMemcpy(c->fsm, host, HR_FSM_SMEM_BYTES, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemset(c->tail, 0, HR_TAIL_WORDS * sizeof(unsigned int)) != cudaSuccess ||
            cudaMemset(c->counters, 0, 256 * sizeof(unsigned long long)) != cudaSuccess) {
            st = fail(c, HR_E_CUDA, "hr_init upload failed");
            break;
        }
    } while (0);
    if (st != HR_OK) {
        hr_destroy(c);
        return st;
    }
    *out = c;
    return HR_OK;
}

extern "C" hr_status hr_set_shard_ex(hr_ctx *c, uint32_t rank, uint32_t count, uint32_t granule_log2)
{
    if (!c || count == 0 || count > 64 || (count & (count - 1)) || rank >= count || 
        granule_log2 > 24)
        return fail(c, HR_E_ARG, "hr_set_shard: bad rank/count/granule");
    if (c->gshadow) return fail(c, HR_E_STATE, "hr_set_shard after hr_shadow_alloc");
    c->gran_log2 = granule_log2;
    c->shard_rank = rank;
    c->shard_count = count;
    c->shard_log2 = 0;
    while ((1u << c->shard_log2) < count) c->shard_log2++;
    return HR_OK;
}

extern "C" hr_status hr_set_warp_tile(hr_ctx *c, uint32_t tile_log2)
{
    if (!c || tile_log2 > 5) return fail(c, HR_E_ARG, "hr_set_warp_tile: tile_log2 must be 0..5");
    c->online_tile_log2 = tile_log2 ? tile_log2 : 5u;
    return HR_OK;
}

extern "C" hr_status hr_set_representatives(hr_ctx *c, uint32_t block_stride, uint32_t warp_stride)
{
    if (!c || block_stride == 0 || warp_stride == 0) return HR_E_ARG;
    c->rep_bstride = block_stride;
    c->rep_wstride = warp_stride;
    return HR_OK;
}

extern "C" hr_status hr_set_shard(hr_ctx *c, uint32_t rank, uint32_t count)
{
    return hr_set_shard_ex(c, rank, count, 3);
}

extern "C" hr_status hr_shadow_alloc(hr_ctx *c, hr_space space, uint64_t base_word, uint64_t n_words,
                                     void **dev_region)
{
    if (!c) return HR_E_ARG;
    CU(cudaSetDevice(c->device));
    if (space == HR_SHARED) {
        const uint64_t per = (c->cfg.options & HR_OPT_FINITE_HISTORY) ? 16 : (c->cfg.options & HR_OPT_SMEM32) ? 4 : 8;
        if (base_word != 0 || n_words * per + HR_FSM_SMEM_BYTES + 32 * sizeof(hr_pool_smem) > 227 * 1024)
            return fail(c, HR_E_ARG, "shared shadow too large: %llu words", (unsigned long long)n_words);
        c->smem_words_max = (uint32_t)n_words;
        if (dev_region) *dev_region = nullptr;
        return HR_OK;
    }
    if (space != HR_GLOBAL || n_words == 0 || base_word + n_words > (1ull << 61))
        return fail(c, HR_E_ARG, "bad global region");
    for (int b = 0; b < 2; b++)
        if (c->gbuf[b]) { cudaFree(c->gbuf[b]); c->gbuf[b] = nullptr; }
    c->gshadow = nullptr;
    /* local slice: this shard's granules, packed in stripe order */
    uint64_t gran = (n_words + (1ull << c->gran_log2) - 1) >> c->gran_log2;
    uint64_t local_gran = (gran + c->shard_count - 1) >> c->shard_log2;
    uint64_t local = local_gran << c->gran_log2;
    c->double_shadow = (c->cfg.options & HR_OPT_DOUBLE_SHADOW) != 0;
    c->shadow_bytes = (c->cfg.options & HR_OPT_FINITE_HISTORY) ? 16 : 8;
    for (int b = 0; b < (c->double_shadow ? 2 : 1); b++) {
        if (cudaMalloc(&c->gbuf[b], local * c->shadow_bytes) != cudaSuccess)
            return fail(c, HR_E_NOMEM, "cudaMalloc(%llu B) for the global shadow failed",
                        (unsigned long long)(local * c->shadow_bytes));
        CU(cudaMemset(c->gbuf[b], 0, local * c->shadow_bytes));
        c->dirty[b] = false;
    }
    if (c->double_shadow && !c->side) {
        CU(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        for (int b = 0; b < 2; b++) {
            CU(cudaEventCreateWithFlags(&c->used_done[b], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c->reset_done[b], cudaEventDisableTiming));
            CU(cudaEventRecord(c->reset_done[b], c->side));
        }
    }
    if (!c->cfg.spill_capacity) {
        /* automatic spill: one record per local shadow word, within [2^16, 2^24] */
        const uint32_t want = (uint32_t)std::min<uint64_t>(HR_SPILL_AUTO_MAX, std::max<uint64_t>(HR_SPILL_MIN, local));
        if (want > c->spill_cap) {
            hr_race *nr = nullptr;
            const size_t ring_bytes = sizeof(hr_race) * (size_t)c->cfg.ring_capacity;
            if (cudaMalloc(&nr, ring_bytes + sizeof(hr_race) * (size_t)want) != cudaSuccess)
                return fail(c, HR_E_NOMEM, "spill store of %u records failed", want);
            CU(cudaDeviceSynchronize());
            /* keep what the ring and spill hold (hr_shadow_alloc is normally called before any kernel) */
            CU(cudaMemcpy(nr, c->ring, ring_bytes + sizeof(hr_race) * (size_t)c->spill_cap, cudaMemcpyDeviceToDevice));
            cudaFree(c->ring);
            c->ring = nr;
            c->spill_cap = want;
        }
    }
    c->scan_pending = false;
    c->gcur = 0;
    c->epoch_tag = 0;
    c->gshadow = c->gbuf[0];
    c->gbase = base_word;
    c->gwords = n_words;
    c->glocal = local;
    if (dev_region) *dev_region = c->gshadow;
    return HR_OK;
}

/* Zero one shadow buffer on stream `s`, with HR_OPT_TIMING events. */
static hr_status reset_buffer(hr_ctx *c, int b, cudaStream_t s)
{
    bool timing = c->cfg.options & HR_OPT_TIMING;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, s)); }
    CU(cudaMemsetAsync(c->gbuf[b], 0, c->glocal * c->shadow_bytes, s));
    if (timing) { CU(cudaEventRecord(e1, s)); c->ev_reset.push_back({e0, e1}); }
    c->dirty[b] = false;
    return HR_OK;
}

/* a9 overflow recovery of the kernel that used the current global shadow:
 * one launch, ordered after that kernel and before the shadow is reset or its
 * epoch tag retired; on the device it returns at once unless the kernel
 * dropped a global race record (hr_spill_scan_kernel). */
static hr_status enqueue_spill_scan(hr_ctx *c, cudaStream_t s)
{
    if (!c->scan_pending || !c->gshadow || c->shadow_bytes != 8) return HR_OK;
    c->scan_pending = false;
    const uint64_t blocks = std::min<uint64_t>(148ull * 4ull, (c->glocal + 255) / 256);
    c->launches++;
    hr_spill_scan_kernel<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, s>>>(
        make_dev(c, c->last_kernel), c->gshadow, c->glocal, (c->cfg.options & HR_OPT_LAZY_RESET) ? c->epoch_tag : 0u);
    CU(cudaGetLastError());
    return HR_OK;
}

extern "C" hr_status hr_kernel_begin(hr_ctx *c, void *stream)
{
    if (!c) return HR_E_ARG;
    CU(cudaSetDevice(c->device));
    c->stream = (cudaStream_t)stream;
    if (!c->gshadow) return HR_OK;
    if (hr_status st = enqueue_spill_scan(c, c->stream)) return st;
    if (c->cfg.options & HR_OPT_LAZY_RESET) {
        /* epoch tags 1..15: words of earlier kernels read as INIT (hr__live);
         * the shadow is zeroed for real only before a tag would be reused */
        if (c->dirty[0] && c->epoch_tag == 15) {
            hr_status st = reset_buffer(c, 0, c->stream);
            if (st) return st;
            c->epoch_tag = 0;
        }
        c->epoch_tag++;
        c->dirty[0] = true;
        return HR_OK;
    }
    if (!c->double_shadow) {
        if (c->dirty[0]) { hr_status st = reset_buffer(c, 0, c->stream); if (st) return st; }
        c->dirty[0] = true;
        return HR_OK;
    }
    /* double shadow: the last kernel's buffer is zeroed on the side stream
     * (after that kernel, overlapping the next one); the other becomes current */
    const int prev = c->gcur, next = prev ^ 1;
    if (c->dirty[prev]) {
        CU(cudaEventRecord(c->used_done[prev], c->stream));
        CU(cudaStreamWaitEvent(c->side, c->used_done[prev], 0));
        hr_status st = reset_buffer(c, prev, c->side);
        if (st) return st;
        CU(cudaEventRecord(c->reset_done[prev], c->side));
    }
    CU(cudaStreamWaitEvent(c->stream, c->reset_done[next], 0));
    c->gcur = next;
    c->gshadow = c->gbuf[next];
    c->dirty[next] = true;
    return HR_OK;
}

/* Kernel choice from warp-length tail, record density of the access rows and
 * the shared-space share (measured on C1, C3, C4, C5 and C5 shards —
 * profiles/r01_kernel_choice.md):
 *   max warp > 16x the mean warp (a few very long warps) -> pooled, 64 registers
 *   < 90% access records in access rows (sparse), unless a small grid
 *     (< 2048 warps: latency bound) at >= 50%          -> pooled, 32 registers
 *   otherwise a row kernel: 64 registers if >= 50% of the accesses are shared
 *   (SMEM shadow: issue bound) or the grid is small, else 32 registers
 *   (global shadow: occupancy hides the random DRAM latency).
 * HR_OPT_NO_POOL forces a row kernel, HR_OPT_POOL a pooled one (tail rule
 * kept), HR_OPT_POOL_WIDE the 64-register pooled kernel, HR_OPT_ROW_WIDE the
 * 64-register row kernel. */
enum { HR_K_ROW = 0, HR_K_POOL = 1, HR_K_POOL_WIDE = 2, HR_K_ROW_WIDE = 3 };

static int kernel_choice_rule(hr_ctx *c, double acc, double tot, double maxw, double sumw, double nwarps,
                              double shared);

static int kernel_choice(hr_ctx *c, double acc, double tot, double maxw, double sumw, double nwarps, double shared)
{
    const int k = kernel_choice_rule(c, acc, tot, maxw, sumw, nwarps, shared);
    if (getenv("HR_DEBUG_CHOICE"))
        fprintf(stderr, "hr kernel choice %d: acc %.0f tot %.0f shared %.0f maxw %.0f meanw %.1f nwarps %.0f\n", k, acc,
                tot, shared, maxw, nwarps > 0 ? sumw / nwarps : 0.0, nwarps);
    return k;
}

static int kernel_choice_rule(hr_ctx *c, double acc, double tot, double maxw, double sumw, double nwarps,
                              double shared)
{
    const uint32_t o = c->cfg.options;
    if (o & HR_OPT_ROW_WIDE) return HR_K_ROW_WIDE;
    if (o & HR_OPT_ROW_NARROW) return HR_K_ROW;
    const bool small = nwarps < 2048;
    /* dense traces: the 64-register row kernel when issue or latency bound (a
     * shared-shadow majority, or a small grid), else the 48-register one, which
     * beats the 64-register kernel on the random-DRAM-bound C5 (88.6 vs 90.2 ms,
     * round 2; in round 1 the 32-register one lost to 64 through spills) */
    const int row = (tot > 0 && shared >= 0.5 * acc) || small ? HR_K_ROW_WIDE : HR_K_ROW;
    if (o & HR_OPT_NO_POOL) return row;
    if (o & HR_OPT_POOL_WIDE) return HR_K_POOL_WIDE;
    const bool tail = nwarps > 0 && maxw > 16.0 * (sumw / nwarps);
    if (tail) return HR_K_POOL_WIDE;
    if (o & HR_OPT_POOL) return HR_K_POOL;
    const double dens = tot > 0 ? acc / tot : 1.0;
    if (dens < 0.9 && !(small && dens >= 0.5)) return HR_K_POOL;
    return row;
}

template <typename SRC>
static hr_status choose_kernel(hr_ctx *c, SRC src, const hr_trace *t, const uint64_t *woff, cudaStream_t s, int *kind)
{
    *kind = HR_K_ROW;
    if (t->n_rows == 0) return HR_OK;
    const void *rec = t->format == HR_TRACE_C32 ? (const void *)t->rec32 : (const void *)t->rec;
    auto &cc = c->choice_cache;
    if (cc.kind >= 0 && cc.rec == rec && cc.n_rows == t->n_rows && cc.woff == woff && cc.n_woff == t->n_warp_off &&
        cc.format == t->format && cc.options == c->cfg.options) {
        *kind = cc.kind;                       /* same trace replayed again: no probe, no sync */
        return HR_OK;
    }
    c->launches++;
    hr_density_kernel<SRC><<<1, 1024, 0, s>>>(src, t->n_rows, 2048, woff, t->n_warp_off, c->counters + 8);
    CU(cudaGetLastError());
    unsigned long long h[5] = {0, 0, 0, 0, 0};
    CU(cudaMemcpyAsync(h, c->counters + 8, sizeof h, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *kind = kernel_choice(c, (double)h[0], (double)h[1], (double)h[2], (double)h[3],
                          (double)(t->n_warp_off > 1 ? t->n_warp_off - 1 : 0), (double)h[4]);
    cc.rec = rec; cc.n_rows = t->n_rows; cc.woff = woff; cc.n_woff = t->n_warp_off;
    cc.format = t->format; cc.options = c->cfg.options; cc.kind = *kind;
    return HR_OK;
}

static hr_status check_kernel(hr_ctx *c, const hr_trace *t, uint32_t k)
{
    const uint64_t *kd = t->kdesc + 8ull * k;
    uint64_t blocks = kd[0], warps = kd[1], lanes = kd[2], smem_words = kd[3], woi = kd[4];
    if (blocks == 0) return HR_OK;
    if (blocks > (1ull << 17) || warps < 1 || warps > 32 || lanes < 1 || lanes > 32 || kd[5] > 4)
        return fail(c, HR_E_ARG, "kernel %u: grid %llux%llux%llu outside the 17/5/5-bit tid", k,
                    (unsigned long long)blocks, (unsigned long long)warps, (unsigned long long)lanes);
    if (smem_words > c->smem_words_max)
        return fail(c, HR_E_STATE, "kernel %u needs %llu shared shadow words (registered %u)", k,
                    (unsigned long long)smem_words, c->smem_words_max);
    if (woi + blocks * warps + 1 > t->n_warp_off) return fail(c, HR_E_ARG, "kernel %u: warp_off out of range", k);
    return HR_OK;
}

static hr_status reserve(hr_ctx *c, int i, size_t bytes);

/* A replay kernel with id `kid` was enqueued on the current global shadow. */
static void note_kernel(hr_ctx *c, uint32_t kid)
{
    c->last_kernel = kid;
    c->max_kernel = std::max(c->max_kernel, kid);
    c->have_kernel = true;
    c->scan_pending = true;                      /* its end-of-kernel spill scan is due */
}

/* Compacted replay of blocks [b0, b1) of kernel k (hr_compact.cuh): count and
 * scan the packed rows of every (warp, helper) stream, write them, replay them.
 * Two small synchronous reads size the buffers. */
template <typename SRC>
static hr_status launch_compact(hr_ctx *c, const hr_trace *t, uint32_t k, SRC src, const uint64_t *woff,
                                cudaStream_t s, uint64_t b0, uint64_t b1, uint32_t split, bool abl)
{
    const uint64_t *kd = t->kdesc + 8ull * k;
    const uint64_t warps = kd[1], lanes = kd[2], smem_words = kd[3], woi = kd[4];
    const uint32_t kid = t->kernel_base + k;
    hr_dev d = make_kdev(c, t, k);
    d.block_base = (uint32_t)b0;
    const uint64_t nw = (b1 - b0) * warps;
    const uint64_t *wk = woff + woi + b0 * warps;
    hr_status st;
    if ((st = reserve(c, 6, (nw + 1) * 8)) || (st = reserve(c, 7, (nw + 1) * 8))) return st;
    uint64_t *nseg = (uint64_t *)c->stage[6], *segoff = (uint64_t *)c->stage[7];
    c->launches++;
    hr_cmp_nseg_kernel<<<(unsigned)((nw + 1 + 255) / 256), 256, 0, s>>>(wk, nw, nseg);
    CU(cudaGetLastError());
    size_t tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nseg, segoff, (int64_t)(nw + 1), s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;                   /* scan-init + scan */
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, nseg, segoff, (int64_t)(nw + 1), s));
    uint64_t nsegs = 0;
    CU(cudaMemcpyAsync(&nsegs, segoff + nw, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const uint64_t ncnt = nsegs << split;
    if ((st = reserve(c, 8, (ncnt + 1) * 8)) || (st = reserve(c, 9, (ncnt + 1) * 8))) return st;
    uint64_t *cnt = (uint64_t *)c->stage[8], *rowoff = (uint64_t *)c->stage[9];
    CU(cudaMemsetAsync(cnt + ncnt, 0, 8, s));
    const unsigned wgrid = (unsigned)((nsegs * 32 + 255) / 256);
    if (nsegs) {
        c->launches++;
        hr_cmp_walk_kernel<false, SRC><<<wgrid, 256, 0, s>>>(d, src, wk, segoff, nw, (uint32_t)lanes, split, cnt,
                                                             nullptr, nullptr);
        CU(cudaGetLastError());
    }
    tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, rowoff, (int64_t)(ncnt + 1), s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;                   /* scan-init + scan */
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, cnt, rowoff, (int64_t)(ncnt + 1), s));
    uint64_t nrows = 0;
    CU(cudaMemcpyAsync(&nrows, rowoff + ncnt, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if ((st = reserve(c, 10, (size_t)std::max<uint64_t>(nrows, 1) * 256)) ||
        (st = reserve(c, 11, (size_t)std::max<uint64_t>(nrows, 1) * 32)))
        return st;
    uint64_t *orec = (uint64_t *)c->stage[10];
    uint8_t *otag = (uint8_t *)c->stage[11];
    if (nsegs) {
        c->launches++;
        hr_cmp_walk_kernel<true, SRC><<<wgrid, 256, 0, s>>>(d, src, wk, segoff, nw, (uint32_t)lanes, split, rowoff,
                                                            orec, otag);
        CU(cudaGetLastError());
    }
    const uint32_t nhw = (uint32_t)warps << split;
    const uint32_t stage_off = hr_stage_offset(false, nhw, smem_u64(c, smem_words));
    const size_t smem = (size_t)stage_off + hr_stage_bytes(nhw, 2u, 8u, hr_src_cmp::ROW_BYTES);
    if (smem > 227 * 1024)
        return fail(c, HR_E_ARG, "kernel %u: %zu bytes of shared memory per block (compacted replay)", k, smem);
    void (*kern)(hr_dev, hr_src_cmp, const uint64_t *, const uint64_t *, uint32_t, uint32_t, uint32_t, uint32_t,
                 uint32_t) = abl ? hr_replay_compact_kernel<true> : hr_replay_compact_kernel<false>;
    if (smem > 48 * 1024) CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    c->launches++;
    kern<<<(unsigned)(b1 - b0), nhw * 32u, smem, s>>>(d, hr_src_cmp{orec, otag}, segoff, rowoff, (uint32_t)warps,
                                                      (uint32_t)lanes, (uint32_t)smem_words, stage_off, split);
    CU(cudaGetLastError());
    note_kernel(c, kid);
    return HR_OK;
}

/* Stream-scheduled replay of blocks [b0, b1) of a barrier-free kernel k
 * without shared shadow (hr_streams.cuh).  Two small synchronous reads size
 * the buffers.  *fallback = true (nothing replayed) if the kernel holds a
 * barrier record. */
template <typename SRC>
static hr_status launch_streams(hr_ctx *c, const hr_trace *t, uint32_t k, SRC src, const uint64_t *woff,
                                cudaStream_t s, uint64_t b0, uint64_t b1, bool abl, bool *fallback)
{
    *fallback = false;
    const uint64_t *kd = t->kdesc + 8ull * k;
    const uint64_t warps = kd[1], lanes = kd[2], woi = kd[4];
    const uint32_t kid = t->kernel_base + k;
    hr_dev d = make_kdev(c, t, k);
    d.block_base = (uint32_t)b0;
    const uint64_t nw = (b1 - b0) * warps;
    const uint64_t *wk = woff + woi + b0 * warps;
    hr_status st;
    const size_t n1 = (size_t)(nw + 1);
    if ((st = reserve(c, 12, 3 * n1 * 8)) || (st = reserve(c, 13, 3 * n1 * 8)) || (st = reserve(c, 14, n1)) ||
        (st = reserve(c, 20, 64)))
        return st;
    uint64_t *cntw = (uint64_t *)c->stage[12], *offw = (uint64_t *)c->stage[13];
    uint64_t *nunit = cntw, *nstream = cntw + n1, *nslot = cntw + 2 * n1;
    uint64_t *unitoff = offw, *streamoff = offw + n1, *slotoff = offw + 2 * n1;
    uint8_t *hlog2 = (uint8_t *)c->stage[14];
    unsigned int *ctr = (unsigned int *)c->stage[20];   /* [0] barrier flag, [1] next stream */
    c->launches++;
    hr_st_plan_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, s>>>(wk, nw, nunit, nstream, nslot, hlog2);
    CU(cudaGetLastError());
    size_t tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nunit, unitoff, (int64_t)n1, s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    for (int i = 0; i < 3; i++) {
        size_t tb = tmp;
        c->launches += 2;
        CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tb, cntw + i * n1, offw + i * n1, (int64_t)n1, s));
    }
    uint64_t tot[3];
    for (int i = 0; i < 3; i++) CU(cudaMemcpyAsync(&tot[i], offw + i * n1 + nw, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemsetAsync(ctr, 0, 8, s));
    CU(cudaStreamSynchronize(s));
    const uint64_t nunits = tot[0], ns = tot[1], nslots = tot[2];
    if (ns >= 0xffffffffull) { *fallback = true; return HR_OK; }
    if ((st = reserve(c, 15, (size_t)(nslots + 1) * 8)) || (st = reserve(c, 16, (size_t)(nslots + 1) * 8)) ||
        (st = reserve(c, 17, (size_t)(ns + 1) * 16)) || (st = reserve(c, 18, (size_t)(ns + 1) * 16)) ||
        (st = reserve(c, 19, (size_t)(ns + 1) * 8)))
        return st;
    uint64_t *cnt = (uint64_t *)c->stage[15], *eoff = (uint64_t *)c->stage[16];
    uint64_t *plen = (uint64_t *)c->stage[17], *sbase = plen + (ns + 1);
    uint32_t *swarp = (uint32_t *)c->stage[18], *skey = swarp + (ns + 1), *sid = skey + (ns + 1),
             *stot = sid + (ns + 1);
    uint32_t *skey2 = (uint32_t *)c->stage[19], *order = skey2 + (ns + 1);
    CU(cudaMemsetAsync(cnt + nslots, 0, 8, s));
    const unsigned ugrid = (unsigned)((nunits * 32 + HR_ST_WALK_WARPS * 32 - 1) / (HR_ST_WALK_WARPS * 32));
    if (nunits) {
        c->launches++;
        hr_st_walk_kernel<false, SRC><<<ugrid, HR_ST_WALK_WARPS * 32, 0, s>>>(
            d, src, wk, nw, unitoff, slotoff, streamoff, hlog2, (uint32_t)lanes, cnt, nullptr, nullptr, nullptr,
            nullptr, ctr);
        CU(cudaGetLastError());
    }
    tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, eoff, (int64_t)(nslots + 1), s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, cnt, eoff, (int64_t)(nslots + 1), s));
    c->launches++;
    hr_st_stream_kernel<<<(unsigned)((ns + 1 + 255) / 256), 256, 0, s>>>(streamoff, unitoff, slotoff, nw, ns, eoff,
                                                                         plen, swarp, skey, sid, stot);
    CU(cudaGetLastError());
    tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, plen, sbase, (int64_t)(ns + 1), s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, plen, sbase, (int64_t)(ns + 1), s));
    uint64_t entries = 0;
    unsigned int barrier = 0;
    CU(cudaMemcpyAsync(&entries, sbase + ns, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&barrier, ctr, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (barrier) { *fallback = true; return HR_OK; }
    if ((st = reserve(c, 10, (size_t)std::max<uint64_t>(entries, 32) * 8)) ||
        (st = reserve(c, 11, (size_t)std::max<uint64_t>(entries, 32))))
        return st;
    uint64_t *orec = (uint64_t *)c->stage[10];
    uint8_t *otag = (uint8_t *)c->stage[11];
    /* longest stream first */
    tmp = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp, skey, skey2, sid, order, (int)ns, 0, 32, s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2 + 4;
    CU(cub::DeviceRadixSort::SortPairs(c->stage[5], tmp, skey, skey2, sid, order, (int)ns, 0, 32, s));
    if (nunits) {
        c->launches++;
        hr_st_walk_kernel<true, SRC><<<ugrid, HR_ST_WALK_WARPS * 32, 0, s>>>(
            d, src, wk, nw, unitoff, slotoff, streamoff, hlog2, (uint32_t)lanes, nullptr, eoff, sbase, orec, otag,
            ctr);
        CU(cudaGetLastError());
    }
    c->launches++;
    hr_st_pad_kernel<<<(unsigned)((ns * 32 + 255) / 256), 256, 0, s>>>(sbase, stot, ns, orec, otag);
    CU(cudaGetLastError());
    const size_t smem = hr_streams_smem();
    void (*kern)(hr_dev, hr_src_cmp, const uint64_t *, const uint32_t *, const uint32_t *, uint32_t, uint32_t,
                 unsigned int *) = abl ? hr_replay_streams_kernel<true> : hr_replay_streams_kernel<false>;
    if (smem > 48 * 1024) CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    c->launches++;
    kern<<<(unsigned)(dev_sms * HR_ST_CTAS), HR_ST_WARPS * 32, smem, s>>>(d, hr_src_cmp{orec, otag}, sbase, order, swarp,
                                                                (uint32_t)ns, (uint32_t)warps, ctr + 1);
    CU(cudaGetLastError());
    note_kernel(c, kid);
    return HR_OK;
}

/* Address-binned replay of blocks [b0, b1) of kernel k (hr_binned.cuh): count
 * walk, scan, write walk, bucket-major persistent replay.  One synchronous
 * read sizes the entry buffer.  *fallback = true (nothing replayed) if an
 * entry cannot hold the clocks. */
template <typename SRC>
static hr_status launch_binned(hr_ctx *c, const hr_trace *t, uint32_t k, SRC src, const uint64_t *woff,
                               cudaStream_t s, uint64_t b0, uint64_t b1, bool abl, bool *fallback)
{
    *fallback = false;
    const uint64_t *kd = t->kdesc + 8ull * k;
    const uint64_t warps = kd[1], lanes = kd[2], woi = kd[4];
    const uint32_t kid = t->kernel_base + k;
    hr_dev d = make_kdev(c, t, k);
    d.block_base = (uint32_t)b0;
    const uint32_t nb = (uint32_t)(b1 - b0);
    const uint32_t nbk = (uint32_t)((c->glocal + (1ull << HR_BN_BITS) - 1) >> HR_BN_BITS);
    const uint64_t ns = (uint64_t)nbk * nb;
    hr_status st;
    /* 64-bit counts: the scan's sum type is the input's, and C5 has 2^32 entries */
    if ((st = reserve(c, 22, (size_t)(ns + 1) * 8)) || (st = reserve(c, 23, (size_t)(ns + 1) * 8)) ||
        (st = reserve(c, 20, 64)))
        return st;
    uint64_t *cnt = (uint64_t *)c->stage[22];
    uint64_t *off = (uint64_t *)c->stage[23];
    unsigned int *status = (unsigned int *)c->stage[20];
    unsigned long long *next = (unsigned long long *)((char *)c->stage[20] + 8);
    CU(cudaMemsetAsync(c->stage[20], 0, 16, s));
    CU(cudaMemsetAsync(cnt + ns, 0, 8, s));
    const size_t wsm = hr_bn_walk_smem(nbk);
    void (*wk0)(hr_dev, SRC, const uint64_t *, uint32_t, uint32_t, uint32_t, uint32_t, uint64_t *, const uint64_t *,
                uint64_t *, unsigned int *) = hr_bn_walk_kernel<false, SRC>;
    void (*wk1)(hr_dev, SRC, const uint64_t *, uint32_t, uint32_t, uint32_t, uint32_t, uint64_t *, const uint64_t *,
                uint64_t *, unsigned int *) = hr_bn_walk_kernel<true, SRC>;
    if (wsm > 48 * 1024) {
        CU(cudaFuncSetAttribute(wk0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
        CU(cudaFuncSetAttribute(wk1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    }
    const unsigned wgrid = (nb + HR_BN_WALK_WARPS - 1) / HR_BN_WALK_WARPS;
    const uint64_t *wkoff = woff + woi + b0 * warps;
    c->launches++;
    wk0<<<wgrid, HR_BN_WALK_WARPS * 32, wsm, s>>>(d, src, wkoff, nb, (uint32_t)warps, (uint32_t)lanes, nbk, cnt,
                                                   nullptr, nullptr, status);
    CU(cudaGetLastError());
    size_t tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, (int64_t)(ns + 1), s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, cnt, off, (int64_t)(ns + 1), s));
    uint64_t entries = 0;
    unsigned int hst = 0;
    CU(cudaMemcpyAsync(&entries, off + ns, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&hst, status, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (hst & HR_BN_ST_CANCEL) { *fallback = true; return HR_OK; }
    if ((st = reserve(c, 21, (size_t)std::max<uint64_t>(entries, 1) * 8))) return st;
    uint64_t *ent = (uint64_t *)c->stage[21];
    c->launches++;
    wk1<<<wgrid, HR_BN_WALK_WARPS * 32, wsm, s>>>(d, src, wkoff, nb, (uint32_t)warps, (uint32_t)lanes, nbk, cnt, off,
                                                   ent, status);
    CU(cudaGetLastError());
    const size_t rsm = hr_bn_replay_smem();
    void (*rk)(hr_dev, const uint64_t *, const uint64_t *, uint32_t, uint64_t, unsigned long long *) =
        abl ? hr_bn_replay_kernel<true> : hr_bn_replay_kernel<false>;
    if (rsm > 48 * 1024) CU(cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    c->launches++;
    rk<<<(unsigned)(dev_sms * 2), HR_BN_WARPS * 32, rsm, s>>>(d, ent, off, nb, ns, next);
    CU(cudaGetLastError());
    note_kernel(c, kid);
    return HR_OK;
}

/* Hybrid binned replay (HR_OPT_HYBRID, hr_hybrid.cuh), first half: count the
 * (bucket, block) runs of kernel k's blocks [b0, b1), choose the binned buckets,
 * lay the runs out bucket-major and point d at them (d.hy_*: the row replay
 * then appends those buckets' accesses).  One synchronous read sizes the
 * entries.  d is left untouched (plain row replay) if nothing is binned or the
 * clocks do not fit an entry. */
template <typename SRC>
static hr_status hybrid_prepare(hr_ctx *c, const hr_trace *t, uint32_t k, SRC src, const uint64_t *woff, cudaStream_t s,
                                uint64_t b0, uint64_t b1, hr_dev &d)
{
    const uint64_t *kd = t->kdesc + 8ull * k;
    const uint64_t warps = kd[1], lanes = kd[2], woi = kd[4];
    const uint32_t nb = (uint32_t)(b1 - b0);
    const uint32_t nbk = (uint32_t)((c->glocal + (1ull << HR_HY_BITS) - 1) >> HR_HY_BITS);
    if (nbk == 0 || nbk > HR_HY_MAXBK || nb == 0) return HR_OK;
    const uint64_t nruns = (uint64_t)nbk * nb;
    hr_status st;
    if ((st = reserve(c, 22, (size_t)(nruns + 1) * 8)) || (st = reserve(c, 23, (size_t)(nruns + 1) * 8)) ||
        (st = reserve(c, 20, (size_t)nbk * 16 + 512)))
        return st;
    unsigned long long *cnt = (unsigned long long *)c->stage[22];
    unsigned long long *off = (unsigned long long *)c->stage[23];
    unsigned long long *stat = (unsigned long long *)c->stage[20];
    uint32_t *map = (uint32_t *)((char *)c->stage[20] + (size_t)nbk * 16);
    unsigned int *clk = (unsigned int *)((char *)c->stage[20] + (size_t)nbk * 16 + 128);
    CU(cudaMemsetAsync(c->stage[20], 0, (size_t)nbk * 16 + 512, s));
    CU(cudaMemsetAsync(cnt + nruns, 0, 8, s));
    const uint64_t *wk = woff + woi + b0 * warps;
    if (c->cfg.options & HR_OPT_BIN_ALL) {
        CU(cudaMemsetAsync(map, 0xff, (nbk + 31) / 32 * 4, s));           /* every bucket (tests) */
    } else {
        /* the choice from a sample of 1 in 64 blocks: >= 2^16 accesses scaled, >= half scattered */
        const uint32_t stride = nb >= 4096 ? 64u : 1u;
        c->launches += 2;
        hr_hy_count_kernel<true, SRC><<<(nb + stride - 1) / stride, (unsigned)(warps * 32), (size_t)nbk * 8, s>>>(
            d, src, wk, (uint32_t)warps, (uint32_t)lanes, nbk, nb, stride, map, cnt, stat, clk);
        CU(cudaGetLastError());
        hr_hy_decide_kernel<<<(nbk + 255) / 256, 256, 0, s>>>(stat, nbk, map, std::max<unsigned long long>(1ull, (1ull << 16) / stride));
        CU(cudaGetLastError());
    }
    c->launches++;
    hr_hy_count_kernel<false, SRC><<<nb, (unsigned)(warps * 32), (size_t)nbk * 4, s>>>(
        d, src, wk, (uint32_t)warps, (uint32_t)lanes, nbk, nb, 1u, map, cnt, stat, clk);
    CU(cudaGetLastError());
    size_t tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, (int64_t)(nruns + 1), s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, cnt, off, (int64_t)(nruns + 1), s));
    unsigned long long total = 0;
    unsigned int hclk[2] = {0, 0};
    CU(cudaMemcpyAsync(&total, off + nruns, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(hclk, clk, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    /* exact counts need clocks that never overflow (a thread past its limit stops
     * checking) and that fit an entry */
    if (total == 0 || hclk[0] > HR_HY_BC_MAX || hclk[0] >= d.bc_max || hclk[1] > HR_HY_WC_MAX || hclk[1] >= d.wc_max)
        return HR_OK;
    if ((st = reserve(c, 21, (size_t)total * 8))) return st;
    d.hy_map = map;
    d.hy_off = off;
    d.hy_ent = (unsigned long long *)c->stage[21];
    d.hy_nb = nb;
    d.hy_nbk = nbk;
    return HR_OK;
}

/* second half: check the binned runs bucket by bucket (after the row replay) */
static hr_status hybrid_replay(hr_ctx *c, const hr_dev &d, cudaStream_t s)
{
    hr_status st;
    if ((st = reserve(c, 20, (size_t)d.hy_nbk * 16 + 512))) return st;
    unsigned long long *next = (unsigned long long *)((char *)c->stage[20] + (size_t)d.hy_nbk * 16 + 256);
    CU(cudaMemsetAsync(next, 0, 8, s));
    const size_t rsm = hr_hy_replay_smem(d.hy_nbk);
    if (rsm > 48 * 1024) CU(cudaFuncSetAttribute(hr_hy_replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    c->launches++;
    hr_hy_replay_kernel<<<(unsigned)(dev_sms * HR_HY_MINB), HR_HY_WARPS * 32, rsm, s>>>(d, d.hy_ent, d.hy_off, d.hy_nb, d.hy_nbk,
                                                                             next);
    CU(cudaGetLastError());
    return HR_OK;
}

/* Binned replay (HR_OPT_BINNED) for kernels without shared shadow and at most
 * HR_BN_MAXBK shadow buckets. */
static bool use_binned(const hr_ctx *c, int kind, uint64_t smem_words)
{
    const uint32_t o = c->cfg.options;
    if (smem_words != 0 || c->shadow_bytes != 8 || !c->gshadow || (o & HR_OPT_NO_BINNED)) return false;
    const uint64_t nbk = (c->glocal + (1ull << HR_BN_BITS) - 1) >> HR_BN_BITS;
    if (nbk > HR_BN_MAXBK) return false;
    /* opt-in: measured slower than the row replay on C5 (DESIGN.md §5 item 17) */
    (void)kind;
    return (o & HR_OPT_BINNED) != 0;
}

/* One launch over simulated blocks [b0, b1) of kernel k (the whole kernel in
 * one launch for device traces; block-range chunks for host traces — blocks
 * are unordered by happens-before, so chunked launches replay the same kernel). */
template <typename SRC>
static hr_status launch(hr_ctx *c, const hr_trace *t, uint32_t k, SRC src, const uint64_t *woff, cudaStream_t s,
                        int kind, uint64_t b0, uint64_t b1)
{
    const uint64_t *kd = t->kdesc + 8ull * k;
    uint64_t warps = kd[1], lanes = kd[2], smem_words = kd[3], woi = kd[4];
    uint32_t kid = t->kernel_base + k;
    hr_dev d = make_kdev(c, t, k);
    d.block_base = (uint32_t)b0;
    if (c->shadow_bytes == 16) {                               /* finite-history baseline */
        size_t smem = HR_FSM_SMEM_BYTES + smem_words * 16;
        if (smem > 48 * 1024)
            CU(cudaFuncSetAttribute(hr_fh_replay_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        bool timing = c->cfg.options & HR_OPT_TIMING;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, s)); }
        c->launches++;
        hr_fh_replay_kernel<SRC><<<(unsigned)(b1 - b0), (unsigned)(warps * 32), smem, s>>>(
            d, src, woff + woi + b0 * warps, (uint32_t)warps, (uint32_t)lanes, (uint32_t)smem_words);
        CU(cudaGetLastError());
        if (timing) { CU(cudaEventRecord(e1, s)); c->ev_kernel.push_back({e0, e1}); }
        note_kernel(c, kid);
        return HR_OK;
    }
    /* the pooled and block-serial walks (pooled, compacted, streams, binned, bserial)
     * keep one warp clock per simulated warp: tile kernels, whose tiles carry their
     * own clocks, take the row kernel (64 registers) */
    const bool tiles = kd[5] != 0;
    if (tiles && (kind == HR_K_POOL || kind == HR_K_POOL_WIDE)) kind = HR_K_ROW_WIDE;
    const bool pool = kind == HR_K_POOL || kind == HR_K_POOL_WIDE;
    const bool abl0 = c->cfg.options & (HR_OPT_NO_COALESCE | HR_OPT_NO_FASTEXIT | HR_OPT_SPECULATE | HR_OPT_SMEM32);
    if (use_binned(c, kind, smem_words) && !(c->cfg.options & HR_OPT_BSERIAL) && !tiles) {
        bool timing = c->cfg.options & HR_OPT_TIMING;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, s)); }
        bool fallback = true;
        hr_status st = launch_binned(c, t, k, src, woff, s, b0, b1, abl0, &fallback);
        if (st) return st;
        if (!fallback) {
            if (timing) { CU(cudaEventRecord(e1, s)); c->ev_kernel.push_back({e0, e1}); }
            return HR_OK;
        }
        if (timing) { c->ev_pool.push_back(e0); c->ev_pool.push_back(e1); }
    }
    if (!src.aligned_ok()) return fail(c, HR_E_ARG, "trace records must be 16-byte aligned (TMA staging)");
    /* the wide row kernel stages 16-row C32 chunks: if that and the shadow do not
     * fit one block's shared memory, the narrow row kernel (4-row chunks) runs */
    if (kind == HR_K_ROW_WIDE &&
        (size_t)hr_stage_offset(false, (uint32_t)warps, smem_u64(c, smem_words)) +
                hr_stage_bytes((uint32_t)warps, hr_stage_cfg<true, false, SRC::ROW_BYTES>::NB,
                               hr_stage_cfg<true, false, SRC::ROW_BYTES>::CH, SRC::ROW_BYTES) > 227 * 1024)
        kind = HR_K_ROW;
    const bool wide = kind == HR_K_POOL_WIDE || kind == HR_K_ROW_WIDE;
    const uint32_t nb = wide ? hr_stage_cfg<true>::NB : hr_stage_cfg<false>::NB;
    const uint32_t ch = kind == HR_K_ROW_WIDE ? hr_stage_cfg<true, false, SRC::ROW_BYTES>::CH
                        : wide               ? hr_stage_cfg<true, true, SRC::ROW_BYTES>::CH
                                             : hr_stage_cfg<false>::CH;
    /* long-tailed grids (wide pooled kernel): split each simulated warp over up
     * to 4 CUDA warps of the block (hr_replay_kernel); HR_SPLIT_LOG2 overrides */
    uint32_t split = 0;
    if (kind == HR_K_POOL_WIDE)
        while (split < 2 && (warps << (split + 1)) <= 32) split++;
    if (pool)
        if (const char *e = getenv("HR_SPLIT_LOG2")) {
            split = (uint32_t)atoi(e);
            if (split > 2) split = 2;                           /* <= 4 helpers (hr_cmp_walk_kernel) */
            while (split && (warps << split) > 32) split--;
        }
    if (!pool) split = 0;
    const uint32_t nhw = (uint32_t)warps << split;
    const bool abl = c->cfg.options & (HR_OPT_NO_COALESCE | HR_OPT_NO_FASTEXIT | HR_OPT_SPECULATE | HR_OPT_SMEM32);
    if (kind == HR_K_POOL && t->format == HR_TRACE_U64 && (c->cfg.options & HR_OPT_BSERIAL) && !tiles) {
        const size_t bsm = hr_bserial_smem((uint32_t)smem_words, (c->cfg.options & HR_OPT_SMEM32) != 0);
        if (bsm <= 227 * 1024) {
            void (*bk)(hr_dev, const uint64_t *, const uint64_t *, uint32_t, uint32_t, uint32_t, uint32_t) =
                abl ? hr_replay_bserial_kernel<true> : hr_replay_bserial_kernel<false>;
            if (bsm > 48 * 1024) CU(cudaFuncSetAttribute(bk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
            bool timing = c->cfg.options & HR_OPT_TIMING;
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, s)); }
            const uint32_t nb = (uint32_t)(b1 - b0);
            c->launches++;
            bk<<<(nb + HR_BS_WARPS - 1) / HR_BS_WARPS, HR_BS_WARPS * 32, bsm, s>>>(
                d, t->rec, woff + woi + b0 * warps, nb, (uint32_t)warps, (uint32_t)lanes, (uint32_t)smem_words);
            CU(cudaGetLastError());
            if (timing) { CU(cudaEventRecord(e1, s)); c->ev_kernel.push_back({e0, e1}); }
            note_kernel(c, kid);
            return HR_OK;
        }
    }
    if (kind == HR_K_POOL_WIDE && !(c->cfg.options & HR_OPT_NO_COMPACT)) {
        bool timing = c->cfg.options & HR_OPT_TIMING;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, s)); }
        bool fallback = true;
        hr_status st = HR_OK;
        if (smem_words == 0 && !(c->cfg.options & HR_OPT_NO_STREAMS))
            st = launch_streams(c, t, k, src, woff, s, b0, b1, abl, &fallback);
        if (!st && fallback) st = launch_compact(c, t, k, src, woff, s, b0, b1, split, abl);
        if (st) return st;
        if (timing) { CU(cudaEventRecord(e1, s)); c->ev_kernel.push_back({e0, e1}); }
        return HR_OK;
    }
    size_t smem = (size_t)hr_stage_offset(pool, nhw, smem_u64(c, smem_words)) + hr_stage_bytes(nhw, nb, ch, SRC::ROW_BYTES);
    bool timing = c->cfg.options & HR_OPT_TIMING;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, s)); }   /* the hybrid passes included */
    if ((c->cfg.options & HR_OPT_HYBRID) && !pool && !tiles && !abl && c->shadow_bytes == 8 && c->gshadow) {
        if (hr_status st = hybrid_prepare(c, t, k, src, woff, s, b0, b1, d)) return st;
        if (d.hy_map) {
            d.hy_sa_off = (uint32_t)smem;               /* the block's run positions after the staging */
            smem += (size_t)d.hy_nbk * 8;
        }
    }
    if (smem > 227 * 1024)
        return fail(c, HR_E_ARG, "kernel %u: %zu bytes of shared memory per block (shadow %llu words + staging)", k, smem,
                    (unsigned long long)smem_words);
    void (*kern)(hr_dev, SRC, const uint64_t *, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t);
    if (abl)
        kern = pool ? (wide ? hr_replay_kernel<true, true, true, SRC> : hr_replay_kernel<true, false, true, SRC>)
                    : (wide ? hr_replay_kernel<false, true, true, SRC> : hr_replay_kernel<false, false, true, SRC>);
    else
        kern = pool ? (wide ? hr_replay_kernel<true, true, false, SRC> : hr_replay_kernel<true, false, false, SRC>)
                    : (wide ? hr_replay_kernel<false, true, false, SRC> : hr_replay_kernel<false, false, false, SRC>);
    const uint32_t stage_off = hr_stage_offset(pool, nhw, smem_u64(c, smem_words));
    if (smem > 48 * 1024) CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    c->launches++;
    kern<<<(unsigned)(b1 - b0), nhw * 32u, smem, s>>>(d, src, woff + woi + b0 * warps, (uint32_t)warps, (uint32_t)lanes,
                                                       (uint32_t)smem_words, stage_off, split);
    CU(cudaGetLastError());
    if (d.hy_map)
        if (hr_status st = hybrid_replay(c, d, s)) return st;
    if (timing) { CU(cudaEventRecord(e1, s)); c->ev_kernel.push_back({e0, e1}); }
    note_kernel(c, kid);
    return HR_OK;
}

template <typename SRC>
static hr_status replay(hr_ctx *c, const hr_trace *t, SRC src, const uint64_t *woff, cudaStream_t s)
{
    int kind = HR_K_ROW;
    hr_status st = choose_kernel(c, src, t, woff, s, &kind);
    if (st) return st;
    c->last_kind = kind;
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        if ((st = check_kernel(c, t, k))) return st;
        const uint64_t blocks = t->kdesc[8ull * k];
        if (!blocks) continue;
        if ((st = hr_kernel_begin(c, s))) return st;
        if ((st = launch(c, t, k, src, woff, s, kind, 0, blocks))) return st;
    }
    return HR_OK;
}

static bool trace_ok(const hr_trace *t)
{
    if (!t) return false;
    if (!t->n_kernels) return true;
    if (!t->kdesc || !t->warp_off) return false;
    if (t->format == HR_TRACE_U64) return t->rec != nullptr;
    if (t->format == HR_TRACE_C32) return t->rec32 && t->recop;
    if (t->format == HR_TRACE_PACKED) return t->packed && t->pack_off;
    if (t->format == HR_TRACE_POOLED) return t->rec && t->recop;
    return false;
}

static hr_status dispatch(hr_ctx *c, const hr_trace *t, const uint64_t *rec, const uint32_t *rec32,
                          const uint8_t *recop, const uint64_t *woff)
{
    if (t->format == HR_TRACE_C32) {
        hr_src_c32 src{rec32, recop};
        return replay(c, t, src, woff, c->stream);
    }
    hr_src_u64 src{rec};
    return replay(c, t, src, woff, c->stream);
}

static hr_status replay_packed(hr_ctx *c, const hr_trace *t, bool host);

/* HR_TRACE_POOLED (include/hr.h): every kernel through the compacted replay
 * kernel, one stream per simulated warp (rows = the warp's pools). */
static hr_status replay_pooled(hr_ctx *c, const hr_trace *t)
{
    const hr_src_cmp src{t->rec, (const uint8_t *)t->recop};
    if (!src.aligned_ok()) return fail(c, HR_E_ARG, "pooled trace records must be 16-byte aligned (TMA staging)");
    const bool abl = c->cfg.options & (HR_OPT_NO_COALESCE | HR_OPT_NO_FASTEXIT | HR_OPT_SPECULATE | HR_OPT_SMEM32);
    c->last_kind = HR_K_POOL;
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        hr_status st = check_kernel(c, t, k);
        if (st) return st;
        const uint64_t *kd = t->kdesc + 8ull * k;
        const uint64_t blocks = kd[0], warps = kd[1], lanes = kd[2], smem_words = kd[3], woi = kd[4];
        if (!blocks) continue;
        if (kd[5]) return fail(c, HR_E_ARG, "pooled trace: kernel %u declares warp tiles (one clock per warp)", k);
        if ((st = hr_kernel_begin(c, c->stream))) return st;
        const uint32_t kid = t->kernel_base + k;
        hr_dev d = make_kdev(c, t, k);
        const uint32_t nhw = (uint32_t)warps;
        const uint32_t stage_off = hr_stage_offset(false, nhw, smem_u64(c, smem_words));
        const size_t smem = (size_t)stage_off + hr_stage_bytes(nhw, 2u, 8u, hr_src_cmp::ROW_BYTES);
        if (smem > 227 * 1024) return fail(c, HR_E_ARG, "kernel %u: %zu bytes of shared memory per block", k, smem);
        /* 32-register variant unless HR_OPT_ROW_WIDE (measured on C5 shards) */
        const bool narrow = !(c->cfg.options & HR_OPT_ROW_WIDE);
        void (*kern)(hr_dev, hr_src_cmp, const uint64_t *, const uint64_t *, uint32_t, uint32_t, uint32_t, uint32_t,
                     uint32_t) = abl ? (narrow ? hr_replay_compact_kernel<true, true> : hr_replay_compact_kernel<true>)
                                     : (narrow ? hr_replay_compact_kernel<false, true> : hr_replay_compact_kernel<false>);
        if (smem > 48 * 1024) CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const bool timing = c->cfg.options & HR_OPT_TIMING;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing) { e0 = get_event(c); e1 = get_event(c); CU(cudaEventRecord(e0, c->stream)); }
        c->launches++;
        kern<<<(unsigned)blocks, nhw * 32u, smem, c->stream>>>(d, src, nullptr, t->warp_off + woi, (uint32_t)warps,
                                                                (uint32_t)lanes, (uint32_t)smem_words, stage_off, 0u);
        CU(cudaGetLastError());
        if (timing) { CU(cudaEventRecord(e1, c->stream)); c->ev_kernel.push_back({e0, e1}); }
        note_kernel(c, kid);
    }
    return HR_OK;
}

__global__ void hr_pool_woff_kernel(const uint64_t *__restrict__ segoff, const uint64_t *__restrict__ rowoff,
                                    uint64_t nw, uint64_t base, uint64_t *__restrict__ out)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= nw) out[i] = base + rowoff[segoff[i]];
}

template <typename SRC>
static hr_status pool_trace(hr_ctx *c, const hr_trace *t, SRC src, uint64_t *rec_out, uint8_t *tag_out,
                            uint64_t cap_rows, uint64_t *woff_out, uint64_t *rows, cudaStream_t s)
{
    uint64_t base = 0;
    hr_status st;
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        const uint64_t *kd = t->kdesc + 8ull * k;
        const uint64_t blocks = kd[0], warps = kd[1], lanes = kd[2], woi = kd[4];
        if (!blocks) continue;
        if (blocks > (1ull << 17) || warps < 1 || warps > 32 || lanes < 1 || lanes > 32 ||
            woi + blocks * warps + 1 > t->n_warp_off)
            return fail(c, HR_E_ARG, "hr_pool_trace: kernel %u: bad grid or warp_off range", k);
        if (kd[5]) return fail(c, HR_E_ARG, "hr_pool_trace: kernel %u declares warp tiles (replay it as rows)", k);
        hr_dev d = make_kdev(c, t, k);
        const uint64_t nw = blocks * warps;
        const uint64_t *wk = t->warp_off + woi;
        if ((st = reserve(c, 6, (nw + 1) * 8)) || (st = reserve(c, 7, (nw + 1) * 8))) return st;
        uint64_t *nseg = (uint64_t *)c->stage[6], *segoff = (uint64_t *)c->stage[7];
        c->launches++;
        hr_cmp_nseg_kernel<<<(unsigned)((nw + 1 + 255) / 256), 256, 0, s>>>(wk, nw, nseg);
        CU(cudaGetLastError());
        size_t tmp = 0;
        CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nseg, segoff, (int64_t)(nw + 1), s));
        if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
        c->launches += 2;
        CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, nseg, segoff, (int64_t)(nw + 1), s));
        uint64_t nsegs = 0;
        CU(cudaMemcpyAsync(&nsegs, segoff + nw, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if ((st = reserve(c, 8, (nsegs + 1) * 8)) || (st = reserve(c, 9, (nsegs + 1) * 8))) return st;
        uint64_t *cnt = (uint64_t *)c->stage[8], *rowoff = (uint64_t *)c->stage[9];
        CU(cudaMemsetAsync(cnt + nsegs, 0, 8, s));
        const unsigned wgrid = (unsigned)((nsegs * 32 + 255) / 256);
        if (nsegs) {
            c->launches++;
            hr_cmp_walk_kernel<false, SRC><<<wgrid, 256, 0, s>>>(d, src, wk, segoff, nw, (uint32_t)lanes, 0u, cnt,
                                                                 nullptr, nullptr);
            CU(cudaGetLastError());
        }
        tmp = 0;
        CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, rowoff, (int64_t)(nsegs + 1), s));
        if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
        c->launches += 2;
        CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, cnt, rowoff, (int64_t)(nsegs + 1), s));
        uint64_t nrows = 0;
        CU(cudaMemcpyAsync(&nrows, rowoff + nsegs, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (rec_out) {
            if (base + nrows > cap_rows) return fail(c, HR_E_ARG, "hr_pool_trace: %llu rows > cap %llu",
                                                     (unsigned long long)(base + nrows), (unsigned long long)cap_rows);
            if (nsegs) {
                c->launches++;
                hr_cmp_walk_kernel<true, SRC><<<wgrid, 256, 0, s>>>(d, src, wk, segoff, nw, (uint32_t)lanes, 0u, rowoff,
                                                                    rec_out + base * 32, tag_out + base * 32);
                CU(cudaGetLastError());
            }
            c->launches++;
            hr_pool_woff_kernel<<<(unsigned)((nw + 1 + 255) / 256), 256, 0, s>>>(segoff, rowoff, nw, base,
                                                                                 woff_out + woi);
            CU(cudaGetLastError());
            CU(cudaStreamSynchronize(s));
        }
        base += nrows;
    }
    *rows = base;
    return HR_OK;
}

extern "C" hr_status hr_pool_trace(hr_ctx *c, const hr_trace *in, uint64_t *rec_out, uint8_t *tag_out,
                                   uint64_t cap_rows, uint64_t *warp_off_out, uint64_t *rows, void *stream)
{
    if (!c || !in || !rows || !trace_ok(in) || (in->format != HR_TRACE_U64 && in->format != HR_TRACE_C32) ||
        (rec_out && (!tag_out || !warp_off_out)))
        return fail(c, HR_E_ARG, "hr_pool_trace: bad arguments (U64 or C32 device trace required)");
    CU(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    c->stream = s;
    if (in->format == HR_TRACE_C32)
        return pool_trace(c, in, hr_src_c32{in->rec32, in->recop}, rec_out, tag_out, cap_rows, warp_off_out, rows, s);
    return pool_trace(c, in, hr_src_u64{in->rec}, rec_out, tag_out, cap_rows, warp_off_out, rows, s);
}

/* HR_TRACE_F_SHARD_OWNED for the duration of one replay call */
struct owned_scope {
    hr_ctx *c;
    owned_scope(hr_ctx *ctx, const hr_trace *t) : c(ctx) { c->cur_owned_only = (t->flags & HR_TRACE_F_SHARD_OWNED) != 0; }
    ~owned_scope() { c->cur_owned_only = false; }
};

extern "C" hr_status hr_replay_trace(hr_ctx *c, const hr_trace *t, void *stream)
{
    if (!c || !trace_ok(t)) return fail(c, HR_E_ARG, "null or malformed trace");
    CU(cudaSetDevice(c->device));
    c->stream = (cudaStream_t)stream;
    owned_scope own(c, t);
    if (t->format == HR_TRACE_PACKED) return replay_packed(c, t, false);
    if (t->format == HR_TRACE_POOLED) return replay_pooled(c, t);
    return dispatch(c, t, t->rec, t->rec32, t->recop, t->warp_off);
}

static hr_status reserve(hr_ctx *c, int i, size_t bytes)
{
    if (bytes > c->stage_cap[i]) {
        if (c->stage[i]) cudaFree(c->stage[i]);
        c->stage[i] = nullptr;
        c->stage_cap[i] = 0;
        if (cudaMalloc(&c->stage[i], bytes) != cudaSuccess) return fail(c, HR_E_NOMEM, "staging %zu bytes failed", bytes);
        c->stage_cap[i] = bytes;
    }
    return HR_OK;
}

/* Host-side version of the kernel-choice probe. */
static int host_kernel_choice(hr_ctx *c, const hr_trace *t)
{
    uint64_t acc = 0, tot = 0, sh = 0;
    for (uint32_t s = 0; s < 2048 && t->n_rows; s++) {
        const double u = ((double)s + fmod((double)s * 0.6180339887498949, 1.0)) / 2048.0;   /* as hr_density_kernel */
        uint64_t row = (uint64_t)(u * (double)t->n_rows);
        if (row >= t->n_rows) break;
        uint32_t ops[32], spcs[32];
        bool barrier = false;
        for (uint32_t l = 0; l < 32; l++) {
            uint64_t w;
            if (t->format == HR_TRACE_C32) {
                ops[l] = t->recop[row * 32 + l] & 3u;
                spcs[l] = (t->recop[row * 32 + l] >> 2) & 1u;
                w = t->rec32[row * 32 + l];
            } else {
                ops[l] = (uint32_t)(t->rec[row * 32 + l] >> 62);
                spcs[l] = (uint32_t)(t->rec[row * 32 + l] >> 61) & 1u;
                w = t->rec[row * 32 + l] & ((1ull << 61) - 1);
            }
            barrier |= ops[l] == 3u && w != 0u;
        }
        if (barrier) continue;                     /* as hr_density_kernel: access rows only */
        for (uint32_t l = 0; l < 32; l++) {
            acc += ops[l] != 3u;
            sh += ops[l] != 3u && spcs[l];
            tot++;
        }
    }
    double mx = 0, sm = 0;
    for (uint64_t i = 0; i + 1 < t->n_warp_off; i++) {
        const double len = t->warp_off[i + 1] >= t->warp_off[i] ? (double)(t->warp_off[i + 1] - t->warp_off[i]) : 0.0;
        mx = len > mx ? len : mx;
        sm += len;
    }
    return kernel_choice(c, (double)acc, (double)tot, mx, sm, (double)(t->n_warp_off > 1 ? t->n_warp_off - 1 : 0),
                         (double)sh);
}

/* Host traces: records are copied in block-range chunks on a copy stream and
 * each chunk is replayed as soon as it lands, so the PCIe transfer of chunk
 * i+1 overlaps the replay of chunk i. */
static size_t host_chunk_bytes()
{
    size_t chunk_bytes = (size_t)1 << 30;                       /* ~1 GiB of records per chunk */
    if (const char *e = getenv("HR_HOST_CHUNK_BYTES")) chunk_bytes = (size_t)strtoull(e, nullptr, 10);
    return chunk_bytes < 256 ? 256 : chunk_bytes;
}

/* PACKED traces (host or device resident): per kernel, block-range chunks of
 * ~chunk_bytes of DECODED rows; each chunk's packed bytes are copied on the
 * copy stream (host traces), decoded on `stream` into one U64 staging buffer,
 * then replayed from it.  Decode and replay are ordered on `stream`, so one
 * decode buffer serves every chunk; only the copies run ahead. */
static hr_status replay_packed(hr_ctx *c, const hr_trace *t, bool host)
{
    hr_status st;
    const uint64_t nwo = t->n_warp_off;
    std::vector<uint64_t> hwoff_v, hpoff_v;
    const uint64_t *hwoff = t->warp_off, *hpoff = t->pack_off;
    const uint64_t *dwoff = t->warp_off, *dpoff = t->pack_off;
    const uint8_t *dpacked = t->packed;
    if (!host) {                                   /* plan chunks from host copies of the offsets */
        hwoff_v.resize(nwo);
        hpoff_v.resize(nwo);
        CU(cudaMemcpyAsync(hwoff_v.data(), t->warp_off, nwo * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(hpoff_v.data(), t->pack_off, nwo * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        hwoff = hwoff_v.data();
        hpoff = hpoff_v.data();
    }
    const size_t chunk_rows = host_chunk_bytes() / 256 ? host_chunk_bytes() / 256 : 1;
    /* chunk plan and the largest chunk, before any buffer is (re)allocated */
    struct chunk { uint32_t k; uint64_t b0, b1; };
    std::vector<chunk> plan;
    uint64_t max_rows = 0;
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        if ((st = check_kernel(c, t, k))) return st;
        const uint64_t *kd = t->kdesc + 8ull * k;
        const uint64_t blocks = kd[0], warps = kd[1], woi = kd[4];
        if (!blocks) continue;
        const uint64_t krows = hwoff[woi + blocks * warps] - hwoff[woi];
        uint64_t nchunks = (krows + chunk_rows - 1) / chunk_rows;
        if (nchunks < 1) nchunks = 1;
        if (nchunks > blocks) nchunks = blocks;
        for (uint64_t ci = 0; ci < nchunks; ci++) {
            const uint64_t b0 = blocks * ci / nchunks, b1 = blocks * (ci + 1) / nchunks;
            const uint64_t s0 = woi + b0 * warps, s1 = woi + b1 * warps;
            if (hwoff[s1] < hwoff[s0] || hpoff[s1] < hpoff[s0])
                return fail(c, HR_E_ARG, "packed trace: decreasing warp_off or pack_off");
            plan.push_back({k, b0, b1});
            max_rows = std::max(max_rows, hwoff[s1] - hwoff[s0]);
        }
    }
    if ((st = reserve(c, 2, (size_t)std::max<uint64_t>(max_rows, 1) * 256))) return st;
    uint64_t *dec = (uint64_t *)c->stage[2];
    if (host) {
        const uint64_t total = hpoff[nwo - 1] + HR_PACK_SLACK;
        if ((st = reserve(c, 0, (size_t)nwo * 8))) return st;
        if ((st = reserve(c, 3, (size_t)nwo * 8))) return st;
        if ((st = reserve(c, 1, (size_t)total))) return st;
        if (!c->copy) CU(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        cudaEvent_t start = get_event(c);
        CU(cudaEventRecord(start, c->stream));
        CU(cudaStreamWaitEvent(c->copy, start, 0));
        c->ev_pool.push_back(start);
        CU(cudaMemcpyAsync(c->stage[0], t->warp_off, (size_t)nwo * 8, cudaMemcpyHostToDevice, c->copy));
        CU(cudaMemcpyAsync(c->stage[3], t->pack_off, (size_t)nwo * 8, cudaMemcpyHostToDevice, c->copy));
        dwoff = (const uint64_t *)c->stage[0];
        dpoff = (const uint64_t *)c->stage[3];
        dpacked = (const uint8_t *)c->stage[1];
    }
    int kind = -1;
    int64_t cur_k = -1;
    for (const chunk &ch : plan) {
        const uint64_t *kd = t->kdesc + 8ull * ch.k;
        const uint64_t warps = kd[1], woi = kd[4];
        const uint64_t s0 = woi + ch.b0 * warps, s1 = woi + ch.b1 * warps;
        const uint64_t rbase = hwoff[s0], rows = hwoff[s1] - hwoff[s0];
        if ((int64_t)ch.k != cur_k) {
            if ((st = hr_kernel_begin(c, c->stream))) return st;
            cur_k = ch.k;
        }
        if (host) {
            if (hpoff[s1] > hpoff[s0])
                CU(cudaMemcpyAsync((uint8_t *)c->stage[1] + hpoff[s0], t->packed + hpoff[s0], hpoff[s1] - hpoff[s0],
                                   cudaMemcpyHostToDevice, c->copy));
            cudaEvent_t landed = get_event(c);
            CU(cudaEventRecord(landed, c->copy));
            CU(cudaStreamWaitEvent(c->stream, landed, 0));
            c->ev_pool.push_back(landed);
        }
        if (s1 > s0) {
            const uint64_t threads = (s1 - s0) * 32;
            c->launches++;
            hr_unpack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, c->stream>>>(dpacked, dpoff, dwoff, s0, s1,
                                                                                       rbase, dec);
            CU(cudaGetLastError());
        }
        hr_src_u64 src{dec - rbase * 32};
        if (kind < 0) {
            /* kernel choice: density of the first decoded chunk, tail of all warps */
            if (rows) {
                c->launches++;
                hr_density_kernel<hr_src_u64><<<1, 1024, 0, c->stream>>>(hr_src_u64{dec}, rows, 2048, dwoff, nwo,
                                                                        c->counters + 8);
                CU(cudaGetLastError());
                unsigned long long h[5] = {0, 0, 0, 0, 0};
                CU(cudaMemcpyAsync(h, c->counters + 8, sizeof h, cudaMemcpyDeviceToHost, c->stream));
                CU(cudaStreamSynchronize(c->stream));
                kind = kernel_choice(c, (double)h[0], (double)h[1], (double)h[2], (double)h[3],
                                     (double)(nwo > 1 ? nwo - 1 : 0), (double)h[4]);
            } else {
                kind = HR_K_ROW;
            }
            c->last_kind = kind;
        }
        if ((st = launch(c, t, ch.k, src, dwoff, c->stream, kind, ch.b0, ch.b1))) return st;
    }
    return HR_OK;
}

extern "C" hr_status hr_pack_trace(hr_ctx *c, const hr_trace *in, uint8_t *out, uint64_t cap, uint64_t *pack_off,
                                   uint64_t *bytes, void *stream)
{
    if (!c || !in || !pack_off || !bytes || in->format != HR_TRACE_U64 || !in->rec || !in->warp_off ||
        in->n_warp_off < 1)
        return fail(c, HR_E_ARG, "hr_pack_trace: bad arguments (U64 device trace required)");
    CU(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    c->stream = s;
    hr_status st;
    const uint64_t n = in->n_warp_off;
    const size_t sizes_bytes = ((size_t)n * 8 + 15) & ~(size_t)15;
    if ((st = reserve(c, 4, sizes_bytes + 16))) return st;
    uint64_t *sizes = (uint64_t *)c->stage[4];
    unsigned int *err = (unsigned int *)((char *)c->stage[4] + sizes_bytes);
    CU(cudaMemsetAsync(err, 0, 4, s));
    const unsigned grid = (unsigned)((n * 32 + 255) / 256);
    c->launches++;
    hr_pack_size_kernel<<<grid, 256, 0, s>>>(in->rec, in->warp_off, n, sizes, err);
    CU(cudaGetLastError());
    size_t tmp = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, sizes, pack_off, (int64_t)n, s));
    if ((st = reserve(c, 5, tmp ? tmp : 1))) return st;
    c->launches += 2;                   /* scan-init + scan */
    CU(cub::DeviceScan::ExclusiveSum(c->stage[5], tmp, sizes, pack_off, (int64_t)n, s));
    uint64_t total = 0;
    unsigned int herr = 0;
    CU(cudaMemcpyAsync(&total, pack_off + (n - 1), 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (herr) return fail(c, HR_E_ARG, "hr_pack_trace: decreasing warp_off");
    *bytes = total + HR_PACK_SLACK;
    if (!out) return HR_OK;
    if (cap < total + HR_PACK_SLACK) return fail(c, HR_E_ARG, "hr_pack_trace: cap %llu < %llu", (unsigned long long)cap,
                                                 (unsigned long long)(total + HR_PACK_SLACK));
    c->launches++;
    hr_pack_write_kernel<<<grid, 256, 0, s>>>(in->rec, in->warp_off, n, pack_off, out);
    CU(cudaGetLastError());
    CU(cudaMemsetAsync(out + total, 0, HR_PACK_SLACK, s));
    CU(cudaStreamSynchronize(s));
    return HR_OK;
}

extern "C" hr_status hr_unpack_trace(hr_ctx *c, const hr_trace *in, uint64_t *rec_out, void *stream)
{
    if (!c || !in || !rec_out || in->format != HR_TRACE_PACKED || !in->packed || !in->pack_off || !in->warp_off)
        return fail(c, HR_E_ARG, "hr_unpack_trace: bad arguments (PACKED device trace required)");
    CU(cudaSetDevice(c->device));
    if (in->n_warp_off < 2) return HR_OK;
    const uint64_t nseg = in->n_warp_off - 1;
    c->launches++;
    hr_unpack_kernel<<<(unsigned)((nseg * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        in->packed, in->pack_off, in->warp_off, 0, nseg, 0, rec_out);
    CU(cudaGetLastError());
    return HR_OK;
}

extern "C" hr_status hr_replay_trace_host(hr_ctx *c, const hr_trace *t, void *stream)
{
    if (!c || !trace_ok(t)) return fail(c, HR_E_ARG, "null or malformed trace");
    CU(cudaSetDevice(c->device));
    c->stream = (cudaStream_t)stream;
    owned_scope own(c, t);
    if (t->format == HR_TRACE_PACKED) return replay_packed(c, t, true);
    if (t->format == HR_TRACE_POOLED) return fail(c, HR_E_ARG, "hr_replay_trace_host: POOLED traces are device only");
    const bool c32 = t->format == HR_TRACE_C32;
    hr_status st;
    if ((st = reserve(c, 0, (size_t)t->n_warp_off * 8))) return st;
    if ((st = reserve(c, 1, (size_t)t->n_rows * (c32 ? 128 : 256)))) return st;
    if (c32 && (st = reserve(c, 2, (size_t)t->n_rows * 32))) return st;
    if (!c->copy) CU(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    /* the copy stream may overwrite staging only after earlier work on `stream` */
    cudaEvent_t start = get_event(c);
    CU(cudaEventRecord(start, c->stream));
    CU(cudaStreamWaitEvent(c->copy, start, 0));
    c->ev_pool.push_back(start);
    CU(cudaMemcpyAsync(c->stage[0], t->warp_off, (size_t)t->n_warp_off * 8, cudaMemcpyHostToDevice, c->copy));
    const int kind = host_kernel_choice(c, t);
    c->last_kind = kind;
    const uint64_t *dwoff = (const uint64_t *)c->stage[0];
    const size_t chunk_bytes = host_chunk_bytes();
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        if ((st = check_kernel(c, t, k))) return st;
        const uint64_t *kd = t->kdesc + 8ull * k;
        const uint64_t blocks = kd[0], warps = kd[1], woi = kd[4];
        if (!blocks) continue;
        if ((st = hr_kernel_begin(c, c->stream))) return st;
        const uint64_t krows = t->warp_off[woi + blocks * warps] - t->warp_off[woi];
        const uint64_t row_bytes = c32 ? 160 : 256;
        uint64_t nchunks = (krows * row_bytes + chunk_bytes - 1) / chunk_bytes;
        if (nchunks < 1) nchunks = 1;
        if (nchunks > blocks) nchunks = blocks;
        for (uint64_t ci = 0; ci < nchunks; ci++) {
            const uint64_t b0 = blocks * ci / nchunks, b1 = blocks * (ci + 1) / nchunks;
            const uint64_t r0 = t->warp_off[woi + b0 * warps], r1 = t->warp_off[woi + b1 * warps];
            if (r1 > r0) {
                if (c32) {
                    CU(cudaMemcpyAsync((uint32_t *)c->stage[1] + r0 * 32, t->rec32 + r0 * 32, (r1 - r0) * 128,
                                       cudaMemcpyHostToDevice, c->copy));
                    CU(cudaMemcpyAsync((uint8_t *)c->stage[2] + r0 * 32, t->recop + r0 * 32, (r1 - r0) * 32,
                                       cudaMemcpyHostToDevice, c->copy));
                } else {
                    CU(cudaMemcpyAsync((uint64_t *)c->stage[1] + r0 * 32, t->rec + r0 * 32, (r1 - r0) * 256,
                                       cudaMemcpyHostToDevice, c->copy));
                }
            }
            cudaEvent_t landed = get_event(c);
            CU(cudaEventRecord(landed, c->copy));
            CU(cudaStreamWaitEvent(c->stream, landed, 0));
            c->ev_pool.push_back(landed);
            if (c32) st = launch(c, t, k, hr_src_c32{(const uint32_t *)c->stage[1], (const uint8_t *)c->stage[2]},
                                 dwoff, c->stream, kind, b0, b1);
            else st = launch(c, t, k, hr_src_u64{(const uint64_t *)c->stage[1]}, dwoff, c->stream, kind, b0, b1);
            if (st) return st;
        }
    }
    return HR_OK;
}

static bool race_less(const hr_race &a, const hr_race &b)
{
    if (a.kernel != b.kernel) return a.kernel < b.kernel;
    if (a.space != b.space) return a.space < b.space;
    if (a.block != b.block) return a.block < b.block;
    return a.word < b.word;
}

/* Sort race records by (kernel, space, block, word): LSD radix sort on a
 * 128-bit key (hi = kernel | space | block, lo = word), 16-bit digits, digits
 * that are constant across the input skipped.  O(n) per live digit. */
static void sort_races(std::vector<hr_race> &v)
{
    const size_t n = v.size();
    if (n < 2) return;
    struct K { uint64_t hi, lo; uint32_t idx; };
    std::vector<K> a(n), b(n);
    for (size_t i = 0; i < n; i++) {
        a[i].hi = ((uint64_t)v[i].kernel << 33) | ((uint64_t)v[i].space << 32) | (uint64_t)v[i].block;
        a[i].lo = v[i].word;
        a[i].idx = (uint32_t)i;
    }
    std::vector<size_t> cnt(65536);
    for (int d = 0; d < 8; d++) {
        const bool hi = d >= 4;
        const int sh = 16 * (d & 3);
        auto dig = [&](const K &k) { return (size_t)(((hi ? k.hi : k.lo) >> sh) & 0xffff); };
        std::fill(cnt.begin(), cnt.end(), 0);
        for (size_t i = 0; i < n; i++) cnt[dig(a[i])]++;
        if (cnt[dig(a[0])] == n) continue;             /* constant digit */
        size_t acc = 0;
        for (size_t j = 0; j < 65536; j++) { size_t t = cnt[j]; cnt[j] = acc; acc += t; }
        for (size_t i = 0; i < n; i++) b[cnt[dig(a[i])]++] = a[i];
        a.swap(b);
    }
    std::vector<hr_race> out(n);
    for (size_t i = 0; i < n; i++) out[i] = v[a[i].idx];
    v.swap(out);
}

/* Race-record sort on the device (large reports): stable LSD radix sort by
 * word, then by kernel | space | block, then a gather.  Same order as
 * sort_races. */
__global__ void hr_race_keys_kernel(const hr_race *__restrict__ r, uint32_t n, uint64_t *__restrict__ lo,
                                    uint32_t *__restrict__ idx)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    lo[i] = r[i].word;
    idx[i] = i;
}

__global__ void hr_race_hikeys_kernel(const hr_race *__restrict__ r, const uint32_t *__restrict__ idx, uint32_t n,
                                      uint64_t *__restrict__ hi)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const hr_race &x = r[idx[i]];
    hi[i] = ((uint64_t)x.kernel << 33) | ((uint64_t)x.space << 32) | (uint64_t)x.block;
}

__global__ void hr_race_gather_kernel(const hr_race *__restrict__ r, const uint32_t *__restrict__ idx, uint32_t n,
                                      hr_race *__restrict__ out)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = r[idx[i]];
}

/* Sorted records -> one per address (kernel, space, block, word), keeping the
 * widest scope (a RACE_BLOCK entry plus its later RACE_GRID upgrade, or a ring
 * record plus its shadow-scan duplicate); returns the unique count. */
static size_t unique_races(std::vector<hr_race> &v)
{
    size_t m = 0;
    for (size_t i = 0; i < v.size(); i++) {
        if (m && !race_less(v[m - 1], v[i]) && !race_less(v[i], v[m - 1])) {
            if (v[i].scope > v[m - 1].scope) {
                uint8_t sc = v[i].scope;
                if (v[m - 1].first_kind == 0xff) v[m - 1] = v[i];
                v[m - 1].scope = sc;
            }
            continue;
        }
        v[m++] = v[i];
    }
    return m;
}

/* HR_REPORT_PROFILE=1: stderr line with the host time of each part of a slow
 * (> 5 ms) hr_report call (diagnostic for host-side stalls). */
static double hr__now_ms()
{
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}
static double hr__prof[16];
static int hr__prof_n = 0;
static bool hr__prof_on = false;
#define HR_PROF_MARK() do { if (hr__prof_on && hr__prof_n < 16) hr__prof[hr__prof_n++] = hr__now_ms(); } while (0)

static hr_status sort_races_device(hr_ctx *c, uint32_t n, std::vector<hr_race> &v)
{
    cudaStream_t s = c->stream;
    /* scratch: lo keys (2 buffers), hi keys (2), idx (2), sorted records */
    const size_t nb = (size_t)n;
    size_t off[8];
    size_t tot = 0;
    const size_t sz[7] = {nb * 8, nb * 8, nb * 8, nb * 8, nb * 4, nb * 4, nb * sizeof(hr_race)};
    for (int i = 0; i < 7; i++) { off[i] = tot; tot += (sz[i] + 255) & ~(size_t)255; }
    size_t t1 = 0, t2 = 0;
    /* CUB's temp-size query does device-attribute / occupancy lookups that
     * measured up to 0.8 s on a busy host now and then: cache it per size */
    if (c->sort_tmp_n == n) {
        t1 = c->sort_tmp_bytes;
    } else {
        CU(cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr, (uint32_t *)nullptr,
                                           (uint32_t *)nullptr, (int)n, 0, 64, s));
        c->sort_tmp_n = n;
        c->sort_tmp_bytes = t1;
    }
    t2 = t1;
    off[7] = tot;
    tot += std::max(t1, t2);
    hr_status st = reserve(c, 5, tot);
    if (st) return st;
    HR_PROF_MARK();
    char *b = (char *)c->stage[5];
    uint64_t *lo0 = (uint64_t *)(b + off[0]), *lo1 = (uint64_t *)(b + off[1]);
    uint64_t *hi0 = (uint64_t *)(b + off[2]), *hi1 = (uint64_t *)(b + off[3]);
    uint32_t *ix0 = (uint32_t *)(b + off[4]), *ix1 = (uint32_t *)(b + off[5]);
    hr_race *sorted = (hr_race *)(b + off[6]);
    void *tmp = b + off[7];
    const unsigned g = (n + 255) / 256;
    c->launches++;
    hr_race_keys_kernel<<<g, 256, 0, s>>>(c->ring, n, lo0, ix0);
    CU(cudaGetLastError());
    HR_PROF_MARK();
    size_t tb = t1;
    c->launches += 10;                  /* onesweep, 64-bit keys: histogram + scan + 8 passes */
    CU(cub::DeviceRadixSort::SortPairs(tmp, tb, lo0, lo1, ix0, ix1, (int)n, 0, 64, s));
    HR_PROF_MARK();
    c->launches++;
    hr_race_hikeys_kernel<<<g, 256, 0, s>>>(c->ring, ix1, n, hi0);
    CU(cudaGetLastError());
    HR_PROF_MARK();
    tb = t1;
    c->launches += 10;                  /* onesweep, 64-bit keys: histogram + scan + 8 passes */
    CU(cub::DeviceRadixSort::SortPairs(tmp, tb, hi0, hi1, ix1, ix0, (int)n, 0, 64, s));
    HR_PROF_MARK();
    c->launches++;
    hr_race_gather_kernel<<<g, 256, 0, s>>>(c->ring, ix0, n, sorted);
    CU(cudaGetLastError());
    HR_PROF_MARK();
    if (n > c->rep_cap) {
        if (c->rep_host) cudaFreeHost(c->rep_host);
        c->rep_host = nullptr;
        c->rep_cap = 0;
        if (cudaHostAlloc((void **)&c->rep_host, nb * sizeof(hr_race), cudaHostAllocDefault) != cudaSuccess)
            return fail(c, HR_E_NOMEM, "pinned report staging of %zu records failed", nb);
        c->rep_cap = n;
    }
    CU(cudaMemcpyAsync(c->rep_host, sorted, nb * sizeof(hr_race), cudaMemcpyDeviceToHost, s));
    HR_PROF_MARK();
    CU(cudaStreamSynchronize(s));
    v.assign(c->rep_host, c->rep_host + n);
    return HR_OK;
}


/* ---- asynchronous report (hr_report_async): a13 on the device ----
 * The ring is sorted at its full capacity (entries past the tail get the
 * largest keys, so the tail count never has to reach the host), run heads of
 * equal (kernel, space, block, word) are flagged and scanned, and each head
 * writes its merged record (widest scope) straight into pinned host memory. */
__global__ void hr_arep_keys_kernel(const hr_race *__restrict__ r, const unsigned int *__restrict__ tail, uint32_t cap,
                                    uint64_t *__restrict__ lo, uint32_t *__restrict__ idx)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cap) return;
    const uint32_t n = min(*tail, cap);
    lo[i] = i < n ? r[i].word : ~0ull;
    idx[i] = i;
}

__global__ void hr_arep_hikeys_kernel(const hr_race *__restrict__ r, const unsigned int *__restrict__ tail,
                                      const uint32_t *__restrict__ idx, uint32_t cap, uint64_t *__restrict__ hi)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cap) return;
    const uint32_t n = min(*tail, cap);
    const uint32_t j = idx[i];
    if (j >= n) { hi[i] = ~0ull; return; }
    const hr_race &x = r[j];
    hi[i] = ((uint64_t)x.kernel << 33) | ((uint64_t)x.space << 32) | (uint64_t)x.block;
}

__device__ __forceinline__ bool hr__same_addr(const hr_race &a, const hr_race &b)
{
    return a.kernel == b.kernel && a.space == b.space && a.block == b.block && a.word == b.word;
}

__global__ void hr_arep_heads_kernel(const hr_race *__restrict__ r, const unsigned int *__restrict__ tail,
                                     const uint32_t *__restrict__ idx, uint32_t cap, uint32_t *__restrict__ head)
{
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= cap) return;
    const uint32_t n = min(*tail, cap);
    head[p] = p < n && (p == 0 || !hr__same_addr(r[idx[p]], r[idx[p - 1]])) ? 1u : 0u;
}

/* one thread per run head: the run's first record with the widest scope of
 * the run (as unique_races on the host) */
__global__ void hr_arep_emit_kernel(const hr_race *__restrict__ r, const unsigned int *__restrict__ tail,
                                    const uint32_t *__restrict__ idx, const uint32_t *__restrict__ head,
                                    const uint32_t *__restrict__ pos, uint32_t cap, hr_race *out, uint32_t out_cap,
                                    uint32_t *hdr)
{
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = min(*tail, cap);
    if (p == 0) {
        hdr[0] = n ? pos[n - 1] + head[n - 1] : 0u;
        hdr[1] = tail[1];
        hdr[2] = *tail;
        hdr[3] = tail[2] | tail[3];             /* spill records or unspilled drops: collect -> hr_report */
    }
    if (p >= n || !head[p] || pos[p] >= out_cap) return;
    hr_race x = r[idx[p]];
    for (uint32_t q = p + 1; q < n && !head[q]; q++) {
        const hr_race &y = r[idx[q]];
        if (y.scope > x.scope) {
            const uint8_t sc = y.scope;
            if (x.first_kind == 0xff) x = y;
            x.scope = sc;
        }
    }
    out[pos[p]] = x;
}

/* The small-set report in one CTA: when the ring holds at most HR_AREP_SMALL
 * records, sort their (hi, lo, ring index) keys — the order of the two stable
 * CUB sorts — with a bitonic network in shared memory, flag the run heads,
 * scan them and emit each run's merged record, as the kernels above do.  A
 * larger ring sets the graph's conditional so that the CUB path (the IF body)
 * runs instead; the host never learns the count.  Cost: one launch, O(n log^2 n)
 * shared-memory work, instead of sorting the whole ring capacity every report. */
#define HR_AREP_SMALL 8192u
#define HR_AREP_SMALL_THREADS 1024u
static constexpr size_t HR_AREP_SMALL_SMEM = (size_t)HR_AREP_SMALL * 20u;

__global__ void __launch_bounds__(HR_AREP_SMALL_THREADS)
    hr_arep_small_kernel(const hr_race *__restrict__ r, const unsigned int *__restrict__ tail, uint32_t cap,
                         hr_race *out, uint32_t out_cap, uint32_t *hdr, cudaGraphConditionalHandle big,
                         unsigned long long *big_launches, uint32_t body_launches)
{
    extern __shared__ __align__(16) unsigned char hr_smem[];
    uint64_t *khi = reinterpret_cast<uint64_t *>(hr_smem), *klo = khi + HR_AREP_SMALL;
    uint32_t *kix = reinterpret_cast<uint32_t *>(klo + HR_AREP_SMALL);
    __shared__ uint32_t wsum[HR_AREP_SMALL_THREADS / 32u];
    const uint32_t n = min(*tail, cap);
    if (n > HR_AREP_SMALL) {
        if (threadIdx.x == 0) {
            cudaGraphSetConditional(big, 1u);
            atomicAdd(big_launches, (unsigned long long)body_launches);
        }
        return;
    }
    uint32_t np = 1;
    while (np < n) np <<= 1;
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
        if (i < n) {
            const hr_race &x = r[i];
            khi[i] = ((uint64_t)x.kernel << 33) | ((uint64_t)x.space << 32) | (uint64_t)x.block;
            klo[i] = x.word;
        } else {
            khi[i] = klo[i] = ~0ull;                  /* padding: after every record */
        }
        kix[i] = i;
    }
    __syncthreads();
    /* bitonic network over np keys; pair q of a stage compares i and i + j */
    for (uint32_t k = 2; k <= np; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t q = threadIdx.x; q < np / 2u; q += blockDim.x) {
                const uint32_t i = (q / j) * 2u * j + (q % j), l = i + j;
                const uint64_t ah = khi[i], bh = khi[l], al = klo[i], bl = klo[l];
                const uint32_t ai = kix[i], bi = kix[l];
                const bool gt = ah > bh || (ah == bh && (al > bl || (al == bl && ai > bi)));
                if (gt == ((i & k) == 0u)) {
                    khi[i] = bh; khi[l] = ah;
                    klo[i] = bl; klo[l] = al;
                    kix[i] = bi; kix[l] = ai;
                }
            }
            __syncthreads();
        }
    /* run heads over contiguous chunks, a block-wide exclusive scan of their counts */
    const uint32_t ch = (n + blockDim.x - 1u) / blockDim.x;
    const uint32_t p0 = min(n, threadIdx.x * ch), p1 = min(n, p0 + ch);
    uint32_t heads = 0;
    for (uint32_t p = p0; p < p1; p++) heads += (p == 0u || !hr__same_addr(r[kix[p]], r[kix[p - 1]])) ? 1u : 0u;
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t inc = heads;
#pragma unroll
    for (uint32_t o = 1; o < 32u; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31u) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < blockDim.x / 32u ? wsum[lane] : 0u;
#pragma unroll
        for (uint32_t o = 1; o < 32u; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += v;
        }
        wsum[lane] = s;                               /* inclusive warp prefix */
    }
    __syncthreads();
    uint32_t pos = inc - heads + (w ? wsum[w - 1] : 0u);
    if (threadIdx.x == 0) {
        hdr[0] = wsum[blockDim.x / 32u - 1u];
        hdr[1] = tail[1];
        hdr[2] = *tail;
        hdr[3] = tail[2] | tail[3];
    }
    for (uint32_t p = p0; p < p1; p++) {
        if (p != 0u && hr__same_addr(r[kix[p]], r[kix[p - 1]])) continue;
        if (pos < out_cap) {
            hr_race x = r[kix[p]];
            for (uint32_t q = p + 1; q < n && hr__same_addr(r[kix[q]], x); q++) {
                const hr_race &y = r[kix[q]];
                if (y.scope > x.scope) {
                    const uint8_t sc = y.scope;
                    if (x.first_kind == 0xff) x = y;
                    x.scope = sc;
                }
            }
            out[pos] = x;
        }
        pos++;
    }
}

static hr_status report_async(hr_ctx *c, cudaStream_t s, hr_race *out, uint32_t out_cap, uint32_t *hdr);

extern "C" hr_status hr_report_async(hr_ctx *c, void *stream)
{
    if (!c) return HR_E_ARG;
    CU(cudaSetDevice(c->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
    if (!c->arep_host) {
        const size_t bytes = (size_t)c->cfg.ring_capacity * sizeof(hr_race);
        if (cudaHostAlloc((void **)&c->arep_host, bytes, cudaHostAllocMapped) != cudaSuccess)
            return fail(c, HR_E_NOMEM, "pinned mapped report buffer of %zu bytes failed", bytes);
        CU(cudaHostGetDevicePointer((void **)&c->arep_dev, c->arep_host, 0));
        if (cudaHostAlloc((void **)&c->arep_hdr_host, 16, cudaHostAllocMapped) != cudaSuccess)
            return fail(c, HR_E_NOMEM, "pinned report header failed");
        CU(cudaHostGetDevicePointer((void **)&c->arep_hdr_dev, c->arep_hdr_host, 0));
        CU(cudaEventCreateWithFlags(&c->arep_ev, cudaEventDisableTiming));
    }
    if (hr_status st = report_async(c, s, c->arep_dev, c->cfg.ring_capacity, c->arep_hdr_dev)) return st;
    CU(cudaEventRecord(c->arep_ev, s));
    c->arep_pending = true;
    return HR_OK;
}

extern "C" hr_status hr_report_async_to(hr_ctx *c, void *stream, hr_race *out, uint32_t out_cap, uint32_t *hdr)
{
    if (!c || !hdr || (out_cap && !out)) return fail(c, HR_E_ARG, "hr_report_async_to: bad arguments");
    CU(cudaSetDevice(c->device));
    return report_async(c, stream ? (cudaStream_t)stream : c->stream, out, out_cap, hdr);
}

/* arguments of the full-capacity report path (scratch carved by report_async) */
struct arep_args {
    uint64_t *lo0, *lo1, *hi0, *hi1;
    uint32_t *ix0, *ix1, *head, *pos;
    void *tmp;
    hr_race *out;
    uint32_t out_cap;
    uint32_t *hdr;
    int lo_bits, hi_bits;
};

static uint32_t arep_body_launches(const arep_args &a)
{
    /* keys, sort (onesweep: histogram + scan + one pass per 8 bits), hi keys, sort,
     * heads, scan (2), emit */
    return 1u + (2u + (a.lo_bits + 7) / 8) + 1u + (2u + (a.hi_bits + 7) / 8) + 1u + 2u + 1u;
}

/* The full-capacity path: sort the whole ring (entries past the tail as the
 * largest keys), flag and scan the run heads, emit. */
static hr_status arep_enqueue_sort(hr_ctx *c, cudaStream_t s, const arep_args &a)
{
    const uint32_t cap = c->cfg.ring_capacity;
    const unsigned g = (cap + 255) / 256;
    size_t tb = c->arep_tmp_bytes;
    hr_arep_keys_kernel<<<g, 256, 0, s>>>(c->ring, c->tail, cap, a.lo0, a.ix0);
    CU(cudaGetLastError());
    CU(cub::DeviceRadixSort::SortPairs(a.tmp, tb, a.lo0, a.lo1, a.ix0, a.ix1, (int)cap, 0, a.lo_bits, s));
    hr_arep_hikeys_kernel<<<g, 256, 0, s>>>(c->ring, c->tail, a.ix1, cap, a.hi0);
    CU(cudaGetLastError());
    tb = c->arep_tmp_bytes;
    CU(cub::DeviceRadixSort::SortPairs(a.tmp, tb, a.hi0, a.hi1, a.ix1, a.ix0, (int)cap, 0, a.hi_bits, s));
    hr_arep_heads_kernel<<<g, 256, 0, s>>>(c->ring, c->tail, a.ix0, cap, a.head);
    CU(cudaGetLastError());
    tb = c->arep_tmp_bytes;
    CU(cub::DeviceScan::ExclusiveSum(a.tmp, tb, a.head, a.pos, (int)cap, s));
    hr_arep_emit_kernel<<<g, 256, 0, s>>>(c->ring, c->tail, a.ix0, a.head, a.pos, cap, a.out, a.out_cap, a.hdr);
    CU(cudaGetLastError());
    return HR_OK;
}

/* (Re)build the report graph for these arguments: a kernel node (the small-set
 * kernel, which sets the IF condition when the ring holds more than
 * HR_AREP_SMALL records) followed by a conditional IF node whose body is the
 * full-capacity path, captured from arep_enqueue_sort. */
static hr_status arep_graph_build(hr_ctx *c, const arep_args &a)
{
    const uint32_t cap = c->cfg.ring_capacity;
    const hr_ctx::arep_key_t key = {a.out, a.hdr, c->arep_scratch, c->ring, a.out_cap, cap, a.lo_bits, a.hi_bits};
    for (int i = 0; i < 2; i++) {
        const hr_ctx::arep_key_t &k = c->arep_g[i].key;
        if (c->arep_g[i].exec && k.out == key.out && k.hdr == key.hdr && k.scratch == key.scratch &&
            k.ring == key.ring && k.out_cap == key.out_cap && k.cap == key.cap && k.lo_bits == key.lo_bits &&
            k.hi_bits == key.hi_bits) {
            c->arep_exec = c->arep_g[i].exec;
            c->arep_lru = 1 - i;
            return HR_OK;
        }
    }
    const int slot = c->arep_lru;
    c->arep_exec = nullptr;
    if (c->arep_g[slot].exec) { cudaGraphExecDestroy(c->arep_g[slot].exec); c->arep_g[slot].exec = nullptr; }
    if (c->arep_g[slot].graph) { cudaGraphDestroy(c->arep_g[slot].graph); c->arep_g[slot].graph = nullptr; }
    if (!c->arep_cap) CU(cudaStreamCreateWithFlags(&c->arep_cap, cudaStreamNonBlocking));
    if (!c->arep_big) {
        CU(cudaMalloc(&c->arep_big, sizeof(unsigned long long)));
        CU(cudaMemset(c->arep_big, 0, sizeof(unsigned long long)));
    }
    CU(cudaFuncSetAttribute(hr_arep_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)HR_AREP_SMALL_SMEM));
    cudaGraph_t g = nullptr;
    CU(cudaGraphCreate(&g, 0));
    c->arep_g[slot].graph = g;
    cudaGraphConditionalHandle big;
    CU(cudaGraphConditionalHandleCreate(&big, g, 0u, cudaGraphCondAssignDefault));
    const hr_race *ring = c->ring;
    const unsigned int *tail = c->tail;
    hr_race *out = a.out;
    uint32_t out_cap = a.out_cap, capv = cap, body = arep_body_launches(a);
    uint32_t *hdr = a.hdr;
    unsigned long long *bigc = c->arep_big;
    void *kargs[] = {(void *)&ring, (void *)&tail, (void *)&capv, (void *)&out, (void *)&out_cap,
                     (void *)&hdr, (void *)&big, (void *)&bigc, (void *)&body};
    cudaKernelNodeParams kp = {};
    kp.func = (void *)hr_arep_small_kernel;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(HR_AREP_SMALL_THREADS);
    kp.sharedMemBytes = (unsigned)HR_AREP_SMALL_SMEM;
    kp.kernelParams = kargs;
    cudaGraphNode_t kn = nullptr, cn = nullptr;
    CU(cudaGraphAddKernelNode(&kn, g, nullptr, 0, &kp));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = big;
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    CU(cudaGraphAddNode(&cn, g, &kn, 1, &np));
    cudaGraph_t bodyg = np.conditional.phGraph_out[0];
    CU(cudaStreamBeginCaptureToGraph(c->arep_cap, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    const hr_status st = arep_enqueue_sort(c, c->arep_cap, a);
    cudaGraph_t captured = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->arep_cap, &captured);
    if (st) return st;
    CU(ec);
    CU(cudaGraphInstantiate(&c->arep_g[slot].exec, g, 0));
    c->arep_g[slot].key = key;
    c->arep_exec = c->arep_g[slot].exec;
    c->arep_lru = 1 - slot;
    return HR_OK;
}

/* a13 on the device (hr_report_async / hr_report_async_to): enqueue on `s` the
 * end-of-kernel spill scan, the sorts, the run-head merge and the emit into
 * out[0, out_cap) + hdr[4]. */
static hr_status report_async(hr_ctx *c, cudaStream_t s, hr_race *out, uint32_t out_cap, uint32_t *hdr)
{
    const uint32_t cap = c->cfg.ring_capacity;
    if (hr_status st = enqueue_spill_scan(c, s)) return st;
    /* scratch: lo keys x2, hi keys x2, idx x2, head flags, positions, CUB temp */
    const size_t nb = cap;
    size_t off[9], tot = 0;
    const size_t sz[8] = {nb * 8, nb * 8, nb * 8, nb * 8, nb * 4, nb * 4, nb * 4, nb * 4};
    for (int i = 0; i < 8; i++) { off[i] = tot; tot += (sz[i] + 255) & ~(size_t)255; }
    if (!c->arep_tmp_bytes) {
        size_t t1 = 0, t2 = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint64_t *)nullptr, (uint64_t *)nullptr, (uint32_t *)nullptr,
                                           (uint32_t *)nullptr, (int)cap, 0, 64, s));
        CU(cub::DeviceScan::ExclusiveSum(nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr, (int)cap, s));
        c->arep_tmp_bytes = std::max(t1, t2);
    }
    off[8] = tot;
    tot += c->arep_tmp_bytes;
    if (tot > c->arep_scratch_bytes) {
        if (c->arep_scratch) cudaFree(c->arep_scratch);
        c->arep_scratch = nullptr;
        c->arep_scratch_bytes = 0;
        if (cudaMalloc(&c->arep_scratch, tot) != cudaSuccess) return fail(c, HR_E_NOMEM, "report scratch failed");
        c->arep_scratch_bytes = tot;
    }
    char *b = (char *)c->arep_scratch;
    uint64_t *lo0 = (uint64_t *)(b + off[0]), *lo1 = (uint64_t *)(b + off[1]);
    uint64_t *hi0 = (uint64_t *)(b + off[2]), *hi1 = (uint64_t *)(b + off[3]);
    uint32_t *ix0 = (uint32_t *)(b + off[4]), *ix1 = (uint32_t *)(b + off[5]);
    uint32_t *head = (uint32_t *)(b + off[6]), *pos = (uint32_t *)(b + off[7]);
    void *tmp = b + off[8];
    /* only the key bits that can be set: words < max(global end, shared words),
     * hi = kernel << 33 | space << 32 | block with kernel <= last_kernel; the
     * padding keys (~0) stay the largest within the range, and the sorts are
     * stable, so real records still precede them (fewer radix passes) */
    auto bits_of = [](uint64_t v) { int b = 0; while (b < 64 && (v >> b)) b++; return b; };
    int lo_bits = std::max(1, std::min(64, bits_of(std::max<uint64_t>(c->gbase + c->gwords, c->smem_words_max))));
    int hi_bits = std::min(64, 33 + bits_of((uint64_t)std::max(c->max_kernel, c->last_kernel) + 1));
    if (c->online_used) lo_bits = hi_bits = 64;  /* online kernels: caller-chosen ids and instance sizes */
    const arep_args a = {lo0, lo1, hi0, hi1, ix0, ix1, head, pos, tmp, out, out_cap, hdr, lo_bits, hi_bits};
    if (!c->arep_no_graph) {
        const hr_status st = arep_graph_build(c, a);
        if (st == HR_OK) {
            c->launches++;                             /* the small-set kernel; the IF body counts itself */
            CU(cudaGraphLaunch(c->arep_exec, s));
            return HR_OK;
        }
        if (st != HR_E_CUDA) return st;
        cudaGetLastError();
        c->arep_no_graph = true;                   /* e.g. a driver without conditional nodes */
    }
    c->launches += arep_body_launches(a);
    return arep_enqueue_sort(c, s, a);
}

extern "C" hr_status hr_report_collect(hr_ctx *c, hr_race *out, size_t cap, size_t *n_out, uint32_t *flags_out)
{
    if (!c || !n_out || (cap && !out)) return fail(c, HR_E_ARG, "hr_report_collect: bad arguments");
    if (!c->arep_pending) return fail(c, HR_E_STATE, "hr_report_collect without hr_report_async");
    CU(cudaSetDevice(c->device));
    CU(cudaEventSynchronize(c->arep_ev));
    c->arep_pending = false;
    const uint32_t m = c->arep_hdr_host[0], flags = c->arep_hdr_host[1];
    if (c->arep_hdr_host[3])                             /* ring overflow: the spill needs the full path */
        return hr_report(c, out, cap, n_out, flags_out);
    *n_out = m;
    if (flags_out) *flags_out = flags;
    const size_t w = std::min<size_t>(m, cap);
    if (w) memcpy(out, c->arep_host, w * sizeof(hr_race));
    return m > cap ? fail(c, HR_E_ARG, "hr_report_collect: %u races, capacity %zu", m, cap) : HR_OK;
}

extern "C" hr_status hr_report(hr_ctx *c, hr_race *out, size_t cap, size_t *n_out, uint32_t *flags_out)
{
    if (!c || !n_out || (cap && !out)) return fail(c, HR_E_ARG, "hr_report: bad arguments");
    static const bool prof = getenv("HR_REPORT_PROFILE") != nullptr;
    hr__prof_on = prof;
    hr__prof_n = 0;
    HR_PROF_MARK();
    CU(cudaSetDevice(c->device));
    if (hr_status st = enqueue_spill_scan(c, c->stream)) return st;
    CU(cudaStreamSynchronize(c->stream));
    HR_PROF_MARK();
    unsigned int hdr[HR_TAIL_WORDS];
    CU(cudaMemcpy(hdr, c->tail, sizeof hdr, cudaMemcpyDeviceToHost));
    HR_PROF_MARK();
    /* ring [0, n_ring) then spill [ring_capacity, ring_capacity + n_spill): the spill is
     * only written after a drop, i.e. with a full ring, so the two are contiguous */
    const uint32_t n_ring = std::min<uint32_t>(hdr[0], c->cfg.ring_capacity);
    const uint32_t n_spill = std::min<uint32_t>(hdr[2], c->spill_cap);
    if (n_spill && n_ring != c->cfg.ring_capacity)
        return fail(c, HR_E_STATE, "hr_report: spill records with a ring that is not full (%u of %u)", n_ring,
                    c->cfg.ring_capacity);
    const uint32_t n = n_ring + n_spill;
    uint32_t flags = hdr[1];
    const bool incomplete = (flags & HR_F_INCOMPLETE) || hdr[3] != 0u;
    if (hdr[3] != 0u) flags |= HR_F_INCOMPLETE;
    std::vector<hr_race> &v = c->rep;
    v.clear();
    bool sorted = false;
    if (n >= 4096) {                            /* large report: sort on the device */
        hr_status st = sort_races_device(c, n, v);
        if (st) return st;
        sorted = true;
    } else {
        v.resize(n);
        if (n) CU(cudaMemcpy(v.data(), c->ring, n * sizeof(hr_race), cudaMemcpyDeviceToHost));
    }
    HR_PROF_MARK();
    if (!sorted) sort_races(v);
    const size_t m = unique_races(v);
    HR_PROF_MARK();
    *n_out = m;
    if (flags_out) *flags_out = flags;
    size_t w = std::min(m, cap);
    if (w) memcpy(out, v.data(), w * sizeof(hr_race));
    HR_PROF_MARK();
    if (prof && hr__prof_n > 1 && hr__prof[hr__prof_n - 1] - hr__prof[0] > 5.0) {
        fprintf(stderr, "hr_report slow:");
        for (int i = 1; i < hr__prof_n; i++) fprintf(stderr, " %.2f", hr__prof[i] - hr__prof[i - 1]);
        fprintf(stderr, " ms (sync, hdr, reserve, keys, sort1, hikeys, sort2, gather, d2h-enq, d2h-sync, unique, copy-out)\n");
    }
    if (m > cap) return fail(c, HR_E_ARG, "hr_report: %zu races, capacity %zu", m, cap);
    if (incomplete)
        return fail(c, HR_E_INCOMPLETE, "hr_report: racy set incomplete (%s)",
                    hdr[3] ? "a block's dropped shared race records were never spilled (hr_thread_end missing)"
                           : "spill store full: raise hr_config.spill_capacity");
    return HR_OK;
}

/* Merge of per-shard race sets (include/hr.h): host only, no CUDA call. */
extern "C" hr_status hr_merge_races(const hr_race *in, size_t n, hr_race *out, size_t cap, size_t *n_out)
{
    if (!n_out || (n && !in) || (cap && !out)) return HR_E_ARG;
    /* scratch kept across calls: fresh multi-MB vectors cost a page fault per 4 KiB */
    static thread_local std::vector<hr_race> v, tmp;
    v.assign(in, in + n);
    /* the input is usually a concatenation of sorted shard reports: merge its
     * natural runs pairwise (log2(runs) sequential passes); radix-sort otherwise */
    std::vector<size_t> run{0};
    for (size_t i = 1; i < n; i++)
        if (race_less(v[i], v[i - 1])) run.push_back(i);
    run.push_back(n);
    if (run.size() - 1 > 64) {
        sort_races(v);
    } else if (run.size() > 2) {
        tmp.resize(n);
        while (run.size() > 2) {
            std::vector<size_t> nr{0};
            for (size_t r = 0; r + 1 < run.size(); r += 2) {
                const size_t a = run[r], b = run[r + 1], e = r + 2 < run.size() ? run[r + 2] : b;
                std::merge(v.begin() + a, v.begin() + b, v.begin() + b, v.begin() + e, tmp.begin() + a, race_less);
                nr.push_back(e);
            }
            v.swap(tmp);
            run.swap(nr);
        }
    }
    const size_t m = unique_races(v);
    *n_out = m;
    const size_t w = std::min(m, cap);
    if (w) memcpy(out, v.data(), w * sizeof(hr_race));
    return m > cap ? HR_E_ARG : HR_OK;
}

/* Per-pair race classes post-pass (include/hr.h). */
template <typename SRC>
static hr_status classes_launch(hr_ctx *c, const hr_trace *t, SRC src, const unsigned char *ctab,
                                const hr_class_entry *tab, uint64_t mask, unsigned long long *sh, unsigned int *cls,
                                uint32_t kinds, cudaStream_t s)
{
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        hr_status st = check_kernel(c, t, k);
        if (st) return st;
        const uint64_t *kd = t->kdesc + 8ull * k;
        if (!kd[0]) continue;
        hr_dev d = make_kdev(c, t, k);
        size_t smem = HR_FSM_SMEM_BYTES + HR_CLASS_TABLES_BYTES;
        c->launches++;
        hr_classes_kernel<SRC><<<(unsigned)kd[0], (unsigned)(kd[1] * 32), smem, s>>>(
            d, src, t->warp_off + kd[4], (uint32_t)kd[1], (uint32_t)kd[2], ctab, tab, mask, sh, cls, kinds);
        CU(cudaGetLastError());
    }
    return HR_OK;
}

extern "C" hr_status hr_race_classes(hr_ctx *c, const hr_trace *t, const hr_race *races, size_t n,
                                     uint8_t *classes_out, void *stream)
{
    if (!c || !trace_ok(t) || (n && (!races || !classes_out))) return fail(c, HR_E_ARG, "hr_race_classes: bad arguments");
    if (t->format == HR_TRACE_PACKED || t->format == HR_TRACE_POOLED)
        return fail(c, HR_E_ARG, "hr_race_classes: U64 or C32 traces only");
    CU(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) return HR_OK;
    uint64_t cap = 64;
    while (cap < 2 * n) cap <<= 1;
    std::vector<hr_class_entry> tab(cap);
    for (auto &e : tab) { e.word = 0; e.key = ~0ull; e.slot = 0; e.pad = 0; }
    for (size_t i = 0; i < n; i++) {
        const uint64_t key = ((uint64_t)races[i].kernel << 33) | ((uint64_t)races[i].space << 32) | races[i].block;
        uint64_t h = hr__class_hash(races[i].word, key) & (cap - 1);
        while (tab[h].key != ~0ull) h = (h + 1) & (cap - 1);
        tab[h].word = races[i].word;
        tab[h].key = key;
        tab[h].slot = (uint32_t)i;
    }
    unsigned char *ctab = nullptr;
    hr_class_entry *dtab = nullptr;
    unsigned long long *sh = nullptr;
    unsigned int *cls = nullptr;
    hr_status st = HR_OK;
    if (cudaMalloc(&ctab, HR_CLASS_TABLES_BYTES) != cudaSuccess || cudaMalloc(&dtab, cap * sizeof(hr_class_entry)) != cudaSuccess ||
        cudaMalloc(&sh, n * 4 * sizeof(unsigned long long)) != cudaSuccess || cudaMalloc(&cls, n * sizeof(unsigned int)) != cudaSuccess) {
        st = fail(c, HR_E_NOMEM, "hr_race_classes: device allocation failed");
    } else {
        uint32_t kinds = 0;
        for (int i = 0; i < 4; i++) kinds |= (uint32_t)hr_class_kinds_init[i] << (8 * i);
        cudaMemcpyAsync(ctab, hr_class_tables_init, HR_CLASS_TABLES_BYTES, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dtab, tab.data(), cap * sizeof(hr_class_entry), cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(sh, 0, n * 4 * sizeof(unsigned long long), s);
        cudaMemsetAsync(cls, 0, n * sizeof(unsigned int), s);
        if (t->format == HR_TRACE_C32)
            st = classes_launch(c, t, hr_src_c32{t->rec32, t->recop}, ctab, dtab, cap - 1, sh, cls, kinds, s);
        else
            st = classes_launch(c, t, hr_src_u64{t->rec}, ctab, dtab, cap - 1, sh, cls, kinds, s);
        if (!st) {
            std::vector<unsigned int> h(n);
            if (cudaMemcpyAsync(h.data(), cls, n * sizeof(unsigned int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess)
                st = fail(c, HR_E_CUDA, "hr_race_classes: %s", cudaGetErrorString(cudaGetLastError()));
            else
                for (size_t i = 0; i < n; i++) classes_out[i] = (uint8_t)h[i];
        }
    }
    cudaFree(ctab); cudaFree(dtab); cudaFree(sh); cudaFree(cls);
    return st;
}

extern "C" hr_status hr_reset_report(hr_ctx *c)
{
    if (!c) return HR_E_ARG;
    CU(cudaSetDevice(c->device));
    CU(cudaMemsetAsync(c->tail, 0, HR_TAIL_WORDS * sizeof(unsigned int), c->stream));
    CU(cudaMemsetAsync(c->counters, 0, 4 * sizeof(unsigned long long), c->stream));
    CU(cudaMemsetAsync(c->counters + HR_CNT_BASE, 0, 4 * HR_CNT_SLICES * sizeof(unsigned long long), c->stream));
    c->have_kernel = false;
    c->online_used = false;
    return HR_OK;
}

extern "C" hr_status hr_counters(hr_ctx *c, uint64_t out[4])
{
    if (!c || !out) return HR_E_ARG;
    CU(cudaSetDevice(c->device));
    CU(cudaStreamSynchronize(c->stream));
    uint64_t sl[4 * HR_CNT_SLICES];
    CU(cudaMemcpy(sl, c->counters + HR_CNT_BASE, sizeof sl, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4; i++) {
        out[i] = 0;
        for (uint32_t k = 0; k < HR_CNT_SLICES; k++) out[i] += sl[4 * k + i];
    }
    return HR_OK;
}

extern "C" hr_status hr_replay_timing(hr_ctx *c, double *reset_ms, uint64_t *n_resets, double *kernel_ms,
                                      uint64_t *n_kernels)
{
    if (!c) return HR_E_ARG;
    CU(cudaSetDevice(c->device));
    double acc[2] = {0, 0};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *lists[2] = {&c->ev_reset, &c->ev_kernel};
    for (int i = 0; i < 2; i++) {
        for (auto &pr : *lists[i]) {
            CU(cudaEventSynchronize(pr.second));
            float ms = 0;
            CU(cudaEventElapsedTime(&ms, pr.first, pr.second));
            acc[i] += ms;
            c->ev_pool.push_back(pr.first);
            c->ev_pool.push_back(pr.second);
        }
    }
    if (reset_ms) *reset_ms = acc[0];
    if (n_resets) *n_resets = c->ev_reset.size();
    if (kernel_ms) *kernel_ms = acc[1];
    if (n_kernels) *n_kernels = c->ev_kernel.size();
    c->ev_reset.clear();
    c->ev_kernel.clear();
    return HR_OK;
}

extern "C" hr_status hr_launch_count(hr_ctx *c, uint64_t *n)
{
    if (!c || !n) return HR_E_ARG;
    uint64_t big = 0;
    if (c->arep_big) {                          /* kernels the report graph's IF body ran */
        CU(cudaSetDevice(c->device));
        CU(cudaDeviceSynchronize());
        CU(cudaMemcpy(&big, c->arep_big, sizeof big, cudaMemcpyDeviceToHost));
        CU(cudaMemset(c->arep_big, 0, sizeof big));
    }
    *n = c->launches + big;
    c->launches = 0;
    return HR_OK;
}

extern "C" hr_status hr_fsm_table(uint8_t *table2048, uint8_t *flags32)
{
    if (table2048) memcpy(table2048, hr_fsm_table_init, HR_FSM_BYTES);
    if (flags32) memcpy(flags32, hr_fsm_flags_init, 32);
    return HR_OK;
}

extern "C" hr_status hr_device_view(hr_ctx *c, void *out, size_t size)
{
    if (!c || !out || size < sizeof(hr_dev)) return fail(c, HR_E_ARG, "hr_device_view: need %zu bytes", sizeof(hr_dev));
    hr_dev d = make_dev(c, c->last_kernel);
    memcpy(out, &d, sizeof d);
    c->online_used = true;                      /* a user kernel will run on this view */
    c->scan_pending = true;
    c->have_kernel = true;
    return HR_OK;
}

extern "C" const char *hr_last_error(hr_ctx *c) { return c ? c->err : "null context"; }

extern "C" void hr_destroy(hr_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->side) cudaStreamSynchronize(c->side);
    for (int b = 0; b < 2; b++) {
        if (c->gbuf[b]) cudaFree(c->gbuf[b]);
        if (c->used_done[b]) cudaEventDestroy(c->used_done[b]);
        if (c->reset_done[b]) cudaEventDestroy(c->reset_done[b]);
    }
    if (c->side) cudaStreamDestroy(c->side);
    if (c->copy) { cudaStreamSynchronize(c->copy); cudaStreamDestroy(c->copy); }
    if (c->ring) cudaFree(c->ring);
    if (c->tail) cudaFree(c->tail);
    if (c->counters) cudaFree(c->counters);
    if (c->fsm) cudaFree(c->fsm);
    for (int i = 0; i < 24; i++)
        if (c->stage[i]) cudaFree(c->stage[i]);
    if (c->rep_host) cudaFreeHost(c->rep_host);
    if (c->arep_host) cudaFreeHost(c->arep_host);
    if (c->arep_hdr_host) cudaFreeHost(c->arep_hdr_host);
    if (c->arep_scratch) cudaFree(c->arep_scratch);
    if (c->arep_ev) cudaEventDestroy(c->arep_ev);
    for (auto &ag : c->arep_g) {
        if (ag.exec) cudaGraphExecDestroy(ag.exec);
        if (ag.graph) cudaGraphDestroy(ag.graph);
    }
    if (c->arep_cap) cudaStreamDestroy(c->arep_cap);
    if (c->arep_big) cudaFree(c->arep_big);
    for (auto &pr : c->ev_reset) { c->ev_pool.push_back(pr.first); c->ev_pool.push_back(pr.second); }
    for (auto &pr : c->ev_kernel) { c->ev_pool.push_back(pr.first); c->ev_pool.push_back(pr.second); }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    delete c;
}
