/*
 * hr.h — C ABI of the B200-native HiRace per-access race check
 * (arXiv 2401.04701, "HiRace: Accurate and Fast Source-Level Race Checking
 * of GPU Programs").  Citations: PAPER.md:n = /root/reference/PAPER.md line n
 * (section given alongside).
 *
 * The method: every monitored word data[k] has a shadow word shadow[k]
 * holding <State, TID, BC, WC> (Fig. ssm_shadow); every
 * read / write / atomic runs Algorithm 1 "UpdateShadow":
 * atomic read, label = (access, checkSync, compareTids), flat-array FSM
 * lookup, pack, atomicCAS until it succeeds.  A word
 * whose FSM enters RACE is reported once per unique address.
 *
 * This header is the host side.  The device side (hr_check_read/_write/
 * _atomic, hr_syncthreads/_syncwarp) is the header-only hr_device.cuh.
 *
 * Conventions (all entry points):
 *   - extern "C", C99 types only; no exceptions or aborts cross the ABI.
 *   - every host call returns hr_status (0 = HR_OK, < 0 = error); CUDA
 *     errors map to HR_E_CUDA with the text in hr_last_error(ctx).
 *   - "device" pointers are CUDA device pointers of ctx->device; "host"
 *     pointers are ordinary (ideally pinned) host memory.
 *   - stream arguments are cudaStream_t passed as void* (NULL = legacy stream).
 *   - one ctx per (device, stream); host calls on one ctx are not re-entrant.
 *   - nothing is allocated on the check path: all device memory is owned by
 *     the ctx and allocated in hr_init / hr_shadow_alloc.
 */
#ifndef HR_H_
#define HR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HR_OK = 0,
    HR_E_ARG = -1,     /* invalid argument (NULL, widths, sizes, grid too large) */
    HR_E_NOMEM = -2,   /* device or host allocation failed */
    HR_E_CUDA = -3,    /* CUDA runtime error; see hr_last_error */
    HR_E_STATE = -4,   /* call out of order (e.g. replay before hr_shadow_alloc) */
    HR_E_INCOMPLETE = -5 /* hr_report / hr_report_collect: the racy set written is NOT complete —
                            the spill store (hr_config.spill_capacity) overflowed, or a block whose
                            shared race records the full ring dropped never called hr_thread_end
                            (flags carry HR_F_INCOMPLETE; n_out counts what was recovered) */
} hr_status;

typedef enum { HR_GLOBAL = 0, HR_SHARED = 1 } hr_space;          /* PAPER.md:257 memory spaces */
typedef enum { HR_READ = 0, HR_WRITE = 1, HR_ATOMIC = 2 } hr_kind; /* PAPER.md:565 "third class" */
typedef enum { HR_SCOPE_BLOCK = 1, HR_SCOPE_GRID = 2 } hr_scope;  /* DESIGN.md reading R4 */

/* Sticky device-side conditions, surfaced by hr_report (never fatal). */
enum {
    HR_F_CLOCK_OVERFLOW = 1u,      /* a BC/WC clock overflowed: later checks of that thread
                                      skipped, earlier races kept (PAPER.md:540 footnote) */
    HR_F_RING_OVERFLOW = 2u,       /* report ring full (a warning): the dropped records were recovered
                                      into the spill store (end-of-kernel global shadow scan, end-of-block
                                      shared instance scan), so the set is still exact unless
                                      HR_F_INCOMPLETE is also set */
    HR_F_MODEL_VIOLATION = 4u,     /* unknown control record / sub-warp sync */
    HR_F_BARRIER_DIVERGENCE = 8u,  /* barrier record not uniform across a warp's lanes */
    HR_F_UNMONITORED = 16u,        /* global access outside the registered shadow region */
    HR_F_INCOMPLETE = 32u          /* overflow recovery failed: the spill store was full, or (as
                                      HR_E_INCOMPLETE) a dropped shared record was never spilled;
                                      or (HR_OPT_HYBRID) a run's appends disagreed with its count */
};

/* Shadow word layout ("5 bits ... 8 bytes of memory per address"):
 *   [63:59] state  [58:32] tid = block:17 | warp:5 | lane:5  [31:wc_bits] bc  [wc_bits-1:0] wc
 * state_bits must be 5 and tid_bits 27; bc_bits + wc_bits must be 32.
 * Defaults (hr_init with cfg == NULL): 5/27/16/16, ring 1<<20 records, device 0,
 * spill capacity automatic.
 *
 * Report storage (a9, "report races on unique memory addresses"):
 * racy words are appended to the ring as they are found.  When the ring is
 * full, dropped records are recovered into the spill store: after each kernel
 * (before its global shadow is reset) a device-side scan copies every RACE word
 * of that kernel's global shadow there if the kernel dropped a global record,
 * and each block that dropped a shared record copies its instance's RACE words
 * there at block end.  The report is the sorted union of ring and spill, so it
 * stays exact until the spill itself is full (HR_F_INCOMPLETE, HR_E_INCOMPLETE).
 * spill_capacity 0 = automatic: max(2^16, min(2^24, local global shadow words)),
 * fixed when hr_shadow_alloc registers the global region (24 B per record). */
typedef struct {
    uint8_t state_bits, tid_bits, bc_bits, wc_bits;
    uint32_t ring_capacity;   /* race records the device ring holds (>= 1) */
    int device;               /* CUDA device ordinal */
    uint32_t options;         /* HR_OPT_* bits */
    uint32_t spill_capacity;  /* records of the overflow spill store; 0 = automatic (above) */
} hr_config;

enum {
    HR_OPT_NO_COALESCE = 1u,   /* disable same-address lane coalescing (a3), for ablations */
    HR_OPT_NO_FASTEXIT = 2u,   /* disable label-insensitive fast exits (a7), for ablations */
    HR_OPT_TIMING = 4u,        /* record CUDA events around every shadow reset and replay launch */
    HR_OPT_NO_SPECULATE = 8u,  /* accepted, no effect: loading the shadow word first is the default
                                  (HR_OPT_SPECULATE below is the ablation) */
    HR_OPT_NO_POOL = 16u,      /* replay row by row (default: chosen from sampled record density,
                                  shared share and warp-length tail, see hr_host.cu kernel_choice) */
    HR_OPT_POOL = 32u,         /* replay with warp pools of valid accesses (sparse traces) */
    HR_OPT_DOUBLE_SHADOW = 64u, /* two global shadows: the kernel-boundary reset (a11) of one runs on a
                                   side stream while the next kernel uses the other (2x shadow memory) */
    HR_OPT_FINITE_HISTORY = 128u, /* BASELINE, not HiRace: iGUARD-style 16-byte records (one reader, one
                                   writer) checked with the same replay, for the
                                   paper's comparisons (Listing 4 eviction, memory); shadow scan off */
    HR_OPT_POOL_WIDE = 256u,     /* force the 64-register pooled kernel (few very long warps) */
    HR_OPT_ROW_WIDE = 512u,      /* force the 64-register row kernel (chosen by default for
                                    shared-shadow heavy traces and small grids) */
    HR_OPT_NO_COMPACT = 1024u,   /* long-tailed grids: replay the rows as they are instead of
                                    packing each long warp's accesses first (hr_compact.cuh) */
    HR_OPT_SMEM32 = 4096u,       /* 32-bit shared-shadow words with the block implicit (SURVEY
                                    §8(f)-4, "configurable and can be reduced"): state 5 |
                                    warp 5 | lane 5 | bc 9 | wc 8.  Halves the SMEM shadow; caps
                                    the block / warp clocks at 511 / 255 (past them a thread stops
                                    checking and HR_F_CLOCK_OVERFLOW is latched).  Not with
                                    HR_OPT_FINITE_HISTORY. */
    HR_OPT_LAZY_RESET = 8192u,   /* a11 without the per-kernel shadow memset: each
                                    kernel writes a 4-bit epoch tag (1..15) into bits [31:28] of the
                                    clock word, a global word with another tag reads as INIT, and
                                    hr_kernel_begin zeroes the shadow only before a tag is reused
                                    (every 15 kernels).  Caps the block clock at 2^(28 - wc_bits) - 1
                                    (4095 at the default 16/16).  Not with FINITE_HISTORY or
                                    DOUBLE_SHADOW; wc_bits <= 24. */
    HR_OPT_BSERIAL = 16384u,     /* sparse U64 traces (pooled replay): one CUDA warp replays a whole
                                    simulated block epoch by epoch (hr_bserial.cuh) */
    HR_OPT_ROW_NARROW = 65536u,  /* force the 48-register row kernel (the default for dense global traces) */
    HR_OPT_BINNED = 262144u,     /* address-binned replay (hr_binned.cuh) for kernels without shared
                                    shadow: accesses regrouped per (shadow bucket of 64 MB, block) in
                                    happens-before order and checked bucket by bucket so the random
                                    shadow RMWs hit L2.  Opt-in: exact, but measured slower than the
                                    row replay on C5 (161 vs 90 ms, DESIGN.md §5 item 17) */
    HR_OPT_NO_BINNED = 524288u,  /* never use the binned replay (the default) */
    HR_OPT_HYBRID = 1048576u,    /* hybrid binned replay (csrc/hr_hybrid.cuh) for row-replayed kernels
                                    without warp tiles: shadow buckets of 32 MB whose accesses arrive
                                    mostly scattered are binned — the row replay appends their accesses
                                    to (bucket, block) runs in happens-before order and a bucket-major
                                    pass checks them with the bucket's shadow in L2 — the rest is
                                    checked by the row replay as usual */
    HR_OPT_BIN_ALL = 2097152u,   /* with HR_OPT_HYBRID: bin every touched bucket (tests) */
    HR_OPT_NO_STREAMS = 131072u, /* long-tailed barrier-free kernels without shared shadow: use the
                                    per-block compacted replay instead of the stream-scheduled one
                                    (hr_streams.cuh: hub warps fanned out over helper streams that
                                    any CUDA warp of any CTA replays, longest first) */
    HR_OPT_SPECULATE = 2048u     /* ablation: global reads/writes skip Algorithm 1's first atomic read
                                    and CAS against INIT (the CAS return is the read when it fails).
                                    Measured slower: a failed CAS costs an L2 atomic round trip that
                                    a load followed by an unchanged-word exit does not */
};

/* One unique racy address.  24 bytes.
 *   word       global: word index; shared: word index inside the block's __shared__ instance
 *   block      shared: simulated block of the instance; global: 0xFFFFFFFF
 *   kernel     kernel index (trace kernel index + hr_trace.kernel_base)
 *   first_tid  packed tid of the access that moved the word into RACE (diagnostic only)
 *   space      hr_space;  scope: hr_scope
 *   first_kind hr_kind of that access; prev_state: FSM state before it (diagnostic only) */
typedef struct {
    uint64_t word;
    uint32_t block;
    uint32_t kernel;
    uint32_t first_tid;
    uint8_t space, scope, first_kind, prev_state;
} hr_race;

/* hr_trace.flags */
enum {
    HR_TRACE_F_SHARD_OWNED = 1u  /* every global access record of the trace targets a word of this ctx's
                                    address shard (the trace was partitioned for this rank, as
                                    tracegen's C5 shard generator and multigpu.shard_trace do): the
                                    replay skips the per-access owner hash.  A record the shard does
                                    not own would then be checked here too; the region check and the
                                    shard-local index are unchanged.  No effect on an unsharded ctx. */
};

/* Record encodings of an hr_trace. */
enum {
    HR_TRACE_U64 = 0,   /* rec: one u64 record per lane and row (any word < 2^61) */
    HR_TRACE_C32 = 1,   /* rec32 + recop: 160 B per row instead of 256 (words < 2^32) */
    HR_TRACE_PACKED = 2, /* packed + pack_off: lossless variable-length rows (below), made by hr_pack_trace */
    HR_TRACE_POOLED = 3  /* rec + recop: pooled rows (below), made by hr_pool_trace */
};

/* HR_TRACE_POOLED: the same access streams re-laid out as warp pools (not in
 * the paper: a replay input layout for sparse traces, e.g. address shards,
 * whose rows carry few accesses).  Row r holds 32 entries: rec[r*32 + i] a
 * U64-layout record and recop[r*32 + i] (u8) the simulated lane it belongs
 * to.  A row is either a barrier row copied verbatim (tags = lanes) or up to
 * 32 accesses of ONE simulated warp inside one epoch, in record order (row-
 * major, lanes ascending), NOP-padded at its end; warp_off gives each warp's
 * rows as for U64.  Lanes of one row are unordered by happens-before (same
 * warp, same epochs) and each thread's accesses keep program order, so a row
 * is checked as one pool (same-word entries folded in order).  Device only
 * (hr_replay_trace); not for hr_replay_trace_host / hr_race_classes. */

/* HR_TRACE_PACKED: a lossless, transfer-oriented encoding of the U64 rows
 * (not in the paper: it shrinks the host->device bytes of hr_replay_trace_host).
 * Segment i (0 <= i < n_warp_off-1) encodes the rows [warp_off[i], warp_off[i+1])
 * (warp_off must be non-decreasing) and occupies bytes [pack_off[i], pack_off[i+1])
 * of `packed`; every pack_off is a multiple of 4.  A segment of n rows is
 *   n header bytes h_j, zero-padded to a multiple of 4, then n row bodies.
 * With k = h & 63, affine = h & 64, uniform = h & 128, a row body is
 *   k == 62 (raw):  the 32 u64 records verbatim (256 B, as lo/hi u32 pairs)
 *   otherwise:      nibbles: uniform ? one u32 whose low 4 bits apply to every lane
 *                                    : four u32, lane l at bits 4*(l%8) of u32 l/8
 *                   if k != 63:  base (u64 as lo, hi u32)
 *                                if !affine && k > 0: k u32 words holding lane l's
 *                                k-bit delta at bits [l*k, l*k+k) (little-endian)
 * A nibble is op | x << 2: for op 0..2 (access) x = space and the word is
 * base + lane (affine), base + delta_l, or base (k == 0); for op 3 (control)
 * x = the control word (0..2) and no word bits are used.  Exception: an affine
 * row with k = 1 or 2 (affine rows carry no deltas) holds every lane as a read
 * or write of space k - 1, and its nibbles are one u32 bit mask instead (bit l
 * set = lane l writes): body = mask, base (12 bytes; 8 with the uniform bit set,
 * which a mask row otherwise never has: a base below 2^32 in one u32); and an
 * affine row with
 * 3 <= k <= 61 is a k-bit delta row whose base fits 32 bits: the base is one
 * u32 (nibbles, base u32, deltas).  k == 63 means the
 * row has no access lanes (no base).  Rows a nibble cannot express (a control
 * record with word > 2 or the space bit set) use the raw form.  The decoder
 * reads up to 8 bytes past a segment's last body; allocate `packed` with 16
 * bytes of slack (hr_pack_trace's size query includes them). */

/* A batch of synthetic access streams (tracegen/format.py documents the layout).
 *   rec       DEVICE, n_rows*32 uint64 records; row r, lane l at rec[r*32+l]:
 *             [63:62] op (0 R, 1 W, 2 A, 3 control) [61] space [60:0] word;
 *             control words: 0 NOP, 1 __syncthreads, 2 __syncwarp
 *   kdesc     HOST, n_kernels x 8 uint64: blocks, warps, lanes(<=32), smem_words,
 *             warp_off_index, tile_log2, 0, 0 — tile_log2 (0..4): 0 = whole-warp
 *             __syncwarp records; 1..4 = the kernel's warp-level barriers are tiles
 *             of 2^tile_log2 lanes (a __syncwarp record held by whole tiles is one
 *             barrier per tile; reading R8 in DESIGN.md).  Tile
 *             kernels are replayed by the row kernel (one clock per lane);
 *             HR_TRACE_POOLED / hr_pool_trace reject them (HR_E_ARG)
 *   warp_off  DEVICE, uint64 absolute row offsets; warp w of kernel k owns rows
 *             [warp_off[woi+w], warp_off[woi+w+1]) with woi = kdesc[k][4]
 *   The ctx never takes ownership.  For hr_replay_trace_host, rec and warp_off are
 *   HOST pointers instead (copied to ctx-owned device staging buffers). */
typedef struct {
    const uint64_t *rec;
    uint64_t n_rows;
    const uint64_t *kdesc;
    uint32_t n_kernels;
    uint32_t kernel_base;
    const uint64_t *warp_off;
    uint64_t n_warp_off;
    /* format HR_TRACE_C32 (rec unused): same rows, split into
     *   rec32  n_rows*32 u32: word (control code for control records)
     *   recop  n_rows*32 u8: op | space << 2
     * decoded in the kernel to the u64 record above; same ownership rules. */
    uint32_t format;
    uint32_t flags;           /* HR_TRACE_F_* (below) */
    const uint32_t *rec32;
    const uint8_t *recop;
    /* format HR_TRACE_PACKED (rec, rec32, recop unused; n_rows and warp_off as
     * for U64):  packed  the segments described above;
     *            pack_off  n_warp_off u64 byte offsets into packed.
     * Same ownership rules; HOST pointers for hr_replay_trace_host. */
    const uint8_t *packed;
    const uint64_t *pack_off;
} hr_trace;

typedef struct hr_ctx hr_ctx;   /* opaque */

/* Create a context on cfg->device: uploads the FSM table, allocates the report
 * ring and the flags word.  cfg == NULL selects the defaults above. */
hr_status hr_init(const hr_config *cfg, hr_ctx **out);

/* Address sharding for multi-GPU replay: this ctx checks only
 * the global words whose shadow granule g = (word - base) >> granule_log2 has
 * hr_shard_owner(g, log2(count)) == rank, and the shared instances of
 * simulated blocks with block % count == rank.  Granules are dealt out in
 * stripes of `count` consecutive granules, one granule of each stripe per
 * rank, the assignment rotated per stripe by a hash of the stripe index; a
 * rank's shadow holds its granules packed in stripe order (local granule
 * index = g >> log2(count)).  count must be a power of two <= 64.  Call before
 * hr_shadow_alloc.  Default: rank 0 of 1. */
hr_status hr_set_shard(hr_ctx *ctx, uint32_t rank, uint32_t count);

/* Representative threads ("the memory footprint can be reduced
 * by tracking only representative threads for user-defined symmetric work
 * groups instead of tracking all threads"): from the next replay or online
 * kernel on, only threads of simulated blocks with block % block_stride == 0
 * and warps with warp % warp_stride == 0 are checked; the others still take
 * part in barriers.  The result is exactly the race set of the trace
 * restricted to those threads; races that need a non-representative thread
 * are not seen (the user asserts the symmetry).  1, 1 = every thread
 * (default).  HR_E_ARG on a zero stride. */
hr_status hr_set_representatives(hr_ctx *ctx, uint32_t block_stride, uint32_t warp_stride);

/* Warp tiles of online kernels (PAPER.md:264 __syncwarp's mask; cooperative
 * groups tiled_partition<2^tile_log2>): from the next hr_device_view on, the
 * kernel's warp-level barriers are hr_syncwarp_mask calls over whole tiles of
 * 2^tile_log2 lanes, each ordering exactly its tile.  0 or 5 = whole warps
 * (default).  Replayed traces declare their tile in kdesc[5] instead. */
hr_status hr_set_warp_tile(hr_ctx *ctx, uint32_t tile_log2);

/* Same with a shard granule of 2^granule_log2 words (0..24; hr_set_shard uses
 * 3 = 8 words, 64 B of shadow: on C5 it balances the Zipf-hot atomic words
 * best; 9 = 4 KiB leaves the hottest granule's rank 1.2x slower at N = 8).  Smaller granules spread power-law hot words over
 * more ranks; the rotation keeps a block's warps from landing on one rank
 * when a granule is a warp row (granule_log2 5). */
hr_status hr_set_shard_ex(hr_ctx *ctx, uint32_t rank, uint32_t count, uint32_t granule_log2);

/* Register a shadow region ("For each shared memory variable, a
 * shadow value data structure is allocated").
 *   HR_GLOBAL: words [base_word, base_word + n_words) get a 1:1 8-byte shadow in
 *     HBM (only this shard's granules are materialised); *dev_region (if not
 *     NULL) receives the device pointer.  Replaces any previous global region.
 *   HR_SHARED: per-block __shared__ shadow of n_words words (staged in SMEM by the
 *     replay kernel, zero = INIT at block start); base_word must be 0;
 *     *dev_region (if not NULL) receives NULL.  n_words * 8 must fit SMEM with the
 *     FSM table (<= 227 KB). */
hr_status hr_shadow_alloc(hr_ctx *ctx, hr_space space, uint64_t base_word, uint64_t n_words,
                          void **dev_region);

/* New kernel epoch: a kernel boundary orders everything, so the global shadow
 * is reset to INIT (all-zero words) on `stream`; skipped if
 * no kernel used it since the last reset.  Before that, the end-of-kernel spill
 * scan of the previous kernel is enqueued (one launch; it returns at once
 * unless that kernel's ring records overflowed).  With HR_OPT_DOUBLE_SHADOW the
 * other (already zero) buffer becomes current and the used one is zeroed on a
 * side stream after its kernel completes.  Online kernels: call it BEFORE
 * hr_device_view for the kernel (the view carries the buffer and epoch tag). */
hr_status hr_kernel_begin(hr_ctx *ctx, void *stream);

/* Replay every kernel of `t` on `stream`: for each kernel, hr_kernel_begin then
 * one launch whose grid mirrors the traced grid; each CUDA thread walks its
 * simulated thread's records and runs the per-access check; __syncthreads /
 * __syncwarp records execute real barriers and advance BC / WC.  Asynchronous;
 * races accumulate in the ring until hr_report / hr_reset_report. */
hr_status hr_replay_trace(hr_ctx *ctx, const hr_trace *t, void *stream);

/* Same with t->rec and t->warp_off in HOST memory: the records are copied to
 * ctx-owned device staging buffers on `stream`, then replayed.  Block-range
 * chunks are copied on a side stream so the copy of chunk i+1 overlaps the
 * replay of chunk i.  PACKED traces are decoded on the device chunk by chunk
 * into one u64 staging buffer right before each chunk's replay (on `stream`).
 * On a device-resident PACKED trace hr_replay_trace does the same decode
 * (and synchronously reads warp_off/pack_off to the host to plan chunks). */
hr_status hr_replay_trace_host(hr_ctx *ctx, const hr_trace *t, void *stream);

/* Encode a DEVICE trace `in` (format U64) as HR_TRACE_PACKED on `stream`.
 *   out == NULL: size query, *bytes receives the packed size (with the 16-byte
 *                slack), pack_off (DEVICE, in->n_warp_off u64) is filled.
 *   out != NULL: out (DEVICE, cap bytes) receives the segments; pack_off is
 *                filled again; HR_E_ARG if cap < the size.
 * Synchronises `stream`.  HR_E_ARG on a decreasing warp_off.  The trace's
 * other fields (kdesc, warp_off, n_rows) are shared with the packed trace. */
hr_status hr_pack_trace(hr_ctx *ctx, const hr_trace *in, uint8_t *out, uint64_t cap, uint64_t *pack_off,
                        uint64_t *bytes, void *stream);

/* Re-lay a DEVICE trace `in` (U64 or C32) out as HR_TRACE_POOLED on `stream`:
 *   rec_out == NULL: size query, *rows receives the pooled row count;
 *   otherwise rec_out (DEVICE, cap_rows*32 u64), tag_out (DEVICE, cap_rows*32
 *   u8) and warp_off_out (DEVICE, in->n_warp_off u64; warp offsets for the
 *   same kdesc) receive the pooled trace; HR_E_ARG if cap_rows < *rows.
 * Accesses this ctx's address shard does not own are dropped (an unsharded
 * ctx keeps all).  Synchronises `stream`. */
hr_status hr_pool_trace(hr_ctx *ctx, const hr_trace *in, uint64_t *rec_out, uint8_t *tag_out, uint64_t cap_rows,
                        uint64_t *warp_off_out, uint64_t *rows, void *stream);

/* Decode a DEVICE HR_TRACE_PACKED trace `in` into U64 rows: rec_out (DEVICE,
 * in->n_rows*32 u64) receives row r of every segment at rec_out[r*32..];
 * rows no segment covers are not written.  Asynchronous on `stream`. */
hr_status hr_unpack_trace(hr_ctx *ctx, const hr_trace *in, uint64_t *rec_out, void *stream);

/* Synchronise the ctx's last stream and return the unique racy addresses,
 * sorted by (kernel, space, block, word), one record per address with the
 * widest scope observed.  n_out receives the number of races (may exceed cap:
 * then only cap are written and HR_E_ARG is returned).  flags_out (may be NULL)
 * receives the sticky HR_F_* word.  Enqueues the end-of-kernel spill scan of
 * the last kernel first (a no-op on the device unless it dropped a record).
 * The result is the union of the ring and the spill store (see hr_config);
 * HR_E_INCOMPLETE (after writing what was recovered) if that is not the whole
 * racy set.  Witness fields (first_tid, first_kind, prev_state) of a record
 * recovered by a scan are the stored accessor and 0xff. */
hr_status hr_report(hr_ctx *ctx, hr_race *out, size_t cap, size_t *n_out, uint32_t *flags_out);

/* hr_report without a host round trip (a13 on the device, "report races
 * on unique memory addresses"): enqueue on `stream` (NULL = the ctx's last
 * stream) the sort of the ring's records, the merge of equal addresses
 * (widest scope) and the write of the result into pinned host memory owned by
 * the ctx.  Returns at once; nothing waits for the GPU, so a caller can
 * enqueue the next kernel's checks behind it.  Each call replaces the previous
 * result.  Runs as one CUDA graph whose first kernel reads the record count on
 * the device: up to 8192 records are sorted and merged by that one CTA in
 * shared memory; more take the graph's conditional branch, two radix sorts of
 * ring_capacity keys (the host never learns the count). */
hr_status hr_report_async(hr_ctx *ctx, void *stream);

/* The same device-side report into caller-owned DEVICE memory, for a
 * device-resident exchange (the race-set allgather of the
 * address-sharded replay runs on these buffers, no host round trip):
 *   out  DEVICE, out_cap hr_race records: the sorted unique set (the first
 *        out_cap of it);
 *   hdr  DEVICE, 4 uint32: [0] unique count (may exceed out_cap), [1] sticky
 *        flags, [2] raw ring records, [3] non-zero if the ring overflowed (the
 *        set then lives partly in the spill store: call hr_report).
 * Enqueued on `stream` (NULL = the ctx's last stream); returns at once.  The
 * buffers must stay valid until the stream reaches the report. */
hr_status hr_report_async_to(hr_ctx *ctx, void *stream, hr_race *out, uint32_t out_cap, uint32_t *hdr);

/* Wait for the last hr_report_async and copy its result out, with the same
 * contract as hr_report.  If the ring had overflowed it runs hr_report (the
 * shadow scan) instead.  HR_E_STATE without a pending hr_report_async. */
hr_status hr_report_collect(hr_ctx *ctx, hr_race *out, size_t cap, size_t *n_out, uint32_t *flags_out);

/* Merge race sets, HOST only (no CUDA call, no
 * ctx): `in` holds n hr_race records, e.g. the concatenated hr_report results
 * of N address shards after an allgather; `out` (host, cap records) receives
 * them sorted by (kernel, space, block, word), one record per address with the
 * widest scope.  *n_out = the unique count; HR_E_ARG if it exceeds cap (then
 * cap records are written) or on NULL arguments.  in and out may not overlap. */
hr_status hr_merge_races(const hr_race *in, size_t n, hr_race *out, size_t cap, size_t *n_out);

/* Per-pair race classes of already reported racy addresses:
 * `races` are the n records hr_report returned for this same device trace `t`
 * (same kernel_base); the trace is replayed again through four class-projected
 * FSMs (fsm_classes.inc) for those addresses only.  classes_out[i] (host, n
 * bytes) receives bit0 W-W, bit1 R-W, bit2 A-W, bit3 A-R: the kind pairs among
 * the race pairs of races[i].  Schedule-independent; synchronises `stream`;
 * temporary device memory ~ 32 B per race + the hash table. */
hr_status hr_race_classes(hr_ctx *ctx, const hr_trace *t, const hr_race *races, size_t n, uint8_t *classes_out,
                          void *stream);

/* Clear the ring, its counter and the flags word (asynchronous on the last stream). */
hr_status hr_reset_report(hr_ctx *ctx);

/* Device-side counters since the last hr_reset_report: [0] checked accesses,
 * [1] failed CAS (Algorithm 1 retries), [2] a7 fast exits (no atomic), [3]
 * committed CAS.  Maintained only by builds with -DHR_COUNTERS (a diagnostic
 * build: per-access atomics); zero otherwise.  Synchronises. */
hr_status hr_counters(hr_ctx *ctx, uint64_t out[4]);

/* With HR_OPT_TIMING: synchronise and return the summed device time (ms) and
 * count of the shadow resets and replay-kernel launches since the last call
 * (events recorded on the launching stream), then clear them. */
hr_status hr_replay_timing(hr_ctx *ctx, double *reset_ms, uint64_t *n_resets, double *kernel_ms,
                           uint64_t *n_kernels);

/* Number of device kernels this ctx launched since the last call (every
 * __global__ launch of libhirace, including the kernels of its CUB scans (2)
 * and radix sorts (2 + one onesweep pass per 8 key bits: 10 for the 64-bit
 * sorts of hr_report)), then clear it.  hr_report_async runs as one CUDA graph:
 * its small-set kernel always, the full-capacity sort path (keys, 2 sorts over
 * the key bits that can be set, heads, scan, emit) only when the ring held more
 * than 8192 records — that path counts its own kernels on the device, so this
 * call synchronises the device to read them.  Lets a harness state how many
 * kernels ran inside a timed region. */
hr_status hr_launch_count(hr_ctx *ctx, uint64_t *n_launches);

/* Copy of the compiled-in FSM table (2048 bytes, index state<<6|kind<<4|sync<<2|rel)
 * and per-state flags (32 bytes).  Either pointer may be NULL. */
hr_status hr_fsm_table(uint8_t *table2048, uint8_t *flags32);

/* Copy the packed device context (struct hr_dev in hr_device.cuh, by value)
 * for a user kernel instrumented online into hr_dev_out (size >= sizeof(hr_dev)).
 * Take it after hr_kernel_begin for that kernel: it holds the current global
 * shadow buffer and epoch tag.  The kernel's id (hr_dev.kernel_id) may be set
 * by the caller; every thread must call hr_thread_begin first and
 * hr_thread_end last (ring-overflow recovery of shared races). */
hr_status hr_device_view(hr_ctx *ctx, void *hr_dev_out, size_t size);

const char *hr_last_error(hr_ctx *ctx);
void hr_destroy(hr_ctx *ctx);

#ifdef __cplusplus
}
#endif

/* The address-shard owner function (hr_set_shard above), inline so that
 * trace partitioners and the device check agree on it. */
#ifdef __CUDACC__
#define HR_HD __host__ __device__ __forceinline__
#else
#define HR_HD static inline
#endif
HR_HD uint32_t hr_shard_rot(uint64_t stripe, uint32_t log2n)
{
    return log2n ? ((uint32_t)(stripe ^ (stripe >> 32)) * 0x9E3779B1u) >> (32u - log2n) : 0u;
}
HR_HD uint32_t hr_shard_owner(uint64_t granule, uint32_t log2n)
{
    return ((uint32_t)granule + hr_shard_rot(granule >> log2n, log2n)) & ((1u << log2n) - 1u);
}
/* inverse: the granule of `rank` in stripe `stripe` */
HR_HD uint64_t hr_shard_granule(uint64_t stripe, uint32_t rank, uint32_t log2n)
{
    return (stripe << log2n) | ((rank - hr_shard_rot(stripe, log2n)) & ((1u << log2n) - 1u));
}
#endif /* HR_H_ */
