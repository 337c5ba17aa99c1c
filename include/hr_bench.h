/*
 * hr_bench.h — online-instrumentation benchmark kernels (C ABI).
 *
 * Real CUDA kernels of three BASELINE configs, each built twice from one
 * template: plain, and instrumented with the device API of hr_device.cuh
 * (hr_thread_begin, hr_check_read/_write/_atomic, hr_syncthreads), the way
 * the paper's wrapper instruments every access.  Their
 * ratio is the paper's instrumented-vs-uninstrumented slowdown (PAPER.md:868,
 * 898).  Each instrumented kernel performs exactly the access stream of the
 * corresponding tracegen generator, so its race report is checked against the
 * oracle on that trace (tests/test_gpu_online.py).
 *
 * Monitored data live in one int array `data` (device, caller-owned); shadow
 * word k <-> data[k].  The ctx must have a global region
 * covering the words used (base 0) and a shared budget >= the kernel's.
 * `instrumented` = 0 runs the plain kernel (ctx may be NULL).  `kernel_id` is
 * written into race records.  Streams are cudaStream_t as void*.  Returns
 * hr_status; launches are asynchronous.
 */
#ifndef HR_BENCH_H_
#define HR_BENCH_H_

#include <stdint.h>

#include "hr.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C1: 1 block x 32 threads, __shared__ s[256]; data[0, rounds*256) input,
 * data[rounds*256 + r] outputs.  removed: -1 none, 0 after the load,
 * s in {128..1} after reduction step s (tracegen.programs.c1_tree_reduction). */
hr_status hrb_c1(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int rounds, int removed, int *data,
                 void *stream);

/* C1 written with the transparent wrapper of hr_array.cuh (always instrumented). */
hr_status hrb_c1_array(hr_ctx *ctx, uint32_t kernel_id, int rounds, int removed, int *data, void *stream);

/* C3: (n/16)^2 blocks x 256 threads, two 18x18 SMEM tiles, `sweeps` Jacobi
 * sweeps; data[0, n*n) input, data[n*n, 2n*n) output; removed = sweep whose
 * trailing barrier is dropped, -1 none (tracegen.stencil.stencil_trace). */
hr_status hrb_c3(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int n, int sweeps, int removed, int *data,
                 void *stream);

/* C4 BFS level L (thread per vertex, n vertices, CSR rp/col on device):
 * data[0, n) = level[]; flevel = final BFS levels (unmonitored, device) decide
 * the frontier (flevel[v] == L) and the writes (flevel[x] == L+1) so the access
 * stream equals tracegen.c4's.  racy: plain reads/writes; else atomics. */
hr_status hrb_c4_level(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int racy, uint32_t n,
                       const uint64_t *rp, const uint32_t *col, const int *flevel, int level, int *data,
                       void *stream);

/* C4 histogram of out-degree into data[n, n+1024) (bin = min(deg, 1023)). */
hr_status hrb_c4_hist(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int racy, uint32_t n,
                      const uint64_t *rp, int *data, void *stream);

/* Sub-warp __syncwarp(mask) online (hr_syncwarp_mask): 1 block x
 * 32 threads; lane l writes data[l]; lanes 0..15 call __syncwarp(0x0000ffff);
 * lane l reads data[(l & 16) | ((l + 1) & 15)] and writes data[32 + l]
 * (unmonitored).  Monitored words [0, 32). */
hr_status hrb_masked_sync(hr_ctx *ctx, uint32_t kernel_id, int *data, void *stream);

/* Uninstrumented replay of a device trace (hr.h's hr_trace): the same grid,
 * record walk and barriers as hr_replay_trace, but each global record performs
 * only the raw 4-byte data access (read / write / atomicAdd on data[word] for
 * global records, on the block's __shared__ int[smem_words] for shared ones;
 * global words >= data_words skipped).  The denominator of the replay slowdown
 * (SURVEY §8(d) "Slowdown"). */
hr_status hrb_raw_replay(const hr_trace *t, int *data, uint64_t data_words, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HR_BENCH_H_ */
