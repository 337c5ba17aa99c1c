/*
 * hr_online.cu — online-instrumented benchmark kernels (include/hr_bench.h).
 *
 * Each kernel is one template compiled twice: INSTR = false is the plain
 * kernel; INSTR = true calls the device API before every monitored access and
 * replaces __syncthreads by hr_syncthreads, as the paper's wrapper does for
 * operator[] and the barrier primitives.  The access order
 * per thread matches the tracegen generators record for record.
 */
#include <cuda_runtime.h>

#include "hr.h"
#include "hr_bench.h"
#include "hr_array.cuh"
#include "hr_device.cuh"
#include "hr_records.cuh"

namespace {

/* run-time options the fast (I = 2) instantiation does not read */
inline bool rt_opts(const hr_dev &d)
{
    return d.options & (HR_OPT_NO_COALESCE | HR_OPT_NO_FASTEXIT | HR_OPT_SPECULATE | HR_OPT_SMEM32);
}

template <int I>
__device__ __forceinline__ void chk(const hr_dev &d, hr_thr &t, hr_space sp, uint64_t w, int kind)
{
    if (I) {
        /* I = 1: options read at run time; I = 2: a ctx without ablation / SMEM32 options */
        if (kind == HR_READ) hr_check_read<I == 1>(d, t, sp, w);
        else if (kind == HR_WRITE) hr_check_write<I == 1>(d, t, sp, w);
        else hr_check_atomic<I == 1>(d, t, sp, w);
    }
}

template <int I>
__device__ __forceinline__ void bar(const hr_dev &d, hr_thr &t)
{
    if (I) hr_syncthreads(d, t);
    else __syncthreads();
}

/* ---- C1: tree reduction, 1 block x 32 threads ---- */
template <int I>
__global__ void __launch_bounds__(32) c1_kernel(hr_dev d, int *data, int rounds, int removed)
{
    __shared__ int s[256];
    __shared__ __align__(16) unsigned char fsm[HR_FSM_SMEM_BYTES];
    __shared__ unsigned long long sh[I ? 256 : 1];
    hr_thr t;
    if (I) t = hr_thread_begin(d, fsm, sh, 256);
    const int lane = threadIdx.x;
    const int out = rounds * 256;
    for (int r = 0; r < rounds; r++) {
        for (int i = lane; i < 256; i += 32) {
            chk<I>(d, t, HR_GLOBAL, r * 256 + i, HR_READ);
            int v = data[r * 256 + i];
            chk<I>(d, t, HR_SHARED, i, HR_WRITE);
            s[i] = v;
        }
        if (removed != 0) bar<I>(d, t);
        for (int st = 128; st >= 1; st >>= 1) {
            for (int i = lane; i < st; i += 32) {
                chk<I>(d, t, HR_SHARED, i, HR_READ);
                int a = s[i];
                chk<I>(d, t, HR_SHARED, i + st, HR_READ);
                int b = s[i + st];
                chk<I>(d, t, HR_SHARED, i, HR_WRITE);
                s[i] = a + b;
            }
            if (removed != st) bar<I>(d, t);
        }
        if (lane == 0) {
            chk<I>(d, t, HR_SHARED, 0, HR_READ);
            int v = s[0];
            chk<I>(d, t, HR_GLOBAL, out + r, HR_WRITE);
            data[out + r] = v;
        }
        bar<I>(d, t);
    }
    if (I) hr_thread_end(d, t);
}

/* ---- C1 again, written against the transparent wrapper (hr_array.cuh):
 * the kernel body reads like the uninstrumented code ---- */
__global__ void __launch_bounds__(32) c1_array_kernel(hr_dev d, int *data, int rounds, int removed)
{
    __shared__ int s_raw[256];
    __shared__ __align__(16) unsigned char fsm[HR_FSM_SMEM_BYTES];
    __shared__ unsigned long long sh[256];
    hr_ctx_dev ctx(d, fsm, sh, 256);
    hr_array<int> g(ctx, data, HR_GLOBAL, 0);
    hr_array<int> s(ctx, s_raw, HR_SHARED, 0);
    const int lane = threadIdx.x, out = rounds * 256;
    for (int r = 0; r < rounds; r++) {
        for (int i = lane; i < 256; i += 32) s[i] = g[r * 256 + i];
        if (removed != 0) ctx.syncthreads();
        for (int st = 128; st >= 1; st >>= 1) {
            for (int i = lane; i < st; i += 32) {
                int a = s[i];
                int b = s[i + st];
                s[i] = a + b;
            }
            if (removed != st) ctx.syncthreads();
        }
        if (lane == 0) g[out + r] = s[0];
        ctx.syncthreads();
    }
    ctx.end();
}

/* ---- C3: 2D Jacobi stencil through two SMEM tiles ---- */
template <int I>
__global__ void __launch_bounds__(256) c3_kernel(hr_dev d, int *data, int n, int sweeps, int removed)
{
    constexpr int T = 16, H = 18, TILE = H * H;
    __shared__ int tile[2][TILE];
    __shared__ __align__(16) unsigned char fsm[HR_FSM_SMEM_BYTES];
    __shared__ unsigned long long sh[I ? 2 * TILE : 1];
    hr_thr t;
    if (I) t = hr_thread_begin(d, fsm, sh, 2 * TILE);
    const int ltid = threadIdx.x, ty = ltid / T, tx = ltid % T;
    const int tiles = n / T, bx = blockIdx.x % tiles, by = blockIdx.x / tiles;
    for (int k = 0; k < 2; k++) {
        const int cell = ltid + 256 * k;
        if (cell < TILE) {
            const int hy = cell / H, hx = cell % H;
            const int gy = min(max(by * T + hy - 1, 0), n - 1), gx = min(max(bx * T + hx - 1, 0), n - 1);
            chk<I>(d, t, HR_GLOBAL, (uint64_t)gy * n + gx, HR_READ);
            int v = data[gy * n + gx];
            chk<I>(d, t, HR_SHARED, cell, HR_WRITE);
            tile[0][cell] = v;
        }
    }
    bar<I>(d, t);
    int src = 0, dst = 1;
    const int c = (ty + 1) * H + (tx + 1);
    for (int s = 0; s < sweeps; s++) {
        const int offs[5] = {0, -H, H, -1, 1};
        int acc = 0;
#pragma unroll
        for (int o = 0; o < 5; o++) {
            chk<I>(d, t, HR_SHARED, src * TILE + c + offs[o], HR_READ);
            acc += tile[src][c + offs[o]];
        }
        chk<I>(d, t, HR_SHARED, dst * TILE + c, HR_WRITE);
        tile[dst][c] = acc / 5;
        if (s != removed) bar<I>(d, t);
        src ^= 1;
        dst ^= 1;
    }
    const int gy = by * T + ty, gx = bx * T + tx;
    chk<I>(d, t, HR_SHARED, src * TILE + c, HR_READ);
    int v = tile[src][c];
    chk<I>(d, t, HR_GLOBAL, (uint64_t)n * n + (uint64_t)gy * n + gx, HR_WRITE);
    data[n * n + gy * n + gx] = v;
    if (I) hr_thread_end(d, t);
}

/* ---- C4: BFS level step and degree histogram, thread per vertex ---- */
template <int I>
__global__ void __launch_bounds__(256) c4_level_kernel(hr_dev d, int *data, uint32_t n, const uint64_t *rp,
                                                       const uint32_t *col, const int *flevel, int L, int racy)
{
    __shared__ __align__(16) unsigned char fsm[HR_FSM_SMEM_BYTES];
    __shared__ unsigned long long sh[1];
    hr_thr t;
    if (I) t = hr_thread_begin(d, fsm, sh, 0);
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    if (racy) {
        chk<I>(d, t, HR_GLOBAL, v, HR_READ);
        volatile int lv = data[v];
        (void)lv;
    } else {
        chk<I>(d, t, HR_GLOBAL, v, HR_ATOMIC);
        atomicOr(&data[v], 0);
    }
    if (flevel[v] != L) return;
    for (uint64_t k = rp[v]; k < rp[v + 1]; k++) {
        const uint32_t x = col[k];
        if (racy) {
            chk<I>(d, t, HR_GLOBAL, x, HR_READ);
            volatile int lx = data[x];
            (void)lx;
            if (flevel[x] == L + 1) {
                chk<I>(d, t, HR_GLOBAL, x, HR_WRITE);
                data[x] = L + 1;
            }
        } else {
            chk<I>(d, t, HR_GLOBAL, x, HR_ATOMIC);
            atomicMin(&data[x], L + 1);
        }
    }
}

template <int I>
__global__ void __launch_bounds__(256) c4_hist_kernel(hr_dev d, int *data, uint32_t n, const uint64_t *rp,
                                                      int racy)
{
    __shared__ __align__(16) unsigned char fsm[HR_FSM_SMEM_BYTES];
    __shared__ unsigned long long sh[1];
    hr_thr t;
    if (I) t = hr_thread_begin(d, fsm, sh, 0);
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint64_t deg = rp[v + 1] - rp[v];
    const uint64_t bin = n + (deg < 1023 ? deg : 1023);
    if (racy) {
        chk<I>(d, t, HR_GLOBAL, bin, HR_READ);
        int h = data[bin];
        chk<I>(d, t, HR_GLOBAL, bin, HR_WRITE);
        data[bin] = h + 1;
    } else {
        chk<I>(d, t, HR_GLOBAL, bin, HR_ATOMIC);
        atomicAdd(&data[bin], 1);
    }
}

/* ---- sub-warp __syncwarp(mask), online: lane l writes word l,
 * lanes 0..15 meet a __syncwarp(0x0000ffff) (hr_syncwarp_mask: no happens-before
 * edge, HR_F_MODEL_VIOLATION), then lane l reads its tile neighbour's word ---- */
__global__ void __launch_bounds__(32) masked_sync_kernel(hr_dev d, int *data)
{
    __shared__ __align__(16) unsigned char fsm[HR_FSM_SMEM_BYTES];
    __shared__ unsigned long long sh[1];
    hr_thr t = hr_thread_begin(d, fsm, sh, 0);
    const uint32_t lane = threadIdx.x;
    hr_check_write(d, t, HR_GLOBAL, lane);
    data[lane] = (int)lane;
    if (lane < 16u) hr_syncwarp_mask(d, t, 0x0000ffffu);
    const uint32_t r = (lane & 16u) | ((lane + 1u) & 15u);
    hr_check_read(d, t, HR_GLOBAL, r);
    data[32 + lane] = data[r];
    hr_thread_end(d, t);
}

/* ---- uninstrumented replay: the same record walk and barriers as
 * hr_replay_kernel, but each access is the raw data access (4-byte word) ---- */
template <typename SRC>
__global__ void __launch_bounds__(1024, 2) raw_replay_kernel(SRC src, const uint64_t *__restrict__ woff,
                                                             uint32_t warps, uint32_t lanes, int *data,
                                                             uint64_t data_words, uint32_t smem_words)
{
    extern __shared__ int sdata[];                        /* the block's __shared__ data instance */
    for (uint32_t i = threadIdx.x; i < smem_words; i += blockDim.x) sdata[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * warps + warp;
    const uint64_t r0 = woff[gw], r1 = woff[gw + 1];
    const bool active = lane < lanes;
    const uint64_t n = r1 - r0;
    typename SRC::raw_t x1 = (active && n > 0) ? src.load(r0, lane) : SRC::nop();
    typename SRC::raw_t x2 = (active && n > 1) ? src.load(r0 + 1, lane) : SRC::nop();
    int acc = 0;
    for (uint64_t i = 0; i < n; i++) {
        const uint64_t x = SRC::decode(x1);
        x1 = x2;
        x2 = (active && i + 2 < n) ? src.load(r0 + i + 2, lane) : SRC::nop();
        const uint32_t op = (uint32_t)(x >> 62);
        const uint64_t w = x & HR_WORD_MASK;
        const unsigned st = __ballot_sync(0xffffffffu, op == 3u && w == 1u);
        const unsigned sw = __ballot_sync(0xffffffffu, op == 3u && w == 2u);
        if (st) { __syncthreads(); continue; }
        if (sw) { __syncwarp(); continue; }
        if (op == 3u) continue;
        if ((x >> 61) & 1u) {                                /* shared data access */
            if (w >= smem_words) continue;
            if (op == 0u) acc += ((volatile int *)sdata)[w];
            else if (op == 1u) ((volatile int *)sdata)[w] = (int)i;
            else atomicAdd(&sdata[w], 1);
            continue;
        }
        if (w >= data_words) continue;
        if (op == 0u) acc += __ldcg(&data[w]);
        else if (op == 1u) data[w] = (int)i;
        else atomicAdd(&data[w], 1);
    }
    if (acc == 0x7fffffff) data[0] = acc;
}

hr_status prepare(hr_ctx *ctx, int instrumented, uint32_t kernel_id, void *stream, hr_dev *d)
{
    memset(d, 0, sizeof *d);
    if (!instrumented) return HR_OK;
    if (!ctx) return HR_E_ARG;
    /* kernel boundary first (fresh global shadow / next epoch tag, and the end-of-kernel
     * spill scan of the previous kernel), then the view of the state this kernel uses */
    hr_status st = hr_kernel_begin(ctx, stream);
    if (st) return st;
    st = hr_device_view(ctx, d, sizeof *d);
    if (st) return st;
    d->kernel_id = kernel_id;
    return HR_OK;
}

hr_status launched()
{
    return cudaGetLastError() == cudaSuccess ? HR_OK : HR_E_CUDA;
}

}  // namespace

extern "C" hr_status hrb_raw_replay(const hr_trace *t, int *data, uint64_t data_words, void *stream)
{
    if (!t) return HR_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    for (uint32_t k = 0; k < t->n_kernels; k++) {
        const uint64_t *kd = t->kdesc + 8ull * k;
        if (kd[0] == 0) continue;
        const dim3 g((unsigned)kd[0]), b((unsigned)(kd[1] * 32));
        const uint32_t sw = (uint32_t)kd[3];
        if (t->format == HR_TRACE_C32)
            raw_replay_kernel<<<g, b, sw * 4, s>>>(hr_src_c32{t->rec32, t->recop}, t->warp_off + kd[4],
                                                   (uint32_t)kd[1], (uint32_t)kd[2], data, data_words, sw);
        else
            raw_replay_kernel<<<g, b, sw * 4, s>>>(hr_src_u64{t->rec}, t->warp_off + kd[4], (uint32_t)kd[1],
                                                   (uint32_t)kd[2], data, data_words, sw);
        if (cudaGetLastError() != cudaSuccess) return HR_E_CUDA;
    }
    return HR_OK;
}

extern "C" hr_status hrb_masked_sync(hr_ctx *ctx, uint32_t kernel_id, int *data, void *stream)
{
    hr_dev d;
    hr_status st = prepare(ctx, 1, kernel_id, stream, &d);
    if (st) return st;
    masked_sync_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d, data);
    return launched();
}

extern "C" hr_status hrb_c1(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int rounds, int removed, int *data,
                            void *stream)
{
    hr_dev d;
    hr_status st = prepare(ctx, instrumented, kernel_id, stream, &d);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (!instrumented) c1_kernel<0><<<1, 32, 0, s>>>(d, data, rounds, removed);
    else if (rt_opts(d)) c1_kernel<1><<<1, 32, 0, s>>>(d, data, rounds, removed);
    else c1_kernel<2><<<1, 32, 0, s>>>(d, data, rounds, removed);
    return launched();
}

extern "C" hr_status hrb_c1_array(hr_ctx *ctx, uint32_t kernel_id, int rounds, int removed, int *data,
                                  void *stream)
{
    hr_dev d;
    hr_status st = prepare(ctx, 1, kernel_id, stream, &d);
    if (st) return st;
    c1_array_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d, data, rounds, removed);
    return launched();
}

extern "C" hr_status hrb_c3(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int n, int sweeps, int removed,
                            int *data, void *stream)
{
    if (n % 16) return HR_E_ARG;
    hr_dev d;
    hr_status st = prepare(ctx, instrumented, kernel_id, stream, &d);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned blocks = (unsigned)((n / 16) * (n / 16));
    if (!instrumented) c3_kernel<0><<<blocks, 256, 0, s>>>(d, data, n, sweeps, removed);
    else if (rt_opts(d)) c3_kernel<1><<<blocks, 256, 0, s>>>(d, data, n, sweeps, removed);
    else c3_kernel<2><<<blocks, 256, 0, s>>>(d, data, n, sweeps, removed);
    return launched();
}

extern "C" hr_status hrb_c4_level(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int racy, uint32_t n,
                                  const uint64_t *rp, const uint32_t *col, const int *flevel, int level, int *data,
                                  void *stream)
{
    hr_dev d;
    hr_status st = prepare(ctx, instrumented, kernel_id, stream, &d);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned blocks = (n + 255) / 256;
    if (!instrumented) c4_level_kernel<0><<<blocks, 256, 0, s>>>(d, data, n, rp, col, flevel, level, racy);
    else if (rt_opts(d)) c4_level_kernel<1><<<blocks, 256, 0, s>>>(d, data, n, rp, col, flevel, level, racy);
    else c4_level_kernel<2><<<blocks, 256, 0, s>>>(d, data, n, rp, col, flevel, level, racy);
    return launched();
}

extern "C" hr_status hrb_c4_hist(hr_ctx *ctx, int instrumented, uint32_t kernel_id, int racy, uint32_t n,
                                 const uint64_t *rp, int *data, void *stream)
{
    hr_dev d;
    hr_status st = prepare(ctx, instrumented, kernel_id, stream, &d);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned blocks = (n + 255) / 256;
    if (!instrumented) c4_hist_kernel<0><<<blocks, 256, 0, s>>>(d, data, n, rp, racy);
    else if (rt_opts(d)) c4_hist_kernel<1><<<blocks, 256, 0, s>>>(d, data, n, rp, racy);
    else c4_hist_kernel<2><<<blocks, 256, 0, s>>>(d, data, n, rp, racy);
    return launched();
}
