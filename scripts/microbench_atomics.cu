// Microbenchmark of the primitives the check is built from, on B200:
// 64-bit CAS / relaxed loads on random or coalesced words, HBM-resident or
// L2-resident, with 1..4 independent operations in flight per thread.
// Gives the atomic roofline denominator (SURVEY §8(d) "L2-atomic roofline:
// not published for B200. Measure it").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

template <int OP, int ILP, bool COAL>
__global__ void kern(unsigned long long *a, uint64_t mask, int iters, unsigned long long *sink)
{
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; it++) {
        uint64_t idx[ILP];
#pragma unroll
        for (int k = 0; k < ILP; k++) {
            uint64_t h = mix(tid * 1315423911ull + (uint64_t)(it * ILP + k) * 0x1234567ull);
            idx[k] = COAL ? (((h >> 5) << 5) + (threadIdx.x & 31)) & mask : h & mask;
            if (COAL) idx[k] = ((mix((tid >> 5) * 77 + it * ILP + k) << 5) + (threadIdx.x & 31)) & mask;
        }
        unsigned long long r[ILP];
#pragma unroll
        for (int k = 0; k < ILP; k++) {
            if (OP == 0) r[k] = atomicCAS(&a[idx[k]], 0ull, tid + 1);           // CAS (first touch wins)
            else if (OP == 1) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r[k]) : "l"(&a[idx[k]]));
            else if (OP == 2) r[k] = atomicCAS(&a[idx[k]], 0xdeadull, tid + 1);  // always-failing CAS
            else if (OP == 3) { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r[k]) : "l"(&a[idx[k]]));
                   r[k] = atomicCAS(&a[idx[k]], r[k], r[k] + 1); }              // load + dependent CAS
            else { a[idx[k]] = tid + 1; r[k] = 0; }                              // plain 8-byte store
        }
#pragma unroll
        for (int k = 0; k < ILP; k++) acc += r[k];
    }
    if (acc == 42) *sink = acc;
}

template <int OP, int ILP, bool COAL>
void run(const char *name, unsigned long long *a, uint64_t words, int blocks, int threads, int iters,
         unsigned long long *sink)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemset(a, 0, words * 8);
    kern<OP, ILP, COAL><<<blocks, threads>>>(a, words - 1, 1, sink);   // warm
    cudaMemset(a, 0, words * 8);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<OP, ILP, COAL><<<blocks, threads>>>(a, words - 1, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * ILP;
    printf("%-34s words=2^%-2d ilp=%d thr=%d: %8.2f Gop/s  (%.3f ms, %.2f us/op/thread)\n", name,
           63 - __builtin_clzll(words), ILP, blocks * threads, ops / ms / 1e6, ms,
           ms * 1e3 / (iters * ILP));
}

int main(int argc, char **argv)
{
    /* optional: cudaLimitMaxL2FetchGranularity in bytes (0..128), and "big" to run only 2^32 words */
    if (argc > 1) {
        size_t g = (size_t)atoi(argv[1]), got = 0;
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("L2 fetch granularity limit set %zu, reads back %zu\n", g, got);
    }
    const bool only_big = argc > 2;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *a, *sink;
    uint64_t big = 1ull << 32;           // 32 GiB: HBM-resident, cold
    uint64_t small = 1ull << 23;         // 64 MiB: L2-resident
    cudaMalloc(&a, big * 8);
    cudaMalloc(&sink, 8);
    int blocks = nsm * 8, thr = 256, it = 64;
    printf("SMs %d, threads %d\n", nsm, blocks * thr);
    for (int lg = only_big ? 32 : 22; lg <= 32; lg += 1) {
        uint64_t w = 1ull << lg;
        run<1, 4, false>("LD random sweep", a, w, blocks, thr, it, sink);
        run<0, 4, false>("CAS random sweep", a, w, blocks, thr, it, sink);
    }
    run<4, 4, false>("ST random", a, big, blocks, thr, it, sink);
    run<3, 1, false>("LD+CAS random", a, big, blocks, thr, it, sink);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
