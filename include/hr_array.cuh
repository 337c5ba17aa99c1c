/*
 * hr_array.cuh — transparent online instrumentation.
 *
 * The paper instruments user code with "a templated wrapper class to monitor
 * user data structures ... The wrapper then overrides relevant operators (for
 * example, the subscript or array index operator operator[]) to intercept
 * memory access events and update the associated shadow value transparently.
 * This approach also requires overriding other relevant functions, such as
 * atomic functions and synchronization primitives.".
 *
 * hr_array<T> wraps a global or __shared__ array of 4-byte elements whose
 * element i is monitored word base + i:
 *
 *     hr_ctx_dev  ctx(d);                          // per-thread checker state
 *     hr_array<int> a(ctx, data, HR_GLOBAL, 0);    // data[k] <-> shadow word k
 *     int v = a[i];         // hr_check_read, then the load
 *     a[j] = v + 1;         // hr_check_write, then the store
 *     a[j] += 2;            // read then write (two checked accesses)
 *     hr_atomic_add(a, k, 1);   // hr_check_atomic, then atomicAdd
 *     ctx.syncthreads();        // hr_syncthreads: barrier + block clock
 *     ctx.end();                // hr_thread_end: last statement of every thread
 *
 * All checks run the same device core as the replay (hr_device.cuh).
 */
#ifndef HR_ARRAY_CUH_
#define HR_ARRAY_CUH_

#include "hr_device.cuh"

/* Per-thread checker state: the device view plus this thread's registers. */
struct hr_ctx_dev {
    const hr_dev &d;
    hr_thr t;
    __device__ hr_ctx_dev(const hr_dev &dev, unsigned char *smem_fsm, unsigned long long *smem_shadow,
                          uint32_t smem_words)
        : d(dev), t(hr_thread_begin(dev, smem_fsm, smem_shadow, smem_words)) {}
    __device__ __forceinline__ void syncthreads() { hr_syncthreads(d, t); }
    __device__ __forceinline__ void syncwarp() { hr_syncwarp(d, t); }
    /* end of the block's checks (hr_thread_end): every thread, after its last access */
    __device__ __forceinline__ void end() { hr_thread_end(d, t); }
};

template <typename T>
struct hr_array {
    static_assert(sizeof(T) == 4, "hr_array monitors 4-byte words (reading R5)");
    hr_ctx_dev &c;
    T *data;
    hr_space space;
    uint64_t base;          /* monitored word of element 0 */

    __device__ hr_array(hr_ctx_dev &ctx, T *p, hr_space sp, uint64_t base_word)
        : c(ctx), data(p), space(sp), base(base_word) {}

    struct ref {
        hr_array &a;
        uint64_t i;
        __device__ __forceinline__ operator T() const
        {
            hr_check_read(a.c.d, a.c.t, a.space, a.base + i);
            return a.data[i];
        }
        __device__ __forceinline__ ref &operator=(T v)
        {
            hr_check_write(a.c.d, a.c.t, a.space, a.base + i);
            a.data[i] = v;
            return *this;
        }
        __device__ __forceinline__ ref &operator=(const ref &o) { return *this = (T)o; }
        __device__ __forceinline__ ref &operator+=(T v) { return *this = (T)(*this) + v; }
        __device__ __forceinline__ ref &operator-=(T v) { return *this = (T)(*this) - v; }
    };

    __device__ __forceinline__ ref operator[](uint64_t i) { return ref{*this, i}; }
};

/* atomics: a third class of memory action */
template <typename T>
__device__ __forceinline__ T hr_atomic_add(hr_array<T> &a, uint64_t i, T v)
{
    hr_check_atomic(a.c.d, a.c.t, a.space, a.base + i);
    return atomicAdd(&a.data[i], v);
}

template <typename T>
__device__ __forceinline__ T hr_atomic_min(hr_array<T> &a, uint64_t i, T v)
{
    hr_check_atomic(a.c.d, a.c.t, a.space, a.base + i);
    return atomicMin(&a.data[i], v);
}

template <typename T>
__device__ __forceinline__ T hr_atomic_cas(hr_array<T> &a, uint64_t i, T cmp, T v)
{
    hr_check_atomic(a.c.d, a.c.t, a.space, a.base + i);
    return atomicCAS(&a.data[i], cmp, v);
}

#endif /* HR_ARRAY_CUH_ */
