// common.cuh -- shared device helpers of the mpjsvd CUDA path (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define MPJ_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) {                             \
            mpj_record_cuda_error(_e, #expr, __FILE__, __LINE__); \
            return _e == cudaErrorMemoryAllocation ? -6 : -4; \
        }                                                    \
    } while (0)

void mpj_record_cuda_error(cudaError_t e, const char* what, const char* file, int line);

// mpjsvd_options.diag_timing of the call in progress on this host thread (set at every entry point)
extern thread_local int g_mpj_diag;
extern thread_local int g_mpj_qrp_pe;   // options.qrp_panel_stages (-1 auto)

// count of kernel launches issued by the engine (reported in stats)
extern thread_local int64_t g_mpj_launches;
#define MPJ_LAUNCHED() (++g_mpj_launches)

// Raise a kernel's dynamic shared-memory limit on the CURRENT device (the attribute is per
// device; cached per (kernel, device) under a lock, so handles on several GPUs or threads are safe).
cudaError_t mpj_set_smem(const void* fn, size_t bytes);
template <typename F>
static inline cudaError_t set_smem(F* fn, size_t bytes) { return mpj_set_smem(reinterpret_cast<const void*>(fn), bytes); }

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---- device helpers ------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide deterministic sum (fixed tree).  `red` must hold >= 32 T.
// All threads receive the result.  Contains two __syncthreads().
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T r = (lane < nw) ? red[lane] : T(0);
    r = warp_sum(r);
    __syncthreads();
    return r;
}
template <typename T>
__device__ __forceinline__ T block_max(T v, T* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T r = (lane < nw) ? red[lane] : T(0);
    r = warp_max(r);
    __syncthreads();
    return r;
}

// wall-clock nanoseconds (for spin-wait time-outs that must not depend on the clock rate,
// time-slicing or a sanitizer's slowdown)
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// a consumer gives up waiting for a producer after this long (a hung producer, not a slow one)
constexpr unsigned long long MPJ_SPIN_TIMEOUT_NS = 120ull * 1000000000ull;

// atomic max of a non-negative double via its bit pattern (exact, order-free)
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// Circle-method (round-robin) schedule, closed form:
// slot j of round r over M slots holds 0 if j == 0, else 1 + ((j-1-r) mod (M-1)).
__device__ __host__ __forceinline__ int rr_slot(int r, int j, int M) {
    if (j == 0) return 0;
    int v = (j - 1 - r) % (M - 1);
    if (v < 0) v += M - 1;
    return 1 + v;
}
