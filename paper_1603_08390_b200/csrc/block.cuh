// Block-level primitives used by the scan and merge kernels.
#pragma once

#include "common.cuh"

namespace genie {

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
    return x;
}

// Exclusive scan over the whole block.  `sums` is shared scratch of >= 32
// elements.  Every thread must call it.  Returns the exclusive prefix and the
// block total.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* sums, T& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    const T incl = warp_inclusive_scan(v);
    if (lane == 31) sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? sums[lane] : T(0);
        w = warp_inclusive_scan(w);
        if (lane < nwarps) sums[lane] = w;
    }
    __syncthreads();
    const T off = warp ? sums[warp - 1] : T(0);
    total = sums[nwarps - 1];
    __syncthreads();
    return off + incl - v;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sums) {
    T total;
    block_exclusive_scan(v, sums, total);
    return total;
}

// In-place ascending bitonic sort of n (power of two) keys in shared memory.
__device__ __forceinline__ void bitonic_sort_smem(uint64_t* keys, uint32_t n) {
    for (uint32_t size = 2; size <= n; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace genie
