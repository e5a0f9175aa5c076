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

// Leaves the k smallest of n distinct keys (n <= 16 * blockDim.x) sorted
// ascending in keys[0, min(k, n)).  MSD radix selection of the k-th smallest
// key over the bytes where the keys differ, then a bitonic sort of the k
// winners only.  `scratch` is >= 256 + 8 u32 of shared memory.
__device__ inline void select_k_smallest(uint64_t* keys, uint32_t n, uint32_t k, uint32_t* scratch) {
    uint32_t* hist = scratch;
    uint32_t* ctl = scratch + 256;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    if (k >= n || n <= 256) {
        uint32_t N = 1;
        while (N < n) N <<= 1;
        for (uint32_t i = n + tid; i < N; i += blockDim.x) keys[i] = ~0ull;
        __syncthreads();
        bitonic_sort_smem(keys, N);
        return;
    }
    // bytes where the keys differ
    uint64_t lo = ~0ull, hi = 0;
    for (uint32_t i = tid; i < n; i += blockDim.x) {
        lo = min(lo, keys[i]);
        hi = max(hi, keys[i]);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    if (tid == 0) {
        reinterpret_cast<uint64_t*>(ctl)[0] = ~0ull;
        reinterpret_cast<uint64_t*>(ctl)[1] = 0;
    }
    __syncthreads();
    if (lane == 0) {
        atomicMin(reinterpret_cast<unsigned long long*>(ctl), lo);
        atomicMax(reinterpret_cast<unsigned long long*>(ctl) + 1, hi);
    }
    __syncthreads();
    lo = reinterpret_cast<uint64_t*>(ctl)[0];
    hi = reinterpret_cast<uint64_t*>(ctl)[1];
    __syncthreads();
    const int b0 = 7 - (__clzll(lo ^ hi) >> 3);  // highest byte where keys differ
    // bytes above b0 are common to all keys
    uint64_t prefix = b0 >= 7 ? 0ull : (lo & ~((1ull << (8 * (b0 + 1))) - 1ull));
    uint32_t need = k;  // rank of the cutoff among keys matching the prefix
    for (int b = b0; b >= 0; --b) {
        for (uint32_t i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const int sh = 8 * b;
        for (uint32_t i = tid; i < n; i += blockDim.x) {
            const uint64_t x = keys[i];
            if (b == 7 || ((x ^ prefix) >> (sh + 8)) == 0) atomicAdd(&hist[(x >> sh) & 0xffu], 1u);
        }
        __syncthreads();
        if (tid < 32) {  // smallest digit whose cumulative count reaches need
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = hist[lane * 8 + j];
                tot += c[j];
            }
            const uint32_t incl = warp_inclusive_scan(tot);
            const uint32_t before = incl - tot;
            const bool mine = before < need && incl >= need;
            if (mine) {
                uint32_t run = before, d = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (run + c[j] >= need) {
                        d = j;
                        break;
                    }
                    run += c[j];
                }
                ctl[4] = lane * 8 + d;
                ctl[5] = run;
            }
        }
        __syncthreads();
        prefix |= uint64_t(ctl[4]) << sh;
        need -= ctl[5];
        __syncthreads();
    }
    // prefix is now the k-th smallest key: keep keys <= prefix (exactly k)
    uint64_t mine[16];
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t i = tid + j * blockDim.x;
        mine[j] = i < n ? keys[i] : ~0ull;
        cnt += (i < n && mine[j] <= prefix) ? 1u : 0u;
    }
    if (tid == 0) ctl[6] = 0;
    __syncthreads();
    uint32_t pos = cnt ? atomicAdd(&ctl[6], cnt) : 0u;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t i = tid + j * blockDim.x;
        if (i < n && mine[j] <= prefix) keys[pos++] = mine[j];
    }
    uint32_t N = 1;
    while (N < k) N <<= 1;
    __syncthreads();
    for (uint32_t i = k + tid; i < N; i += blockDim.x) keys[i] = ~0ull;
    __syncthreads();
    bitonic_sort_smem(keys, N);
}

}  // namespace genie
