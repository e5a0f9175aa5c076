// Shared device/host helpers for libgenie_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "genie/genie.h"

namespace genie {

// ---------------------------------------------------------------- errors

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GENIE_CUDA(call)                                                                 \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::genie::Error(GENIE_ERR_CUDA, std::string(#call) + ": " +             \
                                                     cudaGetErrorString(e_));            \
    } while (0)

inline int set_err(char* err, size_t errlen, int code, const std::string& msg) {
    if (err && errlen) {
        std::strncpy(err, msg.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return code;
}

template <typename Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
    try {
        return fn();
    } catch (const Error& e) {
        return set_err(err, errlen, e.code, e.what());
    } catch (const std::bad_alloc&) {
        return set_err(err, errlen, GENIE_ERR_CUDA, "host allocation failed");
    } catch (const std::exception& e) {
        return set_err(err, errlen, GENIE_ERR_INVARIANT, e.what());
    }
}

// RAII device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // grows (never shrinks); contents are not preserved
    void reserve(size_t count) {
        if (count <= n && p) return;
        release();
        size_t bytes = (count ? count : 1) * sizeof(T);
        GENIE_CUDA(cudaMalloc(&p, bytes));
        n = count;
    }
};

// ---------------------------------------------------------------- device

// splitmix64 finalizer (rng.hpp:25-30)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

#ifndef GENIE_LDG_MODE
#define GENIE_LDG_MODE 0
#endif
__device__ __forceinline__ uint4 ldg_stream_v4(const uint32_t* p) {
#if GENIE_LDG_MODE == 1
    return __ldg(reinterpret_cast<const uint4*>(p));
#elif GENIE_LDG_MODE == 2
    return __ldcg(reinterpret_cast<const uint4*>(p));
#else
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
#endif
}

template <typename T>
__device__ __forceinline__ uint64_t lower_bound_dev(const T* a, uint64_t n, T key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t m = (lo + hi) >> 1;
        if (a[m] < key) lo = m + 1;
        else hi = m;
    }
    return lo;
}

template <typename T>
__device__ __forceinline__ uint64_t upper_bound_dev(const T* a, uint64_t n, T key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t m = (lo + hi) >> 1;
        if (a[m] <= key) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// cpq.hpp:63-68
__host__ __device__ __forceinline__ uint32_t width_for(uint64_t max_count) {
    if (max_count <= 15u) return 4;
    if (max_count <= 255u) return 8;
    if (max_count <= 65535u) return 16;
    return 32;
}

__host__ __device__ __forceinline__ uint64_t bit_ceil64(uint64_t v) {
    uint64_t c = 1;
    while (c < v) c <<= 1;
    return c;
}

// Result order key: ascending key == (count desc, id asc) (cpq.hpp:37-40).
__host__ __device__ __forceinline__ uint64_t order_key(uint32_t id, uint32_t count) {
    return (static_cast<uint64_t>(0xffffffffu - count) << 32) | id;
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t key) { return static_cast<uint32_t>(key); }
__host__ __device__ __forceinline__ uint32_t key_count(uint64_t key) {
    return 0xffffffffu - static_cast<uint32_t>(key >> 32);
}

int sm_count(int device);

}  // namespace genie
