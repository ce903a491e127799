// Error channel, launch helpers and warp/block primitives shared by the .cu files.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cinr {

int set_error(const char* fmt, ...);
int check_launch(const char* what);
int device_sms();
int kernel_ctas_per_sm(const void* fn, int threads, int smem);

inline int grid_for(int64_t n, int block, int cap_per_sm = 16) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)device_sms() * cap_per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-brick miss counters: lanes reporting the same brick add once (match.any + popc).
__device__ __forceinline__ void warp_aggregated_add(int32_t* counters, long long key) {
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, key);
    const int leader = __ffs(peers) - 1;
    if ((int)(threadIdx.x & 31) == leader) atomicAdd(counters + key, __popc(peers));
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace cinr
