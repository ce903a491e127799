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

// TMA bulk copies global -> shared (cp.async.bulk, SASS UBLKCP) completing on one
// mbarrier.  Usage: thread 0 calls tma_stage_begin(bar, total bytes), then
// tma_stage_copy for each region (16-byte aligned addresses, sizes multiples of 16);
// after a __syncthreads() every thread calls tma_stage_wait(bar).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_stage_begin(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_stage_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tma_stage_wait(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "TMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra TMA_WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar))
        : "memory");
}
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
