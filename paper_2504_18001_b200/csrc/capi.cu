// C-ABI plumbing: thread-local error channel, device properties.
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/cinr_b200.h"
#include "util.cuh"

namespace cinr {

static thread_local char g_err[512] = {0};

int set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return -1;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error("%s: %s", what, cudaGetErrorString(e));
    return 0;
}

int device_sms() {
    static thread_local int dev = -1, sms = 0;
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        if (sms <= 0) sms = 148;
        dev = d;
    }
    return sms;
}

// Resident CTAs per SM of `fn` at (threads, dynamic smem), after making sure its
// dynamic shared-memory limit admits `smem` (the limit only ever grows: lowering it
// for a small launch would break a later larger one).  The driver calls run once per
// (device, kernel, size), not per frame.
int kernel_ctas_per_sm(const void* fn, int threads, int smem) {
    struct Limit {
        const void* fn;
        int dev, smem_max;
    };
    struct Occ {
        const void* fn;
        int dev, threads, smem, per_sm;
    };
    static thread_local Limit lim[32];
    static thread_local Occ occ[64];
    static thread_local int nl = 0, no = 0;
    int d = 0;
    cudaGetDevice(&d);
    int li = -1;
    for (int i = 0; i < nl; i++)
        if (lim[i].fn == fn && lim[i].dev == d) li = i;
    if (li < 0) {
        li = nl < 32 ? nl++ : 0;
        lim[li] = Limit{fn, d, 0};
    }
    if (smem > lim[li].smem_max) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        lim[li].smem_max = smem;
    }
    for (int i = 0; i < no; i++)
        if (occ[i].fn == fn && occ[i].dev == d && occ[i].threads == threads && occ[i].smem == smem)
            return occ[i].per_sm;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    occ[no < 64 ? no++ : 0] = Occ{fn, d, threads, smem, per_sm};
    return per_sm;
}

}  // namespace cinr

extern "C" const char* vcb_last_error(void) { return cinr::g_err; }
extern "C" int32_t vcb_abi_version(void) { return 1; }
extern "C" int32_t vcb_device_sm_count(void) { return cinr::device_sms(); }

// Host-only: sizeof of every ABI struct, so bindings can verify their layouts
// without a GPU.
extern "C" int32_t vcb_struct_sizes(int64_t* out, int32_t n) {
    const int64_t s[] = {(int64_t)sizeof(VcbCamera),     (int64_t)sizeof(VcbMarchStatic), (int64_t)sizeof(VcbProbeStatic),
                         (int64_t)sizeof(VcbField),      (int64_t)sizeof(VcbBrickGeom),   (int64_t)sizeof(VcbFrameStats),
                         (int64_t)sizeof(VcbCacheState), (int64_t)sizeof(VcbFrameParams), (int64_t)sizeof(VcbMaintParams),
                         (int64_t)sizeof(VcbPtParams), (int64_t)sizeof(VcbTrainParams)};
    const int k = (int)(sizeof(s) / sizeof(s[0]));
    for (int i = 0; i < n && i < k; i++) out[i] = s[i];
    return k;
}
