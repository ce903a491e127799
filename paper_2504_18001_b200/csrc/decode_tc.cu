// Tensor-core INR decoder (sm_100a tcgen05): hash-grid encode on CUDA cores,
// the 16->32->32 MLP layers as tcgen05.mma (kind::f16, M=128 rows per CTA,
// fp32 accumulators in TMEM), output layer + sigmoid in the epilogue.
//
// Reference: inr/encoding.py:119-134 (encode), inr/mlp.py:39-53 (forward),
// inr/model.py:88-89 (InrField clip).  The reference MLP runs in f32 (OpenBLAS
// sgemm); to keep f32-level accuracy on 16-bit tensor inputs every operand is
// split x = hi + lo (both fp16) and each product is hi*hi + hi*lo + lo*hi
// (three MMAs into one accumulator; the lo*lo term is below f32 rounding).
//
// Shared-memory operands use the canonical no-swizzle K-major layout: 8x8
// fp16 "core matrices" (8 rows x 16 bytes), core (row-group g, k-chunk c) at
// byte g*SBO + c*LBO.  One elected thread issues the MMAs; completion is
// signalled through tcgen05.commit -> mbarrier; warps read their 32 TMEM
// lanes (= tile rows) with tcgen05.ld.32x32b.x32.
#include <cuda_fp16.h>

#include <cstdint>

#include "common.cuh"
#include "fields.cuh"
#include "util.cuh"

namespace cinr {

constexpr int kTcRows = 128;  // UMMA M

// byte offset of element (row, k) in a K-major no-swizzle operand tile
__device__ __forceinline__ uint32_t core_off(int row, int k, uint32_t lbo, uint32_t sbo) {
    return (uint32_t)(row >> 3) * sbo + (uint32_t)(k >> 3) * lbo + (uint32_t)(row & 7) * 16u + (uint32_t)(k & 7) * 2u;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (sm100)
    // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
    return d;
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (0u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, int accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void split_store(unsigned char* base, uint32_t off_hi_lo_delta, uint32_t off, float x) {
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *reinterpret_cast<__half*>(base + off) = h;
    *reinterpret_cast<__half*>(base + off + off_hi_lo_delta) = l;
}

constexpr uint32_t kA0Lbo = 128, kA0Sbo = 256, kA1Lbo = 128, kA1Sbo = 512;
constexpr uint32_t kW0Lbo = 128, kW0Sbo = 256, kW1Lbo = 128, kW1Sbo = 512;

// Position source: points (f64 xyz) or brick samples (flat keys + geometry).
struct TcPointsSrc {
    const double* pos;
    __device__ void get(long long i, double& x, double& y, double& z) const {
        x = pos[3 * i];
        y = pos[3 * i + 1];
        z = pos[3 * i + 2];
    }
};

struct TcBricksSrc {
    VcbBrickGeom G;
    const int64_t* keys;
    __device__ void get(long long t, double& x, double& y, double& z) const {
        const long long b = G.b, b3 = b * b * b;
        const long long ki = t / b3, s = t - ki * b3;
        const long long flat = keys[ki];
        int lod = 0;
        while (lod + 1 < G.n_lod && flat >= G.offset[lod + 1]) lod++;
        const long long lin = flat - G.offset[lod];
        const long long gx = G.grid[lod][0], gy = G.grid[lod][1];
        const long long ix = lin % gx, iy = (lin / gx) % gy, iz = lin / (gx * gy);
        const long long sx = s % b, sy = (s / b) % b, sz = s / (b * b);
        long long nx = (ix > 0 ? ix * (b << lod) - 1 : 0) + (sx << lod);
        long long ny = (iy > 0 ? iy * (b << lod) - 1 : 0) + (sy << lod);
        long long nz = (iz > 0 ? iz * (b << lod) - 1 : 0) + (sz << lod);
        nx = nx < G.dims[0] - 1 ? nx : G.dims[0] - 1;
        ny = ny < G.dims[1] - 1 ? ny : G.dims[1] - 1;
        nz = nz < G.dims[2] - 1 ? nz : G.dims[2] - 1;
        x = ((double)nx + 0.5) / (double)G.dims[0];
        y = ((double)ny + 0.5) / (double)G.dims[1];
        z = ((double)nz + 0.5) / (double)G.dims[2];
    }
};

// ---------------------------------------------------------------------------
// v2: one persistent CTA per SM, eight independent 128-row warpgroup pipelines
// (own operand tiles, TMEM columns, mbarrier and named barrier), sharing one
// shared-memory copy of the weights and of the dense (coarse) hash-grid levels.
// Random-position decode is bound by the table gathers; levels staged in shared
// memory replace scattered L1 gathers by bank accesses.  Measured on B200 (2^24
// random points): 8 groups + levels 0-2 in shared memory 6.8e9 samples/s; 8 groups,
// no staged levels 6.5e9; 6 groups + levels 0-4 4.8e9 (the big tables crowd L1);
// (a first version with six independent 128-thread CTAs per SM reached 5.9e9).
#ifndef TC2_GROUPS
#define TC2_GROUPS 8
#endif
#ifndef TC2_BUDGET_KB
#define TC2_BUDGET_KB 24
#endif
constexpr int kTc2Groups = TC2_GROUPS;
constexpr int kTc2Threads = kTc2Groups * kTcRows;
constexpr int kTc2TableBudget = TC2_BUDGET_KB * 1024;  // bytes of dense levels kept in shared memory

struct Tc2Group {
    // A1 (layer-1 input) reuses A0's bytes: A0 is dead once the layer-0 MMAs completed
    union {
        alignas(128) unsigned char a0[2][kTcRows * 16 * 2];
        alignas(128) unsigned char a1[2][kTcRows * 32 * 2];
    };
    alignas(8) uint64_t mbar;
};

struct Tc2Smem {
    alignas(128) unsigned char w0[2][32 * 16 * 2];
    alignas(128) unsigned char w1[2][32 * 32 * 2];
    float b0[32], b1[32], w2[32], b2;
    uint32_t tmem;
    Tc2Group g[kTc2Groups];
};

// encoding.py:91-134 for one level of the default 2-feature grid, table row pointer given
__device__ __forceinline__ void encode_level2(const VcbField& F, int l, const float2* tab, double x, double y,
                                              double z, float* acc) {
    const int r = F.res[l];
    const double rd = (double)r;
    double u[3] = {x * rd, y * rd, z * rd};
    uint32_t c0[3];
    double fr[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        long long ci = (long long)floor(u[a]);
        ci = ci < 0 ? 0 : (ci > r - 1 ? r - 1 : ci);
        c0[a] = (uint32_t)ci;
        fr[a] = u[a] - (double)ci;
    }
    const double wx[2] = {1.0 - fr[0], fr[0]}, wy[2] = {1.0 - fr[1], fr[1]}, wz[2] = {1.0 - fr[2], fr[2]};
    const uint32_t side = (uint32_t)(r + 1);
    const uint32_t mask = (uint32_t)(F.table_size - 1);
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
        const uint32_t vx = c0[0] + dx, vy = c0[1] + dy, vz = c0[2] + dz;
        const uint32_t idx = F.dense[l] ? vx + side * vy + side * side * vz
                                        : ((vx * 2654435761u) ^ (vy * 2246822519u) ^ (vz * 3266489917u)) & mask;
        const float w = (float)(wx[dx] * wy[dy] * wz[dz]);
        const float2 v = tab[idx];
        s0 += w * v.x;
        s1 += w * v.y;
    }
    acc[0] = s0;
    acc[1] = s1;
}

template <class Src>
__global__ void __launch_bounds__(kTc2Threads, 1) k_inr_decode_tc2(const __grid_constant__ VcbField F, Src src,
                                                                   long long n, float* out, int32_t* nonfinite,
                                                                   int n_smem_levels, const int64_t* n_keys_dev,
                                                                   long long per_key) {
    // device-side item count (maintenance dispatches without a host round trip)
    if (n_keys_dev != nullptr) n = *n_keys_dev * per_key;
    if (n <= 0) return;
    extern __shared__ __align__(128) unsigned char dsm2[];
    Tc2Smem& sm = *reinterpret_cast<Tc2Smem*>(dsm2);
    float2* s_tab = reinterpret_cast<float2*>(dsm2 + ((sizeof(Tc2Smem) + 127) & ~size_t(127)));
    const int tid = threadIdx.x, warp = tid >> 5;
    const int grp = tid / kTcRows, row = tid % kTcRows;
    // ---- weights (hi/lo split, K-major core layout), biases, dense levels
    const float* W0 = F.weights;
    const float* W1 = F.weights + 32 * 16;
    const float* W2 = W1 + 32 * 32;
    for (int e = tid; e < 32 * 16; e += kTc2Threads)
        split_store(&sm.w0[0][0], sizeof(sm.w0[0]), core_off(e / 16, e % 16, kW0Lbo, kW0Sbo), __ldg(W0 + e));
    for (int e = tid; e < 32 * 32; e += kTc2Threads)
        split_store(&sm.w1[0][0], sizeof(sm.w1[0]), core_off(e / 32, e % 32, kW1Lbo, kW1Sbo), __ldg(W1 + e));
    if (tid < 32) {
        sm.b0[tid] = __ldg(F.biases + tid);
        sm.b1[tid] = __ldg(F.biases + 32 + tid);
        sm.w2[tid] = __ldg(W2 + tid);
    }
    const long long tab_rows = n_smem_levels > 0 ? F.tab_off[n_smem_levels] : 0;  // levels are contiguous
    const float2* gtab = reinterpret_cast<const float2*>(F.tables);
    // the dense levels are a plain copy: one TMA bulk copy (whole 16-byte rows; the smem
    // region is rounded up to match)
    __shared__ __align__(8) uint64_t tma_bar;
    if (tid == 0) {
        const uint32_t bytes = ((uint32_t)tab_rows * 8u + 15u) & ~15u;
        tma_stage_begin(&tma_bar, bytes);
        if (bytes) tma_stage_copy(s_tab, gtab, bytes, &tma_bar);
        sm.b2 = __ldg(F.biases + 64);
    }
    if (row == 0) {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(&sm.g[grp].mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.tmem);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tma_stage_wait(&tma_bar);
    Tc2Group& G = sm.g[grp];
    const uint32_t tmem = sm.tmem + (uint32_t)(grp * 64);  // 64 columns per group: D0 | D1
    const uint32_t sa0 = (uint32_t)__cvta_generic_to_shared(&G.a0[0][0]);
    const uint32_t sa1 = (uint32_t)__cvta_generic_to_shared(&G.a1[0][0]);
    const uint32_t sw0 = (uint32_t)__cvta_generic_to_shared(&sm.w0[0][0]);
    const uint32_t sw1 = (uint32_t)__cvta_generic_to_shared(&sm.w1[0][0]);
    const uint32_t da0 = sizeof(G.a0[0]), da1 = sizeof(G.a1[0]), dw0 = sizeof(sm.w0[0]), dw1 = sizeof(sm.w1[0]);
    constexpr uint32_t ID = idesc_f16(kTcRows, 32);
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;  // a warp reads its TMEM lane quarter
    const int bar_id = 1 + grp;
    auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kTcRows) : "memory"); };
    uint32_t phase = 0;
    const long long stride = (long long)gridDim.x * kTc2Groups * kTcRows;
    for (long long t0 = ((long long)blockIdx.x * kTc2Groups + grp) * kTcRows; t0 < n; t0 += stride) {
        const long long i = t0 + row;
        float feat[16];
        if (i < n) {
            double x, y, z;
            src.get(i, x, y, z);
#pragma unroll
            for (int l = 0; l < 8; l++) {
                const float2* tab = l < n_smem_levels ? s_tab + F.tab_off[l] : gtab + F.tab_off[l];
                encode_level2(F, l, tab, x, y, z, feat + 2 * l);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; k++) feat[k] = 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 16; k++) split_store(&G.a0[0][0], da0, core_off(row, k, kA0Lbo, kA0Sbo), feat[k]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        group_sync();
        if (row == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            mma_f16(tmem, umma_desc(sa0, kA0Lbo, kA0Sbo), umma_desc(sw0, kW0Lbo, kW0Sbo), ID, 0);
            mma_f16(tmem, umma_desc(sa0, kA0Lbo, kA0Sbo), umma_desc(sw0 + dw0, kW0Lbo, kW0Sbo), ID, 1);
            mma_f16(tmem, umma_desc(sa0 + da0, kA0Lbo, kA0Sbo), umma_desc(sw0, kW0Lbo, kW0Sbo), ID, 1);
            mma_commit(&G.mbar);
        }
        mbar_wait(&G.mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float h[32];
        tmem_ld32(tmem + lane_base, h);
#pragma unroll
        for (int c = 0; c < 32; c++) {
            const float a = h[c] + sm.b0[c];
            split_store(&G.a1[0][0], da1, core_off(row, c, kA1Lbo, kA1Sbo), a > 0.0f ? a : 0.0f);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        group_sync();
        if (row == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d1 = tmem + 32;
#pragma unroll
            for (int s2 = 0; s2 < 2; s2++) {
                const uint32_t ko = (uint32_t)s2 * 2u * kA1Lbo, kw = (uint32_t)s2 * 2u * kW1Lbo;
                mma_f16(d1, umma_desc(sa1 + ko, kA1Lbo, kA1Sbo), umma_desc(sw1 + kw, kW1Lbo, kW1Sbo), ID, s2);
                mma_f16(d1, umma_desc(sa1 + ko, kA1Lbo, kA1Sbo), umma_desc(sw1 + dw1 + kw, kW1Lbo, kW1Sbo), ID, 1);
                mma_f16(d1, umma_desc(sa1 + da1 + ko, kA1Lbo, kA1Sbo), umma_desc(sw1 + kw, kW1Lbo, kW1Sbo), ID, 1);
            }
            mma_commit(&G.mbar);
        }
        mbar_wait(&G.mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmem_ld32(tmem + lane_base + 32, h);
        float zo = 0.0f;
#pragma unroll
        for (int c = 0; c < 32; c++) {
            const float a = h[c] + sm.b1[c];
            zo += (a > 0.0f ? a : 0.0f) * sm.w2[c];
        }
        zo += sm.b2;
        float v = F.out_sigmoid ? 1.0f / (1.0f + expf(-zo)) : (zo < 0.0f ? 0.0f : (zo > 1.0f ? 1.0f : zo));
        if (i < n) {
            if (!isfinite(v)) *nonfinite = 1;
            if (F.clip01) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
            out[i] = v;
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        group_sync();  // operand tiles and TMEM columns are reused by the next tile
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sm.tmem));
}

// dense levels (coarsest first) whose tables fit the shared-memory budget
static int tc2_smem_levels(const VcbField& F) {
    int L = 0;
    while (L < F.levels && F.dense[L] && F.tab_off[L + 1] * 8 <= kTc2TableBudget) L++;
    return L;
}

template <class Src>
static int launch_tc2(const VcbField& F, const Src& src, long long n, float* out, int32_t* nonfinite,
                      cudaStream_t st, const int64_t* n_keys_dev = nullptr, long long per_key = 0) {
    const int L = tc2_smem_levels(F);
    const size_t smem = ((sizeof(Tc2Smem) + 127) & ~size_t(127)) + (((size_t)(L > 0 ? F.tab_off[L] : 0) * 8 + 15) & ~size_t(15));
    kernel_ctas_per_sm((const void*)k_inr_decode_tc2<Src>, kTc2Threads, (int)smem);  // raises the smem limit once
    const long long tiles = (n + kTcRows - 1) / kTcRows;
    long long grid = (tiles + kTc2Groups - 1) / kTc2Groups;
    if (grid > device_sms()) grid = device_sms();
    if (grid < 1) grid = 1;
    k_inr_decode_tc2<Src><<<(int)grid, kTc2Threads, smem, st>>>(F, src, n, out, nonfinite, L, n_keys_dev, per_key);
    return 0;
}

// Brick decode for maintenance: up to max_keys keys, count read on the device.
int inr_bricks_tc_dev(const VcbField& F, const VcbBrickGeom& G, const int64_t* keys, const int64_t* n_keys_dev,
                      int max_keys, float* out, int32_t* nonfinite, cudaStream_t st) {
    const long long b3 = G.b * G.b * G.b;
    launch_tc2(F, TcBricksSrc{G, keys}, (long long)max_keys * b3, out, nonfinite, st, n_keys_dev, b3);
    return 0;
}

}  // namespace cinr

using namespace cinr;


extern "C" int32_t vcb_inr_points_tc(const VcbField* f, int64_t n, const double* pos, float* out, int32_t* nonfinite,
                                     void* stream) {
    if (n <= 0) return 0;
    if (f->kind != 0 || !inr_is_default(*f)) return set_error("inr_points_tc: only the default 8x2/16-32-32-1 INR");
    launch_tc2(*f, TcPointsSrc{pos}, n, out, nonfinite, (cudaStream_t)stream);
    return check_launch("inr_points_tc");
}

extern "C" int32_t vcb_inr_bricks_tc(const VcbField* f, const VcbBrickGeom* g, int64_t n_keys, const int64_t* keys,
                                     float* out, int32_t* nonfinite, void* stream) {
    if (n_keys <= 0) return 0;
    if (f->kind != 0 || !inr_is_default(*f)) return set_error("inr_bricks_tc: only the default 8x2/16-32-32-1 INR");
    const long long n = n_keys * g->b * g->b * g->b;
    launch_tc2(*f, TcBricksSrc{*g, keys}, n, out, nonfinite, (cudaStream_t)stream);
    return check_launch("inr_bricks_tc");
}
