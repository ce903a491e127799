// Field evaluation on device: hash-grid INR (encoding.py:91-134 + mlp.py:39-53
// + model.py:65-89), trilinear lattice (fields.py:165-221) and the analytic
// volumes (fields.py:131-158).  Values come back as float with the reference's
// [0,1] clip; non-finite INR outputs raise a flag (ModelCorruptError path).
#pragma once
#include "common.cuh"

namespace cinr {

// Weights staged in shared memory once per CTA (the whole default MLP is 6.5 KB).
struct MlpSmem {
    float* w;  // packed like VcbField.weights
    float* b;
};

__device__ __forceinline__ int mlp_param_count(const VcbField& F, int& nb) {
    int nw = 0;
    nb = 0;
    for (int L = 0; L < F.n_layers; L++) {
        nw += F.widths[L] * F.widths[L + 1];
        nb += F.widths[L + 1];
    }
    return nw;
}

__device__ __forceinline__ void stage_mlp(const VcbField& F, float* smem, MlpSmem& m) {
    int nb;
    int nw = mlp_param_count(F, nb);
    for (int i = threadIdx.x; i < nw; i += blockDim.x) smem[i] = __ldg(F.weights + i);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) smem[nw + i] = __ldg(F.biases + i);
    m.w = smem;
    m.b = smem + nw;
}

// encoding.py:91-116 + 119-134 for one level; accumulates F features into acc.
template <int NF>
__device__ __forceinline__ void encode_level(const VcbField& F, int l, double x, double y, double z, float* acc) {
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
    const float* tab = F.tables + F.tab_off[l] * NF;
    float s[NF];
#pragma unroll
    for (int f = 0; f < NF; f++) s[f] = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
        const uint32_t vx = c0[0] + dx, vy = c0[1] + dy, vz = c0[2] + dz;
        // dense: x + s*y + s^2*z; hashed: (x*p0 ^ y*p1 ^ z*p2) & (T-1) — only the
        // low 32 bits of the uint64 products matter under the power-of-two mask
        uint32_t idx = F.dense[l] ? vx + side * vy + side * side * vz
                                  : ((vx * 2654435761u) ^ (vy * 2246822519u) ^ (vz * 3266489917u)) & mask;
        const float w = (float)(wx[dx] * wy[dy] * wz[dz]);
        const float* row = tab + (size_t)idx * NF;
        if (NF == 2) {
            float2 v = __ldg(reinterpret_cast<const float2*>(row));
            s[0] += w * v.x;
            s[1] += w * v.y;
        } else {
#pragma unroll
            for (int f = 0; f < NF; f++) s[f] += w * __ldg(row + f);
        }
    }
#pragma unroll
    for (int f = 0; f < NF; f++) acc[f] = s[f];
}

// Default network (8 levels x 2 features -> 32 -> 32 -> 1): fully unrolled, registers.
// The reference multiplies with OpenBLAS sgemm (fused multiply-adds, tolerance-only
// parity, P14), so the products are explicit FMAs (immune to -fmad=false in the
// march translation units) and weights come from shared memory four at a time.
template <int IN, int H>
__device__ __forceinline__ float mlp_2h(const float* feat, const MlpSmem& m, int out_sigmoid) {
    const float4* w0 = reinterpret_cast<const float4*>(m.w);
    const float4* w1 = reinterpret_cast<const float4*>(m.w + IN * H);
    const float* w2 = m.w + IN * H + H * H;
    const float* b0 = m.b;
    const float* b1 = b0 + H;
    const float* b2 = b1 + H;
    float h0[H];
#pragma unroll
    for (int o = 0; o < H; o++) {
        float a = 0.0f;
#pragma unroll
        for (int k = 0; k < IN / 4; k++) {
            const float4 wv = w0[o * (IN / 4) + k];
            a = __fmaf_rn(feat[4 * k], wv.x, a);
            a = __fmaf_rn(feat[4 * k + 1], wv.y, a);
            a = __fmaf_rn(feat[4 * k + 2], wv.z, a);
            a = __fmaf_rn(feat[4 * k + 3], wv.w, a);
        }
        a = __fadd_rn(a, b0[o]);
        h0[o] = a > 0.0f ? a : 0.0f;
    }
    float h1[H];
#pragma unroll
    for (int o = 0; o < H; o++) {
        float a = 0.0f;
#pragma unroll
        for (int k = 0; k < H / 4; k++) {
            const float4 wv = w1[o * (H / 4) + k];
            a = __fmaf_rn(h0[4 * k], wv.x, a);
            a = __fmaf_rn(h0[4 * k + 1], wv.y, a);
            a = __fmaf_rn(h0[4 * k + 2], wv.z, a);
            a = __fmaf_rn(h0[4 * k + 3], wv.w, a);
        }
        a = __fadd_rn(a, b1[o]);
        h1[o] = a > 0.0f ? a : 0.0f;
    }
    float zo = 0.0f;
#pragma unroll
    for (int k = 0; k < H; k++) zo = __fmaf_rn(h1[k], w2[k], zo);
    zo = __fadd_rn(zo, b2[0]);
    if (out_sigmoid) return 1.0f / (1.0f + expf(-zo));
    return zo < 0.0f ? 0.0f : (zo > 1.0f ? 1.0f : zo);
}

// Any HashGridConfig/MLPConfig within the ABI limits (local-memory arrays).
static __device__ __noinline__ float inr_generic(const VcbField& F, double x, double y, double z, const MlpSmem& m) {
    float a[128], zv[128];  // widths up to 128 (device.py checks)
    int k = 0;
    for (int l = 0; l < F.levels; l++) {
        const int nf = F.feats;
        const int r = F.res[l];
        const double rd = (double)r;
        double u[3] = {x * rd, y * rd, z * rd};
        uint32_t c0[3];
        double fr[3];
        for (int q = 0; q < 3; q++) {
            long long ci = (long long)floor(u[q]);
            ci = ci < 0 ? 0 : (ci > r - 1 ? r - 1 : ci);
            c0[q] = (uint32_t)ci;
            fr[q] = u[q] - (double)ci;
        }
        const double wx[2] = {1.0 - fr[0], fr[0]}, wy[2] = {1.0 - fr[1], fr[1]}, wz[2] = {1.0 - fr[2], fr[2]};
        const uint32_t side = (uint32_t)(r + 1);
        const uint32_t mask = (uint32_t)(F.table_size - 1);
        for (int f = 0; f < nf; f++) a[k + f] = 0.0f;
        for (int c = 0; c < 8; c++) {
            const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
            const uint32_t vx = c0[0] + dx, vy = c0[1] + dy, vz = c0[2] + dz;
            uint32_t idx = F.dense[l] ? vx + side * vy + side * side * vz
                                      : ((vx * 2654435761u) ^ (vy * 2246822519u) ^ (vz * 3266489917u)) & mask;
            const float w = (float)(wx[dx] * wy[dy] * wz[dz]);
            const float* row = F.tables + (F.tab_off[l] + (long long)idx) * nf;
            for (int f = 0; f < nf; f++) a[k + f] += w * __ldg(row + f);
        }
        k += nf;
    }
    const float* w = m.w;
    const float* b = m.b;
    for (int L = 0; L < F.n_layers; L++) {
        const int din = F.widths[L], dout = F.widths[L + 1];
        for (int o = 0; o < dout; o++) {
            float s = 0.0f;
            for (int q = 0; q < din; q++) s += a[q] * w[o * din + q];
            zv[o] = s + b[o];
        }
        w += din * dout;
        b += dout;
        if (L + 1 < F.n_layers)
            for (int o = 0; o < dout; o++) a[o] = zv[o] > 0.0f ? zv[o] : 0.0f;
    }
    const float zo = zv[0];
    if (F.out_sigmoid) return 1.0f / (1.0f + expf(-zo));
    return zo < 0.0f ? 0.0f : (zo > 1.0f ? 1.0f : zo);
}

__host__ __device__ __forceinline__ bool inr_is_default(const VcbField& F) {
    return F.levels == 8 && F.feats == 2 && F.n_layers == 3 && F.widths[0] == 16 && F.widths[1] == 32 &&
           F.widths[2] == 32 && F.widths[3] == 1;
}

// kFast: the default 8x2 -> 32 -> 32 -> 1 network, fully in registers; the
// generic path uses local arrays (a per-thread stack), so it is only compiled
// into the kernel variants that need it.
template <bool kFast>
__device__ __forceinline__ float inr_eval(const VcbField& F, double x, double y, double z, const MlpSmem& m) {
    if constexpr (kFast) {
        float feat[16];
#pragma unroll
        for (int l = 0; l < 8; l++) encode_level<2>(F, l, x, y, z, feat + 2 * l);
        return mlp_2h<16, 32>(feat, m, F.out_sigmoid);
    } else {
        return inr_generic(F, x, y, z, m);
    }
}

// fields.py:165-199 trilinear_lattice via RawLatticeField._evaluate (u = pos*dims - 0.5)
__device__ __forceinline__ float lattice_eval(const VcbField& F, double x, double y, double z) {
    const long long vx = F.lx, vy = F.ly, vz = F.lz;
    double ux = clampd(DSUB(DMUL(x, (double)vx), 0.5), 0.0, (double)(vx - 1));
    double uy = clampd(DSUB(DMUL(y, (double)vy), 0.5), 0.0, (double)(vy - 1));
    double uz = clampd(DSUB(DMUL(z, (double)vz), 0.5), 0.0, (double)(vz - 1));
    long long x0 = (long long)floor(ux), y0 = (long long)floor(uy), z0 = (long long)floor(uz);
    long long x1 = x0 + 1 < vx - 1 ? x0 + 1 : vx - 1;
    long long y1 = y0 + 1 < vy - 1 ? y0 + 1 : vy - 1;
    long long z1 = z0 + 1 < vz - 1 ? z0 + 1 : vz - 1;
    double fx = DSUB(ux, (double)x0), fy = DSUB(uy, (double)y0), fz = DSUB(uz, (double)z0);
    const float* L = F.lattice;
#define LAT(zz, yy, xx) __ldg(L + ((zz) * vy + (yy)) * vx + (xx))
    float c000 = LAT(z0, y0, x0), c100 = LAT(z0, y0, x1), c010 = LAT(z0, y1, x0), c110 = LAT(z0, y1, x1);
    float c001 = LAT(z1, y0, x0), c101 = LAT(z1, y0, x1), c011 = LAT(z1, y1, x0), c111 = LAT(z1, y1, x1);
#undef LAT
    double c00 = DADD((double)c000, DMUL((double)FSUB(c100, c000), fx));
    double c10 = DADD((double)c010, DMUL((double)FSUB(c110, c010), fx));
    double c01 = DADD((double)c001, DMUL((double)FSUB(c101, c001), fx));
    double c11 = DADD((double)c011, DMUL((double)FSUB(c111, c011), fx));
    double c0 = DADD(c00, DMUL(DSUB(c10, c00), fy));
    double c1 = DADD(c01, DMUL(DSUB(c11, c01), fy));
    return __double2float_rn(DADD(c0, DMUL(DSUB(c1, c0), fz)));
}

// fields.py:131-148 (+ ProceduralField clip, 126-128)
__device__ __forceinline__ float procedural_eval(int kind, double x, double y, double z) {
    double v;
    if (kind == 0 || kind == 1) {
        double a = DSUB(x, 0.5), b = DSUB(y, 0.5), c = DSUB(z, 0.5);
        double d = __dsqrt_rn(DADD(DADD(DMUL(a, a), DMUL(b, b)), DMUL(c, c)));
        if (kind == 0) v = DSUB(1.0, d);
        else v = DSUB(0.5, DMUL(0.5, cos(__ddiv_rn(DMUL(DMUL(2.0, 3.141592653589793), d), 0.125))));
    } else {
        double qx = DSUB(DMUL(2.0, x), 1.0), qy = DSUB(DMUL(2.0, y), 1.0), qz = DSUB(DMUL(2.0, z), 1.0);
        double r = __dsqrt_rn(DADD(DMUL(qx, qx), DMUL(qy, qy)));
        const double fm = 6.0, al = 0.25, pi = 3.141592653589793;
        double rho = cos(DMUL(DMUL(DMUL(2.0, pi), fm), cos(__ddiv_rn(DMUL(pi, r), 2.0))));
        v = __ddiv_rn(DADD(DSUB(1.0, sin(__ddiv_rn(DMUL(pi, qz), 2.0))), DMUL(al, DADD(1.0, rho))),
                      DMUL(2.0, DADD(1.0, al)));
    }
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return __double2float_rn(v);
}

// kInr: 0 = field is not an INR (no MLP code compiled in), 1 = default INR
// (register-resident fast path), 2 = any other INR shape (generic path).
template <int kInr>
__device__ __forceinline__ float field_eval(const VcbField& F, double x, double y, double z, const MlpSmem& m,
                                            int* nonfinite) {
    if constexpr (kInr != 0) {
        float v = inr_eval<kInr == 1>(F, x, y, z, m);
        if (!isfinite(v)) {
            if (nonfinite) *nonfinite = 1;
        }
        if (F.clip01) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
        return v;
    } else {
        if (F.kind == 1) return lattice_eval(F, x, y, z);
        return procedural_eval(F.proc, x, y, z);
    }
}

__host__ __device__ __forceinline__ int inr_mode(const VcbField& F) {
    return F.kind != 0 ? 0 : (inr_is_default(F) ? 1 : 2);
}

// launch helper: KERNEL is a template name taking <int kInr>
#define CINR_DISPATCH_INR(F, KERNEL, GRID, BLOCK, SMEM, STREAM, ...)                                   \
    do {                                                                                               \
        switch (inr_mode(F)) {                                                                         \
            case 1: KERNEL<1><<<(GRID), (BLOCK), (SMEM), (STREAM)>>>(__VA_ARGS__); break;              \
            case 2:                                                                                    \
                if ((SMEM) > 48 * 1024)                                                                \
                    cudaFuncSetAttribute(KERNEL<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (SMEM)); \
                KERNEL<2><<<(GRID), (BLOCK), (SMEM), (STREAM)>>>(__VA_ARGS__);                          \
                break;                                                                                 \
            default: KERNEL<0><<<(GRID), (BLOCK), (SMEM), (STREAM)>>>(__VA_ARGS__); break;             \
        }                                                                                              \
    } while (0)

}  // namespace cinr
