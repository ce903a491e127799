// Warp-cooperative INR inference for the frame kernel's miss phase (the default
// 8x2 hash grid + 16-32-32-1 MLP, encoding.py:91-134, mlp.py:39-53): 32 samples per
// warp, the two hidden layers on the tensor cores with mma.sync m16n8k16 (fp16
// operands split hi + lo, fp32 accumulation: hi*hi + hi*lo + lo*hi, so the
// products keep f32-level accuracy like the tcgen05 decoder).
//
// Lane (g, c) = (lane >> 2, lane & 3) encodes hash-grid levels c and c + 4 of the
// warp's samples g, g + 8, 16 + g, 24 + g: exactly the A-fragment elements it owns
// for the two 16-row tiles, so no feature shuffles are needed.  Layer-0
// accumulators become layer-1 A fragments in place (the m16n8 D layout of two
// adjacent N tiles is the m16n8k16 A layout).
#pragma once
#include <cuda_fp16.h>

#include "fields.cuh"

namespace cinr {

// B fragments of W0 (4 N tiles) and W1 (2 K steps x 4 N tiles) per lane, hi/lo
// packed: {b0_hi, b1_hi, b0_lo, b1_lo}; plus f32 biases and the output row.
struct MlpFrag {
    uint4 w0[4][32];
    uint4 w1[2][4][32];
    float b0[32], b1[32], w2[32], b2;
};

__device__ __forceinline__ uint32_t h2pack(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
    const __half xh = __float2half_rn(x), yh = __float2half_rn(y);
    hi = h2pack(xh, yh);
    lo = h2pack(__float2half_rn(x - __half2float(xh)), __float2half_rn(y - __half2float(yh)));
}

// Stage the fragments (one CTA, all threads); W is packed (out, in) per layer like VcbField.
__device__ __forceinline__ void stage_mlp_frag(const VcbField& F, MlpFrag* s) {
    const float* W0 = F.weights;            // [32][16]
    const float* W1 = F.weights + 32 * 16;  // [32][32]
    const float* W2 = W1 + 32 * 32;
    for (int e = threadIdx.x; e < 4 * 32; e += blockDim.x) {
        const int j = e / 32, l = e % 32, g = l >> 2, c = l & 3, n = 8 * j + g;
        uint4 v;
        split2(__ldg(W0 + n * 16 + 2 * c), __ldg(W0 + n * 16 + 2 * c + 1), v.x, v.z);
        split2(__ldg(W0 + n * 16 + 2 * c + 8), __ldg(W0 + n * 16 + 2 * c + 9), v.y, v.w);
        s->w0[j][l] = v;
    }
    for (int e = threadIdx.x; e < 2 * 4 * 32; e += blockDim.x) {
        const int ks = e / 128, j = (e / 32) % 4, l = e % 32, g = l >> 2, c = l & 3, n = 8 * j + g;
        const int k0 = 16 * ks + 2 * c;
        uint4 v;
        split2(__ldg(W1 + n * 32 + k0), __ldg(W1 + n * 32 + k0 + 1), v.x, v.z);
        split2(__ldg(W1 + n * 32 + k0 + 8), __ldg(W1 + n * 32 + k0 + 9), v.y, v.w);
        s->w1[ks][j][l] = v;
    }
    for (int e = threadIdx.x; e < 32; e += blockDim.x) {
        s->b0[e] = __ldg(F.biases + e);
        s->b1[e] = __ldg(F.biases + 32 + e);
        s->w2[e] = __ldg(W2 + e);
    }
    if (threadIdx.x == 0) s->b2 = __ldg(F.biases + 64);
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A (hi, lo) x B (hi, lo) with the lo*lo term dropped
__device__ __forceinline__ void mma_split(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint4 b) {
    mma16816(d, ah[0], ah[1], ah[2], ah[3], b.x, b.y);
    mma16816(d, ah[0], ah[1], ah[2], ah[3], b.z, b.w);
    mma16816(d, al[0], al[1], al[2], al[3], b.x, b.y);
}

// All 32 lanes call this converged; (x, y, z) is the lane's sample position (any
// value for inactive lanes).  Returns the INR output of the lane's own sample
// (before the InrField clip), the same function as inr_eval<true>.
__device__ __forceinline__ float inr_warp_default(const VcbField& F, const MlpFrag* fr, double x, double y,
                                                  double z) {
    const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
    // levels c and c + 4 of samples g, g + 8, 16 + g, 24 + g
    float f[4][2][2];  // [sample slot][level c / c+4][feature]
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const int src = g + 8 * s;
        const double sx = __shfl_sync(0xffffffffu, x, src), sy = __shfl_sync(0xffffffffu, y, src),
                     sz = __shfl_sync(0xffffffffu, z, src);
        encode_level<2>(F, c, sx, sy, sz, f[s][0]);
        encode_level<2>(F, c + 4, sx, sy, sz, f[s][1]);
    }
    float h0[2][4][4];  // [M tile][N tile][accumulator]
#pragma unroll
    for (int mt = 0; mt < 2; mt++) {
        uint32_t ah[4], al[4];
        split2(f[2 * mt][0][0], f[2 * mt][0][1], ah[0], al[0]);          // row g, level c
        split2(f[2 * mt + 1][0][0], f[2 * mt + 1][0][1], ah[1], al[1]);  // row g + 8, level c
        split2(f[2 * mt][1][0], f[2 * mt][1][1], ah[2], al[2]);          // row g, level c + 4
        split2(f[2 * mt + 1][1][0], f[2 * mt + 1][1][1], ah[3], al[3]);  // row g + 8, level c + 4
#pragma unroll
        for (int j = 0; j < 4; j++) {
            float d[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            mma_split(d, ah, al, fr->w0[j][lane]);
            const float bb0 = fr->b0[8 * j + 2 * c], bb1 = fr->b0[8 * j + 2 * c + 1];
            h0[mt][j][0] = fmaxf(d[0] + bb0, 0.0f);
            h0[mt][j][1] = fmaxf(d[1] + bb1, 0.0f);
            h0[mt][j][2] = fmaxf(d[2] + bb0, 0.0f);
            h0[mt][j][3] = fmaxf(d[3] + bb1, 0.0f);
        }
    }
    float zpart[2][2];  // [M tile][row g / g + 8]: this lane's 8 columns of h1 . w2
#pragma unroll
    for (int mt = 0; mt < 2; mt++) {
        float d1[4][4];
#pragma unroll
        for (int j = 0; j < 4; j++) d1[j][0] = d1[j][1] = d1[j][2] = d1[j][3] = 0.0f;
#pragma unroll
        for (int ks = 0; ks < 2; ks++) {
            uint32_t ah[4], al[4];
            split2(h0[mt][2 * ks][0], h0[mt][2 * ks][1], ah[0], al[0]);
            split2(h0[mt][2 * ks][2], h0[mt][2 * ks][3], ah[1], al[1]);
            split2(h0[mt][2 * ks + 1][0], h0[mt][2 * ks + 1][1], ah[2], al[2]);
            split2(h0[mt][2 * ks + 1][2], h0[mt][2 * ks + 1][3], ah[3], al[3]);
#pragma unroll
            for (int j = 0; j < 4; j++) mma_split(d1[j], ah, al, fr->w1[ks][j][lane]);
        }
        float p0 = 0.0f, p1 = 0.0f;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int n0 = 8 * j + 2 * c;
            const float bb0 = fr->b1[n0], bb1 = fr->b1[n0 + 1], w0v = fr->w2[n0], w1v = fr->w2[n0 + 1];
            p0 = __fmaf_rn(fmaxf(d1[j][0] + bb0, 0.0f), w0v, p0);
            p0 = __fmaf_rn(fmaxf(d1[j][1] + bb1, 0.0f), w1v, p0);
            p1 = __fmaf_rn(fmaxf(d1[j][2] + bb0, 0.0f), w0v, p1);
            p1 = __fmaf_rn(fmaxf(d1[j][3] + bb1, 0.0f), w1v, p1);
        }
        zpart[mt][0] = p0;
        zpart[mt][1] = p1;
    }
    // sum the four lanes of group g: z of samples g, g + 8, 16 + g, 24 + g
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            zpart[mt][h] += __shfl_xor_sync(0xffffffffu, zpart[mt][h], 1);
            zpart[mt][h] += __shfl_xor_sync(0xffffffffu, zpart[mt][h], 2);
        }
    // lane s takes its sample's value from group s & 7, slot s >> 3
    const int src = 4 * (lane & 7), slot = lane >> 3;
    const float z0 = __shfl_sync(0xffffffffu, zpart[0][0], src), z1 = __shfl_sync(0xffffffffu, zpart[0][1], src),
                z2 = __shfl_sync(0xffffffffu, zpart[1][0], src), z3 = __shfl_sync(0xffffffffu, zpart[1][1], src);
    float zo = slot == 0 ? z0 : (slot == 1 ? z1 : (slot == 2 ? z2 : z3));
    zo += fr->b2;
    if (F.out_sigmoid) return 1.0f / (1.0f + expf(-zo));
    return zo < 0.0f ? 0.0f : (zo > 1.0f ? 1.0f : zo);
}

}  // namespace cinr
