// INR training on sm_100a: inr/train.py:16-132 (loss_and_grads + Adam / SGD) for
// the default network (8x2 hash grid -> 16 -> 32 -> 32 -> 1), SURVEY §8f row 3.
//
// One optimizer step = four launches on the caller's stream, no host sync:
//   k_tr_positions  the batch rng.random((B, 3)) of numpy's PCG64 stream (train.py:120):
//                   draw d of the stream = the seeded state jumped d + 1 steps
//   k_field_points  targets = field_src.sample_batch(pos) (the field decoders)
//   k_tr_step       per sample: encode (encoding.py:119-134) -> MLP forward
//                   (mlp.py:39-53) -> MSE gradient -> MLP backward (mlp.py:56-74) ->
//                   encode_backward (encoding.py:137-150) as f64 atomics into the
//                   table gradients; the weight/bias gradients are reduced per CTA
//                   from shared memory and added once per CTA; the loss sum likewise
//   k_tr_update     [gradient-norm clip, train.py:78-85] Adam (51-75) or SGD (40-48);
//                   skipped from the first non-finite loss on (train.py:123-127)
// Gradients accumulate in f64 (the reference's bincount is f64; its sgemm sums are
// f32): parity with the reference is to tolerance (atomics order), the positions
// and the optimizer arithmetic are the reference's.
#include <cmath>

#include "common.cuh"
#include "fields.cuh"
#include "util.cuh"

namespace cinr {

typedef unsigned __int128 u128;

constexpr int kTrB = 96;    // samples per CTA (5 CTAs = 15 warps per SM at <= 136 registers)
constexpr int kTrS = kTrB + 1;  // padded column stride: activations are stored feature-major

struct TrJump {
    u64 m_lo, m_hi, p_lo, p_hi;
};

__global__ void k_tr_init(VcbTrainParams P) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    TrJump* J = reinterpret_cast<TrJump*>(P.jump);
    u128 m = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    u128 c = ((u128)P.pcg_inc[1] << 64) | P.pcg_inc[0];
    for (int j = 0; j < 64; j++) {
        J[j] = TrJump{(u64)m, (u64)(m >> 64), (u64)c, (u64)(c >> 64)};
        c = (m + 1) * c;
        m = m * m;
    }
    P.scratch[0] = 0.0;  // gradient norm^2
    P.scratch[1] = 0.0;  // diverged flag
}

__device__ __forceinline__ double tr_pcg_out(u128 s) {
    const u64 hi = (u64)(s >> 64), lo = (u64)s;
    const u64 x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    const u64 out = (x >> r) | (x << ((64u - r) & 63u));
    return (double)(out >> 11) * 1.1102230246251565e-16;
}

// pos[i][a] = draw (draw0 + step*3B + 3i + a)
// P.scratch[1] != 0: an earlier step's loss was non-finite (k_tr_after); the run has
// diverged and every later step's kernels return at once (train.py:123-127 stops there).
__device__ __forceinline__ bool tr_diverged(const VcbTrainParams& P) { return P.scratch[1] != 0.0; }

__global__ void k_tr_positions(VcbTrainParams P, long long step) {
    if (tr_diverged(P)) return;
    const TrJump* J = reinterpret_cast<const TrJump*>(P.jump);
    const u128 A = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    const u128 inc = ((u128)P.pcg_inc[1] << 64) | P.pcg_inc[0];
    const u128 s0 = ((u128)P.pcg_state[1] << 64) | P.pcg_state[0];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.batch;
         i += (long long)gridDim.x * blockDim.x) {
        u64 delta = P.draw0 + (u64)step * 3ull * (u64)P.batch + 3ull * (u64)i + 1ull;
        u128 s = s0;
        for (int j = 0; delta; j++, delta >>= 1) {
            if (delta & 1) {
                const TrJump e = J[j];
                s = s * (((u128)e.m_hi << 64) | e.m_lo) + (((u128)e.p_hi << 64) | e.p_lo);
            }
        }
        P.pos[3 * i] = tr_pcg_out(s);
        s = s * A + inc;
        P.pos[3 * i + 1] = tr_pcg_out(s);
        s = s * A + inc;
        P.pos[3 * i + 2] = tr_pcg_out(s);
    }
}

struct TrSmem {
    float feat[16][kTrS];  // [feature][sample]; d2 is recomputed from delta, h1 and W2
    float h0[32][kTrS];
    float h1[32][kTrS];
    float d1[32][kTrS];
    float delta[kTrB];
    double red[kTrB / 32];
};

// one CTA = kTrB samples; thread t owns sample blockIdx.x*kTrB + t
template <bool kSig>
__global__ void __launch_bounds__(kTrB, 5) k_tr_step(VcbTrainParams P, long long step) {
    extern __shared__ __align__(16) unsigned char tr_smem[];
    if (tr_diverged(P)) return;
    TrSmem& S = *reinterpret_cast<TrSmem*>(tr_smem);
    const VcbField& F = P.model;
    const float* W0 = F.weights + F.w_off[0];  // [32][16]
    const float* W1 = F.weights + F.w_off[1];  // [32][32]
    const float* W2 = F.weights + F.w_off[2];  // [1][32]
    const float* B0 = F.biases + F.b_off[0];
    const float* B1 = F.biases + F.b_off[1];
    const float* B2 = F.biases + F.b_off[2];
    const int t = threadIdx.x;
    const long long i = (long long)blockIdx.x * kTrB + t;
    const bool live = i < P.batch;
    double err2 = 0.0;
    float feat[16], h0[32], h1[32];
    double x = 0.0, y = 0.0, z = 0.0;
    float delta = 0.0f;
    if (live) {
        x = P.pos[3 * i];
        y = P.pos[3 * i + 1];
        z = P.pos[3 * i + 2];
#pragma unroll
        for (int l = 0; l < 8; l++) encode_level<2>(F, l, x, y, z, feat + 2 * l);
#pragma unroll
        for (int j = 0; j < 32; j++) {
            float a = 0.0f;
#pragma unroll
            for (int m = 0; m < 16; m++) a = __fmaf_rn(feat[m], __ldg(W0 + j * 16 + m), a);
            a = __fadd_rn(a, __ldg(B0 + j));
            h0[j] = a > 0.0f ? a : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 32; k++) {
            float a = 0.0f;
#pragma unroll
            for (int j = 0; j < 32; j++) a = __fmaf_rn(h0[j], __ldg(W1 + k * 32 + j), a);
            a = __fadd_rn(a, __ldg(B1 + k));
            h1[k] = a > 0.0f ? a : 0.0f;
        }
        float zo = 0.0f;
#pragma unroll
        for (int k = 0; k < 32; k++) zo = __fmaf_rn(h1[k], __ldg(W2 + k), zo);
        zo = __fadd_rn(zo, __ldg(B2));
        // train.py:30-32 + mlp.py:58-61 (d_z in f64, delta cast to the weights' f32)
        double dz;
        float yo;
        if (kSig) {
            yo = 1.0f / (1.0f + expf(-zo));
            const double err = (double)yo - (double)P.targets[i];
            err2 = err * err;
            const double dy = 2.0 * err / (double)P.batch;
            dz = dy * (double)yo * (double)(1.0f - yo);
        } else {
            yo = zo < 0.0f ? 0.0f : (zo > 1.0f ? 1.0f : zo);
            const double err = (double)yo - (double)P.targets[i];
            err2 = err * err;
            const double dy = 2.0 * err / (double)P.batch;
            dz = (zo > 0.0f && zo < 1.0f) ? dy : 0.0;
        }
        delta = (float)dz;
    }
    // rows for the CTA's weight-gradient reductions
#pragma unroll
    for (int m = 0; m < 16; m++) S.feat[m][t] = live ? feat[m] : 0.0f;
#pragma unroll
    for (int j = 0; j < 32; j++) {
        S.h0[j][t] = live ? h0[j] : 0.0f;
        S.h1[j][t] = live ? h1[j] : 0.0f;
    }
    S.delta[t] = delta;
    // backward (mlp.py:64-74): d2 = (delta W2) * [h1 > 0]; d1 = (d2 W1) * [h0 > 0]; dfeat = d1 W0
    float d2[32];
#pragma unroll
    for (int k = 0; k < 32; k++) {
        d2[k] = h1[k] > 0.0f ? delta * __ldg(W2 + k) : 0.0f;
    }
    float d1[32];
#pragma unroll
    for (int j = 0; j < 32; j++) {
        float a = 0.0f;
#pragma unroll
        for (int k = 0; k < 32; k++) a = __fmaf_rn(d2[k], __ldg(W1 + k * 32 + j), a);
        d1[j] = h0[j] > 0.0f ? a : 0.0f;
        S.d1[j][t] = live ? d1[j] : 0.0f;
    }
    if (live) {
        float df[16];
#pragma unroll
        for (int m = 0; m < 16; m++) {
            float a = 0.0f;
#pragma unroll
            for (int j = 0; j < 32; j++) a = __fmaf_rn(d1[j], __ldg(W0 + j * 16 + m), a);
            df[m] = a;
        }
        // encode_backward (encoding.py:137-150): table[idx] += w (f64) * dfeat (as f64)
        double* gt = P.grads;
#pragma unroll 1
        for (int l = 0; l < 8; l++) {
            const int r = F.res[l];
            const double rd = (double)r;
            const double u[3] = {x * rd, y * rd, z * rd};
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
            const double g0 = (double)df[2 * l], g1 = (double)df[2 * l + 1];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int dx = c & 1, dy = (c >> 1) & 1, dz2 = (c >> 2) & 1;
                const uint32_t vx = c0[0] + dx, vy = c0[1] + dy, vz = c0[2] + dz2;
                const uint32_t idx = F.dense[l] ? vx + side * vy + side * side * vz
                                                : ((vx * 2654435761u) ^ (vy * 2246822519u) ^ (vz * 3266489917u)) & mask;
                const double w = wx[dx] * wy[dy] * wz[dz2];
                double* row = gt + (F.tab_off[l] + (long long)idx) * 2;
                atomicAdd(row, w * g0);
                atomicAdd(row + 1, w * g1);
            }
        }
    }
    // loss sum (f64)
    err2 = warp_sum(err2);
    if ((t & 31) == 0) S.red[t >> 5] = err2;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int w = 0; w < kTrB / 32; w++) s += S.red[w];
        atomicAdd(P.loss + step, s);
    }
    // weight / bias gradients of this CTA's samples (mlp.py:68-73), one f64 atomic each
    const long long wbase = P.n_table_params;
    const long long bbase = wbase + P.n_weights;
    for (int e = t; e < 1633; e += kTrB) {
        float acc = 0.0f;
        long long dst;
        if (e < 512) {  // dW0[j][m] = sum d1[j] feat[m]
            const int j = e >> 4, m = e & 15;
            for (int s = 0; s < kTrB; s++) acc = __fmaf_rn(S.d1[j][s], S.feat[m][s], acc);
            dst = wbase + F.w_off[0] + e;
        } else if (e < 1536) {  // dW1[k][j] = sum d2[k] h0[j]
            const int q = e - 512, k = q >> 5, j = q & 31;
            const float w2k = __ldg(W2 + k);
            for (int s = 0; s < kTrB; s++) {
                const float d2 = S.h1[k][s] > 0.0f ? S.delta[s] * w2k : 0.0f;  // (delta W2) * [h1 > 0]
                acc = __fmaf_rn(d2, S.h0[j][s], acc);
            }
            dst = wbase + F.w_off[1] + q;
        } else if (e < 1568) {  // dW2[k] = sum delta h1[k]
            const int k = e - 1536;
            for (int s = 0; s < kTrB; s++) acc = __fmaf_rn(S.delta[s], S.h1[k][s], acc);
            dst = wbase + F.w_off[2] + k;
        } else if (e < 1600) {
            const int j = e - 1568;
            for (int s = 0; s < kTrB; s++) acc = __fadd_rn(acc, S.d1[j][s]);
            dst = bbase + F.b_off[0] + j;
        } else if (e < 1632) {
            const int k = e - 1600;
            const float w2k = __ldg(W2 + k);
            for (int s = 0; s < kTrB; s++) acc = __fadd_rn(acc, S.h1[k][s] > 0.0f ? S.delta[s] * w2k : 0.0f);
            dst = bbase + F.b_off[1] + k;
        } else {
            for (int s = 0; s < kTrB; s++) acc = __fadd_rn(acc, S.delta[s]);
            dst = bbase + F.b_off[2];
        }
        if (acc != 0.0f) atomicAdd(P.grads + dst, (double)acc);
    }
}

__device__ __forceinline__ float* tr_param(const VcbTrainParams& P, long long q) {
    if (q < P.n_table_params) return const_cast<float*>(P.model.tables) + q;
    q -= P.n_table_params;
    if (q < P.n_weights) return const_cast<float*>(P.model.weights) + q;
    return const_cast<float*>(P.model.biases) + (q - P.n_weights);
}

// train.py:81: sum of the f32 gradients squared, in f64
__global__ void k_tr_gnorm(VcbTrainParams P) {
    if (tr_diverged(P)) return;
    double s = 0.0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P.n_params;
         q += (long long)gridDim.x * blockDim.x) {
        const double g = (double)(float)P.grads[q];
        s += g * g;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(P.scratch, s);
}

__global__ void k_tr_update(VcbTrainParams P, long long step, double bc1, double bc2) {
    // train.py:123-127: a non-finite loss stops the run before this step's update
    const double ls = P.loss[step];
    const bool stop = !isfinite(ls) || P.scratch[1] != 0.0 || P.optimizer == 2;  // 2: learning rate 0
    float scale = 1.0f;
    bool clip = false;
    if (P.flags & 4) {  // clip_norm given (None = no clipping; 0 zeroes the gradients, train.py:78-85)
        const double total = sqrt(P.scratch[0]);
        if (!(total <= P.clip_norm || total == 0.0)) {
            clip = true;
            scale = (float)(P.clip_norm / total);
        }
    }
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P.n_params;
         q += (long long)gridDim.x * blockDim.x) {
        float g = (float)P.grads[q];
        P.grads[q] = 0.0;
        if (stop) continue;
        if (clip) g = g * scale;
        float* p = tr_param(P, q);
        if (P.optimizer == 0) {
            double m = P.m[q] * P.beta1;
            m = m + (double)((float)(1.0 - P.beta1) * g);
            double v = P.v[q] * P.beta2;
            v = v + (1.0 - P.beta2) * ((double)g * (double)g);
            P.m[q] = m;
            P.v[q] = v;
            const double upd = P.lr * (m / bc1) / (sqrt(v / bc2) + P.eps);
            *p = *p - (float)upd;
        } else {
            *p = *p - (float)P.lr * g;
        }
    }
}

__global__ void k_tr_after(VcbTrainParams P, long long step) {
    P.scratch[0] = 0.0;
    if (!isfinite(P.loss[step])) P.scratch[1] = 1.0;
}

}  // namespace cinr

using namespace cinr;

extern "C" int32_t vcb_field_points(const VcbField* f, int64_t n, const double* pos, float* out, int32_t* nonfinite,
                                    void* stream);

extern "C" int64_t vcb_train_workspace_bytes(int64_t batch) {
    (void)batch;
    return 64 * (int64_t)sizeof(TrJump) + 64;
}

extern "C" int32_t vcb_train_steps(const VcbTrainParams* pp, void* stream_) {
    const VcbTrainParams& P = *pp;
    cudaStream_t st = (cudaStream_t)stream_;
    if (P.model.kind != 0 || !inr_is_default(P.model) || P.model.feats != 2)
        return set_error("train_steps: the GPU trainer supports the default 8x2 hash grid + 16-32-32-1 MLP");
    if (P.batch < 1 || P.steps < 0) return set_error("train_steps: batch %lld, steps %lld", (long long)P.batch,
                                                     (long long)P.steps);
    if (P.optimizer < 0 || P.optimizer > 2) return set_error("train_steps: optimizer %d", P.optimizer);
    const int smem = (int)sizeof(TrSmem);
    const void* fn = P.model.out_sigmoid ? (const void*)k_tr_step<true> : (const void*)k_tr_step<false>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_tr_init<<<1, 32, 0, st>>>(P);
    const int gp = grid_for(P.batch, 256);
    const int gs = (int)((P.batch + kTrB - 1) / kTrB);
    const int gu = grid_for(P.n_params, 256);
    long long launches = 1;
    for (long long s = 0; s < P.steps; s++) {
        if (!(P.flags & 1)) {
            k_tr_positions<<<gp, 256, 0, st>>>(P, s);
            int32_t rc = vcb_field_points(&P.target, P.batch, P.pos, P.targets, P.nonfinite, st);
            if (rc != 0) return rc;
        }
        if (P.model.out_sigmoid) k_tr_step<true><<<gs, kTrB, smem, st>>>(P, s);
        else k_tr_step<false><<<gs, kTrB, smem, st>>>(P, s);
        if (P.flags & 2) {
            launches += 1;
            continue;  // loss_and_grads: gradients stay in P.grads
        }
        if (P.flags & 4) k_tr_gnorm<<<gu, 256, 0, st>>>(P);
        const double t = (double)(P.step0 + s + 1);
        const double bc1 = 1.0 - std::pow(P.beta1, t), bc2 = 1.0 - std::pow(P.beta2, t);
        k_tr_update<<<gu, 256, 0, st>>>(P, s, bc1, bc2);
        k_tr_after<<<1, 1, 0, st>>>(P, s);
        launches += 5 + ((P.flags & 4) ? 1 : 0);
    }
    return check_launch("train_steps");
}
