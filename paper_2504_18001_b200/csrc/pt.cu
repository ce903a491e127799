// Volumetric path tracing on sm_100a (compiled with -fmad=false): the
// reference's second render mode, render/pathtrace.py:28-146, on the same
// cached sampler as the ray march (sampler.py:196-280).
//
// Frame: raygen + ordered compaction of box hits (the ray bundle, camera.py:129-154),
// then per sample-per-pixel
//   walk(primary)  Woodcock delta tracking of every bundle ray (trace_free_flight,
//                  pathtrace.py:28-98) + ordered compaction of the hits into shadow rays
//   walk(shadow)   one delta-tracked shadow ray per hit toward the light (101-109)
//   accumulate     tf.eval(v) * (ambient + (1 - ambient) * vis), or the background (130-142)
// and a final pass writing total / spp and hits / spp (143-146).
//
// A walk is one persistent cooperative kernel (one 512-thread CTA per SM) that
// runs the reference's wavefront iterations with three grid barriers each:
//   1 classify: position, outside test, macro cell, majorant, cell exit; empty
//     cells hop or escape; the rest draw a free flight (done by the previous
//     iteration's compaction for every survivor, so only iteration 0 has its own pass)
//   2 draws: dense rays ranked in ray order take numpy PCG64 draw D + rank
//     (rng.random(dense.size), line 79), free flight t - log1p(-xi)/mu
//   3 sample: settled rays ranked in ray order are one VolumeSampler.sample batch
//     (XorShift32 lane = rank, with the reference's lane-pool reseeding,
//     sampler.py:206-213), MRPD probe + miss filing + true-miss INR, then the
//     acceptance draw D + n_dense + rank (line 91)
//   4 ordered compaction of the rays still walking, fused with their classification
//     for the next iteration (dense counts land on the CTA owning the new slot).
// Ranks come from per-CTA counts (each CTA owns a contiguous chunk of the active
// list) plus a block scan, so every draw index, lane and list position equals the
// reference's.  The PCG64 state of draw D is a jump of the seeded state by D + 1
// steps (a radix-16 table of LCG jumps built on the device per frame: a CTA keeps the
// state at the start of each 512-ray round and a lane jumps by its rank, at most three
// table steps); log1p is glibc's
// algorithm (the FMA build numpy calls on x86-64), bit-identical.
#include <cstdio>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"

namespace cinr {

typedef unsigned __int128 u128;

constexpr int kPtThreads = 512;
constexpr int kPtMaxTf = 64;
constexpr int kPtMaxCtas = 1024;

struct PtJump {
    u64 m_lo, m_hi, p_lo, p_hi;
};

// Sampler / PCG bookkeeping carried across the walks of one frame.
struct PtRng {
    u64 draws;        // numpy PCG64 draws consumed this frame
    long long pool;   // XorShift32 lanes seeded this frame (0 = not yet, sampler.py:206)
    long long salt;   // _reseed_salt
    unsigned gen;     // lane generation (lanes seeded lazily: stored generation != gen -> reseed)
    unsigned pad;
    u64 base;         // splitmix64(seed ^ frame' * GOLDEN) of generation gen
    long long iters;  // walk iterations (stats)
    int nonfinite;
    int sh_n;         // shadow rays of the current sample
    long long pad2[8];
};

struct PtWs {
    double* t[2];      // walk state: [0] primary, [1] shadow
    double* thit[2];
    float* vhit[2];
    int* list[2];
    uint8_t* flag;
    uint8_t* flag2;    // second list-flag buffer (walk rebalancing)
    double* exitb;     // [n] cell exit of a dense ray (classify -> draw)
    float* mub;        // [n] majorant of a settled ray's cell (mu[~empty][~crossed], line 91)
    double* sh_o;      // [3n] shadow origins (primary hit points)
    double* sh_tend;   // [n] t_far of the shadow ray
    int* sh_of;        // [n] primary ray -> shadow ray (-1 = no hit)
    double* total;     // [3n]
    double* hits;      // [n]
    unsigned long long* lane;  // [n] XorShift32 lane: (generation << 32) | state
    int* cnt;          // [4][kPtMaxCtas]
    unsigned* bar;
    PtRng* rng;
    PtJump* jump;      // [64] binary jump table (A^2^j, C_j)
    PtJump* j16;       // [16][16] radix-16 jump table: digit d, value v -> jump by v*16^d
};

inline int64_t pt_ws_layout(int64_t n, void* base, PtWs* s) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    size_t o_t[2], o_th[2], o_vh[2], o_l[2];
    for (int b = 0; b < 2; b++) {
        o_t[b] = take((size_t)n * 8);
        o_th[b] = take((size_t)n * 8);
        o_vh[b] = take((size_t)n * 4);
        o_l[b] = take((size_t)n * 4);
    }
    size_t o_f = take((size_t)n);
    size_t o_f2 = take((size_t)n);
    size_t o_ex = take((size_t)n * 8);
    size_t o_mub = take((size_t)n * 4);
    size_t o_sho = take((size_t)n * 24);
    size_t o_sht = take((size_t)n * 8);
    size_t o_shof = take((size_t)n * 4);
    size_t o_tot = take((size_t)n * 24);
    size_t o_hit = take((size_t)n * 8);
    size_t o_ls = take((size_t)n * 8);
    size_t o_cnt = take((size_t)4 * kPtMaxCtas * 4);
    size_t o_bar = take(64);
    size_t o_rng = take(sizeof(PtRng));
    size_t o_j = take(64 * sizeof(PtJump));
    size_t o_j16 = take(256 * sizeof(PtJump));
    if (base && s) {
        char* p = (char*)base;
        for (int b = 0; b < 2; b++) {
            s->t[b] = (double*)(p + o_t[b]);
            s->thit[b] = (double*)(p + o_th[b]);
            s->vhit[b] = (float*)(p + o_vh[b]);
            s->list[b] = (int*)(p + o_l[b]);
        }
        s->flag = (uint8_t*)(p + o_f);
        s->flag2 = (uint8_t*)(p + o_f2);
        s->exitb = (double*)(p + o_ex);
        s->mub = (float*)(p + o_mub);
        s->sh_o = (double*)(p + o_sho);
        s->sh_tend = (double*)(p + o_sht);
        s->sh_of = (int*)(p + o_shof);
        s->total = (double*)(p + o_tot);
        s->hits = (double*)(p + o_hit);
        s->lane = (unsigned long long*)(p + o_ls);
        s->cnt = (int*)(p + o_cnt);
        s->bar = (unsigned*)(p + o_bar);
        s->rng = (PtRng*)(p + o_rng);
        s->jump = (PtJump*)(p + o_j);
        s->j16 = (PtJump*)(p + o_j16);
    }
    return (int64_t)align_up(off, 256);
}

// ------------------------------------------------------------------ numerics
// glibc's log1p (the fdlibm algorithm with the Estrin polynomial, in the FMA
// build x86-64 dispatches to); identical to it on 4e7 inputs in [-1, 0], the
// edge regions included (oracle test).
__device__ __forceinline__ double pt_log1p(double x) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
                 Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                 Lp7 = 1.479819860511658591e-01;
    double f = 0.0, c = 0.0, u;
    int hu = 0;
    const int hx = __double2hiint(x), ax = hx & 0x7fffffff;
    int k = 1;
    if (hx < 0x3FDA827A) {
        if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : nan("");
        if (ax < 0x3e200000) {
            if (ax < 0x3c900000) return x;
            return fma(-DMUL(x, x), 0.5, x);
        }
        if (hx > 0 || hx <= (int)0xbfd2bec3) {
            k = 0;
            f = x;
            hu = 1;
        }
    }
    if (hx >= 0x7ff00000) return DADD(x, x);
    if (k != 0) {
        if (hx < 0x43400000) {
            u = DADD(1.0, x);
            hu = __double2hiint(u);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? DSUB(1.0, DSUB(u, x)) : DSUB(x, DSUB(u, 1.0));
            c = __ddiv_rn(c, u);
        } else {
            u = x;
            hu = __double2hiint(u);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
        } else {
            k += 1;
            u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
            hu = (0x00100000 - hu) >> 2;
        }
        f = DSUB(u, 1.0);
    }
    const double hfsq = DMUL(DMUL(0.5, f), f);
    const double dk = (double)k;
    if (hu == 0) {
        if (f == 0.0) {
            if (k == 0) return 0.0;
            c = fma(dk, ln2_lo, c);
            return fma(dk, ln2_hi, c);
        }
        const double R = DMUL(hfsq, fma(-0.66666666666666666, f, 1.0));
        if (k == 0) return DSUB(f, R);
        return fma(dk, ln2_hi, -DSUB(DSUB(R, fma(dk, ln2_lo, c)), f));
    }
    const double s = __ddiv_rn(f, DADD(2.0, f));
    const double z = DMUL(s, s);
    const double z2 = DMUL(z, z), z4 = DMUL(z2, z2), z6 = DMUL(z4, z2);
    const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
    double R = fma(z, Lp1, DMUL(z2, R2));
    R = fma(z4, R3, R);
    R = fma(R4, z6, R);
    if (k == 0) return DSUB(f, DSUB(hfsq, DMUL(s, DADD(hfsq, R))));
    return fma(dk, ln2_hi, -DSUB(DSUB(hfsq, DADD(DMUL(s, DADD(hfsq, R)), fma(dk, ln2_lo, c))), f));
}

// numpy PCG64 (XSL-RR 128/64): uniform of draw d (0-based) of the stream seeded at s0
__device__ __forceinline__ double pcg_uniform_at(u128 s0, u64 d, const PtJump* __restrict__ J) {
    u64 delta = d + 1;
    u128 s = s0;
    for (int j = 0; delta; j++, delta >>= 1) {
        if (delta & 1) {
            const PtJump e = J[j];
            s = s * (((u128)e.m_hi << 64) | e.m_lo) + (((u128)e.p_hi << 64) | e.p_lo);
        }
    }
    const u64 hi = (u64)(s >> 64), lo = (u64)s;
    const u64 x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    const u64 out = (x >> r) | (x << ((64u - r) & 63u));
    return (double)(out >> 11) * 1.1102230246251565e-16;  // 2^-53
}

// state jumped by delta steps with the radix-16 table (at most one step per hex digit)
__device__ __forceinline__ u128 pcg_jump16(u128 s, u64 delta, const PtJump* J) {
    for (int d = 0; delta; d++, delta >>= 4) {
        const int v = (int)(delta & 15);
        if (v) {
            const PtJump e = J[d * 16 + v];
            s = s * (((u128)e.m_hi << 64) | e.m_lo) + (((u128)e.p_hi << 64) | e.p_lo);
        }
    }
    return s;
}

__device__ __forceinline__ double pcg_out(u128 s) {
    const u64 hi = (u64)(s >> 64), lo = (u64)s;
    const u64 x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    const u64 out = (x >> r) | (x << ((64u - r) & 63u));
    return (double)(out >> 11) * 1.1102230246251565e-16;  // 2^-53
}

// np.interp(x, xp, fp) for sorted xp (numpy/core/src/multiarray/compiled_base.c arr_interp)
__device__ __forceinline__ double np_interp(double x, const double* xp, const double* fp, int n, int stride) {
    if (x > xp[(n - 1) * stride]) return fp[(n - 1) * stride];
    if (x < xp[0]) return fp[0];
    int j = 0;
    while (j + 1 < n && xp[(j + 1) * stride] <= x) j++;
    if (j == n - 1) return fp[j * stride];
    const double xj = xp[j * stride], xj1 = xp[(j + 1) * stride], fj = fp[j * stride], fj1 = fp[(j + 1) * stride];
    if (xj == x) return fj;
    const double slope = __ddiv_rn(DSUB(fj1, fj), DSUB(xj1, xj));
    double r = DADD(DMUL(slope, DSUB(x, xj)), fj);
    if (r != r) {
        r = DADD(DMUL(slope, DSUB(x, xj1)), fj1);
        if (r != r && fj == fj1) r = fj;
    }
    return r;
}

// ------------------------------------------------------------------ grid helpers
__device__ __forceinline__ void pt_barrier(unsigned* bar, unsigned& target) {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// exclusive block rank of flag f (512 threads) and the block total
__device__ __forceinline__ int pt_block_rank(bool f, int* s_w, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_w[warp] = __popc(b);
    __syncthreads();
    if (warp == 0) {
        const int v = lane < kPtThreads / 32 ? s_w[lane] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < kPtThreads / 32) s_w[lane] = x - v;
        if (lane == 31) s_w[32] = x;
    }
    __syncthreads();
    const int r = s_w[warp] + __popc(b & ((1u << lane) - 1u));
    total = s_w[32];
    __syncthreads();
    return r;
}

// (prefix over CTAs < c, total) of a per-CTA count array
__device__ __forceinline__ void pt_cta_prefix(const int* cnt, long long* s, long long& pre, long long& tot) {
    long long a = 0, b = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        const int v = __ldcg(cnt + i);
        b += v;
        if (i < (int)blockIdx.x) a += v;
    }
    a = warp_sum(a);
    b = warp_sum(b);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s[2 * warp] = a;
        s[2 * warp + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long x = 0, y = 0;
        for (int w = 0; w < kPtThreads / 32; w++) {
            x += s[2 * w];
            y += s[2 * w + 1];
        }
        s[64] = x;
        s[65] = y;
    }
    __syncthreads();
    pre = s[64];
    tot = s[65];
    __syncthreads();
}

// prefix + total + max of a per-CTA count array
__device__ __forceinline__ void pt_cta_prefix_max(const int* cnt, long long* s, long long& pre, long long& tot,
                                                  long long& mx) {
    long long a = 0, b = 0, c = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        const int v = __ldcg(cnt + i);
        b += v;
        c = v > c ? v : c;
        if (i < (int)blockIdx.x) a += v;
    }
    a = warp_sum(a);
    b = warp_sum(b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long y = __shfl_xor_sync(0xffffffffu, c, o);
        c = y > c ? y : c;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s[3 * warp] = a;
        s[3 * warp + 1] = b;
        s[3 * warp + 2] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long x = 0, y = 0, z = 0;
        for (int w = 0; w < kPtThreads / 32; w++) {
            x += s[3 * w];
            y += s[3 * w + 1];
            z = s[3 * w + 2] > z ? s[3 * w + 2] : z;
        }
        s[64] = x;
        s[65] = y;
        s[66] = z;
    }
    __syncthreads();
    pre = s[64];
    tot = s[65];
    mx = s[66];
    __syncthreads();
}

__device__ __forceinline__ void pt_chunk(long long n, long long& lo, long long& hi) {
    const long long ch = (n + gridDim.x - 1) / gridDim.x;
    lo = (long long)blockIdx.x * ch;
    if (lo > n) lo = n;
    hi = lo + ch;
    if (hi > n) hi = n;
}

// ------------------------------------------------------------------ one walk step
struct PtWalk {
    const int* n_dev;  // ray count on the device, or nullptr: n_const
    long long n_const;
    const double* o;  // per ray [3n] when o_stride == 3, else oc
    const double* d;
    const double* t0;
    const double* tend;
    double oc[3], dc[3], t0c;
    int o_stride, d_stride, t0_stride;
    int which;        // 0 primary, 1 shadow
    int mu_smem;      // majorant grid staged in shared memory after the MLP weights
    int mu_off;       // its float offset in the dynamic shared memory
};

struct PtGeo {
    float mu;
    double exit_t;
    bool outside, at_end;
};

// pathtrace.py:54-68 for one ray
__device__ __forceinline__ PtGeo pt_geo(const VcbFrameParams& p, float dens_f, double ox, double oy, double oz,
                                        double dx, double dy, double dz, double t, double tend,
                                        const float* mu_grid = nullptr) {
    PtGeo g;
    const double px = DADD(ox, DMUL(dx, t)), py = DADD(oy, DMUL(dy, t)), pz = DADD(oz, DMUL(dz, t));
    const double lo = -1e-12, hi = 1.000000000001;
    g.outside = px < lo || py < lo || pz < lo || px > hi || py > hi || pz > hi;
    g.mu = 0.0f;
    g.exit_t = 0.0;
    g.at_end = false;
    if (g.outside) return g;
    long long cx = (long long)floor(__ddiv_rn(px, p.adv.cwx));
    long long cy = (long long)floor(__ddiv_rn(py, p.adv.cwy));
    long long cz = (long long)floor(__ddiv_rn(pz, p.adv.cwz));
    cx = cx < 0 ? 0 : (cx > p.adv.gx - 1 ? p.adv.gx - 1 : cx);
    cy = cy < 0 ? 0 : (cy > p.adv.gy - 1 ? p.adv.gy - 1 : cy);
    cz = cz < 0 ? 0 : (cz > p.adv.gz - 1 ? p.adv.gz - 1 : cz);
    const long long cell = (cz * p.adv.gy + cy) * p.adv.gx + cx;
    g.mu = FMUL(mu_grid ? mu_grid[cell] : __ldg(p.mu + cell), dens_f);
    // _cell_exit (21-25)
    const double bx = DMUL((double)(cx + (dx > 0.0 ? 1 : 0)), p.adv.cwx);
    const double by = DMUL((double)(cy + (dy > 0.0 ? 1 : 0)), p.adv.cwy);
    const double bz = DMUL((double)(cz + (dz > 0.0 ? 1 : 0)), p.adv.cwz);
    const double tx = fabs(dx) > 1e-14 ? __ddiv_rn(DSUB(bx, ox), dx) : INFINITY;
    const double ty = fabs(dy) > 1e-14 ? __ddiv_rn(DSUB(by, oy), dy) : INFINITY;
    const double tz = fabs(dz) > 1e-14 ? __ddiv_rn(DSUB(bz, oz), dz) : INFINITY;
    double m = tx < ty ? tx : ty;
    m = m < tz ? m : tz;
    const double tn = DADD(t, 1e-9);
    const double cell_exit = m > tn ? m : tn;
    g.at_end = cell_exit >= DSUB(tend, 1e-9);
    g.exit_t = cell_exit < tend ? cell_exit : tend;
    return g;
}

// VolumeSampler.sample for one settled ray at rank `lane` of its batch (sampler.py:196-280):
// lane RNG (lazily reseeded generations), |pos - camera| distance, MRPD probe + stamp,
// miss filing at the requested LoD, true-miss inference at clamp_normalized(pos).
template <int kInr>
__device__ __forceinline__ float pt_sample(const VcbFrameParams& p, const PtWs& s, const PtRng& R, const MlpSmem& mlp,
                                           long long lane, double px, double py, double pz,
                                           unsigned long long& c_ex, unsigned long long& c_fb,
                                           unsigned long long& c_ms) {
    const double hi_n = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
    float v = 0.0f;
    bool miss = true;
    if (p.cached) {
        double u = 0.0;
        if (p.probe.mode != 2) {
            const unsigned long long w = __ldcg(s.lane + lane);
            uint32_t st = ((unsigned)(w >> 32) == R.gen) ? (uint32_t)w : lane_seed(R.base, (u64)lane);
            st = xorshift32(st);
            __stcg(s.lane + lane, ((unsigned long long)R.gen << 32) | st);
            u = DMUL((double)st, 2.3283064365386963e-10);
        }
        const double ex = DSUB(px, p.cam.origin[0]), ey = DSUB(py, p.cam.origin[1]), ez = DSUB(pz, p.cam.origin[2]);
        const double dist = __dsqrt_rn(DADD(DADD(DMUL(ex, ex), DMUL(ey, ey)), DMUL(ez, ez)));
        int rq, slot;
        const int sv = probe_one(px, py, pz, dist, u, p.probe, p.table, p.pool, (long long*)p.last_used,
                                 p.cache_frame, v, rq, slot);
        if (sv != rq) {
            // mrpd.py:215-225 miss filing at the requested LoD (native clipped)
            const i64 span = p.probe.b << rq;
            const double nx = clampd(DSUB(DMUL(px, p.probe.vx), 0.5), 0.0, DSUB(p.probe.vx, 1.0));
            const double ny = clampd(DSUB(DMUL(py, p.probe.vy), 0.5), 0.0, DSUB(p.probe.vy, 1.0));
            const double nz = clampd(DSUB(DMUL(pz, p.probe.vz), 0.5), 0.0, DSUB(p.probe.vz, 1.0));
            const i64 bx = clampi((i64)floor(cell_div(DADD(nx, 1.0), (double)span)), 0, p.probe.grid[rq][0] - 1);
            const i64 by = clampi((i64)floor(cell_div(DADD(ny, 1.0), (double)span)), 0, p.probe.grid[rq][1] - 1);
            const i64 bz = clampi((i64)floor(cell_div(DADD(nz, 1.0), (double)span)), 0, p.probe.grid[rq][2] - 1);
            warp_aggregated_add(p.miss_count,
                                p.probe.offset[rq] + bx + p.probe.grid[rq][0] * (by + p.probe.grid[rq][1] * bz));
        }
        miss = sv < 0;
        if (!miss) {
            c_ex += (sv == rq);
            c_fb += (sv != rq);
        }
    }
    if (miss) {
        c_ms++;
        v = field_eval<kInr>(p.field, clampd(px, 0.0, hi_n), clampd(py, 0.0, hi_n), clampd(pz, 0.0, hi_n), mlp,
                             &s.rng->nonfinite);
    }
    return v;
}

// shadow ray j of primary ray i hit at th: origin o + d th, t_far = intersect_aabb(points,
// light)[1] (camera.py:95-110, pathtrace.py:101-108)
template <class FO, class FD>
__device__ __forceinline__ void pt_shadow_ray(const VcbPtParams& q, const PtWs& s, long long j, int i, double th,
                                              FO& ray_o, FD& ray_d) {
    double ox, oy, oz, dx, dy, dz;
    ray_o(i, ox, oy, oz);
    ray_d(i, dx, dy, dz);
    const double px = DADD(ox, DMUL(dx, th)), py = DADD(oy, DMUL(dy, th)), pz = DADD(oz, DMUL(dz, th));
    s.sh_o[3 * j] = px;
    s.sh_o[3 * j + 1] = py;
    s.sh_o[3 * j + 2] = pz;
    const double o3[3] = {px, py, pz};
    double tfar = INFINITY;
    for (int a = 0; a < 3; a++) {
        const double da = q.light[a];
        double tl, th2;
        if (da != 0.0) {
            const double inv = __ddiv_rn(1.0, da);
            tl = DMUL(DSUB(0.0, o3[a]), inv);
            th2 = DMUL(DSUB(1.0, o3[a]), inv);
        } else {
            const bool inside = o3[a] >= 0.0 && o3[a] <= 1.0;
            tl = inside ? -INFINITY : INFINITY;
            th2 = inside ? INFINITY : -INFINITY;
        }
        const double mx = tl > th2 ? tl : th2;
        tfar = (a == 0 || mx < tfar) ? mx : tfar;
    }
    s.sh_tend[j] = tfar;
}

struct PtSmem {
    PtJump j16[256];
    double tf[kPtMaxTf * 5];
    long long red[70];
    int w[40];
};

template <int kInr>
__global__ void __launch_bounds__(kPtThreads, 1)
    k_pt_walk(VcbFrameParams p, VcbPtParams q, FrameWs fw, PtWs s, PtWalk wk) {
    __shared__ PtSmem sm;
    extern __shared__ __align__(16) float smem[];
    MlpSmem mlp;
    if (kInr != 0) stage_mlp(p.field, smem, mlp);
    const float* MUG = nullptr;  // majorant grid in shared memory when it fits
    if (wk.mu_smem) {
        float* g = smem + wk.mu_off;
        const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
        for (long long c = threadIdx.x; c < cells; c += blockDim.x) g[c] = __ldg(p.mu + c);
        MUG = g;
    }
    for (int i = threadIdx.x; i < q.n_tf * 5; i += blockDim.x) sm.tf[i] = q.tf[i];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sm.j16[i] = s.j16[i];
    unsigned target = 0;
    const int W = wk.which;
    double* T = s.t[W];
    double* TH = s.thit[W];
    float* VH = s.vhit[W];
    const float dens_f = __double2float_rn(q.density);
    const double hi_n = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
    // frame-level sampler/PCG state (identical in every CTA, written back by CTA 0)
    PtRng R = *s.rng;
    const u128 s0 = ((u128)q.pcg_state[1] << 64) | q.pcg_state[0];
    unsigned long long c_req = 0, c_ex = 0, c_fb = 0, c_ms = 0;
    __syncthreads();
    // PCG64 state after the R.draws draws consumed so far (draw x = out(state after x+1 steps))
    u128 SD = pcg_jump16(s0, R.draws, sm.j16);

    auto ray_o = [&](int r, double& x, double& y, double& z) {
        if (wk.o_stride) {
            x = __ldcg(wk.o + 3 * r);
            y = __ldcg(wk.o + 3 * r + 1);
            z = __ldcg(wk.o + 3 * r + 2);
        } else {
            x = wk.oc[0];
            y = wk.oc[1];
            z = wk.oc[2];
        }
    };
    auto ray_d = [&](int r, double& x, double& y, double& z) {
        if (wk.d_stride) {
            x = __ldcg(wk.d + 3 * r);
            y = __ldcg(wk.d + 3 * r + 1);
            z = __ldcg(wk.d + 3 * r + 2);
        } else {
            x = wk.dc[0];
            y = wk.dc[1];
            z = wk.dc[2];
        }
    };
    int* cnt0 = s.cnt;
    int* cnt1 = s.cnt + kPtMaxCtas;
    int* cnt2 = s.cnt + 2 * kPtMaxCtas;

    // ---- init: walking = t < t_end (line 48), ordered list of walking rays
    const long long n = wk.n_dev ? (long long)__ldcg(wk.n_dev) : wk.n_const;
    long long lo, hi;
    pt_chunk(n, lo, hi);
    {
        int cnt = 0;
        for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const double t0 = wk.t0_stride ? __ldcg(wk.t0 + i) : wk.t0c;
            T[i] = t0;
            TH[i] = INFINITY;
            VH[i] = 0.0f;
            cnt += t0 < __ldcg(wk.tend + i);
        }
        cnt = warp_sum(cnt);
        if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(cnt0 + blockIdx.x, cnt);
    }
    pt_barrier(s.bar, target);
    long long pre, m;
    pt_cta_prefix(cnt0, sm.red, pre, m);
    for (long long b0 = lo; b0 < hi; b0 += blockDim.x) {
        const long long i = b0 + threadIdx.x;
        bool f = false;
        if (i < hi) f = __ldcg(T + i) < __ldcg(wk.tend + i);
        int tot;
        const int r = pt_block_rank(f, sm.w, tot);
        if (f) s.list[0][pre + r] = (int)i;
        pre += tot;
    }
    long long k = 0;
    for (; k < q.max_walk && m > 0; k++) {
        const int* in = s.list[k & 1];
        int* out = s.list[(k + 1) & 1];
        uint8_t* FLc = (k & 1) ? s.flag2 : s.flag;  // flags of list k / list k+1
        uint8_t* FLn = (k & 1) ? s.flag : s.flag2;
        pt_barrier(s.bar, target);  // list k, its flags and dense counts complete
        pt_chunk(m, lo, hi);
        // phase 1: classify (54-75); from iteration 1 on the compaction of the previous
        // iteration has classified every survivor already
        if (k == 0) {
            int cnt = 0;
            for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const int r = __ldcg(in + i);
                double ox, oy, oz, dx, dy, dz;
                ray_o(r, ox, oy, oz);
                ray_d(r, dx, dy, dz);
                const double t = __ldcg(T + r), te = __ldcg(wk.tend + r);
                const PtGeo g = pt_geo(p, dens_f, ox, oy, oz, dx, dy, dz, t, te, MUG);
                uint8_t cls = 0;
                if (!g.outside) {
                    if (g.mu <= 0.0f) {
                        if (!g.at_end) {
                            __stcg(T + r, DADD(g.exit_t, 1e-9));
                            cls = 1;
                        }
                    } else {
                        // dense: keep mu, the cell exit and at_end for the draw phase
                        __stcg(s.mub + i, g.mu);
                        __stcg(s.exitb + i, g.exit_t);
                        cls = g.at_end ? 4 : 2;
                        cnt++;
                    }
                }
                __stcg(FLc + i, cls);
            }
            cnt = warp_sum(cnt);
            if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(cnt1 + blockIdx.x, cnt);
            if (threadIdx.x == 0) cnt0[blockIdx.x] = 0;
            pt_barrier(s.bar, target);
        } else if (threadIdx.x == 0) {
            cnt0[blockIdx.x] = 0;  // survivor counts of iteration k-1 were consumed before the barrier
        }
        long long pre_d, n_dense;
        pt_cta_prefix(cnt1, sm.red, pre_d, n_dense);
        // phase 2: free-flight draws of the dense rays (77-88)
        {
            int cnt = 0;
            u128 Sr = pcg_jump16(SD, (u64)pre_d, sm.j16);  // state before this round's first draw
            for (long long b0 = lo; b0 < hi; b0 += blockDim.x) {
                const long long i = b0 + threadIdx.x;
                uint8_t cls = 0;
                int r = 0;
                if (i < hi) {
                    cls = __ldcg(FLc + i);
                    r = __ldcg(in + i);
                }
                const bool dense = cls == 2 || cls == 4;
                int tot;
                const int rk = pt_block_rank(dense, sm.w, tot);
                if (dense) {
                    const double t = __ldcg(T + r);
                    const float mu = __ldcg(s.mub + i);
                    const double exit_t = __ldcg(s.exitb + i);
                    const double xi = pcg_out(pcg_jump16(Sr, (u64)rk + 1, sm.j16));
                    const double tc = DSUB(t, __ddiv_rn(pt_log1p(-xi), (double)mu));
                    if (tc >= exit_t) {
                        if (cls == 4) {
                            cls = 0;
                        } else {
                            __stcg(T + r, DADD(exit_t, 1e-9));
                            cls = 1;
                        }
                    } else {
                        __stcg(T + r, tc);
                        cls = 3;
                        cnt++;
                    }
                    __stcg(FLc + i, cls);
                }
                pre_d += tot;
            Sr = pcg_jump16(Sr, (u64)tot, sm.j16);
            }
            cnt = warp_sum(cnt);
            if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(cnt2 + blockIdx.x, cnt);
        }
        pt_barrier(s.bar, target);
        long long pre_s, n_set;
        pt_cta_prefix(cnt2, sm.red, pre_s, n_set);
        if (threadIdx.x == 0) cnt1[blockIdx.x] = 0;
        // VolumeSampler.sample lane pool (sampler.py:206-213)
        if (n_set > 0) {
            if (R.pool == 0) {
                R.pool = n_set;
                R.salt = 0;
                R.gen += 1;
                R.base = splitmix64((u64)q.lane_seed ^ ((u64)q.lane_frame * 0x9E3779B97F4A7C15ull));
            } else if (R.pool < n_set) {
                R.salt += 1;
                R.pool = n_set;
                R.gen += 1;
                const u64 fr = (u64)q.lane_frame * 1000003ull + (u64)R.salt;
                R.base = splitmix64((u64)q.lane_seed ^ (fr * 0x9E3779B97F4A7C15ull));
            }
        }
        // phase 3: sample the settled rays, accept or reject (89-97)
        {
            int cnt = 0;
            u128 Sr = pcg_jump16(SD, (u64)(n_dense + pre_s), sm.j16);
            for (long long b0 = lo; b0 < hi; b0 += blockDim.x) {
                const long long i = b0 + threadIdx.x;
                uint8_t cls = 0;
                int r = 0;
                if (i < hi) {
                    cls = __ldcg(FLc + i);
                    r = __ldcg(in + i);
                }
                int tot;
                const int rk = pt_block_rank(cls == 3, sm.w, tot);
                if (cls == 3) {
                    double ox, oy, oz, dx, dy, dz;
                    ray_o(r, ox, oy, oz);
                    ray_d(r, dx, dy, dz);
                    const double t = __ldcg(T + r);
                    const double px = DADD(ox, DMUL(dx, t)), py = DADD(oy, DMUL(dy, t)), pz = DADD(oz, DMUL(dz, t));
                    c_req++;
                    const float v = pt_sample<kInr>(p, s, R, mlp, pre_s + rk, px, py, pz, c_ex, c_fb, c_ms);
                    // sigma = tf.opacity(values) * pt_density; accept = xi < sigma / mu
                    const double vv = clampd((double)v, 0.0, 1.0);
                    const double sig = DMUL(np_interp(vv, sm.tf, sm.tf + 4, q.n_tf, 5), q.density);
                    const double xi = pcg_out(pcg_jump16(Sr, (u64)rk + 1, sm.j16));
                    if (xi < __ddiv_rn(sig, (double)__ldcg(s.mub + i))) {
                        __stcg(TH + r, t);
                        __stcg(VH + r, v);
                        cls = 0;
                    } else {
                        cls = 1;
                    }
                }
                if (cls == 1) cls = __ldcg(T + r) < __ldcg(wk.tend + r) ? 1 : 0;  // walking &= t < t_end
                if (i < hi) __stcg(FLc + i, cls);
                cnt += cls;
                pre_s += tot;
                Sr = pcg_jump16(Sr, (u64)tot, sm.j16);
            }
            cnt = warp_sum(cnt);
            if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(cnt0 + blockIdx.x, cnt);
        }
        R.draws += (u64)(n_dense + n_set);
        SD = pcg_jump16(SD, (u64)(n_dense + n_set), sm.j16);
        pt_barrier(s.bar, target);
        long long pre_v, m_next;
        pt_cta_prefix(cnt0, sm.red, pre_v, m_next);
        if (threadIdx.x == 0) cnt2[blockIdx.x] = 0;
        // phase 4: ordered compaction of the walking rays, fused with their classification
        // for iteration k+1 (a ray retired by it keeps its slot with flag 0 and leaves at the
        // next compaction); dense counts go to the CTA that owns the slot in iteration k+1
        const long long ch_next = (m_next + gridDim.x - 1) / gridDim.x;
        for (long long b0 = lo; b0 < hi; b0 += blockDim.x) {
            const long long i = b0 + threadIdx.x;
            bool f = false;
            if (i < hi) f = __ldcg(FLc + i) != 0;
            int tot;
            const int rk = pt_block_rank(f, sm.w, tot);
            if (f) {
                const long long dst = pre_v + rk;
                const int r = __ldcg(in + i);
                __stcg(out + dst, r);
                double ox, oy, oz, dx, dy, dz;
                ray_o(r, ox, oy, oz);
                ray_d(r, dx, dy, dz);
                const double t = __ldcg(T + r), te = __ldcg(wk.tend + r);
                const PtGeo g = pt_geo(p, dens_f, ox, oy, oz, dx, dy, dz, t, te, MUG);
                uint8_t cls = 0;
                if (!g.outside) {
                    if (g.mu <= 0.0f) {
                        if (!g.at_end) {
                            __stcg(T + r, DADD(g.exit_t, 1e-9));
                            cls = 1;
                        }
                    } else {
                        __stcg(s.mub + dst, g.mu);
                        __stcg(s.exitb + dst, g.exit_t);
                        cls = g.at_end ? 4 : 2;
                        warp_aggregated_add(cnt1, dst / ch_next);
                    }
                }
                __stcg(FLn + dst, cls);
            }
            pre_v += tot;
        }
        m = m_next;
    }
    R.iters += k;
    // stats
    c_req = warp_sum(c_req);
    c_ex = warp_sum(c_ex);
    c_fb = warp_sum(c_fb);
    c_ms = warp_sum(c_ms);
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* st = reinterpret_cast<unsigned long long*>(p.stats);
        if (c_req) atomicAdd(st + 0, c_req);
        if (c_ex) atomicAdd(st + 1, c_ex);
        if (c_fb) atomicAdd(st + 2, c_fb);
        if (c_ms) atomicAdd(st + 3, c_ms);
    }
    if (W == 0) {
        // shadow rays of the hits, in ray order (pathtrace.py:132-138, 101-108)
        pt_barrier(s.bar, target);
        pt_chunk(n, lo, hi);
        {
            // cnt2 is zero here: reset after the last iteration's third barrier, unused since
            int cnt = 0;
            for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) cnt += isfinite(__ldcg(TH + i)) ? 1 : 0;
            cnt = warp_sum(cnt);
            if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(cnt2 + blockIdx.x, cnt);
        }
        pt_barrier(s.bar, target);
        long long pre_h, n_h;
        pt_cta_prefix(cnt2, sm.red, pre_h, n_h);
        for (long long b0 = lo; b0 < hi; b0 += blockDim.x) {
            const long long i = b0 + threadIdx.x;
            double th = INFINITY;
            if (i < hi) th = __ldcg(TH + i);
            const bool f = isfinite(th);
            int tot;
            const int rk = pt_block_rank(f, sm.w, tot);
            if (i < hi) s.sh_of[i] = f ? (int)(pre_h + rk) : -1;
            if (f) pt_shadow_ray(q, s, pre_h + rk, (int)i, th, ray_o, ray_d);
            pre_h += tot;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) s.rng->sh_n = (int)n_h;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s.rng->draws = R.draws;
        s.rng->pool = R.pool;
        s.rng->salt = R.salt;
        s.rng->gen = R.gen;
        s.rng->base = R.base;
        s.rng->iters = R.iters;
    }
}


__device__ __forceinline__ int pt_block_sum(int v, int* s_w) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = 0;
    for (int w = 0; w < kPtThreads / 32; w++) t += s_w[w];
    __syncthreads();
    return t;
}

// Two grid barriers per wavefront iteration (walk schedule 1).  Each CTA owns a
// contiguous range of the walk's rays for the whole walk and keeps the ones still
// walking in its own segment of the list, in ray order, so the global order is CTA
// order then list order and a rank is (counts of the CTAs before) + (block rank).
//   barrier A: dense counts of this iteration published
//   draws:     free flights of the dense rays (draw D + dense rank)
//   barrier B: settled counts published
//   sample:    settled rays sampled + accepted (lane = settled rank, draw D + n_dense +
//              settled rank); then, fused, walking &= t < t_end, the in-place compaction
//              of the CTA's list and the classification of the next iteration (outside,
//              majorant, cell exit; empty cells hop), whose dense count is published
// Rays that the next classification retires (outside / escaping an empty cell) leave
// the list one iteration early; they draw nothing, so every draw, lane and value is
// the reference's.
template <int kInr>
__global__ void __launch_bounds__(kPtThreads, 1)
    k_pt_walk2(VcbFrameParams p, VcbPtParams q, FrameWs fw, PtWs s, PtWalk wk) {
    __shared__ PtSmem sm;
    extern __shared__ __align__(16) float smem[];
    MlpSmem mlp;
    if (kInr != 0) stage_mlp(p.field, smem, mlp);
    for (int i = threadIdx.x; i < q.n_tf * 5; i += blockDim.x) sm.tf[i] = q.tf[i];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sm.j16[i] = s.j16[i];
    unsigned target = 0;
    const int W = wk.which;
    double* T = s.t[W];
    double* TH = s.thit[W];
    float* VH = s.vhit[W];
    const float dens_f = __double2float_rn(q.density);
    PtRng R = *s.rng;
    const u128 s0 = ((u128)q.pcg_state[1] << 64) | q.pcg_state[0];
    unsigned long long c_req = 0, c_ex = 0, c_fb = 0, c_ms = 0;
    __syncthreads();
    // PCG64 state after the R.draws draws consumed so far (draw x = out(state after x+1 steps))
    u128 SD = pcg_jump16(s0, R.draws, sm.j16);
    auto ray_o = [&](int r, double& x, double& y, double& z) {
        if (wk.o_stride) {
            x = __ldcg(wk.o + 3 * r);
            y = __ldcg(wk.o + 3 * r + 1);
            z = __ldcg(wk.o + 3 * r + 2);
        } else {
            x = wk.oc[0];
            y = wk.oc[1];
            z = wk.oc[2];
        }
    };
    auto ray_d = [&](int r, double& x, double& y, double& z) {
        if (wk.d_stride) {
            x = __ldcg(wk.d + 3 * r);
            y = __ldcg(wk.d + 3 * r + 1);
            z = __ldcg(wk.d + 3 * r + 2);
        } else {
            x = wk.dc[0];
            y = wk.dc[1];
            z = wk.dc[2];
        }
    };
    // pathtrace.py:54-75 for ray r at parameter t: 0 retired, 1 hopped (t moved), 2 dense
    auto classify = [&](int r, double t) -> uint8_t {
        double ox, oy, oz, dx, dy, dz;
        ray_o(r, ox, oy, oz);
        ray_d(r, dx, dy, dz);
        const PtGeo g = pt_geo(p, dens_f, ox, oy, oz, dx, dy, dz, t, __ldcg(wk.tend + r));
        if (g.outside) return 0;
        if (g.mu > 0.0f) return 2;
        if (g.at_end) return 0;
        __stcg(T + r, DADD(g.exit_t, 1e-9));
        return 1;
    };
    int* cntD = s.cnt;
    int* cntS = s.cnt + kPtMaxCtas;
    int* cntL = s.cnt + 2 * kPtMaxCtas;
    int* cntH = s.cnt + 3 * kPtMaxCtas;
    const long long n = wk.n_dev ? (long long)__ldcg(wk.n_dev) : wk.n_const;
    long long own_lo, own_hi;
    pt_chunk(n, own_lo, own_hi);
    int cur = 0;  // list / flag buffer generation (flips on a rebalance)
    int* L = s.list[0] + own_lo;
    uint8_t* FL = s.flag + own_lo;
    float* MU = s.mub + own_lo;
    // init (line 44-48) + classification of iteration 0
    long long len = 0;
    int nd = 0;
    for (long long b0 = own_lo; b0 < own_hi; b0 += blockDim.x) {
        const long long i = b0 + threadIdx.x;
        uint8_t cls = 0;
        if (i < own_hi) {
            const double t0 = wk.t0_stride ? __ldcg(wk.t0 + i) : wk.t0c;
            __stcg(T + i, t0);
            __stcg(TH + i, (double)INFINITY);
            __stcg(VH + i, 0.0f);
            if (t0 < __ldcg(wk.tend + i)) cls = classify((int)i, t0);
        }
        int tot;
        const int rk = pt_block_rank(cls != 0, sm.w, tot);
        if (cls) {
            __stcg(L + len + rk, (int)i);
            __stcg(FL + len + rk, cls);
        }
        nd += cls == 2;
        len += tot;
    }
    nd = pt_block_sum(nd, sm.w);
    if (threadIdx.x == 0) {
        cntD[blockIdx.x] = nd;
        cntL[blockIdx.x] = (int)len;
    }
    long long k = 0;
    for (;; k++) {
        pt_barrier(s.bar, target);  // A
        long long pre_d, n_dense, pre_l, m, maxl;
        pt_cta_prefix(cntD, sm.red, pre_d, n_dense);
        pt_cta_prefix_max(cntL, sm.red, pre_l, m, maxl);
        if (m == 0 || k >= q.max_walk) break;
        const long long ch = (m + gridDim.x - 1) / gridDim.x;
        if ((maxl + kPtThreads - 1) / kPtThreads > (ch + kPtThreads - 1) / kPtThreads) {
            // rebalance: the lists, concatenated in CTA order (= ray order), re-split evenly
            int* Lb = s.list[cur ^ 1];
            uint8_t* FLb = cur ? s.flag : s.flag2;
            for (long long j = threadIdx.x; j < len; j += blockDim.x) {
                __stcg(Lb + pre_l + j, __ldcg(L + j));
                __stcg(FLb + pre_l + j, __ldcg(FL + j));
            }
            pt_barrier(s.bar, target);
            cur ^= 1;
            long long lo2 = (long long)blockIdx.x * ch;
            if (lo2 > m) lo2 = m;
            long long hi2 = lo2 + ch;
            if (hi2 > m) hi2 = m;
            L = Lb + lo2;
            FL = FLb + lo2;
            MU = s.mub + lo2;
            len = hi2 - lo2;
            int nd2 = 0;
            for (long long j = threadIdx.x; j < len; j += blockDim.x) nd2 += __ldcg(FL + j) == 2;
            nd2 = pt_block_sum(nd2, sm.w);
            if (threadIdx.x == 0) cntD[blockIdx.x] = nd2;
            pt_barrier(s.bar, target);
            pt_cta_prefix(cntD, sm.red, pre_d, n_dense);
        }
        // free flights of the dense rays (77-88)
        int ns = 0;
        u128 Sr = pcg_jump16(SD, (u64)pre_d, sm.j16);  // state before this round's first draw
        for (long long b0 = 0; b0 < len; b0 += blockDim.x) {
            const long long j = b0 + threadIdx.x;
            uint8_t cls = 0;
            int r = 0;
            if (j < len) {
                cls = __ldcg(FL + j);
                r = __ldcg(L + j);
            }
            int tot;
            const int rk = pt_block_rank(cls == 2, sm.w, tot);
            if (cls == 2) {
                double ox, oy, oz, dx, dy, dz;
                ray_o(r, ox, oy, oz);
                ray_d(r, dx, dy, dz);
                const double t = __ldcg(T + r), te = __ldcg(wk.tend + r);
                const PtGeo g = pt_geo(p, dens_f, ox, oy, oz, dx, dy, dz, t, te);
                const double xi = pcg_out(pcg_jump16(Sr, (u64)rk + 1, sm.j16));
                const double tc = DSUB(t, __ddiv_rn(pt_log1p(-xi), (double)g.mu));
                if (tc >= g.exit_t) {
                    if (g.at_end) {
                        cls = 0;
                    } else {
                        __stcg(T + r, DADD(g.exit_t, 1e-9));
                        cls = 1;
                    }
                } else {
                    __stcg(T + r, tc);
                    __stcg(MU + j, g.mu);
                    cls = 3;
                    ns++;
                }
                __stcg(FL + j, cls);
            }
            pre_d += tot;
            Sr = pcg_jump16(Sr, (u64)tot, sm.j16);
        }
        ns = pt_block_sum(ns, sm.w);
        if (threadIdx.x == 0) cntS[blockIdx.x] = ns;
        pt_barrier(s.bar, target);  // B
        long long pre_s, n_set;
        pt_cta_prefix(cntS, sm.red, pre_s, n_set);
        // VolumeSampler.sample lane pool (sampler.py:206-213)
        if (n_set > 0) {
            if (R.pool == 0) {
                R.pool = n_set;
                R.salt = 0;
                R.gen += 1;
                R.base = splitmix64((u64)q.lane_seed ^ ((u64)q.lane_frame * 0x9E3779B97F4A7C15ull));
            } else if (R.pool < n_set) {
                R.salt += 1;
                R.pool = n_set;
                R.gen += 1;
                const u64 fr = (u64)q.lane_frame * 1000003ull + (u64)R.salt;
                R.base = splitmix64((u64)q.lane_seed ^ (fr * 0x9E3779B97F4A7C15ull));
            }
        }
        // sample + accept (89-97), walking &= t < t_end, compaction, next classification
        long long new_len = 0;
        Sr = pcg_jump16(SD, (u64)(n_dense + pre_s), sm.j16);
        nd = 0;
        for (long long b0 = 0; b0 < len; b0 += blockDim.x) {
            const long long j = b0 + threadIdx.x;
            uint8_t cls = 0;
            int r = 0;
            if (j < len) {
                cls = __ldcg(FL + j);
                r = __ldcg(L + j);
            }
            int tot;
            const int rk = pt_block_rank(cls == 3, sm.w, tot);
            if (cls == 3) {
                double ox, oy, oz, dx, dy, dz;
                ray_o(r, ox, oy, oz);
                ray_d(r, dx, dy, dz);
                const double t = __ldcg(T + r);
                const double px = DADD(ox, DMUL(dx, t)), py = DADD(oy, DMUL(dy, t)), pz = DADD(oz, DMUL(dz, t));
                c_req++;
                const float v = pt_sample<kInr>(p, s, R, mlp, pre_s + rk, px, py, pz, c_ex, c_fb, c_ms);
                const double vv = clampd((double)v, 0.0, 1.0);
                const double sig = DMUL(np_interp(vv, sm.tf, sm.tf + 4, q.n_tf, 5), q.density);
                const double xi = pcg_out(pcg_jump16(Sr, (u64)rk + 1, sm.j16));
                if (xi < __ddiv_rn(sig, (double)__ldcg(MU + j))) {
                    __stcg(TH + r, t);
                    __stcg(VH + r, v);
                    cls = 0;
                } else {
                    cls = 1;
                }
            }
            uint8_t nc = 0;
            if (cls == 1) {
                const double t = __ldcg(T + r);
                if (t < __ldcg(wk.tend + r)) nc = classify(r, t);
            }
            int tot2;
            const int rk2 = pt_block_rank(nc != 0, sm.w, tot2);  // all reads of L/FL/MU above precede it
            if (nc) {
                __stcg(L + new_len + rk2, r);
                __stcg(FL + new_len + rk2, nc);
            }
            nd += nc == 2;
            new_len += tot2;
            pre_s += tot;
            Sr = pcg_jump16(Sr, (u64)tot, sm.j16);
        }
        R.draws += (u64)(n_dense + n_set);
        SD = pcg_jump16(SD, (u64)(n_dense + n_set), sm.j16);
        len = new_len;
        nd = pt_block_sum(nd, sm.w);
        if (threadIdx.x == 0) {
            cntD[blockIdx.x] = nd;
            cntL[blockIdx.x] = (int)len;
        }
    }
    R.iters += k;
    c_req = warp_sum(c_req);
    c_ex = warp_sum(c_ex);
    c_fb = warp_sum(c_fb);
    c_ms = warp_sum(c_ms);
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* st = reinterpret_cast<unsigned long long*>(p.stats);
        if (c_req) atomicAdd(st + 0, c_req);
        if (c_ex) atomicAdd(st + 1, c_ex);
        if (c_fb) atomicAdd(st + 2, c_fb);
        if (c_ms) atomicAdd(st + 3, c_ms);
    }
    if (W == 0) {
        // shadow rays of the hits, in ray order (pathtrace.py:132-138, 101-108)
        int nh = 0;
        for (long long i = own_lo + threadIdx.x; i < own_hi; i += blockDim.x) nh += isfinite(__ldcg(TH + i)) ? 1 : 0;
        nh = pt_block_sum(nh, sm.w);
        if (threadIdx.x == 0) cntH[blockIdx.x] = nh;
        pt_barrier(s.bar, target);
        long long pre_h, n_h;
        pt_cta_prefix(cntH, sm.red, pre_h, n_h);
        for (long long b0 = own_lo; b0 < own_hi; b0 += blockDim.x) {
            const long long i = b0 + threadIdx.x;
            double th = INFINITY;
            if (i < own_hi) th = __ldcg(TH + i);
            const bool f = isfinite(th);
            int tot;
            const int rk = pt_block_rank(f, sm.w, tot);
            if (i < own_hi) s.sh_of[i] = f ? (int)(pre_h + rk) : -1;
            if (f) pt_shadow_ray(q, s, pre_h + rk, (int)i, th, ray_o, ray_d);
            pre_h += tot;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) s.rng->sh_n = (int)n_h;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s.rng->draws = R.draws;
        s.rng->pool = R.pool;
        s.rng->salt = R.salt;
        s.rng->gen = R.gen;
        s.rng->base = R.base;
        s.rng->iters = R.iters;
    }
}

// PCG jump table + per-frame state (pathtrace.py:117 seeding happened on the host)
__global__ void k_pt_init(VcbPtParams q, PtWs s) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    u128 m = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    u128 c = ((u128)q.pcg_inc[1] << 64) | q.pcg_inc[0];
    for (int j = 0; j < 64; j++) {
        s.jump[j].m_lo = (u64)m;
        s.jump[j].m_hi = (u64)(m >> 64);
        s.jump[j].p_lo = (u64)c;
        s.jump[j].p_hi = (u64)(c >> 64);
        c = (m + 1) * c;
        m = m * m;
    }
    // radix-16 table: step = jump by 16^d; entry v = step composed v times
    u128 sm_ = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    u128 sc_ = ((u128)q.pcg_inc[1] << 64) | q.pcg_inc[0];
    for (int d = 0; d < 16; d++) {
        u128 em = 1, ec = 0;
        for (int v = 0; v < 16; v++) {
            s.j16[d * 16 + v] = PtJump{(u64)em, (u64)(em >> 64), (u64)ec, (u64)(ec >> 64)};
            // (em, ec) then one more step (sm_, sc_): s -> sm_ (em s + ec) + sc_
            ec = sm_ * ec + sc_;
            em = sm_ * em;
        }
        sm_ = em;  // 16 steps of the old step = the next digit's step
        sc_ = ec;
    }
    PtRng r = {};
    *s.rng = r;
}

// pathtrace.py:132-142: one sample's color per bundle ray, summed in f64
__global__ void k_pt_accumulate(VcbFrameParams p, VcbPtParams q, FrameWs fw, PtWs s) {
    __shared__ double tf[kPtMaxTf * 5];
    for (int i = threadIdx.x; i < q.n_tf * 5; i += blockDim.x) tf[i] = q.tf[i];
    __syncthreads();
    const int n = *fw.live;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double th = s.thit[0][i];
        double r = p.bg[0], g = p.bg[1], b = p.bg[2];
        if (isfinite(th)) {
            const int j = s.sh_of[i];
            const double vis = isinf(s.thit[1][j]) ? 1.0 : 0.0;
            const double shade = DADD(q.ambient, DMUL(DSUB(1.0, q.ambient), vis));
            const double v = clampd((double)s.vhit[0][i], 0.0, 1.0);
            r = DMUL(np_interp(v, tf, tf + 1, q.n_tf, 5), shade);
            g = DMUL(np_interp(v, tf, tf + 2, q.n_tf, 5), shade);
            b = DMUL(np_interp(v, tf, tf + 3, q.n_tf, 5), shade);
            s.hits[i] = DADD(s.hits[i], 1.0);
        }
        s.total[3 * i] = DADD(s.total[3 * i], r);
        s.total[3 * i + 1] = DADD(s.total[3 * i + 1], g);
        s.total[3 * i + 2] = DADD(s.total[3 * i + 2], b);
    }
}

// pathtrace.py:143-146
__global__ void k_pt_finalize(VcbFrameParams p, VcbPtParams q, FrameWs fw, PtWs s) {
    const int n = *fw.live;
    const double spp = (double)q.spp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float4 o;
        o.x = __double2float_rn(__ddiv_rn(s.total[3 * i], spp));
        o.y = __double2float_rn(__ddiv_rn(s.total[3 * i + 1], spp));
        o.z = __double2float_rn(__ddiv_rn(s.total[3 * i + 2], spp));
        o.w = __double2float_rn(__ddiv_rn(s.hits[i], spp));
        reinterpret_cast<float4*>(p.image)[frame_pixel(p, fw.ray_pix[i])] = o;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.stats->rays = n;
        p.stats->iterations = s.rng->iters;
        p.stats->nonfinite = s.rng->nonfinite;
    }
}

__global__ void k_pt_walk_stats(VcbFrameParams p, PtWs s) {
    p.stats->iterations = s.rng->iters;
    p.stats->nonfinite = s.rng->nonfinite;
}

// diagnostics: log1p(x[i]) and the uniform of PCG64 draw idx[i] of the stream at pcg
__global__ void k_pt_debug_math(int64_t n, const double* x, double* lg, u64 s_lo, u64 s_hi, u64 i_lo, u64 i_hi,
                                const u64* idx, double* uni) {
    __shared__ PtJump J[64];
    if (threadIdx.x == 0) {
        u128 m = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
        u128 c = ((u128)i_hi << 64) | i_lo;
        for (int j = 0; j < 64; j++) {
            J[j] = PtJump{(u64)m, (u64)(m >> 64), (u64)c, (u64)(c >> 64)};
            c = (m + 1) * c;
            m = m * m;
        }
    }
    __syncthreads();
    const u128 s0 = ((u128)s_hi << 64) | s_lo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        lg[i] = pt_log1p(x[i]);
        uni[i] = pcg_uniform_at(s0, idx[i], J);
    }
}

void launch_rays(const VcbFrameParams& p, const FrameWs& w, cudaStream_t st);
extern thread_local long long g_launches;

// walk schedule: 0 (default) three barriers per iteration with the active list re-split
// evenly every iteration; 1 two barriers per iteration with per-CTA ray ownership and
// rebalancing on demand (bit-identical, ~5% slower: the imbalance costs more than the
// two barriers it saves)
static const void* pt_kernel(int mode, int impl) {
    if (impl == 1) {
        if (mode == 1) return (const void*)k_pt_walk2<1>;
        if (mode == 2) return (const void*)k_pt_walk2<2>;
        return (const void*)k_pt_walk2<0>;
    }
    if (mode == 1) return (const void*)k_pt_walk<1>;
    if (mode == 2) return (const void*)k_pt_walk<2>;
    return (const void*)k_pt_walk<0>;
}

}  // namespace cinr

using namespace cinr;

extern "C" int64_t vcb_pt_workspace_bytes(int64_t max_rays) { return pt_ws_layout(max_rays, nullptr, nullptr); }

// trace_free_flight (pathtrace.py:28-98) on caller rays: one walk, results copied out.
extern "C" int32_t vcb_trace_free_flight(const VcbFrameParams* pp, const VcbPtParams* qq, int64_t n, const double* o,
                                         const double* d, const double* t0, const double* t1, double* t_hit,
                                         float* v_hit, uint64_t* draws, void* stream_) {
    const VcbFrameParams& p = *pp;
    const VcbPtParams& q = *qq;
    cudaStream_t st = (cudaStream_t)stream_;
    if (n < 0 || n > 0x7fffffff) return set_error("trace_free_flight: %lld rays", (long long)n);
    if (q.n_tf < 2 || q.n_tf > kPtMaxTf) return set_error("trace_free_flight: %d transfer-function points", q.n_tf);
    PtWs s;
    const int64_t need = pt_ws_layout(n, q.workspace, &s);
    if (need > q.workspace_bytes)
        return set_error("trace_free_flight: workspace too small (%lld < %lld)", (long long)q.workspace_bytes,
                         (long long)need);
    const int mode = inr_mode(p.field);
    const void* fn = pt_kernel(mode, p.impl == 1 ? 1 : 0);
    int smem = 0;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        smem = (nw + nb) * 4;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int G = device_sms();
    if (G > kPtMaxCtas) G = kPtMaxCtas;
    if (n > 0) cudaMemsetAsync(s.lane, 0xFF, (size_t)n * 8, st);
    cudaMemsetAsync(s.cnt, 0, (size_t)4 * kPtMaxCtas * 4, st);
    cudaMemsetAsync(s.bar, 0, 64, st);
    k_pt_init<<<1, 32, 0, st>>>(q, s);
    PtWalk wk = {};
    wk.n_const = n;
    wk.o = o;
    wk.o_stride = 3;
    wk.d = d;
    wk.d_stride = 3;
    wk.t0 = t0;
    wk.t0_stride = 1;
    wk.tend = t1;
    wk.which = 1;
    VcbFrameParams pc = p;
    VcbPtParams qc = q;
    FrameWs wc = {};
    PtWs sc = s;
    void* args[5] = {&pc, &qc, &wc, &sc, &wk};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, G, kPtThreads, args, smem, st);
    if (e != cudaSuccess)
        return set_error("trace_free_flight: cooperative launch (%d CTAs): %s", G, cudaGetErrorString(e));
    k_pt_walk_stats<<<1, 1, 0, st>>>(p, s);
    if (n > 0) {
        cudaMemcpyAsync(t_hit, s.thit[1], (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(v_hit, s.vhit[1], (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
    }
    unsigned long long dr = 0;
    cudaMemcpyAsync(&dr, &s.rng->draws, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e2 != cudaSuccess) return set_error("trace_free_flight: %s", cudaGetErrorString(e2));
    if (draws) *draws = dr;
    g_launches = 2;
    return check_launch("trace_free_flight");
}

extern "C" int32_t vcb_debug_pt_math(int64_t n, const double* x, double* log1p_out, const uint64_t* pcg,
                                     const uint64_t* draw_idx, double* uniform_out, void* stream) {
    if (n <= 0) return 0;
    k_pt_debug_math<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x, log1p_out, pcg[0], pcg[1], pcg[2], pcg[3],
                                                                         (const u64*)draw_idx, uniform_out);
    return check_launch("debug_pt_math");
}

extern "C" int32_t vcb_pathtrace_frame(const VcbFrameParams* pp, const VcbPtParams* qq, void* stream_) {
    const VcbFrameParams& p = *pp;
    const VcbPtParams& q = *qq;
    cudaStream_t st = (cudaStream_t)stream_;
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    if (npix == 0) return 0;
    if (q.n_tf < 2 || q.n_tf > kPtMaxTf) return set_error("pathtrace_frame: %d transfer-function points", q.n_tf);
    if (q.spp < 1) return set_error("pathtrace_frame: samples_per_pixel %d", q.spp);
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    FrameWs w;
    const int64_t need = frame_ws_layout(npix, max_it, p.workspace, &w);
    if (need > p.workspace_bytes)
        return set_error("pathtrace_frame: frame workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)need);
    PtWs s;
    const int64_t need2 = pt_ws_layout(npix, q.workspace, &s);
    if (need2 > q.workspace_bytes)
        return set_error("pathtrace_frame: workspace too small (%lld < %lld)", (long long)q.workspace_bytes,
                         (long long)need2);
    const int mode = inr_mode(p.field);
    const void* fn = pt_kernel(mode, p.impl == 1 ? 1 : 0);
    int smem = 0;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        smem = (nw + nb) * 4;
    }
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    const int mu_off = (smem / 4 + 3) & ~3;
    const bool mu_smem = p.impl != 1 && (long long)mu_off * 4 + cells * 4 <= 200 * 1024;
    if (mu_smem) smem = mu_off * 4 + (int)cells * 4;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPtThreads, smem);
    if (per_sm < 1) return set_error("pathtrace_frame: walk kernel does not fit one CTA per SM");
    int G = device_sms();
    if (G > kPtMaxCtas) G = kPtMaxCtas;
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(w.ctr_iter, 0, w.ctr_iter_bytes, st);
    cudaMemsetAsync(s.lane, 0xFF, (size_t)npix * 8, st);
    cudaMemsetAsync(s.total, 0, (size_t)npix * 24, st);
    cudaMemsetAsync(s.hits, 0, (size_t)npix * 8, st);
    cudaMemsetAsync(s.cnt, 0, (size_t)4 * kPtMaxCtas * 4, st);
    k_pt_init<<<1, 32, 0, st>>>(q, s);
    launch_rays(p, w, st);
    long long launches = 3;
    PtWalk prim = {};
    prim.n_dev = w.live;
    prim.d = w.ray_dir;
    prim.d_stride = 3;
    prim.o_stride = 0;
    for (int a = 0; a < 3; a++) prim.oc[a] = p.cam.origin[a];
    prim.t0 = w.ray_ten;
    prim.t0_stride = 1;
    prim.tend = w.ray_tex;
    prim.which = 0;
    prim.mu_smem = mu_smem ? 1 : 0;
    prim.mu_off = mu_off;
    PtWalk shad = {};
    shad.n_dev = &s.rng->sh_n;
    shad.o = s.sh_o;
    shad.o_stride = 3;
    shad.d_stride = 0;
    for (int a = 0; a < 3; a++) shad.dc[a] = q.light[a];
    shad.t0c = 1e-6;
    shad.t0_stride = 0;
    shad.tend = s.sh_tend;
    shad.which = 1;
    shad.mu_smem = mu_smem ? 1 : 0;
    shad.mu_off = mu_off;
    VcbFrameParams pc = p;
    VcbPtParams qc = q;
    FrameWs wc = w;
    PtWs sc = s;
    const int grid_acc = grid_for(npix, 256);
    for (int k = 0; k < q.spp; k++) {
        for (int walk = 0; walk < 2; walk++) {
            PtWalk wk = walk == 0 ? prim : shad;
            cudaMemsetAsync(s.bar, 0, 64, st);
            cudaMemsetAsync(s.cnt, 0, (size_t)4 * kPtMaxCtas * 4, st);
            void* args[5] = {&pc, &qc, &wc, &sc, &wk};
            cudaError_t e = cudaLaunchCooperativeKernel(fn, G, kPtThreads, args, smem, st);
            if (e != cudaSuccess)
                return set_error("pathtrace_frame: cooperative launch (%d CTAs): %s", G, cudaGetErrorString(e));
            launches++;
        }
        k_pt_accumulate<<<grid_acc, 256, 0, st>>>(p, q, w, s);
        launches++;
    }
    k_pt_finalize<<<grid_acc, 256, 0, st>>>(p, q, w, s);
    g_launches = launches + 1;
    return check_launch("pathtrace_frame");
}
