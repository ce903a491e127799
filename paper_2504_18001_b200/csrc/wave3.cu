// One-barrier persistent wavefront march (default frame kernel), sm_100a, -fmad=false.
//
// Same iteration semantics as the reference's wavefront loop
// (render/raymarch.py:72-115): iteration k advances every live ray, the rays
// that sample are ranked in ray order (that rank is the RNG lane, P5, and the
// slot in the next compacted buffer, P18), probed, shaded, and retired when
// dead.  Schedule, one CTA per SM, all iterations in one cooperative launch:
//
//   state S_k   slots [0, m_k), m_k = n_{k-1}; a slot holds a sample of
//               iteration k (ray id, tmid, dt, cursor, colour, T) or id -1.
//               Slots form groups of 32 (one warp), groups form stripes of 32.
//               Whoever wrote S_k also counted its sampling slots per group
//               and per stripe.
//   barrier     the only grid-wide sync of an iteration (one counter per
//               barrier instance, no reset).
//   scan        every CTA scans the m_k/1024 stripe counts in shared memory.
//   phase k     warps take groups (first by warp id, then from a global ticket:
//               dynamic balance across the whole GPU; the next group's slot ids
//               are prefetched); a group's rank base = stripe prefix + the warp's
//               own scan of the earlier group counts of that stripe; then per
//               lane: stochastic LoD + MRPD probe + trilinear + stamp + miss
//               filing (kernels.py:166-273, sampler.py:236-275); shade
//               (kernels.py:322-355); and, in the same thread, the advance of
//               iteration k+1 (kernels.py:35-137) straight into slot `rank` of
//               S_{k+1} plus its group/stripe counts.
//   misses      true misses (sampler.py:276-279) are queued instead of being
//               inferred inline; after the barrier, an iteration that queued any
//               runs one dense miss phase (inference, shade, advance, count)
//               and one more barrier.  Steady-state frames have none.  For the
//               default INR the phase infers 32 misses per warp with the hidden
//               layers on the tensor cores (mlp_warp.cuh).
//
// The majorant grid, the transfer-function LUT and the MLP weights (as mma
// B fragments for the default INR) live in shared memory; per-sample state is
// SoA so every warp access is coalesced.  Bit-exactness: all addressing, cursor,
// LoD and compositing arithmetic is the reference's f64/f32 sequence without FMA
// contraction (common.cuh); only inferred INR values are tolerance-level (P14).
#include <cstddef>
#include <cstdio>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"
#include "mlp_warp.cuh"

namespace cinr {

constexpr int kW3MaxStripeScan = 16384;     // stripes scanned in shared memory (16.7 M rays)
constexpr long long kW3MuSmemCells = 36864;  // f32 majorants in smem up to 144 KB

constexpr long long kW3OccMaxCells = 1ll << 20;
constexpr int kW3LutMax = 4096;
constexpr int kW3TraceIters = 512;  // diagnostics: per-CTA timestamps of the first iterations
constexpr int kW3TraceCtas = 1024;

struct W3Ws {
    int32_t* id[2];
    double* tmid[2];
    double* dt[2];
    long long* cur[2];
    double* cr[2];
    double* cg[2];
    double* cb[2];
    double* tr[2];
    int* gcnt;           // [3][maxg] sampling slots per group of S_k (k % 3)
    int* scnt;           // [3][maxs] per stripe (32 groups)
    int* mlist;          // queued true misses (slots of S_{k+1})
    int* nmiss;          // [max_it + 2]
    int* tick;           // [max_it + 2] group tickets (0 = prologue, k + 1 = phase k)
    unsigned int* bar;   // [2 * (max_it + 2)] arrivals per barrier instance
    unsigned int* trace; // [kW3TraceIters][kW3TraceCtas][3] globaltimer low words (timing frames)
    long long maxg, maxs;
    // dynamic shared-memory carve (bytes)
    int sm_lut, sm_mu, sm_occ, sm_mlp, sm_sc, sm_total;
};

inline int64_t w3_layout(int64_t n, int32_t max_it, void* base, W3Ws* s) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    const int64_t maxg = (n + 31) / 32 + 1;
    const int64_t maxs = (maxg + 31) / 32 + 1;
    const int64_t ns = maxg * 32;  // whole groups, so 16-byte group copies stay in bounds
    size_t o_id[2], o_tm[2], o_dt[2], o_cur[2], o_c[2][4];
    for (int b = 0; b < 2; b++) {
        o_id[b] = take((size_t)ns * 4);
        o_tm[b] = take((size_t)ns * 8);
        o_dt[b] = take((size_t)ns * 8);
        o_cur[b] = take((size_t)ns * 8);
        for (int q = 0; q < 4; q++) o_c[b][q] = take((size_t)ns * 8);
    }
    size_t o_g = take((size_t)maxg * 3 * 4);
    size_t o_s = take((size_t)maxs * 3 * 4);
    size_t o_ml = take((size_t)n * 4 + 4);
    size_t o_nm = take((size_t)(max_it + 2) * 4);
    size_t o_tk = take((size_t)(max_it + 2) * 4);
    size_t o_bar = take((size_t)(max_it + 2) * 2 * 4);
    size_t o_tr = take((size_t)kW3TraceIters * kW3TraceCtas * 3 * 4);
    if (base && s) {
        char* p = (char*)base;
        for (int b = 0; b < 2; b++) {
            s->id[b] = (int32_t*)(p + o_id[b]);
            s->tmid[b] = (double*)(p + o_tm[b]);
            s->dt[b] = (double*)(p + o_dt[b]);
            s->cur[b] = (long long*)(p + o_cur[b]);
            s->cr[b] = (double*)(p + o_c[b][0]);
            s->cg[b] = (double*)(p + o_c[b][1]);
            s->cb[b] = (double*)(p + o_c[b][2]);
            s->tr[b] = (double*)(p + o_c[b][3]);
        }
        s->gcnt = (int*)(p + o_g);
        s->scnt = (int*)(p + o_s);
        s->mlist = (int*)(p + o_ml);
        s->nmiss = (int*)(p + o_nm);
        s->tick = (int*)(p + o_tk);
        s->bar = (unsigned int*)(p + o_bar);
        s->trace = (unsigned int*)(p + o_tr);
        s->maxg = maxg;
        s->maxs = maxs;
    }
    return (int64_t)align_up(off, 256);
}

int64_t wave3_ws_bytes(int64_t npix, int max_it) {
    if (max_it > kMaxIterCap) max_it = kMaxIterCap;
    return frame_ws_layout(npix, max_it, nullptr, nullptr) + w3_layout(npix, max_it, nullptr, nullptr);
}

// Grid barrier instance `b`: every CTA adds one arrival to its own counter and
// waits for all G (no reset, so no second round trip for the last arriver).
__device__ __forceinline__ void w3_barrier(unsigned int* bar, int b, unsigned int G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int* c = bar + b;
        // release: the CTA's writes (ordered before by bar.sync) become visible with the arrival
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        } while (v < G);
    }
    __syncthreads();
}

// Slot ids of group gg of S_k and the counts of the earlier groups of its stripe.
__device__ __forceinline__ void w3_fetch(const W3Ws& s, int b, const int* gcur, long long m, long long ng,
                                         long long gg, int lane, int& id_o, int& gc_o) {
    const long long ii = gg * 32 + lane;
    id_o = (gg < ng && ii < m) ? __ldcg(s.id[b] + ii) : -1;
    const long long gg0 = gg & ~31ll;
    gc_o = (gg < ng && gg0 + lane < gg) ? __ldcg(gcur + gg0 + lane) : 0;
}

// exclusive block scan of a[0..L) in place (shared memory); returns the total
template <int NT>
__device__ __forceinline__ int w3_scan_array(int* a, int L, int* wsum) {
    constexpr int NW = NT / 32;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int per = (L + NT - 1) / NT;
    const int lo = t * per, hi = min(lo + per, L);
    int sum = 0;
    for (int i = lo; i < hi; i++) sum += a[i];
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int wb = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < NW; q++) {
        const int v = wsum[q];
        wb += (q < warp) ? v : 0;
        tot += v;
    }
    int run = wb + x - sum;
    for (int i = lo; i < hi; i++) {
        const int v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
    return tot;
}

__device__ __forceinline__ void w3_retire(const VcbFrameParams& p, int pix, double cr, double cg, double cb,
                                          double tr) {
    // raymarch.py:57-60: rgb = color + T*bg, alpha = 1 - T, then .astype(float32)
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

struct W3Smem {
    int4 lv[VCB_MAX_LOD];  // per LoD: brick grid + page-table offset (no indexed constant loads)
    int wsum[32];
    unsigned long long cnt[3];
};

struct W3Ctx {
    double ox, oy, oz;
    const float* mu_s;
    const uint32_t* occ;
};

// After the shade of a live sample: the advance of iteration k+1 (or the
// iteration-cap flush) and the write of slot j of S_{k+1}.  Returns the
// sampling flag of slot j.
#ifdef CINR_STATS
// diagnostics build: FrameCounters.pad as u64 [skip-loop steps, advances, max steps in one advance];
// FrameWs.mq_pos as u64 [groups, cycles per phase stage 0..5] summed over warps
#define W3_NSKIP , &nskip
#define W3_T(q)                                                   \
    do {                                                          \
        __syncwarp(__activemask());                               \
        const long long t_ = clock64();                           \
        st_cyc[q] += t_ - t_prev;                                 \
        t_prev = t_;                                              \
    } while (0)
#else
#define W3_NSKIP
#define W3_T(q) \
    do {        \
    } while (0)
#endif

__device__ __forceinline__ int w3_next(const VcbFrameParams& p, const FrameWs& w, const W3Ws& s, const W3Ctx& c,
                                       int nb, bool last, int id, long long j, double dx, double dy, double dz,
                                       double ten, double tex, long long cur, double cr, double cg, double cb,
                                       double tr, int pix) {
    int f = 0;
    AdvanceOut a;
    if (!last) {
        double cf = __longlong_as_double(cur);
        i64 ck = cur;
#ifdef CINR_STATS
        int nskip = 0;
        const long long ta0 = clock64();
#endif
        f = advance_one(c.ox, c.oy, c.oz, dx, dy, dz, ten, tex, cf, ck, p.adv, p.mu, a, c.occ, c.mu_s W3_NSKIP);
#ifdef CINR_STATS
        if (a.tmid == -1234.5) asm volatile("trap;");
        const long long ta1 = clock64();
        atomicAdd(reinterpret_cast<unsigned long long*>(w.ctr->pad) + 5, (unsigned long long)(ta1 - ta0));
        atomicAdd(reinterpret_cast<unsigned long long*>(w.ctr->pad) + 6, 1ull);
#endif
#ifdef CINR_STATS
        {
            // warp-aggregated so the counters do not perturb the stage timings much
            const unsigned am = __activemask();
            int tot = nskip, mx = nskip;
            for (int o = 16; o > 0; o >>= 1) {
                const int ot = __shfl_xor_sync(am, tot, o), om = __shfl_xor_sync(am, mx, o);
                if ((am >> ((threadIdx.x & 31) ^ o)) & 1u) {
                    tot += ot;
                    mx = max(mx, om);
                }
            }
            if ((threadIdx.x & 31) == __ffs(am) - 1) {
                unsigned long long* st = reinterpret_cast<unsigned long long*>(w.ctr->pad);
                atomicAdd(st, (unsigned long long)tot);
                atomicAdd(st + 1, (unsigned long long)__popc(am));
                atomicMax(st + 2, (unsigned long long)mx);
                atomicAdd(st + 3, (unsigned long long)mx);  // sum over warps of the slowest lane
                atomicAdd(st + 4, 1ull);
            }
        }
#endif
        cur = p.adv.adaptive ? __double_as_longlong(cf) : (long long)ck;
    }
    if (f) {
        __stcg(s.id[nb] + j, id);
        __stcg(s.tmid[nb] + j, a.tmid);
        __stcg(s.dt[nb] + j, a.dt);
        __stcg(s.cur[nb] + j, cur);
        __stcg(s.cr[nb] + j, cr);
        __stcg(s.cg[nb] + j, cg);
        __stcg(s.cb[nb] + j, cb);
        __stcg(s.tr[nb] + j, tr);
    } else {
        w3_retire(p, pix, cr, cg, cb, tr);
        __stcg(s.id[nb] + j, -1);
    }
    return f;
}

// Counts of the next buffer for one warp whose flagged lanes hold consecutive
// ranks starting at jb (so at most two groups): one atomic per group and stripe.
__device__ __forceinline__ void w3_count_next(int* gnx, int* snx, long long jb, long long j, int f) {
    const int lane = threadIdx.x & 31;
    const long long ga = jb >> 5;
    const unsigned fa = __ballot_sync(0xffffffffu, f && (j >> 5) == ga);
    const unsigned fb = __ballot_sync(0xffffffffu, f && (j >> 5) != ga);
    if (lane == 0) {
        if (fa) {
            atomicAdd(gnx + ga, __popc(fa));
            atomicAdd(snx + (ga >> 5), __popc(fa));
        }
        if (fb) {
            atomicAdd(gnx + ga + 1, __popc(fb));
            atomicAdd(snx + ((ga + 1) >> 5), __popc(fb));
        }
    }
}

// Frame scheduler (VcbFrameParams.miss_budget): whether this lane's queued true miss
// may be decoded (counted in misses_resolved) or is left undecoded and not composited
// (deferred_misses).  Warp-aggregated; call with every lane of the warp.
__device__ __forceinline__ bool w3_budget(const VcbFrameParams& p, const FrameWs& w, bool want) {
    const unsigned nb = __ballot_sync(__activemask(), want);
    if (!nb) return false;
    const int lane = threadIdx.x & 31, leader = __ffs(nb) - 1;
    unsigned long long base = 0;
    if (p.miss_budget >= 0 && lane == leader)
        base = atomicAdd(reinterpret_cast<unsigned long long*>(&w.ctr->pad[2]), (unsigned long long)__popc(nb));
    base = __shfl_sync(__activemask(), base, leader);
    const bool ok = want && (p.miss_budget < 0 || (long long)(base + __popc(nb & ((1u << lane) - 1u))) < p.miss_budget);
    const unsigned okb = __ballot_sync(__activemask(), ok);
    if (lane == leader) {
        if (okb) atomicAdd((unsigned long long*)&p.stats->misses_resolved, (unsigned long long)__popc(okb));
        if (nb & ~okb) atomicAdd((unsigned long long*)&p.stats->deferred_misses, (unsigned long long)__popc(nb & ~okb));
    }
    return ok;
}

// One queued true miss of iteration k-1 (sampler.py:276-279): field inference at the
// sample, shade, then the advance of iteration k into the same slot of S_k.  Out of
// line, so the register-hungry inference does not raise the phase's register budget.
template <int kInr>
static __device__ __noinline__ void w3_miss_item(const VcbFrameParams& p, const FrameWs& w, const W3Ws& s,
                                                 const W3Ctx c, const MlpSmem mlp, const float* lut, bool smem_lut,
                                                 long long q, int b, bool last, int* gnx, int* snx) {
    const double hmax = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
    const long long j = __ldcg(s.mlist + q);
    const int id = __ldcg(s.id[b] + j);
    const double tmid = __ldcg(s.tmid[b] + j), dt = __ldcg(s.dt[b] + j);
    const long long cur = __ldcg(s.cur[b] + j);
    double cr = __ldcg(s.cr[b] + j), cg = __ldcg(s.cg[b] + j), cb = __ldcg(s.cb[b] + j), tr = __ldcg(s.tr[b] + j);
    const double dx = __ldg(w.ray_dir + 3 * id), dy = __ldg(w.ray_dir + 3 * id + 1), dz = __ldg(w.ray_dir + 3 * id + 2);
    const double px = DADD(c.ox, DMUL(dx, tmid)), py = DADD(c.oy, DMUL(dy, tmid)), pz = DADD(c.oz, DMUL(dz, tmid));
    bool dead = false;
    if (w3_budget(p, w, true)) {
        int bad = 0;
        const float v = field_eval<kInr>(p.field, clampd(px, 0.0, hmax), clampd(py, 0.0, hmax),
                                         clampd(pz, 0.0, hmax), mlp, &bad);
        if (bad) w.ctr->nonfinite = 1;
        dead = smem_lut ? shade_one<true>(v, dt, lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg, cb,
                                          tr)
                        : shade_one<false>(v, dt, lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg,
                                           cb, tr);
    }
    int f = 0;
    if (dead) {
        w3_retire(p, __ldg(w.ray_pix + id), cr, cg, cb, tr);
        __stcg(s.id[b] + j, -1);
    } else {
        f = w3_next(p, w, s, c, b, last, id, j, dx, dy, dz, __ldg(w.ray_ten + id), __ldg(w.ray_tex + id), cur, cr,
                    cg, cb, tr, __ldg(w.ray_pix + id));
    }
    if (f) {
        atomicAdd(gnx + (j >> 5), 1);
        atomicAdd(snx + (j >> 10), 1);
    }
}

// The default INR's queued misses, 32 per warp: warp-cooperative inference with the
// hidden layers on the tensor cores (mlp_warp.cuh), then per lane the same shade /
// advance / publish as w3_miss_item.  Called converged by whole warps.
static __device__ __noinline__ void w3_miss_warp(const VcbFrameParams& p, const FrameWs& w, const W3Ws& s,
                                                 const W3Ctx c, const MlpFrag* fr, const float* lut, bool smem_lut,
                                                 long long base, int nm, int b, bool last, int* gnx, int* snx) {
    const double hmax = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
    const long long q = base + (threadIdx.x & 31);
    const bool active = q < nm;
    long long j = 0, cur = 0;
    int id = 0;
    double tmid = 0.0, dt = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, tr = 1.0, dx = 0.0, dy = 0.0, dz = 0.0;
    double px = 0.5, py = 0.5, pz = 0.5;
    if (active) {
        j = __ldcg(s.mlist + q);
        id = __ldcg(s.id[b] + j);
        tmid = __ldcg(s.tmid[b] + j);
        dt = __ldcg(s.dt[b] + j);
        cur = __ldcg(s.cur[b] + j);
        cr = __ldcg(s.cr[b] + j);
        cg = __ldcg(s.cg[b] + j);
        cb = __ldcg(s.cb[b] + j);
        tr = __ldcg(s.tr[b] + j);
        dx = __ldg(w.ray_dir + 3 * id);
        dy = __ldg(w.ray_dir + 3 * id + 1);
        dz = __ldg(w.ray_dir + 3 * id + 2);
        px = clampd(DADD(c.ox, DMUL(dx, tmid)), 0.0, hmax);
        py = clampd(DADD(c.oy, DMUL(dy, tmid)), 0.0, hmax);
        pz = clampd(DADD(c.oz, DMUL(dz, tmid)), 0.0, hmax);
    }
    const bool granted = w3_budget(p, w, active);
    float v = 0.0f;
    if (__any_sync(0xffffffffu, granted)) v = inr_warp_default(p.field, fr, px, py, pz);
    if (!active) return;
    bool dead = false;
    if (granted) {
        if (!isfinite(v)) w.ctr->nonfinite = 1;
        if (p.field.clip01) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
        dead = smem_lut ? shade_one<true>(v, dt, lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg, cb,
                                          tr)
                        : shade_one<false>(v, dt, lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg,
                                           cb, tr);
    }
    int f = 0;
    if (dead) {
        w3_retire(p, __ldg(w.ray_pix + id), cr, cg, cb, tr);
        __stcg(s.id[b] + j, -1);
    } else {
        f = w3_next(p, w, s, c, b, last, id, j, dx, dy, dz, __ldg(w.ray_ten + id), __ldg(w.ray_tex + id), cur, cr,
                    cg, cb, tr, __ldg(w.ray_pix + id));
    }
    if (f) {
        atomicAdd(gnx + (j >> 5), 1);
        atomicAdd(snx + (j >> 10), 1);
    }
}

template <int kInr, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_wave3_march(const __grid_constant__ VcbFrameParams p, const __grid_constant__ FrameWs w,
                  const __grid_constant__ W3Ws s, int max_it) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ W3Smem sm;
    const int G = gridDim.x, cta = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;

    // ---- stage read-only tables in shared memory
    float* s_lut = s.sm_lut >= 0 ? reinterpret_cast<float*>(dsm + s.sm_lut) : nullptr;
    if (s_lut)
        for (int i = threadIdx.x; i < p.lut_size * 4; i += NT) s_lut[i] = __ldg(p.lut + i);
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    W3Ctx c;
    c.ox = p.cam.origin[0];
    c.oy = p.cam.origin[1];
    c.oz = p.cam.origin[2];
    c.mu_s = nullptr;
    c.occ = nullptr;
    if (s.sm_mu >= 0) {
        float* m = reinterpret_cast<float*>(dsm + s.sm_mu);
        for (long long i = threadIdx.x; i < cells; i += NT) m[i] = __ldg(p.mu + i);
        c.mu_s = m;
    } else if (s.sm_occ >= 0) {
        uint32_t* occ = reinterpret_cast<uint32_t*>(dsm + s.sm_occ);
        const int nwords = (int)((cells + 31) >> 5);
        for (int wd = threadIdx.x >> 5; wd < nwords; wd += NT / 32) {
            const long long q = (long long)wd * 32 + lane;
            const unsigned b = __ballot_sync(0xffffffffu, q < cells && __ldg(p.mu + q) > 0.0f);
            if (lane == 0) occ[wd] = b;
        }
        c.occ = occ;
    }
    MlpSmem mlp;
    mlp.w = mlp.b = nullptr;
    const MlpFrag* mfrag = nullptr;
    if (kInr == 1 && s.sm_mlp >= 0) {
        // default INR: B fragments for the tensor-core miss inference
        stage_mlp_frag(p.field, reinterpret_cast<MlpFrag*>(dsm + s.sm_mlp));
        mfrag = reinterpret_cast<const MlpFrag*>(dsm + s.sm_mlp);
    } else if (kInr != 0 && s.sm_mlp >= 0) {
        stage_mlp(p.field, reinterpret_cast<float*>(dsm + s.sm_mlp), mlp);
    }
    int* s_sc = reinterpret_cast<int*>(dsm + s.sm_sc);
    const float* lut = s_lut ? s_lut : p.lut;
    if (threadIdx.x < 3) sm.cnt[threadIdx.x] = 0;
    if (threadIdx.x <= p.probe.max_lod && threadIdx.x < VCB_MAX_LOD)
        sm.lv[threadIdx.x] = make_int4((int)p.probe.grid[threadIdx.x][0], (int)p.probe.grid[threadIdx.x][1],
                                       (int)p.probe.grid[threadIdx.x][2], (int)p.probe.offset[threadIdx.x]);
    __syncthreads();

    unsigned c_ex = 0, c_fb = 0, c_ms = 0;  // per-thread sample counts (< 2^32)
    long long req = 0;

    // diagnostics (timing frames): per CTA and iteration, globaltimer after the
    // barrier, after the scan and when all of the CTA's warps finished the phase
    const bool tracing = (p.timing & 2) != 0;  // bit 1: per-iteration trace (diagnostics only)
    const bool trace = tracing && threadIdx.x == 0 && cta < kW3TraceCtas;
    auto stamp = [&](int kk, int what) {
        if (trace && kk < kW3TraceIters) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            s.trace[((long long)kk * kW3TraceCtas + cta) * 3 + what] = (unsigned int)t;
        }
    };

    // ---- prologue: advance of iteration 0 over the ray list (slot i = ray i)
    const long long n0 = __ldcg(w.live);
    {
        const long long ng = (n0 + 31) >> 5;
        const long long nw = (long long)G * (NT / 32);
        for (long long g = (long long)cta * (NT / 32) + (threadIdx.x >> 5);;) {
            if (g >= ng) break;
            long long gnext = 0;
            if (lane == 0) gnext = nw + atomicAdd(s.tick, 1);
            const long long i = g * 32 + lane;
            int f = 0;
            if (i < n0) {
                const int id = (int)i;
                const long long cur0 = p.adv.adaptive ? __double_as_longlong(__ldg(w.ray_ten + id)) : 0ll;
                f = w3_next(p, w, s, c, 0, max_it <= 0, id, i, __ldg(w.ray_dir + 3 * i), __ldg(w.ray_dir + 3 * i + 1),
                            __ldg(w.ray_dir + 3 * i + 2), __ldg(w.ray_ten + i), __ldg(w.ray_tex + i), cur0, 0.0,
                            0.0, 0.0, 1.0, __ldg(w.ray_pix + i));
            }
            const int cnt = __popc(__ballot_sync(0xffffffffu, f));
            if (lane == 0) {
                __stcg(s.gcnt + g, cnt);
                if (cnt) atomicAdd(s.scnt + (g >> 5), cnt);
            }
            g = __shfl_sync(0xffffffffu, gnext, 0);
        }
    }

    int k = 0, nbar = 0;
    long long m = n0;  // slots in S_k
    int iters = 0;
    for (;; k++) {
        w3_barrier(s.bar, nbar++, G);
        stamp(k, 0);
        // one round of loads after the barrier: queued misses of k-1, the stripe counts
        // and the first group of S_k (the last two again if a miss phase changes them)
        const int nm = (k > 0) ? __ldcg(s.nmiss + (k - 1)) : 0;
        const long long ng = (m + 31) >> 5;
        const int ns = (int)((ng + 31) >> 5);
        const int* gcur = s.gcnt + (k % 3) * s.maxg;
        const long long g_first = (long long)cta * (NT / 32) + (threadIdx.x >> 5);
        int id_nx = -1, gc_nx = 0;
        if (k < max_it) {
            for (int t = threadIdx.x; t < ns; t += NT) s_sc[t] = __ldcg(s.scnt + (k % 3) * s.maxs + t);
            w3_fetch(s, k & 1, gcur, m, ng, g_first, lane, id_nx, gc_nx);
        }
        if (k > 0) {
            // ---------------- miss phase of iteration k-1 (sampler.py:276-279)
            if (nm > 0) {
                const int b = k & 1;  // S_k
                int* gnx = s.gcnt + (k % 3) * s.maxg;
                int* snx = s.scnt + (k % 3) * s.maxs;
                const bool last = (k == max_it);
                if (kInr == 1) {
                    for (long long qb = ((long long)cta * (NT / 32) + (threadIdx.x >> 5)) * 32; qb < nm;
                         qb += (long long)G * NT)
                        w3_miss_warp(p, w, s, c, mfrag, lut, s_lut != nullptr, qb, nm, b, last, gnx, snx);
                } else {
                    for (long long q = (long long)cta * NT + threadIdx.x; q < nm; q += (long long)G * NT)
                        w3_miss_item<kInr>(p, w, s, c, mlp, lut, s_lut != nullptr, q, b, last, gnx, snx);
                }
                w3_barrier(s.bar, nbar++, G);
                if (k < max_it) {
                    for (int t = threadIdx.x; t < ns; t += NT) s_sc[t] = __ldcg(s.scnt + (k % 3) * s.maxs + t);
                    w3_fetch(s, k & 1, gcur, m, ng, g_first, lane, id_nx, gc_nx);
                }
            }
        }
        if (k >= max_it) {
            iters = max_it;
            break;
        }
        // ---------------- scan of the stripe counts of S_k
        __syncthreads();
        const long long nk = w3_scan_array<NT>(s_sc, ns, sm.wsum);
        stamp(k, 1);
        if (tracing && cta == 0 && threadIdx.x == 0) w.live[k + 1] = (int)nk;
        if (nk == 0) {
            iters = (n0 == 0) ? 0 : k + 1;
            break;
        }
        req += nk;
        // zero the counters of S_{k+2} (last read by the scan of k-1, next written by phase k+1)
        {
            const long long nz = (nk + 31) >> 5;
            int* gz = s.gcnt + ((k + 2) % 3) * s.maxg;
            int* sz = s.scnt + ((k + 2) % 3) * s.maxs;
            for (long long i = (long long)cta * NT + threadIdx.x; i < nz; i += (long long)G * NT) gz[i] = 0;
            for (long long i = (long long)cta * NT + threadIdx.x; i < ((nz + 31) >> 5); i += (long long)G * NT)
                sz[i] = 0;
            if (cta == 0 && threadIdx.x == 0) s.nmiss[k + 1] = 0;
        }

        // ---------------- phase k: warps take groups of S_k from the ticket
        {
            const int b = k & 1, nb = (k + 1) & 1;
            int* gnx = s.gcnt + ((k + 1) % 3) * s.maxg;
            int* snx = s.scnt + ((k + 1) % 3) * s.maxs;
            const bool last = (k + 1 == max_it);
            // first group by warp id, then from the ticket (no atomics at all when
            // the iteration has fewer groups than the grid has warps)
            int* tick = s.tick + (k + 1);
            const long long nw = (long long)G * (NT / 32);
            long long g = g_first;
            // slot ids and earlier-group counts of a group, loaded one group ahead
            auto fetch = [&](long long gg, int& id_o, int& gc_o) { w3_fetch(s, b, gcur, m, ng, gg, lane, id_o, gc_o); };
            const bool use_rng = p.cached && p.probe.mode != 2;
#ifdef CINR_STATS
            long long st_cyc[7] = {0, 0, 0, 0, 0, 0, 0};
            long long t_prev = clock64();
#endif
            while (g < ng) {
                W3_T(6);
                long long gnext = 0;
                if (lane == 0) gnext = nw + atomicAdd(tick, 1);
                const long long i = g * 32 + lane;
                const int id = id_nx;
                // rank base: stripe prefix + earlier groups of the stripe
                const long long jb = (long long)s_sc[g >> 5] + warp_sum(gc_nx);
                const unsigned bal = __ballot_sync(0xffffffffu, id >= 0);
                const long long j = jb + __popc(bal & lt_mask);
                // this group's state (SoA slots through L2; ray data through the read-only path)
                double tmid = 0.0, dt = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, tr = 0.0;
                double dx = 0.0, dy = 0.0, dz = 0.0, ten = 0.0, tex = 0.0;
                long long cur = 0;
                int pix = 0;
                uint32_t r_prev = 0u;
                if (id >= 0) {
                    tmid = __ldcg(s.tmid[b] + i);
                    dt = __ldcg(s.dt[b] + i);
                    cur = __ldcg(s.cur[b] + i);
                    cr = __ldcg(s.cr[b] + i);
                    cg = __ldcg(s.cg[b] + i);
                    cb = __ldcg(s.cb[b] + i);
                    tr = __ldcg(s.tr[b] + i);
                    dx = __ldg(w.ray_dir + 3 * id);
                    dy = __ldg(w.ray_dir + 3 * id + 1);
                    dz = __ldg(w.ray_dir + 3 * id + 2);
                    ten = __ldg(w.ray_ten + id);
                    tex = __ldg(w.ray_tex + id);
                    pix = __ldg(w.ray_pix + id);
                    if (use_rng && k > 0) r_prev = __ldcg(w.rng + j);
                }
                const long long g_nx = __shfl_sync(0xffffffffu, gnext, 0);
                fetch(g_nx, id_nx, gc_nx);
                // the sample position as the advance computed it: o + d * tmid
                const double px = DADD(c.ox, DMUL(dx, tmid)), py = DADD(c.oy, DMUL(dy, tmid)),
                             pz = DADD(c.oz, DMUL(dz, tmid));
                W3_T(0);
                int f = 0, queued = 0;
                if (id >= 0) {
                    float v = 0.0f;
#ifdef CINR_STATS
                    if (px == -1234.5 || dt == -1.0 || cr == -1.0 || tr == -1.0) asm volatile("trap;");
#endif
                    W3_T(1);
                    if (!p.cached) {
                        queued = 1;
                    } else {
                        double u = 0.0;
                        if (use_rng) {
                            uint32_t r = (k == 0) ? lane_seed(p.rng_base, (u64)j) : r_prev;
                            r = xorshift32(r);
                            __stcg(w.rng + j, r);
                            u = DMUL((double)r, 2.3283064365386963e-10);  // / 2^32, exact
                        }
                        double dist = tmid;
                        if (p.paged_dist) {
                            const double ex = DSUB(px, c.ox), ey = DSUB(py, c.oy), ez = DSUB(pz, c.oz);
                            dist = __dsqrt_rn(DADD(DADD(DMUL(ex, ex), DMUL(ey, ey)), DMUL(ez, ez)));
                        }
                        int rq, slot, rflat;
                        const int sv = probe_one(px, py, pz, dist, u, p.probe, p.table, p.pool,
                                                 (long long*)p.last_used, p.cache_frame, v, rq, slot, sm.lv, &rflat);
                        if (sv != rq) {
                            if (p.probe.b_pow2 != 0) {
                                warp_aggregated_add(p.miss_count, (i64)rflat);  // the probe's requested brick
                            } else {
                                // mrpd.py:215-225 miss filing at the requested LoD (native clipped, P6)
                                const i64 span = p.probe.b << rq;
                                const double nx = clampd(DSUB(DMUL(px, p.probe.vx), 0.5), 0.0, DSUB(p.probe.vx, 1.0));
                                const double ny = clampd(DSUB(DMUL(py, p.probe.vy), 0.5), 0.0, DSUB(p.probe.vy, 1.0));
                                const double nz = clampd(DSUB(DMUL(pz, p.probe.vz), 0.5), 0.0, DSUB(p.probe.vz, 1.0));
                                const int4 q = sm.lv[rq];
                                const i64 bx = clampi((i64)floor(cell_div(DADD(nx, 1.0), (double)span)), 0, q.x - 1);
                                const i64 by = clampi((i64)floor(cell_div(DADD(ny, 1.0), (double)span)), 0, q.y - 1);
                                const i64 bz = clampi((i64)floor(cell_div(DADD(nz, 1.0), (double)span)), 0, q.z - 1);
                                warp_aggregated_add(p.miss_count, (i64)q.w + bx + (i64)q.x * (by + (i64)q.y * bz));
                            }
                        }
                        if (sv < 0) {
                            queued = 1;
                        } else {
                            c_ex += (sv == rq);
                            c_fb += (sv != rq);
                        }
                    }
#ifdef CINR_STATS
                    if (v == -1234.5f) asm volatile("trap;");
#endif
                    W3_T(2);
                    if (queued) {
                        // the sample itself goes to slot j; the miss phase infers, shades, advances
                        c_ms += 1;
                        __stcg(s.id[nb] + j, id);
                        __stcg(s.tmid[nb] + j, tmid);
                        __stcg(s.dt[nb] + j, dt);
                        __stcg(s.cur[nb] + j, cur);
                        __stcg(s.cr[nb] + j, cr);
                        __stcg(s.cg[nb] + j, cg);
                        __stcg(s.cb[nb] + j, cb);
                        __stcg(s.tr[nb] + j, tr);
                    } else {
                        const bool dead = s_lut ? shade_one<true>(v, dt, lut, p.lut_size, p.adv.adaptive,
                                                                  p.adv.dt_base, p.term, cr, cg, cb, tr)
                                                : shade_one<false>(v, dt, lut, p.lut_size, p.adv.adaptive,
                                                                   p.adv.dt_base, p.term, cr, cg, cb, tr);
                        W3_T(3);
                        if (dead) {
                            w3_retire(p, pix, cr, cg, cb, tr);
                            __stcg(s.id[nb] + j, -1);
                        } else {
                            f = w3_next(p, w, s, c, nb, last, id, j, dx, dy, dz, ten, tex, cur, cr, cg, cb, tr, pix);
                        }
                    }
                }
                W3_T(4);
                // queue this warp's true misses (one atomic per warp)
                const unsigned qb = __ballot_sync(0xffffffffu, queued);
                if (qb) {
                    int qbase = 0;
                    if (lane == 0) qbase = atomicAdd(s.nmiss + k, __popc(qb));
                    qbase = __shfl_sync(0xffffffffu, qbase, 0);
                    if (queued) __stcg(s.mlist + qbase + __popc(qb & lt_mask), (int)j);
                }
                w3_count_next(gnx, snx, jb, j, f);
                g = g_nx;
                W3_T(5);
#ifdef CINR_STATS
                st_cyc[6] -= 0;  // stage 6 = loop overhead + ticket (measured at the next top)
#endif
            }
#ifdef CINR_STATS
            if (lane == 0) {
                // light iterations (< 256 groups: one group per warp, pure latency) apart
                unsigned long long* acc = reinterpret_cast<unsigned long long*>(w.mq_pos) + (ng < 256 ? 8 : 0);
                for (int q = 0; q < 7; q++) atomicAdd(acc + 1 + q, (unsigned long long)st_cyc[q]);
                if (st_cyc[0] != 0) atomicAdd(acc, 1ull);
            }
#endif
        }
        if (tracing) {
            __syncthreads();
            stamp(k, 2);
        }
        m = nk;
    }

    // ---- frame counters (FrameStats, mrpd.py:33-41)
    const unsigned long long t_ex = warp_sum((unsigned long long)c_ex);
    const unsigned long long t_fb = warp_sum((unsigned long long)c_fb);
    const unsigned long long t_ms = warp_sum((unsigned long long)c_ms);
    if (lane == 0) {
        atomicAdd(&sm.cnt[0], t_ex);
        atomicAdd(&sm.cnt[1], t_fb);
        atomicAdd(&sm.cnt[2], t_ms);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&p.stats->exact, sm.cnt[0]);
        atomicAdd((unsigned long long*)&p.stats->fallback, sm.cnt[1]);
        atomicAdd((unsigned long long*)&p.stats->miss, sm.cnt[2]);
        if (cta == 0) {
            p.stats->requests = req;
            p.stats->iterations = iters;
            p.stats->rays = n0;
            p.stats->nonfinite = __ldcg(&w.ctr->nonfinite);
        }
    }
}

static const void* wave3_kernel(int mode, int nt) {
    if (nt == 384) return mode == 1 ? (const void*)k_wave3_march<1, 384> : (const void*)k_wave3_march<0, 384>;
    return mode == 1 ? (const void*)k_wave3_march<1, 512>
                     : mode == 2 ? (const void*)k_wave3_march<2, 512> : (const void*)k_wave3_march<0, 512>;
}

void launch_rays(const VcbFrameParams& p, const FrameWs& w, cudaStream_t st);

// nt: threads per CTA (384 = 12 warps at <= 168 registers, the default: the 512-thread
// build spills ~300 B per thread at 128 registers and is 11% slower; 768 = 24 warps at
// <= 80 registers)
int launch_wave3_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used,
                       int nt, int mu_mode) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    FrameWs w;
    const int64_t need = frame_ws_layout(npix, max_it, p.workspace, &w);
    W3Ws s;
    const int64_t need3 = w3_layout(npix, max_it, (char*)p.workspace + need, &s);
    if (need + need3 > p.workspace_bytes)
        return set_error("march_frame: workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)(need + need3));
    const int mode = inr_mode(p.field);
    if (mode == 2) nt = 512;  // the generic INR keeps its arrays on the stack either way
    const int G = device_sms();
    // dynamic shared memory: LUT, majorants (or occupancy bits), MLP weights, stripe prefixes
    int off = 0;
    auto take = [&](int bytes) {
        const int o = (off + 15) & ~15;
        off = o + bytes;
        return o;
    };
    // fixed parts first, then the majorants in whatever shared memory is left
    constexpr int kSmemMax = 227 * 1024;
    s.sm_lut = (p.lut_size <= kW3LutMax) ? take(p.lut_size * 16) : -1;
    s.sm_mlp = -1;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        s.sm_mlp = take(mode == 1 ? (int)sizeof(MlpFrag) : (nw + nb) * 4);
    }
    if (s.maxs > kW3MaxStripeScan)
        return set_error("march_frame: %lld rays exceed the stripe scan budget", (long long)npix);
    s.sm_sc = take((int)s.maxs * 4);
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    s.sm_mu = s.sm_occ = -1;
    if (mu_mode == 0 && cells <= kW3MuSmemCells && off + 16 + cells * 4 <= kSmemMax) s.sm_mu = take((int)cells * 4);
    else if (cells <= kW3OccMaxCells && p.adv.skip_empty && off + 16 + ((cells + 31) >> 5) * 4 <= kSmemMax)
        s.sm_occ = take((int)(((cells + 31) >> 5) * 4));
    s.sm_total = off;
    const void* fn = wave3_kernel(mode, nt);
    const int per_sm = kernel_ctas_per_sm(fn, nt, off);
    if (per_sm < 1)
        return set_error("march_frame: frame kernel does not fit one CTA per SM (%d B shared)", off);
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(w.ctr_iter, 0, w.ctr_iter_bytes, st);
#ifdef CINR_STATS
    cudaMemsetAsync(w.mq_pos, 0, 16 * 8, st);
#endif
    cudaMemsetAsync(s.gcnt, 0, (size_t)s.maxg * 3 * 4, st);
    cudaMemsetAsync(s.scnt, 0, (size_t)s.maxs * 3 * 4, st);
    cudaMemsetAsync(s.nmiss, 0, 8, st);
    cudaMemsetAsync(s.tick, 0, (size_t)(max_it + 2) * 4, st);
    cudaMemsetAsync(s.bar, 0, (size_t)(max_it + 2) * 2 * 4, st);
    launch_rays(p, w, st);
    VcbFrameParams pc = p;
    FrameWs wc = w;
    W3Ws sc = s;
    int mi = max_it;
    void* args[4] = {&pc, &wc, &sc, &mi};
    if (ev) cudaEventRecord(ev[0], st);
    cudaError_t e = cudaLaunchCooperativeKernel(fn, G, nt, args, off, st);
    if (ev) {
        cudaEventRecord(ev[1], st);
        *ev_used = 1;
    }
    if (e != cudaSuccess) return set_error("march_frame: cooperative launch (%d CTAs): %s", G, cudaGetErrorString(e));
    *launches = 3;
    return check_launch("march_frame(wave3)");
}

int wave3_trace(const void* workspace, int64_t npix, int max_it, int n, unsigned int* out, int* live) {
    if (max_it > kMaxIterCap) max_it = kMaxIterCap;
    FrameWs w;
    const int64_t need = frame_ws_layout(npix, max_it, const_cast<void*>(workspace), &w);
    W3Ws s;
    w3_layout(npix, max_it, (char*)workspace + need, &s);
    if (n > kW3TraceIters) n = kW3TraceIters;
    if (cudaMemcpy(out, s.trace, (size_t)n * kW3TraceCtas * 3 * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(live, w.live, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return set_error("frame_trace: %s", cudaGetErrorString(cudaGetLastError()));
    return n;
}

int wave3_counters(const void* workspace, int64_t npix, int max_it, long long* out) {
    if (max_it > kMaxIterCap) max_it = kMaxIterCap;
    FrameWs w;
    frame_ws_layout(npix, max_it, const_cast<void*>(workspace), &w);
    if (cudaMemcpy(out, w.ctr->pad, 7 * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(out + 7, w.mq_pos, 16 * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return set_error("frame_counters: %s", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

}  // namespace cinr
