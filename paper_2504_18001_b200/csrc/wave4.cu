// Barrier-free pipelined wavefront march (sm_100a, -fmad=false).
//
// Same iteration semantics as the reference's wavefront loop
// (render/raymarch.py:72-115): iteration ("level") k advances every live ray,
// the rays that sample are ranked in ray order (the rank is the RNG lane, P5,
// and the slot in the next compacted buffer, P18), probed, shaded and retired
// when dead.  Nothing synchronises the grid.  Instead:
//
//   units     level k's buffer S_k (slots [0, m_k), m_k = n_{k-1}) is cut into
//             units of 32 slots, one warp each.  Warps take (level, unit)
//             tickets in order from one counter per level and move to level
//             k+1 when level k runs out, so several levels are in flight.
//   slots     every slot word carries its level as a tag and is published with
//             release semantics after the slot's state; a unit starts once its
//             32 slots carry tag k (lanes past m_k resolve through n_{k-1}).
//   ranks     a unit's rank base is the sum of the sampling counts of all
//             earlier units of its level: warp-parallel decoupled look-back over
//             per-unit (aggregate | inclusive prefix) words, tagged by level.
//   outputs   a sampling lane of rank j draws lane j's xorshift state (written
//             by the rank-j sample of level k-1), probes with stochastic LoD +
//             MRPD walk + trilinear + stamp + miss filing (kernels.py:166-273,
//             sampler.py:236-275), infers true misses through the field
//             (sampler.py:276-279), shades (kernels.py:322-355), advances to
//             level k+1 (kernels.py:35-137) and publishes slot j of S_{k+1}.
//
// Safety of the double-buffered slots: a unit of level k+1 can only finish its
// look-back after every earlier unit of level k+1 is complete, i.e. after every
// level-k sample of lower rank was processed, so the level-(k+2) slots it writes
// (ranks < its own slots) were already consumed by level k.
#include <cstddef>
#include <cstdio>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"

namespace cinr {

constexpr int kW4Threads = 512;
constexpr int kW4Ring = 64;  // look-back words: levels k and k+64 share a row (8 measurably aborted)
constexpr long long kW4MuSmemCells = 40960;
constexpr long long kW4OccMaxCells = 1ll << 20;
constexpr int kW4LutMax = 4096;
constexpr unsigned long long kW4FlagA = 1ull << 32;
constexpr unsigned long long kW4FlagP = 2ull << 32;
constexpr unsigned long long kW4Pub = 1ull << 63;

struct W4Ws {
    unsigned long long* idt[2];  // (level + 1) << 32 | (uint32) ray id (-1 = no sample); 0 = unwritten
    double* tmid[2];
    double* dt[2];
    long long* cur[2];
    double* cr[2];
    double* cg[2];
    double* cb[2];
    double* tr[2];
    uint32_t* rng[2];            // lane state by rank, written by level k for level k+1
    unsigned long long* look;    // [kW4Ring][maxg] (level + 1) << 34 | flag | value
    unsigned long long* total;   // [max_it + 1]: kW4Pub | n_k once known
    int* tick;                   // [max_it + 2]: tick[0] prologue, tick[k + 1] level k
    int* abort;                  // protocol violation: every warp leaves
    unsigned long long* cnt;     // exact, fallback, miss
    long long maxg, nslots;
    int sm_lut, sm_mu, sm_occ, sm_mlp, sm_total;
};

inline int64_t w4_layout(int64_t n, int32_t max_it, void* base, W4Ws* s) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    const int64_t maxg = (n + 31) / 32 + 1;
    const int64_t ns = maxg * 32;  // slot arrays cover whole units
    size_t o_id[2], o_tm[2], o_dt[2], o_cur[2], o_c[2][4], o_rng[2];
    for (int b = 0; b < 2; b++) {
        o_id[b] = take((size_t)ns * 8);
        o_tm[b] = take((size_t)ns * 8);
        o_dt[b] = take((size_t)ns * 8);
        o_cur[b] = take((size_t)ns * 8);
        for (int q = 0; q < 4; q++) o_c[b][q] = take((size_t)ns * 8);
        o_rng[b] = take((size_t)ns * 4);
    }
    size_t o_look = take((size_t)kW4Ring * maxg * 8);
    size_t o_tot = take((size_t)(max_it + 2) * 8);
    size_t o_tick = take((size_t)(max_it + 2) * 4);
    size_t o_ab = take(16);
    size_t o_cnt = take(64);
    if (base && s) {
        char* p = (char*)base;
        for (int b = 0; b < 2; b++) {
            s->idt[b] = (unsigned long long*)(p + o_id[b]);
            s->tmid[b] = (double*)(p + o_tm[b]);
            s->dt[b] = (double*)(p + o_dt[b]);
            s->cur[b] = (long long*)(p + o_cur[b]);
            s->cr[b] = (double*)(p + o_c[b][0]);
            s->cg[b] = (double*)(p + o_c[b][1]);
            s->cb[b] = (double*)(p + o_c[b][2]);
            s->tr[b] = (double*)(p + o_c[b][3]);
            s->rng[b] = (uint32_t*)(p + o_rng[b]);
        }
        s->look = (unsigned long long*)(p + o_look);
        s->total = (unsigned long long*)(p + o_tot);
        s->tick = (int*)(p + o_tick);
        s->abort = (int*)(p + o_ab);
        s->cnt = (unsigned long long*)(p + o_cnt);
        s->maxg = maxg;
        s->nslots = ns;
    }
    return (int64_t)align_up(off, 256);
}

int64_t wave4_ws_bytes(int64_t npix, int max_it) {
    if (max_it > kMaxIterCap) max_it = kMaxIterCap;
    return frame_ws_layout(npix, max_it, nullptr, nullptr) + w4_layout(npix, max_it, nullptr, nullptr);
}

// Publication protocol.  Mutable state is only ever read through L2 (.cg / strong
// loads), so readers need no L1 invalidation: a warp writes its slot state,
// executes one gpu-scope fence (all lanes, converged) and then stores the tags
// with strong relaxed stores; readers poll with strong relaxed loads and issue
// their .cg state loads only after the poll succeeded.  (ld.acquire would add an
// L1 invalidate per poll and st.release a membar per store.)
__device__ __forceinline__ unsigned long long w4_ld_acq(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void w4_fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void w4_st_rel(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void w4_retire(const VcbFrameParams& p, int pix, double cr, double cg, double cb,
                                          double tr) {
    // raymarch.py:57-60: rgb = color + T*bg, alpha = 1 - T, then .astype(float32)
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

// n_k if already known (n_{-1} = rays), else -1.  Non-blocking.
__device__ __forceinline__ long long w4_known_total(const W4Ws& s, int k, long long n0) {
    if (k < 0) return n0;
    const unsigned long long v = w4_ld_acq(s.total + k);
    return (v & kW4Pub) ? (long long)(v & 0xFFFFFFFFull) : -1;
}

// Try to learn n_k from the last unit of level k (needs n_{k-1}); publishes it.
__device__ __forceinline__ long long w4_try_total(const W4Ws& s, int k, long long n0) {
    long long t = w4_known_total(s, k, n0);
    if (t >= 0) return t;
    const long long m = w4_known_total(s, k - 1, n0);
    if (m < 0) return -1;
    const long long ng = (m + 31) >> 5;
    long long v = -1;
    if (ng == 0) {
        v = 0;
    } else {
        const unsigned long long w = w4_ld_acq(s.look + (long long)(k % kW4Ring) * s.maxg + (ng - 1));
        if ((w >> 34) == (unsigned long long)(k + 1) && (w & (3ull << 32)) == kW4FlagP)
            v = (long long)(w & 0xFFFFFFFFull);
        else if ((w >> 34) > (unsigned long long)(k + 1))
            atomicExch(s.abort, 1);
    }
    if (v >= 0) w4_st_rel(s.total + k, kW4Pub | (unsigned long long)v);
    return v;
}

// Warp-parallel decoupled look-back: exclusive prefix of unit t (t > 0) of level k.
__device__ __forceinline__ long long w4_lookback(const W4Ws& s, int k, long long t) {
    const int lane = threadIdx.x & 31;
    const unsigned long long tag = (unsigned long long)(k + 1);
    const unsigned long long* row = s.look + (long long)(k % kW4Ring) * s.maxg;
    long long acc = 0, base = t - 1;
    for (;;) {
        const long long idx = base - lane;
        unsigned long long w = kW4FlagP;  // virtual prefix 0 before unit 0
        if (idx >= 0) {
            int spins = 0;
            for (;;) {
                w = w4_ld_acq(row + idx);
                const unsigned long long wt = w >> 34;
                if (wt == tag && (w & (3ull << 32)) != 0) break;
                if (wt > tag || *(volatile int*)s.abort) {
                    atomicExch(s.abort, 1);
                    w = kW4FlagP;
                    break;
                }
                if (++spins > 8) __nanosleep(32);
            }
        }
        const bool isP = (w & (3ull << 32)) == kW4FlagP;
        const unsigned pm = __ballot_sync(0xffffffffu, isP);
        long long v = (long long)(w & 0xFFFFFFFFull);
        if (pm) {
            const int first = __ffs(pm) - 1;
            if (lane > first) v = 0;
            acc += warp_sum(v);
            return acc;
        }
        acc += warp_sum(v);
        base -= 32;
    }
}

struct W4Ctx {
    double ox, oy, oz;
    const float* mu_s;
    const uint32_t* occ;
    const float* lut;
    bool smem_lut;
};

template <int kInr>
static __device__ __noinline__ float w4_infer(const VcbField& F, double x, double y, double z, const MlpSmem mlp,
                                              int* bad) {
    return field_eval<kInr>(F, x, y, z, mlp, bad);
}

// Prologue unit: the advance of level 0 for rays [32t, 32t + 32) into S_0 (slot = ray).
__device__ __forceinline__ void w4_prologue(const VcbFrameParams& p, const FrameWs& w, const W4Ws& s,
                                            const W4Ctx& c, long long t, long long n0, int max_it) {
    const int lane = threadIdx.x & 31;
    const long long i = t * 32 + lane;
    const int id = (int)i;
    int f = 0;
    if (i < n0) {
    double cf = __ldg(w.ray_ten + id);
    i64 ck = 0;
    AdvanceOut a;
    if (max_it > 0)
        f = advance_one(c.ox, c.oy, c.oz, __ldg(w.ray_dir + 3 * i), __ldg(w.ray_dir + 3 * i + 1),
                        __ldg(w.ray_dir + 3 * i + 2), __ldg(w.ray_ten + i), __ldg(w.ray_tex + i), cf, ck, p.adv,
                        p.mu, a, c.occ, c.mu_s);
    if (f) {
        __stcg(s.tmid[0] + i, a.tmid);
        __stcg(s.dt[0] + i, a.dt);
        __stcg(s.cur[0] + i, p.adv.adaptive ? __double_as_longlong(cf) : (long long)ck);
        __stcg(s.cr[0] + i, 0.0);
        __stcg(s.cg[0] + i, 0.0);
        __stcg(s.cb[0] + i, 0.0);
        __stcg(s.tr[0] + i, 1.0);
    } else {
        w4_retire(p, __ldg(w.ray_pix + id), 0.0, 0.0, 0.0, 1.0);
    }
    }
    __syncwarp();
    w4_fence_release();
    if (i < n0) w4_st_rel(s.idt[0] + i, (1ull << 32) | (unsigned long long)(uint32_t)(f ? id : -1));
}

enum { kW4Done = 0, kW4Void = 1, kW4End = 2 };

// Unit t of level k.  Returns kW4Void when t is past the level's last unit and
// kW4End when the frame has no level k (n_{k-1} == 0) or was aborted.
template <int kInr>
__device__ __forceinline__ int w4_unit(const VcbFrameParams& p, const FrameWs& w, const W4Ws& s, const W4Ctx& c,
                                       const MlpSmem& mlp, int k, long long t, long long n0, int max_it,
                                       unsigned long long& c_ex, unsigned long long& c_fb,
                                       unsigned long long& c_ms) {
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int b = k & 1, nb = (k + 1) & 1;
    const long long i = t * 32 + lane;
    long long m = w4_known_total(s, k - 1, n0);
    if (m == 0) return kW4End;
    if (m > 0 && t >= ((m + 31) >> 5)) return kW4Void;
    // ---- wait for this unit's slots (tag k + 1) or for n_{k-1} to rule lanes out
    int id = -1;
    bool resolved = false;
    int spins = 0;
    for (;;) {
        if (!resolved) {
            if (m >= 0 && i >= m) {
                resolved = true;
            } else if (i < s.nslots) {
                const unsigned long long v = w4_ld_acq(s.idt[b] + i);
                if ((v >> 32) == (unsigned long long)(k + 1)) {
                    resolved = true;
                    id = (int)(uint32_t)v;
                }
            }
        }
        if (__all_sync(0xffffffffu, resolved)) break;
        if (m < 0) {
            long long v = 0;
            if (lane == 0) v = w4_try_total(s, k - 1, n0);
            m = __shfl_sync(0xffffffffu, v, 0);
            if (m == 0) return kW4End;
            if (m > 0 && t >= ((m + 31) >> 5)) return kW4Void;
        }
        if (*(volatile int*)s.abort) return kW4End;
        if (++spins > 4) __nanosleep(64);
    }
    __syncwarp();
    // ---- rank base by look-back; opportunistically publish n_k from the last unit
    const unsigned bal = __ballot_sync(0xffffffffu, id >= 0);
    const long long nu = __popc(bal);
    unsigned long long* my = s.look + (long long)(k % kW4Ring) * s.maxg + t;
    const unsigned long long tag = (unsigned long long)(k + 1) << 34;
    long long E = 0;
    if (t == 0) {
        if (lane == 0) w4_st_rel(my, tag | kW4FlagP | (unsigned long long)nu);
    } else {
        if (lane == 0) w4_st_rel(my, tag | kW4FlagA | (unsigned long long)nu);
        E = w4_lookback(s, k, t);
        if (lane == 0) w4_st_rel(my, tag | kW4FlagP | (unsigned long long)(E + nu));
    }
    if (lane == 0) {
        if (m < 0) m = w4_known_total(s, k - 1, n0);
        if (m >= 0 && t == ((m + 31) >> 5) - 1) w4_st_rel(s.total + k, kW4Pub | (unsigned long long)(E + nu));
    }
    __syncwarp();
    const bool last = (k + 1 >= max_it);
    const long long j = E + __popc(bal & lt_mask);
    int f = 0;
    if (id >= 0) {
    // ---- the sample of rank j
    const double tmid = __ldcg(s.tmid[b] + i), dt = __ldcg(s.dt[b] + i);
    long long cur = __ldcg(s.cur[b] + i);
    double cr = __ldcg(s.cr[b] + i), cg = __ldcg(s.cg[b] + i), cb = __ldcg(s.cb[b] + i), tr = __ldcg(s.tr[b] + i);
    const double dx = __ldg(w.ray_dir + 3 * id), dy = __ldg(w.ray_dir + 3 * id + 1), dz = __ldg(w.ray_dir + 3 * id + 2);
    // the sample position as the advance computed it: o + d * tmid
    const double px = DADD(c.ox, DMUL(dx, tmid)), py = DADD(c.oy, DMUL(dy, tmid)), pz = DADD(c.oz, DMUL(dz, tmid));
    float v = 0.0f;
    bool miss = !p.cached;
    if (p.cached) {
        double u = 0.0;
        if (p.probe.mode != 2) {
            uint32_t r = (k == 0) ? lane_seed(p.rng_base, (u64)j) : __ldcg(s.rng[b] + j);
            r = xorshift32(r);
            __stcg(s.rng[nb] + j, r);
            u = DMUL((double)r, 2.3283064365386963e-10);  // / 2^32, exact
        }
        double dist = tmid;
        if (p.paged_dist) {
            const double ex = DSUB(px, c.ox), ey = DSUB(py, c.oy), ez = DSUB(pz, c.oz);
            dist = __dsqrt_rn(DADD(DADD(DMUL(ex, ex), DMUL(ey, ey)), DMUL(ez, ez)));
        }
        int rq, slot;
        const int sv = probe_one(px, py, pz, dist, u, p.probe, p.table, p.pool, (long long*)p.last_used,
                                 p.cache_frame, v, rq, slot);
        if (sv != rq) {
            // mrpd.py:215-225 miss filing at the requested LoD (native clipped, P6)
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
        if (sv < 0) {
            miss = true;
        } else {
            c_ex += (sv == rq);
            c_fb += (sv != rq);
        }
    }
    if (miss) {
        // sampler.py:276-279: the field at clip(world, 0, nextafter(1, 0))
        const double hmax = 0.99999999999999989;
        int bad = 0;
        v = w4_infer<kInr>(p.field, clampd(px, 0.0, hmax), clampd(py, 0.0, hmax), clampd(pz, 0.0, hmax), mlp, &bad);
        if (bad) w.ctr->nonfinite = 1;
        c_ms += 1;
    }
    const bool dead = c.smem_lut ? shade_one<true>(v, dt, c.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term,
                                                   cr, cg, cb, tr)
                                 : shade_one<false>(v, dt, c.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term,
                                                    cr, cg, cb, tr);
    AdvanceOut a;
    if (!dead && !last) {
        double cf = __longlong_as_double(cur);
        i64 ck = cur;
        f = advance_one(c.ox, c.oy, c.oz, dx, dy, dz, __ldg(w.ray_ten + id), __ldg(w.ray_tex + id), cf, ck, p.adv,
                        p.mu, a, c.occ, c.mu_s);
        cur = p.adv.adaptive ? __double_as_longlong(cf) : (long long)ck;
    }
    if (f) {
        __stcg(s.tmid[nb] + j, a.tmid);
        __stcg(s.dt[nb] + j, a.dt);
        __stcg(s.cur[nb] + j, cur);
        __stcg(s.cr[nb] + j, cr);
        __stcg(s.cg[nb] + j, cg);
        __stcg(s.cb[nb] + j, cb);
        __stcg(s.tr[nb] + j, tr);
    } else {
        w4_retire(p, __ldg(w.ray_pix + id), cr, cg, cb, tr);
    }
    }
    // publish slot j of S_{k+1}: state, one fence for the warp, then the tag
    __syncwarp();
    w4_fence_release();
    if (id >= 0 && !last)
        w4_st_rel(s.idt[nb] + j, ((unsigned long long)(k + 2) << 32) | (unsigned long long)(uint32_t)(f ? id : -1));
    return kW4Done;
}

template <int kInr>
__global__ void __launch_bounds__(kW4Threads, 1)
    k_wave4_march(const __grid_constant__ VcbFrameParams p, const __grid_constant__ FrameWs w,
                  const __grid_constant__ W4Ws s, int max_it) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int lane = threadIdx.x & 31;
    // ---- stage read-only tables in shared memory
    float* s_lut = s.sm_lut >= 0 ? reinterpret_cast<float*>(dsm + s.sm_lut) : nullptr;
    if (s_lut)
        for (int i = threadIdx.x; i < p.lut_size * 4; i += kW4Threads) s_lut[i] = __ldg(p.lut + i);
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    W4Ctx c;
    c.ox = p.cam.origin[0];
    c.oy = p.cam.origin[1];
    c.oz = p.cam.origin[2];
    c.mu_s = nullptr;
    c.occ = nullptr;
    c.lut = s_lut ? s_lut : p.lut;
    c.smem_lut = s_lut != nullptr;
    if (s.sm_mu >= 0) {
        float* mm = reinterpret_cast<float*>(dsm + s.sm_mu);
        for (long long i = threadIdx.x; i < cells; i += kW4Threads) mm[i] = __ldg(p.mu + i);
        c.mu_s = mm;
    } else if (s.sm_occ >= 0) {
        uint32_t* occ = reinterpret_cast<uint32_t*>(dsm + s.sm_occ);
        const int nwords = (int)((cells + 31) >> 5);
        for (int wd = threadIdx.x >> 5; wd < nwords; wd += kW4Threads / 32) {
            const long long q = (long long)wd * 32 + lane;
            const unsigned bb = __ballot_sync(0xffffffffu, q < cells && __ldg(p.mu + q) > 0.0f);
            if (lane == 0) occ[wd] = bb;
        }
        c.occ = occ;
    }
    MlpSmem mlp;
    mlp.w = mlp.b = nullptr;
    if (kInr != 0 && s.sm_mlp >= 0) stage_mlp(p.field, reinterpret_cast<float*>(dsm + s.sm_mlp), mlp);
    __syncthreads();

    const long long n0 = __ldcg(w.live);
    unsigned long long c_ex = 0, c_fb = 0, c_ms = 0;
    // ---- prologue units (rays -> S_0), then levels in order
    {
        const long long ngp = (n0 + 31) >> 5;
        for (;;) {
            long long t = 0;
            if (lane == 0) t = atomicAdd(s.tick, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= ngp) break;
            w4_prologue(p, w, s, c, t, n0, max_it);
        }
    }
    int k = 0;
    while (k < max_it) {
        long long t = 0;
        if (lane == 0) t = atomicAdd(s.tick + k + 1, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        const int r = w4_unit<kInr>(p, w, s, c, mlp, k, t, n0, max_it, c_ex, c_fb, c_ms);
        if (r == kW4End) break;
        if (r == kW4Void) k++;
    }
    if (k >= max_it && lane == 0) {
        // the capped frame's last level: make sure n_{max_it-1} gets published
        int spins = 0;
        while (w4_try_total(s, max_it - 1, n0) < 0 && !*(volatile int*)s.abort)
            if (++spins > 4) __nanosleep(128);
    }
    c_ex = warp_sum(c_ex);
    c_fb = warp_sum(c_fb);
    c_ms = warp_sum(c_ms);
    if (lane == 0) {
        if (c_ex) atomicAdd(s.cnt + 0, c_ex);
        if (c_fb) atomicAdd(s.cnt + 1, c_fb);
        if (c_ms) atomicAdd(s.cnt + 2, c_ms);
    }
}

// FrameStats from the per-level totals (mrpd.py:33-41 + sampler counters).
__global__ void k_wave4_stats(VcbFrameParams p, FrameWs w, W4Ws s, int max_it) {
    const long long n0 = w.live[0];
    long long req = 0;
    int it = 0;
    if (n0 > 0) {
        it = max_it;
        for (int k = 0; k < max_it; k++) {
            const unsigned long long v = s.total[k];
            const long long nk = (v & kW4Pub) ? (long long)(v & 0xFFFFFFFFull) : 0;
            if (nk == 0) {
                it = k + 1;
                break;
            }
            req += nk;
        }
    }
    p.stats->requests = req;
    p.stats->iterations = it;
    p.stats->rays = n0;
    p.stats->exact += s.cnt[0];
    p.stats->fallback += s.cnt[1];
    p.stats->miss += s.cnt[2];
    p.stats->misses_resolved = s.cnt[2];
    p.stats->nonfinite = w.ctr->nonfinite | (*s.abort ? 2 : 0);
}

static const void* wave4_kernel(int mode) {
    return mode == 1 ? (const void*)k_wave4_march<1>
                     : mode == 2 ? (const void*)k_wave4_march<2> : (const void*)k_wave4_march<0>;
}

void launch_rays(const VcbFrameParams& p, const FrameWs& w, cudaStream_t st);

int launch_wave4_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    FrameWs w;
    const int64_t need = frame_ws_layout(npix, max_it, p.workspace, &w);
    W4Ws s;
    const int64_t need4 = w4_layout(npix, max_it, (char*)p.workspace + need, &s);
    if (need + need4 > p.workspace_bytes)
        return set_error("march_frame: workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)(need + need4));
    const int mode = inr_mode(p.field);
    const int G = device_sms();
    int off = 0;
    auto take = [&](int bytes) {
        const int o = (off + 15) & ~15;
        off = o + bytes;
        return o;
    };
    s.sm_lut = (p.lut_size <= kW4LutMax) ? take(p.lut_size * 16) : -1;
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    s.sm_mu = s.sm_occ = -1;
    if (cells <= kW4MuSmemCells) s.sm_mu = take((int)cells * 4);
    else if (cells <= kW4OccMaxCells && p.adv.skip_empty) s.sm_occ = take((int)(((cells + 31) >> 5) * 4));
    s.sm_mlp = -1;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        s.sm_mlp = take((nw + nb) * 4);
    }
    s.sm_total = off;
    const void* fn = wave4_kernel(mode);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, off > 0 ? off : 1);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kW4Threads, off);
    if (per_sm < 1)
        return set_error("march_frame: frame kernel does not fit one CTA per SM (%d B shared)", off);
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(w.ctr_iter, 0, w.ctr_iter_bytes, st);
    cudaMemsetAsync(s.idt[0], 0, (size_t)s.nslots * 8, st);
    cudaMemsetAsync(s.idt[1], 0, (size_t)s.nslots * 8, st);
    cudaMemsetAsync(s.look, 0, (size_t)kW4Ring * s.maxg * 8, st);
    cudaMemsetAsync(s.total, 0, (size_t)(max_it + 2) * 8, st);
    cudaMemsetAsync(s.tick, 0, (size_t)(max_it + 2) * 4, st);
    cudaMemsetAsync(s.abort, 0, 16, st);
    cudaMemsetAsync(s.cnt, 0, 64, st);
    launch_rays(p, w, st);
    VcbFrameParams pc = p;
    FrameWs wc = w;
    W4Ws sc = s;
    int mi = max_it;
    void* args[4] = {&pc, &wc, &sc, &mi};
    if (ev) cudaEventRecord(ev[0], st);
    cudaError_t e = cudaLaunchCooperativeKernel(fn, G * per_sm, kW4Threads, args, off, st);
    if (ev) {
        cudaEventRecord(ev[1], st);
        *ev_used = 1;
    }
    if (e != cudaSuccess)
        return set_error("march_frame: cooperative launch (%d CTAs): %s", G * per_sm, cudaGetErrorString(e));
    k_wave4_stats<<<1, 1, 0, st>>>(p, w, s, max_it);
    *launches = 4;
    return check_launch("march_frame(wave4)");
}

}  // namespace cinr
