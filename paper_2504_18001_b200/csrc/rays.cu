// Throughput-mode frame kernel ("fast path"), sm_100a, -fmad=false.
//
// One persistent CTA per SM; every lane owns one primary ray at a time and
// marches it to completion with the ray state in registers:
//
//   ticket -> pixel (8x4 pixel tiles per warp, so a warp's rays stay coherent)
//   raygen  (kernels.py:376-411; background for rays that miss the box)
//   loop    advance (kernels.py:35-137) -> stochastic LoD + MRPD probe +
//           trilinear + stamp + miss filing (kernels.py:166-273,
//           sampler.py:236-275) -> true-miss inference (sampler.py:276-279)
//           -> shade (kernels.py:322-355) -> early termination / iteration cap
//           (raymarch.py:72-117)
//   retire  rgb = color + T*bg, alpha = 1 - T (raymarch.py:57-60); the lane takes
//           the next ticket.
//
// There is no grid barrier and no per-iteration state round trip through HBM:
// the only global traffic is the sample's page-table entry and brick corners,
// the miss counters and the retired pixel.  The per-sample arithmetic is the
// parity path's (common.cuh) bit for bit; what differs is the RNG lane of the
// stochastic LoD.  The reference numbers lanes by the sample's rank among the
// samples of a wavefront iteration (sampler.py:206-213, P5), which needs a
// grid-wide scan per iteration.  Here lane = the ray's global film pixel
// (row * W + column): seed lane_seed(frame base, pixel) (sampler.py:39-45),
// one xorshift32 step per sample of that ray (sampler.py:51-58).  Same
// per-sample distribution (E[LoD] = D), and it needs no ordering, so band
// partitions of a frame draw exactly the numbers the whole frame would.  With
// LodPolicy(mode="off") no number is drawn and frames are bit-identical to the
// parity schedule (images, counters, stamps, miss reports).
//
// True misses are inferred by the warp that meets them: for the default INR the
// whole warp runs the tensor-core inference (mlp_warp.cuh, 32 samples per call)
// whenever any lane holds a miss, so its values are the parity path's.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"
#include "mlp_warp.cuh"

namespace cinr {

struct RmCfg {
    int sm_lut, sm_mu, sm_occ, sm_mlp;  // dynamic shared-memory offsets (-1 = not staged)
    int tiles_x;                         // 8-pixel tile columns
    int max_it;
    int max_skip;                        // empty macro cells one lane crosses per loop turn (0 = all)
    long long n_tickets;                 // 32 per 8x4 tile
    uint32_t* coarse;                    // [words] non-empty 4x4x4 super-cells (kFast 2), in the workspace
    int coarse_words;
    double4* ray_a;                      // [n] dx, dy, dz, t_enter of the box-hitting rays
    double2* ray_b;                      // [n] t_exit, (local pixel, film pixel) as two int32
    int* n_rays;                         // rays in the list (written by k_ray_setup)
    // a mapped host image: k_ray_setup lists the background pixels from the end of ray_b
    // and k_bg_fill stores them on a side stream while the march runs
    int* n_bg;
    int bg_list;
    long long cap;
};

// workspace after frame_ws_layout(0, ...): the ray list
constexpr int kCoarseMaxWords = 48 * 1024 / 4;  // super-cell bits kept in shared memory (48 KB)

inline int64_t rays_layout(int64_t npix, void* base, RmCfg* c) {
    const size_t a = align_up((size_t)npix * sizeof(double4), 256);
    const size_t b = align_up((size_t)npix * sizeof(double2), 256);
    const size_t o = align_up((size_t)kCoarseMaxWords * 4, 256);
    if (base && c) {
        c->ray_a = reinterpret_cast<double4*>(base);
        c->ray_b = reinterpret_cast<double2*>((char*)base + a);
        c->coarse = reinterpret_cast<uint32_t*>((char*)base + a + b);
    }
    return (int64_t)(a + b + o);
}

// Bitmask of the 4x4x4 super-cells of the macro grid holding any cell with a positive
// majorant (one warp per 32 super-cells; recomputed each frame, ~67 MB read at 4096^3).
__global__ void k_coarse_occ(const float* __restrict__ mu, int gx, int gy, int gz, uint32_t* out, int words) {
    const int lane = threadIdx.x & 31;
    const int sgx = (gx + 3) >> 2, sgy = (gy + 3) >> 2, sgz = (gz + 3) >> 2;
    const long long nsc = (long long)sgx * sgy * sgz;
    for (long long wd = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; wd < words;
         wd += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long sc = wd * 32 + lane;
        bool any = false;
        if (sc < nsc) {
            const int sx = (int)(sc % sgx), sy = (int)((sc / sgx) % sgy), sz = (int)(sc / ((long long)sgx * sgy));
            for (int z = sz * 4; z < min(sz * 4 + 4, gz) && !any; z++)
                for (int y = sy * 4; y < min(sy * 4 + 4, gy) && !any; y++)
                    for (int x = sx * 4; x < min(sx * 4 + 4, gx); x++)
                        if (__ldg(mu + x + (long long)gx * (y + (long long)gy * z)) > 0.0f) {
                            any = true;
                            break;
                        }
        }
        const unsigned b = __ballot_sync(0xffffffffu, any);
        if (lane == 0) out[wd] = b;
    }
}

int64_t rays_ws_bytes(int64_t npix, int max_it) {
    if (max_it > kMaxIterCap) max_it = kMaxIterCap;
    return frame_ws_layout(0, max_it, nullptr, nullptr) + rays_layout(npix, nullptr, nullptr);
}

// Ray setup (kernels.py:376-411, camera.py:129-154): tickets walk 8x4 pixel tiles; box
// hits are appended to the ray list warp by warp (list order is irrelevant here: the
// RNG lane is the pixel), every other pixel gets the background (raymarch.py:33-35).
__global__ void __launch_bounds__(256) k_ray_setup(const __grid_constant__ VcbFrameParams p, RmCfg cfg) {
    const int lane = threadIdx.x & 31;
    const int W = p.cam.width, H = p.cam.height, rows = p.cam.rows;
    const float4 bgv = make_float4((float)p.bg[0], (float)p.bg[1], (float)p.bg[2], 0.0f);
    if (blockIdx.x == 0 && threadIdx.x < sizeof(VcbFrameStats) / 8)
        reinterpret_cast<long long*>(p.stats)[threadIdx.x] = 0;  // the march accumulates after this kernel
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); t0 < cfg.n_tickets; t0 += stride) {
        const long long t = t0 + lane;
        const long long tile = t >> 5;
        const int x = (int)(tile % cfg.tiles_x) * 8 + (lane & 7);
        const int yl = (int)(tile / cfg.tiles_x) * 4 + (lane >> 3);
        bool keep = false;
        Ray r;
        int film_row = 0;
        if (x < W && yl < rows) {
            film_row = p.cam.row0 + yl * p.cam.row_step;
            double fx, fy;
            film_coord(x, film_row, W, H, fx, fy);
            r = make_ray(fx, fy, p.cam);
            keep = r.keep;
            if (!keep && !cfg.bg_list) reinterpret_cast<float4*>(p.image)[frame_pixel(p, (long long)yl * W + x)] = bgv;
        }
        const unsigned kb = __ballot_sync(0xffffffffu, keep);
        if (cfg.bg_list) {
            const bool bgp = x < W && yl < rows && !keep;
            const unsigned bm = __ballot_sync(0xffffffffu, bgp);
            int bb = 0;
            if (lane == 0 && bm) bb = atomicAdd(cfg.n_bg, __popc(bm));
            bb = __shfl_sync(0xffffffffu, bb, 0);
            if (bgp) {
                const long long j = cfg.cap - 1 - (bb + __popc(bm & ((1u << lane) - 1u)));
                cfg.ray_b[j] = make_double2(0.0, __hiloint2double(0, yl * W + x));
            }
        }
        int base = 0;
        if (lane == 0 && kb) base = atomicAdd(cfg.n_rays, __popc(kb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
            const int j = base + __popc(kb & ((1u << lane) - 1u));
            cfg.ray_a[j] = make_double4(r.dx, r.dy, r.dz, r.t0);
            cfg.ray_b[j] = make_double2(r.t1, __hiloint2double(film_row * W + x, yl * W + x));
        }
    }
}

// The background pixels k_ray_setup listed (bg_list), stored into the mapped host image
// by one CTA on a side stream while the march runs on the other SMs: their PCIe writes
// (~40% of a 1024^2 frame) then overlap the march instead of preceding it.
__global__ void __launch_bounds__(1024) k_bg_fill(const __grid_constant__ VcbFrameParams p, RmCfg cfg) {
    const float4 bgv = make_float4((float)p.bg[0], (float)p.bg[1], (float)p.bg[2], 0.0f);
    const long long n = __ldcg(cfg.n_bg);
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double2 rb = __ldcs(cfg.ray_b + (cfg.cap - 1 - i));
        reinterpret_cast<float4*>(p.image)[frame_pixel(p, __double2loint(rb.y))] = bgv;
    }
}

struct RmSmem {
    int4 lv[VCB_MAX_LOD];       // per LoD: brick grid + page-table offset (no indexed constant loads)
    unsigned long long cnt[7];  // exact, fallback, miss, samples, rays, decoded misses, deferred misses
    int max_k;
};

__device__ __forceinline__ void rm_retire(const VcbFrameParams& p, long long pix, double cr, double cg, double cb,
                                          double tr) {
    // raymarch.py:57-60: rgb = color + T*bg, alpha = 1 - T, then .astype(float32)
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

// The default INR at 32 positions of the warp (out of line: the inference's
// registers do not count against the march loop's budget).  Called converged.
static __device__ __noinline__ float rm_infer_warp(const VcbField& F, const MlpFrag* fr, double x, double y,
                                                   double z) {
    return inr_warp_default(F, fr, x, y, z);
}

template <int kInr>
static __device__ __noinline__ float rm_infer_lane(const VcbField& F, double x, double y, double z,
                                                   const MlpSmem m, int* bad) {
    return field_eval<kInr>(F, x, y, z, m, bad);
}

// kFast = 1: majorants and LUT in shared memory, adaptive steps, empty-space
// skipping (every BASELINE config): the run-time switches are folded away, which
// halves the loop's code (instruction-cache misses were a fifth of the stalls).
// (Memoising the adaptive step's division per ray costs 5 registers and spills: slower.)
template <int kInr, int NT, int kFast>
__global__ void __launch_bounds__(NT, 1)
    k_ray_march(const __grid_constant__ VcbFrameParams p, FrameCounters* ctr, const __grid_constant__ RmCfg cfg) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ RmSmem sm;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const double hmax = 0.99999999999999989;  // np.nextafter(1.0, 0.0)

    // ---- read-only tables in shared memory: LUT, majorants (or occupancy bits), MLP.
    // The LUT, the majorant grid and the super-cell bits are plain copies: one TMA bulk
    // copy each (cp.async.bulk), completing on one mbarrier, while the threads stage the
    // rest.
    __shared__ __align__(8) uint64_t tma_bar;
    float* s_lut = cfg.sm_lut >= 0 ? reinterpret_cast<float*>(dsm + cfg.sm_lut) : nullptr;
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    const float* mu_s = nullptr;
    const uint32_t* occ = nullptr;
    const uint32_t lut_bytes = s_lut ? (uint32_t)p.lut_size * 16u : 0u;
    const uint32_t mu_bytes = 0u;  // (the majorant grid: by the threads, measured faster at config 2)
    const uint32_t co_bytes = kFast >= 2 ? ((uint32_t)cfg.coarse_words * 4u + 15u) & ~15u : 0u;
    if (threadIdx.x == 0) {
        tma_stage_begin(&tma_bar, lut_bytes + mu_bytes + co_bytes);
        if (lut_bytes) tma_stage_copy(s_lut, p.lut, lut_bytes, &tma_bar);
        if (mu_bytes) tma_stage_copy(dsm + cfg.sm_mu, p.mu, mu_bytes, &tma_bar);
        if (co_bytes) tma_stage_copy(dsm + cfg.sm_occ, cfg.coarse, co_bytes, &tma_bar);
    }
    if (cfg.sm_mu >= 0) {
        float* m = reinterpret_cast<float*>(dsm + cfg.sm_mu);
        for (long long i = mu_bytes / 4 + threadIdx.x; i < cells; i += NT) m[i] = __ldg(p.mu + i);
        mu_s = m;
    } else if (kFast == 2) {
        occ = reinterpret_cast<const uint32_t*>(dsm + cfg.sm_occ);
    } else if (cfg.sm_occ >= 0) {
        uint32_t* o = reinterpret_cast<uint32_t*>(dsm + cfg.sm_occ);
        const int nwords = (int)((cells + 31) >> 5);
        for (int wd = threadIdx.x >> 5; wd < nwords; wd += NT / 32) {
            const long long q = (long long)wd * 32 + lane;
            const unsigned b = __ballot_sync(0xffffffffu, q < cells && __ldg(p.mu + q) > 0.0f);
            if (lane == 0) o[wd] = b;
        }
        occ = o;
    }
    MlpSmem mlp;
    mlp.w = mlp.b = nullptr;
    const MlpFrag* mfrag = nullptr;
    if (kInr == 1 && cfg.sm_mlp >= 0) {
        stage_mlp_frag(p.field, reinterpret_cast<MlpFrag*>(dsm + cfg.sm_mlp));
        mfrag = reinterpret_cast<const MlpFrag*>(dsm + cfg.sm_mlp);
    } else if (kInr != 0 && cfg.sm_mlp >= 0) {
        stage_mlp(p.field, reinterpret_cast<float*>(dsm + cfg.sm_mlp), mlp);
    }
    if (threadIdx.x <= p.probe.max_lod && threadIdx.x < VCB_MAX_LOD)
        sm.lv[threadIdx.x] = make_int4((int)p.probe.grid[threadIdx.x][0], (int)p.probe.grid[threadIdx.x][1],
                                       (int)p.probe.grid[threadIdx.x][2], (int)p.probe.offset[threadIdx.x]);
    if (threadIdx.x < 7) sm.cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) sm.max_k = 0;
    __syncthreads();
    tma_stage_wait(&tma_bar);
    const float* lut = s_lut ? s_lut : p.lut;

    const double ox = p.cam.origin[0], oy = p.cam.origin[1], oz = p.cam.origin[2];
    const bool use_rng = p.cached && p.probe.mode != 2;
    const bool adaptive = p.adv.adaptive != 0;

    // per-lane ray state
    bool has = false;
    int k = 0;               // samples taken by the lane's ray (the wavefront iteration index)
    long long pix = 0;       // local (band) pixel index
    double dx = 0.0, dy = 0.0, dz = 0.0, ten = 0.0, tex = 0.0;
    long long cur = 0;       // cursor_f bits (adaptive) or cursor_k
    double cr = 0.0, cg = 0.0, cb = 0.0, tr = 1.0;
    uint32_t rs = 0u;
    unsigned c_ex = 0, c_fb = 0, c_ms = 0, c_rays = 0, c_res = 0, c_def = 0;
    unsigned long long c_smp = 0;
    int max_k = 0, bad = 0;
    const long long n_list = __ldcg(cfg.n_rays);
    bool exhausted = n_list == 0;

    for (;;) {
        // ---- refill: lanes without a ray take the next rays of the list (one atomic per warp)
        if (!exhausted) {
            const unsigned need = __ballot_sync(0xffffffffu, !has);
            if (need) {
                long long base = 0;
                if (lane == 0) base = atomicAdd(&ctr->ticket_rays, __popc(need));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base + __popc(need) >= n_list) exhausted = true;
                if (!has) {
                    const long long t = base + __popc(need & lt_mask);
                    if (t < n_list) {
                        const double2* pa = reinterpret_cast<const double2*>(cfg.ray_a + t);
                        const double2 ra0 = __ldcs(pa), ra1 = __ldcs(pa + 1);
                        const double2 rb = __ldcs(cfg.ray_b + t);
                        has = true;
                        k = 0;
                        dx = ra0.x;
                        dy = ra0.y;
                        dz = ra1.x;
                        ten = ra1.y;
                        tex = rb.x;
                        pix = __double2loint(rb.y);
                        cur = adaptive ? __double_as_longlong(ten) : 0ll;
                        cr = cg = cb = 0.0;
                        tr = 1.0;
                        c_rays++;
                        if (use_rng) rs = lane_seed(p.rng_base, (u64)(unsigned)__double2hiint(rb.y));
                    }
                }
            }
        }
        if (!__any_sync(0xffffffffu, has)) break;

        // ---- advance (or the iteration-cap flush, raymarch.py:117); a lane crossing empty
        // space stops after max_skip cells and resumes the same advance next turn
        int samp = 0;
        AdvanceOut a;
        a.px = a.py = a.pz = 0.5;
        a.dt = a.tmid = 0.0;
        if (has) {
            int f = 0;
            if (k < cfg.max_it) {
                double cf = __longlong_as_double(cur);
                i64 ck = cur;
                if constexpr (kFast != 0)
                    f = advance_impl<kFast>(ox, oy, oz, dx, dy, dz, ten, tex, cf, ck, p.adv, p.mu, a, occ, mu_s,
                                            nullptr, cfg.max_skip);
                else
                    f = advance_one(ox, oy, oz, dx, dy, dz, ten, tex, cf, ck, p.adv, p.mu, a, occ, mu_s, nullptr,
                                    cfg.max_skip);
                cur = adaptive ? __double_as_longlong(cf) : (long long)ck;
            }
            if (f == 2) {
                // mid-advance: no sample this turn
            } else if (f) {
                samp = 1;
                k++;
            } else {
                rm_retire(p, pix, cr, cg, cb, tr);
                has = false;
                max_k = max(max_k, k);
            }
        }

        // ---- probe (stochastic LoD, MRPD walk, trilinear, stamp, miss filing)
        float v = 0.0f;
        int needinf = 0;
        if (samp) {
            c_smp++;
            if (!p.cached) {
                needinf = 1;
            } else {
                double u = 0.0;
                if (use_rng) {
                    rs = xorshift32(rs);
                    u = DMUL((double)rs, 2.3283064365386963e-10);  // / 2^32, exact
                }
                double dist = a.tmid;
                if (p.paged_dist) {
                    const double ex = DSUB(a.px, ox), ey = DSUB(a.py, oy), ez = DSUB(a.pz, oz);
                    dist = __dsqrt_rn(DADD(DADD(DMUL(ex, ex), DMUL(ey, ey)), DMUL(ez, ez)));
                }
                int rq, slot, rflat;
                const int sv = probe_one<kFast ? 1 : -1>(a.px, a.py, a.pz, dist, u, p.probe, p.table, p.pool,
                                         (long long*)p.last_used, p.cache_frame, v, rq, slot, sm.lv, &rflat);
                if (sv != rq) {
                    if (kFast || p.probe.b_pow2 != 0) {
                        warp_aggregated_add(p.miss_count, (i64)rflat);  // the probe's requested brick
                    } else {
                        // mrpd.py:215-225 miss filing at the requested LoD (native clipped, P6)
                        const i64 span = p.probe.b << rq;
                        const double nx = clampd(DSUB(DMUL(a.px, p.probe.vx), 0.5), 0.0, DSUB(p.probe.vx, 1.0));
                        const double ny = clampd(DSUB(DMUL(a.py, p.probe.vy), 0.5), 0.0, DSUB(p.probe.vy, 1.0));
                        const double nz = clampd(DSUB(DMUL(a.pz, p.probe.vz), 0.5), 0.0, DSUB(p.probe.vz, 1.0));
                        const int4 q = sm.lv[rq];
                        const i64 bx = clampi((i64)floor(cell_div(DADD(nx, 1.0), (double)span)), 0, q.x - 1);
                        const i64 by = clampi((i64)floor(cell_div(DADD(ny, 1.0), (double)span)), 0, q.y - 1);
                        const i64 bz = clampi((i64)floor(cell_div(DADD(nz, 1.0), (double)span)), 0, q.z - 1);
                        warp_aggregated_add(p.miss_count, (i64)q.w + bx + (i64)q.x * (by + (i64)q.y * bz));
                    }
                }
                if (sv < 0) {
                    needinf = 1;
                } else {
                    c_ex += (sv == rq);
                    c_fb += (sv != rq);
                }
            }
        }

        // ---- frame scheduler: a true miss is decoded only within the frame's budget; past
        // it the sample is filed (above) but not composited (p.miss_budget < 0: unbounded,
        // sampler.py:276-279)
        c_ms += needinf;
        if (p.miss_budget >= 0) {
            const unsigned nb = __ballot_sync(0xffffffffu, needinf);
            if (nb) {
                long long base = 0;
                if (lane == __ffs(nb) - 1) base = atomicAdd((unsigned long long*)&ctr->pad[2], (unsigned long long)__popc(nb));
                base = __shfl_sync(0xffffffffu, base, __ffs(nb) - 1);
                if (needinf && base + __popc(nb & lt_mask) >= p.miss_budget) {
                    needinf = 0;
                    samp = 0;  // not composited
                    c_def++;
                }
            }
        }

        // ---- true-miss inference (sampler.py:276-279): clip(world, 0, nextafter(1, 0))
        if (kInr == 1) {
            if (__any_sync(0xffffffffu, needinf)) {
                const double qx = needinf ? clampd(a.px, 0.0, hmax) : 0.5;
                const double qy = needinf ? clampd(a.py, 0.0, hmax) : 0.5;
                const double qz = needinf ? clampd(a.pz, 0.0, hmax) : 0.5;
                float vi = rm_infer_warp(p.field, mfrag, qx, qy, qz);
                if (needinf) {
                    if (!isfinite(vi)) bad = 1;
                    if (p.field.clip01) vi = vi < 0.0f ? 0.0f : (vi > 1.0f ? 1.0f : vi);
                    v = vi;
                }
            }
        } else if (needinf) {
            v = rm_infer_lane<kInr>(p.field, clampd(a.px, 0.0, hmax), clampd(a.py, 0.0, hmax),
                                    clampd(a.pz, 0.0, hmax), mlp, &bad);
        }
        c_res += needinf;

        // ---- shade + early termination
        if (samp) {
            const bool dead = (kFast || s_lut) ? shade_one<true>(v, a.dt, lut, p.lut_size, kFast ? 1 : p.adv.adaptive,
                                                                 p.adv.dt_base, p.term, cr, cg, cb, tr)
                                    : shade_one<false>(v, a.dt, lut, p.lut_size, p.adv.adaptive, p.adv.dt_base,
                                                       p.term, cr, cg, cb, tr);
            if (dead) {
                rm_retire(p, pix, cr, cg, cb, tr);
                has = false;
                max_k = max(max_k, k);
            }
        }
    }

    // ---- frame counters (FrameStats, mrpd.py:33-41)
    if (bad) atomicExch((unsigned long long*)&p.stats->nonfinite, 1ull);
    const unsigned long long t_ex = warp_sum((unsigned long long)c_ex);
    const unsigned long long t_fb = warp_sum((unsigned long long)c_fb);
    const unsigned long long t_ms = warp_sum((unsigned long long)c_ms);
    const unsigned long long t_sm = warp_sum(c_smp);
    const unsigned long long t_ry = warp_sum((unsigned long long)c_rays);
    const unsigned long long t_rs = warp_sum((unsigned long long)c_res);
    const unsigned long long t_df = warp_sum((unsigned long long)c_def);
    int mk = max_k;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    if (lane == 0) {
        atomicAdd(&sm.cnt[0], t_ex);
        atomicAdd(&sm.cnt[1], t_fb);
        atomicAdd(&sm.cnt[2], t_ms);
        atomicAdd(&sm.cnt[3], t_sm);
        atomicAdd(&sm.cnt[4], t_ry);
        if (t_rs) atomicAdd(&sm.cnt[5], t_rs);
        if (t_df) atomicAdd(&sm.cnt[6], t_df);
        atomicMax(&sm.max_k, mk);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        VcbFrameStats* S = p.stats;
        atomicAdd((unsigned long long*)&S->exact, sm.cnt[0]);
        atomicAdd((unsigned long long*)&S->fallback, sm.cnt[1]);
        atomicAdd((unsigned long long*)&S->miss, sm.cnt[2]);
        atomicAdd((unsigned long long*)&S->misses_resolved, sm.cnt[5]);
        if (sm.cnt[6]) atomicAdd((unsigned long long*)&S->deferred_misses, sm.cnt[6]);
        atomicAdd((unsigned long long*)&S->requests, sm.cnt[3]);
        atomicAdd((unsigned long long*)&S->rays, sm.cnt[4]);
        // wavefront iterations the parity schedule runs: the longest ray's samples + 1
        if (sm.cnt[4]) atomicMax((long long*)&S->iterations, (long long)sm.max_k + 1);
    }
}

static const void* ray_kernel(int mode, int nt, int fast) {
    if (fast == 2)
        return mode == 1 ? (const void*)k_ray_march<1, 512, 2>
                         : mode == 2 ? (const void*)k_ray_march<2, 512, 2> : (const void*)k_ray_march<0, 512, 2>;
    if (fast) {
        if (nt == 640)
            return mode == 1 ? (const void*)k_ray_march<1, 640, 1>
                             : mode == 2 ? (const void*)k_ray_march<2, 640, 1> : (const void*)k_ray_march<0, 640, 1>;
        return mode == 1 ? (const void*)k_ray_march<1, 512, 1>
                         : mode == 2 ? (const void*)k_ray_march<2, 512, 1> : (const void*)k_ray_march<0, 512, 1>;
    }
    return mode == 1 ? (const void*)k_ray_march<1, 512, 0>
                     : mode == 2 ? (const void*)k_ray_march<2, 512, 0> : (const void*)k_ray_march<0, 512, 0>;
}

// The side stream (and its two events) k_bg_fill runs on, one set per device.
static bool bg_side_stream(cudaStream_t* s, cudaEvent_t* a, cudaEvent_t* b) {
    static cudaStream_t streams[64] = {};
    static cudaEvent_t evs[64][2] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    if (streams[dev] == nullptr) {
        if (cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&evs[dev][0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&evs[dev][1], cudaEventDisableTiming) != cudaSuccess)
            return false;
    }
    *s = streams[dev];
    *a = evs[dev][0];
    *b = evs[dev][1];
    return true;
}

// nt: threads per CTA (one CTA per SM); max_skip: see advance_impl
int launch_ray_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used,
                     int nt, int max_skip) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    FrameWs w;
    const int64_t need0 = frame_ws_layout(0, max_it, p.workspace, &w);
    RmCfg cfg;
    const int64_t need = need0 + rays_layout(npix, (char*)p.workspace + need0, &cfg);
    if (need > p.workspace_bytes)
        return set_error("march_frame: workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)need);
    const int mode = inr_mode(p.field);
    cfg.max_it = max_it;
    cfg.max_skip = max_skip;
    cfg.tiles_x = (p.cam.width + 7) / 8;
    cfg.n_tickets = (long long)cfg.tiles_x * ((p.cam.rows + 3) / 4) * 32;
    cfg.n_rays = &w.ctr->pad[0];
    cfg.n_bg = &w.ctr->pad[4];
    cfg.cap = npix;
    {
        cudaPointerAttributes pa;
        cfg.bg_list = cudaPointerGetAttributes(&pa, p.image) == cudaSuccess && pa.type == cudaMemoryTypeHost ? 1 : 0;
        cudaGetLastError();
    }
    if (cfg.n_tickets >= (1ll << 31)) return set_error("march_frame: %lld pixels exceed the ticket range", (long long)npix);
    if (((uintptr_t)p.lut | (uintptr_t)p.mu) & 15)
        return set_error("march_frame: the LUT and majorant arrays must be 16-byte aligned (TMA)");
    int off = 0;
    auto take = [&](int bytes) {
        const int o = (off + 15) & ~15;
        off = o + bytes;
        return o;
    };
    constexpr int kSmemMax = 227 * 1024;
    cfg.sm_lut = (p.lut_size <= 4096) ? take(p.lut_size * 16) : -1;
    cfg.sm_mlp = -1;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        cfg.sm_mlp = take(mode == 1 ? (int)sizeof(MlpFrag) : (nw + nb) * 4);
    }
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    cfg.sm_mu = cfg.sm_occ = -1;
    // CINR_FORCE_SUPERCELL (tests only): the large-grid specialisation (super-cell bits,
    // super-cell jumps) on any macro grid, so small scenes exercise it against the oracle
    const bool force_sc = getenv("CINR_FORCE_SUPERCELL") != nullptr;
    if (force_sc) {
    } else if (off + 16 + cells * 4 <= kSmemMax) cfg.sm_mu = take((int)cells * 4);
    else if (p.adv.skip_empty && off + 16 + ((cells + 31) >> 5) * 4 <= kSmemMax)
        cfg.sm_occ = take((int)(((cells + 31) >> 5) * 4));
    // (the specialised kernels also assume power-of-two brick spans: shift-based LoD walk)
    const bool spec_ok = p.adv.adaptive && p.adv.skip_empty && p.probe.b_pow2 != 0;
    int fast = (cfg.sm_mu >= 0 && cfg.sm_lut >= 0 && spec_ok) ? 1 : 0;
    cfg.coarse_words = 0;
    if (!fast && cfg.sm_occ < 0 && cfg.sm_lut >= 0 && spec_ok && cells > 0) {
        // majorants too large for shared memory (4096^3: 256^3 cells): super-cell bits
        const long long nsc = (long long)((p.adv.gx + 3) / 4) * ((p.adv.gy + 3) / 4) * ((p.adv.gz + 3) / 4);
        const int words = (int)((nsc + 31) / 32);
        if (words <= kCoarseMaxWords) {
            // (the plain occupancy bitmask chosen above is dropped in this mode)
            cfg.sm_occ = take((words * 4 + 15) & ~15);  // whole 16-byte rows for the TMA copy
            cfg.coarse_words = words;
            fast = 2;
        }
    }
    if (mode == 2 || !fast) nt = 512;
    if (fast >= 2) nt = 512;
    if (off > kSmemMax) return set_error("march_frame: %d B of shared memory needed", off);
    const void* fn = ray_kernel(mode, nt, fast);
    const int per_sm = kernel_ctas_per_sm(fn, nt, off);
    if (per_sm < 1) return set_error("march_frame: ray kernel does not fit one CTA per SM (%d B shared)", off);
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    const int G = device_sms();
    if (ev) cudaEventRecord(ev[0], st);
    if (fast >= 2)
        k_coarse_occ<<<grid_for((int64_t)cfg.coarse_words * 32, 256), 256, 0, st>>>(
            p.mu, (int)p.adv.gx, (int)p.adv.gy, (int)p.adv.gz, cfg.coarse, cfg.coarse_words);
    k_ray_setup<<<grid_for(cfg.n_tickets, 256), 256, 0, st>>>(p, cfg);
    cudaStream_t side = nullptr;
    cudaEvent_t ev_setup = nullptr, ev_bg = nullptr;
    if (cfg.bg_list && bg_side_stream(&side, &ev_setup, &ev_bg)) {
        cudaEventRecord(ev_setup, st);
        cudaStreamWaitEvent(side, ev_setup, 0);
        k_bg_fill<<<1, 1024, 0, side>>>(p, cfg);
        cudaEventRecord(ev_bg, side);
    } else if (cfg.bg_list) {
        return set_error("march_frame: no side stream for the background pixels");
    }
    VcbFrameParams pc = p;
    FrameCounters* ctr = w.ctr;
    void* args[3] = {&pc, &ctr, &cfg};
    // with a mapped image one SM is left to k_bg_fill
    cudaError_t e = cudaLaunchKernel(fn, cfg.bg_list ? G - 1 : G, nt, args, off, st);
    if (cfg.bg_list) cudaStreamWaitEvent(st, ev_bg, 0);
    if (ev) {
        cudaEventRecord(ev[1], st);
        *ev_used = 1;
    }
    if (e != cudaSuccess) return set_error("march_frame: ray kernel launch: %s", cudaGetErrorString(e));
    *launches = (fast >= 2 ? 3 : 2) + (cfg.bg_list ? 1 : 0);
    return check_launch("march_frame(rays)");
}

}  // namespace cinr
