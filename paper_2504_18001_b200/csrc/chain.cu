// Persistent chained ray march (the default frame kernel), sm_100a, -fmad=false.
//
// The reference's wavefront (raymarch.py:72-115) synchronises all rays every
// iteration; its only cross-ray coupling is the RNG lane of a sample, which is
// the sample's rank among all rays sampling in that iteration (P5: lane j =
// j-th entry of flatnonzero(sample_mask)).  Here every CTA owns a contiguous
// range of the (row-major, box-compacted) rays for the whole frame and runs its
// iterations on its own.  The only exchange is one prefix count per (CTA,
// iteration): after its advance pass a CTA publishes how many of its rays
// sample, and learns how many sample before it by a warp-parallel decoupled
// look-back over the CTAs below it (CTAs that finished publish a final marker
// and count as zero).  Low CTAs run ahead, high CTAs trail; no grid barrier.
//
// Lane states live in one global array: lane j is advanced once per iteration
// by whichever ray holds rank j.  The previous holder's write is ordered before
// the next holder's read through the release/acquire of the look-back words.
//
// True misses (sampler.py:276-279) are inferred inline, after the probe phase,
// by the CTA that owns the ray (the same field decoder as the brick fill).
#include <cstdio>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"

namespace cinr {

constexpr int kChainThreads = 256;
constexpr int kChainMaxPerSm = 4;

struct ChainWs {
    int32_t* ray_pix;       // [M]
    double* ray_dir;        // [3M]
    double* ray_ten;        // [M]
    double* ray_tex;        // [M]
    long long* cur;         // [M] cursor_f bits / cursor_k
    double* col;            // [3M]
    double* tr;             // [M]
    double* tmp;            // [5M] advance outputs (px,py,pz,dt,tmid) by ray
    uint32_t* rng;          // [M] lane states
    uint16_t* lists;        // [2 * M] per-CTA live lists (ray offsets within range)
    unsigned long long* status;  // [(max_it + 1) * G]
    unsigned long long* fin;     // [G]
    unsigned long long* cnt;     // [4] exact, fallback, miss, requests
    int* iters;                  // [0] max iterations run, [1] non-finite inference flag
};

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void retire_px(const VcbFrameParams& p, int pix, double cr, double cg, double cb,
                                          double tr) {
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

struct ChainSmem {
    int n_live;
    int n_next;
    int n_samp;
    int n_miss;
    long long prefix;
    int warp_tot[kChainThreads / 32];
    unsigned long long cnt[4];
};

// Exclusive block scan of one flag per thread; returns the block total.
__device__ __forceinline__ int block_scan(int flag, int* warp_tot, int& excl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kChainThreads / 32; i++) {
        const int t = warp_tot[i];
        base += (i < warp) ? t : 0;
        tot += t;
    }
    excl = base + wpre;
    __syncthreads();
    return tot;
}

template <int kInr>
__global__ void __launch_bounds__(kChainThreads, 2) k_chain_march(VcbFrameParams p, ChainWs w, const int* nrays, int G,
                                                               int max_it, unsigned int tag) {
    extern __shared__ __align__(16) unsigned char dsmem[];
    __shared__ ChainSmem sm;
    const int t = blockIdx.x;
    const long long M = *nrays;
    const long long r0 = M * t / G, r1 = M * (t + 1) / G;
    const int nr = (int)(r1 - r0);
    // dynamic smem: [MLP weights][flags nr bytes][miss list nr ints]
    float* mlp_s = reinterpret_cast<float*>(dsmem);
    int mlp_floats = 0;
    if (p.field.kind == 0) {
        int nb;
        mlp_floats = mlp_param_count(p.field, nb) + nb;
    }
    uint8_t* flags = reinterpret_cast<uint8_t*>(dsmem + ((mlp_floats * 4 + 15) & ~15));
    int* missq = reinterpret_cast<int*>(flags + ((nr + 15) & ~15));
    MlpSmem mlp;
    if (p.field.kind == 0) stage_mlp(p.field, mlp_s, mlp);
    uint16_t* live_a = w.lists + 2 * r0;
    uint16_t* live_b = live_a + nr;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) live_a[i] = (uint16_t)i;
    if (threadIdx.x < 4) sm.cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) sm.n_live = nr;
    __syncthreads();
    const double ox = p.cam.origin[0], oy = p.cam.origin[1], oz = p.cam.origin[2];
    const unsigned long long tagw = (unsigned long long)tag << 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int k = 0;
    for (; k < max_it; k++) {
        const int n = sm.n_live;
        if (n == 0) break;
        uint16_t* cur_list = (k & 1) ? live_b : live_a;
        uint16_t* next_list = (k & 1) ? live_a : live_b;
        // ---- phase A: advance every live ray (kernels.py:35-137); flags in smem
        int cnt_local = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const long long r = r0 + cur_list[i];
            int f = 0;
            if (w.tr[r] >= 0.0) {  // negative trans marks a ray retired by shading
                long long cb = w.cur[r];
                double cf = __longlong_as_double(cb);
                i64 ck = cb;
                AdvanceOut a;
                f = advance_one(ox, oy, oz, w.ray_dir[3 * r], w.ray_dir[3 * r + 1], w.ray_dir[3 * r + 2],
                                w.ray_ten[r], w.ray_tex[r], cf, ck, p.adv, p.mu, a);
                w.cur[r] = p.adv.adaptive ? __double_as_longlong(cf) : ck;
                if (f) {
                    double* tp = w.tmp + 5 * r;
                    tp[0] = a.px;
                    tp[1] = a.py;
                    tp[2] = a.pz;
                    tp[3] = a.dt;
                    tp[4] = a.tmid;
                } else {
                    retire_px(p, w.ray_pix[r], w.col[3 * r], w.col[3 * r + 1], w.col[3 * r + 2], w.tr[r]);
                }
            }
            flags[i] = (uint8_t)f;
            cnt_local += f;
        }
        cnt_local = warp_sum(cnt_local);
        if (lane == 0) sm.warp_tot[warp] = cnt_local;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int i = 0; i < kChainThreads / 32; i++) tot += sm.warp_tot[i];
            sm.n_samp = tot;
            sm.n_miss = 0;
            // publish this CTA's aggregate for iteration k (lane writes of k-1 precede it)
            __threadfence();
            st_release_u64(w.status + (size_t)k * G + t,
                           tagw | (t == 0 ? kFlagP : kFlagA) | (unsigned long long)tot);
        }
        __syncthreads();
        // ---- look-back: samples before this CTA at iteration k
        if (warp == 0) {
            long long acc = 0;
            if (t > 0) {
                long long base = t - 1;
                for (;;) {
                    const long long idx = base - lane;
                    unsigned long long s;
                    if (idx < 0) {
                        s = kFlagP;
                    } else {
                        for (;;) {
                            const unsigned long long fw = ld_acquire_u64(w.fin + idx);
                            if ((fw >> 32) == tag && (long long)(fw & 0xFFFFFFFFull) <= k) {
                                s = kFlagA;  // finished before iteration k: contributes nothing
                                break;
                            }
                            s = ld_acquire_u64(w.status + (size_t)k * G + idx);
                            if ((s >> 32) == tag && (s & (3ull << 30)) != 0) break;
                        }
                    }
                    const bool isP = (s & (3ull << 30)) == kFlagP;
                    const unsigned pm = __ballot_sync(0xffffffffu, isP);
                    long long v = (long long)(s & kValMask);
                    if (pm) {
                        const int first = __ffs(pm) - 1;
                        if (lane > first) v = 0;
                        acc += warp_sum(v);
                        break;
                    }
                    acc += warp_sum(v);
                    base -= 32;
                }
                if (lane == 0)
                    st_release_u64(w.status + (size_t)k * G + t,
                                   tagw | kFlagP | (unsigned long long)(acc + sm.n_samp));
            }
            if (lane == 0) {
                __threadfence();
                sm.prefix = acc;
            }
        }
        __syncthreads();
        const long long prefix = sm.prefix;
        // ---- phase B: rank, probe (stochastic LoD + MRPD walk), miss filing, shade
        int run = 0;  // samples in earlier chunks of this CTA's list
        for (int c0 = 0; c0 < n; c0 += blockDim.x) {
            const int i = c0 + threadIdx.x;
            const int f = (i < n) ? flags[i] : 0;
            int ex;
            const int tot = block_scan(f, sm.warp_tot, ex);
            if (f) {
                const long long r = r0 + cur_list[i];
                const long long j = prefix + run + ex;  // global rank = RNG lane
                const int slot_local = run + ex;        // position in the next live list
                const double* tp = w.tmp + 5 * r;
                const double px = tp[0], py = tp[1], pz = tp[2], dt = tp[3], tmid = tp[4];
                double cr = w.col[3 * r], cg = w.col[3 * r + 1], cb = w.col[3 * r + 2], tr = w.tr[r];
                int dead = 0, miss = 0;
                if (!p.cached) {
                    miss = 1;
                } else {
                    double u = 0.0;
                    if (p.probe.mode != 2) {
                        uint32_t s = (k == 0) ? lane_seed(p.rng_base, (u64)j) : __ldcg(w.rng + j);
                        s = xorshift32(s);
                        __stcg(w.rng + j, s);
                        u = DMUL((double)s, 2.3283064365386963e-10);
                    }
                    double dist = tmid;
                    if (p.paged_dist) {
                        const double ex_ = DSUB(px, ox), ey = DSUB(py, oy), ez = DSUB(pz, oz);
                        dist = __dsqrt_rn(DADD(DADD(DMUL(ex_, ex_), DMUL(ey, ey)), DMUL(ez, ez)));
                    }
                    float v;
                    int rq, slot;
                    const int sv = probe_one(px, py, pz, dist, u, p.probe, p.table, p.pool,
                                             (long long*)p.last_used, p.cache_frame, v, rq, slot);
                    if (sv != rq) {
                        const i64 span = p.probe.b << rq;
                        const double nx = clampd(DSUB(DMUL(px, p.probe.vx), 0.5), 0.0, DSUB(p.probe.vx, 1.0));
                        const double ny = clampd(DSUB(DMUL(py, p.probe.vy), 0.5), 0.0, DSUB(p.probe.vy, 1.0));
                        const double nz = clampd(DSUB(DMUL(pz, p.probe.vz), 0.5), 0.0, DSUB(p.probe.vz, 1.0));
                        const i64 bx = clampi((i64)floor(cell_div(DADD(nx, 1.0), (double)span)), 0, p.probe.grid[rq][0] - 1);
                        const i64 by = clampi((i64)floor(cell_div(DADD(ny, 1.0), (double)span)), 0, p.probe.grid[rq][1] - 1);
                        const i64 bz = clampi((i64)floor(cell_div(DADD(nz, 1.0), (double)span)), 0, p.probe.grid[rq][2] - 1);
                        warp_aggregated_add(p.miss_count, p.probe.offset[rq] + bx + p.probe.grid[rq][0] *
                                                                                 (by + p.probe.grid[rq][1] * bz));
                    }
                    if (sv < 0) {
                        miss = 1;
                    } else {
                        atomicAdd(&sm.cnt[sv == rq ? 0 : 1], 1ull);
                        dead = shade_one(v, dt, p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg,
                                         cb, tr);
                    }
                }
                if (miss) {
                    const int q = atomicAdd(&sm.n_miss, 1);
                    missq[q] = (int)(r - r0);
                } else {
                    w.col[3 * r] = cr;
                    w.col[3 * r + 1] = cg;
                    w.col[3 * r + 2] = cb;
                    if (dead) {
                        retire_px(p, w.ray_pix[r], cr, cg, cb, tr);
                        w.tr[r] = -1.0;
                    } else {
                        w.tr[r] = tr;
                    }
                }
                next_list[slot_local] = (uint16_t)(r - r0);
            }
            run += tot;
        }
        __syncthreads();
        // ---- phase C: true misses of this CTA -> field inference -> shade
        const int nm = sm.n_miss;
        if (nm) {
            if (threadIdx.x == 0) atomicAdd(&sm.cnt[2], (unsigned long long)nm);
            const double hi = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
            for (int q = threadIdx.x; q < nm; q += blockDim.x) {
                const long long r = r0 + missq[q];
                const double* tp = w.tmp + 5 * r;
                const float v = field_eval<kInr>(p.field, clampd(tp[0], 0.0, hi), clampd(tp[1], 0.0, hi),
                                           clampd(tp[2], 0.0, hi), mlp, &w.iters[1]);
                double cr = w.col[3 * r], cg = w.col[3 * r + 1], cb = w.col[3 * r + 2], tr = w.tr[r];
                const bool dead = shade_one(v, tp[3], p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr,
                                            cg, cb, tr);
                w.col[3 * r] = cr;
                w.col[3 * r + 1] = cg;
                w.col[3 * r + 2] = cb;
                if (dead) {
                    retire_px(p, w.ray_pix[r], cr, cg, cb, tr);
                    w.tr[r] = -1.0;
                } else {
                    w.tr[r] = tr;
                }
            }
        }
        if (threadIdx.x == 0) {
            sm.cnt[3] += (unsigned long long)sm.n_samp;
            sm.n_live = sm.n_samp;
        }
        __syncthreads();
    }
    // rays alive at the iteration cap are flushed as they stand (raymarch.py:117)
    if (k == max_it) {
        const int n = sm.n_live;
        uint16_t* cur_list = (k & 1) ? live_b : live_a;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const long long r = r0 + cur_list[i];
            if (w.tr[r] >= 0.0) retire_px(p, w.ray_pix[r], w.col[3 * r], w.col[3 * r + 1], w.col[3 * r + 2], w.tr[r]);
        }
    }
    if (threadIdx.x == 0) {
        // no samples from this CTA at iterations >= k
        __threadfence();
        st_release_u64(w.fin + t, tagw | (unsigned long long)k);
        atomicAdd(&w.cnt[0], sm.cnt[0]);
        atomicAdd(&w.cnt[1], sm.cnt[1]);
        atomicAdd(&w.cnt[2], sm.cnt[2]);
        atomicAdd(&w.cnt[3], sm.cnt[3]);
        atomicMax(&w.iters[0], k);
    }
}

// Box-hit rays, row-major, compacted in order (camera.py:144-154) + initial state.
__global__ void __launch_bounds__(kTile) k_chain_rays(VcbFrameParams p, FrameWs fw, ChainWs w, unsigned int tag) {
    __shared__ ScanSmem sm;
    const int W = p.cam.width, H = p.cam.height;
    const int64_t n = (int64_t)W * p.cam.rows;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    for (;;) {
        if (threadIdx.x == 0) sm.tile = atomicAdd(&fw.ctr->ticket_rays, 1);
        __syncthreads();
        const int64_t tile = sm.tile;
        __syncthreads();
        if (tile >= ntiles) break;
        const int64_t i = tile * kTile + threadIdx.x;
        Ray r;
        int flag = 0;
        if (i < n) {
            double fx, fy;
            film_coord((int)(i % W), p.cam.row0 + (int)(i / W) * p.cam.row_step, W, H, fx, fy);
            r = make_ray(fx, fy, p.cam);
            flag = r.keep;
            reinterpret_cast<float4*>(p.image)[frame_pixel(p, i)] = make_float4((float)p.bg[0], (float)p.bg[1], (float)p.bg[2], 0.0f);
        }
        long long excl;
        const uint32_t total = ordered_scan(flag, tile, fw.status, tag, sm, excl);
        if (flag) {
            const long long j = excl;
            w.ray_pix[j] = (int32_t)i;
            w.ray_dir[3 * j] = r.dx;
            w.ray_dir[3 * j + 1] = r.dy;
            w.ray_dir[3 * j + 2] = r.dz;
            w.ray_ten[j] = r.t0;
            w.ray_tex[j] = r.t1;
            w.cur[j] = p.adv.adaptive ? __double_as_longlong(r.t0) : 0ll;
            w.col[3 * j] = 0.0;
            w.col[3 * j + 1] = 0.0;
            w.col[3 * j + 2] = 0.0;
            w.tr[j] = 1.0;
        }
        if (tile == ntiles - 1 && threadIdx.x == kTile - 1) fw.live[0] = (int32_t)total;
    }
}

__global__ void k_chain_stats(VcbFrameParams p, FrameWs fw, ChainWs w) {
    p.stats->exact = (long long)w.cnt[0];
    p.stats->fallback = (long long)w.cnt[1];
    p.stats->miss = (long long)w.cnt[2];
    p.stats->requests = (long long)w.cnt[3];
    p.stats->iterations = w.iters[0];
    p.stats->rays = fw.live[0];
    p.stats->misses_resolved = (long long)w.cnt[2];
    p.stats->nonfinite = w.iters[1];
}

// workspace: FrameWs (its ray-compaction part) + ChainWs arrays
int64_t chain_ws_layout(int64_t n, int max_it, int G, void* base, FrameWs* fw, ChainWs* w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    const int64_t tiles = (n + kTile - 1) / kTile + 1;
    size_t o_st = take((size_t)tiles * 8), o_ctr = take(sizeof(FrameCounters)), o_it = take(64);
    size_t o_pix = take(n * 4), o_dir = take(n * 24), o_ten = take(n * 8), o_tex = take(n * 8), o_cur = take(n * 8),
           o_col = take(n * 24), o_tr = take(n * 8), o_tmp = take(n * 40), o_rng = take(n * 4), o_lists = take(n * 4),
           o_cst = take((size_t)(max_it + 1) * G * 8), o_fin = take((size_t)G * 8), o_cnt = take(64),
           o_iters = take(64);
    if (base) {
        char* b = (char*)base;
        fw->status = (unsigned long long*)(b + o_st);
        fw->max_tiles = tiles;
        fw->ctr = (FrameCounters*)(b + o_ctr);
        fw->live = (int*)(b + o_it);
        w->ray_pix = (int32_t*)(b + o_pix);
        w->ray_dir = (double*)(b + o_dir);
        w->ray_ten = (double*)(b + o_ten);
        w->ray_tex = (double*)(b + o_tex);
        w->cur = (long long*)(b + o_cur);
        w->col = (double*)(b + o_col);
        w->tr = (double*)(b + o_tr);
        w->tmp = (double*)(b + o_tmp);
        w->rng = (uint32_t*)(b + o_rng);
        w->lists = (uint16_t*)(b + o_lists);
        w->status = (unsigned long long*)(b + o_cst);
        w->fin = (unsigned long long*)(b + o_fin);
        w->cnt = (unsigned long long*)(b + o_cnt);
        w->iters = (int*)(b + o_iters);
    }
    return (int64_t)align_up(off, 256);
}

static const void* chain_kernel(int mode) {
    return mode == 1 ? (const void*)k_chain_march<1> : mode == 2 ? (const void*)k_chain_march<2> : (const void*)k_chain_march<0>;
}

static int chain_grid(int mode, int smem_bytes) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chain_kernel(mode), kChainThreads, smem_bytes);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > kChainMaxPerSm) per_sm = kChainMaxPerSm;
    return per_sm * device_sms();
}

int64_t chain_ws_bytes(int64_t npix, int max_it) {
    FrameWs fw;
    ChainWs w;
    return chain_ws_layout(npix, max_it < kMaxIterCap ? max_it : kMaxIterCap, kChainMaxPerSm * device_sms(), nullptr,
                           &fw, &w);
}

int launch_chain_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev,
                       int* ev_used) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    const int mode = inr_mode(p.field);
    int mlp_bytes = 0;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        mlp_bytes = (nw + nb) * 4;
    }
    // the grid fixes rays per CTA, which sizes the dynamic smem: iterate to a fixpoint
    int G = chain_grid(mode, 0);
    int smem = 0;
    for (int pass = 0; pass < 4; pass++) {
        const int64_t per = (npix + G - 1) / G + 1;
        smem = ((mlp_bytes + 15) & ~15) + (int)((per + 15) & ~15) + (int)(per * 4) + 64;
        if (smem > 48 * 1024) cudaFuncSetAttribute(chain_kernel(mode), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int G2 = chain_grid(mode, smem);
        if (G2 >= G) break;
        G = G2;
    }
    if ((npix + G - 1) / G > 65535) return set_error("march_frame: too many rays per CTA (%lld)", (long long)npix);
    FrameWs fw;
    ChainWs w;
    const int64_t need = chain_ws_layout(npix, max_it, kChainMaxPerSm * device_sms(), p.workspace, &fw, &w);
    if (need > p.workspace_bytes)
        return set_error("march_frame: workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)need);
    cudaMemsetAsync(fw.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(fw.live, 0, 64, st);
    cudaMemsetAsync(w.cnt, 0, 64, st);
    cudaMemsetAsync(w.iters, 0, 64, st);
    k_chain_rays<<<device_sms() * 4, kTile, 0, st>>>(p, fw, w, p.epoch * 16384u + 16383u);
    // every CTA of the chained march must be resident at once: the cooperative
    // launch guarantees it (and fails loudly instead of deadlocking if it cannot)
    VcbFrameParams pc = p;
    ChainWs wc = w;
    const int* nr = fw.live;
    int Gi = G, mi = max_it;
    unsigned int tg = p.epoch * 16384u;
    void* args[6] = {&pc, &wc, (void*)&nr, &Gi, &mi, &tg};
    if (ev) cudaEventRecord(ev[0], st);
    cudaError_t e = cudaLaunchCooperativeKernel(chain_kernel(mode), G, kChainThreads, args, smem, st);
    if (ev) {
        cudaEventRecord(ev[1], st);
        *ev_used = 1;
    }
    if (e != cudaSuccess) return set_error("march_frame: cooperative launch (%d CTAs): %s", G, cudaGetErrorString(e));
    k_chain_stats<<<1, 1, 0, st>>>(p, fw, w);
    *launches = 3;
    return check_launch("march_frame(chain)");
}

}  // namespace cinr
