// Two-phase persistent wavefront march (default frame kernel), sm_100a, -fmad=false.
//
// Same iteration semantics as wave.cu (render/raymarch.py:72-115), different
// synchronisation: every iteration is
//   phase A  every CTA advances its round-robin tiles of the live buffer
//            (kernels.py:35-137), retires finished rays, stores each sampling
//            ray's advance output and one count per tile;
//   barrier
//   scan     each CTA scans all tile counts at once (block scan in shared
//            memory) -> the rank base of its tiles = the reference's RNG lanes
//            (P5) and the survivors' slots in the next buffer;
//   phase B  probe with stochastic LoD + MRPD walk + trilinear + stamps + miss
//            filing (kernels.py:166-273), inline true-miss inference
//            (sampler.py:276-279), shade (kernels.py:322-355), ordered write;
//   barrier
// No look-back chains: the rank of every tile is known after one barrier.
#include <cstddef>
#include <cstdio>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"

namespace cinr {

constexpr int kW2Threads = 256;
constexpr int kW2MaxTiles = 8192;  // tiles per iteration held in shared memory for the scan
constexpr long long kW2OccMaxCells = 1ll << 18;

struct W2Smem {
    int warp_tot[kW2Threads / 32];
    int tile_base[kW2MaxTiles];  // exclusive prefix of tile counts (this iteration)
    unsigned long long cnt[3];
};

__device__ __forceinline__ void w2_retire(const VcbFrameParams& p, int pix, double cr, double cg, double cb, double tr) {
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

__device__ __forceinline__ void w2_barrier(unsigned int* count, volatile unsigned int* gen, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned int*)gen, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// block-wide exclusive scan of one int per thread
__device__ __forceinline__ int w2_block_scan(int v, int* warp_tot, int& excl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kW2Threads / 32; i++) {
        const int t = warp_tot[i];
        base += (i < warp) ? t : 0;
        tot += t;
    }
    excl = base + x - v;
    __syncthreads();
    return tot;
}

template <int kInr>
__global__ void __launch_bounds__(kW2Threads, 2) k_wave2_march(VcbFrameParams p, FrameWs w, int max_it,
                                                               unsigned int* bar) {
    extern __shared__ __align__(16) unsigned char dsmem[];
    __shared__ W2Smem sm;
    MlpSmem mlp;
    int mlp_floats = 0;
    if (p.field.kind == 0) {
        int nb;
        mlp_floats = mlp_param_count(p.field, nb) + nb;
        stage_mlp(p.field, reinterpret_cast<float*>(dsmem), mlp);
    }
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    uint32_t* occ = nullptr;
    if (cells <= kW2OccMaxCells && p.adv.skip_empty) {
        occ = reinterpret_cast<uint32_t*>(dsmem + ((mlp_floats * 4 + 15) & ~15));
        const int nwords = (int)((cells + 31) >> 5);
        for (int wd = threadIdx.x >> 5; wd < nwords; wd += blockDim.x >> 5) {
            const long long c = (long long)wd * 32 + (threadIdx.x & 31);
            const unsigned b = __ballot_sync(0xffffffffu, c < cells && __ldg(p.mu + c) > 0.0f);
            if ((threadIdx.x & 31) == 0) occ[wd] = b;
        }
    }
    if (threadIdx.x < 3) sm.cnt[threadIdx.x] = 0;
    __syncthreads();
    const double ox = p.cam.origin[0], oy = p.cam.origin[1], oz = p.cam.origin[2];
    const int G = gridDim.x;
    int* tile_cnt = reinterpret_cast<int*>(w.status);  // per-tile sampling counts (reused each iteration)
    unsigned long long c_ex = 0, c_fb = 0, c_ms = 0;
    int k = 0;
    for (; k < max_it; k++) {
        const long long n = __ldcg(&w.live[k]);
        if (n == 0) break;
        const LiveBuf in = w.buf[k & 1];
        const LiveBuf out = w.buf[(k + 1) & 1];
        const long long rounds = (n + (long long)kTile * G - 1) / ((long long)kTile * G);
        const long long ntiles = rounds * G;
        // ---------------- phase A: advance
        for (long long tile = blockIdx.x; tile < ntiles; tile += G) {
            const long long lo = tile * n / ntiles, hi = (tile + 1) * n / ntiles;
            const long long i = lo + threadIdx.x;
            int flag = 0;
            if (i < hi) {
                const int32_t id = __ldcg(in.id + i);
                if (id >= 0) {
                    const long long cur = __ldcg(in.cur + i);
                    double cf = __longlong_as_double(cur);
                    i64 ck = cur;
                    AdvanceOut a;
                    flag = advance_one(ox, oy, oz, w.ray_dir[3 * id], w.ray_dir[3 * id + 1], w.ray_dir[3 * id + 2],
                                       w.ray_ten[id], w.ray_tex[id], cf, ck, p.adv, p.mu, a, occ);
                    if (flag) {
                        double* tp = w.mq_pos + 6 * i;  // advance outputs by live slot
                        __stcg(tp + 0, a.px);
                        __stcg(tp + 1, a.py);
                        __stcg(tp + 2, a.pz);
                        __stcg(tp + 3, a.dt);
                        __stcg(tp + 4, a.tmid);
                        __stcg(reinterpret_cast<long long*>(tp) + 5,
                               p.adv.adaptive ? __double_as_longlong(cf) : (long long)ck);
                    } else {
                        w2_retire(p, w.ray_pix[id], __ldcg(in.col + 3 * i), __ldcg(in.col + 3 * i + 1),
                                  __ldcg(in.col + 3 * i + 2), __ldcg(in.tr + i));
                    }
                }
            }
            if (i < hi) w.pix_keep[i] = (uint8_t)flag;  // sampling flag by live slot
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            const int wc = __popc(__ballot_sync(0xffffffffu, flag));
            if (lane == 0) sm.warp_tot[warp] = wc;
            __syncthreads();
            if (threadIdx.x == 0) {
                int t = 0;
#pragma unroll
                for (int q = 0; q < kW2Threads / 32; q++) t += sm.warp_tot[q];
                __stcg(tile_cnt + tile, t);
            }
            __syncthreads();
        }
        w2_barrier(bar, bar + 1, G);
        // ---------------- scan of all tile counts (redundantly in every CTA)
        {
            int carry = 0;
            for (long long t0 = 0; t0 < ntiles; t0 += kW2Threads) {
                const long long t = t0 + threadIdx.x;
                const int v = t < ntiles ? __ldcg(tile_cnt + t) : 0;
                int ex;
                const int tot = w2_block_scan(v, sm.warp_tot, ex);
                if (t < ntiles && t < kW2MaxTiles) sm.tile_base[t] = carry + ex;
                carry += tot;
            }
            if (blockIdx.x == 0 && threadIdx.x == 0) w.live[k + 1] = carry;
            __syncthreads();
        }
        // ---------------- phase B: rank, probe, miss filing, inference, shade, ordered write
        for (long long tile = blockIdx.x; tile < ntiles; tile += G) {
            const long long lo = tile * n / ntiles, hi = (tile + 1) * n / ntiles;
            const long long i = lo + threadIdx.x;
            const int flag = (i < hi) ? (int)w.pix_keep[i] : 0;
            int ex;
            w2_block_scan(flag, sm.warp_tot, ex);
            if (flag) {
                const long long j = (long long)sm.tile_base[tile] + ex;
                const int32_t id = __ldcg(in.id + i);
                const double* tp = w.mq_pos + 6 * i;
                const double px = __ldcg(tp + 0), py = __ldcg(tp + 1), pz = __ldcg(tp + 2), dt = __ldcg(tp + 3),
                             tmid = __ldcg(tp + 4);
                const long long curn = __ldcg(reinterpret_cast<const long long*>(tp) + 5);
                double cr = __ldcg(in.col + 3 * i), cg = __ldcg(in.col + 3 * i + 1), cb = __ldcg(in.col + 3 * i + 2),
                       tr = __ldcg(in.tr + i);
                int miss = 0, dead = 0;
                float v = 0.0f;
                if (!p.cached) {
                    miss = 1;
                } else {
                    double u = 0.0;
                    if (p.probe.mode != 2) {
                        uint32_t s = (k == 0) ? lane_seed(p.rng_base, (u64)j) : __ldcg(w.rng + j);
                        s = xorshift32(s);
                        __stcg(w.rng + j, s);
                        u = DMUL((double)s, 2.3283064365386963e-10);  // / 2^32, exact
                    }
                    double dist = tmid;
                    if (p.paged_dist) {
                        const double ex_ = DSUB(px, ox), ey = DSUB(py, oy), ez = DSUB(pz, oz);
                        dist = __dsqrt_rn(DADD(DADD(DMUL(ex_, ex_), DMUL(ey, ey)), DMUL(ez, ez)));
                    }
                    int rq, slot;
                    const int sv = probe_one(px, py, pz, dist, u, p.probe, p.table, p.pool, (long long*)p.last_used,
                                             p.cache_frame, v, rq, slot);
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
                        c_ex += (sv == rq);
                        c_fb += (sv != rq);
                    }
                }
                if (miss) {
                    const double hmax = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
                    int bad = 0;
                    v = field_eval<kInr>(p.field, clampd(px, 0.0, hmax), clampd(py, 0.0, hmax), clampd(pz, 0.0, hmax),
                                         mlp, &bad);
                    if (bad) w.ctr->nonfinite = 1;
                    c_ms += 1;
                }
                dead = shade_one(v, dt, p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg, cb, tr);
                if (dead) w2_retire(p, w.ray_pix[id], cr, cg, cb, tr);
                __stcg(out.id + j, dead ? -1 : id);
                __stcg(out.cur + j, curn);
                __stcg(out.col + 3 * j, cr);
                __stcg(out.col + 3 * j + 1, cg);
                __stcg(out.col + 3 * j + 2, cb);
                __stcg(out.tr + j, tr);
            }
        }
        w2_barrier(bar, bar + 1, G);
    }
    if (k == max_it) {
        const long long n = __ldcg(&w.live[k]);
        const LiveBuf in = w.buf[k & 1];
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)G * blockDim.x) {
            const int32_t id = __ldcg(in.id + i);
            if (id >= 0)
                w2_retire(p, w.ray_pix[id], __ldcg(in.col + 3 * i), __ldcg(in.col + 3 * i + 1),
                          __ldcg(in.col + 3 * i + 2), __ldcg(in.tr + i));
        }
    }
    c_ex = warp_sum(c_ex);
    c_fb = warp_sum(c_fb);
    c_ms = warp_sum(c_ms);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sm.cnt[0], c_ex);
        atomicAdd(&sm.cnt[1], c_fb);
        atomicAdd(&sm.cnt[2], c_ms);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&p.stats->exact, sm.cnt[0]);
        atomicAdd((unsigned long long*)&p.stats->fallback, sm.cnt[1]);
        atomicAdd((unsigned long long*)&p.stats->miss, sm.cnt[2]);
        if (blockIdx.x == 0) p.stats->iterations = k;
    }
}

__global__ void k_wave2_stats(VcbFrameParams p, FrameWs w) {
    long long req = 0;
    for (int k = 1; k <= (int)p.stats->iterations; k++) req += w.live[k];
    p.stats->requests = req;
    p.stats->rays = w.live[0];
    p.stats->misses_resolved = p.stats->miss;
    p.stats->nonfinite = w.ctr->nonfinite;
}

static const void* wave2_kernel(int mode) {
    return mode == 1 ? (const void*)k_wave2_march<1>
                     : mode == 2 ? (const void*)k_wave2_march<2> : (const void*)k_wave2_march<0>;
}

void launch_rays(const VcbFrameParams& p, const FrameWs& w, cudaStream_t st);

int launch_wave2_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    FrameWs w;
    const int64_t need = frame_ws_layout(npix, max_it, p.workspace, &w);
    if (need > p.workspace_bytes)
        return set_error("march_frame: workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)need);
    const int mode = inr_mode(p.field);
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
    if (cells <= kW2OccMaxCells && p.adv.skip_empty) smem = ((smem + 15) & ~15) + (int)(((cells + 31) >> 5) * 4);
    cudaFuncSetAttribute(wave2_kernel(mode), cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 0 ? smem : 1);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wave2_kernel(mode), kW2Threads, smem);
    if (per_sm < 1) per_sm = 1;
    int G = per_sm * device_sms();
    // the scan keeps one prefix per tile in shared memory
    if ((npix + (long long)kTile * G - 1) / ((long long)kTile * G) * G > kW2MaxTiles)
        return set_error("march_frame: %lld rays exceed the two-phase tile budget", (long long)npix);
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(w.ctr_iter, 0, w.ctr_iter_bytes, st);
    launch_rays(p, w, st);
    VcbFrameParams pc = p;
    FrameWs wc = w;
    int mi = max_it;
    unsigned int* bar = reinterpret_cast<unsigned int*>((char*)w.ctr + offsetof(FrameCounters, pad));
    void* args[4] = {&pc, &wc, &mi, (void*)&bar};
    if (ev) cudaEventRecord(ev[0], st);
    cudaError_t e = cudaLaunchCooperativeKernel(wave2_kernel(mode), G, kW2Threads, args, smem, st);
    if (ev) {
        cudaEventRecord(ev[1], st);
        *ev_used = 1;
    }
    if (e != cudaSuccess) return set_error("march_frame: cooperative launch (%d CTAs): %s", G, cudaGetErrorString(e));
    k_wave2_stats<<<1, 1, 0, st>>>(p, w);
    *launches = 4;
    return check_launch("march_frame(wave2)");
}

}  // namespace cinr
