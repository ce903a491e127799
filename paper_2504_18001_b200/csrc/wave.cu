// Persistent wavefront ray march (default frame kernel), sm_100a, -fmad=false.
//
// One cooperative launch runs every iteration of the reference's wavefront
// loop (render/raymarch.py:72-115).  Per iteration k the live rays sit,
// compacted in the reference's order (row-major pixels among box hits, P18),
// in buffer k&1.  CTAs take 256-ray tiles of it by ticket; a tile advances its
// rays (kernels.py:35-137), ranks the sampling ones with a decoupled look-back
// over earlier tiles (that rank is the reference's RNG lane, P5, and the ray's
// slot in the next buffer), probes with stochastic LoD + MRPD walk + trilinear
// (kernels.py:166-273), files misses, infers true misses inline
// (sampler.py:276-279) and shades (kernels.py:322-355) — ray state stays in
// registers for the whole tile.  One grid barrier separates iterations.
// Work is balanced dynamically every iteration (all SMs share all live rays).
#include <cstddef>
#include <cstdio>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"

namespace cinr {

constexpr int kWaveThreads = 256;
constexpr long long kOccMaxCells = 1ll << 18;  // 32 KB of shared memory
static_assert(kWaveThreads == kTile, "tile = one ray per thread");

struct WaveSmem {
    ScanSmem scan;
    long long wsum[kWaveThreads / 32];
    unsigned long long cnt[3];
};

__device__ __forceinline__ void retire_w(const VcbFrameParams& p, int pix, double cr, double cg, double cb, double tr) {
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

// sense-reversing grid barrier over the cooperative grid
__device__ __forceinline__ void grid_barrier(unsigned int* count, volatile unsigned int* gen, unsigned int nblocks) {
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

// Rank of each sampling ray of tile (round r, column c) of iteration k.  Every
// tile publishes its own count (agg) and, once known, its inclusive prefix
// (incl).  A tile reads, in parallel, the aggs of the c tiles before it in its
// round plus the incl of the last tile of the previous round: one step instead
// of a 32-wide walk back through the round.
__device__ __forceinline__ long long round_scan(int flag, long long tile, int G, unsigned long long* agg,
                                                unsigned long long* incl, unsigned int tag, WaveSmem& sm,
                                                long long& rank, long long& total_incl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) sm.scan.warp_tot[warp] = __popc(bal);
    __syncthreads();
    int wbase = 0, btot = 0;
#pragma unroll
    for (int i = 0; i < kWaveThreads / 32; i++) {
        const int t = sm.scan.warp_tot[i];
        wbase += (i < warp) ? t : 0;
        btot += t;
    }
    const unsigned long long tagw = (unsigned long long)tag << 32;
    if (threadIdx.x == 0) st_volatile_u64(agg + tile, tagw | (unsigned long long)btot);
    const long long r = tile / G, c = tile - r * G, base = r * G;
    long long acc = 0;
    for (long long q = threadIdx.x; q < c; q += blockDim.x) {
        unsigned long long s;
        do {
            s = ld_volatile_u64(agg + base + q);
        } while ((s >> 32) != tag);
        acc += (long long)(s & 0xFFFFFFFFull);
    }
    if (threadIdx.x == blockDim.x - 1 && r > 0) {
        unsigned long long s;
        do {
            s = ld_volatile_u64(incl + base - 1);
        } while ((s >> 32) != tag);
        acc += (long long)(s & 0xFFFFFFFFull);
    }
    acc = warp_sum(acc);
    if (lane == 0) sm.wsum[warp] = acc;
    __syncthreads();
    long long pre = 0;
#pragma unroll
    for (int i = 0; i < kWaveThreads / 32; i++) pre += sm.wsum[i];
    if (threadIdx.x == 0) st_volatile_u64(incl + tile, tagw | (unsigned long long)(pre + btot));
    rank = pre + wbase + wpre;
    total_incl = pre + btot;
    __syncthreads();  // sm reuse by the next tile
    return pre;
}

template <int kInr>
__global__ void __launch_bounds__(kWaveThreads, 2) k_wave_march(VcbFrameParams p, FrameWs w, int max_it,
                                                                unsigned int* bar) {
    extern __shared__ __align__(16) unsigned char dsmem[];
    __shared__ WaveSmem sm;
    MlpSmem mlp;
    int mlp_floats = 0;
    if (p.field.kind == 0) {
        int nb;
        mlp_floats = mlp_param_count(p.field, nb) + nb;
        stage_mlp(p.field, reinterpret_cast<float*>(dsmem), mlp);
    }
    // non-empty-cell bitmask of the macro grid in shared memory (when it fits)
    const long long cells = p.adv.gx * p.adv.gy * p.adv.gz;
    uint32_t* occ = nullptr;
    if (cells <= kOccMaxCells && p.adv.skip_empty) {
        occ = reinterpret_cast<uint32_t*>(dsmem + ((mlp_floats * 4 + 15) & ~15));
        const int nwords = (int)((cells + 31) >> 5);
        for (int wd = threadIdx.x >> 5; wd < nwords; wd += blockDim.x >> 5) {
            const long long c = (long long)wd * 32 + (threadIdx.x & 31);
            const unsigned b = __ballot_sync(0xffffffffu, c < cells && __ldg(p.mu + c) > 0.0f);
            if ((threadIdx.x & 31) == 0) occ[wd] = b;
        }
    }
    __syncthreads();
    if (threadIdx.x < 3) sm.cnt[threadIdx.x] = 0;
    const double ox = p.cam.origin[0], oy = p.cam.origin[1], oz = p.cam.origin[2];
    const int lane = threadIdx.x & 31;
    unsigned long long c_ex = 0, c_fb = 0, c_ms = 0;
    int k = 0;
    for (; k < max_it; k++) {
        const long long n = __ldcg(&w.live[k]);
        if (n == 0) break;
        const LiveBuf in = w.buf[k & 1];
        const LiveBuf out = w.buf[(k + 1) & 1];
        // even tiles: the iteration's n rays split into G * rounds tiles of <= 256,
        // so every CTA works the same number of rounds (no partial last round)
        const int G = gridDim.x;
        const long long rounds = (n + (long long)kTile * G - 1) / ((long long)kTile * G);
        const long long ntiles = rounds * G;
        const unsigned int tag = p.epoch * 16384u + (unsigned int)k;
        // static round-robin: CTA c walks tiles c, c+G, c+2G, ... in increasing order,
        // so every rank predecessor is done or in flight (no deadlock)
        for (long long tile = blockIdx.x; tile < ntiles; tile += G) {
            const long long lo = tile * n / ntiles, hi = (tile + 1) * n / ntiles;
            const long long i = lo + threadIdx.x;
            int flag = 0;
            int32_t id = -1;
            double cf = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, tr = 1.0;
            i64 ck = 0;
            AdvanceOut a;
            if (i < hi) {
                id = __ldcg(in.id + i);
                if (id >= 0) {
                    const long long cur = __ldcg(in.cur + i);
                    cf = __longlong_as_double(cur);
                    ck = cur;
                    cr = __ldcg(in.col + 3 * i);
                    cg = __ldcg(in.col + 3 * i + 1);
                    cb = __ldcg(in.col + 3 * i + 2);
                    tr = __ldcg(in.tr + i);
                    flag = advance_one(ox, oy, oz, w.ray_dir[3 * id], w.ray_dir[3 * id + 1], w.ray_dir[3 * id + 2],
                                       w.ray_ten[id], w.ray_tex[id], cf, ck, p.adv, p.mu, a, occ);
                    if (!flag) retire_w(p, w.ray_pix[id], cr, cg, cb, tr);
                }
            }
            long long j;
            const uint32_t total = ordered_scan(flag, tile, w.status, tag, sm.scan, j);
            if (tile == ntiles - 1 && threadIdx.x == kTile - 1) w.live[k + 1] = (int)total;
            int miss = 0, dead = 0;
            float v = 0.0f;
            if (flag) {
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
                    double dist = a.tmid;
                    if (p.paged_dist) {
                        const double ex = DSUB(a.px, ox), ey = DSUB(a.py, oy), ez = DSUB(a.pz, oz);
                        dist = __dsqrt_rn(DADD(DADD(DMUL(ex, ex), DMUL(ey, ey)), DMUL(ez, ez)));
                    }
                    int rq, slot;
                    const int sv = probe_one(a.px, a.py, a.pz, dist, u, p.probe, p.table, p.pool,
                                             (long long*)p.last_used, p.cache_frame, v, rq, slot);
                    if (sv != rq) {
                        const i64 span = p.probe.b << rq;
                        const double nx = clampd(DSUB(DMUL(a.px, p.probe.vx), 0.5), 0.0, DSUB(p.probe.vx, 1.0));
                        const double ny = clampd(DSUB(DMUL(a.py, p.probe.vy), 0.5), 0.0, DSUB(p.probe.vy, 1.0));
                        const double nz = clampd(DSUB(DMUL(a.pz, p.probe.vz), 0.5), 0.0, DSUB(p.probe.vz, 1.0));
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
                        dead = shade_one(v, a.dt, p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg,
                                         cb, tr);
                        if (dead) retire_w(p, w.ray_pix[id], cr, cg, cb, tr);
                    }
                }
            }
            // true misses: infer through the field (inputs clamped to
            // [0, nextafter(1,0)], sampler.py:119-120), then shade
            {
                if (miss) {
                    const double hi = 0.99999999999999989;
                    int bad = 0;
                    v = field_eval<kInr>(p.field, clampd(a.px, 0.0, hi), clampd(a.py, 0.0, hi), clampd(a.pz, 0.0, hi),
                                         mlp, &bad);
                    if (bad) w.ctr->nonfinite = 1;
                    c_ms += 1;
                    dead = shade_one(v, a.dt, p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg, cb,
                                     tr);
                    if (dead) retire_w(p, w.ray_pix[id], cr, cg, cb, tr);
                }
            }
            if (flag) {
                __stcg(out.id + j, dead ? -1 : id);
                __stcg(out.cur + j, p.adv.adaptive ? __double_as_longlong(cf) : (long long)ck);
                __stcg(out.col + 3 * j, cr);
                __stcg(out.col + 3 * j + 1, cg);
                __stcg(out.col + 3 * j + 2, cb);
                __stcg(out.tr + j, tr);
            }
        }
        grid_barrier(bar, bar + 1, gridDim.x);
    }
    // rays alive at the iteration cap are flushed as they stand (raymarch.py:117)
    if (k == max_it) {
        const long long n = __ldcg(&w.live[k]);
        const LiveBuf in = w.buf[k & 1];
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
            const int32_t id = __ldcg(in.id + i);
            if (id >= 0)
                retire_w(p, w.ray_pix[id], __ldcg(in.col + 3 * i), __ldcg(in.col + 3 * i + 1), __ldcg(in.col + 3 * i + 2),
                         __ldcg(in.tr + i));
        }
    }
    // counters: warp-reduce, one shared add per warp, one global add per CTA
    c_ex = warp_sum(c_ex);
    c_fb = warp_sum(c_fb);
    c_ms = warp_sum(c_ms);
    if (lane == 0) {
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

__global__ void k_wave_stats(VcbFrameParams p, FrameWs w) {
    long long req = 0;
    for (int k = 1; k <= (int)p.stats->iterations; k++) req += w.live[k];
    p.stats->requests = req;
    p.stats->rays = w.live[0];
    p.stats->misses_resolved = p.stats->miss;
    p.stats->nonfinite = w.ctr->nonfinite;
}

static const void* wave_kernel(int mode) {
    return mode == 1 ? (const void*)k_wave_march<1> : mode == 2 ? (const void*)k_wave_march<2> : (const void*)k_wave_march<0>;
}

void launch_rays(const VcbFrameParams& p, const FrameWs& w, cudaStream_t st);

int launch_wave_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used) {
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
    if (cells <= kOccMaxCells && p.adv.skip_empty) smem = ((smem + 15) & ~15) + (int)(((cells + 31) >> 5) * 4);
    if (smem > 48 * 1024) cudaFuncSetAttribute(wave_kernel(mode), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wave_kernel(mode), kWaveThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int G = per_sm * device_sms();
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(w.ctr_iter, 0, w.ctr_iter_bytes, st);
    launch_rays(p, w, st);
    VcbFrameParams pc = p;
    FrameWs wc = w;
    int mi = max_it;
    unsigned int* bar = reinterpret_cast<unsigned int*>((char*)w.ctr + offsetof(FrameCounters, pad));  // count, gen
    void* args[4] = {&pc, &wc, &mi, (void*)&bar};
    if (ev) cudaEventRecord(ev[0], st);
    cudaError_t e = cudaLaunchCooperativeKernel(wave_kernel(mode), G, kWaveThreads, args, smem, st);
    if (ev) {
        cudaEventRecord(ev[1], st);
        *ev_used = 1;
    }
    if (e != cudaSuccess) return set_error("march_frame: cooperative launch (%d CTAs): %s", G, cudaGetErrorString(e));
    k_wave_stats<<<1, 1, 0, st>>>(p, w);
    *launches = 4;
    return check_launch("march_frame(wave)");
}

}  // namespace cinr
