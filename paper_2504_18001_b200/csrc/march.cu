// Wavefront cached ray march on sm_100a (compiled with -fmad=false).
//
// Frame structure (render/raymarch.py:25-120, sampler.py:196-280):
//   raygen + ordered compaction of box-hitting rays (camera.py:129-154)
//   for k < max_iterations while rays live:
//     k_march_iter  : advance -> sample rank via decoupled look-back (= the
//                     reference's RNG lane / compaction index) -> probe with
//                     stochastic LoD + MRPD walk + trilinear -> stamp -> miss
//                     counting -> shade hits -> ordered write of survivors
//     k_miss_shade  : true misses inferred through the field, then shaded
//   flush of rays alive at the iteration cap (raymarch.py:117)
//
// Ray order is the reference's row-major pixel order restricted to box hits,
// preserved by every compaction, so the rank of a ray among the rays sampling
// in iteration k equals the lane index numpy's flatnonzero() gives it (P5/P18).
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "fields.cuh"
#include "march.cuh"

namespace cinr {

// ----------------------------------------------------------------- operator passes
__global__ void k_raygen_pass(int64_t n, const double* __restrict__ base, const double* __restrict__ rot,
                              const double* __restrict__ origin, double tan_h, double tan_v, double* dirs,
                              double* t0, double* t1, uint8_t* keep) {
    VcbCamera c;
    for (int i = 0; i < 9; i++) c.rot[i] = rot[i];
    for (int i = 0; i < 3; i++) c.origin[i] = origin[i];
    c.tan_h = tan_h;
    c.tan_v = tan_v;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        Ray r = make_ray(base[2 * i], base[2 * i + 1], c);
        dirs[3 * i] = r.dx;
        dirs[3 * i + 1] = r.dy;
        dirs[3 * i + 2] = r.dz;
        t0[i] = r.t0;
        t1[i] = r.t1;
        keep[i] = r.keep ? 1 : 0;
    }
}

__global__ void k_advance_pass(int64_t n, const double* __restrict__ o, const double* __restrict__ d,
                               const double* __restrict__ t_en, const double* __restrict__ t_ex, double* cursor_f,
                               int64_t* cursor_k, const uint8_t* __restrict__ active, VcbMarchStatic S,
                               const float* __restrict__ mu, double* out_pos, double* out_dt, double* out_tmid,
                               uint8_t* sample_mask, uint8_t* done_mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        sample_mask[i] = 0;
        done_mask[i] = 0;
        if (!active[i]) continue;
        double cf = cursor_f[i];
        i64 ck = cursor_k[i];
        AdvanceOut a;
        int s = advance_one(o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1], d[3 * i + 2], t_en[i],
                            t_ex[i], cf, ck, S, mu, a);
        cursor_f[i] = cf;
        cursor_k[i] = ck;
        if (!s) {
            done_mask[i] = 1;
            continue;
        }
        out_pos[3 * i] = a.px;
        out_pos[3 * i + 1] = a.py;
        out_pos[3 * i + 2] = a.pz;
        out_dt[i] = a.dt;
        out_tmid[i] = a.tmid;
        sample_mask[i] = 1;
    }
}

__global__ void k_probe_pass(int64_t n, const double* __restrict__ pos, const double* __restrict__ dist,
                             const double* __restrict__ u, VcbProbeStatic P, const int32_t* __restrict__ table,
                             const float* __restrict__ pool, int64_t* last_used, int64_t frame, float* values,
                             int8_t* served, int8_t* req, unsigned long long* counts) {
    unsigned long long ex = 0, fb = 0, ms = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v;
        int rq, slot;
        int sv = probe_one(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], dist[i], u[i], P, table, pool,
                           (long long*)last_used, frame, v, rq, slot);
        values[i] = v;
        served[i] = (int8_t)sv;
        req[i] = (int8_t)rq;
        int gap = sv - rq;
        ex += gap == 0;
        fb += gap > 0;
        ms += gap < 0;
    }
    ex = warp_sum(ex);
    fb = warp_sum(fb);
    ms = warp_sum(ms);
    if ((threadIdx.x & 31) == 0) {
        if (ex) atomicAdd(counts + 0, ex);
        if (fb) atomicAdd(counts + 1, fb);
        if (ms) atomicAdd(counts + 2, ms);
    }
}

__global__ void k_shade_pass(int64_t n, const int64_t* __restrict__ rows, const float* __restrict__ values,
                             const double* __restrict__ dt, const float* __restrict__ lut, int lut_size, int adaptive,
                             double dt_base, double term, double* color, double* trans, uint8_t* dead) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = rows[j];
        double cr = color[3 * i], cg = color[3 * i + 1], cb = color[3 * i + 2], tr = trans[i];
        bool d = shade_one(values[j], dt[j], lut, lut_size, adaptive, dt_base, term, cr, cg, cb, tr);
        color[3 * i] = cr;
        color[3 * i + 1] = cg;
        color[3 * i + 2] = cb;
        trans[i] = tr;
        if (d) dead[j] = 1;
    }
}

__global__ void k_pow_dd(int64_t n, const double* x, const double* y, double* out, int accurate) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = accurate ? pow_dd_accurate(x[i], y[i]) : pow_dd(x[i], y[i]);
}

// ----------------------------------------------------------------- frame march
__device__ __forceinline__ void retire(const VcbFrameParams& p, int pix, double cr, double cg, double cb, double tr) {
    // raymarch.py:57-60: rgb = color + T*bg, alpha = 1 - T, then .astype(float32)
    float4 o;
    o.x = __double2float_rn(DADD(cr, DMUL(tr, p.bg[0])));
    o.y = __double2float_rn(DADD(cg, DMUL(tr, p.bg[1])));
    o.z = __double2float_rn(DADD(cb, DMUL(tr, p.bg[2])));
    o.w = __double2float_rn(DSUB(1.0, tr));
    reinterpret_cast<float4*>(p.image)[frame_pixel(p, pix)] = o;
}

// Pixel pass: background everywhere (raymarch.py:33-35), box hits flagged.
__global__ void k_raygen_frame(VcbFrameParams p, FrameWs w) {
    const int W = p.cam.width, H = p.cam.height;
    const int64_t n = (int64_t)W * p.cam.rows;
    float4 bg = make_float4((float)p.bg[0], (float)p.bg[1], (float)p.bg[2], 0.0f);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double fx, fy;
        film_coord((int)(i % W), p.cam.row0 + (int)(i / W) * p.cam.row_step, W, H, fx, fy);
        Ray r = make_ray(fx, fy, p.cam);
        reinterpret_cast<float4*>(p.image)[frame_pixel(p, i)] = bg;
        w.pix_keep[i] = r.keep ? 1 : 0;
    }
}

// Ordered compaction of box hits -> ray arrays + initial live state (camera.py:144-154,
// raymarch.py:50-56).  Same decoupled look-back as the march iterations.
__global__ void __launch_bounds__(kTile) k_compact_rays(VcbFrameParams p, FrameWs w) {
    __shared__ ScanSmem sm;
    const int W = p.cam.width, H = p.cam.height;
    const int64_t n = (int64_t)W * p.cam.rows;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    for (;;) {
        if (threadIdx.x == 0) sm.tile = atomicAdd(&w.ctr->ticket_rays, 1);
        __syncthreads();
        const int64_t tile = sm.tile;
        __syncthreads();
        if (tile >= ntiles) break;
        const int64_t i = tile * kTile + threadIdx.x;
        int flag = (i < n) ? w.pix_keep[i] : 0;
        long long excl;
        uint32_t total = ordered_scan(flag, tile, w.status, p.epoch * 16384u + 16383u, sm, excl);
        if (flag) {
            double fx, fy;
            film_coord((int)(i % W), p.cam.row0 + (int)(i / W) * p.cam.row_step, W, H, fx, fy);
            Ray r = make_ray(fx, fy, p.cam);
            const int64_t j = excl;
            w.ray_pix[j] = (int32_t)i;
            w.ray_dir[3 * j] = r.dx;
            w.ray_dir[3 * j + 1] = r.dy;
            w.ray_dir[3 * j + 2] = r.dz;
            w.ray_ten[j] = r.t0;
            w.ray_tex[j] = r.t1;
            LiveBuf b = w.buf[0];
            b.id[j] = (int32_t)j;
            b.cur[j] = p.adv.adaptive ? __double_as_longlong(r.t0) : 0ll;
            b.col[3 * j] = 0.0;
            b.col[3 * j + 1] = 0.0;
            b.col[3 * j + 2] = 0.0;
            b.tr[j] = 1.0;
        }
        if (tile == ntiles - 1 && threadIdx.x == kTile - 1) {
            w.live[0] = (int32_t)total;
        }
    }
}

// One wavefront iteration.  Input: live buffer k&1 (entries [0, live[k])).
// Output: sampling rays compacted in order into buffer (k+1)&1 at their rank.
__global__ void __launch_bounds__(kTile) k_march_iter(VcbFrameParams p, FrameWs w, int k,
                                                      unsigned long long* host_live) {
    __shared__ ScanSmem sm;
    __shared__ unsigned long long cnt[4];
    const int64_t n = __ldcg(&w.live[k]);
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && host_live)
            host_live[k + 1] = (unsigned long long)p.epoch << 32;
        return;
    }
    const LiveBuf in = w.buf[k & 1];
    const LiveBuf out = w.buf[(k + 1) & 1];
    const int64_t ntiles = (n + kTile - 1) / kTile;
    if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
    const double ox = p.cam.origin[0], oy = p.cam.origin[1], oz = p.cam.origin[2];
    for (;;) {
        if (threadIdx.x == 0) sm.tile = atomicAdd(&w.ticket[k], 1);
        __syncthreads();
        const int64_t tile = sm.tile;
        __syncthreads();
        if (tile >= ntiles) break;
        const int64_t i = tile * kTile + threadIdx.x;
        int flag = 0;
        int32_t id = -1;
        double cf = 0.0, cr = 0.0, cg = 0.0, cb = 0.0, tr = 1.0;
        i64 ck = 0;
        AdvanceOut a;
        if (i < n) {
            id = in.id[i];
            if (id >= 0) {
                long long cur = in.cur[i];
                cf = __longlong_as_double(cur);
                ck = cur;
                cr = in.col[3 * i];
                cg = in.col[3 * i + 1];
                cb = in.col[3 * i + 2];
                tr = in.tr[i];
                flag = advance_one(ox, oy, oz, w.ray_dir[3 * id], w.ray_dir[3 * id + 1], w.ray_dir[3 * id + 2],
                                   w.ray_ten[id], w.ray_tex[id], cf, ck, p.adv, p.mu, a);
                if (!flag) retire(p, w.ray_pix[id], cr, cg, cb, tr);
            }
        }
        long long j;
        uint32_t total = ordered_scan(flag, tile, w.status, p.epoch * 16384u + (uint32_t)k, sm, j);
        if (tile == ntiles - 1 && threadIdx.x == kTile - 1) {
            w.live[k + 1] = (int32_t)total;
            if (host_live) host_live[k + 1] = ((unsigned long long)p.epoch << 32) | total;
        }
        if (flag) {
            int dead = 0, queued = 0;
            if (!p.cached) {
                queued = 1;
            } else {
                double u = 0.0;
                if (p.probe.mode != 2) {
                    uint32_t s = (k == 0) ? lane_seed(p.rng_base, (u64)j) : w.rng[j];
                    s = xorshift32(s);
                    w.rng[j] = s;
                    u = DMUL((double)s, 2.3283064365386963e-10);  // / 2^32, exact
                }
                double dist = a.tmid;
                if (p.paged_dist) {
                    double ex = DSUB(a.px, ox), ey = DSUB(a.py, oy), ez = DSUB(a.pz, oz);
                    dist = __dsqrt_rn(DADD(DADD(DMUL(ex, ex), DMUL(ey, ey)), DMUL(ez, ez)));
                }
                float v;
                int rq, slot;
                int sv = probe_one(a.px, a.py, a.pz, dist, u, p.probe, p.table, p.pool, (long long*)p.last_used,
                                   p.cache_frame, v, rq, slot);
                if (sv != rq) {
                    // mrpd.py:215-225 miss filing at the requested LoD; native clipped
                    // to [0, V-1] (sampler.py:271-275), owner floor((p+1)/span)
                    const i64 span = p.probe.b << rq;
                    double nx = clampd(DSUB(DMUL(a.px, p.probe.vx), 0.5), 0.0, DSUB(p.probe.vx, 1.0));
                    double ny = clampd(DSUB(DMUL(a.py, p.probe.vy), 0.5), 0.0, DSUB(p.probe.vy, 1.0));
                    double nz = clampd(DSUB(DMUL(a.pz, p.probe.vz), 0.5), 0.0, DSUB(p.probe.vz, 1.0));
                    i64 bx = clampi((i64)floor(cell_div(DADD(nx, 1.0), (double)span)), 0, p.probe.grid[rq][0] - 1);
                    i64 by = clampi((i64)floor(cell_div(DADD(ny, 1.0), (double)span)), 0, p.probe.grid[rq][1] - 1);
                    i64 bz = clampi((i64)floor(cell_div(DADD(nz, 1.0), (double)span)), 0, p.probe.grid[rq][2] - 1);
                    i64 key = p.probe.offset[rq] + bx + p.probe.grid[rq][0] * (by + p.probe.grid[rq][1] * bz);
                    warp_aggregated_add(p.miss_count, key);
                }
                if (sv < 0) {
                    queued = 1;
                    atomicAdd(&cnt[3], 1ull);
                } else {
                    atomicAdd(&cnt[sv == rq ? 1 : 2], 1ull);
                    dead = shade_one(v, a.dt, p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg, cb,
                                     tr);
                    if (dead) retire(p, w.ray_pix[id], cr, cg, cb, tr);
                }
            }
            if (queued) {
                int q = atomicAdd(&w.nmiss[k], 1);
                w.mq_slot[q] = (int32_t)j;
                w.mq_pos[3 * q] = a.px;
                w.mq_pos[3 * q + 1] = a.py;
                w.mq_pos[3 * q + 2] = a.pz;
                w.mq_dt[q] = a.dt;
            }
            out.id[j] = dead ? -1 : id;
            out.cur[j] = p.adv.adaptive ? __double_as_longlong(cf) : ck;
            out.col[3 * j] = cr;
            out.col[3 * j + 1] = cg;
            out.col[3 * j + 2] = cb;
            out.tr[j] = tr;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (cnt[1]) atomicAdd((unsigned long long*)&p.stats->exact, cnt[1]);
        if (cnt[2]) atomicAdd((unsigned long long*)&p.stats->fallback, cnt[2]);
        if (cnt[3]) atomicAdd((unsigned long long*)&p.stats->miss, cnt[3]);
    }
}

void launch_rays(const VcbFrameParams& p, const FrameWs& w, cudaStream_t st) {
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    k_raygen_frame<<<grid_for(npix, 256), 256, 0, st>>>(p, w);
    k_compact_rays<<<device_sms() * 4, kTile, 0, st>>>(p, w);
}

// True misses of iteration k: infer through the field (sampler.py:145-154 with
// clamp_normalized, 119-120), then shade the ray sitting at output slot j.
template <int kInr>
__global__ void k_miss_shade(VcbFrameParams p, FrameWs w, int k) {
    extern __shared__ __align__(16) float smem[];
    const int nm = __ldcg(&w.nmiss[k]);
    if (nm == 0) return;
    MlpSmem m;
    if (p.field.kind == 0) {
        stage_mlp(p.field, smem, m);
        __syncthreads();
    }
    const LiveBuf out = w.buf[(k + 1) & 1];
    const double hi = 0.99999999999999989;  // np.nextafter(1.0, 0.0)
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nm; q += gridDim.x * blockDim.x) {
        double x = clampd(w.mq_pos[3 * q], 0.0, hi);
        double y = clampd(w.mq_pos[3 * q + 1], 0.0, hi);
        double z = clampd(w.mq_pos[3 * q + 2], 0.0, hi);
        float v = field_eval<kInr>(p.field, x, y, z, m, &w.ctr->nonfinite);
        const int j = w.mq_slot[q];
        const int32_t id = out.id[j];
        double cr = out.col[3 * j], cg = out.col[3 * j + 1], cb = out.col[3 * j + 2], tr = out.tr[j];
        bool dead = shade_one(v, w.mq_dt[q], p.lut, p.lut_size, p.adv.adaptive, p.adv.dt_base, p.term, cr, cg, cb,
                              tr);
        out.col[3 * j] = cr;
        out.col[3 * j + 1] = cg;
        out.col[3 * j + 2] = cb;
        out.tr[j] = tr;
        if (dead) {
            retire(p, w.ray_pix[id], cr, cg, cb, tr);
            out.id[j] = -1;
        }
    }
}

// Rays still alive after max_iterations are flushed as they stand (raymarch.py:117).
__global__ void k_flush(VcbFrameParams p, FrameWs w, int k) {
    const int64_t n = __ldcg(&w.live[k]);
    const LiveBuf in = w.buf[k & 1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t id = in.id[i];
        if (id < 0) continue;
        retire(p, w.ray_pix[id], in.col[3 * i], in.col[3 * i + 1], in.col[3 * i + 2], in.tr[i]);
    }
}

__global__ void k_frame_stats(VcbFrameParams p, FrameWs w, int kmax) {
    // requests = sum of sampling counts over iterations; iterations run
    long long req = 0;
    int it = 0;
    for (int k = 1; k <= kmax; k++) {
        int v = w.live[k];
        req += v;
        if (v > 0) it = k;
    }
    p.stats->requests += req;
    p.stats->iterations = it;
    p.stats->rays = w.live[0];
    long long mres = 0;
    for (int k = 0; k < kmax; k++) mres += w.nmiss[k];
    p.stats->misses_resolved = mres;
    if (!p.cached) p.stats->miss += req;
    p.stats->nonfinite = w.ctr->nonfinite;
}

}  // namespace cinr

using namespace cinr;

namespace cinr {
int launch_wave3_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used,
                       int nt, int mu_mode);
int64_t wave3_ws_bytes(int64_t npix, int max_it);
int launch_ray_frame(const VcbFrameParams& p, cudaStream_t st, long long* launches, cudaEvent_t* ev, int* ev_used,
                     int nt, int max_skip);
int64_t rays_ws_bytes(int64_t npix, int max_it);
int wave3_trace(const void* workspace, int64_t npix, int max_it, int n, unsigned int* out, int* live);
int wave3_counters(const void* workspace, int64_t npix, int max_it, long long* out);
}  // namespace cinr

extern "C" int64_t vcb_frame_workspace_bytes(int64_t max_rays, int32_t max_iterations) {
    // the parity schedule's layout (includes frame_ws_layout; the throughput
    // schedule uses only its counters)
    const int64_t a = wave3_ws_bytes(max_rays, max_iterations), b = rays_ws_bytes(max_rays, max_iterations);
    return a > b ? a : b;
}

extern "C" int32_t vcb_raygen_pass(int64_t n, const double* base, const double* rot, const double* origin,
                                   double tan_h, double tan_v, double* dirs, double* t0, double* t1, uint8_t* keep,
                                   void* stream) {
    if (n <= 0) return 0;
    k_raygen_pass<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, base, rot, origin, tan_h, tan_v, dirs, t0,
                                                                       t1, keep);
    return check_launch("raygen_pass");
}

extern "C" int32_t vcb_debug_pow(int64_t n, const double* x, const double* y, double* out, void* stream) {
    if (n <= 0) return 0;
    k_pow_dd<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x, y, out, 0);
    return check_launch("debug_pow");
}

extern "C" int32_t vcb_debug_pow_accurate(int64_t n, const double* x, const double* y, double* out, void* stream) {
    if (n <= 0) return 0;
    k_pow_dd<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x, y, out, 1);
    return check_launch("debug_pow_accurate");
}

extern "C" int32_t vcb_advance_pass(int64_t n, const double* o, const double* d, const double* t_en,
                                    const double* t_ex, double* cursor_f, int64_t* cursor_k, const uint8_t* active,
                                    const VcbMarchStatic* s, const float* mu, double* out_pos, double* out_dt,
                                    double* out_tmid, uint8_t* sample_mask, uint8_t* done_mask, void* stream) {
    if (n <= 0) return 0;
    k_advance_pass<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, o, d, t_en, t_ex, cursor_f, cursor_k,
                                                                        active, *s, mu, out_pos, out_dt, out_tmid,
                                                                        sample_mask, done_mask);
    return check_launch("advance_pass");
}

extern "C" int32_t vcb_probe_pass(int64_t n, const double* pos, const double* dist, const double* u,
                                  const VcbProbeStatic* p, const int32_t* table, const float* pool,
                                  int64_t* last_used, int64_t frame, float* values, int8_t* served, int8_t* req,
                                  int64_t* counts, void* stream) {
    if (n <= 0) return 0;
    k_probe_pass<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        n, pos, dist, u, *p, table, pool, last_used, frame, values, served, req, (unsigned long long*)counts);
    return check_launch("probe_pass");
}

extern "C" int32_t vcb_shade_pass(int64_t n, const int64_t* rows, const float* values, const double* dt,
                                  const float* lut, int64_t lut_size, int32_t adaptive, double dt_base, double term,
                                  double* color, double* trans, uint8_t* dead, void* stream) {
    if (n <= 0) return 0;
    k_shade_pass<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, rows, values, dt, lut, (int)lut_size,
                                                                      adaptive, dt_base, term, color, trans, dead);
    return check_launch("shade_pass");
}

namespace cinr {
thread_local long long g_launches = 0;
static thread_local std::vector<cudaEvent_t> g_ev;
static thread_local int g_ev_used = 0;
}  // namespace cinr

static unsigned long long* mapped_live(int n, unsigned long long** dev) {
    // pinned + mapped host array the iteration kernels write live counts into,
    // so the host loop can stop issuing iterations without a stream sync
    static thread_local unsigned long long* host = nullptr;
    static thread_local unsigned long long* devp = nullptr;
    static thread_local int cap = 0;
    if (cap < n) {
        if (host) cudaFreeHost(host);
        if (cudaHostAlloc((void**)&host, (size_t)n * 8, cudaHostAllocMapped) != cudaSuccess) {
            host = nullptr;
            cap = 0;
            *dev = nullptr;
            return nullptr;
        }
        cudaHostGetDevicePointer((void**)&devp, host, 0);
        cap = n;
    }
    *dev = devp;
    return host;
}

extern "C" int32_t vcb_march_frame(const VcbFrameParams* pp, void* stream_) {
    const VcbFrameParams& p = *pp;
    cudaStream_t st = (cudaStream_t)stream_;
    // this frame's counters (the ray path's setup kernel clears them itself)
    const bool ray_path = p.impl >= 10 && p.impl <= 14 && (int64_t)p.cam.width * p.cam.rows > 0;
    if (!ray_path) cudaMemsetAsync(p.stats, 0, sizeof(VcbFrameStats), st);
    if (p.impl != 1) {
        if ((int64_t)p.cam.width * p.cam.rows == 0) return 0;
        g_ev_used = 0;
        if (p.timing) {
            while (g_ev.size() < 2) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                g_ev.push_back(e);
            }
        }
        cudaEvent_t* ev = p.timing ? g_ev.data() : nullptr;
        if (p.impl == 9) return launch_wave3_frame(p, st, &g_launches, ev, &g_ev_used, 512, 0);
        if (p.impl == 10) return launch_ray_frame(p, st, &g_launches, ev, &g_ev_used, 512, 2);
        if (p.impl == 11) return launch_ray_frame(p, st, &g_launches, ev, &g_ev_used, 512, 1);
        if (p.impl == 12) return launch_ray_frame(p, st, &g_launches, ev, &g_ev_used, 640, 1);
        if (p.impl == 13) return launch_ray_frame(p, st, &g_launches, ev, &g_ev_used, 512, 0);
        if (p.impl == 14) return launch_ray_frame(p, st, &g_launches, ev, &g_ev_used, 640, 2);
        return launch_wave3_frame(p, st, &g_launches, ev, &g_ev_used, 384, 0);
    }
    const int64_t npix = (int64_t)p.cam.width * p.cam.rows;
    const int max_it = p.max_iterations < kMaxIterCap ? p.max_iterations : kMaxIterCap;
    FrameWs w;
    int64_t need = frame_ws_layout(npix, max_it, p.workspace, &w);
    if (need > p.workspace_bytes)
        return set_error("march_frame: workspace too small (%lld < %lld)", (long long)p.workspace_bytes,
                         (long long)need);
    if (npix == 0) return 0;
    unsigned long long* dlive = nullptr;
    volatile unsigned long long* hlive = mapped_live(max_it + 2, &dlive);
    cudaMemsetAsync(w.ctr, 0, sizeof(FrameCounters), st);
    cudaMemsetAsync(w.ctr_iter, 0, w.ctr_iter_bytes, st);
    const int sms = device_sms();
    k_raygen_frame<<<grid_for(npix, 256), 256, 0, st>>>(p, w);
    k_compact_rays<<<sms * 4, kTile, 0, st>>>(p, w);
    const int iter_grid = sms * kItersPerSm;
    int smem_mlp = 0;
    if (p.field.kind == 0) {
        int nw = 0, nb = 0;
        for (int L = 0; L < p.field.n_layers; L++) {
            nw += p.field.widths[L] * p.field.widths[L + 1];
            nb += p.field.widths[L + 1];
        }
        smem_mlp = (nw + nb) * (int)sizeof(float);

    }
    // Chunks of iterations are queued back to back; before queueing chunk c+1 the
    // host waits for chunk c-1 and stops once its last live count (tagged with this
    // frame's epoch) is zero.  Iterations past the end exit on live[k] == 0.
    const int chunk = 16;
    g_launches = 2;
    if (p.timing) {
        while ((int)g_ev.size() < 2 * max_it) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            g_ev.push_back(e);
        }
    }
    g_ev_used = 0;
    cudaEvent_t ev[2];
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    int chunk_end[2] = {-1, -1};
    int k = 0, ci = 0;
    bool stop = false;
    while (k < max_it && !stop) {
        const int kend = k + chunk < max_it ? k + chunk : max_it;
        for (; k < kend; k++) {
            if (p.timing) cudaEventRecord(g_ev[2 * k], st);
            k_march_iter<<<iter_grid, kTile, 0, st>>>(p, w, k, dlive);
            if (p.timing) cudaEventRecord(g_ev[2 * k + 1], st);
            CINR_DISPATCH_INR(p.field, k_miss_shade, sms * 4, 256, smem_mlp, st, p, w, k);
            g_launches += 2;
        }
        if (p.timing) g_ev_used = k;
        cudaEventRecord(ev[ci & 1], st);
        chunk_end[ci & 1] = kend;
        ci++;
        const int older = ci & 1;
        if (hlive && chunk_end[older] >= 0) {
            cudaEventSynchronize(ev[older]);
            const unsigned long long v = hlive[chunk_end[older]];
            if ((uint32_t)(v >> 32) == p.epoch && (uint32_t)v == 0u) stop = true;
        }
    }
    k_flush<<<grid_for(npix, 256), 256, 0, st>>>(p, w, k);
    k_frame_stats<<<1, 1, 0, st>>>(p, w, k);
    g_launches += 2;
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    return check_launch("march_frame");
}

extern "C" int32_t vcb_march_timing(int32_t n_iters, double* ms_total, int64_t* launches) {
    double tot = 0.0;
    int n = n_iters < g_ev_used ? n_iters : g_ev_used;
    for (int k = 0; k < n; k++) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, g_ev[2 * k], g_ev[2 * k + 1]) != cudaSuccess)
            return set_error("march_timing: %s", cudaGetErrorString(cudaGetLastError()));
        tot += ms;
    }
    *ms_total = tot;
    *launches = n;
    return 0;
}

extern "C" int64_t vcb_last_launch_count(void) { return g_launches; }

// Diagnostics of the last timing=1 frame of the default schedule.
extern "C" int32_t vcb_frame_trace(const void* workspace, int64_t max_rays, int32_t max_iterations, int32_t n,
                                   uint32_t* stamps, int32_t* live) {
    return wave3_trace(workspace, max_rays, max_iterations, n, stamps, live);
}

// Diagnostics: the 23 u64 counters a CINR_STATS build of the default schedule keeps.
extern "C" int32_t vcb_frame_counters(const void* workspace, int64_t max_rays, int32_t max_iterations,
                                      int64_t* out23) {
    return wave3_counters(workspace, max_rays, max_iterations, (long long*)out23);
}
