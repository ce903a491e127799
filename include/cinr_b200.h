/*
 * cinr_b200.h — C ABI of the B200-native cached-INR ray-march path.
 *
 * Plain C structs + device pointers + sizes; no torch types.  Every entry
 * point returns 0 on success or a negative status, with the message available
 * from vcb_last_error() (thread-local).  Streams are passed as `void*`
 * (a cudaStream_t; NULL = legacy default stream).  Callers own all memory.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/voxcache/):
 *
 *   Operator ABI (Stage A drop-in: one export per numba pass; the reference
 *   resolves these module attributes at call time, so a plugin swaps them):
 *     vcb_raygen_pass   <- render/kernels.py:426 raygen_pass   (_raygen_one 376-411)
 *     vcb_advance_pass  <- render/kernels.py:160 advance_pass  (_advance_one 35-137)
 *     vcb_probe_pass    <- render/kernels.py:316 probe_pass    (_probe_one 166-273)
 *     vcb_shade_pass    <- render/kernels.py:370 shade_pass    (_shade_one 322-355)
 *   Field / decoder ABI (the Field.sample_batch duck type, fields.py:89-97):
 *     vcb_field_points  <- InrField/RawLatticeField/ProceduralField.sample_batch
 *                          (inr/model.py:65-89, encoding.py:119-134, mlp.py:39-53,
 *                          fields.py:165-221, fields.py:131-158)
 *     vcb_field_bricks  <- scheduler.py:127-134 fulfill (+ brickmath.py:125-139
 *                          sample_positions), written straight into a pool/staging slab
 *     vcb_macro_minmax  <- macrocell.py:49-74 build (lattice decode + dilated min/max)
 *   Session ABI (Stage B drop-in: the GPU-resident RenderSession):
 *     vcb_march_frame   <- render/raymarch.py:25-120 raymarch_frame with the
 *                          VolumeSampler probe/miss path (sampler.py:196-280)
 *     vcb_pathtrace_frame <- render/pathtrace.py:112-146 pathtrace_frame (trace_free_flight
 *                          28-98, _light_visibility 101-109) on the same sampler
 *     vcb_maintenance   <- session.py:132-142 _maintenance: Mrpd.drain_miss_reports
 *                          (mrpd.py:263), RequestTable.report_many/select_batch
 *                          (scheduler.py:60-101), InlineLoader collect/dispatch
 *                          (scheduler.py:137-172), Mrpd.insert + BrickPool.acquire_slot
 *                          (mrpd.py:229-256, pool.py:55-68)
 */
#ifndef CINR_B200_H
#define CINR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VCB_MAX_LOD 32
#define VCB_MAX_LEVELS 16
#define VCB_MAX_LAYERS 8

/* camera.py:129-138: origin, rot = [right, up, fwd] as columns (row-major 3x3),
 * tan_h = tan(fov/2)*aspect, tan_v = tan(fov/2).  A session may render a
 * subset of the film rows (sort-first multi-GPU): local row j is film row
 * row0 + j*row_step, `rows` rows in total (row0=0, row_step=1, rows=height
 * for the whole frame). */
typedef struct {
    double origin[3];
    double rot[9];
    double tan_h, tan_v;
    int32_t width, height;
    int32_t row0, row_step, rows, pad_;
} VcbCamera;

/* advance_pass scalars (kernels.py:35-39). gx/gy/gz macro grid, cw* cell widths. */
typedef struct {
    int32_t adaptive, skip_empty;
    double dt_base, mu_floor;
    int64_t gx, gy, gz;
    double cwx, cwy, cwz;
} VcbMarchStatic;

/* probe_pass scalars (kernels.py:166-170) + packed table geometry (mrpd.py:91-114). */
typedef struct {
    double vx, vy, vz, lod_scale;
    int32_t mode;    /* 0 corrected, 1 as_printed, 2 off (sampler.py:233) */
    int32_t max_lod;
    int64_t b;       /* brick size */
    int32_t b_pow2;  /* 1 if every span B<<L is a power of two */
    int32_t pad_;
    int64_t grid[VCB_MAX_LOD][3];
    int64_t offset[VCB_MAX_LOD];
} VcbProbeStatic;

/* Field descriptor: kind 0 = hash-grid INR, 1 = lattice, 2 = procedural. */
typedef struct {
    int32_t kind;
    /* INR (HashGridConfig / MLPConfig, encoding.py:30-64, mlp.py:13-25) */
    int32_t levels, feats, out_sigmoid, n_layers;
    int64_t table_size;
    int32_t res[VCB_MAX_LEVELS];
    int32_t dense[VCB_MAX_LEVELS];
    int64_t tab_off[VCB_MAX_LEVELS];       /* row offset of each level */
    int32_t widths[VCB_MAX_LAYERS + 1];    /* input, hidden..., 1 */
    int64_t w_off[VCB_MAX_LAYERS], b_off[VCB_MAX_LAYERS];
    const float *tables;                   /* [rows][feats] */
    const float *weights;                  /* packed (out,in) row-major per layer */
    const float *biases;
    /* lattice (z,y,x) f32 */
    const float *lattice;
    int64_t lx, ly, lz;
    /* procedural: 0 sphere, 1 shells, 2 marschner_lobb_like (fields.py:131-148) */
    int32_t proc;
    int32_t clip01;                        /* InrField clip (model.py:88-89) */
} VcbField;

/* Brick geometry for decode (brickmath.py:87-139). */
typedef struct {
    int64_t dims[3];
    int64_t b;
    int32_t n_lod, pad_;
    int64_t grid[VCB_MAX_LOD][3];
    int64_t offset[VCB_MAX_LOD];
} VcbBrickGeom;

/* Per-frame device counters (FrameStats, mrpd.py:33-41 + sampler counters). */
typedef struct {
    int64_t requests, exact, fallback, miss;
    int64_t iterations, rays;
    int64_t misses_resolved;
    int64_t nonfinite;      /* true-miss inference produced NaN/Inf (ModelCorruptError) */
    int64_t deferred_misses; /* true misses left undecoded by the frame's decode budget (not composited) */
    int64_t pad_[7];
} VcbFrameStats;

/* Device-resident cache bookkeeping (pool free list, loader, counters). */
typedef struct {
    int64_t next_free;      /* free slots are [next_free, S) — pool.py:46,57-58 */
    int64_t loaded_total;   /* mrpd.py:84-85 */
    int64_t n_staged;       /* bricks dispatched last maintenance (InlineLoader._staged) */
    int64_t staged_frame;
    int64_t decode_error;   /* non-finite decode -> reinsert (scheduler.py:164-168) */
    int64_t bricks_loaded;  /* this maintenance */
    int64_t deferred, inserted;
    int64_t n_inflight;
    int64_t n_reports, n_pending, n_batch;
    int64_t pad_[4];
} VcbCacheState;

typedef struct {
    VcbCamera cam;
    VcbMarchStatic adv;
    VcbProbeStatic probe;
    int32_t cached;          /* 0 = uncached baseline (session.py:63-70) */
    int32_t paged_dist;      /* 1 = |pos-cam| distances (sampler.py:135 numpy path) */
    int64_t cache_frame;     /* probe stamp clock (P11) */
    uint64_t rng_base;       /* splitmix64(seed ^ frame*GOLDEN), sampler.py:41 */
    double term;
    double bg[3];
    int32_t lut_size;
    int32_t max_iterations;
    uint32_t epoch;          /* monotonic per call; tags look-back status words */
    int32_t timing;          /* bit 0: bracket the frame kernel(s) with CUDA events; bit 1: record the
                                default schedule's per-iteration trace (vcb_frame_trace) */
    const float *mu;         /* majorants [gz][gy][gx] */
    const float *lut;        /* [lut_size][4] */
    const int32_t *table;    /* dense logical MRPD, all LoDs */
    const float *pool;       /* [S][B][B][B] */
    int64_t *last_used;      /* [S] */
    int32_t *miss_count;     /* per brick, all LoDs */
    VcbField field;          /* true-miss inference */
    float *image;            /* [H][W][4] */
    VcbFrameStats *stats;    /* device */
    void *workspace;
    int64_t workspace_bytes;
    int32_t impl;            /* march schedule.  Parity (the reference's RNG lanes = sample rank per
                                wavefront iteration, sampler.py:206-213): 0 = one-barrier persistent
                                wavefront, 384 threads/CTA (default), 9 = the same at 512 threads,
                                1 = one launch per iteration (cross-check).  Throughput (RNG lane = film
                                pixel, no grid barrier, one persistent ray per lane): 10 = 512 threads/CTA,
                                skip budget 2 (default); 11 = 512, 1; 12 = 640, 1; 13 = 512, unbounded;
                                14 = 640, 2.  Path tracing: 1 = four-barrier walk, otherwise the default
                                walk */
    int32_t image_global;    /* 0: image is this session's band [rows][W][4]; 1: image is the whole
                                frame [height][W][4] (possibly a peer GPU's buffer mapped over NVLink)
                                and local row j lands on film row row0 + j*row_step */
    int64_t miss_budget;     /* frame scheduler: true misses the frame may decode (sampler.py:276-279 is
                                unbounded: -1); past it a true miss is filed but not composited */
} VcbFrameParams;

typedef struct {
    VcbBrickGeom geom;
    int64_t total;           /* bricks over all LoDs */
    int64_t slots;
    int64_t session_frame;
    int32_t max_requests, ranking;
    int64_t rank_clamp;
    int32_t lin_bits, lod_bits;
    int32_t *table;
    float *pool;
    int64_t *owner;          /* [S] flat brick id or -1 */
    int64_t *last_used;
    int32_t *miss_count;
    int64_t *req_base;       /* -1 absent */
    int64_t *req_hits;
    VcbCacheState *state;
    float *staging;          /* [max_requests][B^3] */
    int64_t *staged_keys;    /* [max_requests] flat brick ids in batch order */
    void *workspace;
    int64_t workspace_bytes;
    int64_t *dbg_reports;    /* optional [total][2] (flat id, count), NULL to skip */
    VcbField field;
    const VcbFrameStats *frame_stats; /* optional: the frame just rendered (device).  nonfinite set: the
                                        whole maintenance is skipped on the device, as the reference raises
                                        RenderError before _maintenance runs (sampler.py:149-152,
                                        session.py:107-112).  misses_resolved: the decode budget's share
                                        the frame already used */
    int64_t decode_budget;   /* frame scheduler: samples decoded per frame (true misses + brick batch);
                                -1 = unbounded (the reference: max_requests bricks, all misses).  The batch
                                is min(max_requests, max(1, (budget - misses_resolved) / B^3)) bricks */
    int32_t defer_decode;    /* 1: the batch is decoded by vcb_maint_decode (on another stream, overlapping
                                the next frame; inserted at the next maintenance as InlineLoader /
                                ThreadLoader collect() would); 0: decoded inside this call */
    int32_t pad2_;
    int32_t *pending_list;   /* [total] bricks with a request-table entry (req_base >= 0), any order;
                                kept by the maintenance (new keys appended, popped keys compacted out) */
    int32_t *list_counts;    /* [1] pending_list entries; both null = k_pending scans every brick */
} VcbMaintParams;

/* Path tracing (render/pathtrace.py:112-146, session.py:108-109): samples_per_pixel
 * delta-tracked paths per pixel with one shadow ray each, on the VolumeSampler of the
 * frame params (cache probe, miss filing, true-miss inference).  The PCG64 stream is
 * numpy's default_rng(splitmix64((seed & 0xFFFFFFFF) ^ frame)) seeded on the host. */
typedef struct {
    int32_t spp;             /* SessionConfig.samples_per_pixel */
    int32_t max_walk;        /* _MAX_WALK (pathtrace.py:18) */
    double density;          /* RenderSettings.pt_density */
    double ambient;          /* RenderSettings.pt_ambient */
    double light[3];         /* -light_dir / |light_dir| (pathtrace.py:103-104) */
    int32_t n_tf, pad_;
    const double *tf;        /* [n_tf][5] TransferFunction.points (x, r, g, b, a), device */
    uint64_t pcg_state[2];   /* PCG64 state (lo, hi) after seeding */
    uint64_t pcg_inc[2];     /* PCG64 increment (lo, hi) */
    uint64_t lane_seed;      /* VolumeSampler.seed (lane reseeding, sampler.py:206-213) */
    int64_t lane_frame;      /* VolumeSampler.frame */
    void *workspace;         /* vcb_pt_workspace_bytes(width*rows) bytes */
    int64_t workspace_bytes;
} VcbPtParams;

/* INR training (inr/train.py:16-132): `steps` optimizer steps of MSE on batches of
 * rng.random((batch, 3)) positions of numpy's PCG64 stream (default_rng(seed) state,
 * draw0 draws already consumed), targets from the target field's decoder. */
typedef struct {
    VcbField model;          /* default 8x2 hash grid + 16-32-32-1 MLP; its device tables/weights/biases
                                are updated in place */
    VcbField target;         /* the field fitted (lattice / procedural / INR) */
    int64_t batch, steps, step0;   /* step0 = optimizer steps already taken (Adam t) */
    int32_t optimizer;             /* 0 = Adam (train.py:51-75), 1 = SGD (40-48), 2 = none (lr 0) */
    int32_t flags;                 /* bit 0: pos/targets given by the caller (no PCG batch, no decode);
                                      bit 1: keep the gradients (loss_and_grads, train.py:16-37: no update);
                                      bit 2: clip by the global norm clip_norm (train.py:78-85; unset = None) */
    double lr, beta1, beta2, eps, clip_norm;
    uint64_t pcg_state[2], pcg_inc[2];
    uint64_t draw0;
    int64_t n_table_params, n_weights, n_params;  /* flat parameter order: tables, weights, biases */
    double *grads, *m, *v;   /* [n_params] f64; grads zero on entry and left zero */
    double *pos;             /* [batch][3] */
    float *targets;          /* [batch] */
    double *loss;            /* [steps] per-step sum of squared errors (zeroed by the caller) */
    double *scratch;         /* [8] */
    int32_t *nonfinite;      /* target-decode flag */
    void *jump;              /* vcb_train_workspace_bytes(batch) bytes */
} VcbTrainParams;

const char *vcb_last_error(void);
int32_t vcb_abi_version(void);
int32_t vcb_device_sm_count(void);
/* host-only: sizeof of VcbCamera, VcbMarchStatic, VcbProbeStatic, VcbField, VcbBrickGeom,
 * VcbFrameStats, VcbCacheState, VcbFrameParams, VcbMaintParams (ABI self-check) */
int32_t vcb_struct_sizes(int64_t *out, int32_t n);

/* ---- operator ABI (device pointers, row-major arrays as in kernels.py) */
int32_t vcb_raygen_pass(int64_t n, const double *base_dirs, const double *rot, const double *origin, double tan_h,
                        double tan_v, double *dirs, double *t0, double *t1, uint8_t *keep, void *stream);
int32_t vcb_advance_pass(int64_t n, const double *o, const double *d, const double *t_en, const double *t_ex,
                         double *cursor_f, int64_t *cursor_k, const uint8_t *active, const VcbMarchStatic *s,
                         const float *mu, double *out_pos, double *out_dt, double *out_tmid, uint8_t *sample_mask,
                         uint8_t *done_mask, void *stream);
int32_t vcb_probe_pass(int64_t n, const double *pos, const double *dist, const double *u, const VcbProbeStatic *p,
                       const int32_t *table, const float *pool, int64_t *last_used, int64_t frame, float *values,
                       int8_t *served, int8_t *req, int64_t *counts /* device [3] */, void *stream);
int32_t vcb_shade_pass(int64_t n, const int64_t *rows, const float *values, const double *dt, const float *lut,
                       int64_t lut_size, int32_t adaptive, double dt_base, double term, double *color, double *trans,
                       uint8_t *dead, void *stream);

/* diagnostics: the shade's accurate pow, out[i] = x[i]**y[i] (x in (0,1], y > 0) */
int32_t vcb_debug_pow(int64_t n, const double *x, const double *y, double *out, void *stream);
/* The same pow through its double-double phase only (the fast phase's cross-check). */
int32_t vcb_debug_pow_accurate(int64_t n, const double *x, const double *y, double *out, void *stream);

/* ---- field / decoder ABI */
int32_t vcb_field_points(const VcbField *f, int64_t n, const double *pos, float *out, int32_t *nonfinite,
                         void *stream);
int32_t vcb_field_bricks(const VcbField *f, const VcbBrickGeom *g, int64_t n_keys, const int64_t *keys,
                         float *out, int32_t *nonfinite, void *stream);
/* Tensor-core (tcgen05) decoder for the default INR shape (8x2 hash grid,
 * 16->32->32->1): the same contract as vcb_field_points / vcb_field_bricks. */
int32_t vcb_inr_points_tc(const VcbField *f, int64_t n, const double *pos, float *out, int32_t *nonfinite,
                          void *stream);
int32_t vcb_inr_bricks_tc(const VcbField *f, const VcbBrickGeom *g, int64_t n_keys, const int64_t *keys,
                          float *out, int32_t *nonfinite, void *stream);
int32_t vcb_macro_minmax(const VcbField *f, const int64_t *dims, int64_t cell, float *vmin, float *vmax,
                         void *stream);

/* macrocell.py:120-128 update_majorants on the device: mu[c] = f32(max of bin_max over
 * bins [int(vmin[c]*bins), int(vmax[c]*bins)]), bin_max = opacity_bin_maxima (host, f64). */
int32_t vcb_update_majorants(const float *vmin, const float *vmax, int64_t n, const double *bin_max, int32_t bins,
                             float *mu, void *stream);

/* image_io.py:14-21 to_rgba8 on the device: out[i] = uint8(clip(f64(image[i]), 0, 1) * 255 + 0.5)
 * for the n_pixels RGBA f32 pixels of image (frame streaming, protocol.py:59-61). */
int32_t vcb_frame_rgba8(const float *image, int64_t n_pixels, uint8_t *out, void *stream);

/* ---- training ABI */
int64_t vcb_train_workspace_bytes(int64_t batch);
int32_t vcb_train_steps(const VcbTrainParams *p, void *stream);

/* ---- session ABI */
int64_t vcb_frame_workspace_bytes(int64_t max_rays, int32_t max_iterations);
int32_t vcb_march_frame(const VcbFrameParams *p, void *stream);
/* render/pathtrace.py:112-146 pathtrace_frame with the VolumeSampler probe/miss path;
 * the maintenance that follows is vcb_maintenance as for the ray march. */
int64_t vcb_pt_workspace_bytes(int64_t max_rays);
int32_t vcb_pathtrace_frame(const VcbFrameParams *p, const VcbPtParams *q, void *stream);
/* render/pathtrace.py:28-98 trace_free_flight(scene, origins, directions, t_start, t_end, rng)
 * on n caller rays (device arrays; o/d [n][3]) with the sampler, macro grid and field of p and
 * the density / TF / PCG stream of q (q.spp unused); q.workspace holds vcb_pt_workspace_bytes(n).
 * Synchronous: on return t_hit (+inf = escaped), v_hit are written and *draws (host) is the
 * number of PCG64 draws consumed (the caller advances its generator by it). */
int32_t vcb_trace_free_flight(const VcbFrameParams *p, const VcbPtParams *q, int64_t n, const double *o,
                              const double *d, const double *t0, const double *t1, double *t_hit, float *v_hit,
                              uint64_t *draws, void *stream);
/* diagnostics: log1p_out[i] = glibc log1p(x[i]); uniform_out[i] = numpy PCG64 random() of
 * draw draw_idx[i] (0-based) of the stream at pcg = {state lo, state hi, inc lo, inc hi};
 * pcg is a HOST pointer, the rest device pointers */
int32_t vcb_debug_pt_math(int64_t n, const double *x, double *log1p_out, const uint64_t *pcg,
                          const uint64_t *draw_idx, double *uniform_out, void *stream);
/* After the stream of a timing=1 frame has completed: summed device time (ms) and
 * count of the first `n_iters` iteration-kernel launches (the ray-march kernel). */
int32_t vcb_march_timing(int32_t n_iters, double *ms_total, int64_t *launches);
/* Diagnostics after a timing=1 frame of the default schedule (synchronous): for
 * iteration k < n (n <= 512) and CTA c < 1024, stamps[(k*1024 + c)*3 + {0,1,2}] =
 * low 32 bits of %globaltimer after the grid barrier, after the rank scan and when
 * the CTA finished its phase; live[k+1] = samples of iteration k (live[0] = rays).
 * Returns the number of iterations copied. */
int32_t vcb_frame_trace(const void *workspace, int64_t max_rays, int32_t max_iterations, int32_t n,
                        uint32_t *stamps, int32_t *live);
/* Diagnostics: 23 u64 counters of the last frame kept by a -DCINR_STATS build
 * ([0..2] skip-loop steps, advances, max steps of one advance; [8..14] summed
 * warp cycles per phase stage; zeros otherwise). */
int32_t vcb_frame_counters(const void *workspace, int64_t max_rays, int32_t max_iterations, int64_t *out23);
/* Kernels launched by this thread's last march_frame + maintenance calls. */
int64_t vcb_last_launch_count(void);
int64_t vcb_maint_workspace_bytes(int64_t total_bricks, int64_t slots, int32_t max_requests);
int32_t vcb_maintenance(const VcbMaintParams *p, void *stream);
/* The decode (fulfill, scheduler.py:127-134) of the batch the last vcb_maintenance with
 * defer_decode = 1 selected, on `stream`: the caller orders it after that maintenance
 * and before the next one (events), so it overlaps the next frame's march. */
int32_t vcb_maint_decode(const VcbMaintParams *p, void *stream);
/* The maintenance as one CUDA graph (north_star subsystem 4: the per-frame launch
 * sequence captured once, replayed per frame).  vcb_maint_graph_create captures
 * vcb_maintenance's launches for `p`; every field but session_frame must stay the same
 * for the graph's life (the caller keys the graph on them).  vcb_maint_graph_launch
 * sets session_frame in the captured kernels and launches the graph on `stream`: the
 * results are vcb_maintenance's. */
/* Brick-decode sharing across ranks (SURVEY §8e "optional brick sharing"; the
 * collectives are the caller's).  vcb_share_keys writes [n, staged keys...] of the last
 * maintenance (max_requests + 1 int64).  With those rows of all `world` ranks,
 * vcb_share_plan lists the distinct keys this rank owns (owner = splitmix64(key) % world;
 * up to `cap`, in key order: counts[0]), where each of its own batch keys sits in the
 * gathered slabs (src[i] = owner * cap + slot, -1 = decode locally) and the keys to
 * decode locally (ovf_keys / ovf_idx, counts[1]).  vcb_share_decode decodes a device-
 * counted key list (the owned keys, the local ones); vcb_share_scatter fills the staging
 * slab from the gathered slabs and the local bricks, merges the owners' decode-failure
 * flags and runs the failure path (scheduler.py:164-168) — the state equals the
 * unshared maintenance's. */
int32_t vcb_share_keys(const VcbMaintParams *p, int64_t *out, void *stream);
int32_t vcb_share_plan(const int64_t *all_keys, int32_t world, int32_t rank, int32_t max_requests, int32_t cap,
                       int64_t *own_keys, int64_t *counts, int32_t *src, int64_t *ovf_keys, int32_t *ovf_idx,
                       void *stream);
int32_t vcb_share_decode(const VcbMaintParams *p, const int64_t *keys, const int64_t *n_keys, int32_t max_keys,
                         float *out, int32_t *nonfinite, void *stream);
int32_t vcb_share_scatter(const VcbMaintParams *p, const float *gathered, const int32_t *flags, int32_t cap,
                          const int32_t *src, const float *ovf_out, const int32_t *ovf_idx, const int64_t *counts,
                          const int32_t *ovf_flag, void *stream);
int32_t vcb_maint_graph_create(const VcbMaintParams *p, void **graph);
int32_t vcb_maint_graph_launch(void *graph, const VcbMaintParams *p, void *stream);
void vcb_maint_graph_destroy(void *graph);

#ifdef __cplusplus
}
#endif
#endif
