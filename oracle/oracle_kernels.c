/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Plain-C restatement of the reference's
 * per-item loops (voxcache, /root/reference/pkg/src/voxcache/render/kernels.py)
 * and of the INR forward pass (inr/encoding.py, inr/mlp.py).  It is the CPU
 * checker the CUDA path is compared against, and the `cpu_baseline` /
 * `--impl reference` arm of bench.py.  Nothing in the product links this.
 *
 * Build: oracle/build_oracle.sh (gcc -O2 -ffp-contract=off -fopenmp).
 * Arithmetic is IEEE double/float without contraction so results are
 * bit-identical to the numba (LLVM, no fastmath) passes.  `pow` is glibc's,
 * the same libm numba lowers `**` to.
 *
 * Parity pinned by tests/test_oracle_golden.py against fixtures that
 * tests/golden/make_golden.py recorded from the real reference.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef int64_t i64;

/* CPython float floor division, Objects/floatobject.c float_floor_div, which
 * numba reproduces for `a // b` on floats (used at kernels.py:210-212). */
static double py_floordiv(double vx, double wx) {
    double mod = fmod(vx, wx);
    double div = (vx - mod) / wx;
    if (mod) {
        if ((wx < 0) != (mod < 0)) { mod += wx; div -= 1.0; }
    }
    double floordiv;
    if (div) {
        floordiv = floor(div);
        if (div - floordiv > 0.5) floordiv += 1.0;
    } else {
        floordiv = copysign(0.0, vx / wx);
    }
    return floordiv;
}

/* ---------------------------------------------------------------- raygen
 * kernels.py:376-411 (_raygen_one).  rot is row-major [3][3]. */
void orc_raygen(i64 n, const double *base, const double *rot, const double *origin,
                double tan_h, double tan_v, double *dirs, double *t0, double *t1, uint8_t *keep) {
#pragma omp parallel for schedule(static) if (n >= 6144)
    for (i64 i = 0; i < n; i++) {
        double bx = base[2 * i] * tan_h, by = base[2 * i + 1] * tan_v;
        double dx = rot[0] * bx + rot[1] * by + rot[2];
        double dy = rot[3] * bx + rot[4] * by + rot[5];
        double dz = rot[6] * bx + rot[7] * by + rot[8];
        double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
        dx *= inv; dy *= inv; dz *= inv;
        dirs[3 * i] = dx; dirs[3 * i + 1] = dy; dirs[3 * i + 2] = dz;
        double tn = -INFINITY, tf = INFINITY;
        int ok = 1;
        double dd[3] = {dx, dy, dz};
        for (int a = 0; a < 3; a++) {
            double oa = origin[a], da = dd[a];
            if (da != 0.0) {
                double ta = (0.0 - oa) / da, tb = (1.0 - oa) / da;
                if (ta > tb) { double t = ta; ta = tb; tb = t; }
                if (ta > tn) tn = ta;
                if (tb < tf) tf = tb;
            } else if (oa < 0.0 || oa > 1.0) {
                ok = 0;
            }
        }
        if (tn < 0.0) tn = 0.0;
        keep[i] = ok && (tf > tn);
        t0[i] = tn;
        t1[i] = tf;
    }
}

/* ---------------------------------------------------------------- advance
 * kernels.py:35-137 (_advance_one).  o,d: [n][3]. */
typedef struct {
    const double *o, *d, *t_en, *t_ex;
    double *cursor_f;
    i64 *cursor_k;
    const uint8_t *active;
    int adaptive, skip_empty;
    double dt_base, mu_floor;
    const float *mu;
    i64 gx, gy, gz;
    double cwx, cwy, cwz;
    double *out_pos, *out_dt, *out_tmid;
    uint8_t *sample_mask, *done_mask;
} orc_advance_args;

static i64 clampi(i64 v, i64 lo, i64 hi) { return v < lo ? lo : (v > hi ? hi : v); }

void orc_advance(i64 n, const orc_advance_args *A) {
#pragma omp parallel for schedule(static) if (n >= 6144)
    for (i64 i = 0; i < n; i++) {
        A->sample_mask[i] = 0;
        A->done_mask[i] = 0;
        if (!A->active[i]) continue;
        double ox = A->o[3 * i], oy = A->o[3 * i + 1], oz = A->o[3 * i + 2];
        double dx = A->d[3 * i], dy = A->d[3 * i + 1], dz = A->d[3 * i + 2];
        double end = A->t_ex[i];
        double t_c = A->adaptive ? A->cursor_f[i] : A->t_en[i] + ((double)A->cursor_k[i] + 0.5) * A->dt_base;
        for (;;) {
            if (t_c >= end) { A->done_mask[i] = 1; break; }
            double px = ox + dx * t_c, py = oy + dy * t_c, pz = oz + dz * t_c;
            i64 cx = clampi((i64)(px / A->cwx), 0, A->gx - 1);
            i64 cy = clampi((i64)(py / A->cwy), 0, A->gy - 1);
            i64 cz = clampi((i64)(pz / A->cwz), 0, A->gz - 1);
            float mu = A->mu[cx + A->gx * (cy + A->gy * cz)];
            if (A->skip_empty && mu <= 0.0f) {
                double tx, ty, tz;
                if (dx > 0.0) tx = ((double)(cx + 1) * A->cwx - ox) / dx;
                else if (dx < 0.0) tx = ((double)cx * A->cwx - ox) / dx;
                else tx = INFINITY;
                if (dy > 0.0) ty = ((double)(cy + 1) * A->cwy - oy) / dy;
                else if (dy < 0.0) ty = ((double)cy * A->cwy - oy) / dy;
                else ty = INFINITY;
                if (dz > 0.0) tz = ((double)(cz + 1) * A->cwz - oz) / dz;
                else if (dz < 0.0) tz = ((double)cz * A->cwz - oz) / dz;
                else tz = INFINITY;
                double te = fmin(tx, fmin(ty, tz));
                if (te < t_c + 1e-9) te = t_c + 1e-9;
                if (A->adaptive) {
                    t_c = te + 1e-9;
                } else {
                    i64 jump = (i64)ceil((te - A->t_en[i]) / A->dt_base - 0.5);
                    if (jump < A->cursor_k[i] + 1) jump = A->cursor_k[i] + 1;
                    A->cursor_k[i] = jump;
                    t_c = A->t_en[i] + ((double)jump + 0.5) * A->dt_base;
                }
                continue;
            }
            if (A->adaptive) {
                double base = A->skip_empty ? (double)mu : 1.0;
                if (base < A->mu_floor) base = A->mu_floor;
                double step = A->dt_base / base;
                double limit = end - t_c;
                if (step > limit) step = limit;
                if (step < 1e-9) step = 1e-9;
                double tm = t_c + 0.5 * step;
                A->out_pos[3 * i] = ox + dx * tm;
                A->out_pos[3 * i + 1] = oy + dy * tm;
                A->out_pos[3 * i + 2] = oz + dz * tm;
                A->out_dt[i] = step;
                A->out_tmid[i] = tm;
                A->cursor_f[i] = t_c + step;
            } else {
                A->out_pos[3 * i] = px;
                A->out_pos[3 * i + 1] = py;
                A->out_pos[3 * i + 2] = pz;
                A->out_dt[i] = A->dt_base;
                A->out_tmid[i] = t_c;
                A->cursor_k[i] += 1;
            }
            A->sample_mask[i] = 1;
            break;
        }
    }
}

/* ---------------------------------------------------------------- probe
 * kernels.py:166-273 (_probe_one) + the count fold of _probe_serial. */
typedef struct {
    const double *pos, *dist, *u;
    double lod_scale;
    int mode; /* 0 corrected, 1 as_printed, 2 off */
    double vx, vy, vz;
    i64 max_lod, b;
    const int32_t *table;
    const i64 *offsets, *grids; /* grids [L+1][3] */
    const float *pool;
    i64 *last_used;
    i64 frame;
    float *values;
    int8_t *served, *req;
} orc_probe_args;

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

void orc_probe(i64 n, const orc_probe_args *P, i64 *counts /* exact, fallback, miss */) {
    i64 ex = 0, fb = 0, ms = 0;
#pragma omp parallel for schedule(static) reduction(+ : ex, fb, ms) if (n >= 6144)
    for (i64 i = 0; i < n; i++) {
        i64 b = P->b;
        double px = clampd(P->pos[3 * i] * P->vx - 0.5, 0.0, P->vx - 1.0);
        double py = clampd(P->pos[3 * i + 1] * P->vy - 0.5, 0.0, P->vy - 1.0);
        double pz = clampd(P->pos[3 * i + 2] * P->vz - 0.5, 0.0, P->vz - 1.0);
        double dd = P->dist[i] * P->lod_scale;
        i64 base_l = (i64)floor(dd);
        double frac = dd - (double)base_l;
        i64 lod = base_l;
        if (P->mode == 0) lod += (P->u[i] < frac) ? 1 : 0;
        else if (P->mode == 1) lod += (P->u[i] > frac) ? 1 : 0;
        lod = clampi(lod, 0, P->max_lod);
        P->req[i] = (int8_t)lod;
        i64 served = -1;
        float val = 0.0f;
        for (i64 level = lod; level <= P->max_lod; level++) {
            i64 span = b << level;
            i64 ggx = P->grids[3 * level], ggy = P->grids[3 * level + 1], ggz = P->grids[3 * level + 2];
            i64 ix = clampi((i64)py_floordiv(px + 1.0, (double)span), 0, ggx - 1);
            i64 iy = clampi((i64)py_floordiv(py + 1.0, (double)span), 0, ggy - 1);
            i64 iz = clampi((i64)py_floordiv(pz + 1.0, (double)span), 0, ggz - 1);
            int32_t slot = P->table[P->offsets[level] + ix + ggx * (iy + ggy * iz)];
            if (slot < 0) continue;
            double stride = (double)((i64)1 << level);
            double lx = clampd((px - (double)(ix * span - (ix > 0 ? 1 : 0))) / stride, 0.0, (double)b - 1.0);
            double ly = clampd((py - (double)(iy * span - (iy > 0 ? 1 : 0))) / stride, 0.0, (double)b - 1.0);
            double lz = clampd((pz - (double)(iz * span - (iz > 0 ? 1 : 0))) / stride, 0.0, (double)b - 1.0);
            i64 x0 = (i64)lx, y0 = (i64)ly, z0 = (i64)lz;
            if (x0 > b - 2) x0 = b - 2;
            if (y0 > b - 2) y0 = b - 2;
            if (z0 > b - 2) z0 = b - 2;
            float fx = (float)(lx - (double)x0), fy = (float)(ly - (double)y0), fz = (float)(lz - (double)z0);
            float hx = 1.0f - fx, hy = 1.0f - fy, hz = 1.0f - fz;
            const float *c = P->pool + (((i64)slot * b + z0) * b + y0) * b + x0;
            i64 sy = b, sz = b * b;
            float c00 = c[0] * hx + c[1] * fx;
            float c10 = c[sy] * hx + c[sy + 1] * fx;
            float c01 = c[sz] * hx + c[sz + 1] * fx;
            float c11 = c[sz + sy] * hx + c[sz + sy + 1] * fx;
            val = (c00 * hy + c10 * fy) * hz + (c01 * hy + c11 * fy) * fz;
            served = level;
            P->last_used[slot] = P->frame;
            break;
        }
        P->values[i] = val;
        P->served[i] = (int8_t)served;
        i64 gap = served - lod;
        if (gap == 0) ex++;
        else if (gap > 0) fb++;
        else ms++;
    }
    counts[0] = ex; counts[1] = fb; counts[2] = ms;
}

/* ---------------------------------------------------------------- shade
 * kernels.py:322-355 (_shade_one).  lut [size][4] f32. */
void orc_shade(i64 n, const i64 *rows, const float *values, const double *dt, const float *lut, i64 size,
               int adaptive, double dt_base, double term, double *color, double *trans, uint8_t *dead) {
#pragma omp parallel for schedule(static) if (n >= 6144)
    for (i64 j = 0; j < n; j++) {
        i64 i = rows[j];
        float v = values[j];
        if (v < 0.0f) v = 0.0f;
        else if (v > 1.0f) v = 1.0f;
        double q = (double)v * (double)(size - 1);
        i64 i0 = (i64)q;
        if (i0 > size - 2) i0 = size - 2;
        float f = (float)(q - (double)i0);
        float g = 1.0f - f;
        const float *l0 = lut + 4 * i0, *l1 = lut + 4 * (i0 + 1);
        float r = l0[0] * g + l1[0] * f;
        float gg = l0[1] * g + l1[1] * f;
        float bb = l0[2] * g + l1[2] * f;
        float a = l0[3] * g + l1[3] * f;
        double alpha = (double)a;
        if (adaptive) {
            double ratio = dt[j] / dt_base;
            if (alpha > 1.0 - 1e-12) alpha = 1.0 - 1e-12;
            if (alpha * ratio < 1e-4) alpha = alpha * ratio;
            else alpha = 1.0 - pow(1.0 - alpha, ratio);
        }
        double w = trans[i] * alpha;
        color[3 * i] += w * (double)r;
        color[3 * i + 1] += w * (double)gg;
        color[3 * i + 2] += w * (double)bb;
        trans[i] *= 1.0 - alpha;
        if (trans[i] < term) dead[j] = 1;
    }
}

/* ---------------------------------------------------------------- INR
 * Hash-grid encode (encoding.py:91-134) and MLP forward (mlp.py:39-53),
 * InrField clip (model.py:88-89).  Reductions are sequential in f32 (the
 * reference's einsum / sgemm orders are unspecified: tolerance parity, P14). */
typedef struct {
    i64 levels, feats;
    const i64 *res;        /* per level resolution */
    const uint8_t *dense;  /* per level dense flag */
    const i64 *tab_off;    /* per level row offset into tables */
    i64 table_size;
    const float *tables;   /* concatenated [rows][feats] */
    i64 n_layers;          /* weight matrices incl. output */
    const i64 *dims;       /* n_layers+1 widths */
    const float *const *W; /* (out,in) row-major */
    const float *const *B;
    int out_sigmoid;
} orc_inr_args;

static const uint64_t HP0 = 2654435761ull, HP1 = 2246822519ull, HP2 = 3266489917ull;

void orc_inr_encode(i64 n, const double *pos, const orc_inr_args *M, float *feat /* [n][levels*feats] */) {
    i64 nf = M->feats, od = M->levels * M->feats;
#pragma omp parallel for schedule(static) if (n >= 4096)
    for (i64 s = 0; s < n; s++) {
        for (i64 l = 0; l < M->levels; l++) {
            i64 r = M->res[l];
            double u[3], fr[3];
            uint64_t c0[3];
            for (int a = 0; a < 3; a++) {
                u[a] = pos[3 * s + a] * (double)r;
                double fl = floor(u[a]);
                i64 ci = (i64)fl;
                ci = clampi(ci, 0, r - 1);
                c0[a] = (uint64_t)ci;
                fr[a] = u[a] - (double)ci;
            }
            double wx[2] = {1.0 - fr[0], fr[0]}, wy[2] = {1.0 - fr[1], fr[1]}, wz[2] = {1.0 - fr[2], fr[2]};
            float acc[16];
            for (i64 f = 0; f < nf; f++) acc[f] = 0.0f;
            uint64_t side = (uint64_t)(r + 1);
            for (int c = 0; c < 8; c++) {
                int ddx = c & 1, ddy = (c >> 1) & 1, ddz = (c >> 2) & 1;
                uint64_t vx = c0[0] + ddx, vy = c0[1] + ddy, vz = c0[2] + ddz;
                uint64_t idx = M->dense[l] ? vx + side * vy + side * side * vz
                                           : ((vx * HP0) ^ (vy * HP1) ^ (vz * HP2)) & (uint64_t)(M->table_size - 1);
                float w = (float)(wx[ddx] * wy[ddy] * wz[ddz]);
                const float *row = M->tables + (M->tab_off[l] + (i64)idx) * nf;
                for (i64 f = 0; f < nf; f++) acc[f] += w * row[f];
            }
            for (i64 f = 0; f < nf; f++) feat[s * od + l * nf + f] = acc[f];
        }
    }
}

void orc_inr_mlp(i64 n, const float *feat, const orc_inr_args *M, float *out) {
#pragma omp parallel for schedule(static) if (n >= 4096)
    for (i64 s = 0; s < n; s++) {
        float a[256], z[256];
        i64 w0 = M->dims[0];
        for (i64 k = 0; k < w0; k++) a[k] = feat[s * w0 + k];
        for (i64 L = 0; L < M->n_layers; L++) {
            i64 din = M->dims[L], dout = M->dims[L + 1];
            for (i64 o = 0; o < dout; o++) {
                float accum = 0.0f;
                const float *wr = M->W[L] + o * din;
                for (i64 k = 0; k < din; k++) accum += a[k] * wr[k];
                z[o] = accum + M->B[L][o];
            }
            if (L + 1 < M->n_layers)
                for (i64 o = 0; o < dout; o++) a[o] = z[o] > 0.0f ? z[o] : 0.0f;
        }
        float zo = z[0], y;
        if (M->out_sigmoid) y = 1.0f / (1.0f + expf(-zo));
        else y = zo < 0.0f ? 0.0f : (zo > 1.0f ? 1.0f : zo);
        out[s] = y;
    }
}

/* ---------------------------------------------------------------- lattice
 * fields.py:165-199 trilinear_lattice, as RawLatticeField._evaluate (202-221)
 * calls it: u = pos*dims - 0.5; arithmetic in f64, result rounded to f32. */
void orc_lattice_sample(i64 n, const double *pos, const float *lat, i64 vx, i64 vy, i64 vz, float *out) {
#pragma omp parallel for schedule(static) if (n >= 4096)
    for (i64 s = 0; s < n; s++) {
        double x = clampd(pos[3 * s] * (double)vx - 0.5, 0.0, (double)(vx - 1));
        double y = clampd(pos[3 * s + 1] * (double)vy - 0.5, 0.0, (double)(vy - 1));
        double z = clampd(pos[3 * s + 2] * (double)vz - 0.5, 0.0, (double)(vz - 1));
        i64 x0 = (i64)floor(x), y0 = (i64)floor(y), z0 = (i64)floor(z);
        i64 x1 = x0 + 1 < vx - 1 ? x0 + 1 : vx - 1;
        i64 y1 = y0 + 1 < vy - 1 ? y0 + 1 : vy - 1;
        i64 z1 = z0 + 1 < vz - 1 ? z0 + 1 : vz - 1;
        double fx = x - (double)x0, fy = y - (double)y0, fz = z - (double)z0;
#define L(zz, yy, xx) lat[((zz) * vy + (yy)) * vx + (xx)]
        float c000 = L(z0, y0, x0), c100 = L(z0, y0, x1), c010 = L(z0, y1, x0), c110 = L(z0, y1, x1);
        float c001 = L(z1, y0, x0), c101 = L(z1, y0, x1), c011 = L(z1, y1, x0), c111 = L(z1, y1, x1);
#undef L
        double c00 = (double)c000 + (double)(c100 - c000) * fx;
        double c10 = (double)c010 + (double)(c110 - c010) * fx;
        double c01 = (double)c001 + (double)(c101 - c001) * fx;
        double c11 = (double)c011 + (double)(c111 - c011) * fx;
        double c0 = c00 + (c10 - c00) * fy;
        double c1 = c01 + (c11 - c01) * fy;
        out[s] = (float)(c0 + (c1 - c0) * fz);
    }
}
