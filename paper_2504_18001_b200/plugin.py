"""Stage A drop-in: the reference's four numba passes served by the sm_100a kernels.

Signatures, argument meaning and in-place outputs are those of
voxcache/render/kernels.py (raygen_pass 426, advance_pass 160, probe_pass 316,
shade_pass 370).  Each call copies its numpy arguments to the device, runs the
C-ABI pass, and copies every mutated array back (the reference contract is
caller-owned arrays written in place).  `install(voxcache.render.kernels)`
swaps the module attributes the reference resolves at call time
(raymarch.py:73,87; sampler.py:242; camera.py:144), so the reference's own
RenderSession, tests and harness run on the GPU unchanged.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .device import ptr, require_cuda


def _d(a, dtype=None):
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return torch.from_numpy(arr).to("cuda", non_blocking=False)


def raygen_pass(base_dirs, rot, origin, tan_half_h, tan_half_v, dirs, t0_out, t1_out, keep):
    require_cuda()
    n = base_dirs.shape[0]
    if n == 0:
        return
    b, r, o = _d(base_dirs, np.float64), _d(rot, np.float64), _d(origin, np.float64)
    dd = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    a0 = torch.empty(n, dtype=torch.float64, device="cuda")
    a1 = torch.empty(n, dtype=torch.float64, device="cuda")
    k = torch.empty(n, dtype=torch.uint8, device="cuda")
    N.call("vcb_raygen_pass", n, ptr(b), ptr(r), ptr(o), float(tan_half_h), float(tan_half_v), ptr(dd), ptr(a0),
           ptr(a1), ptr(k), 0)
    dirs[...] = dd.cpu().numpy()
    t0_out[...] = a0.cpu().numpy()
    t1_out[...] = a1.cpu().numpy()
    keep[...] = k.cpu().numpy().astype(bool)


def advance_pass(o, d, t_en, t_ex, cursor_f, cursor_k, active, adaptive, skip_empty, dt_base, mu_floor, mu_flat,
                 gx, gy, gz, cwx, cwy, cwz, out_pos, out_dt, out_tmid, sample_mask, done_mask):
    require_cuda()
    n = o.shape[0]
    if n == 0:
        return
    s = N.VcbMarchStatic(int(bool(adaptive)), int(bool(skip_empty)), float(dt_base), float(mu_floor), int(gx), int(gy),
                         int(gz), float(cwx), float(cwy), float(cwz))
    to, td, te, tx = _d(o, np.float64), _d(d, np.float64), _d(t_en, np.float64), _d(t_ex, np.float64)
    cf, ck = _d(cursor_f, np.float64), _d(cursor_k, np.int64)
    act = _d(np.asarray(active).view(np.uint8))
    mu = _d(mu_flat, np.float32)
    op = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    odt = torch.empty(n, dtype=torch.float64, device="cuda")
    otm = torch.empty(n, dtype=torch.float64, device="cuda")
    sm = torch.empty(n, dtype=torch.uint8, device="cuda")
    dm = torch.empty(n, dtype=torch.uint8, device="cuda")
    N.call("vcb_advance_pass", n, ptr(to), ptr(td), ptr(te), ptr(tx), ptr(cf), ptr(ck), ptr(act), C.byref(s), ptr(mu),
           ptr(op), ptr(odt), ptr(otm), ptr(sm), ptr(dm), 0)
    cursor_f[...] = cf.cpu().numpy()
    cursor_k[...] = ck.cpu().numpy()
    smh = sm.cpu().numpy().astype(bool)
    # untouched output slots keep whatever the caller had (numba writes only sampled rows)
    rows = np.flatnonzero(smh)
    out_pos[rows] = op.cpu().numpy()[rows]
    out_dt[rows] = odt.cpu().numpy()[rows]
    out_tmid[rows] = otm.cpu().numpy()[rows]
    sample_mask[...] = smh
    done_mask[...] = dm.cpu().numpy().astype(bool)


def probe_static(lod_scale, mode, vx, vy, vz, max_lod, brick_size, offsets, grids):
    p = N.VcbProbeStatic()
    p.vx, p.vy, p.vz, p.lod_scale = float(vx), float(vy), float(vz), float(lod_scale)
    p.mode, p.max_lod, p.b = int(mode), int(max_lod), int(brick_size)
    p.b_pow2 = 1 if (int(brick_size) & (int(brick_size) - 1)) == 0 else 0
    g = np.asarray(grids, dtype=np.int64).reshape(-1, 3)
    for l in range(int(max_lod) + 1):
        for a in range(3):
            p.grid[l][a] = int(g[l, a])
        p.offset[l] = int(offsets[l])
    return p


def probe_pass(pos, dist, u, lod_scale, stochastic_mode, vx, vy, vz, max_lod, brick_size, table_flat, table_offsets,
               grids, pool_flat, last_used, frame, out_values, out_served, out_req):
    require_cuda()
    n = pos.shape[0]
    if n == 0:
        return 0, 0, 0
    p = probe_static(lod_scale, stochastic_mode, vx, vy, vz, max_lod, brick_size, table_offsets, grids)
    tp, td, tu = _d(pos, np.float64), _d(dist, np.float64), _d(u, np.float64)
    tab, pool, lu = _d(table_flat, np.int32), _d(pool_flat, np.float32), _d(last_used, np.int64)
    vals = torch.empty(n, dtype=torch.float32, device="cuda")
    srv = torch.empty(n, dtype=torch.int8, device="cuda")
    req = torch.empty(n, dtype=torch.int8, device="cuda")
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    N.call("vcb_probe_pass", n, ptr(tp), ptr(td), ptr(tu), C.byref(p), ptr(tab), ptr(pool), ptr(lu), int(frame),
           ptr(vals), ptr(srv), ptr(req), ptr(cnt), 0)
    out_values[...] = vals.cpu().numpy()
    out_served[...] = srv.cpu().numpy()
    out_req[...] = req.cpu().numpy()
    last_used[...] = lu.cpu().numpy()
    c = cnt.cpu().numpy()
    return int(c[0]), int(c[1]), int(c[2])


def shade_pass(rows, values, dt_i, lut, adaptive, dt_base, term_threshold, color, trans, dead_mask):
    require_cuda()
    n = rows.shape[0]
    if n == 0:
        return
    tr_, tv, tdt = _d(rows, np.int64), _d(values, np.float32), _d(dt_i, np.float64)
    tl = _d(lut, np.float32)
    tc, tt = _d(color, np.float64), _d(trans, np.float64)
    dm = _d(np.asarray(dead_mask).view(np.uint8))
    N.call("vcb_shade_pass", n, ptr(tr_), ptr(tv), ptr(tdt), ptr(tl), int(lut.shape[0]), int(bool(adaptive)),
           float(dt_base), float(term_threshold), ptr(tc), ptr(tt), ptr(dm), 0)
    color[...] = tc.cpu().numpy()
    trans[...] = tt.cpu().numpy()
    dead_mask[...] = dm.cpu().numpy().astype(bool)


PASSES = {"raygen_pass": raygen_pass, "advance_pass": advance_pass, "probe_pass": probe_pass,
          "shade_pass": shade_pass}


def install(kernels_module):
    """Swap the reference's pass attributes for the GPU ones; returns an undo callable."""
    saved = {k: getattr(kernels_module, k) for k in PASSES}
    for k, fn in PASSES.items():
        setattr(kernels_module, k, fn)

    def undo():
        for k, fn in saved.items():
            setattr(kernels_module, k, fn)

    return undo
