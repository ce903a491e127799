"""GPU-resident drop-in for voxcache.session.RenderSession (session.py:26-152).

Same constructor, methods, FrameRecord and frame cycle:
    render (vcb_march_frame) -> maintenance (vcb_maintenance) -> tick.
The cache, request table and loader staging live in HBM; the host issues two
C-ABI calls per frame and reads back one small stats block (plus the image
when the caller wants it on the host, as the reference API returns it).

Loader semantics are the reference InlineLoader (P12): a batch dispatched at
maintenance f is decoded into a staging slab on the GPU right away and
inserted at maintenance f+1.  `loader="thread"` maps to the same deterministic
schedule (the GPU decode of one batch always completes within a frame).
"""

from __future__ import annotations

import ctypes as C
import time
import weakref
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _native as N
from . import macrocell
from .cache import CacheConfig, DeviceCache
from .device import device_field, ptr, require_cuda, stream_ptr
from .errors import ConfigError, ModelCorruptError, RenderError
from .render import PT_MAX_WALK, RenderSettings, base_step, camera_frame_setup, pcg64_seeded_state
from .sampler import (MASK64, MODES, LodPolicy, effective_lod_scale, force_max_scale, frame_rng_base,
                      splitmix64)
from .scheduler import SchedulerConfig


@dataclass
class SessionConfig:
    cached: bool = True
    mode: str = "raymarch"
    loader: str = "thread"
    cache: CacheConfig = dc_field(default_factory=CacheConfig)
    scheduler: SchedulerConfig = dc_field(default_factory=SchedulerConfig)
    policy: LodPolicy = dc_field(default_factory=LodPolicy)
    settings: RenderSettings = dc_field(default_factory=RenderSettings)
    macro_cell_size: int = 16
    samples_per_pixel: int = 1
    seed: int = 0


@dataclass
class FrameRecord:
    frame: int
    wall_s: float
    fps: float
    samples: int
    true_misses: int
    fallback_hits: int
    exact_hits: int
    occupancy: float
    bricks_loaded: int
    bricks_loaded_total: int
    requests_inflight: int


_EPOCH = [1]


def _next_epoch() -> int:
    _EPOCH[0] = (_EPOCH[0] + 1) & 0x3FFFF or 1
    return _EPOCH[0]


class RenderSession:
    """Owns the device render state for one viewer/bench run."""

    def __init__(self, field_src, tf, camera, config: SessionConfig, macro=None, device=None, debug=False,
                 stream=None, march="parity"):
        self.device = require_cuda(device)
        if config.mode not in ("raymarch", "pathtrace"):
            raise ValueError(f"unknown mode {config.mode!r}")
        if config.loader not in ("inline", "thread"):
            raise ValueError(f"unknown loader kind {config.loader!r}")
        self.field = field_src
        self.config = config
        self.dims = tuple(int(d) for d in field_src.domain.dims)
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self._dfield = device_field(field_src, self.device)
        with torch.cuda.stream(self.stream):
            self.macro = macro if macro is not None else macrocell.build(field_src, self.dims,
                                                                          config.macro_cell_size, self.device)
        self.tf = tf
        self._set_majorants(tf)
        self.camera = camera
        self.debug = debug
        if config.cached:
            with torch.cuda.stream(self.stream):
                self.cache = DeviceCache(self.dims, config.cache, config.scheduler, self.device, debug=debug)
        else:
            self.cache = None
        self.frame = 0
        self.mode = config.mode
        self._ws = None
        self._img = None
        # the frame's counters and the cache's state words share one device buffer, so the
        # FrameRecord needs a single device-to-host copy per frame
        ns = C.sizeof(N.VcbFrameStats) // 8
        self._dev_stats = torch.zeros(ns + (self.cache.state.numel() if self.cache else 0), dtype=torch.int64,
                                      device=self.device)
        self._stats = self._dev_stats[:ns]
        if self.cache is not None:
            with torch.cuda.stream(self.stream):
                self._dev_stats[ns:].copy_(self.cache.state)
            self.cache.state = self._dev_stats[ns:]
        self._host_stats = torch.zeros(self._dev_stats.numel(), dtype=torch.int64).pin_memory()
        self.last_frame_stats = {}
        self.timing = False  # CUDA-event time the frame kernel (bench)
        self.trace = False  # record the per-iteration trace (diagnostics)
        self.impl = 0  # march schedule (VcbFrameParams.impl), set through `march`
        self.march = march
        self.band = (0, 1)  # film rows row0, row0+step, ... (sort-first multi-GPU)
        self.maint_graph = True  # replay the maintenance as one CUDA graph (False: kernel by kernel)
        self._share = None  # parallel.BrickShare: brick decodes shared across ranks (share_decode)
        self._target = None  # whole-frame buffer written in place (fused sort-first gather)
        self._pin_free = []  # pinned host frames released by callers
        # loader="thread" (the reference's default, a background decode thread): the batch a
        # maintenance selects is decoded on a decode stream while the next frame marches, and
        # inserted by the next maintenance (the inline cadence, P12, so state is identical)
        self._dstream = torch.cuda.Stream(self.device) if (config.loader == "thread" and config.cached) else None
        self._cstream = torch.cuda.Stream(self.device)  # device-to-host image copies
        self._ev_image = torch.cuda.Event()
        # this session's own timing events (the library's per-thread ones would be shared
        # by every session driven from the same thread)
        self._ev_t0, self._ev_t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self._timed_launches = 0
        self._ev_decoded = None

    MARCH_SCHEDULES = {"parity": 0, "throughput": 10}

    @property
    def march(self) -> str:
        """Frame-kernel schedule: "parity" (default) numbers the stochastic-LoD RNG lanes
        by sample rank per wavefront iteration exactly as the reference (sampler.py:206-213),
        so cache state is bit-exact; "throughput" marches one persistent ray per GPU lane
        with lane = film pixel (same per-sample distribution, no grid barriers; bit-exact
        with "parity" when LodPolicy.mode == "off")."""
        for k, v in self.MARCH_SCHEDULES.items():
            if v == self.impl:
                return k
        return f"impl{self.impl}"

    @march.setter
    def march(self, name: str):
        if name not in self.MARCH_SCHEDULES:
            raise ValueError(f"unknown march schedule {name!r} (parity | throughput)")
        self.impl = self.MARCH_SCHEDULES[name]

    def share_decode(self, ctx, cap=None):
        """Decode each frame's brick batch jointly with the other ranks of `ctx`
        (parallel.BrickShare): every distinct requested brick is decoded once, by its
        owner rank, and all-gathered.  Same cache state as decoding alone; with
        loader="thread" the decode then runs on the session stream.  ctx=None turns it off."""
        from .parallel import BrickShare

        self._sync_decode()
        self._share = BrickShare(ctx, self, cap) if ctx is not None else None

    def set_band(self, row0: int, row_step: int):
        """Render only film rows row0 + j*row_step (one rank's share of a frame)."""
        if row_step < 1 or not 0 <= row0 < row_step:
            raise ValueError("band needs 0 <= row0 < row_step")
        self.band = (int(row0), int(row_step))

    def set_frame_target(self, target):
        """Write this session's rows straight into `target`, a whole-frame (H, W, 4) f32
        CUDA tensor (e.g. rank 0's frame mapped over NVLink by symmetric memory), at
        film rows row0 + j*row_step: the sort-first gather fused into the frame kernel.
        None restores the session's own band image."""
        if target is not None:
            if target.dtype != torch.float32 or target.dim() != 3 or target.shape[2] != 4 or not target.is_cuda:
                raise ValueError("frame target must be a CUDA f32 tensor of shape (H, W, 4)")
            if not target.is_contiguous():
                raise ValueError("frame target must be contiguous")
        self._target = target

    def _band_rows(self, H: int) -> int:
        row0, step = self.band
        return max(0, (H - row0 + step - 1) // step)

    # -- control (session.py:78-101)
    def _set_majorants(self, tf):
        """macrocell.update_majorants on the device (vcb_update_majorants): the macro
        grid's min/max stay resident; a TF change recomputes the majorants in place."""
        m = self.macro
        if getattr(self, "_vminmax", None) is None:
            self._vminmax = (torch.from_numpy(np.ascontiguousarray(m.value_min, dtype=np.float32)).to(self.device),
                             torch.from_numpy(np.ascontiguousarray(m.value_max, dtype=np.float32)).to(self.device))
            self._mu = torch.empty(self._vminmax[0].shape, dtype=torch.float32, device=self.device)
        bm = torch.from_numpy(macrocell.opacity_bin_maxima(tf)).to(self.device)
        vmin, vmax = self._vminmax
        with torch.cuda.device(self.device):  # the session stream's device, whatever is current
            N.call("vcb_update_majorants", ptr(vmin), ptr(vmax), vmin.numel(), ptr(bm), bm.numel(), ptr(self._mu),
                   stream_ptr(self.stream))
        self._bm = bm  # keep alive until the stream ran
        self._lut = torch.from_numpy(np.ascontiguousarray(tf.lookup_table(), dtype=np.float32)).to(self.device)
        # control points for the path tracer's np.interp (tf.opacity / tf.eval, transfer.py:28-56)
        self._tfp = torch.from_numpy(np.array(tf.points, dtype=np.float64)).to(self.device)

    def set_camera(self, camera):
        self.camera = camera

    def set_transfer_function(self, tf):
        self.tf = tf
        self._set_majorants(tf)

    def set_lod_scale(self, scale: float):
        self.config.policy.lod_scale = float(scale)

    def set_mode(self, mode: str):
        if mode not in ("raymarch", "pathtrace"):
            raise ValueError(f"unknown mode {mode!r}")
        self.mode = mode

    def _sync_decode(self):
        """Order the session stream after an outstanding deferred decode."""
        if self._ev_decoded is not None:
            self.stream.wait_event(self._ev_decoded)

    def reset_cache(self):
        if self.cache is not None:
            self._sync_decode()
            with torch.cuda.stream(self.stream):
                self.cache.reset()
        self.frame = 0

    # -- frame cycle (session.py:105-130)
    def _static_key(self, W, H):
        """Everything the frame parameters depend on besides the camera pose and the
        per-frame clocks (settings are re-read each frame, as the reference does)."""
        cfg = self.config
        s = cfg.settings
        m, c = self.macro, self.cache
        return (W, H, self.band, tuple(m.grid_dims), m.cell_size, ptr(self._lut), self._lut.shape[0], ptr(self._mu),
                bytes(self._dfield.desc), ptr(c.table) if c is not None else 0, ptr(self._stats),
                s.adaptive_step, s.skip_empty, s.base_step_scale, s.mu_floor, s.early_termination,
                tuple(s.background), s.max_iterations, cfg.policy.mode, getattr(cfg.scheduler, "decode_budget", None))

    def _frame_template(self, W, H):
        """The frame parameters that stay fixed between frames, as raw bytes (host
        submission is on the frame's critical path: the GPU waits for the first launch)."""
        cfg = self.config
        s = cfg.settings
        p = N.VcbFrameParams()
        p.cam.width, p.cam.height = W, H
        row0, step = self.band
        p.cam.row0, p.cam.row_step, p.cam.rows = row0, step, self._band_rows(H)
        vx, vy, vz = self.dims
        m = self.macro
        p.adv.adaptive = 1 if s.adaptive_step else 0
        p.adv.skip_empty = 1 if s.skip_empty else 0
        p.adv.dt_base = base_step(self.dims, s)
        p.adv.mu_floor = float(s.mu_floor)
        p.adv.gx, p.adv.gy, p.adv.gz = m.grid_dims
        p.adv.cwx, p.adv.cwy, p.adv.cwz = m.cell_size / vx, m.cell_size / vy, m.cell_size / vz
        pol = cfg.policy
        if pol.mode not in MODES:
            raise ValueError(f"unknown stochastic lod mode {pol.mode!r}")
        c = self.cache
        if c is not None:
            lay = c.layout
            p.probe.vx, p.probe.vy, p.probe.vz = float(vx), float(vy), float(vz)
            p.probe.mode = MODES[pol.mode]
            p.probe.max_lod = c.max_lod
            p.probe.b = lay.brick_size
            p.probe.b_pow2 = 1 if (lay.brick_size & (lay.brick_size - 1)) == 0 else 0
            for l in range(c.max_lod + 1):
                for a in range(3):
                    p.probe.grid[l][a] = lay.grids[l][a]
                p.probe.offset[l] = lay.offsets[l]
            p.cached = 1
            p.paged_dist = 1 if c.paged else 0
            p.table, p.pool, p.last_used, p.miss_count = ptr(c.table), ptr(c.pool), ptr(c.last_used), ptr(c.miss_count)
        p.term = float(s.early_termination)
        for a in range(3):
            p.bg[a] = float(s.background[a])
        p.lut_size = self._lut.shape[0]
        p.max_iterations = int(s.max_iterations)
        p.mu, p.lut = ptr(self._mu), ptr(self._lut)
        p.field = self._dfield.desc
        budget = getattr(cfg.scheduler, "decode_budget", None)
        p.miss_budget = -1 if budget is None else int(budget)
        p.stats = ptr(self._stats)
        self._ws_need = N.load().vcb_frame_workspace_bytes(W * p.cam.rows, p.max_iterations)
        return bytes(p)

    def _frame_params(self, image):
        cam = self.camera
        cfg = self.config
        W, H = int(cam.width), int(cam.height)
        key = self._static_key(W, H)
        if getattr(self, "_tmpl_key", None) != key:
            self._tmpl = self._frame_template(W, H)
            self._tmpl_key = key
        p = N.VcbFrameParams.from_buffer_copy(self._tmpl)
        # per frame: the camera pose, the LoD scale of the preload ramp, the clocks
        origin, rot, tan_h, tan_v, box_dist = camera_frame_setup(cam)
        p.cam.origin[:] = origin
        p.cam.rot[:] = rot
        p.cam.tan_h, p.cam.tan_v = tan_h, tan_v
        c = self.cache
        if c is not None:
            force = force_max_scale(c.max_lod, box_dist)
            p.probe.lod_scale = effective_lod_scale(cfg.policy, self.frame, force)
            p.cache_frame = c.frame
        p.rng_base = frame_rng_base(cfg.seed, self.frame)
        p.epoch = _next_epoch()
        p.timing = (1 if self.timing else 0) | (2 if self.trace else 0)
        p.impl = self.impl
        p.image = ptr(image)
        p.image_global = 1 if (self._target is not None and image is self._target) else 0
        if self._ws is None or self._ws.numel() < self._ws_need:
            self._ws = torch.empty(self._ws_need, dtype=torch.uint8, device=self.device)
        p.workspace = ptr(self._ws)
        p.workspace_bytes = self._ws.numel()
        return p

    def _pt_params(self, p, pcg=None, n_rays=None):
        """pathtrace_frame's scalars (pathtrace.py:112-117, 101-104): the numpy PCG64
        stream of default_rng(splitmix64((seed & 0xFFFFFFFF) ^ frame)) as seeded state,
        the normalised light direction, the TF control points."""
        cfg = self.config
        s = cfg.settings
        q = N.VcbPtParams()
        q.spp = int(cfg.samples_per_pixel)
        q.max_walk = PT_MAX_WALK
        q.density = float(s.pt_density)
        q.ambient = float(s.pt_ambient)
        light = -np.asarray(s.light_dir, dtype=np.float64)
        light /= np.linalg.norm(light)
        for a in range(3):
            q.light[a] = float(light[a])
        q.n_tf = int(self._tfp.shape[0])
        q.tf = ptr(self._tfp)
        if pcg is None:
            pcg = pcg64_seeded_state(splitmix64((cfg.seed & 0xFFFFFFFF) ^ self.frame))
        st, inc = pcg
        q.pcg_state[0], q.pcg_state[1] = st & MASK64, st >> 64
        q.pcg_inc[0], q.pcg_inc[1] = inc & MASK64, inc >> 64
        q.lane_seed = cfg.seed & MASK64
        q.lane_frame = self.frame
        n_rays = int(p.cam.width) * int(p.cam.rows) if n_rays is None else int(n_rays)
        need = N.load().vcb_pt_workspace_bytes(n_rays)
        if getattr(self, "_pt_ws", None) is None or self._pt_ws.numel() < need:
            self._pt_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        q.workspace = ptr(self._pt_ws)
        q.workspace_bytes = self._pt_ws.numel()
        return q

    def trace_free_flight(self, origins, directions, t_start, t_end, rng):
        """pathtrace.py:28-98 `trace_free_flight(scene, ...)` on this session's sampler,
        macro grid and settings: delta-track each ray to its first real collision.
        `rng` is a numpy Generator (PCG64); it is advanced by the draws the walk used,
        exactly as the reference's calls would have.  Returns (t_hit, value) host arrays,
        t_hit = +inf for rays that escape.  The sampler starts a fresh lane pool."""
        st = rng.bit_generator.state
        if st.get("bit_generator") != "PCG64":
            raise ValueError("trace_free_flight needs a numpy PCG64 generator (np.random.default_rng)")
        o = np.ascontiguousarray(np.asarray(origins, dtype=np.float64).reshape(-1, 3))
        n = o.shape[0]
        d = np.ascontiguousarray(np.broadcast_to(np.asarray(directions, dtype=np.float64), (n, 3)))
        t0 = np.ascontiguousarray(np.broadcast_to(np.asarray(t_start, dtype=np.float64), (n,)))
        t1 = np.ascontiguousarray(np.broadcast_to(np.asarray(t_end, dtype=np.float64), (n,)))
        dev = [torch.from_numpy(np.array(a)).to(self.device) for a in (o, d, t0, t1)]
        t_hit = torch.empty(n, dtype=torch.float64, device=self.device)
        v_hit = torch.empty(n, dtype=torch.float32, device=self.device)
        if self._img is None:
            self._img = torch.empty((1, 1, 4), dtype=torch.float32, device=self.device)
        draws = np.zeros(1, dtype=np.uint64)
        with torch.cuda.stream(self.stream):
            self._stats.zero_()
            p = self._frame_params(self._img)
            q = self._pt_params(p, pcg=(int(st["state"]["state"]), int(st["state"]["inc"])), n_rays=n)
            N.call("vcb_trace_free_flight", C.byref(p), C.byref(q), n, *(ptr(a) for a in dev), ptr(t_hit),
                   ptr(v_hit), draws.ctypes.data, stream_ptr(self.stream))
        if int(self._stats[7].item()):
            raise RenderError("miss resolution failed: inference produced non-finite outputs")
        rng.bit_generator.advance(int(draws[0]))
        return t_hit.cpu().numpy(), v_hit.cpu().numpy()

    def render_frame_device(self, out=None):
        """Render + maintenance on the session stream; returns the device image
        (H, W, 4) f32 without synchronising.  `collect_record()` finishes the frame.
        out: a (rows, W, 4) f32 buffer the frame kernels write instead (render_frame
        passes a pinned host frame: the pixels cross PCIe as the rays retire)."""
        W, H = int(self.camera.width), int(self.camera.height)
        R = self._band_rows(H)
        if out is not None:
            if tuple(out.shape) != (R, W, 4) or out.dtype != torch.float32:
                raise ValueError(f"frame buffer {tuple(out.shape)} {out.dtype} != {(R, W, 4)} float32")
            img = out
        elif self._target is not None:
            if tuple(self._target.shape) != (H, W, 4):
                raise ValueError(f"frame target shape {tuple(self._target.shape)} != {(H, W, 4)}")
            img = self._target
        else:
            if self._img is None or self._img.shape != (R, W, 4):
                self._img = torch.empty((R, W, 4), dtype=torch.float32, device=self.device)
            img = self._img
        with torch.cuda.stream(self.stream):
            if self.mode == "pathtrace":
                self._stats.zero_()  # (vcb_march_frame clears its counters itself)
            p = self._frame_params(img)
            if self.mode == "pathtrace":
                if self.band != (0, 1):
                    # one PCG64 stream orders the whole bundle (pathtrace.py:117-131): a band
                    # would draw different numbers than the full frame
                    raise ConfigError("path tracing renders whole frames; use alternate-frame rendering")
                q = self._pt_params(p)
                N.call("vcb_pathtrace_frame", C.byref(p), C.byref(q), stream_ptr(self.stream))
            else:
                if self.timing:
                    self._ev_t0.record(self.stream)
                N.call("vcb_march_frame", C.byref(p), stream_ptr(self.stream))
                if self.timing:
                    self._ev_t1.record(self.stream)
                    self._timed_launches = N.load().vcb_last_launch_count()
            # the image is final here: a host copy can overlap the maintenance below
            self._ev_image.record(self.stream)
            if self.cache is not None:
                # a frame whose true-miss inference failed raises RenderError in collect_record
                # without advancing the clocks; its maintenance skips itself on the device
                if self._ev_decoded is not None:
                    self.stream.wait_event(self._ev_decoded)  # the batch this maintenance inserts
                self.cache.maintenance(self.frame, self._dfield.desc, self.stream, frame_stats=ptr(self._stats),
                                       defer_decode=self._dstream is not None or self._share is not None,
                                       graph=self.maint_graph)
                if self._share is not None:
                    self._share.run(self.cache._last_params, self.stream)
                elif self._dstream is not None:
                    sel = torch.cuda.Event()
                    sel.record(self.stream)
                    self._dstream.wait_event(sel)
                    self.cache.decode(self._dstream)
                    self._ev_decoded = torch.cuda.Event()
                    self._ev_decoded.record(self._dstream)
            # one small D2H for the FrameRecord counters and the cache state
            self._host_stats.copy_(self._dev_stats, non_blocking=True)
        return img

    def collect_record(self, t0: float) -> FrameRecord:
        self.stream.synchronize()
        hs = self._host_stats.numpy()
        ns = self._stats.numel()
        fs = {f[0]: int(hs[i]) for i, f in enumerate(N.VcbFrameStats._fields_) if f[0] != "pad_"}
        self.last_frame_stats = fs
        if fs["nonfinite"]:
            raise RenderError("miss resolution failed: inference produced non-finite outputs")
        wall = time.perf_counter() - t0
        c = self.cache
        if c is not None:
            st = {f[0]: int(hs[ns + i]) for i, f in enumerate(N.VcbCacheState._fields_) if f[0] != "pad_"}
            self.last_cache_state = st
            rec = FrameRecord(self.frame, wall, 1.0 / wall if wall > 0 else float("inf"), fs["requests"], fs["miss"],
                              fs["fallback"], fs["exact"], 1.0 - (c.slots - st["next_free"]) / c.slots,
                              st["bricks_loaded"], st["loaded_total"], st["n_inflight"])
            c.frame += 1
        else:
            rec = FrameRecord(self.frame, wall, 1.0 / wall if wall > 0 else float("inf"), fs["requests"], fs["miss"],
                              0, 0, 0.0, 0, 0, 0)
        self.frame += 1
        return rec

    def render_frame(self):
        """Render, then run the maintenance phase; returns (image f32[H,W,4] on host, FrameRecord).
        The frame kernels store the pixels straight into a pinned host frame (mapped
        memory), so the image transfer overlaps the march instead of following it."""
        t0 = time.perf_counter()
        if self._target is None:
            host = self._pinned((self._band_rows(int(self.camera.height)), int(self.camera.width), 4))
            self.render_frame_device(out=host)
            rec = self.collect_record(t0)
            out = host.numpy()
            weakref.finalize(out, self._pin_free.append, host)
            return out, rec
        img = self.render_frame_device()
        host = self._pinned(tuple(img.shape))
        # the copy waits only for the frame kernel, not for the maintenance after it
        self._cstream.wait_event(self._ev_image)
        with torch.cuda.stream(self._cstream):
            host.copy_(img, non_blocking=True)
            img.record_stream(self._cstream)
        rec = self.collect_record(t0)
        self._cstream.synchronize()
        out = host.numpy()
        # the caller owns the array; its pinned buffer returns to the pool when it dies
        weakref.finalize(out, self._pin_free.append, host)
        return out, rec

    def render_frame_rgba8(self):
        """render_frame() for streaming: the frame is quantised on the device exactly as
        image_io.to_rgba8 (image_io.py:14-21) and 4 bytes per pixel cross PCIe.
        Returns (uint8 (H, W, 4) host array, FrameRecord)."""
        t0 = time.perf_counter()
        img = self.render_frame_device()
        if getattr(self, "_rgba8", None) is None or tuple(self._rgba8.shape) != tuple(img.shape):
            self._rgba8 = torch.empty(tuple(img.shape), dtype=torch.uint8, device=self.device)
        host = torch.empty(tuple(img.shape), dtype=torch.uint8, pin_memory=True)
        with torch.cuda.stream(self.stream):
            N.call("vcb_frame_rgba8", ptr(img), img.numel() // 4, ptr(self._rgba8), stream_ptr(self.stream))
            host.copy_(self._rgba8, non_blocking=True)
        rec = self.collect_record(t0)
        return host.numpy(), rec

    def _pinned(self, shape):
        """A pinned host frame buffer from the session's pool (pinned allocation costs
        milliseconds, so buffers released by the caller are reused)."""
        while self._pin_free:
            t = self._pin_free.pop()
            if tuple(t.shape) == shape:
                return t
        return torch.empty(shape, dtype=torch.float32, pin_memory=True)

    def reserve_host_frames(self, k: int = 2):
        """Pre-allocate k pinned host frames of the current camera's shape, so a loop
        that holds the previous frame while rendering the next never allocates."""
        H, W = int(self.camera.height), int(self.camera.width)
        shape = (self._band_rows(H), W, 4)
        have = sum(1 for t in self._pin_free if tuple(t.shape) == shape)
        for _ in range(max(0, k - have)):
            self._pin_free.append(torch.empty(shape, dtype=torch.float32, pin_memory=True))

    def march_kernel_time(self):
        """(ms, frames) of the frame-kernel call (ray setup + march) in the last
        timing=True frame, from this session's CUDA events on its stream."""
        self._ev_t1.synchronize()
        return self._ev_t0.elapsed_time(self._ev_t1), 1

    def frame_trace(self):
        """Per-iteration diagnostics of the last timing=True frame (default schedule):
        per CTA, ns from the iteration's earliest barrier exit to barrier exit, scan
        done and phase done; plus samples per iteration."""
        self.stream.synchronize()
        it = min(int(self.last_frame_stats.get("iterations", 0)), 512)
        W = int(self.camera.width)
        rows = self._band_rows(int(self.camera.height))
        max_it = int(self.config.settings.max_iterations)
        st = np.zeros((max(it, 1), 1024, 3), np.uint32)
        lv = np.zeros(it + 2, np.int32)
        n = N.load().vcb_frame_trace(ptr(self._ws), W * rows, max_it, it, st.ctypes.data, lv.ctypes.data)
        G = N.load().vcb_device_sm_count()
        st = st[:n, :G].astype(np.int64)
        t0 = st[:, :, 0].min(axis=1, keepdims=True)
        rel = ((st - t0[:, :, None]) % (1 << 32)).astype(np.int64)
        return {"samples": lv[1:n + 1].tolist(), "rays": int(lv[0]), "iters": int(n),
                "bar": rel[:, :, 0].tolist(), "scan": rel[:, :, 1].tolist(), "phase": rel[:, :, 2].tolist()}

    def frame_counters(self):
        """The u64 diagnostics counters of the last frame (CINR_STATS builds)."""
        self.stream.synchronize()
        W = int(self.camera.width)
        rows = self._band_rows(int(self.camera.height))
        out = np.zeros(23, np.int64)
        N.call("vcb_frame_counters", ptr(self._ws), W * rows, int(self.config.settings.max_iterations),
               out.ctypes.data)
        return out.tolist()

    def export_state(self):
        """Full device state as host arrays (tables, pool, owners, stamps, requests,
        staged loader batch): lets another implementation resume this session."""
        self._sync_decode()
        self.stream.synchronize()
        c = self.cache
        d = c.dump()
        st = d["state"]
        b3 = c.config.brick_size ** 3
        n = st["n_staged"]
        d["pool"] = c.pool.cpu().numpy()
        d["next_free"] = st["next_free"]
        d["loaded_total"] = st["loaded_total"]
        keys = c.staged_keys[:n].cpu().numpy()
        offs = np.asarray(c.layout.offsets, dtype=np.int64)
        l = np.searchsorted(offs, keys, side="right") - 1
        d["staged_keys"] = np.stack([l, keys - offs[l]], axis=1).reshape(-1, 2)
        d["staged_data"] = c.staging[: n * b3].cpu().numpy().reshape(n, b3)
        d["session_frame"] = self.frame
        return d

    def debug_state(self):
        """Reference-shaped per-frame state (tables, owner, stamps, requests, batch, reports)."""
        self._sync_decode()
        self.stream.synchronize()
        d = self.cache.dump()
        d["batch"] = self.cache.batch()
        d["reports"] = self.cache.reports()
        return d

    def close(self):
        self._sync_decode()
        self.stream.synchronize()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
