#!/usr/bin/env python
"""Headline benchmark: cached-INR ray-march frames/s at 1024^2 (BASELINE.json config 2).

Workload (configs[1]): 512^3 volume decoded from the random-init hash-grid INR
(HashGridConfig()/MLPConfig(), seed 0, parameters re-drawn uniform(-0.7,0.7) from
default_rng(42)), 16^3 bricks, 32^3-slot pool (537 MB), 1024x1024 frames on the
orbit (center .5, radius 2.2, 120 frames/rev, 20 deg elevation, fov 45),
warm_body(0.5, 0.9), LodPolicy(1.2, preload 20), 40 requests/frame, inline
loader (deterministic), seed 0.  A step = one RenderSession.render_frame()
(render + maintenance), the reference's fps definition (session.py:107-113).

  value : frames/s with everything resident in HBM (device-side render + stats
          readback), CUDA events on the session stream, L2 flushed between frames
  e2e   : the same frames through the public API render_frame() returning the
          host image (D2H inside the timed region)
  cpu_baseline : the CPU oracle (restated reference, all host threads) rendering
          the same steady-state frame from the GPU session's exact cache state

Multi-GPU (torchrun, N>1): by default alternate-frame rendering — rank r renders
the whole 1024^2 orbit frames r, r+N, ... with its own cache and the frames are
all-gathered with NCCL each step (scaling "weak": N frames per step);
`--mp tiles` renders sort-first row bands of every frame instead (scaling
"strong"; limited by the ~190 dependent iterations per frame).

`--impl reference` times the CPU oracle port alone (the reference path has no GPU
code) on a bounded sample of the same workload; see the JSON `cpu_baseline.sample`.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec at 1024^2 (cached INR render, 512^3 random-init INR, config 2)"
UNIT = "frames/s"
BYTES_PER_SAMPLE = 40  # 8 f32 corners + 1 i32 page-table entry + 1 f32 majorant


def workload(res=1024, volume=512, pool=32):
    return dict(workload="config2_cached_inr_raymarch", volume=f"{volume}^3 random-init INR (8x2 hash grid, 16-32-32-1)",
                image=f"{res}x{res}", brick=16, pool_slots=pool ** 3, orbit="r=2.2, 120 frames/rev, elev 20, fov 45",
                tf="warm_body(0.5,0.9)", lod_policy="scale 1.2, preload 20, corrected", max_requests=40,
                loader="inline", l2="flushed (256 MB write) between timed frames")


def make_model(volume):
    import paper_2504_18001_b200 as P

    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((volume,) * 3), seed=0)
    r = np.random.default_rng(42)
    m.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in m.parameters()])
    return m


def load_macro(volume):
    f = ROOT / "bench_data" / f"macro_inr{volume}_c16.npz"
    if f.exists():
        d = np.load(f)
        return d["vmin"], d["vmax"], "bench_data (CPU-oracle-built, shared by every arm)"
    return None, None, "built on the GPU (vcb_macro_minmax)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic():
    f = ROOT / "profiles" / "ncu_frame_kernel.json"
    if f.exists():
        try:
            return json.loads(f.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


# --------------------------------------------------------------------------- CPU arms
def cpu_oracle_frame_from_state(state, macro, res_frac, frame_idx, volume, frames=1):
    """Steady-state frames of the oracle, resumed from the GPU session's exact state."""
    from oracle import cinr_oracle as O

    t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
    fld = O.InrFieldOracle((volume,) * 3, t, w, b, O.DEFAULT_GRID)
    cfg = O.Config(dims=(volume,) * 3, brick=16, pool=(32, 32, 32), max_requests=40, lod_scale=1.2, preload=20)
    sess = O.OracleSession(fld, O.warm_body_points(0.5, 0.9), cfg, macro_minmax_arrays=macro)
    O.load_session_state(sess, state)
    res = int(1024 * res_frac)
    wall = 0.0
    for f in range(frames):
        pos = O.orbit_camera((0.5, 0.5, 0.5), 2.2, 120, frame_idx + f)
        sess.set_camera(pos, (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0, res, res)
        img, rec = sess.render_frame()
        wall += rec.wall_s
    return wall / frames, img, rec


def run_reference_arm(args):
    """`--impl reference`: the CPU oracle port (the reference has no GPU path) on all
    host threads, rendering the same orbit frames as the GPU arm (warm-up frames
    0..W-1 untimed, then frames W.., at most --ref-max-steps of them timed) at the
    same resolution, so the cache state evolves exactly as on the GPU."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cinr_oracle as O

    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    vmin, vmax, msrc = load_macro(args.volume)
    t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
    fld = O.InrFieldOracle((args.volume,) * 3, t, w, b, O.DEFAULT_GRID)
    if vmin is None:
        vmin, vmax = O.macro_minmax_streamed(fld, (args.volume,) * 3, 16)
    cfg = O.Config(dims=(args.volume,) * 3, brick=16, pool=(32, 32, 32), max_requests=40, lod_scale=1.2, preload=20)
    sess = O.OracleSession(fld, O.warm_body_points(0.5, 0.9), cfg, macro_minmax_arrays=(vmin, vmax))
    res = args.ref_res or args.res
    timed = max(1, min(args.steps, args.ref_max_steps))
    walls = []
    for f in range(args.warmup + timed):
        pos = O.orbit_camera((0.5, 0.5, 0.5), 2.2, 120, f)
        sess.set_camera(pos, (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0, res, res)
        img, rec = sess.render_frame()
        if f >= args.warmup:
            walls.append(rec.wall_s)
    scale = (res * res) / (args.res * args.res)
    fps = len(walls) / sum(walls) * scale if walls else 0.0
    sample = (f"oracle port (C+numpy restatement of voxcache, OpenMP {cores} threads): orbit frames "
              f"{args.warmup}..{args.warmup + timed - 1} (the GPU arm's first {timed} timed frames) at {res}^2 after "
              f"warm-up frames 0..{args.warmup - 1}; render + maintenance wall time per frame"
              + (f", fps scaled x{scale:.4f} (pixel ratio) to {args.res}^2" if scale != 1.0 else ""))
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 / fps if fps else None, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": workload(args.res, args.volume), "impl": "reference",
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--volume", type=int, default=512)
    ap.add_argument("--ref-res", type=int, default=0, help="reference arm resolution (0 = --res)")
    ap.add_argument("--ref-max-steps", type=int, default=8, help="reference arm: at most this many timed frames")
    ap.add_argument("--cpu-frac", type=float, default=1.0, help="oracle baseline image fraction of --res")
    ap.add_argument("--cpu-frames", type=int, default=3, help="oracle baseline frames (from the GPU state)")
    ap.add_argument("--decode-n", type=int, default=1 << 24, help="isolated INR decode batch (0 = skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--uncached-steps", type=int, default=5, help="frames of the no-cache INR baseline (0 = skip)")
    ap.add_argument("--train-steps", type=int, default=50,
                    help="INR training steps at batch 65536 (inr/train.py on the GPU; 0 = skip)")
    ap.add_argument("--pt-steps", type=int, default=5,
                    help="frames of the path-trace mode (pathtrace.py, spp 1) cached and uncached (0 = skip)")
    ap.add_argument("--mp", default="auto", choices=["auto", "frames", "tiles"],
                    help="N>1: 'frames' = alternate-frame rendering (each GPU renders whole 1024^2 frames of the orbit "
                         "with its own cache, frames gathered over NCCL; weak scaling, the default), 'tiles' = sort-first "
                         "row bands of every frame (strong scaling)")
    ap.add_argument("--fused-gather", action="store_true",
                    help="N>1: ranks write pixels straight into rank 0's frame (symmetric memory) instead of NCCL all-gather")
    ap.add_argument("--schedule", type=int, default=0,
                    help="march schedule (VcbFrameParams.impl): 0 one-barrier wavefront (default), 4 two-phase, 5 = 0 at 768 threads")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch

    from paper_2504_18001_b200 import parallel
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.macrocell import MacroCellGrid, layout
    from paper_2504_18001_b200.session import SessionConfig

    import paper_2504_18001_b200 as P

    ctx = parallel.init_from_env()
    dev = torch.device("cuda", ctx.local_rank)
    torch.cuda.set_device(dev)
    model = make_model(args.volume)
    fld = model.as_field()
    vmin, vmax, msrc = load_macro(args.volume)
    t_macro = None
    if vmin is None:
        from paper_2504_18001_b200 import macrocell

        t0 = time.perf_counter()
        mg = macrocell.build(fld, (args.volume,) * 3, 16, dev)
        t_macro = time.perf_counter() - t0
    else:
        grid, _, _ = layout((args.volume,) * 3, 16)
        mg = MacroCellGrid(16, (args.volume,) * 3, grid, vmin, vmax, np.ones_like(vmin))
    cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                        scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20),
                        settings=P.RenderSettings(), seed=0)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=args.res, height=args.res)
    mp = ("frames" if ctx.world > 1 else "single") if args.mp == "auto" else args.mp
    if ctx.world == 1:
        mp = "single"
    afr = mp == "frames"
    sess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, bands=not afr)
    sess.impl = args.schedule
    per_step = ctx.world if afr else 1  # 1024^2 frames completed per step, whole job

    def cam(f):
        # alternate-frame rendering: rank r renders orbit frames r, r + N, r + 2N, ...
        return traj.camera_at(f * ctx.world + ctx.rank if afr else f)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = sess.stream
    fused = None
    if args.fused_gather and ctx.world > 1 and ctx.backend == "nccl" and not afr:
        try:
            fused = parallel.FusedGather(ctx, sess, args.res, args.res)
        except Exception as exc:  # no peer mapping here: keep the NCCL all-gather
            print(f"fused gather unavailable ({exc}); using NCCL all-gather", file=sys.stderr)
            fused = None

    def gather(img):
        if afr:
            return parallel.gather_frames(ctx, img, st)
        if fused is not None:
            return fused.finish(st)
        return parallel.gather_frame(ctx, img, st, args.res)

    def frame_device(f):
        sess.set_camera(cam(f))
        t0 = time.perf_counter()
        img = sess.render_frame_device()
        return img, t0

    # warm-up (cold cache fills; untimed)
    verbose = bool(os.environ.get("CINR_BENCH_VERBOSE"))
    for f in range(args.warmup):
        if ctx.world == 1 and f >= args.warmup - 2:
            # the last warm-up frames go through the public call too (pins its host frame buffers)
            sess.set_camera(cam(f))
            t0 = time.perf_counter()
            _, rec = sess.render_frame()
        else:
            img, t0 = frame_device(f)
            gather(img)
            rec = sess.collect_record(t0)
        if verbose:
            print(f"warm {f}: {rec.wall_s * 1e3:.2f} ms samples {rec.samples} miss {rec.true_misses} "
                  f"fb {rec.fallback_hits} it {sess.last_frame_stats.get('iterations')} "
                  f"rays {sess.last_frame_stats.get('rays')} occ {rec.occupancy:.3f}", file=sys.stderr)
    torch.cuda.synchronize()

    # ---- timed: device-resident frames, one CUDA event pair per frame on the session stream
    sess.timing = True
    sess.trace = bool(os.environ.get("CINR_TRACE"))
    times, samples, march_ms, march_launches, launches, recs = [], 0, 0.0, 0, 0, []
    from paper_2504_18001_b200 import _native as N

    with ClockSampler(ctx.local_rank) as clk:
        for i in range(args.steps):
            f = args.warmup + i
            flush.zero_()
            torch.cuda.synchronize()
            parallel.barrier(ctx)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            img, t0 = frame_device(f)
            gather(img)
            e1.record(st)
            rec = sess.collect_record(t0)
            launches += N.load().vcb_last_launch_count()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            times.append(parallel.max_over_ranks(ctx, ms))
            samples += rec.samples
            recs.append(rec)
            if verbose:
                print(f"timed {f}: {ms:.3f} ms samples {rec.samples} miss {rec.true_misses} "
                      f"it {sess.last_frame_stats.get('iterations')}", file=sys.stderr)
            if os.environ.get("CINR_STATS"):
                print("counters", f, sess.frame_counters(), file=sys.stderr)
            km, kn = sess.march_kernel_time()
            march_ms += km
            march_launches += kn
    if os.environ.get("CINR_TRACE"):
        Path(os.environ["CINR_TRACE"]).write_text(json.dumps(sess.frame_trace()))
    sess.timing = False
    total_ms = sum(times)
    fps = per_step * args.steps / (total_ms / 1000.0)
    samples_all = parallel.sum_over_ranks(ctx, samples)

    # ---- e2e through the public API (host image out), continuing the orbit
    e2e = None
    if not args.no_e2e:
        import gc

        _ = None  # drop the warm-up frame; the loop holds one frame while rendering the next
        sess.reserve_host_frames(2)

        gc.collect()
        gc.disable()  # no collector pauses inside the timed public-API frames
        walls = []
        for i in range(args.steps):
            f = args.warmup + args.steps + i
            flush.zero_()
            torch.cuda.synchronize()
            parallel.barrier(ctx)
            sess.set_camera(cam(f))
            t0 = time.perf_counter()
            if ctx.world == 1 or afr:
                img_h, rec = sess.render_frame()  # AFR: every rank returns its whole frame to its host
            else:
                img = sess.render_frame_device()
                full = gather(img)
                img_h = full.cpu().numpy() if ctx.rank == 0 else None
                rec = sess.collect_record(t0)
            walls.append(parallel.max_over_ranks(ctx, (time.perf_counter() - t0) * 1000.0))
        gc.enable()
        if verbose:
            print("e2e walls ms:", [round(x, 2) for x in walls], file=sys.stderr)
        h2d = len(bytes(N.VcbFrameParams())) + len(bytes(N.VcbMaintParams()))
        e2e = {"value": per_step * args.steps / (sum(walls) / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "median_ms": statistics.median(walls), "max_ms": max(walls),
               "d2h_bytes_per_step": args.res * args.res * 16 + 256,
               "note": "RenderSession.render_frame(): camera/params by value, image f32[H,W,4] copied to host"}

    # ---- CPU baseline (rank 0, N=1): the oracle renders the first timed frame's successor
    cpu = None
    if ctx.world == 1 and not args.no_cpu_baseline:
        try:
            state = sess.export_state()
            frac = args.cpu_frac
            wall, oimg, orec = cpu_oracle_frame_from_state(state, (mg.value_min, mg.value_max), frac, sess.frame,
                                                            args.volume, args.cpu_frames)
            cores = os.cpu_count() or 1
            cpu = {"value": (frac * frac) / wall, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": (f"{args.cpu_frames} frames (orbit frames {sess.frame}..{sess.frame + args.cpu_frames - 1}) "
                              f"rendered by the oracle port (C+numpy restatement of voxcache, OpenMP {cores} threads), "
                              f"resumed from the GPU session's exact cache/request/loader state, at "
                              f"{int(args.res * frac)}^2; mean render+maintenance {wall:.2f}s/frame"
                              + (f", fps scaled by the pixel ratio {frac * frac:.4f}" if frac != 1.0 else ""))}
        except Exception as exc:  # the baseline is reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}

    # ---- the paper's comparison: the same frames without the brick cache (every
    # sample inferred through the INR, session.py:63-70), device-timed like `value`
    uncached = None
    if ctx.world == 1 and args.uncached_steps > 0:
        ucfg = SessionConfig(cached=False, loader="inline", cache=cfg.cache, scheduler=cfg.scheduler,
                             policy=cfg.policy, settings=cfg.settings, seed=0)
        usess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), ucfg, macro=mg)
        usess.impl = args.schedule
        ust = usess.stream
        uts, usamp = [], 0
        for i in range(args.uncached_steps + 1):
            f = args.warmup + i
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ust)
            usess.set_camera(traj.camera_at(f))
            t0 = time.perf_counter()
            usess.render_frame_device()
            e1.record(ust)
            urec = usess.collect_record(t0)
            torch.cuda.synchronize()
            if i > 0:  # the first frame is warm-up
                uts.append(e0.elapsed_time(e1))
                usamp += urec.samples
        ufps = len(uts) / (sum(uts) / 1000.0)
        uncached = {"fps": ufps, "cache_speedup": fps / ufps, "frames": len(uts),
                    "inr_samples_per_s": usamp / (sum(uts) / 1000.0),
                    "note": "same orbit frames rendered with SessionConfig(cached=False): every sample decoded "
                            "through the INR inside the frame kernel (true-miss path)"}
        del usess

    # ---- the paper's second FPS column: the path tracer (render/pathtrace.py) on the same
    # model, orbit and cache configuration, cached and uncached, device-timed like `value`
    pathtrace = None
    if ctx.world == 1 and args.pt_steps > 0:
        pathtrace = {"spp": 1, "note": "SessionConfig(mode='pathtrace', samples_per_pixel=1): delta-tracked primary "
                                       "walk + one shadow ray per hit, numpy-PCG64-exact draws, same sampler/cache"}
        for label, cached in (("cached", True), ("uncached", False)):
            pcfg = SessionConfig(cached=cached, mode="pathtrace", samples_per_pixel=1, loader="inline",
                                 cache=cfg.cache, scheduler=cfg.scheduler, policy=cfg.policy, settings=cfg.settings,
                                 seed=0)
            psess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), pcfg, macro=mg)
            pst = psess.stream
            pts, psamp, piters = [], 0, 0
            for i in range(args.warmup + args.pt_steps):
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(pst)
                psess.set_camera(traj.camera_at(args.warmup + i))
                t0 = time.perf_counter()
                psess.render_frame_device()
                e1.record(pst)
                prec = psess.collect_record(t0)
                torch.cuda.synchronize()
                if i >= args.warmup:
                    pts.append(e0.elapsed_time(e1))
                    psamp += prec.samples
                    piters += psess.last_frame_stats.get("iterations", 0)
            pathtrace[label] = {"fps": len(pts) / (sum(pts) / 1000.0), "ms_per_frame": statistics.mean(pts),
                                "samples_per_frame": psamp / len(pts), "walk_iterations_per_frame": piters / len(pts),
                                "frames": len(pts)}
            del psess
        pathtrace["cache_speedup"] = pathtrace["cached"]["fps"] / pathtrace["uncached"]["fps"]

    # ---- INR training (inr/train.py): Adam steps at the reference's
    # default batch on a 64^3 lattice target, device-timed
    training = None
    if ctx.world == 1 and args.train_steps > 0:
        from paper_2504_18001_b200.train import psnr_on_lattice, train

        lat = np.random.default_rng(9).random((64, 64, 64)).astype(np.float32)
        tfield = P.RawLatticeField(lat, P.FieldDomain((64, 64, 64)))
        tmodel = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((64, 64, 64)), seed=0)
        train(tmodel, tfield, steps=3, seed=1)  # warm-up (module load, allocations)
        tmodel = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((64, 64, 64)), seed=0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tres = train(tmodel, tfield, steps=args.train_steps, seed=2)
        e1.record()
        torch.cuda.synchronize()
        tms = e0.elapsed_time(e1) / args.train_steps
        training = {"ms_per_step": tms, "batch": 65536, "samples_per_s": 65536 / (tms / 1000.0),
                    "steps": args.train_steps, "loss_first_last": [float(tres.loss_trace[0]), tres.final_loss],
                    "note": "train(model, field, steps, batch_size=65536, adam lr 1e-2): PCG64 batch, target decode, "
                            "fused forward/backward + f64 scatter-add, Adam; timed on the current stream incl. the "
                            "host round trip of the loss trace"}

    decode = None
    if ctx.rank == 0 and args.decode_n > 0:
        try:
            sys.path.insert(0, str(ROOT / "tools"))
            import decode_bench

            decode = decode_bench.run(args.decode_n, reps=3)
        except Exception as exc:
            decode = {"error": str(exc)}
    peak, peak_src = measured_peak_hbm()
    achieved = (samples_all * BYTES_PER_SAMPLE) / (march_ms / 1000.0) / 1e9 if march_ms > 0 else None
    if ctx.rank == 0:
        last = recs[-1]
        line = {
            "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if afr else "strong", "vs_baseline": None, "dtype": "f64 addressing + f32 samples",
            "data": "synthetic (random-init INR weights, procedural orbit)",
            "config": {**workload(args.res, args.volume),
                       "parallelism": (f"alternate-frame rendering x{ctx.world} (private cache per GPU, NCCL frame gather)"
                                       if afr else f"sort-first bands x{ctx.world}" + (", fused peer-write gather" if fused else "")),
                       "macro": msrc},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": profiled_traffic(),
                         "kernel": "k_wave3_march (persistent cooperative, one grid barrier per iteration: rank+probe+shade+next advance; queued miss inference)",
                         "algorithmic_bytes": f"{BYTES_PER_SAMPLE} B/sample x samples per launch",
                         "launches": march_launches, "avg_launch_us": 1000.0 * march_ms / max(march_launches, 1),
                         "march_share_of_step": (march_ms / ctx.world) / total_ms if total_ms else None,
                         "peak_source": peak_src},
            "cpu_baseline": cpu, "e2e": e2e, "inr_decode": decode, "uncached_inr_baseline": uncached,
            "pathtrace": pathtrace, "inr_training": training,
            "clocks": clk.summary(), "gpu_launches": launches,
            "samples_per_frame": samples_all / (args.steps * per_step),
            "inr_samples_per_frame": float(np.mean([r.true_misses for r in recs])) + 40 * 16 ** 3,
            "hit_rate": 1.0 - sum(r.true_misses for r in recs) / max(1, sum(r.samples for r in recs)),
            "last_record": {k: getattr(last, k) for k in ("frame", "samples", "true_misses", "fallback_hits",
                                                          "exact_hits", "occupancy", "bricks_loaded_total")},
        }
        if t_macro is not None:
            line["macro_build_s"] = t_macro
        print(json.dumps(line), flush=True)
    parallel.shutdown(ctx)


if __name__ == "__main__":
    main()
