#!/usr/bin/env python
"""Headline benchmark: cached-INR ray-march frames/s at 1024^2 (BASELINE.json config 2).

Workload (configs[1]): 512^3 volume decoded from the random-init hash-grid INR
(HashGridConfig()/MLPConfig(), seed 0, parameters re-drawn uniform(-0.7,0.7) from
default_rng(42)), 16^3 bricks, 32^3-slot pool (537 MB), 1024x1024 frames on the
orbit (center .5, radius 2.2, 120 frames/rev, 20 deg elevation, fov 45),
warm_body(0.5, 0.9), LodPolicy(1.2, preload 20), 40 requests/frame, inline
loader (deterministic), seed 0.  A step = one RenderSession.render_frame()
(render + maintenance), the reference's fps definition (session.py:107-113).

Steady state (PAPER.md:278 measures "after the effects of pre-loading have
disappeared"): the session is pre-rolled --preroll frames along the orbit
(default 200, i.e. 1.7 revolutions, far past the 20-frame preload ramp), then W
warm-up and K timed frames follow.  The same K frames from a cold start (frames
W..W+K-1, inside the preload ramp) are reported as `ramp_window`.

  value : frames/s, device-resident (render + maintenance + stats readback), CUDA
          events on the session stream, L2 flushed (256 MB write) between frames
  e2e   : W untimed, then K timed frames through the public API render_frame(),
          which returns the host image (the 16 MB image crosses PCIe inside the
          timed region: the frame kernels store it into mapped pinned memory)
  parity: the CPU oracle resumes the GPU session's exact state and renders the
          next frames; image, FrameRecord counters and post-maintenance cache
          state (tables, owners, stamps, requests, batch) are compared
  cpu_baseline : those oracle frames' wall time (all host threads)

Frame kernel (`--march`): "throughput" (default) marches one
persistent ray per GPU lane, the stochastic-LoD RNG lane being the film pixel;
"parity" is the wavefront that numbers RNG lanes by sample rank exactly as the
reference (sampler.py:206-213).  The other schedule is measured on the same
frames as `other_schedule`.  The oracle restates whichever lane rule is benched.

Multi-GPU (torchrun, N>1): sort-first tiles by default — rank r renders film rows
r, r+N, ... of every frame with a private cache and the RGBA8 bands are gathered
to rank 0 with NCCL on a comm stream that overlaps the next frame (scaling
"strong"); `--mp frames` is alternate-frame rendering instead.

`--impl reference` times the CPU oracle port alone (the reference has no GPU
path) on a bounded sample of the same workload; see its `cpu_baseline.sample`.
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
KERNEL = {"throughput": "k_ray_march (persistent, one ray per lane, pixel RNG lanes; + k_ray_setup)",
          "parity": "k_wave3_march (persistent cooperative wavefront, one grid barrier per iteration, rank RNG lanes)"}


def workload(res=1024, volume=512, pool=32, preroll=200):
    return dict(workload="config2_cached_inr_raymarch", volume=f"{volume}^3 random-init INR (8x2 hash grid, 16-32-32-1)",
                image=f"{res}x{res}", brick=16, pool_slots=pool ** 3, orbit="r=2.2, 120 frames/rev, elev 20, fov 45",
                tf="warm_body(0.5,0.9)", lod_policy="scale 1.2, preload 20, corrected", max_requests=40,
                loader="inline", steady_state=f"timed after a {preroll}-frame pre-roll (PAPER.md:278)",
                l2="flushed (256 MB write) between timed frames")


def make_model(volume):
    import paper_2504_18001_b200 as P

    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((volume,) * 3), seed=0)
    r = np.random.default_rng(42)
    m.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in m.parameters()])
    return m


def load_bench_macro(volume):
    """The oracle-built macro grid (oracle/make_bench_macro.py) — the reference arm's
    input, and the GPU build's parity check."""
    f = ROOT / "bench_data" / f"macro_inr{volume}_c16.npz"
    if f.exists():
        d = np.load(f)
        return d["vmin"], d["vmax"]
    return None, None


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


def profiled_traffic(march):
    f = ROOT / "profiles" / f"ncu_frame_kernel_{march}.json"
    if f.exists():
        try:
            return json.loads(f.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def oracle_session(volume, macro, rng):
    from oracle import cinr_oracle as O

    t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
    fld = O.InrFieldOracle((volume,) * 3, t, w, b, O.DEFAULT_GRID)
    cfg = O.Config(dims=(volume,) * 3, brick=16, pool=(32,) * 3, max_requests=40, lod_scale=1.2, preload=20,
                   seed=0, rng=rng)
    return O.OracleSession(fld, O.warm_body_points(0.5, 0.9), cfg, macro_minmax_arrays=macro)


# --------------------------------------------------------------------------- reference arm
def run_reference_arm(args):
    """`--impl reference`: the CPU oracle port (the reference has no GPU path) on all
    host threads, with the reference's own RNG lanes.  Steady state as the GPU arm:
    the orbit is pre-rolled (at --ref-preroll-res to stay within minutes; the bricks a
    frame requests depend on distance, not on resolution, so the cache reaches the
    same kind of steady state), then W warm-up and at most --ref-max-steps timed
    frames at full resolution."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cinr_oracle as O

    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    vmin, vmax = load_bench_macro(args.volume)
    if vmin is None:
        t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
        fld = O.InrFieldOracle((args.volume,) * 3, t, w, b, O.DEFAULT_GRID)
        vmin, vmax = O.macro_minmax_streamed(fld, (args.volume,) * 3, 16)
    sess = oracle_session(args.volume, (vmin, vmax), "rank")
    pre_res = args.ref_preroll_res
    t0 = time.perf_counter()
    for f in range(args.preroll):
        sess.set_camera(O.orbit_camera((0.5, 0.5, 0.5), 2.2, 120, f), (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0,
                        pre_res, pre_res)
        sess.render_frame()
    t_pre = time.perf_counter() - t0
    timed = max(1, min(args.steps, args.ref_max_steps))
    walls = []
    for i in range(args.warmup + timed):
        f = args.preroll + i
        sess.set_camera(O.orbit_camera((0.5, 0.5, 0.5), 2.2, 120, f), (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0,
                        args.res, args.res)
        img, rec = sess.render_frame()
        if i >= args.warmup:
            walls.append(rec.wall_s)
    fps = len(walls) / sum(walls)
    f0 = args.preroll + args.warmup
    sample = (f"oracle port (C+numpy restatement of voxcache, OpenMP {cores} threads, the reference's rank RNG lanes): "
              f"orbit frames {f0}..{f0 + timed - 1} at {args.res}^2 after a {args.preroll}-frame pre-roll at "
              f"{pre_res}^2 ({t_pre:.0f} s) and {args.warmup} warm-up frames; render + maintenance wall time per frame")
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus, "steps": timed,
            "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / fps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 addressing + f32 samples",
            "data": "synthetic (random-init INR weights, procedural orbit)",
            "config": workload(args.res, args.volume, preroll=args.preroll), "impl": "reference",
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm helpers
def session_config(P, SessionConfig, pool=32, preload=20, cached=True, mode="raymarch"):
    return SessionConfig(cached=cached, mode=mode, samples_per_pixel=1, loader="inline",
                         cache=P.CacheConfig(brick_size=16, pool_dims=(pool,) * 3),
                         scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, preload),
                         settings=P.RenderSettings(), seed=0)


def device_frames(sess, cam, frames, flush, st, timing=False, gather=None, ctx=None):
    """Render `frames` (orbit indices) device-resident; per-frame CUDA-event ms on the
    session stream (max over ranks), records, march-kernel ms and launch counts."""
    import torch

    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200 import parallel

    sess.timing = timing
    out = dict(ms=[], recs=[], march_ms=0.0, march_launches=0, launches=0)
    for f in frames:
        flush.zero_()
        torch.cuda.synchronize()
        if ctx is not None:
            parallel.barrier(ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c = cam(f)  # the trajectory's camera object (harness work, outside the step)
        e0.record(st)
        sess.set_camera(c)
        t0 = time.perf_counter()
        img = sess.render_frame_device()
        if gather is not None:
            gather(img)
        e1.record(st)
        rec = sess.collect_record(t0)
        out["launches"] += N.load().vcb_last_launch_count()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out["ms"].append(parallel.max_over_ranks(ctx, ms) if ctx is not None else ms)
        out["recs"].append(rec)
        if timing:
            km, kn = sess.march_kernel_time()
            out["march_ms"] += km
            out["march_launches"] += kn
    sess.timing = False
    return out


def preroll(sess, cam, n, start=0):
    for f in range(start, start + n):
        sess.set_camera(cam(f))
        t0 = time.perf_counter()
        sess.render_frame_device()
        sess.collect_record(t0)


def roofline(samples, march_ms, launches, peak, peak_src, march, share=None, profile=None):
    """`profile`: the ncu capture whose DRAM bytes are this kernel's `traffic`
    (profiles/ncu_frame_kernel_<profile>.json; default <march>, the config-2 captures;
    None-valued for workloads without a capture)."""
    achieved = samples * BYTES_PER_SAMPLE / (march_ms / 1000.0) / 1e9 if march_ms > 0 else None
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None,
            "traffic": profiled_traffic(profile if profile is not None else march),
            "kernel": KERNEL.get(march, march),
            "algorithmic_bytes": f"{BYTES_PER_SAMPLE} B/sample x {samples / max(launches, 1):.0f} samples per launch",
            "launches": launches, "avg_launch_us": 1000.0 * march_ms / max(launches, 1), "march_share_of_step": share,
            "peak_source": peak_src}


def state_of(sess):
    d = sess.cache.dump()
    d["batch"] = sess.cache.batch()
    return d


def oracle_state(osess):
    c = osess.cache
    ents = sorted((k[0], k[1], v[0], v[1]) for k, v in osess.req.entries.items())
    return dict(tables=c.table, owner=c.owner, last_used=c.last_used,
                entries=np.array(ents, dtype=np.int64).reshape(-1, 4),
                batch=np.array(osess.last_batch, dtype=np.int64).reshape(-1, 2))


def parity_leg(sess, macro, args, march, traj):
    """The oracle resumes the GPU session's exact state (tables, pool, owners, stamps,
    requests, staged batch) and renders the next --cpu-frames frames with the lane rule
    of the benched schedule; the GPU renders the same frames.  Returns (parity, cpu)."""
    from oracle import cinr_oracle as O

    cores = os.cpu_count() or 1
    state = sess.export_state()
    f0 = int(state["session_frame"])
    osess = oracle_session(args.volume, macro, "pixel" if march == "throughput" else "rank")
    O.load_session_state(osess, state)
    res = {"frames": [], "tolerance": "image <= 1e-3 abs and >= 60 dB PSNR (decoded INR values, P14); FrameRecord "
                                      "counters and post-maintenance cache state bit-exact",
           "oracle_rng_lanes": "pixel" if march == "throughput" else "rank (the reference's)"}
    walls = []
    ok = True
    for i in range(args.cpu_frames):
        f = f0 + i
        c = traj.camera_at(f)
        sess.set_camera(c)
        img, rec = sess.render_frame()
        gs = state_of(sess)
        osess.set_camera(c.position, (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0, args.res, args.res)
        oimg, orec = osess.render_frame()
        walls.append(orec.wall_s)
        os_ = oracle_state(osess)
        diff = float(np.abs(img - oimg).max())
        mse = float(np.mean((img[..., :3].astype(np.float64) - oimg[..., :3]) ** 2))
        psnr = float(10 * np.log10(1.0 / mse)) if mse > 0 else float("inf")
        rec_eq = (rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits, rec.bricks_loaded) == \
                 (orec.samples, orec.true_misses, orec.fallback_hits, orec.exact_hits, orec.bricks_loaded)
        st_eq = {k: bool(np.array_equal(np.asarray(gs[k]), np.asarray(os_[k])))
                 for k in ("tables", "owner", "last_used", "entries", "batch")}
        fr_ok = diff <= 1e-3 and psnr >= 60.0 and rec_eq and all(st_eq.values())
        ok = ok and fr_ok
        res["frames"].append({"frame": f, "image_max_abs": diff, "psnr_db": psnr if np.isfinite(psnr) else "inf",
                              "record_equal": rec_eq, "state_equal": st_eq, "samples": rec.samples,
                              "true_misses": rec.true_misses})
    res["pass"] = ok
    wall = float(np.mean(walls))
    cpu = {"value": 1.0 / wall, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": (f"{args.cpu_frames} steady-state frames (orbit frames {f0}..{f0 + args.cpu_frames - 1}) at "
                      f"{args.res}^2 rendered by the oracle port (C+numpy restatement of voxcache, OpenMP {cores} "
                      f"threads) resumed from the GPU session's exact state; mean render+maintenance "
                      f"{wall:.2f} s/frame")}
    return res, cpu


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--volume", type=int, default=512)
    ap.add_argument("--preroll", type=int, default=200, help="orbit frames rendered before warm-up (steady state)")
    ap.add_argument("--march", default="throughput", choices=["throughput", "parity"])
    ap.add_argument("--schedule", type=int, default=None, help="override VcbFrameParams.impl (A/B of variants)")
    ap.add_argument("--ref-preroll-res", type=int, default=128, help="reference arm: pre-roll resolution")
    ap.add_argument("--ref-max-steps", type=int, default=8, help="reference arm: at most this many timed frames")
    ap.add_argument("--cpu-frames", type=int, default=4, help="oracle parity/baseline frames (from the GPU state)")
    ap.add_argument("--decode-n", type=int, default=1 << 24, help="isolated INR decode batch (0 = skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ramp", action="store_true", help="skip the cold-start (preload ramp) window")
    ap.add_argument("--no-other", action="store_true", help="skip the other march schedule")
    ap.add_argument("--config3-steps", type=int, default=10, help="config 3 (4096^3 virtual) timed frames (0 = skip)")
    ap.add_argument("--config3-preroll", type=int, default=60)
    ap.add_argument("--config5-steps", type=int, default=5, help="config 5 at N=1 (4096^3, 4K) frames (0 = skip)")
    ap.add_argument("--config5-preroll", type=int, default=20)
    ap.add_argument("--config1", type=int, default=1, help="config 1 (64^3, 256^2, 120-frame orbit) side result")
    ap.add_argument("--config4-frames", type=int, default=40, help="config 4 (2048^3, 1080p) frames (0 = skip)")
    ap.add_argument("--uncached-steps", type=int, default=5, help="frames of the no-cache INR baseline (0 = skip)")
    ap.add_argument("--scheduler-frames", type=int, default=8, help="frame-scheduler cold-start frames (0 = skip)")
    ap.add_argument("--budget", type=int, default=1 << 20, help="decode budget (samples/frame) of that comparison")
    ap.add_argument("--train-steps", type=int, default=50,
                    help="INR training steps at batch 65536 (inr/train.py on the GPU; 0 = skip)")
    ap.add_argument("--pt-steps", type=int, default=5,
                    help="frames of the path-trace mode (pathtrace.py, spp 1) cached and uncached (0 = skip)")
    ap.add_argument("--mp", default="tiles", choices=["tiles", "frames"],
                    help="N>1: 'tiles' = sort-first film-row bands of every frame, RGBA8 bands gathered to rank 0 "
                         "(strong scaling, default); 'frames' = alternate-frame rendering (weak scaling)")
    ap.add_argument("--share-decode", action="store_true",
                    help="N>1: decode each distinct requested brick once, on its owner rank, and all-gather "
                         "(RenderSession.share_decode; the cache state is unchanged)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch

    from paper_2504_18001_b200 import macrocell, parallel
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import SessionConfig

    import paper_2504_18001_b200 as P

    ctx = parallel.init_from_env()
    dev = torch.device("cuda", ctx.local_rank)
    torch.cuda.set_device(dev)
    model = make_model(args.volume)
    fld = model.as_field()
    # macro grid: built on the GPU from the field lattice (vcb_macro_minmax), timed
    # separately and checked against the oracle-built grid the reference arm uses
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mg = macrocell.build(fld, (args.volume,) * 3, 16, dev)
    torch.cuda.synchronize()
    macro_ms = (time.perf_counter() - t0) * 1000.0
    ovmin, ovmax = load_bench_macro(args.volume)
    macro_info = {"build_ms": macro_ms, "cells": int(np.prod(mg.grid_dims)), "source": "GPU (vcb_macro_minmax)"}
    if ovmin is not None:
        macro_info["max_abs_diff_vs_oracle_grid"] = float(max(np.abs(mg.value_min - ovmin).max(),
                                                              np.abs(mg.value_max - ovmax).max()))
    macro_np = (np.asarray(mg.value_min), np.asarray(mg.value_max))

    cfg = session_config(P, SessionConfig)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=args.res, height=args.res)
    afr = ctx.world > 1 and args.mp == "frames"
    sess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, bands=not afr)
    sess.march = args.march
    if args.schedule is not None:
        sess.impl = args.schedule
    if args.share_decode and ctx.world > 1:
        sess.share_decode(ctx)
    per_step = ctx.world if afr else 1  # 1024^2 frames completed per step, whole job

    def cam(f):
        # alternate-frame rendering: rank r renders orbit frames r, r + N, r + 2N, ...
        return traj.camera_at(f * ctx.world + ctx.rank if afr else f)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = sess.stream
    gatherer = parallel.FrameGather(ctx, sess, args.res, args.res, frames=afr) if ctx.world > 1 else None
    gather = gatherer.submit if gatherer is not None else None

    # ---- pre-roll to the steady state, then warm-up (untimed)
    preroll(sess, cam, args.preroll)
    for f in range(args.preroll, args.preroll + args.warmup):
        if ctx.world == 1 and f >= args.preroll + args.warmup - 2:
            sess.set_camera(cam(f))
            sess.render_frame()  # the last warm-up frames go through the public call (pins its host buffers)
        else:
            device_frames(sess, cam, [f], flush, st, gather=gather, ctx=ctx)
    torch.cuda.synchronize()

    # ---- timed: device-resident frames
    f_timed = args.preroll + args.warmup
    with ClockSampler(ctx.local_rank) as clk:
        t = device_frames(sess, cam, range(f_timed, f_timed + args.steps), flush, st, timing=True, gather=gather,
                          ctx=ctx)
    total_ms = sum(t["ms"])
    fps = per_step * args.steps / (total_ms / 1000.0)
    samples = sum(r.samples for r in t["recs"])
    samples_all = parallel.sum_over_ranks(ctx, samples)
    march_all = parallel.sum_over_ranks(ctx, t["march_ms"])
    launches_all = int(parallel.sum_over_ranks(ctx, t["march_launches"]))

    # ---- e2e through the public API (host image out), continuing the orbit
    e2e = None
    f_e2e = f_timed + args.steps
    if not args.no_e2e:
        import gc

        sess.reserve_host_frames(2)
        gc.collect()
        gc.disable()  # no collector pauses inside the timed public-API frames
        walls = []
        # W untimed public-API frames first (first-call setup: pinned frames, side stream)
        for i in range(-args.warmup, args.steps):
            f = f_e2e + args.warmup + i
            flush.zero_()
            torch.cuda.synchronize()
            parallel.barrier(ctx)
            sess.set_camera(cam(f))
            t0 = time.perf_counter()
            if ctx.world == 1 or afr:
                img_h, rec = sess.render_frame()  # AFR: every rank returns its whole frame to its host
            else:
                img = sess.render_frame_device()
                gatherer.submit(img)
                rec = sess.collect_record(t0)
                img_h = gatherer.host_frame() if ctx.rank == 0 else None
            wall = parallel.max_over_ranks(ctx, (time.perf_counter() - t0) * 1000.0)
            if i >= 0:
                walls.append(wall)
        gc.enable()
        h2d = len(bytes(P._native.VcbFrameParams())) + len(bytes(P._native.VcbMaintParams()))
        d2h = args.res * args.res * (16 if ctx.world == 1 or afr else 4) + 256
        e2e = {"value": per_step * args.steps / (sum(walls) / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "median_ms": statistics.median(walls), "max_ms": max(walls), "d2h_bytes_per_step": d2h,
               "note": ("RenderSession.render_frame(): camera/params by value, image f32[H,W,4] stored into mapped pinned host "
                         "memory by the frame kernels (box-hit pixels by the march's lanes, background by a side-stream "
                         "kernel)"
                        if ctx.world == 1 or afr else
                        "render_frame_device + RGBA8 band gather to rank 0 + one RGBA8 frame D2H on rank 0")}

    # ---- parity at the benched size + CPU baseline (rank 0, N=1)
    parity, cpu = None, None
    if ctx.world == 1 and not args.no_cpu_baseline:
        try:
            parity, cpu = parity_leg(sess, macro_np, args, args.march, traj)
        except Exception as exc:  # reported, never fatal
            import traceback

            traceback.print_exc()
            parity = {"error": str(exc)}
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    last = t["recs"][-1]
    del sess
    torch.cuda.empty_cache()

    peak, peak_src = measured_peak_hbm()
    side = {}
    if ctx.world == 1:
        # ---- the other march schedule on the same steady-state frames
        if not args.no_other:
            other = "parity" if args.march == "throughput" else "throughput"
            s2 = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
            s2.march = other
            preroll(s2, cam, args.preroll + args.warmup)
            o = device_frames(s2, cam, range(f_timed, f_timed + args.steps), flush, s2.stream, timing=True)
            osamp = sum(r.samples for r in o["recs"])
            side["other_schedule"] = {"march": other, "fps": len(o["ms"]) / (sum(o["ms"]) / 1000.0),
                                      "samples_per_frame": osamp / len(o["ms"]),
                                      "roofline": roofline(osamp, o["march_ms"], o["march_launches"], peak, peak_src,
                                                           other, o["march_ms"] / sum(o["ms"]))}
            del s2
        # ---- the same K frames from a cold start (inside the 20-frame preload ramp)
        if not args.no_ramp:
            s3 = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
            s3.march = args.march
            preroll(s3, cam, args.warmup)
            o = device_frames(s3, cam, range(args.warmup, args.warmup + args.steps), flush, s3.stream)
            lr = o["recs"][-1]
            side["ramp_window"] = {"fps": len(o["ms"]) / (sum(o["ms"]) / 1000.0),
                                   "frames": f"{args.warmup}..{args.warmup + args.steps - 1} from a cold cache",
                                   "last_occupancy": lr.occupancy, "last_fallback_hits": lr.fallback_hits,
                                   "last_samples": lr.samples}
            del s3
        torch.cuda.empty_cache()
        # ---- frame scheduler: cold-start frames with and without a decode budget, and the
        # overlapped (loader="thread") decode at steady state
        if args.scheduler_frames > 0:
            side["frame_scheduler"] = run_frame_scheduler(P, SessionConfig, parallel, ctx, fld, mg, traj, cam, args,
                                                          flush, f_timed)
            torch.cuda.empty_cache()
        # ---- config 3: 4096^3 virtual volume at 1024^2 (B=16, 10 LoD levels), steady state
        if args.config3_steps > 0:
            try:
                side["config3"] = run_config3(P, SessionConfig, OrbitTrajectory, macrocell, args, flush, dev, peak,
                                              peak_src)
            except Exception as exc:
                import traceback

                traceback.print_exc()
                side["config3"] = {"error": str(exc)}
            torch.cuda.empty_cache()
        # ---- configs 1 and 4 at their stated sizes
        if args.config1:
            side["config1"] = run_config1(P, SessionConfig, OrbitTrajectory, args, flush, dev)
        if args.config4_frames > 0:
            side["config4"] = run_config4(P, SessionConfig, OrbitTrajectory, macrocell, args, flush, dev)
            torch.cuda.empty_cache()
        # ---- the paper's comparison: no brick cache (every sample through the INR)
        if args.uncached_steps > 0:
            ucfg = session_config(P, SessionConfig, cached=False)
            us = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), ucfg, macro=mg)
            us.march = args.march
            preroll(us, cam, 1, start=f_timed - 1)
            o = device_frames(us, cam, range(f_timed, f_timed + args.uncached_steps), flush, us.stream)
            ufps = len(o["ms"]) / (sum(o["ms"]) / 1000.0)
            usamp = sum(r.samples for r in o["recs"])
            side["uncached_inr_baseline"] = {
                "fps": ufps, "cache_speedup": fps / ufps, "frames": len(o["ms"]),
                "inr_samples_per_s": usamp / (sum(o["ms"]) / 1000.0),
                "note": "the timed orbit frames with SessionConfig(cached=False): every sample decoded through the "
                        "INR inside the frame kernel (true-miss path), same march schedule"}
            del us
        # ---- the paper's second FPS column: the path tracer, cached and uncached
        if args.pt_steps > 0:
            pt = {"spp": 1, "note": "SessionConfig(mode='pathtrace', samples_per_pixel=1): delta-tracked primary "
                                    "walk + one shadow ray per hit, numpy-PCG64-exact draws, same sampler/cache; "
                                    "frames W..W+k-1 from a cold cache"}
            for label, cached in (("cached", True), ("uncached", False)):
                pcfg = session_config(P, SessionConfig, cached=cached, mode="pathtrace")
                ps = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), pcfg, macro=mg)
                preroll(ps, traj.camera_at, args.warmup)
                o = device_frames(ps, traj.camera_at, range(args.warmup, args.warmup + args.pt_steps), flush,
                                  ps.stream)
                pt[label] = {"fps": len(o["ms"]) / (sum(o["ms"]) / 1000.0), "ms_per_frame": statistics.mean(o["ms"]),
                             "samples_per_frame": sum(r.samples for r in o["recs"]) / len(o["ms"]),
                             "frames": len(o["ms"])}
                del ps
            pt["cache_speedup"] = pt["cached"]["fps"] / pt["uncached"]["fps"]
            side["pathtrace"] = pt
        # ---- INR training (inr/train.py)
        if args.train_steps > 0:
            from paper_2504_18001_b200.train import train

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
            side["inr_training"] = {"ms_per_step": tms, "batch": 65536, "samples_per_s": 65536 / (tms / 1000.0),
                                    "steps": args.train_steps,
                                    "loss_first_last": [float(tres.loss_trace[0]), tres.final_loss],
                                    "note": "train(model, field, steps, batch_size=65536, adam lr 1e-2), timed on the "
                                            "current stream incl. the host round trip of the loss trace"}
    if ctx.rank == 0 and args.decode_n > 0:
        try:
            sys.path.insert(0, str(ROOT / "tools"))
            import decode_bench

            side["inr_decode"] = decode_bench.run(args.decode_n, reps=3)
        except Exception as exc:
            side["inr_decode"] = {"error": str(exc)}

    launches_total = int(parallel.sum_over_ranks(ctx, t["launches"]))  # a collective: every rank
    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if afr else "strong", "vs_baseline": None, "dtype": "f64 addressing + f32 samples",
            "data": "synthetic (random-init INR weights, procedural orbit)",
            "config": workload(args.res, args.volume, preroll=args.preroll),
            "march": args.march if args.schedule is None else f"impl {args.schedule}",
            "parallelism": (f"alternate-frame rendering x{ctx.world} (private cache per GPU, NCCL frame gather)" if afr
                            else f"sort-first film-row bands x{ctx.world} (private cache per GPU, RGBA8 bands "
                                 f"gathered to rank 0 over NCCL on a comm stream"
                                 f"{'; brick decodes shared across ranks' if args.share_decode else ''})"
                            if ctx.world > 1 else "single GPU"),
            "roofline": roofline(samples_all, march_all, launches_all, peak, peak_src, args.march,
                                 (march_all / ctx.world) / total_ms if total_ms else None),
            "cpu_baseline": cpu, "e2e": e2e, "parity": parity, "macro_grid": macro_info,
            "clocks": clk.summary(), "gpu_launches": launches_total,
            "samples_per_frame": samples_all / (args.steps * per_step),
            "hit_rate": 1.0 - sum(r.true_misses for r in t["recs"]) / max(1, samples),
            "last_record": {k: getattr(last, k) for k in ("frame", "samples", "true_misses", "fallback_hits",
                                                          "exact_hits", "occupancy", "bricks_loaded_total")},
            **side,
        }
        print(json.dumps(line), flush=True)
    if gatherer is not None:
        gatherer.close()
    parallel.shutdown(ctx)


def run_frame_scheduler(P, SessionConfig, parallel, ctx, fld, mg, traj, cam, args, flush, f_timed):
    """The first frames of a cold session (every sample a true miss until the coarsest
    brick lands at frame 2, P19) unbounded vs with SchedulerConfig(decode_budget), and
    steady-state fps with loader='thread' (batch decoded on a side stream)."""
    import dataclasses

    out = {"budget_samples_per_frame": args.budget}
    for label, budget in (("unbounded", None), ("budgeted", args.budget)):
        cfg = session_config(P, SessionConfig)
        cfg = dataclasses.replace(cfg, scheduler=dataclasses.replace(cfg.scheduler, decode_budget=budget))
        s = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
        s.march = args.march
        o = device_frames(s, cam, range(args.scheduler_frames), flush, s.stream)
        st = [dict(ms=round(ms, 3), true_misses=r.true_misses) for ms, r in zip(o["ms"], o["recs"])]
        out[label] = {"max_ms": max(o["ms"]), "mean_ms": statistics.mean(o["ms"]), "frames": st}
        del s
    cfg = dataclasses.replace(session_config(P, SessionConfig), loader="thread")
    s = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
    s.march = args.march
    preroll(s, cam, args.preroll + args.warmup)
    o = device_frames(s, cam, range(f_timed, f_timed + args.steps), flush, s.stream)
    out["thread_loader_steady_fps"] = len(o["ms"]) / (sum(o["ms"]) / 1000.0)
    out["note"] = ("budgeted: true misses beyond the budget are filed but not composited, the brick batch gets what "
                   "the misses left (>= 1 brick); thread loader: the batch decodes on a decode stream during the next "
                   "frame's march (state identical to inline)")
    del s
    return out


def run_config3(P, SessionConfig, OrbitTrajectory, macrocell, args, flush, dev, peak, peak_src):
    """BASELINE config 3: 4096^3 virtual volume (the same random-init INR over a 4096^3
    domain), B=16 -> 10 LoD levels (19.4 M bricks), 64^3-slot pool (4.3 GB), 1024^2,
    max_requests 40 (= a decode budget of 163,840 samples per frame plus true misses).
    The macro grid (256^3 cells) is decoded from the field on the GPU."""
    import torch

    from paper_2504_18001_b200.session import RenderSession

    dims = (4096,) * 3
    fld = make_model(4096).as_field()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mg = macrocell.build(fld, dims, 16, dev)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1000.0
    cfg = session_config(P, SessionConfig, pool=64)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=args.res, height=args.res)
    out = {"volume": "4096^3 virtual random-init INR", "brick": 16, "lod_levels": None, "pool_slots": 64 ** 3,
           "macro_build_ms": build_ms, "preroll": args.config3_preroll}
    for march in ("throughput", "parity"):
        s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, device=dev, march=march)
        out["lod_levels"] = s.cache.max_lod + 1
        preroll(s, traj.camera_at, args.config3_preroll)
        f0 = args.config3_preroll
        o = device_frames(s, traj.camera_at, range(f0, f0 + args.config3_steps), flush, s.stream, timing=True)
        smp = sum(r.samples for r in o["recs"])
        lr = o["recs"][-1]
        out[march] = {"fps": len(o["ms"]) / (sum(o["ms"]) / 1000.0), "ms_per_frame": statistics.mean(o["ms"]),
                      "samples_per_frame": smp / len(o["ms"]),
                      "true_misses_per_frame": sum(r.true_misses for r in o["recs"]) / len(o["ms"]),
                      "occupancy": lr.occupancy,
                      "roofline": roofline(smp, o["march_ms"], o["march_launches"], peak, peak_src, march,
                                           o["march_ms"] / sum(o["ms"]), profile=f"{march}_config3")}
        del s
        torch.cuda.empty_cache()
    out["target_60fps_met"] = out["throughput"]["fps"] >= 60.0
    # BASELINE config 5 at N=1: the same 4096^3 volume at 3840x2160 (the per-GPU tile of
    # the sort-first runs is a 1/N row band of this frame)
    if args.config5_steps > 0:
        t5 = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=3840, height=2160)
        s = RenderSession(fld, P.warm_body(0.5, 0.9), t5.camera_at(0), cfg, macro=mg, device=dev, march="throughput")
        preroll(s, t5.camera_at, args.config5_preroll)
        f0 = args.config5_preroll
        o = device_frames(s, t5.camera_at, range(f0, f0 + args.config5_steps), flush, s.stream, timing=True)
        smp = sum(r.samples for r in o["recs"])
        out["config5_n1"] = {"image": "3840x2160", "march": "throughput", "preroll": f0,
                             "fps": len(o["ms"]) / (sum(o["ms"]) / 1000.0), "ms_per_frame": statistics.mean(o["ms"]),
                             "samples_per_frame": smp / len(o["ms"]),
                             "roofline": roofline(smp, o["march_ms"], o["march_launches"], peak, peak_src,
                                                  "throughput", o["march_ms"] / sum(o["ms"]), profile="throughput_config5")}
        del s
        torch.cuda.empty_cache()
    return out


def run_config1(P, SessionConfig, OrbitTrajectory, args, flush, dev):
    """BASELINE config 1 at its stated size: 64^3 random-init INR, B=16, the 2-level
    paged MRPD knobs (direct_table_threshold=8, page_size=4, page_budget=2), 4^3 pool,
    256x256, the 120-frame orbit; fps over the orbit's last 20 frames (harness.py:65-109's
    summary window), device-timed and through render_frame()."""
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.session import RenderSession

    dims = (64,) * 3
    fld = make_model(64).as_field()
    mg = macrocell.build(fld, dims, 16, dev)
    cfg = SessionConfig(cached=True, loader="inline",
                        cache=P.CacheConfig(brick_size=16, pool_dims=(4, 4, 4), direct_table_threshold=8, page_size=4,
                                            page_budget=2),
                        scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20),
                        settings=P.RenderSettings(), seed=0)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=256, height=256)
    out = {"volume": "64^3 random-init INR", "image": "256x256", "orbit_frames": 120, "window": "frames 100-119"}
    for march in ("throughput", "parity"):
        s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, device=dev, march=march)
        preroll(s, traj.camera_at, 100)
        o = device_frames(s, traj.camera_at, range(100, 120), flush, s.stream)
        s2 = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, device=dev, march=march)
        s2.reserve_host_frames(2)
        walls = []
        for f in range(120):
            s2.set_camera(traj.camera_at(f))
            t0 = time.perf_counter()
            s2.render_frame()
            if f >= 100:
                walls.append(time.perf_counter() - t0)
        out[march] = {"fps": len(o["ms"]) / (sum(o["ms"]) / 1000.0), "e2e_fps": len(walls) / sum(walls),
                      "hit_rate": 1.0 - sum(r.true_misses for r in o["recs"]) / max(1, sum(r.samples for r in o["recs"]))}
        del s, s2
    return out


def run_config4(P, SessionConfig, OrbitTrajectory, macrocell, args, flush, dev):
    """BASELINE config 4: 2048^3 random-init INR, 1920x1080, saliency-ranked vs FIFO
    scheduling (SchedulerConfig.ranking_enabled) along the orbit with a transfer-function
    switch at frame 16: frames to a 90% hit rate (harness.py:78-86) and fps."""
    from paper_2504_18001_b200.session import RenderSession

    dims = (2048,) * 3
    fld = make_model(2048).as_field()
    mg = macrocell.build(fld, dims, 16, dev)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1920, height=1080)
    out = {"volume": "2048^3 random-init INR", "image": "1920x1080", "frames": args.config4_frames,
           "event": "warm_body(0.5,0.9) -> warm_body(0.4,0.85) at frame 16"}
    for label, ranked in (("ranked", True), ("fifo", False)):
        cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(48, 48, 48)),
                            scheduler=P.SchedulerConfig(max_requests=40, ranking_enabled=ranked),
                            policy=P.LodPolicy(1.2, 20), settings=P.RenderSettings(), seed=0)
        s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, device=dev,
                          march="throughput")
        recs, ms = [], []
        for f in range(args.config4_frames):
            if f == 16:
                s.set_transfer_function(P.warm_body(0.4, 0.85))
            o = device_frames(s, traj.camera_at, [f], flush, s.stream)
            recs.append(o["recs"][0])
            ms.append(o["ms"][0])
        rates = [(r.samples - r.true_misses) / r.samples if r.samples else 0.0 for r in recs]
        exact = [r.exact_hits / r.samples if r.samples else 0.0 for r in recs]
        to90 = next((i for i, x in enumerate(rates) if x >= 0.9), -1)
        out[label] = {"frames_to_hit_rate_0.9": to90, "fps_last_10": 10 / (sum(ms[-10:]) / 1000.0),
                      "exact_lod_hit_rate_mean": float(np.mean(exact)), "exact_lod_hit_rate_last": exact[-1]}
        del s
    return out


if __name__ == "__main__":
    main()
