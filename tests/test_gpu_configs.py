"""BASELINE configs 1-3 and 5 at their stated sizes, both march schedules — needs a B200.

* config 1 (64^3 random-init INR, 2-level paged MRPD, 256^2, the full 120-frame
  orbit): the parity schedule against the reference's own run
  (tests/golden/session_config1.npz, tests/golden/make_config1.py) frame by frame;
  the throughput schedule against the oracle with pixel RNG lanes.
* config 2 (512^3, 1024^2): after a pre-roll past the preload ramp, the oracle
  resumes the GPU session's exact state and renders the next frame.
* config 3 (4096^3 virtual, 10 LoD levels, 1024^2): the same resumed-frame check.
* config 5 (4096^3, 3840x2160): four sort-first bands with private caches join into
  the single-session frame bit for bit (throughput schedule, stochastic LoD: pixel
  lanes give a band the whole frame's draws).
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402
from oracle_runner import oracle_state, record_array, run_oracle_session  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _record(rec):
    return np.array([rec.frame, rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits, rec.bricks_loaded,
                     rec.bricks_loaded_total, rec.requests_inflight], dtype=np.int64)


def _psnr(a, b):
    mse = float(np.mean((a[..., :3].astype(np.float64) - b[..., :3]) ** 2))
    return 10 * np.log10(1.0 / mse) if mse > 0 else np.inf


def test_config1_full_orbit_vs_reference():
    """120 frames at 256^2: FrameRecords, page tables, owners, request table and
    batches equal the reference's every frame; images within 1e-3 / >= 60 dB."""
    from gpu_runner import run_gpu_session

    g = load_golden("session_config1.npz")
    n = 0
    for f, img, rec, sess in run_gpu_session("config1", macro=(g["macro_vmin"], g["macro_vmax"])):
        np.testing.assert_array_equal(_record(rec), g[f"f{f}_record"], err_msg=f"frame {f} record")
        st = sess.debug_state()
        for k in ("tables", "owner", "entries", "batch"):
            np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")
        if f"f{f}_img" in g:
            ref = g[f"f{f}_img"]
            assert np.abs(img - ref).max() <= 1e-3 and _psnr(img, ref) >= 60.0, f"frame {f}"
        n += 1
    assert n == 120


def test_config1_throughput_vs_oracle_pixel_lanes():
    """The throughput schedule on the config-1 recipe (first 40 frames) equals the
    oracle with the same pixel RNG lanes."""
    import scene_specs
    from gpu_runner import run_gpu_session

    name = "_config1_pix"
    scene_specs.SESSION_SPECS[name] = dict(scene_specs.SESSION_SPECS["config1"], rng="pixel", frames=40)
    try:
        g = load_golden("session_config1.npz")
        macro = (g["macro_vmin"], g["macro_vmax"])
        for (f, img, rec, sess), (_, oimg, orec, osess) in zip(run_gpu_session(name, macro=macro, impl=10),
                                                               run_oracle_session(name, macro=macro)):
            np.testing.assert_array_equal(_record(rec), record_array(orec), err_msg=f"frame {f}")
            st, ost = sess.debug_state(), oracle_state(osess)
            for k in ("tables", "owner", "entries", "batch"):
                np.testing.assert_array_equal(st[k], ost[k], err_msg=f"frame {f} {k}")
            assert np.abs(img - oimg).max() <= 1e-3, f"frame {f}"
    finally:
        scene_specs.SESSION_SPECS.pop(name, None)


def _resumed_frame_check(dims, res, pool, march, preroll, macro_np, mg, seed=0):
    """Pre-roll a GPU session, hand its exact state to the oracle, render the next frame
    on both; image, counters and post-maintenance state must agree."""
    from gpu_runner import product_inr
    from oracle import cinr_oracle as O
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    import paper_2504_18001_b200 as P

    cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(pool,) * 3),
                        scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20),
                        settings=P.RenderSettings(), seed=seed)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=res, height=res)
    sess = RenderSession(product_inr(dims).as_field(), P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg,
                         march=march)
    for f in range(preroll):
        sess.set_camera(traj.camera_at(f))
        sess.render_frame()
    state = sess.export_state()
    sess.set_camera(traj.camera_at(preroll))
    img, rec = sess.render_frame()
    gst = sess.cache.dump()
    gst["batch"] = sess.cache.batch()

    t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
    ocfg = O.Config(dims=dims, brick=16, pool=(pool,) * 3, max_requests=40, lod_scale=1.2, preload=20, seed=seed,
                    rng="pixel" if march == "throughput" else "rank")
    osess = O.OracleSession(O.InrFieldOracle(dims, t, w, b, O.DEFAULT_GRID), O.warm_body_points(0.5, 0.9), ocfg,
                            macro_minmax_arrays=macro_np)
    O.load_session_state(osess, state)
    osess.set_camera(traj.camera_at(preroll).position, (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0, res, res)
    oimg, orec = osess.render_frame()
    assert (rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits, rec.bricks_loaded) == \
           (orec.samples, orec.true_misses, orec.fallback_hits, orec.exact_hits, orec.bricks_loaded)
    assert np.abs(img - oimg).max() <= 1e-3 and _psnr(img, oimg) >= 60.0
    ost = oracle_state(osess)
    for k in ("tables", "owner", "last_used", "entries", "batch"):
        np.testing.assert_array_equal(gst[k], ost[k], err_msg=k)
    return rec


@pytest.mark.parametrize("march", ["parity", "throughput"])
def test_config2_1024_resumed_frame_vs_oracle(march):
    from gpu_runner import product_inr
    from paper_2504_18001_b200 import macrocell

    dims = (512,) * 3
    mg = macrocell.build(product_inr(dims).as_field(), dims, 16)
    rec = _resumed_frame_check(dims, 1024, 32, march, 30, (mg.value_min, mg.value_max), mg)
    assert rec.samples > 10_000_000


def test_config3_coherent_empty_space_supercell_jumps_vs_oracle():
    """4096^3 with spatially coherent empty space (blocks of 8^3 macro cells, 40% empty,
    plus everything outside a ball): the throughput kernel leaves whole empty 4x4x4
    super-cells in one step there (advance_impl<2>); the resumed frame must still equal
    the oracle's cell-by-cell walk bit for bit."""
    from gpu_runner import macro_from

    dims = (4096,) * 3
    rng = np.random.default_rng(11)
    blocks = rng.random((32, 32, 32)) < 0.4
    empty = np.repeat(np.repeat(np.repeat(blocks, 8, 0), 8, 1), 8, 2)
    i = (np.arange(256) + 0.5 - 128.0) ** 2
    empty |= (i[:, None, None] + i[None, :, None] + i[None, None, :]) > 118.0 ** 2
    vmax = np.where(empty, 0.2, 1.0).astype(np.float32)
    vmin = np.zeros_like(vmax)
    rec = _resumed_frame_check(dims, 512, 24, "throughput", 12, (vmin, vmax), macro_from(dims, vmin, vmax))
    assert rec.samples > 1_000_000


def test_config2_forced_supercell_kernel_equals_default():
    """The benched config 2 (512^3 INR, its own macro grid: coherent empty space) with the
    large-grid specialisation forced (CINR_FORCE_SUPERCELL: super-cell bits + jumps over
    empty super-cells) renders the same frames and cache state as the default
    shared-memory-majorant kernel, over a cold-cache orbit."""
    import os

    from gpu_runner import product_inr
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    import paper_2504_18001_b200 as P

    dims = (512,) * 3
    fld = product_inr(dims).as_field()
    mg = macrocell.build(fld, dims, 16)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=512, height=512)

    def run(force):
        if force:
            os.environ["CINR_FORCE_SUPERCELL"] = "1"
        try:
            cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(32,) * 3),
                                scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20),
                                settings=P.RenderSettings(), seed=0)
            s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, march="throughput")
            out = []
            for f in range(0, 48, 4):
                s.set_camera(traj.camera_at(f))
                img, rec = s.render_frame()
                st = s.cache.dump()
                out.append((img.copy(), (rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits,
                                         rec.bricks_loaded), {k: st[k].copy() for k in ("tables", "owner", "last_used",
                                                                                        "entries")}))
            return out
        finally:
            os.environ.pop("CINR_FORCE_SUPERCELL", None)

    a, b = run(False), run(True)
    for f, ((ia, ra, sa), (ib, rb, sb)) in enumerate(zip(a, b)):
        assert ra == rb, f"frame {f}: {ra} vs {rb}"
        np.testing.assert_array_equal(ia, ib, err_msg=f"frame {f} image")
        for k in sa:
            np.testing.assert_array_equal(sa[k], sb[k], err_msg=f"frame {f} {k}")


@pytest.mark.parametrize("march,res", [("parity", 1024), ("throughput", 512)])
def test_config3_4096_resumed_frame_vs_oracle(march, res):
    """4096^3 virtual volume (19.4 M bricks, paged MRPD distances on the reference
    side) with a synthetic 35%-empty macro grid shared by both sides (P16).  (The
    oracle needs ~70 s for a 1024^2 frame at this size, so the throughput schedule is
    checked at 512^2.)"""
    from gpu_runner import macro_from

    dims = (4096,) * 3
    rng = np.random.default_rng(7)
    vmax = np.where(rng.random((256, 256, 256)) < 0.35, 0.2, 1.0).astype(np.float32)
    vmin = np.zeros_like(vmax)
    rec = _resumed_frame_check(dims, res, 24, march, 12, (vmin, vmax), macro_from(dims, vmin, vmax))
    assert rec.samples > 1_000_000


def test_config5_4096_4k_four_bands_join_bit_exact():
    """3840x2160, 4096^3: 1 full-frame session and 4 band sessions (rows r, r+4, ...)
    each with its own cache, throughput schedule, stochastic LoD (corrected).  Once
    every session's cache serves every sample at its requested LoD, values depend only
    on the draws, and the joined bands equal the full frame."""
    from gpu_runner import macro_from, product_inr
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    import paper_2504_18001_b200 as P

    dims = (4096,) * 3
    W, H, world = 3840, 2160, 4
    rng = np.random.default_rng(11)
    vmax = np.where(rng.random((256, 256, 256)) < 0.3, 0.2, 1.0).astype(np.float32)
    mg = macro_from(dims, np.zeros_like(vmax), vmax)
    fld = product_inr(dims).as_field()
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=W, height=H)

    def run(band):
        cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(64, 64, 64)),
                            scheduler=P.SchedulerConfig(max_requests=2048), policy=P.LodPolicy(3.0, 0),
                            settings=P.RenderSettings(), seed=5)
        s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(9), cfg, macro=mg, march="throughput")
        s.set_band(*band)
        # the same number of frames in every session: the draws depend on the frame number
        for _ in range(24):
            img, rec = s.render_frame()
        assert rec.true_misses == 0 and rec.fallback_hits == 0, f"band {band}: cache not warm ({rec})"
        return img

    full = run((0, 1))
    joined = np.empty_like(full)
    for r in range(world):
        joined[r::world] = run((r, world))
    np.testing.assert_array_equal(joined, full)
