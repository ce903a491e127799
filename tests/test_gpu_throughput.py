"""Throughput-mode frame kernel (k_ray_march: one persistent ray per lane, RNG lane =
film pixel) vs the reference and the oracle — needs a B200.

* LodPolicy(mode="off") draws no random numbers, so the throughput schedule must
  reproduce the reference's golden sessions bit for bit (images, records, page
  tables, owners, stamps, request table, miss reports, batches).
* With stochastic LoD it must equal the oracle run with the same lane rule
  (oracle Config.rng="pixel": seeds and xorshift32 steps of sampler.py:39-58,
  lane = row*W + col), bit for bit, over whole cache-pressure sessions.
* Band partitions (sort-first) draw the same numbers as the whole frame, so with
  a shared warm cache the joined bands equal the single frame bit for bit.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402
from oracle_runner import oracle_state, record_array, run_oracle_session  # noqa: E402

THROUGHPUT = [10, 11, 12, 14]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _record(rec):
    return np.array([rec.frame, rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits, rec.bricks_loaded,
                     rec.bricks_loaded_total, rec.requests_inflight], dtype=np.int64)


@pytest.mark.parametrize("impl", THROUGHPUT)
def test_mode_off_session_bit_exact_vs_reference(impl):
    """aniso_b10 (LoD mode off, non-power-of-two bricks, no skipping): the reference's
    golden per-frame state, reproduced by the throughput schedule."""
    from gpu_runner import run_gpu_session

    g = load_golden("session_aniso_b10.npz")
    n = 0
    for f, img, rec, sess in run_gpu_session("aniso_b10", macro=(g["macro_vmin"], g["macro_vmax"]), impl=impl):
        np.testing.assert_array_equal(_record(rec), g[f"f{f}_record"], err_msg=f"frame {f} record")
        st = sess.debug_state()
        for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
            np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")
        assert np.abs(img - g[f"f{f}_img"]).max() <= 1e-6, f"frame {f}"
        n += 1
    assert n == 14


@pytest.mark.parametrize("base", ["pressure", "lattice64", "events", "lattice64_fifo"])
def test_mode_off_throughput_equals_parity(base):
    """The golden recipes with the LoD rule switched off: both schedules, same state."""
    import scene_specs
    from gpu_runner import run_gpu_session

    name = f"_off_{base}"
    spec = dict(scene_specs.SESSION_SPECS[base])
    spec["policy"] = dict(spec["policy"], mode="off")
    spec["frames"] = min(spec["frames"], 12)
    scene_specs.SESSION_SPECS[name] = spec
    try:
        for (f, ia, ra, xa), (_, ib, rb, xb) in zip(run_gpu_session(name, impl=0), run_gpu_session(name, impl=10)):
            np.testing.assert_array_equal(_record(ra), _record(rb), err_msg=f"frame {f}")
            np.testing.assert_array_equal(ia, ib, err_msg=f"frame {f} image")
            da, db = xa.debug_state(), xb.debug_state()
            for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
                np.testing.assert_array_equal(da[k], db[k], err_msg=f"frame {f} {k}")
    finally:
        scene_specs.SESSION_SPECS.pop(name, None)


@pytest.mark.parametrize("base", ["pressure", "lattice64", "events"])
def test_mode_off_supercell_kernel_equals_parity(base, monkeypatch):
    """The large-grid specialisation (super-cell bits, jumps over empty super-cells)
    forced on the small golden scenes: still the parity schedule's state bit for bit."""
    monkeypatch.setenv("CINR_FORCE_SUPERCELL", "1")
    test_mode_off_throughput_equals_parity(base)


@pytest.mark.parametrize("base", ["pressure", "lattice64", "lattice64_paged", "events", "lattice64_fifo", "inr64"])
def test_pixel_lane_sessions_vs_oracle(base):
    """Stochastic LoD with pixel lanes: CUDA throughput schedule == oracle(rng="pixel")."""
    import scene_specs
    from gpu_runner import run_gpu_session

    name = f"_pix_{base}"
    spec = dict(scene_specs.SESSION_SPECS[base], rng="pixel")
    spec["frames"] = min(spec["frames"], 12)
    scene_specs.SESSION_SPECS[name] = spec
    inr = spec["field"] == "inr"
    try:
        g = load_golden(f"session_{base}.npz")
        macro = (g["macro_vmin"], g["macro_vmax"])
        for (f, img, rec, sess), (_, oimg, orec, osess) in zip(run_gpu_session(name, macro=macro, impl=10),
                                                               run_oracle_session(name, macro=macro)):
            np.testing.assert_array_equal(_record(rec), record_array(orec), err_msg=f"frame {f}")
            st, ost = sess.debug_state(), oracle_state(osess)
            keys = ("tables", "owner", "entries", "batch") if inr else ("tables", "owner", "last_used", "entries",
                                                                         "reports", "batch")
            for k in keys:
                np.testing.assert_array_equal(st[k], ost[k], err_msg=f"frame {f} {k}")
            tol = 1e-3 if inr else 1e-6
            assert np.abs(img - oimg).max() <= tol, f"frame {f}"
    finally:
        scene_specs.SESSION_SPECS.pop(name, None)


def test_pixel_lanes_differ_from_rank_lanes_but_match_statistics():
    """Sanity: the stochastic LoD really is on in these runs (pixel lanes change the
    request stream vs rank lanes), yet hit statistics stay close."""
    import scene_specs
    from gpu_runner import run_gpu_session

    recs = {}
    for impl in (0, 10):
        recs[impl] = [r for _, _, r, _ in run_gpu_session("pressure", frames=10, impl=impl)]
    a = [(r.exact_hits, r.fallback_hits) for r in recs[0]]
    b = [(r.exact_hits, r.fallback_hits) for r in recs[10]]
    assert a != b
    sa = sum(r.samples for r in recs[0])
    sb = sum(r.samples for r in recs[10])
    assert abs(sa - sb) / sa < 0.05


def test_bands_join_to_the_frame():
    """Sort-first bands of a throughput frame (each band its own session and cache)
    equal the single frame bit for bit once every session's cache serves every sample
    exactly: values then depend only on the stochastic-LoD draws, and pixel lanes give
    a band the draws the whole frame makes."""
    import paper_2504_18001_b200 as P
    from gpu_runner import product_field, product_tf
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig
    import scene_specs

    spec = scene_specs.SESSION_SPECS["pressure"]
    fld = product_field(spec)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 1.7, 120, width=96, height=80)

    def run(band, frames=14):
        cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=8, pool_dims=(12, 12, 12)),
                            scheduler=P.SchedulerConfig(max_requests=2000), policy=P.LodPolicy(1.5, 0, "corrected"),
                            seed=3)
        s = RenderSession(fld, product_tf(spec["tf"]), traj.camera_at(0), cfg, march="throughput")
        s.set_band(*band)
        for f in range(frames):
            img, rec = s.render_frame()
        assert rec.true_misses == 0 and rec.fallback_hits == 0, (band, rec)
        return img

    full = run((0, 1))
    joined = np.empty_like(full)
    for r in range(3):
        joined[r::3] = run((r, 3))
    np.testing.assert_array_equal(joined, full)


@pytest.mark.parametrize("case", ["odd_size", "iteration_cap", "background", "fixed_steps", "no_skip", "nothing_hit"])
def test_edge_cases_vs_oracle(case):
    """Throughput schedule vs the oracle (pixel lanes) on edge cases: film sizes that
    are not multiples of the 8x4 ray tiles, the iteration cap flushing live rays
    (raymarch.py:117), a coloured background, fixed-ladder steps and no empty-space
    skipping (the generic kernel build), and a camera that misses the volume."""
    import scene_specs
    from gpu_runner import run_gpu_session

    base = dict(scene_specs.SESSION_SPECS["pressure"], rng="pixel", frames=5)
    over = {
        "odd_size": dict(res=(37, 23)),
        "iteration_cap": dict(settings=dict(max_iterations=6)),
        "background": dict(settings=dict(background=(0.2, 0.1, 0.3), early_termination=0.05)),
        "fixed_steps": dict(settings=dict(adaptive_step=False), res=(40, 33)),
        "no_skip": dict(settings=dict(skip_empty=False), res=(41, 30)),
        "nothing_hit": dict(radius=2.2, res=(24, 24), fov_far=True),
    }[case]
    spec = dict(base, **{k: v for k, v in over.items() if k != "fov_far"})
    name = f"_edge_{case}"
    scene_specs.SESSION_SPECS[name] = spec
    try:
        if case == "nothing_hit":
            # a camera looking away from the unit box: background everywhere, no samples
            import paper_2504_18001_b200 as P
            from gpu_runner import product_config, product_field, product_tf
            from paper_2504_18001_b200.session import RenderSession

            cam = P.Camera(position=(3.0, 3.0, 3.0), target=(6.0, 6.0, 6.0), width=24, height=24)
            s = RenderSession(product_field(spec), product_tf(spec["tf"]), cam, product_config(spec),
                              march="throughput")
            img, rec = s.render_frame()
            assert rec.samples == 0 and s.last_frame_stats["rays"] == 0
            assert (img == 0.0).all()
            return
        for (f, img, rec, sess), (_, oimg, orec, osess) in zip(run_gpu_session(name, impl=10),
                                                               run_oracle_session(name)):
            np.testing.assert_array_equal(_record(rec), record_array(orec), err_msg=f"{case} frame {f}")
            st, ost = sess.debug_state(), oracle_state(osess)
            for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
                np.testing.assert_array_equal(st[k], ost[k], err_msg=f"{case} frame {f} {k}")
            assert np.abs(img - oimg).max() <= 1e-6, f"{case} frame {f}"
    finally:
        scene_specs.SESSION_SPECS.pop(name, None)
