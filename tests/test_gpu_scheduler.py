"""Frame scheduler (north_star subsystem 4) — needs a B200.

* decode_budget=None is the reference (every true miss decoded, max_requests
  bricks): covered by every session test; a budget at least as large as a frame's
  demand changes nothing.
* A finite budget bounds what a frame decodes: true misses first (the rest are filed
  but not composited), then the brick batch gets the remainder (at least one brick).
* loader="thread": the batch is decoded on a decode stream overlapping the next
  frame's march and inserted at the next maintenance, so the per-frame state equals
  the reference's inline loader bit for bit.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("impl", [0, 10])
def test_thread_loader_overlapped_decode_matches_reference(impl):
    """The golden 'pressure' session (recorded with the inline loader) replayed with
    loader='thread': decode on its own stream, same state every frame."""
    import scene_specs
    from gpu_runner import run_gpu_session

    name = "_pressure_thread"
    scene_specs.SESSION_SPECS[name] = dict(scene_specs.SESSION_SPECS["pressure"], loader="thread")
    try:
        g = load_golden("session_pressure.npz")
        ref_impl = 0
        sess_frames = run_gpu_session(name, macro=(g["macro_vmin"], g["macro_vmax"]), impl=impl)
        if impl == 0:
            for f, img, rec, sess in sess_frames:
                assert sess._dstream is not None
                st = sess.debug_state()
                for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
                    np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")
                assert np.abs(img - g[f"f{f}_img"]).max() <= 1e-6
        else:
            inline = run_gpu_session("pressure", macro=(g["macro_vmin"], g["macro_vmax"]), impl=impl)
            for (f, img, rec, sess), (_, img2, rec2, sess2) in zip(sess_frames, inline):
                a, b = sess.debug_state(), sess2.debug_state()
                for k in ("tables", "owner", "last_used", "entries", "batch"):
                    np.testing.assert_array_equal(a[k], b[k], err_msg=f"frame {f} {k}")
                np.testing.assert_array_equal(img, img2)
        del ref_impl
    finally:
        scene_specs.SESSION_SPECS.pop(name, None)


def _inr_session(budget, march, cached=True, res=128, max_requests=40):
    import paper_2504_18001_b200 as P
    from gpu_runner import product_inr
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    dims = (256, 256, 256)
    cfg = SessionConfig(cached=cached, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(16, 16, 16)),
                        scheduler=P.SchedulerConfig(max_requests=max_requests, decode_budget=budget),
                        policy=P.LodPolicy(1.2, 0), settings=P.RenderSettings(), seed=0)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=res, height=res)
    return RenderSession(product_inr(dims).as_field(), P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, march=march), traj


@pytest.mark.parametrize("march", ["parity", "throughput"])
def test_budget_bounds_the_cold_frame(march):
    """Frame 0 (nothing resident, no preload ramp: every sample a true miss): with a
    budget of 5000 samples, exactly 5000 misses are decoded, the rest are deferred,
    and the batch shrinks to the one-brick floor; the unbounded run decodes them all."""
    s0, _ = _inr_session(None, march)
    _, r0 = s0.render_frame()
    st0 = s0.last_frame_stats
    assert r0.true_misses > 20000 and st0["misses_resolved"] == r0.true_misses and st0["deferred_misses"] == 0
    s1, _ = _inr_session(5000, march)
    img1, r1 = s1.render_frame()
    st1 = s1.last_frame_stats
    assert st1["misses_resolved"] == 5000
    assert st1["deferred_misses"] == r1.true_misses - 5000
    assert s1.last_cache_state["n_batch"] == 1  # budget spent on misses: the one-brick floor
    assert s0.last_cache_state["n_batch"] == min(40, s0.last_cache_state["n_pending"])
    assert np.isfinite(img1).all()


def test_budget_splits_between_misses_and_bricks():
    """A budget of 40 bricks' worth plus 1000 samples: the frame's misses (all decoded
    while within budget) are charged first, the batch gets floor(rest / 4096)."""
    b3 = 16 ** 3
    budget = 10 * b3 + 1000
    s2, traj = _inr_session(budget, "throughput")
    for f in range(8):
        s2.set_camera(traj.camera_at(f))
        _, rec = s2.render_frame()
        st = s2.last_frame_stats
        used = st["misses_resolved"]
        assert used <= budget
        want = max(1, min(40, (budget - used) // b3))
        assert s2.last_cache_state["n_batch"] <= want
        if s2.last_cache_state["n_pending"] >= want:
            assert s2.last_cache_state["n_batch"] == want, (f, used, s2.last_cache_state)


def test_budget_covering_the_demand_changes_nothing():
    """A budget above every frame's demand gives the unbounded run's images and state."""
    a, traj = _inr_session(None, "parity")
    b, _ = _inr_session(10 ** 9, "parity")
    for f in range(5):
        for s in (a, b):
            s.set_camera(traj.camera_at(f * 7))
        ia, ra = a.render_frame()
        ib, rb = b.render_frame()
        np.testing.assert_array_equal(ia, ib)
        assert (ra.samples, ra.true_misses, ra.exact_hits) == (rb.samples, rb.true_misses, rb.exact_hits)
        da, db = a.debug_state(), b.debug_state()
        for k in ("tables", "owner", "entries", "batch"):
            np.testing.assert_array_equal(da[k], db[k])


def test_budget_caps_uncached_frame_time():
    """The no-cache baseline (every sample inferred) under a budget of 2^18 decodes per
    frame: the frame does a bounded amount of inference and gets faster."""
    import time

    def run(budget):
        s, traj = _inr_session(budget, "throughput", cached=False, res=256)
        s.render_frame()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            s.render_frame()
        return (time.perf_counter() - t0) / 3, s.last_frame_stats

    t_full, st_full = run(None)
    t_cap, st_cap = run(1 << 18)
    assert st_cap["misses_resolved"] == 1 << 18 and st_full["misses_resolved"] > 1 << 18
    assert t_cap < t_full
