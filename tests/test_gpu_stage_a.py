"""Stage A on the GPU box (SURVEY §8b "Recommended staging"): the reference's own
RenderSession — the unmodified `voxcache` package installed into baseline/_ref
(`pip install --no-deps --target baseline/_ref`) — renders the same
frames twice: on its numba CPU passes, and with `plugin.install(voxcache.render.kernels)`
swapping raygen/advance/probe/shade for the sm_100a passes.  Images, FrameRecords and
the reference's own cache state (page tables, pool owners, stamps, request table)
must agree bit for bit.  Skipped where baseline/_ref was not installed."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def vc():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not (REF / "voxcache").is_dir():
        pytest.skip("the reference is not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_stage_a")
    sys.path.insert(0, str(REF))
    import voxcache

    return voxcache


def _ref_session(vc, spec):
    from scene_specs import smoothed_random_lattice
    from voxcache import macrocell
    from voxcache.cache import CacheConfig
    from voxcache.fields import FieldDomain, RawLatticeField
    from voxcache.harness import OrbitTrajectory
    from voxcache.inr import HashGridConfig, InrModel, MLPConfig
    from voxcache.render import warm_body
    from voxcache.render.scene import RenderSettings
    from voxcache.sampler import LodPolicy
    from voxcache.scheduler import SchedulerConfig
    from voxcache.session import RenderSession, SessionConfig

    dims = tuple(spec["dims"])
    if spec["field"] == "inr":
        m = InrModel(HashGridConfig(), MLPConfig(), FieldDomain(dims), seed=0)
        r = np.random.default_rng(42)
        m.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in m.parameters()])
        field = m.as_field()
    else:
        field = RawLatticeField(smoothed_random_lattice(dims, spec["field_seed"]), FieldDomain(dims))
    traj = OrbitTrajectory((0.5, 0.5, 0.5), spec.get("radius", 2.2), 120, width=spec["res"][0], height=spec["res"][1])
    cfg = SessionConfig(cached=True, loader="inline",
                        cache=CacheConfig(brick_size=spec["brick"], pool_dims=tuple(spec["pool"])),
                        scheduler=SchedulerConfig(**spec.get("sched_kw", {})), policy=LodPolicy(**spec["policy"]),
                        settings=RenderSettings(**spec.get("settings", {})), seed=0)
    sess = RenderSession(field, warm_body(*spec["tf"][1:]), traj.camera_at(0), cfg,
                         macro=macrocell.build(field, dims, 16))
    return sess, traj


def _state(sess):
    c = sess.cache
    tabs = [np.asarray(t.entries).copy() for t in c.tables]
    own = [(-1, -1) if k is None else (k.lod, k.linear_index(c.layout.grids[k.lod])) for k in c.pool.owner]
    ents = sorted((e.key.lod, e.key.linear_index(c.layout.grids[e.key.lod]), e.base, e.hits)
                  for e in sess.table._entries.values())
    return tabs, own, c.pool.last_used.copy(), ents


def _run(vc, spec, gpu, frames):
    from paper_2504_18001_b200 import plugin
    from voxcache.render import kernels

    undo = plugin.install(kernels) if gpu else None
    try:
        sess, traj = _ref_session(vc, spec)
        out = []
        for f in range(frames):
            sess.set_camera(traj.camera_at(f * spec.get("cam_step", 1)))
            img, rec = sess.render_frame()
            out.append((img, (rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits, rec.bricks_loaded),
                        _state(sess)))
        return out
    finally:
        if undo is not None:
            undo()


@pytest.mark.parametrize("name", ["pressure", "lattice64_fifo", "inr64"])
def test_reference_session_on_b200_passes(vc, name):
    import scene_specs

    spec = scene_specs.SESSION_SPECS[name]
    frames = min(spec["frames"], 8)
    cpu = _run(vc, spec, False, frames)
    gpu = _run(vc, spec, True, frames)
    for f, ((ia, ra, sa), (ib, rb, sb)) in enumerate(zip(cpu, gpu)):
        assert ra == rb, (name, f, ra, rb)
        np.testing.assert_array_equal(ia, ib, err_msg=f"{name} frame {f} image")
        for x, y in zip(sa[0], sb[0]):
            np.testing.assert_array_equal(x, y)
        assert sa[1] == sb[1] and sa[3] == sb[3], (name, f)
        np.testing.assert_array_equal(sa[2], sb[2])
