"""Replays a tests/scene_specs.py session through the product (GPU) API."""

from __future__ import annotations

import numpy as np

import paper_2504_18001_b200 as P
from paper_2504_18001_b200 import macrocell
from scene_specs import SESSION_SPECS, smoothed_random_lattice


def product_tf(name):
    if name[0] == "warm_body":
        return P.warm_body(*name[1:])
    if name[0] == "grayscale_ramp":
        return P.grayscale_ramp(*name[1:])
    return P.TransferFunction(name[1])


def product_inr(dims, seed=0, redraw=42):
    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain(tuple(dims)), seed=seed)
    if redraw is not None:
        r = np.random.default_rng(redraw)
        m.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in m.parameters()])
    return m


def product_field(spec):
    if spec["field"] == "lattice":
        return P.RawLatticeField(smoothed_random_lattice(spec["dims"], spec["field_seed"]), P.FieldDomain(spec["dims"]))
    if spec["field"] == "inr":
        return product_inr(spec["dims"]).as_field()
    return P.make_procedural(spec["field"], spec["dims"])


def product_config(spec):
    from paper_2504_18001_b200.session import SessionConfig

    return SessionConfig(
        cached=spec.get("cached", True), mode=spec.get("mode", "raymarch"), samples_per_pixel=spec.get("spp", 1),
        loader=spec.get("loader", "inline"),
        cache=P.CacheConfig(brick_size=spec["brick"], pool_dims=tuple(spec["pool"]), **spec.get("cache_kw", {})),
        scheduler=P.SchedulerConfig(**spec.get("sched_kw", {})), policy=P.LodPolicy(**spec["policy"]),
        settings=P.RenderSettings(**spec.get("settings", {})), seed=spec.get("seed", 0),
    )


def macro_from(dims, vmin, vmax, cell=16):
    grid, _, _ = macrocell.layout(dims, cell)
    return macrocell.MacroCellGrid(cell, tuple(dims), grid, np.asarray(vmin, np.float32), np.asarray(vmax, np.float32),
                                   np.ones_like(vmin, dtype=np.float32))


def run_gpu_session(name, macro=None, frames=None, debug=True, impl=0, maint_graph=None, setup=None):
    """Yields (frame, img, record, session).  maint_graph: None = the session default;
    setup(session) runs before the first frame."""
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession

    spec = SESSION_SPECS[name]
    fld = product_field(spec)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), spec.get("radius", 2.2), 120, width=spec["res"][0], height=spec["res"][1])
    mg = macro_from(spec["dims"], *macro) if macro is not None else None
    sess = RenderSession(fld, product_tf(spec["tf"]), traj.camera_at(0), product_config(spec), macro=mg, debug=debug)
    sess.impl = impl
    if maint_graph is not None:
        sess.maint_graph = maint_graph
    if setup is not None:
        setup(sess)
    events = spec.get("events", {})
    for f in range(frames if frames is not None else spec["frames"]):
        ev = events.get(f)
        if ev is not None:
            if ev[0] == "tf":
                sess.set_transfer_function(product_tf(ev[1]))
            elif ev[0] == "reset":
                sess.reset_cache()
            elif ev[0] == "lod_scale":
                sess.set_lod_scale(ev[1])
        sess.set_camera(traj.camera_at(f * spec.get("cam_step", 1)))
        img, rec = sess.render_frame()
        yield f, img, rec, sess
