"""Replays a tests/scene_specs.py session through the CPU oracle (test infra)."""

from __future__ import annotations

import numpy as np

from oracle import cinr_oracle as O
from scene_specs import SESSION_SPECS, smoothed_random_lattice


def tf_points(name):
    if name[0] == "warm_body":
        return O.warm_body_points(*name[1:])
    if name[0] == "grayscale_ramp":
        return O.grayscale_points(*name[1:])
    return np.asarray(name[1], dtype=np.float64)


def oracle_field(spec):
    if spec["field"] == "lattice":
        return O.LatticeField(smoothed_random_lattice(spec["dims"], spec["field_seed"]))
    if spec["field"] == "inr":
        t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
        return O.InrFieldOracle(spec["dims"], t, w, b, O.DEFAULT_GRID)
    raise ValueError(spec["field"])


def oracle_config(spec):
    ck = spec.get("cache_kw", {})
    sk = spec.get("sched_kw", {})
    pol = spec["policy"]
    st = spec.get("settings", {})
    return O.Config(
        dims=tuple(spec["dims"]), brick=spec["brick"], pool=tuple(spec["pool"]),
        direct_threshold=ck.get("direct_table_threshold", 1 << 18),
        max_requests=sk.get("max_requests", 40), ranking=sk.get("ranking_enabled", True),
        rank_clamp=sk.get("rank_clamp", 1000),
        lod_scale=pol.get("lod_scale", 1.0), preload=pol.get("preload_frames", 120), mode=pol.get("mode", "corrected"),
        cached=spec.get("cached", True), seed=spec.get("seed", 0),
        skip_empty=st.get("skip_empty", True), adaptive=st.get("adaptive_step", True),
        base_step_scale=st.get("base_step_scale", 0.5), rng=spec.get("rng", "rank"),
        max_iterations=st.get("max_iterations", 8192), background=tuple(st.get("background", (0.0, 0.0, 0.0))),
        term=st.get("early_termination", 0.01),
    )


def camera_for(spec, f):
    pos = O.orbit_camera((0.5, 0.5, 0.5), spec.get("radius", 2.2), 120, f * spec.get("cam_step", 1))
    w, h = spec["res"]
    return dict(position=pos, target=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0), fov_y=45.0, width=w, height=h)


def run_oracle_session(name, macro=None, frames=None):
    """Yields (frame, img, record, session) per frame."""
    spec = SESSION_SPECS[name]
    fld = oracle_field(spec)
    sess = O.OracleSession(fld, tf_points(spec["tf"]), oracle_config(spec), macro_minmax_arrays=macro)
    events = spec.get("events", {})
    for f in range(frames if frames is not None else spec["frames"]):
        ev = events.get(f)
        if ev is not None:
            if ev[0] == "tf":
                sess.set_tf(tf_points(ev[1]))
            elif ev[0] == "reset":
                sess.reset_cache()
            elif ev[0] == "lod_scale":
                sess.cfg.lod_scale = float(ev[1])
        sess.set_camera(**camera_for(spec, f))
        img, rec = sess.render_frame()
        yield f, img, rec, sess


def oracle_state(sess):
    c = sess.cache
    ents = sorted((k[0], k[1], v[0], v[1]) for k, v in sess.req.entries.items())
    return dict(
        tables=c.table.copy(), owner=c.owner.copy(), last_used=c.last_used.copy(), n_free=len(c.free),
        cache_frame=c.frame,
        entries=np.array(ents, dtype=np.int64).reshape(-1, 4),
        reports=np.array(sorted((k[0], k[1], v) for k, v in sess.last_reports.items()), dtype=np.int64).reshape(-1, 3),
        batch=np.array(sess.last_batch, dtype=np.int64).reshape(-1, 2),
    )


def record_array(rec):
    return np.array([rec.frame, rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits,
                     rec.bricks_loaded, rec.bricks_loaded_total, rec.requests_inflight], dtype=np.int64)
