"""Generate golden fixtures by running the UNMODIFIED reference (`voxcache`) here.

This script is the only place that imports the reference. It must run in the
build container (where /root/reference exists); its outputs are committed as
small `.npz` files under tests/golden/ and are what the oracle and the CUDA
path are pinned against on the GPU box (where /root/reference does not exist).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Capture points (all read-only wrappers, nothing in the reference is modified):
  * per frame, after RenderSession.render_frame (vc/session.py:105-130):
    dense page tables (pagetable.py:22 / :48), pool owner/last_used/free
    (pool.py:44-46), cache.frame, request-table entries (scheduler.py:49),
    the drained miss reports (mrpd.py:263) and the dispatched batch
    (scheduler.py:79), FrameStats (taken before tick_frame), the image.
  * op level: inputs/outputs of kernels.raygen/advance/probe/shade_pass
    (render/kernels.py:160, 316, 370, 426) during one frame.

Path-tracing fixtures (pt_* sessions, pt_flight.npz) are generated with numpy's
AVX-512 dispatch disabled, NPY_DISABLE_CPU_FEATURES="AVX512F AVX512CD AVX512VL
AVX512BW AVX512DQ AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR AVX512VNNI
AVX512IFMA AVX512VBMI AVX512VBMI2 AVX512BITALG AVX512FP16 AVX512VPOPCNTDQ": the free
flights use np.log1p (pathtrace.py:80), which numpy computes with SVML on AVX-512
hosts and with libm's log1p elsewhere (the two differ by 1 ulp on ~7% of inputs).
The fixtures pin the libm semantics, which the device follows.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))  # tests/ for scene_specs

import voxcache  # noqa: E402
from voxcache import macrocell  # noqa: E402
from voxcache.cache import BrickKey, CacheConfig  # noqa: E402
from voxcache.cache.pagetable import DirectTable, PagedTable  # noqa: E402
from voxcache.fields import FieldDomain, RawLatticeField, make_procedural  # noqa: E402
from voxcache.harness import OrbitTrajectory  # noqa: E402
from voxcache.inr import HashGridConfig, InrModel, MLPConfig, encoding  # noqa: E402
from voxcache.render import TransferFunction, grayscale_ramp, kernels, warm_body  # noqa: E402
from voxcache.render.scene import RenderSettings  # noqa: E402
from voxcache.sampler import LodPolicy  # noqa: E402
from voxcache.scheduler import SchedulerConfig, fulfill  # noqa: E402
from voxcache.session import RenderSession, SessionConfig  # noqa: E402

import scene_specs as specs  # noqa: E402  (shared, reference-free scene recipes)


def ref_lattice_field(dims, seed):
    return RawLatticeField(specs.smoothed_random_lattice(dims, seed), FieldDomain(tuple(dims)))


def ref_inr_model(dims, seed=0, redraw=42, grid=None, mlp=None):
    m = InrModel(grid or HashGridConfig(), mlp or MLPConfig(), FieldDomain(tuple(dims)), seed=seed)
    if redraw is not None:
        r = np.random.default_rng(redraw)
        m.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in m.parameters()])
    return m


def make_field(spec):
    kind = spec["field"]
    if kind == "lattice":
        return ref_lattice_field(spec["dims"], spec["field_seed"])
    if kind == "inr":
        return ref_inr_model(spec["dims"]).as_field()
    if kind in ("sphere", "shells", "marschner_lobb_like"):
        return make_procedural(kind, spec["dims"])
    raise ValueError(kind)


def make_tf(name):
    if name[0] == "warm_body":
        return warm_body(*name[1:])
    if name[0] == "grayscale_ramp":
        return grayscale_ramp(*name[1:])
    return TransferFunction(name[1])


def session_config(spec):
    return SessionConfig(
        cached=spec.get("cached", True),
        mode=spec.get("mode", "raymarch"),
        samples_per_pixel=spec.get("spp", 1),
        loader="inline",
        cache=CacheConfig(
            brick_size=spec["brick"],
            pool_dims=tuple(spec["pool"]),
            **spec.get("cache_kw", {}),
        ),
        scheduler=SchedulerConfig(**spec.get("sched_kw", {})),
        policy=LodPolicy(**spec["policy"]),
        settings=RenderSettings(**spec.get("settings", {})),
        seed=spec.get("seed", 0),
    )


def dense_tables(cache):
    out = []
    for lod, t in enumerate(cache.tables):
        n = cache.layout.brick_count(lod)
        if isinstance(t, DirectTable):
            out.append(t.entries.copy())
        else:
            dense = np.full(n, -1, dtype=np.int32)
            for pid, page in t._pages.items():
                lo = pid * t.page_size
                hi = min(lo + t.page_size, n)
                dense[lo:hi] = page[: hi - lo]
            out.append(dense)
    return np.concatenate(out).astype(np.int32)


def key_linear(cache, key):
    return key.linear_index(cache.layout.grids[key.lod])


def run_session(spec, op_capture_frame=None):
    field = make_field(spec)
    tf = make_tf(spec["tf"])
    dims = tuple(spec["dims"])
    macro = macrocell.build(field, dims, 16)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), spec.get("radius", 2.2), 120, width=spec["res"][0], height=spec["res"][1])
    cfg = session_config(spec)
    sess = RenderSession(field, tf, traj.camera_at(0), cfg, macro=macro)
    cache = sess.cache

    captured = {"reports": None, "batch": None}
    if cache is not None:
        orig_drain = cache.drain_miss_reports

        def drain():
            r = orig_drain()
            captured["reports"] = r
            return r

        cache.drain_miss_reports = drain

    def wrap_table(table):
        orig_sel = table.select_batch

        def sel(n, exclude=None):
            b = orig_sel(n, exclude)
            captured["batch"] = list(b)
            return b

        table.select_batch = sel

    if sess.table is not None:
        wrap_table(sess.table)

    ops = {}
    frames = {}
    n_frames = spec["frames"]
    events = spec.get("events", {})
    macro_dump = {"vmin": macro.value_min.copy(), "vmax": macro.value_max.copy()}
    for f in range(n_frames):
        ev = events.get(f)
        if ev is not None:
            if ev[0] == "tf":
                sess.set_transfer_function(make_tf(ev[1]))
            elif ev[0] == "reset":
                sess.reset_cache()
                if sess.table is not None:
                    wrap_table(sess.table)
            elif ev[0] == "lod_scale":
                sess.set_lod_scale(ev[1])
        sess.set_camera(traj.camera_at(f * spec.get("cam_step", 1)))
        captured["reports"] = None
        captured["batch"] = None
        if f == op_capture_frame:
            img, rec, ops = capture_ops(sess)
        else:
            img, rec = sess.render_frame()
        d = {"img": img.astype(np.float32)}
        d["record"] = np.array(
            [rec.frame, rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits,
             rec.bricks_loaded, rec.bricks_loaded_total, rec.requests_inflight],
            dtype=np.int64,
        )
        d["occupancy"] = np.float64(rec.occupancy)
        if cache is not None:
            cache = sess.cache
            d["tables"] = dense_tables(cache)
            own = np.full((cache.pool.slot_count, 2), -1, dtype=np.int64)
            for s, k in enumerate(cache.pool.owner):
                if k is not None:
                    own[s] = (k.lod, key_linear(cache, k))
            d["owner"] = own
            d["last_used"] = cache.pool.last_used.copy()
            d["n_free"] = np.int64(len(cache.pool._free))
            d["cache_frame"] = np.int64(cache.frame)
            ents = sorted(
                (e.key.lod, key_linear(cache, e.key), e.base, e.hits) for e in sess.table._entries.values()
            )
            d["entries"] = np.array(ents, dtype=np.int64).reshape(-1, 4)
            reps = captured["reports"] or {}
            d["reports"] = np.array(
                sorted((k.lod, key_linear(cache, k), c) for k, c in reps.items()), dtype=np.int64
            ).reshape(-1, 3)
            bat = captured["batch"] or []
            d["batch"] = np.array([(k.lod, key_linear(cache, k)) for k in bat], dtype=np.int64).reshape(-1, 2)
        frames[f] = d
    sess.close()
    return frames, ops, macro_dump


def capture_ops(sess):
    """Run one frame with the four kernel passes wrapped; keep a few calls each."""
    store = {"raygen": [], "advance": [], "probe": [], "shade": []}
    orig = {k: getattr(kernels, f"{k}_pass") for k in store}

    def snap(args):
        return [np.array(a, copy=True) if isinstance(a, np.ndarray) else a for a in args]

    def mk(name):
        def fn(*args):
            pre = snap(args)
            ret = orig[name](*args)
            post = snap(args)
            if len(store[name]) < 2:
                store[name].append((pre, post, ret))
            return ret

        return fn

    for k in store:
        setattr(kernels, f"{k}_pass", mk(k))
    try:
        img, rec = sess.render_frame()
    finally:
        for k in store:
            setattr(kernels, f"{k}_pass", orig[k])
    flat = {}
    for name, calls in store.items():
        for ci, (pre, post, ret) in enumerate(calls):
            for ai, (a, b) in enumerate(zip(pre, post)):
                if isinstance(a, np.ndarray):
                    flat[f"{name}{ci}_in{ai}"] = a
                    flat[f"{name}{ci}_out{ai}"] = b
                else:
                    flat[f"{name}{ci}_in{ai}"] = np.asarray(a)
            if ret is not None:
                flat[f"{name}{ci}_ret"] = np.asarray(ret)
    return img, rec, flat


def save_session(name, spec, op_frame=None):
    frames, ops, macro_dump = run_session(spec, op_frame)
    out = {}
    for f, d in frames.items():
        for k, v in d.items():
            out[f"f{f}_{k}"] = v
    out["macro_vmin"] = macro_dump["vmin"]
    out["macro_vmax"] = macro_dump["vmax"]
    np.savez_compressed(HERE / f"session_{name}.npz", **out)
    if ops:
        np.savez_compressed(HERE / f"ops_{name}.npz", **ops)
    print(name, "frames", len(frames), "bytes", (HERE / f"session_{name}.npz").stat().st_size)


def save_inr():
    out = {}
    # default INR (config 1 recipe) and a tiny odd-shaped one
    for tag, grid, mlp_cfg in (
        ("default", HashGridConfig(), MLPConfig()),
        ("tiny", HashGridConfig(levels=3, features_per_entry=3, base_resolution=5, growth_factor=1.7, table_size=64),
         MLPConfig(hidden_width=12, hidden_layers=3, output_activation="clamp")),
    ):
        m = ref_inr_model((64, 64, 64), grid=grid, mlp=mlp_cfg)
        pos = np.random.default_rng(5).random((4096, 3))
        out[f"{tag}_pos"] = pos
        out[f"{tag}_infer"] = m.infer_batch(pos)
        out[f"{tag}_field"] = m.as_field().sample_batch(pos)
        out[f"{tag}_encode"] = encoding.encode(m.grid_config, m.tables, pos[:512])
        out[f"{tag}_resolutions"] = np.array(m.grid_config.resolutions())
        for i, p in enumerate(m.parameters()):
            if p.size <= 4096:
                out[f"{tag}_param{i}"] = p
            out[f"{tag}_param{i}_sha"] = np.frombuffer(hashlib.sha256(p.tobytes()).digest(), dtype=np.uint8)
        # a brick decode through fulfill (scheduler.py:127-134)
        from voxcache.cache import BrickLayout

        lay = BrickLayout((64, 64, 64), 16)
        for key in (BrickKey(1, (1, 0, 1)), BrickKey(0, (4, 4, 4))):
            out[f"{tag}_brick_{key.lod}_{key.index[0]}{key.index[1]}{key.index[2]}"] = fulfill([key], lay, m.as_field())[0].samples
    # un-redrawn seed-0 model (near 0.5 everywhere) to pin the init sequence
    m0 = ref_inr_model((32, 32, 32), redraw=None)
    for i, p in enumerate(m0.parameters()):
        out[f"seed0_param{i}_sha"] = np.frombuffer(hashlib.sha256(p.tobytes()).digest(), dtype=np.uint8)
    np.savez_compressed(HERE / "inr.npz", **out)


def save_fields():
    out = {}
    pos = np.random.default_rng(17).random((3000, 3))
    out["pos"] = pos
    for kind in ("sphere", "shells", "marschner_lobb_like"):
        out[kind] = make_procedural(kind, (32, 32, 32)).sample_batch(pos)
    lat = ref_lattice_field((20, 24, 28), 4)
    out["lattice_values"] = lat.sample_batch(pos)
    out["lattice"] = lat.lattice
    # macro grid + majorants for a TF (macrocell.py:49-128)
    mg = macrocell.build(lat, lat.domain.dims, 8)
    for tname, tf in (("warm", warm_body(0.45, 0.9)), ("gray", grayscale_ramp(0.7))):
        macrocell.update_majorants(mg, tf)
        out[f"major_{tname}"] = mg.majorant.copy()
        out[f"lut_{tname}"] = tf.lookup_table()
    out["macro_vmin"] = mg.value_min
    out["macro_vmax"] = mg.value_max
    np.savez_compressed(HERE / "fields.npz", **out)


def save_brickmath():
    from voxcache.cache import BrickLayout

    out = {}
    cases = [((64, 64, 64), 16), ((512, 512, 512), 16), ((4096, 4096, 4096), 40), ((4096,) * 3, 16),
             ((1000, 600, 300), 17), ((40, 48, 56), 10), ((130, 130, 130), 8), ((2048,) * 3, 16)]
    for ci, (dims, b) in enumerate(cases):
        lay = BrickLayout(dims, b)
        out[f"c{ci}_dims"] = np.array(dims)
        out[f"c{ci}_b"] = np.int64(b)
        out[f"c{ci}_grids"] = np.array(lay.grids, dtype=np.int64)
        rng = np.random.default_rng(ci)
        pos = rng.uniform(-2, np.array(dims) + 1, size=(500, 3))
        for lod in range(min(lay.max_lod + 1, 4)):
            idx, local = lay.locate(pos, lod)
            out[f"c{ci}_pos"] = pos
            out[f"c{ci}_idx{lod}"] = idx
            out[f"c{ci}_local{lod}"] = local
        keys = [BrickKey(l, tuple(int(rng.integers(0, g)) for g in lay.grids[l])) for l in range(lay.max_lod + 1)]
        out[f"c{ci}_keys"] = np.array([(k.lod, *k.index) for k in keys], dtype=np.int64)
        out[f"c{ci}_origins"] = np.array([lay.origin(k) for k in keys], dtype=np.int64)
        if b <= 17:
            nat, norm = lay.sample_positions(keys[min(1, len(keys) - 1)])
            out[f"c{ci}_native"] = nat
            out[f"c{ci}_normalized"] = norm
    np.savez_compressed(HERE / "brickmath.npz", **out)


def save_rng():
    from voxcache.sampler import XorShift32, effective_lod_scale, force_max_scale, splitmix64

    out = {}
    out["splitmix_in"] = np.array([0, 1, 2**63, 0xDEADBEEF, 2**64 - 1], dtype=np.uint64)
    out["splitmix_out"] = splitmix64(out["splitmix_in"])
    x = XorShift32(seed=3, frame=7, lanes=1000)
    out["xs_state0"] = x.state.copy()
    u = [x.uniform(1000 - 100 * i) for i in range(5)]
    out["xs_u"] = np.concatenate(u)
    out["xs_state5"] = x.state.copy()
    pol = LodPolicy(lod_scale=1.2, preload_frames=20)
    out["eff"] = np.array([effective_lod_scale(pol, f, force_max_scale(6, 1.3)) for f in range(25)])
    np.savez_compressed(HERE / "rng.npz", **out)


def main(only=()):
    if not only:
        save_brickmath()
        save_rng()
        save_fields()
        save_inr()
    for name, spec in specs.SESSION_SPECS.items():
        if not only or name in only:
            save_session(name, spec, op_frame=spec.get("op_frame"))


if __name__ == "__main__":
    assert "voxcache" in sys.modules and os.path.isdir("/root/reference")
    main(tuple(sys.argv[1:]))  # optional: only these session names
