"""CUDA path vs the reference (golden fixtures) and the CPU oracle — needs a B200."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402
from oracle_runner import oracle_state, record_array, run_oracle_session  # noqa: E402
from scene_specs import SESSION_SPECS  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_18001_b200 import _native

    _native.load()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _replay_gpu(name, ops, ci):
    from paper_2504_18001_b200 import plugin

    fn = {"raygen": plugin.raygen_pass, "advance": plugin.advance_pass, "probe": plugin.probe_pass,
          "shade": plugin.shade_pass}[name]
    args = []
    ai = 0
    while f"{name}{ci}_in{ai}" in ops:
        a = ops[f"{name}{ci}_in{ai}"]
        args.append(a.copy() if a.ndim else a.item())
        ai += 1
    ret = fn(*args)
    for ai in range(len(args)):
        if f"{name}{ci}_out{ai}" in ops:
            want = ops[f"{name}{ci}_out{ai}"]
            if name == "shade" and ai in (7, 8):
                # color/trans go through 1-(1-a)^r (kernels.py:348).  glibc's pow misrounds
                # ~7e-4 of these inputs (checked against 50-digit decimal); the device pow is
                # correctly rounded, and 1-pow cancels, so allow a 1e-11 relative f64 gap
                # here (the f32 image and every cache decision stay identical)
                np.testing.assert_allclose(args[ai], want, rtol=1e-11, atol=0, err_msg=f"{name}{ci} arg {ai}")
            else:
                np.testing.assert_array_equal(args[ai], want, err_msg=f"{name}{ci} arg {ai}")
    if f"{name}{ci}_ret" in ops:
        np.testing.assert_array_equal(np.asarray(ret), ops[f"{name}{ci}_ret"])


@pytest.mark.parametrize("name", ["raygen", "advance", "probe", "shade"])
def test_operator_passes_bit_exact_vs_reference(name):
    """Stage A: the four C-ABI passes on the reference's own recorded inputs."""
    ops = load_golden("ops_lattice64.npz")
    n = 0
    for ci in range(3):
        if f"{name}{ci}_in0" in ops:
            _replay_gpu(name, ops, ci)
            n += 1
    assert n >= 1


EXACT = ["lattice64", "lattice64_paged", "lattice64_fifo", "aniso_b10", "events", "pressure", "pressure_fifo",
         "pt_lattice64", "pt_pressure", "pt_aniso"]


@pytest.mark.parametrize("name", EXACT)
def test_session_bit_exact_vs_reference(name):
    """Stage B: per-frame page tables, owners, stamps, request table, miss reports,
    dispatched batch, FrameRecord and image equal the reference's."""
    from gpu_runner import run_gpu_session

    g = load_golden(f"session_{name}.npz")
    for f, img, rec, sess in run_gpu_session(name, macro=(g["macro_vmin"], g["macro_vmax"])):
        got = np.array([rec.frame, rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits, rec.bricks_loaded,
                        rec.bricks_loaded_total, rec.requests_inflight], dtype=np.int64)
        np.testing.assert_array_equal(got, g[f"f{f}_record"], err_msg=f"frame {f} record")
        st = sess.debug_state()
        for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
            np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")
        assert st["n_free"] == int(g[f"f{f}_n_free"])
        assert st["cache_frame"] == int(g[f"f{f}_cache_frame"])
        assert rec.occupancy == pytest.approx(float(g[f"f{f}_occupancy"]), abs=0)
        diff = np.abs(img - g[f"f{f}_img"]).max()
        assert diff <= 1e-6, f"frame {f} image max abs diff {diff}"


@pytest.mark.parametrize("name", ["pressure", "events", "lattice64_fifo"])
def test_maintenance_launch_modes_bit_exact_vs_reference(name):
    """The maintenance replayed as one CUDA graph and launched kernel by kernel (the
    mode the session does not use by default) give the reference's state every frame
    (eviction, deferral, TF switch + reset events, FIFO)."""
    from gpu_runner import run_gpu_session
    g = load_golden(f"session_{name}.npz")
    for graph in (True, False):
        for f, img, rec, sess in run_gpu_session(name, macro=(g["macro_vmin"], g["macro_vmax"]), maint_graph=graph):
            st = sess.debug_state()
            for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
                np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"graph={graph} frame {f} {k}")
            assert np.abs(img - g[f"f{f}_img"]).max() <= 1e-6, f"graph={graph} frame {f}"


@pytest.mark.parametrize("name", ["inr64", "inr_uncached", "pt_inr", "pt_inr_uncached"])
def test_session_inr_vs_reference(name):
    """Random-init hash-grid INR: images within 1e-3 abs (>= 60 dB), cache state bit-exact."""
    from gpu_runner import run_gpu_session

    g = load_golden(f"session_{name}.npz")
    cached = SESSION_SPECS[name].get("cached", True)
    for f, img, rec, sess in run_gpu_session(name, macro=(g["macro_vmin"], g["macro_vmax"])):
        ref = g[f"f{f}_img"]
        diff = np.abs(img - ref).max()
        mse = float(np.mean((img[..., :3] - ref[..., :3]) ** 2))
        psnr = 10 * np.log10(1.0 / mse) if mse > 0 else np.inf
        assert diff <= 1e-3 and psnr >= 60.0, f"frame {f}: max {diff}, psnr {psnr}"
        if cached:
            st = sess.debug_state()
            for k in ("tables", "owner", "entries", "batch"):
                np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")


def test_inr_decode_vs_reference():
    import paper_2504_18001_b200 as P
    from gpu_runner import product_inr

    g = load_golden("inr.npz")
    m = product_inr((64, 64, 64))
    pos = g["default_pos"]
    np.testing.assert_allclose(m.infer_batch(pos), g["default_infer"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(m.as_field().sample_batch(pos), g["default_field"], atol=1e-5, rtol=0)
    tiny = P.InrModel(P.HashGridConfig(levels=3, features_per_entry=3, base_resolution=5, growth_factor=1.7,
                                       table_size=64),
                      P.MLPConfig(hidden_width=12, hidden_layers=3, output_activation="clamp"),
                      P.FieldDomain((64, 64, 64)), seed=0)
    r = np.random.default_rng(42)
    tiny.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in tiny.parameters()])
    np.testing.assert_allclose(tiny.infer_batch(g["tiny_pos"]), g["tiny_infer"], atol=1e-5, rtol=0)


@pytest.mark.parametrize("tag", ["w128", "w64x3"])
def test_wide_inr_decode_vs_reference(tag):
    """Wider MLPs than the default (the reference's MLPConfig.hidden_width is free):
    width 128 x 2 and 64 x 3 hidden layers through the generic decoder and inside a
    frame (true misses of an uncached session) against the reference's outputs."""
    import paper_2504_18001_b200 as P

    g = load_golden("inr_wide.npz")
    mlp = (P.MLPConfig(hidden_width=128, hidden_layers=2) if tag == "w128"
           else P.MLPConfig(hidden_width=64, hidden_layers=3, output_activation="clamp"))
    m = P.InrModel(P.HashGridConfig(), mlp, P.FieldDomain((64, 64, 64)), seed=0)
    r = np.random.default_rng(42)
    m.set_parameters([r.uniform(-0.2, 0.2, size=p.shape).astype(np.float32) for p in m.parameters()])
    pos = g[f"{tag}_pos"]
    np.testing.assert_allclose(m.infer_batch(pos), g[f"{tag}_infer"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(m.as_field().sample_batch(pos), g[f"{tag}_field"], atol=1e-5, rtol=0)
    # the same network as the true-miss decoder of both frame schedules
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=48, height=48)
    imgs = []
    for march in ("parity", "throughput"):
        cfg = SessionConfig(cached=False, loader="inline", policy=P.LodPolicy(1.2, 0), seed=0)
        s = RenderSession(m.as_field(), P.grayscale_ramp(0.8), traj.camera_at(3), cfg, march=march)
        img, rec = s.render_frame()
        assert rec.true_misses == rec.samples > 0
        imgs.append(img)
    np.testing.assert_array_equal(imgs[0], imgs[1])  # uncached: no RNG, same values


def test_brick_decode_into_pool_layout():
    """vcb_field_bricks writes [slot][z][y][x] exactly like pool.store (P15)."""
    from gpu_runner import product_inr
    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.cache import BrickLayout
    from paper_2504_18001_b200.device import device_field, ptr

    g = load_golden("inr.npz")
    m = product_inr((64, 64, 64))
    lay = BrickLayout((64, 64, 64), 16)
    keys = []
    refs = []
    for k in [k for k in g if k.startswith("default_brick_")]:
        lod = int(k.split("_")[2])
        idx = [int(c) for c in k.split("_")[3]]
        keys.append(lay.offsets[lod] + idx[0] + lay.grids[lod][0] * (idx[1] + lay.grids[lod][1] * idx[2]))
        refs.append(g[k])
    kt = _dev(np.array(keys, dtype=np.int64))
    out = torch.empty(len(keys) * 16 ** 3, dtype=torch.float32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    geom = lay.geom()
    df = device_field(m.as_field())
    N.call("vcb_field_bricks", C.byref(df.desc), C.byref(geom), len(keys), ptr(kt), ptr(out), ptr(flag), 0)
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy().reshape(len(keys), -1), np.stack(refs), atol=1e-5, rtol=0)


def test_fields_vs_reference():
    import paper_2504_18001_b200 as P

    g = load_golden("fields.npz")
    lat = P.RawLatticeField(g["lattice"], P.FieldDomain((20, 24, 28)))
    np.testing.assert_array_equal(lat.sample_batch(g["pos"]), g["lattice_values"])
    for kind in ("sphere", "shells", "marschner_lobb_like"):
        np.testing.assert_allclose(P.make_procedural(kind, (32, 32, 32)).sample_batch(g["pos"]), g[kind], atol=1e-6)


def test_macro_build_vs_reference():
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import macrocell

    g = load_golden("fields.npz")
    lat = P.RawLatticeField(g["lattice"], P.FieldDomain((20, 24, 28)))
    mg = macrocell.build(lat, (20, 24, 28), 8)
    np.testing.assert_array_equal(mg.value_min, g["macro_vmin"])
    np.testing.assert_array_equal(mg.value_max, g["macro_vmax"])
    s = load_golden("session_inr64.npz")
    from gpu_runner import product_inr

    mi = macrocell.build(product_inr((64, 64, 64)).as_field(), (64, 64, 64), 16)
    np.testing.assert_allclose(mi.value_min, s["macro_vmin"], atol=1e-5)
    np.testing.assert_allclose(mi.value_max, s["macro_vmax"], atol=1e-5)


@pytest.mark.parametrize("seed", [0, 1])
def test_session_vs_oracle_random_scene(seed):
    """Fresh seeded scenes (not in the golden set): CUDA path == CPU oracle, bit for bit."""
    import scene_specs
    from gpu_runner import run_gpu_session

    rng = np.random.default_rng(100 + seed)
    name = f"_rand{seed}"
    scene_specs.SESSION_SPECS[name] = dict(
        field="lattice", field_seed=int(rng.integers(1000)), dims=(int(rng.integers(24, 70)),) * 3,
        tf=("warm_body", float(rng.uniform(0.3, 0.6)), 0.9), brick=int(rng.choice([4, 8, 12, 16])),
        pool=(2, 3, 2), sched_kw=dict(max_requests=int(rng.integers(2, 12)), ranking_enabled=bool(seed == 0)),
        policy=dict(lod_scale=float(rng.uniform(0.3, 2.0)), preload_frames=3,
                    mode=["corrected", "as_printed", "off"][seed % 3]),
        res=(48, 40), frames=10, cam_step=int(rng.integers(1, 12)), radius=float(rng.uniform(1.5, 2.5)),
    )
    try:
        gpu = run_gpu_session(name)
        cpu = run_oracle_session(name)
        for (f, img, rec, sess), (_, oimg, orec, osess) in zip(gpu, cpu):
            got = np.array([rec.frame, rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits,
                            rec.bricks_loaded, rec.bricks_loaded_total, rec.requests_inflight], dtype=np.int64)
            np.testing.assert_array_equal(got, record_array(orec), err_msg=f"frame {f}")
            st, ost = sess.debug_state(), oracle_state(osess)
            for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
                np.testing.assert_array_equal(st[k], ost[k], err_msg=f"frame {f} {k}")
            assert np.abs(img - oimg).max() <= 1e-6
    finally:
        scene_specs.SESSION_SPECS.pop(name, None)


@pytest.mark.parametrize("other", [1, 9])
def test_march_schedules_agree(other):
    """The persistent wavefront (default), the launch-per-iteration wavefront and
    the 512-thread build are schedules of the same arithmetic: identical images
    and cache state."""
    from gpu_runner import run_gpu_session

    g = load_golden("session_pressure.npz")
    m = (g["macro_vmin"], g["macro_vmax"])
    for (f, ia, ra, xa), (_, ib, rb, xb) in zip(run_gpu_session("pressure", macro=m, frames=8, impl=0),
                                               run_gpu_session("pressure", macro=m, frames=8, impl=other)):
        assert (ra.samples, ra.true_misses, ra.exact_hits) == (rb.samples, rb.true_misses, rb.exact_hits)
        np.testing.assert_array_equal(ia, ib)
        da, db = xa.debug_state(), xb.debug_state()
        for k in ("tables", "owner", "last_used", "entries", "batch"):
            np.testing.assert_array_equal(da[k], db[k])


def test_tensor_core_decoder_vs_reference():
    """tcgen05 MLP decoder (split-fp16, fp32 accumulate in TMEM) against the
    reference's INR outputs and the CUDA-core decoder."""
    from gpu_runner import product_inr
    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.cache import BrickLayout
    from paper_2504_18001_b200.device import device_field, ptr

    g = load_golden("inr.npz")
    m = product_inr((64, 64, 64))
    df = device_field(m.as_field())
    pos = np.concatenate([g["default_pos"], np.random.default_rng(9).random((70000, 3))])
    tp = _dev(pos)
    out_tc = torch.empty(len(pos), dtype=torch.float32, device="cuda")
    out_cc = torch.empty(len(pos), dtype=torch.float32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("vcb_inr_points_tc", C.byref(df.desc), len(pos), ptr(tp), ptr(out_tc), ptr(flag), 0)
    N.call("vcb_field_points", C.byref(df.desc), len(pos), ptr(tp), ptr(out_cc), ptr(flag), 0)
    tc, cc = out_tc.cpu().numpy(), out_cc.cpu().numpy()
    n0 = len(g["default_pos"])
    np.testing.assert_allclose(tc[:n0], g["default_field"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(tc, cc, atol=1e-5, rtol=0)
    # brick variant writes the pool layout
    lay = BrickLayout((64, 64, 64), 16)
    keys = []
    refs = []
    for k in [k for k in g if k.startswith("default_brick_")]:
        lod = int(k.split("_")[2])
        idx = [int(c) for c in k.split("_")[3]]
        keys.append(lay.offsets[lod] + idx[0] + lay.grids[lod][0] * (idx[1] + lay.grids[lod][1] * idx[2]))
        refs.append(g[k])
    kt = _dev(np.array(keys, dtype=np.int64))
    out = torch.empty(len(keys) * 16 ** 3, dtype=torch.float32, device="cuda")
    geom = lay.geom()
    N.call("vcb_inr_bricks_tc", C.byref(df.desc), C.byref(geom), len(keys), ptr(kt), ptr(out), ptr(flag), 0)
    np.testing.assert_allclose(out.cpu().numpy().reshape(len(keys), -1), np.stack(refs), atol=1e-5, rtol=0)


def test_update_majorants_on_device_matches_reference_rule():
    """vcb_update_majorants (macrocell.py:120-128 on the device) equals the numpy
    restatement (pinned to the reference by test_majorants_and_lut_vs_reference)
    bit for bit, on random grids with values on bin edges and out of [0, 1]."""
    import torch

    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.device import ptr

    r = np.random.default_rng(11)
    shape = (37, 41, 43)
    a = r.random(shape).astype(np.float32)
    b = r.random(shape).astype(np.float32)
    vmin, vmax = np.minimum(a, b), np.maximum(a, b)
    edges = r.random(shape) < 0.2
    vmin[edges] = np.floor(vmin[edges] * 256) / 256
    vmax[r.random(shape) < 0.05] = 1.25
    vmin[r.random(shape) < 0.05] = -0.5
    for tf in (P.warm_body(0.5, 0.9), P.grayscale_ramp(0.7), P.warm_body(0.35, 0.9)):
        grid = macrocell.MacroCellGrid(16, (1, 1, 1), shape[::-1], vmin, vmax, np.ones(shape, np.float32))
        want = macrocell.update_majorants(grid, tf).majorant
        d_min, d_max = torch.from_numpy(vmin).cuda(), torch.from_numpy(vmax).cuda()
        bm = torch.from_numpy(macrocell.opacity_bin_maxima(tf)).cuda()
        mu = torch.empty_like(d_min)
        N.call("vcb_update_majorants", ptr(d_min), ptr(d_max), d_min.numel(), ptr(bm), bm.numel(), ptr(mu), 0)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(mu.cpu().numpy(), want)


def test_results_do_not_depend_on_workspace_contents():
    """Every workspace is either written before it is read or cleared by the library:
    filling the maintenance and frame workspaces with garbage before every frame
    changes nothing (a stale decode-error flag once delayed the first insert)."""
    from gpu_runner import run_gpu_session

    g = load_golden("session_lattice64.npz")
    macro = (g["macro_vmin"], g["macro_vmax"])
    clean = [(rec.samples, rec.true_misses, rec.exact_hits, img.copy(), sess.debug_state()["tables"])
             for _, img, rec, sess in run_gpu_session("lattice64", macro=macro, frames=6)]
    dirty = []
    gen = run_gpu_session("lattice64", macro=macro, frames=6)
    for f, img, rec, sess in gen:
        dirty.append((rec.samples, rec.true_misses, rec.exact_hits, img.copy(), sess.debug_state()["tables"]))
        sess.cache.workspace.fill_(0xFF)
        if sess._ws is not None:
            sess._ws.fill_(0xA5)
    for a, b in zip(clean, dirty):
        assert a[:3] == b[:3]
        np.testing.assert_array_equal(a[3], b[3])
        np.testing.assert_array_equal(a[4], b[4])
