"""Path tracing (render/pathtrace.py) beyond the recorded sessions:
the two numerical primitives the bit-exactness rests on, and the reference's own
statistical checks (test_render.py:171-244) on the GPU path."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def test_log1p_and_pcg64_match_numpy():
    """Device log1p == glibc's and device PCG64 draw d == numpy's d-th random()."""
    import ctypes

    import torch

    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.device import ptr
    from paper_2504_18001_b200.render import pcg64_seeded_state

    rng = np.random.default_rng(1)
    n = 1 << 21
    x = -rng.random(n)
    x[: 1 << 16] = -0.5 + (rng.random(1 << 16) - 0.5) * 1e-5  # near powers of two (|f| < 2^-20 path)
    x[1 << 16: 1 << 17] = -np.ldexp(rng.random(1 << 16), -rng.integers(20, 60, 1 << 16))  # tiny |x|
    seed = 123456789
    st, inc = pcg64_seeded_state(seed)
    idx = np.concatenate([np.arange(4096, dtype=np.uint64), rng.integers(0, 1 << 40, n - 4096, dtype=np.uint64)])
    ref_rng = np.random.default_rng(seed).random(4096)
    dx = torch.from_numpy(x).cuda()
    di = torch.from_numpy(idx).cuda()
    lg = torch.empty_like(dx)
    un = torch.empty_like(dx)
    pcg = np.array([st & (2**64 - 1), st >> 64, inc & (2**64 - 1), inc >> 64], dtype=np.uint64)
    N.call("vcb_debug_pt_math", n, ptr(dx), ptr(lg), pcg.ctypes.data, ptr(di), ptr(un), None)
    torch.cuda.synchronize()
    # the reference's np.log1p is libm's log1p on hosts without AVX-512; numpy dispatches to
    # SVML on AVX-512 hosts (1-ulp differences in ~7% of inputs), see make_golden.py
    libm = ctypes.CDLL("libm.so.6")
    libm.log1p.restype = ctypes.c_double
    libm.log1p.argtypes = [ctypes.c_double]
    want = np.fromiter((libm.log1p(float(v)) for v in x), dtype=np.float64, count=n)
    np.testing.assert_array_equal(lg.cpu().numpy(), want)
    u = un.cpu().numpy()
    np.testing.assert_array_equal(u[:4096], ref_rng)
    # arbitrary offsets against numpy's own jump (bit_generator.advance)
    for k in rng.integers(4096, n, 64):
        g = np.random.default_rng(seed)
        g.bit_generator.advance(int(idx[k]))
        assert u[k] == g.random()


def _flight_session(lattice, tf, density, cell=16, vminmax=None, **cfg_kw):
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    dims = tuple(int(x) for x in lattice.shape[::-1])
    fld = P.RawLatticeField(np.asarray(lattice, np.float32), P.FieldDomain(dims))
    macro = None
    if vminmax is not None:
        grid, _, _ = macrocell.layout(dims, cell)
        macro = macrocell.MacroCellGrid(cell, dims, grid, np.asarray(vminmax[0], np.float32),
                                        np.asarray(vminmax[1], np.float32), np.ones_like(vminmax[0], np.float32))
    cfg = SessionConfig(cached=False, loader="inline", settings=P.RenderSettings(pt_density=density),
                        macro_cell_size=cell, **cfg_kw)
    cam = P.Camera(position=(0.5, 0.5, -1.5), target=(0.5, 0.5, 0.5), width=8, height=8)
    return RenderSession(fld, tf, cam, cfg, macro=macro)


def test_trace_free_flight_bit_exact_vs_reference():
    """Golden vectors from the reference's trace_free_flight (tests/golden/make_pt_flight.py):
    same collisions, values and PCG64 draws consumed."""
    import paper_2504_18001_b200 as P
    from scene_specs import smoothed_random_lattice
    from conftest import load_golden

    g = load_golden("pt_flight.npz")
    sess = _flight_session(smoothed_random_lattice((32, 32, 32), 3), P.warm_body(0.4, 0.9), 30.0, cell=8,
                           vminmax=(g["vmin"], g["vmax"]))
    rng = np.random.default_rng(77)
    t_hit, v_hit = sess.trace_free_flight(g["o"], g["d"], g["t0"], g["t1"], rng)
    np.testing.assert_array_equal(t_hit, g["t_hit"])
    np.testing.assert_array_equal(v_hit, g["v_hit"])
    assert rng.random() == float(g["after"])  # the generator advanced by exactly the reference's draws
    assert int(sess._stats[0].item()) == int(g["requests"])


def _const_tf(alpha):
    import paper_2504_18001_b200 as P

    return P.TransferFunction([[0.0, 1, 1, 1, alpha], [1.0, 1, 1, 1, alpha]])


def test_mean_free_path_homogeneous():
    """test_render.py:179-191 / acceptance check 11: 1e6 rays into a constant medium."""
    mu = 40.0
    sess = _flight_session(np.ones((16, 16, 16), np.float32), _const_tf(1.0), mu)
    n = 1_000_000
    rng = np.random.default_rng(3)
    origins = np.column_stack([np.full(n, 1e-4), rng.uniform(0.3, 0.7, n), rng.uniform(0.3, 0.7, n)])
    t_hit, _ = sess.trace_free_flight(origins, np.array([1.0, 0.0, 0.0]), np.zeros(n), np.full(n, 1.0), rng)
    flights = t_hit[np.isfinite(t_hit)]
    assert len(flights) > 0.99 * n  # e^-40 escapes
    assert abs(flights.mean() - 1.0 / mu) / (1.0 / mu) <= 0.02


def test_slab_transmittance_within_3_sigma():
    """test_render.py:194-208."""
    sigma = 2.0
    slab = 1.0 - 1e-4
    sess = _flight_session(np.ones((16, 16, 16), np.float32), _const_tf(1.0), sigma)
    n = 100_000
    rng = np.random.default_rng(9)
    origins = np.column_stack([np.full(n, 1e-4), rng.uniform(0.2, 0.8, n), rng.uniform(0.2, 0.8, n)])
    t_hit, _ = sess.trace_free_flight(origins, np.array([1.0, 0.0, 0.0]), np.zeros(n), np.full(n, slab), rng)
    p_hat = np.isinf(t_hit).mean()
    p = np.exp(-sigma * slab)
    se = np.sqrt(p * (1 - p) / n)
    assert abs(p_hat - p) <= 3 * se


def _pt_session(field, tf, res, spp, seed, **settings):
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    cfg = SessionConfig(cached=False, mode="pathtrace", samples_per_pixel=spp, loader="inline",
                        settings=P.RenderSettings(**settings), seed=seed)
    cam = P.Camera(position=(0.5, 0.5, -1.3), target=(0.5, 0.5, 0.5), width=res, height=res)
    return RenderSession(field, tf, cam, cfg)


def test_pathtrace_zero_opacity_background():
    """test_render.py:171-176."""
    import paper_2504_18001_b200 as P

    sess = _pt_session(P.make_procedural("sphere", (16, 16, 16)), _const_tf(0.0), 32, 2, 0, background=(0.1, 0.2, 0.3))
    img, rec = sess.render_frame()
    np.testing.assert_allclose(img[..., :3], np.broadcast_to([0.1, 0.2, 0.3], img[..., :3].shape), atol=1e-6)
    assert (img[..., 3] == 0).all()


def test_pathtrace_variance_scales_inverse_n():
    """test_render.py:222-233: per-pixel variance over independent runs ~ 1/spp."""
    import paper_2504_18001_b200 as P

    tf = P.TransferFunction([[0.0, 1, 0.6, 0.3, 0.0], [1.0, 1, 0.8, 0.5, 0.7]])
    fld = P.make_procedural("sphere", (16, 16, 16))
    spps = [4, 16, 64]
    variances = []
    for spp in spps:
        runs = [_pt_session(fld, tf, 16, spp, 100 + i, pt_density=25.0).render_frame()[0][..., :3] for i in range(8)]
        variances.append(np.var(np.stack(runs), axis=0).mean())
    slope = np.polyfit(np.log(spps), np.log(variances), 1)[0]
    assert -1.35 <= slope <= -0.65, slope


def test_walk_schedules_agree():
    """The two-barrier walk (default) and the four-barrier walk (impl=1) are bit-identical."""
    from gpu_runner import run_gpu_session

    outs = []
    for impl in (0, 1):
        frames = []
        for f, img, rec, sess in run_gpu_session("pt_pressure", frames=4, impl=impl):
            frames.append((img.copy(), rec.samples, rec.true_misses, rec.exact_hits, sess.debug_state()["tables"]))
        outs.append(frames)
    for (a, b) in zip(*outs):
        np.testing.assert_array_equal(a[0], b[0])
        assert a[1:4] == b[1:4]
        np.testing.assert_array_equal(a[4], b[4])
