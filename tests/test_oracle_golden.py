"""Pins the CPU oracle to the real reference (CPU-only; fixtures recorded by
tests/golden/make_golden.py from voxcache itself)."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import cinr_oracle as O
from oracle_runner import oracle_state, record_array, run_oracle_session
from scene_specs import SESSION_SPECS, smoothed_random_lattice


def test_brickmath_golden():
    g = load_golden("brickmath.npz")
    ci = 0
    while f"c{ci}_dims" in g:
        dims = tuple(int(v) for v in g[f"c{ci}_dims"])
        b = int(g[f"c{ci}_b"])
        max_lod, grids = O.layout_grids(dims, b)
        np.testing.assert_array_equal(np.array(grids), g[f"c{ci}_grids"])
        pos = g[f"c{ci}_pos"]
        for lod in range(min(max_lod + 1, 4)):
            idx, local = O.locate(pos, b, lod, grids[lod])
            np.testing.assert_array_equal(idx, g[f"c{ci}_idx{lod}"])
            np.testing.assert_array_equal(local, g[f"c{ci}_local{lod}"])
        keys = g[f"c{ci}_keys"]
        for k, o in zip(keys, g[f"c{ci}_origins"]):
            np.testing.assert_array_equal(O.brick_origin(k[1:], b, int(k[0])), o)
        if f"c{ci}_native" in g:
            k = keys[min(1, len(keys) - 1)]
            nat, norm = O.brick_positions(dims, b, int(k[0]), k[1:])
            np.testing.assert_array_equal(nat, g[f"c{ci}_native"])
            np.testing.assert_array_equal(norm, g[f"c{ci}_normalized"])
        ci += 1
    assert ci >= 8


def test_rng_golden():
    g = load_golden("rng.npz")
    np.testing.assert_array_equal(O.splitmix64(g["splitmix_in"]), g["splitmix_out"])
    st = O.lane_seeds(3, 7, 1000)
    np.testing.assert_array_equal(st, g["xs_state0"])
    u = np.concatenate([O.xorshift_uniform(st, 1000 - 100 * i) for i in range(5)])
    np.testing.assert_array_equal(u, g["xs_u"])
    np.testing.assert_array_equal(st, g["xs_state5"])
    eff = [O.effective_scale(1.2, 20, f, (6 + 1.0) / 1.3) for f in range(25)]
    np.testing.assert_array_equal(np.array(eff), g["eff"])


def test_fields_and_macro_golden():
    g = load_golden("fields.npz")
    lat = O.LatticeField(g["lattice"])
    np.testing.assert_array_equal(lat.sample(g["pos"]), g["lattice_values"])
    np.testing.assert_array_equal(g["lattice"], smoothed_random_lattice((20, 24, 28), 4))
    vmin, vmax = O.macro_minmax(g["lattice"], 8)
    np.testing.assert_array_equal(vmin, g["macro_vmin"])
    np.testing.assert_array_equal(vmax, g["macro_vmax"])
    for name, pts in (("warm", O.warm_body_points(0.45, 0.9)), ("gray", O.grayscale_points(0.7))):
        np.testing.assert_array_equal(O.majorants(pts, vmin, vmax), g[f"major_{name}"])
        np.testing.assert_array_equal(O.tf_lut(pts), g[f"lut_{name}"])


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8)


@pytest.mark.parametrize("tag", ["default", "tiny"])
def test_inr_golden(tag):
    g = load_golden("inr.npz")
    if tag == "default":
        grid, mlp, sig = O.DEFAULT_GRID, O.DEFAULT_MLP, True
    else:
        grid = dict(levels=3, features_per_entry=3, base_resolution=5, growth_factor=1.7, table_size=64)
        mlp, sig = dict(hidden_width=12, hidden_layers=3), False
    t, w, b = O.inr_params_from_seed(grid, mlp)
    for i, p in enumerate(t + w + b):
        np.testing.assert_array_equal(_sha(p), g[f"{tag}_param{i}_sha"])
    fld = O.InrFieldOracle((64, 64, 64), t, w, b, grid, out_sigmoid=sig)
    np.testing.assert_array_equal(fld.res, g[f"{tag}_resolutions"])
    pos = g[f"{tag}_pos"]
    np.testing.assert_allclose(fld.encode(pos[:512]), g[f"{tag}_encode"], atol=2e-6, rtol=0)
    np.testing.assert_allclose(fld.infer(pos), g[f"{tag}_infer"], atol=2e-6, rtol=0)
    np.testing.assert_allclose(fld.sample(pos), g[f"{tag}_field"], atol=2e-6, rtol=0)
    for key in [k for k in g if k.startswith(f"{tag}_brick_")]:
        lod = int(key.split("_")[2])
        idx = [int(c) for c in key.split("_")[3]]
        _, norm = O.brick_positions((64, 64, 64), 16, lod, idx)
        np.testing.assert_allclose(fld.sample(norm), g[key], atol=2e-6, rtol=0)


def test_inr_seed0_init_sequence():
    g = load_golden("inr.npz")
    t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP, redraw=None)
    for i, p in enumerate(t + w + b):
        np.testing.assert_array_equal(_sha(p), g[f"seed0_param{i}_sha"])


def _replay(name, ops):
    """Feed recorded kernel-pass inputs to the oracle pass; outputs must be bit-identical."""
    fn = {"raygen": O.raygen_pass, "advance": O.advance_pass, "probe": O.probe_pass, "shade": O.shade_pass}[name]
    n_calls = 0
    for ci in range(3):
        if f"{name}{ci}_in0" not in ops:
            break
        args = []
        ai = 0
        while f"{name}{ci}_in{ai}" in ops:
            a = ops[f"{name}{ci}_in{ai}"]
            args.append(a.copy() if a.ndim else a.item())
            ai += 1
        ret = fn(*args)
        ai = 0
        while f"{name}{ci}_in{ai}" in ops:
            if f"{name}{ci}_out{ai}" in ops:
                np.testing.assert_array_equal(args[ai], ops[f"{name}{ci}_out{ai}"], err_msg=f"{name}{ci} arg {ai}")
            ai += 1
        if f"{name}{ci}_ret" in ops:
            np.testing.assert_array_equal(np.asarray(ret), ops[f"{name}{ci}_ret"])
        n_calls += 1
    return n_calls


@pytest.mark.parametrize("name", ["raygen", "advance", "probe", "shade"])
def test_kernel_passes_bit_exact(name):
    ops = load_golden("ops_lattice64.npz")
    assert _replay(name, ops) >= 1


EXACT = ["lattice64", "lattice64_paged", "lattice64_fifo", "aniso_b10", "events", "pressure", "pressure_fifo"]


@pytest.mark.parametrize("name", EXACT)
def test_session_state_bit_exact(name):
    g = load_golden(f"session_{name}.npz")
    macro = (g["macro_vmin"], g["macro_vmax"])
    for f, img, rec, sess in run_oracle_session(name, macro=macro):
        np.testing.assert_array_equal(record_array(rec), g[f"f{f}_record"], err_msg=f"frame {f} record")
        st = oracle_state(sess)
        for k in ("tables", "owner", "last_used", "entries", "reports", "batch"):
            np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")
        assert st["n_free"] == int(g[f"f{f}_n_free"]) and st["cache_frame"] == int(g[f"f{f}_cache_frame"])
        assert rec.occupancy == float(g[f"f{f}_occupancy"])
        np.testing.assert_array_equal(img, g[f"f{f}_img"], err_msg=f"frame {f} image")


@pytest.mark.parametrize("name", ["inr64", "inr_uncached"])
def test_session_inr_tolerance(name):
    g = load_golden(f"session_{name}.npz")
    macro = (g["macro_vmin"], g["macro_vmax"])
    same_state = 0
    frames = 0
    for f, img, rec, sess in run_oracle_session(name, macro=macro):
        frames += 1
        d = np.abs(img - g[f"f{f}_img"]).max()
        assert d <= 1e-3, f"frame {f} max abs {d}"
        if sess.cache is not None:
            st = oracle_state(sess)
            same_state += all(np.array_equal(st[k], g[f"f{f}_{k}"]) for k in ("tables", "owner", "entries", "batch"))
    if SESSION_SPECS[name].get("cached", True):
        assert same_state == frames
