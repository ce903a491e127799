"""INR training on the GPU against the reference's own training
runs (tests/golden/make_train.py): the same PCG64 batches, loss trace and final
parameters within tolerance (f32 gradient sums in a different order), and the
reference's divergence semantics."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "adam": dict(steps=24, batch_size=4096, learning_rate=1e-2, optimizer="adam", seed=3, clip_norm=None),
    "adam_2": dict(steps=2, batch_size=4096, learning_rate=1e-2, optimizer="adam", seed=3, clip_norm=None),
    "sgd_clip": dict(steps=12, batch_size=2048, learning_rate=0.5, optimizer="sgd", seed=4, clip_norm=0.05),
    "adam_clip": dict(steps=12, batch_size=3000, learning_rate=3e-3, optimizer="adam", seed=5, clip_norm=0.02),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _setup():
    import paper_2504_18001_b200 as P
    from scene_specs import smoothed_random_lattice

    dims = (32, 32, 32)
    field = P.RawLatticeField(smoothed_random_lattice(dims, 9), P.FieldDomain(dims))
    model = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain(dims), seed=0)
    return model, field


@pytest.mark.parametrize("name", list(CASES))
def test_training_matches_reference(name):
    from conftest import load_golden
    from paper_2504_18001_b200.train import psnr_on_lattice, train

    g = load_golden("train.npz")
    model, field = _setup()
    res = train(model, field, **CASES[name])
    ref = g[f"{name}_loss"]
    rel = np.abs(res.loss_trace - ref) / ref
    print(name, "loss", res.loss_trace[[0, -1]], "ref", ref[[0, -1]], "max rel", rel.max())
    assert rel[0] <= 1e-5, "step-0 loss (same batch, same initial model) differs"
    assert rel.max() <= 2e-3
    params = res.model.parameters()
    nt = len(res.model.tables)
    diffs = []
    for i, p in enumerate(params):
        want = g[f"{name}_p{i}"]
        got = p[g[f"{name}_p{i}_rows"]] if i < nt else p
        diffs.append(np.abs(got - want).ravel())
        if i < nt:
            s = float(np.sum(p, dtype=np.float64))
            assert abs(s - float(g[f"{name}_p{i}_sum"])) <= 1e-3 * max(1.0, abs(s)), f"table {i} sum"
    d = np.concatenate(diffs)
    worst = float(d.max())
    # Adam normalises each gradient: where a parameter's gradient nearly cancels, the f32
    # summation order can flip its sign and move that parameter by up to 2*lr per step
    lr, steps = CASES[name]["learning_rate"], CASES[name]["steps"]
    bound = 2 * lr * steps if CASES[name]["optimizer"] == "adam" else 1e-4
    # after 24 steps at lr 1e-2 the trajectories have drifted apart a little (2% of the
    # parameters by > 1e-4, same loss and PSNR); the short and clipped runs stay within 1e-6
    frac = 0.05 if steps > 16 else 0.01
    print(name, "fraction > 1e-4:", float((d > 1e-4).mean()), "worst", worst)
    assert float((d > 1e-4).mean()) <= frac, f"{(d > 1e-4).mean():.4f} of parameters off by > 1e-4"
    assert worst <= bound
    ps = psnr_on_lattice(res.model, field)
    print(name, "worst param diff", worst, "psnr", ps, "ref", float(g[f"{name}_psnr"]))
    assert abs(ps - float(g[f"{name}_psnr"])) <= 0.05


def test_training_divergence_keeps_last_finite_step():
    """train.py:123-127: a non-finite loss raises TrainingDivergedError with the trace so far."""
    from paper_2504_18001_b200.errors import TrainingDivergedError
    from paper_2504_18001_b200.train import train

    model, field = _setup()
    with pytest.raises(TrainingDivergedError) as ei:
        train(model, field, steps=6, batch_size=1024, learning_rate=1e30, optimizer="sgd", seed=1)
    e = ei.value
    assert e.last_finite_step is not None and len(e.loss_trace) == e.last_finite_step + 1
    assert np.isfinite(e.loss_trace).all()


def test_training_reduces_loss_at_scale():
    """The default batch (65536) for 100 steps: the loss falls and PSNR rises."""
    from paper_2504_18001_b200.train import psnr_on_lattice, train

    model, field = _setup()
    p0 = psnr_on_lattice(model, field)
    res = train(model, field, steps=100, seed=7)
    assert res.final_loss < 0.5 * res.loss_trace[0]
    assert psnr_on_lattice(res.model, field) > p0 + 3.0


def test_loss_and_grads_matches_reference():
    """train.py:16-37 on one batch: the reference's loss and every parameter gradient."""
    from conftest import load_golden
    from paper_2504_18001_b200.train import loss_and_grads

    g = load_golden("train.npz")
    model, _ = _setup()
    loss, grads = loss_and_grads(model, g["lg_pos"], g["lg_targets"])
    assert abs(loss - float(g["lg_loss"])) <= 1e-6 * float(g["lg_loss"])
    nt = len(model.tables)
    for i, gr in enumerate(grads):
        assert gr.dtype == np.float32 and gr.shape == model.parameters()[i].shape
        if i < nt:
            np.testing.assert_allclose(gr[g[f"lg_g{i}_rows"]], g[f"lg_g{i}"], rtol=1e-4, atol=1e-9)
            assert abs(float(np.abs(gr).sum(dtype=np.float64)) - float(g[f"lg_g{i}_sum"])) <= 1e-4 * float(
                g[f"lg_g{i}_sum"]) + 1e-9
        else:
            want = g[f"lg_g{i}"]
            np.testing.assert_allclose(gr, want, rtol=1e-4, atol=1e-6 * float(np.abs(want).max()))


def test_loss_and_grads_finite_differences():
    """test_inr.py:139-160's check in f32 on the default network (randomised weights so the
    ReLUs are not all at their kinks): central differences of the GPU loss against the GPU
    gradient at the largest-gradient entry of every parameter array."""
    from gpu_runner import product_inr
    from paper_2504_18001_b200.train import loss_and_grads

    model = product_inr((32, 32, 32))
    rng = np.random.default_rng(0)
    pos = rng.random((256, 3))
    targets = rng.random(256).astype(np.float32)
    _, grads = loss_and_grads(model, pos, targets)
    eps = 1e-3
    worst = 0.0
    params = model.parameters()
    for i, gr in enumerate(grads):
        k = int(np.argmax(np.abs(gr).reshape(-1)))
        flat = params[i].reshape(-1)
        orig = flat[k]
        flat[k] = orig + eps
        model.set_parameters(params)
        lp, _ = loss_and_grads(model, pos, targets)
        flat[k] = orig - eps
        model.set_parameters(params)
        lm, _ = loss_and_grads(model, pos, targets)
        flat[k] = orig
        model.set_parameters(params)
        fd = (lp - lm) / (2 * eps)
        gv = float(gr.reshape(-1)[k])
        print("fd check", i, k, fd, gv)
        worst = max(worst, abs(fd - gv) / max(abs(fd), abs(gv), 1e-6))
    assert worst <= 2e-2, worst
