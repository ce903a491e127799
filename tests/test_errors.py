"""Error semantics at the boundary (vc/errors.py): the same exception
types as the reference for out-of-domain positions (fields.py:71-80), non-finite
model outputs (model.py:71-74) and failed true-miss inference in a frame
(sampler.py:149-152)."""

import numpy as np
import pytest


def test_out_of_domain_positions_raise_domain_error():
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200.errors import DomainError
    from paper_2504_18001_b200.fields import check_positions

    for bad in ([[0.5, 0.5, 1.0]], [[-1e-9, 0.2, 0.2]], [[0.1, 0.2]]):
        with pytest.raises(DomainError):
            check_positions(np.asarray(bad, dtype=np.float64))
    assert check_positions(np.asarray([[0.0, 0.5, np.nextafter(1.0, 0.0)]])).shape == (1, 3)
    # like the reference's comparisons, NaN coordinates are not rejected here
    assert check_positions(np.asarray([[np.nan, 0.5, 0.5]])).shape == (1, 3)
    assert issubclass(DomainError, P.VoxcacheError)


def _nan_model():
    import paper_2504_18001_b200 as P

    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((32, 32, 32)), seed=0)
    params = [np.asarray(p).copy() for p in m.parameters()]
    params[-1][...] = np.nan  # output bias: every inference is non-finite
    m.set_parameters(params)
    return m


@pytest.mark.gpu
def test_non_finite_inference_raises_model_corrupt_error():
    import torch

    from paper_2504_18001_b200.errors import ModelCorruptError

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    with pytest.raises(ModelCorruptError):
        _nan_model().as_field().sample_batch(np.full((64, 3), 0.5))


@pytest.mark.gpu
def test_failed_miss_inference_in_a_frame_raises_render_error():
    import torch

    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200.errors import RenderError
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=48, height=48)
    grid = np.zeros((2, 2, 2), np.float32)
    from paper_2504_18001_b200.macrocell import MacroCellGrid

    macro = MacroCellGrid(16, (32, 32, 32), (2, 2, 2), grid, grid + 1.0, np.ones_like(grid))
    cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(2, 2, 2)),
                        policy=P.LodPolicy(1.0, 2), seed=0)
    sess = RenderSession(_nan_model().as_field(), P.warm_body(0.3, 0.9), traj.camera_at(0), cfg, macro=macro,
                         debug=True)
    for attempt in range(2):
        with pytest.raises(RenderError):
            sess.render_frame()  # frame 0: every sample is a true miss
        # the reference raises before _maintenance (sampler.py:149-152, session.py:107-112):
        # neither clock advanced, no miss report was drained into the request table, no
        # batch was dispatched, nothing was inserted
        assert sess.frame == 0 and sess.cache.frame == 0, attempt
        st = sess.debug_state()
        assert st["entries"].shape[0] == 0 and st["batch"].shape[0] == 0, attempt
        assert (st["tables"] < 0).all() and (st["owner"] < 0).all(), attempt
        assert int(sess.cache.miss_count.sum().item()) > 0  # the frame's reports wait, undrained


def test_param_fingerprint_sees_in_place_edits():
    """The device copy of a model is keyed on its parameters' content."""
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200.device import _param_fingerprint

    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((16, 16, 16)), seed=0)
    a = _param_fingerprint(m)
    assert _param_fingerprint(m) == a
    m.tables[0][0, 0] += 1.0  # in place, same array object
    assert _param_fingerprint(m) != a


def test_trainer_rejects_non_float32_models():
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200.errors import ConfigError
    from paper_2504_18001_b200.train import train

    class F64Model:  # a reference InrModel built with dtype=np.float64 (duck typed)
        grid_config, mlp_config, dtype = P.HashGridConfig(), P.MLPConfig(), np.dtype(np.float64)

    with pytest.raises(ConfigError):
        train(F64Model(), P.make_procedural("sphere", (16, 16, 16)), steps=1)
