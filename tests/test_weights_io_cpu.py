"""`.cinr` model files: the product reads the reference's own file (tests/golden/
tiny_model.cinr, written by voxcache.inr.weights_io.save_weights) and writes it
back byte for byte; defects raise WeightFormatError (weights_io.py:13-16)."""

import numpy as np
import pytest

from conftest import GOLDEN


def test_reads_reference_file_and_writes_it_back(tmp_path):
    from paper_2504_18001_b200.weights_io import load_weights, save_weights

    model, macro = load_weights(GOLDEN / "tiny_model.cinr")
    ref = np.load(GOLDEN / "tiny_model_params.npz")
    params = model.parameters()
    assert len(params) == len([k for k in ref.files if k.startswith("arr_")])
    for i, p in enumerate(params):
        np.testing.assert_array_equal(np.asarray(p), ref[f"arr_{i}"])
    assert model.domain.dims == (24, 20, 16) and model.domain.value_range == (0.0, 2.0)
    np.testing.assert_array_equal(macro.value_min, ref["vmin"])
    np.testing.assert_array_equal(macro.value_max, ref["vmax"])
    out = tmp_path / "again.cinr"
    save_weights(model, out, macro)
    assert out.read_bytes() == (GOLDEN / "tiny_model.cinr").read_bytes()


@pytest.mark.parametrize("cut", ["magic", "version", "truncated", "shapes"])
def test_defects_raise_weight_format_error(tmp_path, cut):
    from paper_2504_18001_b200.errors import WeightFormatError
    from paper_2504_18001_b200.weights_io import load_weights

    data = bytearray((GOLDEN / "tiny_model.cinr").read_bytes())
    if cut == "magic":
        data[:4] = b"XXXX"
    elif cut == "version":
        data[4] = 2
    elif cut == "truncated":
        data = data[:-5]
    else:
        data = data.replace(b'"params": [[', b'"params": [[9, ', 1)
        data[8:12] = (int.from_bytes(data[8:12], "little") + 3).to_bytes(4, "little")
    f = tmp_path / "bad.cinr"
    f.write_bytes(bytes(data))
    with pytest.raises(WeightFormatError):
        load_weights(f)
