"""Golden vectors for a wide MLP (hidden_width 128, the GPU path's limit): the
UNMODIFIED reference's InrModel.infer_batch / InrField.sample_batch at 4096 points.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_wide_inr.py
"""

from pathlib import Path

import numpy as np
from voxcache.fields import FieldDomain
from voxcache.inr import HashGridConfig, InrModel, MLPConfig

HERE = Path(__file__).resolve().parent


def main():
    out = {}
    for tag, mlp in (("w128", MLPConfig(hidden_width=128, hidden_layers=2)),
                     ("w64x3", MLPConfig(hidden_width=64, hidden_layers=3, output_activation="clamp"))):
        m = InrModel(HashGridConfig(), mlp, FieldDomain((64, 64, 64)), seed=0)
        r = np.random.default_rng(42)
        # smaller redraw range than the default recipe: a 128-wide layer of +-0.7 weights
        # saturates the sigmoid everywhere
        m.set_parameters([r.uniform(-0.2, 0.2, size=p.shape).astype(np.float32) for p in m.parameters()])
        pos = np.random.default_rng(5).random((4096, 3))
        out[f"{tag}_pos"] = pos
        out[f"{tag}_infer"] = m.infer_batch(pos)
        out[f"{tag}_field"] = m.as_field().sample_batch(pos)
    np.savez_compressed(HERE / "inr_wide.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
