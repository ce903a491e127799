"""Writes tests/golden/tiny_model.cinr with the REFERENCE's own save_weights
(voxcache/inr/weights_io.py:63-73), a small INR + macro grid, plus the parameters
as .npz, so the product's .cinr reader/writer is pinned against real files.

Run in the container that has /root/reference:
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_cinr.py
"""
from pathlib import Path

import numpy as np
from voxcache.fields import FieldDomain, make_procedural
from voxcache.inr import HashGridConfig, InrModel, MLPConfig
from voxcache.inr.weights_io import save_weights
from voxcache import macrocell

out = Path(__file__).resolve().parent
model = InrModel(HashGridConfig(levels=3, features_per_entry=2, base_resolution=4, growth_factor=1.5, table_size=64),
                 MLPConfig(hidden_width=8, hidden_layers=2), FieldDomain((24, 20, 16), (0.0, 2.0)), seed=3)
r = np.random.default_rng(5)
model.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in model.parameters()])
macro = macrocell.build(make_procedural("sphere", (24, 20, 16)), (24, 20, 16), 8)
save_weights(model, out / "tiny_model.cinr", macro)
np.savez(out / "tiny_model_params.npz", *[np.asarray(p) for p in model.parameters()],
         vmin=macro.value_min, vmax=macro.value_max)
print("wrote", out / "tiny_model.cinr")
