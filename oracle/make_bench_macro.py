"""Builds the macro-cell min/max grid of the bench volume (512^3 random-init INR,
config 2) with the CPU oracle, so the GPU arm and both CPU arms of bench.py
consume the identical grid (P16).  Output: bench_data/macro_inr512_c16.npz."""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import cinr_oracle as O  # noqa: E402

if __name__ == "__main__":
    V = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    t, w, b = O.inr_params_from_seed(O.DEFAULT_GRID, O.DEFAULT_MLP)
    fld = O.InrFieldOracle((V,) * 3, t, w, b, O.DEFAULT_GRID)
    t0 = time.time()
    vmin, vmax = O.macro_minmax_streamed(fld, (V,) * 3, 16)
    out = ROOT / "bench_data" / f"macro_inr{V}_c16.npz"
    np.savez_compressed(out, vmin=vmin, vmax=vmax, dims=np.array([V] * 3), cell=16)
    print(out, vmin.shape, f"{time.time() - t0:.1f}s", float(vmin.min()), float(vmax.max()))
