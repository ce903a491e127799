"""Golden fixture for BASELINE config 1 at its stated size (scene_specs "config1"):
the UNMODIFIED reference renders the full 120-frame orbit at 256x256; every frame's
FrameRecord and post-maintenance cache state is kept, the image every 20th frame.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_config1.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import make_golden as G  # noqa: E402  (the reference capture wrappers)
import scene_specs as specs  # noqa: E402

IMAGE_EVERY = 20


def main():
    frames, _, macro = G.run_session(specs.SESSION_SPECS["config1"])
    out = {"macro_vmin": macro["vmin"], "macro_vmax": macro["vmax"]}
    for f, d in frames.items():
        for k, v in d.items():
            if k == "img" and f % IMAGE_EVERY != IMAGE_EVERY - 1:
                continue
            out[f"f{f}_{k}"] = v
    np.savez_compressed(HERE / "session_config1.npz", **out)
    print("config1 frames", len(frames), "bytes", (HERE / "session_config1.npz").stat().st_size)


if __name__ == "__main__":
    main()
