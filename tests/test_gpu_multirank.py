"""Sort-first multi-rank rendering on the GPU box (one device shared by the ranks,
gloo carries the gather): the RGBA8 bands FrameGather assembles on rank 0 equal the
single-session frame quantised as image_io.to_rgba8 does — bit for bit."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_bands_on_ranks_join_to_the_frame(tmp_path, world):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "mp.npz"
    env = dict(os.environ, CINR_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tests" / "mp_band_worker.py"),
           str(out)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = np.load(out)
    assert int(d["world"]) == world
    np.testing.assert_array_equal(d["frame"], d["ref"])
