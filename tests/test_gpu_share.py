"""Brick-decode sharing across ranks (parallel.BrickShare, SURVEY §8e "optional brick
sharing") on the GPU box: the state and images of a session that shares its brick
decodes equal those of the same session decoding alone, frame by frame — in one
process (world 1: every key is owned locally) against the reference's goldens, and
with 2-3 ranks sharing one device over gloo, each rank rendering its sort-first band."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("name", ["pressure", "inr64"])
def test_shared_decode_world1_matches_reference(name):
    from gpu_runner import run_gpu_session
    from paper_2504_18001_b200 import parallel

    g = load_golden(f"session_{name}.npz")
    exact = name == "pressure"
    share = lambda sess: sess.share_decode(parallel.Ctx())
    for f, img, rec, sess in run_gpu_session(name, macro=(g["macro_vmin"], g["macro_vmax"]), setup=share):
        assert sess._share is not None
        st = sess.debug_state()
        for k in ("tables", "owner", "entries", "batch") + (("last_used",) if exact else ()):
            np.testing.assert_array_equal(st[k], g[f"f{f}_{k}"], err_msg=f"frame {f} {k}")
        assert np.abs(img - g[f"f{f}_img"]).max() <= (1e-6 if exact else 1e-3), f"frame {f}"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,name", [(2, "pressure"), (3, "inr64")])
def test_shared_decode_across_ranks_equals_alone(tmp_path, world, name):
    frames = 12
    env = dict(os.environ, CINR_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tests" / "mp_share_worker.py"),
           str(tmp_path), name, str(frames)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    alone_total, owned = 0, 0
    for rank in range(world):
        d = np.load(tmp_path / f"rank{rank}.npz")
        assert int(d["world"]) == world
        for f in range(frames):
            for k in ("img", "rec", "tables", "owner", "last_used", "entries", "batch"):
                np.testing.assert_array_equal(d[f"s{f}_{k}"], d[f"a{f}_{k}"], err_msg=f"rank {rank} frame {f} {k}")
            alone_total += len(d[f"a{f}_batch"])
        owned += int(d["owned_total"])
    # the ranks' batches overlap: together they decoded fewer bricks than alone
    assert 0 < owned < alone_total
