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


@pytest.mark.parametrize("name,cap", [("pressure", None), ("inr64", None), ("pressure", 3)])
def test_shared_decode_world1_matches_reference(name, cap):
    """cap=3: most of each batch overflows the owner's slab and is decoded locally."""
    from gpu_runner import run_gpu_session
    from paper_2504_18001_b200 import parallel

    g = load_golden(f"session_{name}.npz")
    exact = name == "pressure"
    share = lambda sess: sess.share_decode(parallel.Ctx(), cap=cap)
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


def _splitmix64(x):
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


@pytest.mark.parametrize("world,mr,cap,seed", [(3, 12, 12, 0), (3, 12, 2, 1), (4, 40, 5, 2), (1, 7, 3, 3)])
def test_share_plan_matches_restatement(world, mr, cap, seed):
    """vcb_share_plan against a direct restatement: owner = splitmix64(key) % world,
    slot = rank among the owner's distinct keys, keys past `cap` decoded locally
    (small caps force the overflow path); duplicates across ranks decoded once."""
    import torch

    from paper_2504_18001_b200 import _native as N

    rng = np.random.default_rng(seed)
    pool = rng.choice(10_000, size=mr * world, replace=False)
    rows = np.full((world, mr + 1), -1, dtype=np.int64)
    for q in range(world):
        n = int(rng.integers(0, mr + 1))
        keys = rng.choice(pool[: max(1, mr * world // 2)], size=min(n, mr * world // 2), replace=False)[:mr]
        rows[q, 0] = len(keys)
        rows[q, 1:1 + len(keys)] = keys
    dev = torch.device("cuda")
    all_keys = torch.from_numpy(rows.ravel()).to(dev)
    for rank in range(world):
        own = torch.full((cap,), -1, dtype=torch.int64, device=dev)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
        src = torch.empty(mr, dtype=torch.int32, device=dev)
        ovf_keys = torch.full((mr,), -1, dtype=torch.int64, device=dev)
        ovf_idx = torch.full((mr,), -1, dtype=torch.int32, device=dev)
        N.call("vcb_share_plan", all_keys.data_ptr(), world, rank, mr, cap, own.data_ptr(), counts.data_ptr(),
               src.data_ptr(), ovf_keys.data_ptr(), ovf_idx.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        distinct = sorted({int(k) for q in range(world) for k in rows[q, 1:1 + rows[q, 0]]})
        owner = {k: _splitmix64(k) % world for k in distinct}
        slots = {k: sorted(v for v in distinct if owner[v] == owner[k]).index(k) for k in distinct}
        mine = [k for k in distinct if owner[k] == rank]
        want_own = [k for k in mine if slots[k] < cap]
        assert int(counts[0]) == len(want_own)
        np.testing.assert_array_equal(own.cpu().numpy()[: len(want_own)], want_own)
        n_mine = int(rows[rank, 0])
        got_src = src.cpu().numpy()
        ovf = {}
        for i in range(n_mine):
            k = int(rows[rank, 1 + i])
            if slots[k] < cap:
                assert got_src[i] == owner[k] * cap + slots[k]
            else:
                assert got_src[i] == -1
                ovf[i] = k
        assert int(counts[1]) == len(ovf)
        oi, ok = ovf_idx.cpu().numpy()[: len(ovf)], ovf_keys.cpu().numpy()[: len(ovf)]
        assert {int(i): int(k) for i, k in zip(oi, ok)} == ovf
