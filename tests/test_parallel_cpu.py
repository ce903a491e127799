"""Sort-first multi-GPU host logic on CPU: world_size 2 over gloo (127.0.0.1)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, W, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2504_18001_b200 import parallel

    ctx = parallel.init_from_env(backend="gloo")
    rows = parallel.rows_of(rank, world, H)
    # the band a rank renders: film row r carries value r*1000 + column
    band = torch.tensor([[[r * 1000.0 + c, rank, 0, 1] for c in range(W)] for r in rows], dtype=torch.float32)
    full = parallel.gather_rows(ctx, band, H)
    mx = parallel.max_over_ranks(ctx, float(rank + 1))
    sm = parallel.sum_over_ranks(ctx, 10.0)
    q.put((rank, full.numpy(), mx, sm))
    parallel.shutdown(ctx)


@pytest.mark.parametrize("H", [7, 8])
def test_interleaved_bands_gather_to_full_frame(H):
    world, W = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    want = np.array([[r * 1000.0 + c for c in range(W)] for r in range(H)])
    for rank, full, mx, sm in res:
        assert full.shape == (H, W, 4)
        np.testing.assert_array_equal(full[..., 0], want)
        np.testing.assert_array_equal(full[..., 1], np.array([[r % world] * W for r in range(H)]))
        assert mx == 2.0 and sm == 20.0


def test_rows_partition_is_exact_cover():
    from paper_2504_18001_b200 import parallel

    for H in (1, 7, 1024, 2160):
        for world in (1, 2, 4, 8):
            rows = sorted(r for k in range(world) for r in parallel.rows_of(k, world, H))
            assert rows == list(range(H))


def _root_worker(rank, world, port, H, W, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2504_18001_b200 import parallel

    ctx = parallel.init_from_env(backend="gloo")
    rows = parallel.rows_of(rank, world, H)
    # RGBA8 band (the FrameGather payload): film row r carries (r, column, rank, 255)
    band = torch.tensor([[[r, c, rank, 255] for c in range(W)] for r in rows], dtype=torch.uint8)
    full = parallel.gather_bands_to_root(ctx, band, H)
    q.put((rank, None if full is None else full.numpy()))
    parallel.shutdown(ctx)


@pytest.mark.parametrize("H,world", [(7, 2), (9, 3)])
def test_rgba8_bands_gather_to_rank0(H, world):
    """Sort-first frame assembly (FrameGather's gather + interleave) over gloo."""
    W = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_root_worker, args=(r, world, port, H, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(1, world):
        assert res[r] is None
    full = res[0]
    assert full.shape == (H, W, 4)
    np.testing.assert_array_equal(full[..., 0], np.repeat(np.arange(H)[:, None], W, axis=1))
    np.testing.assert_array_equal(full[..., 1], np.repeat(np.arange(W)[None, :], H, axis=0))
    np.testing.assert_array_equal(full[..., 2], np.repeat((np.arange(H) % world)[:, None], W, axis=1))


def test_interleave_bands_matches_rows_of():
    from paper_2504_18001_b200 import parallel

    H, world, W = 11, 4, 3
    per = -(-H // world)
    bands = torch.full((world, per, W, 1), -1.0)
    for r in range(world):
        for j, row in enumerate(parallel.rows_of(r, world, H)):
            bands[r, j] = row
    full = parallel.interleave_bands(bands, H)
    np.testing.assert_array_equal(full[:, 0, 0].numpy(), np.arange(H))
