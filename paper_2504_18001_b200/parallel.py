"""Sort-first multi-GPU rendering: one process per GPU, each with a
private cache (MRPD + pool + request table), film rows interleaved across ranks
(rank r renders rows r, r+N, r+2N, ... — balances the orbit's empty borders),
and one NCCL all-gather of the RGBA bands per frame on the session stream.

The same code runs with world_size 1 (no collective) and, for tests on CPU
hosts, with the gloo backend on host tensors (`gather_rows`).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class Ctx:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    backend: str = "none"


def init_from_env(backend=None) -> Ctx:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if ndev and local_world > ndev:
        # more ranks than GPUs (a functional check of the multi-rank path on a small
        # box): ranks share devices round-robin; NCCL cannot, so gloo carries the gather
        local = local % ndev
        backend = backend or "gloo"
    backend = backend or os.environ.get("CINR_DIST_BACKEND") or None
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        be = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if be == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(be, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(be)
        return Ctx(rank, world, local, be)
    return Ctx(rank, world, local, dist.get_backend() if dist.is_initialized() else "none")


def rows_of(rank: int, world: int, height: int):
    """Film rows rendered by `rank` (interleaved assignment)."""
    return list(range(rank, height, world))


def make_session(ctx: Ctx, field_src, tf, camera, config, macro=None, bands: bool = True):
    """A session on this rank's GPU: a sort-first band of every frame (bands=True) or
    whole frames (alternate-frame rendering, bands=False)."""
    from .session import RenderSession

    s = RenderSession(field_src, tf, camera, config, macro=macro, device=torch.device("cuda", ctx.local_rank))
    if bands:
        s.set_band(ctx.rank, ctx.world)
    return s


def gather_frames(ctx: Ctx, img: torch.Tensor, stream=None) -> torch.Tensor:
    """Alternate-frame rendering: every rank's whole frame of this step, stacked
    (world, H, W, 4), all-gathered with NCCL on the render stream."""
    if ctx.world == 1:
        return img.unsqueeze(0)
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        out = torch.empty((ctx.world,) + tuple(img.shape), dtype=img.dtype, device=img.device)
        if ctx.backend == "nccl":
            dist.all_gather_into_tensor(out, img.contiguous())
        else:
            dist.all_gather(list(out.unbind(0)), img.contiguous())
        return out


def gather_rows(ctx: Ctx, band: torch.Tensor, height: int) -> torch.Tensor:
    """All-gather interleaved row bands into the full (H, W, C) frame on every rank."""
    if ctx.world == 1:
        return band
    per = -(-height // ctx.world)
    W, Cc = band.shape[1], band.shape[2]
    pad = torch.zeros((per, W, Cc), dtype=band.dtype, device=band.device)
    pad[: band.shape[0]] = band
    out = torch.empty((ctx.world * per, W, Cc), dtype=band.dtype, device=band.device)
    if ctx.backend == "nccl":
        dist.all_gather_into_tensor(out, pad)
    else:
        dist.all_gather(list(out.view(ctx.world, per, W, Cc).unbind(0)), pad)
    # out[r*per + j] holds film row r + j*world
    full = out.view(ctx.world, per, W, Cc).transpose(0, 1).reshape(per * ctx.world, W, Cc)
    return full[:height]


def gather_frame(ctx: Ctx, img: torch.Tensor, stream=None, height=None) -> torch.Tensor:
    """NCCL all-gather of this frame's row bands, ordered on the render stream."""
    if ctx.world == 1:
        return img
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        return gather_rows(ctx, img, height if height is not None else img.shape[0] * ctx.world)


class FusedGather:
    """Sort-first gather fused into the frame kernel: every rank's march kernel stores
    its retired pixels straight into rank 0's frame buffer over NVLink (a symmetric-
    memory peer mapping; VcbFrameParams.image_global), so the transfer overlaps the
    march instead of following it.  One device-side barrier per frame orders the
    peer stores before rank 0 reads the frame.  Opt-in (bench.py --fused-gather);
    the NCCL all-gather stays the default."""

    def __init__(self, ctx: Ctx, sess, height: int, width: int):
        import torch.distributed._symmetric_memory as symm_mem

        dev = torch.device("cuda", ctx.local_rank)
        self.ctx = ctx
        self.local = symm_mem.empty((height, width, 4), dtype=torch.float32, device=dev)
        self.hdl = symm_mem.rendezvous(self.local, dist.group.WORLD)
        self.target = self.hdl.get_buffer(0, (height, width, 4), torch.float32)
        sess.set_frame_target(self.target)

    def finish(self, stream) -> torch.Tensor:
        """Call after render_frame_device() on every rank; the full frame (rank 0)."""
        with torch.cuda.stream(stream):
            self.hdl.barrier(channel=0)
        return self.local


def barrier(ctx: Ctx):
    if ctx.world > 1:
        dist.barrier()


def _reduce(ctx: Ctx, v: float, op) -> float:
    if ctx.world == 1:
        return v
    dev = torch.device("cuda", ctx.local_rank) if ctx.backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(ctx: Ctx, v: float) -> float:
    return _reduce(ctx, v, dist.ReduceOp.MAX)


def sum_over_ranks(ctx: Ctx, v: float) -> float:
    return _reduce(ctx, v, dist.ReduceOp.SUM)


def shutdown(ctx: Ctx):
    if ctx.world > 1 and dist.is_initialized():
        dist.destroy_process_group()
