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


def interleave_bands(bands: torch.Tensor, height: int) -> torch.Tensor:
    """(world, per, W, C) padded bands -> the (height, W, C) frame: band r's row j is
    film row r + j*world."""
    world, per = bands.shape[0], bands.shape[1]
    return bands.transpose(0, 1).reshape(per * world, *bands.shape[2:])[:height]


def gather_bands_to_root(ctx: Ctx, band: torch.Tensor, height: int, out: torch.Tensor = None):
    """Gather every rank's interleaved row band (padded to ceil(height/world) rows) to
    rank 0; returns the assembled frame on rank 0, None elsewhere.  NCCL on CUDA
    tensors, gloo on host tensors (the CPU tests)."""
    if ctx.world == 1:
        return band
    per = -(-height // ctx.world)
    if band.shape[0] != per:
        pad = torch.zeros((per,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
        pad[: band.shape[0]] = band
        band = pad
    if ctx.rank == 0:
        if out is None:
            out = torch.empty((ctx.world,) + tuple(band.shape), dtype=band.dtype, device=band.device)
        dist.gather(band, gather_list=list(out.unbind(0)), dst=0)
        return interleave_bands(out, height)
    dist.gather(band, gather_list=None, dst=0)
    return None


class FrameGather:
    """Frame assembly for N>1 on a comm stream that overlaps the next frame.

    Sort-first tiles: each rank quantises its film-row band to RGBA8 on the render
    stream (vcb_frame_rgba8 = image_io.to_rgba8, 4 B/pixel instead of 16), then the
    comm stream waits for it and NCCL-gathers the bands to rank 0 while the render
    stream goes on with the next frame.  Alternate-frame rendering gathers whole
    RGBA8 frames the same way.  Two band buffers per rank; the render stream only
    reuses one after the gather that read it has finished."""

    def __init__(self, ctx: Ctx, sess, height: int, width: int, frames: bool = False):
        from . import _native as N
        from .device import ptr, stream_ptr

        self.N, self.ptr, self.stream_ptr = N, ptr, stream_ptr
        self.ctx, self.sess, self.H, self.W, self.frames = ctx, sess, height, width, frames
        dev = torch.device("cuda", ctx.local_rank)
        self.rows = height if frames else -(-height // ctx.world)
        self.comm = torch.cuda.Stream(dev)
        self.bands = [torch.zeros((self.rows, width, 4), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.done = [None, None]
        self.out = [torch.empty((ctx.world, self.rows, width, 4), dtype=torch.uint8, device=dev)
                    for _ in range(2)] if ctx.rank == 0 else None
        self.i = 0
        self.last = None

    def submit(self, img: torch.Tensor):
        """Queue this rank's part of the current frame (img: f32 (rows, W, 4))."""
        k = self.i % 2
        st = self.sess.stream
        if self.done[k] is not None:
            st.wait_event(self.done[k])
        with torch.cuda.stream(st):
            self.N.call("vcb_frame_rgba8", self.ptr(img), img.numel() // 4, self.ptr(self.bands[k]),
                        self.stream_ptr(st))
        ready = torch.cuda.Event()
        ready.record(st)
        if self.ctx.backend != "nccl":
            # gloo (ranks sharing a GPU in the functional checks): through host memory,
            # synchronously
            ready.synchronize()
            band = self.bands[k].cpu()
            outs = [torch.empty_like(band) for _ in range(self.ctx.world)] if self.ctx.rank == 0 else None
            dist.gather(band, gather_list=outs, dst=0)
            if self.ctx.rank == 0:
                self.out[k].copy_(torch.stack(outs))
            self.done[k] = None
            self.last = k
            self.i += 1
            return
        self.comm.wait_event(ready)
        with torch.cuda.stream(self.comm):
            if self.ctx.world > 1:
                dist.gather(self.bands[k], gather_list=list(self.out[k].unbind(0)) if self.ctx.rank == 0 else None,
                            dst=0)
            ev = torch.cuda.Event()
            ev.record(self.comm)
        self.done[k] = ev
        self.last = k
        self.i += 1

    def drain(self):
        self.comm.synchronize()

    def host_frame(self):
        """Rank 0: the last submitted frame(s) as host RGBA8 (H, W, 4), or (world, H, W, 4)
        for alternate-frame rendering."""
        self.comm.synchronize()
        o = self.out[self.last]
        full = o if self.frames else interleave_bands(o, self.H)
        return full.cpu().numpy()

    def close(self):
        self.drain()


class BrickShare:
    """Brick-decode sharing across ranks (SURVEY §8e "optional brick sharing").

    Every rank's maintenance selects its own batch for its private cache.  The batches'
    keys are all-gathered; each distinct key is decoded once, by its owner rank
    (splitmix64(key) % world), into a fixed slab of `cap` bricks; the slabs are
    all-gathered and each rank fills its staging slab from them (vcb_share_*).  With
    sort-first bands the ranks' batches overlap, so a rank decodes about 1/world of
    what it would alone; the cache state is unchanged (the decoder is deterministic
    per key).  NCCL all-gathers on the session stream; gloo (ranks sharing a GPU in the
    functional checks) goes through host memory."""

    def __init__(self, ctx: Ctx, sess, cap=None):
        c = sess.cache
        if c is None:
            raise ValueError("brick sharing needs a cached session")
        self.ctx, self.sess = ctx, sess
        dev = sess.device
        mr = int(c.sched.max_requests)
        b3 = int(c.geom.b) ** 3
        W = ctx.world
        self.mr, self.cap, self.b3 = mr, int(cap) if cap is not None else mr, b3  # cap: slab bricks per owner
        e = lambda n, dt: torch.empty(n, dtype=dt, device=dev)
        self.keys = e(mr + 1, torch.int64)
        self.keys_all = e(W * (mr + 1), torch.int64)
        self.own, self.counts = e(self.cap, torch.int64), torch.zeros(2, dtype=torch.int64, device=dev)
        self.src, self.ovf_keys, self.ovf_idx = e(mr, torch.int32), e(mr, torch.int64), e(mr, torch.int32)
        self.slab, self.flag = e(self.cap * b3, torch.float32), torch.zeros(1, dtype=torch.int32, device=dev)
        self.gathered, self.flags = e(W * self.cap * b3, torch.float32), e(W, torch.int32)
        self.ovf_out, self.ovf_flag = e(mr * b3, torch.float32), torch.zeros(1, dtype=torch.int32, device=dev)
        self.decoded = 0  # bricks this rank decoded (owned + local), host-side count for reports

    def _all_gather(self, out, inp):
        if self.ctx.world == 1:
            out.copy_(inp)
        elif self.ctx.backend == "nccl":
            dist.all_gather_into_tensor(out, inp)
        else:
            torch.cuda.current_stream().synchronize()
            h = inp.cpu()
            parts = [torch.empty_like(h) for _ in range(self.ctx.world)]
            dist.all_gather(parts, h)
            out.copy_(torch.cat(parts))

    def run(self, params, stream):
        """After a maintenance with defer_decode=1 (params: its VcbMaintParams)."""
        import ctypes as C

        from . import _native as N
        from .device import ptr, stream_ptr

        sp, pp = stream_ptr(stream), C.byref(params)
        with torch.cuda.stream(stream):
            N.call("vcb_share_keys", pp, ptr(self.keys), sp)
            self._all_gather(self.keys_all, self.keys)
            N.call("vcb_share_plan", ptr(self.keys_all), self.ctx.world, self.ctx.rank, self.mr, self.cap,
                   ptr(self.own), ptr(self.counts), ptr(self.src), ptr(self.ovf_keys), ptr(self.ovf_idx), sp)
            self.flag.zero_()
            N.call("vcb_share_decode", pp, ptr(self.own), ptr(self.counts), self.cap, ptr(self.slab), ptr(self.flag), sp)
            self._all_gather(self.gathered, self.slab)
            self._all_gather(self.flags, self.flag)
            self.ovf_flag.zero_()
            N.call("vcb_share_decode", pp, ptr(self.ovf_keys), ptr(self.counts[1:]), self.mr, ptr(self.ovf_out),
                   ptr(self.ovf_flag), sp)
            N.call("vcb_share_scatter", pp, ptr(self.gathered), ptr(self.flags), self.cap, ptr(self.src),
                   ptr(self.ovf_out), ptr(self.ovf_idx), ptr(self.counts), ptr(self.ovf_flag), sp)


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
