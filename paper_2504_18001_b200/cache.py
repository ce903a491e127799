"""Multi-resolution page table (MRPD), brick pool and request table on the device.

Host side: brick geometry (voxcache/cache/brickmath.py:25-151) and configs
(mrpd.py:21-29, pool.py:15-33).  Device side (`DeviceCache`): one dense int32
residency table over every LoD (the logical view of DirectTable/PagedTable,
P13; 4096^3@B16 is 78 MB, trivial in 180 GB HBM), the f32 pool [S][B][B][B],
owner/last_used per slot, per-brick miss counters and the request table as
per-brick (base, hits) arrays.  All mutation happens in the maintenance
kernels (csrc/cache.cu); the host only reads state back for diagnostics.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import ptr, stream_ptr


# ----------------------------------------------------------------- brick hierarchy
# The semantics are brickmath.py:25-151's (pinned by tests/golden/brickmath.npz): at
# LoD L a brick holds B samples 2^L voxels apart; along an axis brick k starts at
# native voxel k*B*2^L - 1 (0 for k = 0: P1) and owns the positions p with
# floor((p + 1) / (B*2^L)) = k; an axis needs one brick at L once
# V <= (B-1)*2^L + 1, else ceil((V + 2^L) / (B*2^L)).  Here every per-level quantity
# is a row of a small table built once.

_LOD_LIMIT = 48


def _axis_bricks(v: int, b: int, lod: int) -> int:
    step = 1 << lod
    return 1 if v <= (b - 1) * step + 1 else -(-(v + step) // (b << lod))


def _level_table(dims, b: int):
    """(L+1, 3) brick counts per level until one brick covers the volume."""
    rows = []
    while True:
        lod = len(rows)
        row = tuple(_axis_bricks(v, b, lod) for v in dims)
        rows.append(row)
        if row == (1, 1, 1):
            return rows
        if lod >= _LOD_LIMIT:
            raise ValueError(f"dims {tuple(dims)} need more than {_LOD_LIMIT} LoD levels at brick size {b}")


def max_lod(dims, brick_size: int) -> int:
    """The coarsest LoD (a single brick), brickmath.py:60-67."""
    return len(_level_table(tuple(int(d) for d in dims), int(brick_size))) - 1


@dataclass(frozen=True)
class BrickKey:
    """(LoD, brick index (i, j, k)) — brickmath.py:71-84."""

    lod: int
    index: tuple

    def __post_init__(self):
        object.__setattr__(self, "index", tuple(int(i) for i in self.index))

    def linear_index(self, grid) -> int:
        i, j, k = self.index
        return i + grid[0] * (j + grid[1] * k)


class BrickLayout:
    """A volume's brick hierarchy (brickmath.py:87-151): per-level grids, the flat
    numbering of bricks over all levels (level offsets), brick origins and the
    native/normalized coordinates of a brick's B^3 samples."""

    def __init__(self, dims, brick_size: int):
        if brick_size < 2:
            raise ValueError("brick_size must be >= 2")
        self.dims = tuple(int(d) for d in dims)
        self.brick_size = int(brick_size)
        self.grids = _level_table(self.dims, self.brick_size)
        self.max_lod = len(self.grids) - 1
        counts = np.prod(np.asarray(self.grids, dtype=np.int64), axis=1)
        starts = np.zeros(len(counts), dtype=np.int64)
        np.cumsum(counts[:-1], out=starts[1:])
        self.offsets = [int(v) for v in starts]
        self.total = int(counts.sum())

    # -- numbering
    def brick_count(self, lod: int) -> int:
        gx, gy, gz = self.grids[lod]
        return gx * gy * gz

    def total_bricks(self) -> int:
        return self.total

    def flat(self, key: BrickKey) -> int:
        return self.offsets[key.lod] + key.linear_index(self.grids[key.lod])

    def key_of_flat(self, flat: int) -> BrickKey:
        lod = int(np.searchsorted(self.offsets, flat, side="right")) - 1
        gx, gy, _ = self.grids[lod]
        q, i = divmod(flat - self.offsets[lod], gx)
        k, j = divmod(q, gy)
        return BrickKey(lod, (i, j, k))

    def valid_key(self, key: BrickKey) -> bool:
        return 0 <= key.lod <= self.max_lod and all(0 <= c < n for c, n in zip(key.index, self.grids[key.lod]))

    def keys_at(self, lod: int):
        gx, gy, gz = self.grids[lod]
        for k in range(gz):
            for j in range(gy):
                for i in range(gx):
                    yield BrickKey(lod, (i, j, k))

    # -- geometry
    def _starts(self, index, lod: int):
        """Native voxel of sample 0 of bricks `index` (int64 array) at `lod`."""
        first = index * (self.brick_size << lod)
        return np.where(index > 0, first - 1, first)

    def origin(self, key: BrickKey):
        return tuple(int(v) for v in self._starts(np.asarray(key.index, dtype=np.int64), key.lod))

    def locate(self, positions, lod: int):
        """(brick index, local sample coordinate) of native positions at `lod`."""
        if lod > self.max_lod:
            raise ValueError(f"lod {lod} is coarser than the hierarchy's {self.max_lod}")
        pos = np.asarray(positions, dtype=np.float64)
        idx = np.floor((pos + 1.0) / (self.brick_size << lod)).astype(np.int64)
        np.clip(idx, 0, np.asarray(self.grids[lod], dtype=np.int64) - 1, out=idx)
        local = (pos - self._starts(idx, lod)) / (1 << lod)
        np.clip(local, 0.0, self.brick_size - 1, out=local)
        return idx, local

    def sample_positions(self, key: BrickKey):
        """A brick's B^3 samples, x fastest: native voxels (clipped to the volume) and
        the normalized positions (n + 0.5) / V the field is evaluated at."""
        steps = np.arange(self.brick_size, dtype=np.int64) << key.lod
        z, y, x = np.meshgrid(steps, steps, steps, indexing="ij")
        native = np.column_stack([x.ravel(), y.ravel(), z.ravel()]) + np.asarray(self.origin(key))
        np.clip(native, 0, np.asarray(self.dims, dtype=np.int64) - 1, out=native)
        return native, (native + 0.5) / np.asarray(self.dims, dtype=np.float64)

    def geom(self) -> N.VcbBrickGeom:
        g = N.VcbBrickGeom()
        g.dims[:] = list(self.dims)
        g.b = self.brick_size
        g.n_lod = self.max_lod + 1
        for lod, row in enumerate(self.grids):
            g.grid[lod][:] = list(row)
            g.offset[lod] = self.offsets[lod]
        return g


@dataclass(frozen=True)
class PoolSpec:
    """pool.py:15-33."""

    pool_dims: tuple
    brick_size: int

    @property
    def slot_count(self) -> int:
        px, py, pz = self.pool_dims
        return px * py * pz

    @property
    def voxel_count(self) -> int:
        return self.slot_count * self.brick_size ** 3

    @property
    def byte_size(self) -> int:
        return self.voxel_count * 4


@dataclass(frozen=True)
class CacheConfig:
    """mrpd.py:21-29."""

    brick_size: int = 40
    pool_dims: tuple = (8, 8, 8)
    direct_table_threshold: int = 1 << 18
    page_size: int = 4096
    page_budget: int = 64

    def pool_spec(self) -> PoolSpec:
        return PoolSpec(tuple(self.pool_dims), self.brick_size)


def _bits(v: int) -> int:
    return max(1, int(v).bit_length())


class DeviceCache:
    """GPU-resident Mrpd + BrickPool + RequestTable + InlineLoader staging."""

    def __init__(self, dims, config: CacheConfig, sched, device, debug=False):
        self.config = config
        self.sched = sched
        self.device = device
        self.layout = BrickLayout(dims, config.brick_size)
        lay = self.layout
        if lay.max_lod > 127:
            raise ValueError("LoD arrays are int8 (P17)")
        self.max_lod = lay.max_lod
        counts = [lay.brick_count(l) for l in range(lay.max_lod + 1)]
        # the reference takes its numpy lookup path (|pos-cam| LoD distances) as
        # soon as one LoD table is virtualised (mrpd.py:99-100, sampler.py:131-142)
        self.paged = any(c > config.direct_table_threshold for c in counts)
        self.slots = config.pool_spec().slot_count
        b3 = config.brick_size ** 3
        self.geom = lay.geom()
        mr = int(sched.max_requests)
        if mr < 1:
            raise ValueError("batch size must be >= 1")
        t = lambda n, dt, fill: torch.full((n,), fill, dtype=dt, device=device)
        self.table = t(lay.total, torch.int32, -1)
        self.pool = torch.zeros(self.slots * b3, dtype=torch.float32, device=device)
        self.owner = t(self.slots, torch.int64, -1)
        self.last_used = t(self.slots, torch.int64, -1)
        self.miss_count = t(lay.total, torch.int32, 0)
        self.req_base = t(lay.total, torch.int64, -1)
        self.req_hits = t(lay.total, torch.int64, 0)
        self.state = torch.zeros(C.sizeof(N.VcbCacheState) // 8, dtype=torch.int64, device=device)
        self.staging = torch.zeros(mr * b3, dtype=torch.float32, device=device)
        self.staged_keys = t(mr, torch.int64, -1)
        wsb = N.load().vcb_maint_workspace_bytes(lay.total, self.slots, mr)
        self.workspace = torch.zeros(wsb, dtype=torch.uint8, device=device)
        self._graph, self._graph_key = None, None  # the maintenance CUDA graph (maintenance(graph=True))
        self.dbg_reports = t(2 * lay.total, torch.int64, 0) if debug else None
        # the request table's keys as a compacted list (k_pending reads it instead of
        # scanning every brick's req_base: 19.4 M bricks at 4096^3@B16); list_counts[1]
        self.pending_list = t(lay.total, torch.int32, 0)
        self.list_counts = t(4, torch.int32, 0)
        self.frame = 0  # Mrpd.frame: the probe stamp clock (P11)
        max_lin = max(counts) - 1
        self.lin_bits = _bits(max_lin)
        self.lod_bits = _bits(lay.max_lod)
        if 63 - self.lin_bits - self.lod_bits < 24:
            raise ValueError("brick grid too large for 64-bit request keys")

    def reset(self):
        """mrpd.py:268-276 (Mrpd.frame survives; in-flight loads dropped)."""
        self.table.fill_(-1)
        self.pool.zero_()
        self.owner.fill_(-1)
        self.last_used.fill_(-1)
        self.miss_count.zero_()
        self.req_base.fill_(-1)
        self.req_hits.zero_()
        self.list_counts.zero_()
        self.state.zero_()

    def maint_params(self, session_frame: int, field_desc, frame_stats=None, defer_decode=False) -> N.VcbMaintParams:
        p = N.VcbMaintParams()
        p.geom = self.geom
        p.total = self.layout.total
        p.slots = self.slots
        p.session_frame = session_frame
        p.max_requests = self.sched.max_requests
        p.ranking = 1 if self.sched.ranking_enabled else 0
        p.rank_clamp = self.sched.rank_clamp
        p.lin_bits = self.lin_bits
        p.lod_bits = self.lod_bits
        p.table = ptr(self.table)
        p.pool = ptr(self.pool)
        p.owner = ptr(self.owner)
        p.last_used = ptr(self.last_used)
        p.miss_count = ptr(self.miss_count)
        p.req_base = ptr(self.req_base)
        p.req_hits = ptr(self.req_hits)
        p.state = ptr(self.state)
        p.staging = ptr(self.staging)
        p.staged_keys = ptr(self.staged_keys)
        p.workspace = ptr(self.workspace)
        p.workspace_bytes = self.workspace.numel()
        p.dbg_reports = ptr(self.dbg_reports)
        p.field = field_desc
        p.frame_stats = frame_stats
        p.pending_list, p.list_counts = ptr(self.pending_list), ptr(self.list_counts)
        budget = getattr(self.sched, "decode_budget", None)
        p.decode_budget = -1 if budget is None else int(budget)
        p.defer_decode = 1 if defer_decode else 0
        return p

    def maintenance(self, session_frame: int, field_desc, stream=None, frame_stats=None, defer_decode=False,
                    graph=False):
        """vcb_maintenance.  frame_stats = device address of the frame's VcbFrameStats (a
        failed frame then skips the maintenance on the device; the decode budget's share
        the frame used).  defer_decode: the batch is left for decode() on another stream.
        graph: replay the maintenance as one CUDA graph (vcb_maint_graph_*), captured
        again whenever a parameter other than the session frame changes."""
        p = self.maint_params(session_frame, field_desc, frame_stats, defer_decode)
        self._last_params = p
        if not graph:
            N.call("vcb_maintenance", C.byref(p), stream_ptr(stream))
            return
        q = N.VcbMaintParams.from_buffer_copy(p)
        q.session_frame = 0
        key = bytes(q)
        if self._graph is None or self._graph_key != key:
            self.drop_graph()
            h = C.c_void_p()
            N.call("vcb_maint_graph_create", C.byref(p), C.byref(h))
            self._graph, self._graph_key = h, key
        N.call("vcb_maint_graph_launch", self._graph, C.byref(p), stream_ptr(stream))

    def drop_graph(self):
        if getattr(self, "_graph", None) is not None:
            N.load().vcb_maint_graph_destroy(self._graph)
        self._graph, self._graph_key = None, None

    def __del__(self):
        try:
            self.drop_graph()
        except Exception:
            pass

    def decode(self, stream):
        """The deferred fulfill of the batch the last maintenance selected (vcb_maint_decode)."""
        N.call("vcb_maint_decode", C.byref(self._last_params), stream_ptr(stream))

    # ---- diagnostics (D2H; not on the hot path)
    def state_dict(self):
        s = self.state.cpu().numpy()
        names = [f[0] for f in N.VcbCacheState._fields_ if f[0] != "pad_"]
        return {n: int(s[i]) for i, n in enumerate(names)}

    def occupancy_from(self, st) -> float:
        return 1.0 - (self.slots - st["next_free"]) / self.slots

    def is_mapped(self, key: BrickKey) -> bool:
        return int(self.table[self.layout.flat(key)].item()) >= 0

    def dump(self):
        """Reference-shaped state: dense tables, owner (lod, linear), stamps, requests."""
        lay = self.layout
        offs = np.asarray(lay.offsets, dtype=np.int64)
        own = self.owner.cpu().numpy()
        pairs = np.full((self.slots, 2), -1, dtype=np.int64)
        m = own >= 0
        lods = np.searchsorted(offs, own[m], side="right") - 1
        pairs[m, 0] = lods
        pairs[m, 1] = own[m] - offs[lods]
        base = self.req_base.cpu().numpy()
        hits = self.req_hits.cpu().numpy()
        pend = np.flatnonzero(base >= 0)
        pl = np.searchsorted(offs, pend, side="right") - 1
        ents = np.stack([pl, pend - offs[pl], base[pend], hits[pend]], axis=1) if pend.size else np.zeros((0, 4), np.int64)
        ents = ents[np.lexsort((ents[:, 1], ents[:, 0]))] if pend.size else ents
        st = self.state_dict()
        return dict(tables=self.table.cpu().numpy(), owner=pairs, last_used=self.last_used.cpu().numpy(),
                    n_free=self.slots - st["next_free"], cache_frame=self.frame, entries=ents.astype(np.int64),
                    state=st)

    def batch(self):
        st = self.state_dict()
        keys = self.staged_keys[: st["n_batch"]].cpu().numpy()
        offs = np.asarray(self.layout.offsets, dtype=np.int64)
        l = np.searchsorted(offs, keys, side="right") - 1
        return np.stack([l, keys - offs[l]], axis=1).astype(np.int64).reshape(-1, 2)

    def reports(self):
        st = self.state_dict()
        if self.dbg_reports is None:
            return None
        r = self.dbg_reports[: 2 * st["n_reports"]].cpu().numpy().reshape(-1, 2)
        offs = np.asarray(self.layout.offsets, dtype=np.int64)
        l = np.searchsorted(offs, r[:, 0], side="right") - 1
        out = np.stack([l, r[:, 0] - offs[l], r[:, 1]], axis=1).astype(np.int64)
        return out[np.lexsort((out[:, 1], out[:, 0]))].reshape(-1, 3)
