"""Macro-cell grid (voxcache/macrocell.py:20-128).

`build` decodes the field lattice on the GPU cell by cell (vcb_macro_minmax,
never materialising the lattice) and records min/max dilated by one voxel.
`update_majorants` maps a transfer function to per-cell opacity majorants:
256 value bins, each bin's TF-opacity upper bound (knots and bin edges), then
the max over the inclusive bin range [int(min*256), int(max*256)] per cell.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

OPACITY_BINS = 256


def layout(dims, cell_size: int):
    """macrocell.py:20-24."""
    grid = tuple(-(-int(v) // int(cell_size)) for v in dims)
    cells = grid[0] * grid[1] * grid[2]
    return grid, cells, cells * 8


@dataclass
class MacroCellGrid:
    cell_size: int
    dims: tuple
    grid_dims: tuple
    value_min: np.ndarray  # (gz, gy, gx) f32
    value_max: np.ndarray
    majorant: np.ndarray

    def cell_of(self, native_pos):
        idx = np.floor(np.asarray(native_pos, dtype=np.float64) / self.cell_size).astype(np.int64)
        return np.clip(idx, 0, np.asarray(self.grid_dims, dtype=np.int64) - 1)

    def majorant_at(self, cells):
        return self.majorant[cells[:, 2], cells[:, 1], cells[:, 0]]


def build(field_src, dims=None, cell_size: int = 16, device=None) -> MacroCellGrid:
    if cell_size < 2:
        raise ValueError("cell_size must be >= 2")
    dims = tuple(int(v) for v in (dims if dims is not None else field_src.domain.dims))
    grid, _, _ = layout(dims, cell_size)
    gx, gy, gz = grid
    import torch

    from . import _native as N
    from .device import device_field, ptr, require_cuda, stream_ptr

    dev = require_cuda(device)
    df = device_field(field_src, dev)
    vmin = torch.empty((gz, gy, gx), dtype=torch.float32, device=dev)
    vmax = torch.empty((gz, gy, gx), dtype=torch.float32, device=dev)
    d = (C.c_int64 * 3)(*dims)
    N.call("vcb_macro_minmax", C.byref(df.desc), d, cell_size, ptr(vmin), ptr(vmax), stream_ptr())
    vmin_h, vmax_h = vmin.cpu().numpy(), vmax.cpu().numpy()
    return MacroCellGrid(cell_size, dims, grid, vmin_h, vmax_h, np.ones((gz, gy, gx), dtype=np.float32))


def opacity_bin_maxima(tf, bins: int = OPACITY_BINS) -> np.ndarray:
    """macrocell.py:105-117: upper bound of TF opacity on each value bin."""
    xs = np.unique(np.concatenate([np.linspace(0.0, 1.0, bins + 1), tf.points[:, 0]]))
    alpha = tf.eval(xs)[:, 3]
    out = np.zeros(bins, dtype=np.float64)
    np.maximum.at(out, np.minimum((xs * bins).astype(np.int64), bins - 1), alpha)
    scaled = xs * bins
    edge = np.isclose(scaled, np.round(scaled)) & (xs > 0)
    left = np.clip(np.round(scaled).astype(np.int64) - 1, 0, bins - 1)
    np.maximum.at(out, left[edge], alpha[edge])
    return out


def update_majorants(grid: MacroCellGrid, tf) -> MacroCellGrid:
    """macrocell.py:120-128 (range max by doubling table: max over [lo, hi])."""
    bm = opacity_bin_maxima(tf)
    lo = np.clip((grid.value_min.ravel() * OPACITY_BINS).astype(np.int64), 0, OPACITY_BINS - 1)
    hi = np.clip((grid.value_max.ravel() * OPACITY_BINS).astype(np.int64), 0, OPACITY_BINS - 1)
    hi = np.maximum(hi, lo)
    levels = [bm]
    while (1 << len(levels)) <= OPACITY_BINS:
        prev, h = levels[-1], 1 << (len(levels) - 1)
        levels.append(np.maximum(prev[:-h], prev[h:]))
    width = hi - lo + 1
    k = np.floor(np.log2(width)).astype(np.int64)
    mu = np.empty(lo.shape, dtype=np.float64)
    for lv in np.unique(k):
        sel = k == lv
        t = levels[int(lv)]
        mu[sel] = np.maximum(t[lo[sel]], t[hi[sel] - (1 << int(lv)) + 1])
    grid.majorant = mu.reshape(grid.value_min.shape).astype(np.float32)
    return grid
