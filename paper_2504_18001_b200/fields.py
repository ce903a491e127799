"""Field API (voxcache/fields.py:28-297) backed by sm_100a decoders.

`Field.sample_batch` keeps the reference contract (positions (N,3) in [0,1)^3
-> float32 values in [0,1], DomainError outside) but evaluates on the GPU via
`vcb_field_points`.  Supported kinds: lattice (RawLatticeField), procedural
(sphere / shells / marschner_lobb_like) and the hash-grid INR (inr.InrField).
Reference-package field objects are accepted by duck typing (see
`device_field`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DomainError

PROCEDURAL_KINDS = ("sphere", "shells", "marschner_lobb_like")


@dataclass(frozen=True)
class FieldDomain:
    """fields.py:28-53: voxel extent (Vx, Vy, Vz) and native value range."""

    dims: tuple
    value_range: tuple = (0.0, 1.0)

    def __post_init__(self):
        if len(self.dims) != 3 or any(int(d) < 1 for d in self.dims):
            raise ConfigError(f"dims must be three counts >= 1, got {self.dims}")
        vmin, vmax = self.value_range
        if not vmin <= vmax:
            raise ConfigError(f"value_range must satisfy vmin <= vmax, got {self.value_range}")
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))
        object.__setattr__(self, "value_range", (float(vmin), float(vmax)))

    def normalize(self, native):
        vmin, vmax = self.value_range
        if vmax == vmin:
            return np.zeros_like(np.asarray(native, dtype=np.float64))
        return (np.asarray(native, dtype=np.float64) - vmin) / (vmax - vmin)


def check_positions(positions) -> np.ndarray:
    """fields.py:71-80: shape (N,3), every coordinate in [0,1)."""
    pos = np.asarray(positions, dtype=np.float64)
    if pos.ndim == 1 and pos.size == 3:
        pos = pos.reshape(1, 3)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise DomainError(f"positions must have shape (N, 3), got {pos.shape}")
    if pos.size and ((pos < 0.0).any() or (pos >= 1.0).any()):
        bad = pos[((pos < 0.0) | (pos >= 1.0)).any(axis=1)][0]
        raise DomainError(f"coordinate {tuple(bad)} outside [0,1)^3")
    return np.ascontiguousarray(pos)


class Field:
    """Base scalar field; evaluation happens on the GPU through the field ABI."""

    def __init__(self, domain: FieldDomain):
        self.domain = domain

    def sample_batch(self, positions) -> np.ndarray:
        pos = check_positions(positions)
        if pos.shape[0] == 0:
            return np.zeros(0, dtype=np.float32)
        from .device import device_field, field_points

        return field_points(device_field(self), pos)

    def sample_lattice(self, dims=None) -> np.ndarray:
        vx, vy, vz = dims if dims is not None else self.domain.dims
        zs, ys, xs = np.meshgrid((np.arange(vz) + 0.5) / vz, (np.arange(vy) + 0.5) / vy, (np.arange(vx) + 0.5) / vx,
                                 indexing="ij")
        pos = np.stack([xs.ravel(), ys.ravel(), zs.ravel()], axis=1)
        return self.sample_batch(pos).reshape(vz, vy, vx)


class ProceduralField(Field):
    """fields.py:119-128 analytic field."""

    def __init__(self, kind: str, dims):
        if kind not in PROCEDURAL_KINDS:
            raise ConfigError(f"unknown procedural kind {kind!r}; expected one of {sorted(PROCEDURAL_KINDS)}")
        super().__init__(FieldDomain(tuple(dims), (0.0, 1.0)))
        self.kind = kind


def make_procedural(kind: str, dims) -> ProceduralField:
    """fields.py:158."""
    return ProceduralField(kind, dims)


class RawLatticeField(Field):
    """fields.py:202-225: explicit (Vz,Vy,Vx) lattice, trilinear interpolation."""

    def __init__(self, lattice: np.ndarray, domain: FieldDomain):
        vz, vy, vx = lattice.shape
        if (vx, vy, vz) != domain.dims:
            raise ConfigError(f"lattice shape {lattice.shape} (z,y,x) does not match dims {domain.dims}")
        super().__init__(domain)
        self.lattice = np.ascontiguousarray(lattice, dtype=np.float32)
        self.lattice.flags.writeable = False

    def sample_lattice(self, dims=None):
        if dims is None or tuple(dims) == self.domain.dims:
            return self.lattice
        return super().sample_lattice(dims)
