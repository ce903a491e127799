"""Stochastic LoD policy and per-frame RNG seeding (voxcache/sampler.py:19-100, 283).

Host side computes the per-frame scale and the frame's splitmix64 base; the
per-lane seeds and xorshift32 draws happen inside the march kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


@dataclass
class LodPolicy:
    lod_scale: float = 1.0
    preload_frames: int = 120
    mode: str = "corrected"  # corrected | as_printed | off


MODES = {"corrected": 0, "as_printed": 1, "off": 2}


def splitmix64(x: int) -> int:
    """sampler.py:24-30 on Python ints with explicit 64-bit wrap."""
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def frame_rng_base(seed: int, frame: int) -> int:
    """sampler.py:41: splitmix64(seed ^ frame*GOLDEN); lane j = splitmix64(base + j)."""
    return splitmix64((seed & MASK64) ^ ((frame * GOLDEN) & MASK64))


def effective_lod_scale(policy: LodPolicy, frame: int, force_scale: float) -> float:
    """sampler.py:70-77."""
    k = policy.preload_frames
    if frame >= k or force_scale <= policy.lod_scale:
        return policy.lod_scale
    t = frame / k
    return policy.lod_scale + (force_scale - policy.lod_scale) * (1.0 - t)


def force_max_scale(max_lod: int, min_distance: float) -> float:
    """sampler.py:80-82."""
    return (max_lod + 1.0) / max(min_distance, 1e-6)


def point_to_unit_box(p) -> float:
    """sampler.py:283-285."""
    p = np.asarray(p, dtype=np.float64)
    gap = np.maximum(np.maximum(-p, p - 1.0), 0.0)
    return float(np.linalg.norm(gap))
