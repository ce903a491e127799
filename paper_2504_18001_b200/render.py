"""Render API types: Camera (camera.py:15-66), TransferFunction (transfer.py:13-98),
RenderSettings (scene.py:16-26).  Host-side value objects; the arithmetic that
feeds the kernels (camera basis, LUT, base step) reproduces the reference's
numpy expressions exactly so GPU rays match the reference bit for bit.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ConfigError


@dataclass(frozen=True)
class Camera:
    position: tuple
    target: tuple
    up: tuple = (0.0, 1.0, 0.0)
    fov_y: float = 45.0
    width: int = 256
    height: int = 256

    def __post_init__(self):
        if not 0.0 < self.fov_y < 180.0:
            raise ConfigError(f"fov must be in (0, 180), got {self.fov_y}")
        fwd = np.asarray(self.target, dtype=np.float64) - np.asarray(self.position, dtype=np.float64)
        n = np.linalg.norm(fwd)
        if n == 0:
            raise ConfigError("camera position and target coincide")
        if np.linalg.norm(np.array(_cross(fwd / n, np.asarray(self.up, dtype=np.float64)))) < 1e-9:
            raise ConfigError("up vector is parallel to the view direction")

    def basis(self):
        return camera_basis(self)

    def to_json(self) -> dict:
        return {"position": list(self.position), "target": list(self.target), "up": list(self.up), "fov": self.fov_y,
                "width": self.width, "height": self.height}

    @classmethod
    def from_json(cls, data: dict) -> "Camera":
        return cls(position=tuple(data["position"]), target=tuple(data["target"]),
                   up=tuple(data.get("up", (0.0, 1.0, 0.0))), fov_y=float(data.get("fov", 45.0)),
                   width=int(data.get("width", 256)), height=int(data.get("height", 256)))


def _cross(a, b):
    """np.cross for 3-vectors, component by component as numpy computes it
    (a1*b2 - a2*b1: two roundings, no fused multiply-add), without its array overhead."""
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def camera_basis(cam):
    """camera.py:36-42 (works for any object with position/target/up).  Scalar arithmetic
    with numpy's norms: bit-identical to the array expressions (tests/test_host_cpu.py)."""
    p, t, u = cam.position, cam.target, cam.up
    fwd = (float(t[0]) - float(p[0]), float(t[1]) - float(p[1]), float(t[2]) - float(p[2]))
    n = float(np.linalg.norm(np.array(fwd)))
    fwd = (fwd[0] / n, fwd[1] / n, fwd[2] / n)
    right = _cross(fwd, (float(u[0]), float(u[1]), float(u[2])))
    n = float(np.linalg.norm(np.array(right)))
    right = (right[0] / n, right[1] / n, right[2] / n)
    up = _cross(right, fwd)
    return np.array(fwd), np.array(right), np.array(up)


def camera_rays_setup(cam):
    """camera.py:129-138: rot = [right, up, fwd] columns, tan_h = tan*aspect, tan_v."""
    fwd, right, up = camera_basis(cam)
    rot = np.array([[right[0], up[0], fwd[0]], [right[1], up[1], fwd[1]], [right[2], up[2], fwd[2]]])
    tan_half = np.tan(np.radians(cam.fov_y) / 2.0)
    aspect = cam.width / cam.height
    return rot, float(tan_half * aspect), float(tan_half)


class TransferFunction:
    """Ordered control points (x, r, g, b, a), x strictly increasing from 0 to 1."""

    def __init__(self, points):
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 5 or pts.shape[0] < 2:
            raise ConfigError("transfer function needs >= 2 control points of (x, r, g, b, a)")
        x = pts[:, 0]
        if x[0] != 0.0 or x[-1] != 1.0 or not (np.diff(x) > 0).all():
            raise ConfigError("control point x values must increase strictly from 0 to 1")
        if (pts[:, 1:] < 0).any() or (pts[:, 1:] > 1).any():
            raise ConfigError("color and opacity components must lie in [0,1]")
        self.points = pts
        self.points.flags.writeable = False

    def eval(self, values) -> np.ndarray:
        v = np.clip(np.asarray(values, dtype=np.float64), 0.0, 1.0)
        out = np.empty(v.shape + (4,), dtype=np.float64)
        for c in range(4):
            out[..., c] = np.interp(v, self.points[:, 0], self.points[:, c + 1])
        return out

    def lookup_table(self, size: int = 1024) -> np.ndarray:
        lut = getattr(self, "_lut", None)
        if lut is None or lut.shape[0] != size:
            lut = self.eval(np.linspace(0.0, 1.0, size)).astype(np.float32)
            self._lut = lut
        return lut

    def opacity(self, values) -> np.ndarray:
        v = np.clip(np.asarray(values, dtype=np.float64), 0.0, 1.0)
        return np.interp(v, self.points[:, 0], self.points[:, 4])

    def to_json(self):
        return [{"x": float(p[0]), "rgb": [float(p[1]), float(p[2]), float(p[3])], "a": float(p[4])} for p in self.points]

    @classmethod
    def from_json(cls, data) -> "TransferFunction":
        try:
            pts = [[p["x"], p["rgb"][0], p["rgb"][1], p["rgb"][2], p["a"]] for p in data]
        except (KeyError, TypeError, IndexError) as exc:
            raise ConfigError(f"malformed transfer function JSON: {exc}") from exc
        return cls(pts)

    @classmethod
    def load(cls, path) -> "TransferFunction":
        return cls.from_json(json.loads(Path(path).read_text()))


def grayscale_ramp(max_opacity: float = 1.0) -> TransferFunction:
    return TransferFunction([[0.0, 0.0, 0.0, 0.0, 0.0], [1.0, 1.0, 1.0, 1.0, max_opacity]])


def transparent() -> TransferFunction:
    return TransferFunction([[0.0, 0.0, 0.0, 0.0, 0.0], [1.0, 1.0, 1.0, 1.0, 0.0]])


def warm_body(threshold: float = 0.35, max_opacity: float = 0.9) -> TransferFunction:
    """transfer.py:88-98."""
    t = float(np.clip(threshold, 0.01, 0.95))
    return TransferFunction([[0.0, 0.0, 0.0, 0.1, 0.0], [t, 0.1, 0.05, 0.3, 0.0],
                             [min(t + 0.15, 0.97), 0.9, 0.45, 0.1, 0.55 * max_opacity],
                             [1.0, 1.0, 0.95, 0.8, max_opacity]])


@dataclass
class RenderSettings:
    """scene.py:16-26."""

    base_step_scale: float = 0.5
    mu_floor: float = 1.0 / 16.0
    early_termination: float = 0.01
    background: tuple = (0.0, 0.0, 0.0)
    skip_empty: bool = True
    adaptive_step: bool = True
    max_iterations: int = 8192
    pt_density: float = 60.0
    pt_ambient: float = 0.2
    light_dir: tuple = (-0.5, -0.8, -0.3)


def base_step(dims, settings) -> float:
    """scene.py:41-44."""
    vx, vy, vz = dims
    return settings.base_step_scale * float(np.linalg.norm([1.0 / vx, 1.0 / vy, 1.0 / vz]))


# -- path tracing host scalars (render/pathtrace.py) -----------------------------
PT_MAX_WALK = 100_000  # pathtrace.py:18 _MAX_WALK


def pcg64_seeded_state(seed: int):
    """(state, inc) of numpy's default_rng(seed) (PCG64 after SeedSequence), as the
    path tracer's stream starts (pathtrace.py:117).  The device advances it."""
    st = np.random.default_rng(int(seed)).bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise RuntimeError(f"numpy default_rng is {st['bit_generator']}, expected PCG64")
    return int(st["state"]["state"]), int(st["state"]["inc"])
