"""Render API types: Camera (camera.py:15-66), TransferFunction (transfer.py:13-98),
RenderSettings (scene.py:16-26).  Host-side value objects; the arithmetic that
feeds the kernels (camera basis, LUT, base step) reproduces the reference's
numpy expressions exactly so GPU rays match the reference bit for bit.
"""

from __future__ import annotations

import json
import math
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


_TAN_HALF = {}


def _norm3(v) -> float:
    """np.linalg.norm of a 3-vector: numpy computes sqrt(x.dot(x)) (linalg.norm, ord
    None), so this is that expression without norm's argument handling."""
    a = np.array(v)
    return math.sqrt(a.dot(a))


def camera_frame_setup(cam):
    """camera_rays_setup + the camera's distance to the unit box, flat, for the per-frame
    kernel parameters: (origin3, rot9 row-major, tan_h, tan_v, box_distance).  The
    same operations as camera_basis / camera_rays_setup / point_to_unit_box
    (sampler.py:283-285), bit for bit (tests/test_host_cpu.py); tan(fov/2) is cached per
    fov (np.tan, as before)."""
    p, t, u = cam.position, cam.target, cam.up
    p0, p1, p2 = float(p[0]), float(p[1]), float(p[2])
    fwd = (float(t[0]) - p0, float(t[1]) - p1, float(t[2]) - p2)
    n = _norm3(fwd)
    fwd = (fwd[0] / n, fwd[1] / n, fwd[2] / n)
    right = _cross(fwd, (float(u[0]), float(u[1]), float(u[2])))
    n = _norm3(right)
    right = (right[0] / n, right[1] / n, right[2] / n)
    up = _cross(right, fwd)
    th = _TAN_HALF.get(cam.fov_y)
    if th is None:
        th = _TAN_HALF.setdefault(cam.fov_y, float(np.tan(np.radians(cam.fov_y) / 2.0)))
    gap = (max(max(-p0, p0 - 1.0), 0.0), max(max(-p1, p1 - 1.0), 0.0), max(max(-p2, p2 - 1.0), 0.0))
    return ((p0, p1, p2), (right[0], up[0], fwd[0], right[1], up[1], fwd[1], right[2], up[2], fwd[2]),
            float(th * (cam.width / cam.height)), th, _norm3(gap))


def _checked_points(points) -> np.ndarray:
    """Control points as a read-only (n, 5) f64 array: x from 0 to 1 strictly
    increasing, colour and opacity in [0, 1] (transfer.py:16-27's rules)."""
    pts = np.array(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 5 or len(pts) < 2:
        raise ConfigError("a transfer function is at least two (x, r, g, b, a) rows")
    xs = pts[:, 0]
    if not (xs[0] == 0.0 and xs[-1] == 1.0 and np.all(xs[1:] > xs[:-1])):
        raise ConfigError("transfer-function x must run strictly upward from 0 to 1")
    if np.any((pts[:, 1:] < 0.0) | (pts[:, 1:] > 1.0)):
        raise ConfigError("transfer-function colour/opacity outside [0, 1]")
    pts.flags.writeable = False
    return pts


class TransferFunction:
    """Piecewise-linear colour/opacity of a normalized value (transfer.py:13-78): the
    control points, their interpolation, and the dense LUT the shade samples."""

    def __init__(self, points):
        self.points = _checked_points(points)
        self._tables = {}

    def _interp(self, values, column):
        v = np.clip(np.asarray(values, dtype=np.float64), 0.0, 1.0)
        return np.interp(v, self.points[:, 0], self.points[:, column])

    def eval(self, values) -> np.ndarray:
        """rgba (..., 4) f64 at each value (clamped to [0, 1])."""
        return np.stack([self._interp(values, c) for c in (1, 2, 3, 4)], axis=-1)

    def opacity(self, values) -> np.ndarray:
        return self._interp(values, 4)

    def lookup_table(self, size: int = 1024) -> np.ndarray:
        """(size, 4) f32 rgba at size evenly spaced values; built once per size."""
        if size not in self._tables:
            self._tables[size] = self.eval(np.linspace(0.0, 1.0, size)).astype(np.float32)
        return self._tables[size]

    def to_json(self):
        return [dict(x=float(x), rgb=[float(r), float(g), float(b)], a=float(a)) for x, r, g, b, a in self.points]

    @classmethod
    def from_json(cls, data) -> "TransferFunction":
        try:
            rows = [(e["x"], *e["rgb"][:3], e["a"]) for e in data]
        except (KeyError, TypeError, IndexError) as exc:
            raise ConfigError(f"transfer-function JSON is malformed: {exc}") from exc
        return cls(rows)

    @classmethod
    def load(cls, path) -> "TransferFunction":
        return cls.from_json(json.loads(Path(path).read_text()))


# presets (transfer.py:80-98): the same control points
def grayscale_ramp(max_opacity: float = 1.0) -> TransferFunction:
    return TransferFunction([(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, max_opacity)])


def transparent() -> TransferFunction:
    return grayscale_ramp(0.0)


def warm_body(threshold: float = 0.35, max_opacity: float = 0.9) -> TransferFunction:
    """Transparent below `threshold` (clamped to [0.01, 0.95]), warm and opaque above."""
    t = min(max(float(threshold), 0.01), 0.95)
    return TransferFunction([(0.0, 0.0, 0.0, 0.1, 0.0),
                             (t, 0.1, 0.05, 0.3, 0.0),
                             (min(t + 0.15, 0.97), 0.9, 0.45, 0.1, 0.55 * max_opacity),
                             (1.0, 1.0, 0.95, 0.8, max_opacity)])


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
