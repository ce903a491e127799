"""Hash-grid INR model (voxcache/inr/encoding.py, mlp.py, model.py) with GPU inference.

Parameters live on the host as numpy (same draw order as the reference, so
`InrModel(..., seed=s)` reproduces the reference weights bit for bit) and are
uploaded once per device by `device.device_field`.  Inference runs in the
sm_100a decoder (vcb_field_points / vcb_field_bricks).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, ModelCorruptError
from .fields import Field, FieldDomain, check_positions


@dataclass(frozen=True)
class HashGridConfig:
    """encoding.py:30-64."""

    levels: int = 8
    features_per_entry: int = 2
    base_resolution: int = 4
    growth_factor: float = 1.5
    table_size: int = 1 << 16

    def __post_init__(self):
        if self.levels < 1 or self.features_per_entry < 1:
            raise ConfigError("levels and features_per_entry must be >= 1")
        if self.growth_factor <= 1.0:
            raise ConfigError("growth_factor must be > 1")
        if self.base_resolution < 1:
            raise ConfigError("base_resolution must be >= 1")
        t = self.table_size
        if t < 1 or (t & (t - 1)) != 0:
            raise ConfigError("table_size must be a power of two")

    def resolution(self, level: int) -> int:
        return int(np.floor(self.base_resolution * self.growth_factor ** level))

    def resolutions(self):
        return [self.resolution(l) for l in range(self.levels)]

    def level_is_dense(self, level: int) -> bool:
        return (self.resolution(level) + 1) ** 3 <= self.table_size

    def level_entries(self, level: int) -> int:
        dense = (self.resolution(level) + 1) ** 3
        return dense if dense <= self.table_size else self.table_size

    @property
    def output_dim(self) -> int:
        return self.levels * self.features_per_entry


@dataclass(frozen=True)
class MLPConfig:
    """mlp.py:13-25."""

    hidden_width: int = 32
    hidden_layers: int = 2
    activation: str = "relu"
    output_activation: str = "sigmoid"

    def __post_init__(self):
        if self.hidden_width < 1 or self.hidden_layers < 1:
            raise ConfigError("hidden width and layer count must be >= 1")
        if self.activation != "relu":
            raise ConfigError(f"unsupported activation {self.activation!r}")
        if self.output_activation not in ("sigmoid", "clamp"):
            raise ConfigError(f"unsupported output activation {self.output_activation!r}")


def init_mlp(config: MLPConfig, input_dim: int, rng, dtype=np.float32):
    """mlp.py:28-36: uniform +-1/sqrt(fan_in) weights (out, in), zero biases."""
    dims = [input_dim] + [config.hidden_width] * config.hidden_layers + [1]
    weights, biases = [], []
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        bound = 1.0 / np.sqrt(fan_in)
        weights.append(rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(dtype))
        biases.append(np.zeros(fan_out, dtype=dtype))
    return weights, biases


class InrModel:
    """model.py:14-78: tables coarsest-first, then weights, then biases."""

    def __init__(self, grid_config: HashGridConfig, mlp_config: MLPConfig, domain: FieldDomain, seed: int = 0,
                 dtype=np.float32):
        self.grid_config = grid_config
        self.mlp_config = mlp_config
        self.domain = domain
        self.dtype = np.dtype(dtype)
        if self.dtype != np.float32:
            raise ConfigError("the GPU decoder evaluates float32 models")
        rng = np.random.default_rng(seed)
        self.tables = [
            rng.uniform(-1e-4, 1e-4, size=(grid_config.level_entries(l), grid_config.features_per_entry)).astype(
                self.dtype)
            for l in range(grid_config.levels)
        ]
        self.weights, self.biases = init_mlp(mlp_config, grid_config.output_dim, rng, self.dtype)
        self._version = 0

    def parameters(self):
        return [*self.tables, *self.weights, *self.biases]

    def parameter_names(self):
        return ([f"grid{l}" for l in range(len(self.tables))] + [f"w{i}" for i in range(len(self.weights))]
                + [f"b{i}" for i in range(len(self.biases))])

    def set_parameters(self, params):
        nt, nw = len(self.tables), len(self.weights)
        self.tables = [np.asarray(p, dtype=self.dtype) for p in params[:nt]]
        self.weights = [np.asarray(p, dtype=self.dtype) for p in params[nt:nt + nw]]
        self.biases = [np.asarray(p, dtype=self.dtype) for p in params[nt + nw:]]
        self._version += 1

    def all_finite(self) -> bool:
        return all(np.isfinite(p).all() for p in self.parameters())

    def infer_batch(self, positions) -> np.ndarray:
        """model.py:65-75 on the GPU; non-finite outputs raise ModelCorruptError."""
        pos = check_positions(positions)
        if pos.shape[0] == 0:
            return np.zeros(0, dtype=np.float32)
        from .device import device_field, field_points

        out, bad = field_points(device_field(self.as_field(), clip=False), pos, return_flag=True)
        if bad:
            if not self.all_finite():
                raise ModelCorruptError("model parameters contain non-finite values")
            raise ModelCorruptError("inference produced non-finite outputs")
        return out

    def as_field(self) -> "InrField":
        f = getattr(self, "_field", None)
        if f is None:
            f = InrField(self)
            self._field = f
        return f


class InrField(Field):
    """model.py:81-89: the model as a Field (outputs clipped to [0,1])."""

    def __init__(self, model: InrModel):
        super().__init__(model.domain)
        self.model = model

    def sample_batch(self, positions) -> np.ndarray:
        pos = check_positions(positions)
        if pos.shape[0] == 0:
            return np.zeros(0, dtype=np.float32)
        from .device import device_field, field_points

        out, bad = field_points(device_field(self), pos, return_flag=True)
        if bad:
            raise ModelCorruptError("inference produced non-finite outputs")
        return out
