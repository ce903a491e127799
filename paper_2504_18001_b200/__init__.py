"""B200-native cached-INR volume renderer (drop-in for voxcache's ray-march path).

Public API mirrors the reference package (voxcache): fields, INR model, camera,
transfer function, cache/scheduler/LoD configs and RenderSession.render_frame().
Compute runs in libcinr_b200.so (hand-written sm_100a CUDA); torch only owns
device memory and streams.  There is no CPU fallback.
"""

from .cache import BrickKey, BrickLayout, CacheConfig, PoolSpec
from .errors import (ConfigError, DomainError, IngestionError, ModelCorruptError, RenderError,
                     TrainingDivergedError, VoxcacheError, WeightFormatError)
from .fields import Field, FieldDomain, ProceduralField, RawLatticeField, make_procedural
from .inr import HashGridConfig, InrField, InrModel, MLPConfig
from .render import Camera, RenderSettings, TransferFunction, grayscale_ramp, transparent, warm_body
from .sampler import LodPolicy, effective_lod_scale, force_max_scale
from .scheduler import SchedulerConfig
from .weights_io import load_weights, save_weights

__version__ = "0.1.0"


def __getattr__(name):
    # session/harness/macrocell import torch lazily-heavy modules on first use
    if name in ("RenderSession", "SessionConfig", "FrameRecord"):
        from . import session

        return getattr(session, name)
    if name in ("OrbitTrajectory", "BenchReport", "bench_run"):
        from . import harness

        return getattr(harness, name)
    # voxcache.inr's training API (the function itself is paper_2504_18001_b200.train.train,
    # like voxcache.inr.train.train: the submodule owns the package attribute `train`)
    if name in ("loss_and_grads", "psnr_on_lattice", "TrainResult"):
        import importlib

        mod = importlib.import_module(".train", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
