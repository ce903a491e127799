"""Reference-free scene recipes shared by the golden generator, the oracle tests
and the GPU parity tests. Nothing here imports the reference or the product.

`smoothed_random_lattice` restates the reference test fixture
`random_lattice_field` (pkg/tests/conftest.py:12-22): a seeded uniform lattice,
three passes of a [1/4, 1/2, 1/4] periodic blur (np.roll), then min/max
normalisation — all in float32 exactly as the fixture does it.
"""

from __future__ import annotations

import numpy as np


def smoothed_random_lattice(dims, seed=0, smooth=True):
    vx, vy, vz = dims
    lat = np.random.default_rng(seed).random((vz, vy, vx)).astype(np.float32)
    if smooth:
        for axis in range(3):
            lat = 0.5 * lat + 0.25 * (np.roll(lat, 1, axis) + np.roll(lat, -1, axis))
        lat -= lat.min()
        lat /= max(lat.max(), 1e-9)
    return lat.astype(np.float32)


# Each spec is one inline-loader session recorded frame by frame (golden) and
# replayed by the oracle / CUDA path. Keys:
#   field: lattice | inr | sphere...; dims; tf: ("warm_body", t, a) | ("grayscale_ramp", a)
#   brick, pool, cache_kw (CacheConfig extras), sched_kw (SchedulerConfig),
#   policy (LodPolicy kwargs), settings (RenderSettings kwargs), res (W, H),
#   frames, cam_step (orbit frames per session frame), events {frame: (...)}.
SESSION_SPECS = {
    # config-1 shape on an exactly-reproducible field: B16, 4^3 pool, direct tables
    "lattice64": dict(
        field="lattice", field_seed=7, dims=(64, 64, 64), tf=("warm_body", 0.45, 0.9),
        brick=16, pool=(4, 4, 4), policy=dict(lod_scale=1.2, preload_frames=8),
        res=(96, 96), frames=24, cam_step=5, op_frame=12,
    ),
    # same, forced onto the 2-level paged MRPD (test_cache.py:184-200 knobs):
    # the reference then uses the numpy lookup with |pos-cam| distances (sampler.py:135)
    "lattice64_paged": dict(
        field="lattice", field_seed=7, dims=(64, 64, 64), tf=("warm_body", 0.45, 0.9),
        brick=16, pool=(4, 4, 4), cache_kw=dict(direct_table_threshold=8, page_size=4, page_budget=2),
        policy=dict(lod_scale=1.2, preload_frames=8), res=(64, 64), frames=16, cam_step=5,
    ),
    # FIFO scheduling, as_printed LoD rule, fixed-ladder stepping, tiny pool (eviction + deferral)
    "lattice64_fifo": dict(
        field="lattice", field_seed=11, dims=(64, 64, 64), tf=("warm_body", 0.5, 0.95),
        brick=16, pool=(2, 2, 2), sched_kw=dict(max_requests=6, ranking_enabled=False),
        policy=dict(lod_scale=1.5, preload_frames=4, mode="as_printed"),
        settings=dict(adaptive_step=False), res=(64, 64), frames=20, cam_step=7,
    ),
    # anisotropic dims, non-power-of-two brick (Python float floor-division path), mode off
    "aniso_b10": dict(
        field="lattice", field_seed=3, dims=(40, 48, 56), tf=("warm_body", 0.4, 0.9),
        brick=10, pool=(3, 3, 3), policy=dict(lod_scale=2.0, preload_frames=3, mode="off"),
        settings=dict(skip_empty=False), res=(64, 48), frames=14, cam_step=9, radius=1.9,
    ),
    # control-plane events: TF switch (majorants), reset_cache (two clocks), lod scale change
    "events": dict(
        field="lattice", field_seed=5, dims=(64, 64, 64), tf=("warm_body", 0.45, 0.9),
        brick=16, pool=(3, 3, 3), sched_kw=dict(max_requests=10),
        policy=dict(lod_scale=1.2, preload_frames=5), res=(64, 64), frames=20, cam_step=3,
        events={8: ("tf", ("grayscale_ramp", 0.8)), 12: ("reset",), 15: ("lod_scale", 0.6)},
    ),
    # cache pressure: B8 (729 LoD-0 bricks), 18-slot pool, 7 requests/frame -> pending
    # entries carry over, LRU eviction, deferred inserts, exclusion of mapped keys
    "pressure": dict(
        field="lattice", field_seed=13, dims=(64, 64, 64), tf=("warm_body", 0.4, 0.9),
        brick=8, pool=(3, 3, 2), sched_kw=dict(max_requests=7),
        policy=dict(lod_scale=0.5, preload_frames=2), res=(80, 72), frames=22, cam_step=2, radius=1.7,
    ),
    "pressure_fifo": dict(
        field="lattice", field_seed=13, dims=(64, 64, 64), tf=("warm_body", 0.4, 0.9),
        brick=8, pool=(3, 3, 2), sched_kw=dict(max_requests=7, ranking_enabled=False, rank_clamp=3),
        policy=dict(lod_scale=0.5, preload_frames=2), res=(80, 72), frames=16, cam_step=2, radius=1.7,
    ),
    # config 1 proper: random-init hash-grid INR (values tolerance-checked, P14)
    "inr64": dict(
        field="inr", dims=(64, 64, 64), tf=("warm_body", 0.5, 0.9),
        brick=16, pool=(4, 4, 4), policy=dict(lod_scale=1.2, preload_frames=20),
        res=(64, 64), frames=12, cam_step=10,
    ),
    # BASELINE config 1 at its stated size: 64^3 random-init INR, B16, the 2-level paged
    # MRPD (test_cache.py:184-200 knobs), 4^3 pool, 256x256, the full 120-frame orbit,
    # warm_body(0.5, 0.9), LodPolicy(1.2, preload 20), 40 requests/frame
    # (images kept every 20th frame: tests/golden/make_config1.py)
    "config1": dict(
        field="inr", dims=(64, 64, 64), tf=("warm_body", 0.5, 0.9),
        brick=16, pool=(4, 4, 4), cache_kw=dict(direct_table_threshold=8, page_size=4, page_budget=2),
        policy=dict(lod_scale=1.2, preload_frames=20), res=(256, 256), frames=120, cam_step=1,
    ),
    # uncached INR baseline (every sample inferred; session.py:63-70)
    "inr_uncached": dict(
        field="inr", dims=(32, 32, 32), tf=("warm_body", 0.5, 0.9), cached=False,
        brick=16, pool=(2, 2, 2), policy=dict(lod_scale=1.2, preload_frames=20),
        res=(48, 48), frames=2, cam_step=30,
    ),
    # path tracing (pathtrace.py:112-146, §8f row 2): Woodcock delta tracking over the
    # majorants with the numpy PCG64 stream, the same cached sampler, shadow rays
    "pt_lattice64": dict(
        field="lattice", field_seed=7, dims=(64, 64, 64), tf=("warm_body", 0.45, 0.9), mode="pathtrace", spp=2,
        brick=16, pool=(4, 4, 4), policy=dict(lod_scale=1.2, preload_frames=3),
        settings=dict(pt_density=25.0), res=(48, 48), frames=8, cam_step=5,
    ),
    "pt_pressure": dict(
        field="lattice", field_seed=13, dims=(64, 64, 64), tf=("warm_body", 0.4, 0.9), mode="pathtrace", spp=1,
        brick=8, pool=(3, 3, 2), sched_kw=dict(max_requests=7),
        policy=dict(lod_scale=0.5, preload_frames=2, mode="as_printed"),
        settings=dict(pt_density=60.0, background=(0.1, 0.2, 0.3), light_dir=(0.3, -1.0, 0.2)),
        res=(40, 36), frames=8, cam_step=2, radius=1.7, seed=5,
    ),
    "pt_inr": dict(
        field="inr", dims=(64, 64, 64), tf=("warm_body", 0.5, 0.9), mode="pathtrace", spp=1,
        brick=16, pool=(4, 4, 4), policy=dict(lod_scale=1.2, preload_frames=20),
        settings=dict(pt_density=40.0), res=(40, 40), frames=5, cam_step=10,
    ),
    "pt_inr_uncached": dict(
        field="inr", dims=(32, 32, 32), tf=("warm_body", 0.5, 0.9), mode="pathtrace", spp=1, cached=False,
        brick=16, pool=(2, 2, 2), policy=dict(lod_scale=1.2, preload_frames=20),
        settings=dict(pt_density=40.0), res=(32, 32), frames=2, cam_step=30,
    ),
    # anisotropic dims, non-power-of-two brick, LoD mode off, spp 3, seed 2
    "pt_aniso": dict(
        field="lattice", field_seed=3, dims=(40, 48, 56), tf=("warm_body", 0.4, 0.9), mode="pathtrace", spp=3,
        brick=10, pool=(3, 3, 3), policy=dict(lod_scale=2.0, preload_frames=3, mode="off"),
        settings=dict(pt_density=35.0, pt_ambient=0.35), res=(40, 32), frames=6, cam_step=9, radius=1.9, seed=2,
    ),
}
