"""Request-table configuration (voxcache/scheduler.py:22-40); the table itself
is device-resident (cache.DeviceCache) and driven by the maintenance kernels."""

from __future__ import annotations

from dataclasses import dataclass

RANK_CLAMP = 1000
DEFAULT_MAX_REQUESTS = 40


@dataclass(frozen=True)
class SchedulerConfig:
    max_requests: int = DEFAULT_MAX_REQUESTS
    ranking_enabled: bool = True
    rank_clamp: int = RANK_CLAMP
    # Frame scheduler (this package; north_star subsystem 4): INR samples decoded per
    # frame, true misses first, the brick batch gets the rest (at least one brick).
    # None = the reference's behaviour: every true miss decoded (sampler.py:276-279)
    # and max_requests bricks per frame (scheduler.py:152-169).
    decode_budget: int | None = None

    def __post_init__(self):
        if self.decode_budget is not None and self.decode_budget < 0:
            raise ValueError("decode_budget must be >= 0 (or None for unbounded)")
