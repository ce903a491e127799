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
