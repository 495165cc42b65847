"""Host half of adaptive stale aggregation, mirroring the reference API
(stale.py:42-108): StaleMode, StaleConfig, EpochLossTrace and threshold().
The per-key decision (filter_transmissions, stale.py:154-176) runs on the GPU
(K5, csrc/stale.cu); see EmbeddingCacheGPU / filter_transmissions_gpu."""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import torch

from . import ops


class StaleMode(str, Enum):
    OFF = "off"
    STATIC = "static"
    ADAPTIVE_TIGHTEN = "adaptive-tighten"
    ADAPTIVE_RELAX = "adaptive-relax"


@dataclass(frozen=True)
class StaleConfig:
    mode: StaleMode = StaleMode.OFF
    static_fraction: float = 0.5

    def __post_init__(self):
        object.__setattr__(self, "mode", StaleMode(getattr(self.mode, "value", self.mode)))
        if not 0.0 <= self.static_fraction <= 1.0:
            raise ValueError("static_fraction must be in [0, 1]")

    @classmethod
    def off(cls):
        return cls(StaleMode.OFF)

    @classmethod
    def static(cls, fraction: float):
        return cls(StaleMode.STATIC, fraction)

    @classmethod
    def adaptive(cls, tighten: bool = False):
        return cls(StaleMode.ADAPTIVE_TIGHTEN if tighten else StaleMode.ADAPTIVE_RELAX)

    @classmethod
    def coerce(cls, cfg) -> "StaleConfig":
        """Accept the reference's dynpart.StaleConfig (duck-typed) unchanged."""
        if isinstance(cfg, cls):
            return cfg
        if cfg is None:
            return cls.off()
        return cls(StaleMode(getattr(cfg.mode, "value", cfg.mode)), float(cfg.static_fraction))


@dataclass
class EpochLossTrace:
    losses: list = field(default_factory=list)

    def append(self, loss: float) -> None:
        if not self.losses and loss <= 0:
            raise ValueError("initial loss must be > 0")
        self.losses.append(float(loss))

    def progress(self, r: int) -> float:
        if r < 2:
            raise ValueError("progress is defined from epoch 2 on")
        if len(self.losses) < r - 1:
            raise ValueError(f"no loss recorded for epoch {r - 1}")
        l1 = self.losses[0]
        return (l1 - self.losses[r - 2]) / l1


def threshold(trace: EpochLossTrace, r: int, d_r: float, config: StaleConfig) -> float:
    """stale.py:97-108 verbatim semantics."""
    if d_r < 0:
        raise ValueError("d_r must be >= 0")
    if config.mode is StaleMode.OFF:
        return 0.0
    if config.mode is StaleMode.STATIC:
        return config.static_fraction * d_r
    p = trace.progress(r)
    if config.mode is StaleMode.ADAPTIVE_TIGHTEN:
        return d_r / (1.0 + math.exp(p))
    return d_r / (1.0 + math.exp(-p))


class EmbeddingCacheGPU:
    """Device-resident last-transmitted cache for a fixed key set
    (stale.py:111-130; one copy per boundary key)."""

    def __init__(self, n_keys: int, width: int, device):
        self.values = torch.zeros((n_keys, width), dtype=torch.float32, device=device)
        self.cached = torch.zeros(n_keys, dtype=torch.uint8, device=device)
        self.dist = torch.zeros(n_keys, dtype=torch.float32, device=device)
        self.send = torch.ones(n_keys, dtype=torch.uint8, device=device)
        self.dmax = torch.zeros(1, dtype=torch.float32, device=device)
        self.width = width


def filter_transmissions_gpu(Y, key_rows, cache: EmbeddingCacheGPU, theta: float):
    """K5 on the GPU: the decision half of stale.py:154-176 for rows
    Y[key_rows]; returns the device send mask (uint8). ``theta`` comes from
    threshold() with D_r = the max of dgc_stale_distance (global over ranks)."""
    ops.stale_select(Y, key_rows, cache.dist, theta, cache.values, cache.cached, cache.send,
                     cache.width)
    return cache.send


def cache_gap_gpu(Y, key_rows, cache: EmbeddingCacheGPU):
    """K5 distance half (stale.py:140-151,205-212): fills cache.dist and
    cache.dmax (max over cached keys)."""
    ops.stale_distance(Y, key_rows, cache.values, cache.cached, cache.width, cache.dist, cache.dmax)
    return cache.dmax
