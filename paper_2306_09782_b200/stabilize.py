"""Stabiliser configuration, mirroring fusedtrain/stabilize.py's public types.

The arithmetic of every stabiliser runs on the GPU (K1/K2/K3 in
csrc/lomo_kernels.cu); this module only holds the configuration objects with
the reference's names, argument meaning and validation errors, so code
written against the reference keeps working:

* ``ClipMode``      stabilize.py:45-74   (none / by_value / by_global_norm / by_group_norm)
* ``LossScaler``    stabilize.py:94-127  (power-of-two dynamic scale; the state
                    machine itself runs on device, see ``LOMO.loss_scale``)
* ``Stabilizer``    stabilize.py:130-153 (pass count; scaler + group clip rejected)
* ``StepOutcome``   stabilize.py:77-79
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

from .errors import ConfigError


class ClipKind(Enum):
    NONE = "none"
    BY_VALUE = "by_value"
    BY_GLOBAL_NORM = "by_global_norm"
    BY_GROUP_NORM = "by_group_norm"


@dataclass(frozen=True)
class ClipMode:
    """stabilize.py:45-74."""

    kind: ClipKind = ClipKind.NONE
    threshold: float | None = None
    max_norm: float | None = None
    window: int | None = None

    @staticmethod
    def none() -> "ClipMode":
        return ClipMode()

    @staticmethod
    def by_value(threshold: float) -> "ClipMode":
        if threshold <= 0:
            raise ConfigError(f"clip threshold must be positive, got {threshold}")
        return ClipMode(ClipKind.BY_VALUE, threshold=float(threshold))

    @staticmethod
    def by_global_norm(max_norm: float) -> "ClipMode":
        if max_norm <= 0:
            raise ConfigError(f"max_norm must be positive, got {max_norm}")
        return ClipMode(ClipKind.BY_GLOBAL_NORM, max_norm=float(max_norm))

    @staticmethod
    def by_group_norm(max_norm: float, window: int) -> "ClipMode":
        if max_norm <= 0:
            raise ConfigError(f"max_norm must be positive, got {max_norm}")
        if window < 1:
            raise ConfigError(f"group window must be >= 1, got {window}")
        return ClipMode(ClipKind.BY_GROUP_NORM, max_norm=float(max_norm), window=int(window))


class StepOutcome(Enum):
    APPLIED = "applied"
    SKIPPED_OVERFLOW = "skipped_overflow"


def is_power_of_two(x: float) -> bool:
    """stabilize.py:89-91."""
    mantissa, _ = math.frexp(x)
    return x > 0 and mantissa == 0.5


@dataclass(frozen=True)
class LossScaler:
    """Dynamic loss-scale configuration (stabilize.py:94-113).

    Validation is the reference's; the halve/double state machine
    (stabilize.py:115-127) runs on device inside K3a/K3b.
    """

    scale: float = 2.0 ** 10
    growth_interval: int = 16
    min_scale: float = 1.0
    max_scale: float = 2.0 ** 24

    def __post_init__(self):
        for name, value in (("scale", self.scale), ("min_scale", self.min_scale),
                            ("max_scale", self.max_scale)):
            if not is_power_of_two(value):
                raise ConfigError(f"{name} must be a positive power of two, got {value}")
        if not (self.min_scale <= self.scale <= self.max_scale):
            raise ConfigError(f"scale {self.scale} outside [{self.min_scale}, {self.max_scale}]")
        if self.growth_interval < 1:
            raise ConfigError(f"growth_interval must be >= 1, got {self.growth_interval}")


@dataclass(frozen=True)
class Stabilizer:
    """A clip mode plus an optional scaler; decides the pass count (stabilize.py:130-146)."""

    clip: ClipMode = ClipMode()
    scaler: LossScaler | None = None

    def __post_init__(self):
        if self.scaler is not None and self.clip.kind is ClipKind.BY_GROUP_NORM:
            raise ConfigError(
                "grouped clipping is the single-pass alternative and does not "
                "combine with the loss scaler; use by_global_norm instead"
            )

    @property
    def backward_passes_per_step(self) -> int:
        two = self.scaler is not None or self.clip.kind is ClipKind.BY_GLOBAL_NORM
        return 2 if two else 1
