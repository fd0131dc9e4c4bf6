"""Stabiliser configuration, mirroring fusedtrain/stabilize.py's public types.

The arithmetic of every stabiliser runs on the GPU (K1/K2/K3 in
csrc/lomo_kernels.cu); this module only holds the configuration objects with
the reference's names, argument meaning and validation errors, so code
written against the reference keeps working:

* ``ClipMode``      stabilize.py:45-74   (none / by_value / by_global_norm / by_group_norm)
* ``LossScaler``    stabilize.py:94-127  (power-of-two dynamic scale: the
                    reference's live object -- ``scale``, ``clean_steps``,
                    ``on_overflow()``, ``on_clean()``; under LOMO the state
                    machine runs on device and the optimizer mirrors it here)
* ``Stabilizer``    stabilize.py:130-153 (pass count; scaler + group clip rejected)
* ``StepOutcome``   stabilize.py:77-79
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

from .errors import ConfigError, ScaleUnderflowError


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


class LossScaler:
    """Dynamic loss-scale state machine; the scale is always a power of two
    (stabilize.py:94-127): the reference's names, validation, live
    attributes and methods.

    Under :class:`~paper_2306_09782_b200.LOMO` the halve/double state machine
    runs on the device (K3a halves on overflow, K3b counts clean steps); the
    optimizer copies the device's ``scale`` and ``clean_steps`` into this
    object at each step's status read and applies ``on_clean()`` after an
    applied step (the same arithmetic K3b ran), so ``scaler.scale`` reads as
    the reference's does -- without an extra host sync.
    """

    def __init__(self, scale: float = 2.0 ** 10, growth_interval: int = 16,
                 min_scale: float = 1.0, max_scale: float = 2.0 ** 24):
        for name, value in (("scale", scale), ("min_scale", min_scale),
                            ("max_scale", max_scale)):
            if not is_power_of_two(value):
                raise ConfigError(f"{name} must be a positive power of two, got {value}")
        if not (min_scale <= scale <= max_scale):
            raise ConfigError(f"scale {scale} outside [{min_scale}, {max_scale}]")
        if growth_interval < 1:
            raise ConfigError(f"growth_interval must be >= 1, got {growth_interval}")
        self.scale = float(scale)
        self.growth_interval = int(growth_interval)
        self.min_scale = float(min_scale)
        self.max_scale = float(max_scale)
        self.clean_steps = 0

    def on_overflow(self) -> None:
        """stabilize.py:115-121: halve, or raise when below min_scale."""
        if self.scale / 2.0 < self.min_scale:
            raise ScaleUnderflowError(
                f"loss scale would fall below {self.min_scale}; training diverged")
        self.scale /= 2.0
        self.clean_steps = 0

    def on_clean(self) -> None:
        """stabilize.py:123-127: double after growth_interval clean steps."""
        self.clean_steps += 1
        if self.clean_steps >= self.growth_interval:
            self.scale = min(self.scale * 2.0, self.max_scale)
            self.clean_steps = 0

    def _mirror(self, status) -> None:
        """Copy the device state machine's values (a lomo_status snapshot)."""
        self.scale = float(status.scale)
        self.clean_steps = int(status.clean_steps)

    def __repr__(self) -> str:
        return (f"LossScaler(scale={self.scale}, growth_interval={self.growth_interval}, "
                f"min_scale={self.min_scale}, max_scale={self.max_scale}, "
                f"clean_steps={self.clean_steps})")


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

    def run_step(self, model, batch, lr: float, **lomo_kwargs):
        """One stabilised fused step (stabilize.py:148-153): ``batch`` is
        ``(inputs, targets)`` for ``model.loss`` or a closure returning the
        loss.  Returns ``(loss, StepOutcome)``; the scaler object carries its
        state from step to step, as the reference's does.  (A thin wrapper:
        hooks are registered for this one step -- long loops keep one
        :class:`~paper_2306_09782_b200.LOMO`.)"""
        from .grouped import GroupedLOMO
        from .lomo import LOMO
        if self.clip.kind is ClipKind.BY_GROUP_NORM:
            opt = GroupedLOMO(model, lr, max_norm=self.clip.max_norm, window=self.clip.window,
                              **lomo_kwargs)
        else:
            opt = LOMO(model, lr, stabilizer=self, **lomo_kwargs)
        try:
            loss = opt.step(batch, lr)
            outcome = opt.last_outcome
            return loss, (StepOutcome.APPLIED if outcome is None else outcome)
        finally:
            opt.remove_hooks()


def clip_by_value(grad, threshold: float):
    """stabilize.py:82-86: clamp every element to [-threshold, threshold]
    (NaN stays NaN, as np.clip); K1's ``clip_value`` applies it in place."""
    if threshold <= 0:
        raise ConfigError(f"clip threshold must be positive, got {threshold}")
    return grad.clamp(-threshold, threshold)


def two_pass_norm_clip_step(model, batch, lr: float, max_norm: float, **lomo_kwargs) -> float:
    """stabilize.py:277-280: global-norm-clipped fused step (two passes)."""
    loss, _ = Stabilizer(ClipMode.by_global_norm(max_norm)).run_step(model, batch, lr,
                                                                     **lomo_kwargs)
    return loss


def grouped_norm_clip_step(model, batch, lr: float, max_norm: float, window: int,
                           **lomo_kwargs) -> float:
    """stabilize.py:283-289: single-pass step with per-layer-window clipping."""
    loss, _ = Stabilizer(ClipMode.by_group_norm(max_norm, window)).run_step(model, batch, lr,
                                                                            **lomo_kwargs)
    return loss


def scaled_step(model, batch, lr: float, scaler: LossScaler, clip: ClipMode = ClipMode(),
                **lomo_kwargs):
    """stabilize.py:292-295: loss-scaled fused step under the two-pass protocol."""
    return Stabilizer(clip, scaler).run_step(model, batch, lr, **lomo_kwargs)
