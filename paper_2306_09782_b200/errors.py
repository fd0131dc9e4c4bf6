"""Exception types, named after the reference's (fusedtrain/errors.py:1-37).

Only the ones the fused-update path can raise are mirrored; the error
conventions follow the reference: a non-finite loss without a stabiliser
aborts the step with parameters untouched (optim.py:63-65), and a loss scale
that would fall below its minimum is fatal (stabilize.py:115-119).
"""
from __future__ import annotations


class FusedTrainError(Exception):
    """Base class (errors.py:4-5)."""


class ShapeError(FusedTrainError):
    """Gradient/parameter extents disagree (tape.py:388-393)."""

    def __init__(self, op: str, message: str):
        super().__init__(f"{op}: {message}")
        self.op = op


class TapeStateError(FusedTrainError):
    """Protocol misuse, e.g. fused_backward before grad_norm (tape.py:337-339)."""


class NonFiniteLossError(FusedTrainError):
    """The loss became NaN/inf outside of scaled training (errors.py:28-29)."""


class ScaleUnderflowError(FusedTrainError):
    """The dynamic loss scale fell below its minimum (errors.py:32-33)."""


class ConfigError(FusedTrainError):
    """Invalid optimizer / stabiliser configuration (errors.py:36-37)."""


class NativeError(FusedTrainError):
    """A C-ABI call into liblomo_b200.so returned a non-zero status."""
