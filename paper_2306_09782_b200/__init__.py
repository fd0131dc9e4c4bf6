"""B200-native LOMO fused gradient-compute + parameter-update path.

Drop-in for the per-parameter update hook of the reference ``fusedtrain``
(optim.py:101-132, stabilize.py:130-230): PyTorch autograd drives the
backward, a post-accumulate-grad hook per parameter calls the C-ABI of
``liblomo_b200.so`` (include/lomo_b200.h), whose sm_100a kernels fuse
unscale, overflow detection, clipping, weight decay and ``p -= lr*g``.
"""
from .errors import (ConfigError, FusedTrainError, NativeError, NonFiniteLossError,
                     ScaleUnderflowError, ShapeError, TapeStateError)
from .engine import apply_update
from .grouped import GroupedLOMO
from .lomo import LOMO, lomo_step
from .stabilize import (ClipKind, ClipMode, LossScaler, Stabilizer, StepOutcome, clip_by_value,
                        grouped_norm_clip_step, scaled_step, two_pass_norm_clip_step)

__all__ = [
    "LOMO", "GroupedLOMO", "lomo_step", "apply_update", "ClipKind", "ClipMode", "LossScaler", "Stabilizer", "StepOutcome",
    "clip_by_value", "two_pass_norm_clip_step", "grouped_norm_clip_step", "scaled_step",
    "ConfigError", "FusedTrainError", "NativeError", "NonFiniteLossError",
    "ScaleUnderflowError", "ShapeError", "TapeStateError",
]
