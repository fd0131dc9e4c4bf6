"""GroupedLOMO: single-pass grouped-norm clipping on the GPU
(Stabilizer._grouped_step, fusedtrain/stabilize.py:234-274).

Gradients are retained per window of ``window`` adjacent layers (group =
layer // window, layers in the reference's numbering: embedding 0, decoder
blocks 1..L, final norm + head L+1, zoo.py:150-201).  When the first gradient
of the next group arrives -- and once more after backward -- the finished
group is flushed on the device with the same kernels as the two-pass path:
K2 over the group's gradients, K3a for the group's norm / clip factor /
non-finite skip, then K1 with ``coef`` for each gradient.  A group whose norm
is non-finite is dropped alone (earlier groups were already applied); the
step outcome is SKIPPED_OVERFLOW if any group was dropped.  One backward pass,
no second forward; biased relative to global clipping;
gradient peak = the largest group (pkg/README.md:103-107).
"""
from __future__ import annotations

import re
from typing import Callable

import torch

from . import _lib
from .engine import CudaEngine, dtype_code
from .errors import ConfigError, NonFiniteLossError, TapeStateError
from .lomo import trainable_params
from .stabilize import ClipMode, StepOutcome

_BLOCK = re.compile(r"(?:^|\.)(?:layers|block|blocks|h)[._]?(\d+)(?:\.|__|$)")


def infer_layers(model) -> dict[int, int]:
    """Reference layer index per parameter: decoder block i -> i+1, parameters
    registered before the first block -> 0, after the last block -> L+1."""
    named = [(n.replace("__", "."), p) for n, p in model.named_parameters() if p.requires_grad]
    blocks = []
    for n, _ in named:
        m = _BLOCK.search(n)
        blocks.append(int(m.group(1)) if m else None)
    nblocks = max([b for b in blocks if b is not None], default=-1) + 1
    out, seen_block = {}, False
    for (n, p), b in zip(named, blocks):
        if b is not None:
            seen_block = True
            out[id(p)] = b + 1
        else:
            out[id(p)] = nblocks + 1 if seen_block else 0
    return out


class GroupedLOMO:
    """LOMO with per-layer-window norm clipping in one backward pass.

    Args:
        model: torch module on one CUDA device.
        lr: default learning rate.
        max_norm, window: ``ClipMode.by_group_norm(max_norm, window)``.
        layer_of: optional ``{id(param): layer}``; default :func:`infer_layers`.
        math: ``"f32"`` or ``"f64"``.
    """

    def __init__(self, model, lr: float = 1e-3, max_norm: float = 1.0, window: int = 1, *,
                 layer_of: dict | None = None, math: str = "f32", weight_decay: float = 0.0):
        self.clip = ClipMode.by_group_norm(max_norm, window)  # validation (stabilize.py:65-74)
        params = trainable_params(model)
        dev = params[0].device
        for p in params:
            if p.device != dev:
                raise ConfigError("all parameters must live on one CUDA device")
            dtype_code(p.dtype)
        self.params = params
        self.lr = float(lr)
        self.weight_decay = float(weight_decay)
        self.layer = layer_of if layer_of is not None else infer_layers(model)
        missing = [p for p in params if id(p) not in self.layer]
        if missing:
            raise ConfigError(f"{len(missing)} parameters have no layer index")
        self.engine = CudaEngine(dev, len(params), None, float(max_norm), math)
        self._slot = {id(p): i for i, p in enumerate(reversed(params))}
        self._active = False
        self._buf: list[tuple[torch.Tensor, torch.Tensor]] = []
        self._group = None
        self._probe_flags = _lib.ACCUM_F64 if self.engine.math == _lib.MATH_F64 else 0
        self._skipped_before = 0
        self.last_outcome: StepOutcome | None = None
        self.peak_group_grads = 0
        self._handles = [p.register_post_accumulate_grad_hook(self._hook) for p in params]

    def _hook(self, p: torch.Tensor) -> None:
        if not self._active or p.grad is None:
            return
        g = p.grad if p.grad.is_contiguous() else p.grad.contiguous()
        p.grad = None  # RETAIN in our buffer (stabilize.py:260-266), not in .grad
        group = self.layer[id(p)] // self.clip.window
        if self._group is not None and group != self._group:
            self._flush()
        self._group = group
        self._buf.append((p, g))
        self.peak_group_grads = max(self.peak_group_grads,
                                    sum(x.numel() * x.element_size() for _, x in self._buf))

    def _flush(self) -> None:
        """stabilize.py:239-258 on the device: K2 -> K3a -> K1 for one group."""
        if not self._buf:
            return
        eng = self.engine
        eng.begin(None)                       # fresh slots / overflow for this group
        eng.configure(flags=self._probe_flags)
        for p, g in self._buf:
            eng.probe(g, self._slot[id(p)])
        eng.flush()
        eng.finalize()                        # N, coef = min(1, max_norm/N), skip if !finite
        eng.configure(self._lr, 0.0, self.weight_decay, _lib.USE_SKIP | _lib.USE_COEF)
        for p, g in self._buf:
            eng.update(p, g)
        eng.flush()
        self._buf = []                        # gradients released (stream-ordered)

    def fused_backward(self, loss: torch.Tensor, lr: float | None = None) -> None:
        """One grouped fused pass (stabilize.py:234-274)."""
        if not torch.isfinite(loss.detach()).all():   # _require_finite (optim.py:63-65)
            raise NonFiniteLossError(f"loss is non-finite ({float(loss.detach())}); step aborted")
        for p in self.params:
            if p.grad is not None:
                raise TapeStateError("a parameter already holds a gradient")
        self._lr = self.lr if lr is None else float(lr)
        self._active, self._group = True, None
        try:
            loss.backward()
            self._flush()
        finally:
            self._active, self._buf, self._group = False, [], None
        st = self.engine.read_status()
        skipped = st.steps_skipped > self._skipped_before
        self._skipped_before = st.steps_skipped
        self.last_outcome = StepOutcome.SKIPPED_OVERFLOW if skipped else StepOutcome.APPLIED

    def step(self, closure: Callable[[], torch.Tensor], lr: float | None = None) -> float:
        loss = closure()
        self.fused_backward(loss, lr)
        return float(loss.detach())

    def state_nbytes(self) -> int:
        return 0

    def remove_hooks(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []
