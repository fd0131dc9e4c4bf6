"""LOMO: the fused gradient-compute + parameter-update optimizer (B200 path).

Public API (the north-star names, OpenLMLab LOMO style)::

    opt = LOMO(model, lr, clip_grad_norm=None, loss_scale=None)
    loss = model(...)                 # forward (PyTorch)
    opt.grad_norm(loss)               # pass 1 (only when two passes are needed)
    opt.fused_backward(loss, lr)      # pass 2 / the single fused pass

plus the reference's step protocol as an adapter (``step(closure, lr)``,
fusedtrain/optim.py:118-132 and stabilize.py:148-230) so the parity tests
read like the reference's.

How the reference maps onto this file:

* ``Tape.backward(loss_grad, hook)`` + ``_deliver`` (tape.py:330-405) is
  replaced by torch autograd plus one ``register_post_accumulate_grad_hook``
  per parameter; the hook receives the complete gradient exactly once,
  calls the C-ABI (csrc/lomo_kernels.cu) on the current CUDA stream and
  then drops ``p.grad`` -- the ``Disposition.CONSUME`` equivalent, so at
  most one gradient tensor is alive at a time (optim.py:1-7, tape.py:399-401).
* the hook bodies -- ``apply_update`` (optim.py:52-54), the value-clip hook
  (stabilize.py:165-171), ``probe_hook`` (:190-200), ``update_hook``
  (:215-224) -- are the device kernels K1/K2; the norm decision and the
  loss-scale state machine (:201-213, :94-127) are K3 on device.  The host
  reads the 128-byte step status once per step (the one sync), never per
  parameter.
"""
from __future__ import annotations

import math
from typing import Callable, Iterable

import torch

from . import _lib
from .dispatch import HookDispatcher
from .errors import (ConfigError, NonFiniteLossError, ScaleUnderflowError, ShapeError,
                     TapeStateError)
from .stabilize import ClipKind, ClipMode, LossScaler, Stabilizer, StepOutcome

_DTYPE_CODE = {
    torch.float32: _lib.F32,
    torch.float16: _lib.F16,
    torch.bfloat16: _lib.BF16,
    torch.float64: _lib.F64,
}
_MATH_CODE = {"f32": _lib.MATH_F32, "f64": _lib.MATH_F64}

_PROBE = 1
_UPDATE = 2


def dtype_code(dtype: torch.dtype) -> int:
    try:
        return _DTYPE_CODE[dtype]
    except KeyError:
        raise ConfigError(f"unsupported parameter dtype {dtype}") from None


def _stabilizer_from_args(clip_grad_norm, clip_grad_value, loss_scale) -> Stabilizer | None:
    if clip_grad_norm is not None and clip_grad_value is not None:
        raise ConfigError("clip_grad_norm and clip_grad_value are mutually exclusive")
    clip = ClipMode.none()
    if clip_grad_norm is not None and clip_grad_norm > 0:
        clip = ClipMode.by_global_norm(clip_grad_norm)
    elif clip_grad_value is not None and clip_grad_value > 0:
        clip = ClipMode.by_value(clip_grad_value)
    scaler = None
    if isinstance(loss_scale, LossScaler):
        scaler = loss_scale
    elif loss_scale is not None and loss_scale is not False:
        scaler = LossScaler(scale=float(2.0 ** 10 if loss_scale is True else loss_scale))
    if clip.kind is ClipKind.NONE and scaler is None:
        return None
    return Stabilizer(clip, scaler)


class LOMO:
    """Fused update: each gradient is consumed on the GPU the moment it exists.

    Args:
        model: a ``torch.nn.Module`` (or an iterable of parameters) on one CUDA
            device; parameters of dtype fp32/fp16/bf16/fp64, contiguous.
        lr: default learning rate (``fused_backward`` takes it per call).
        clip_grad_norm: global-norm clip (two passes, stabilize.py:180-230).
        loss_scale: ``None`` (off), an initial power-of-two scale, or a
            :class:`LossScaler` (dynamic scaling, two passes).
        clip_grad_value: value clip threshold (single pass, stabilize.py:163-176).
        weight_decay: decoupled decay ``p *= 1 - lr*wd`` (0 = the reference).
        stabilizer: alternatively, the reference's :class:`Stabilizer`.
        math: ``"f32"`` (fp32 arithmetic, the hot path) or ``"f64"`` (the
            reference's float64 arithmetic, rounded directly to storage).
    """

    def __init__(self, model, lr: float = 1e-3, clip_grad_norm: float | None = None,
                 loss_scale=None, *, clip_grad_value: float | None = None,
                 weight_decay: float = 0.0, stabilizer: Stabilizer | None = None,
                 math: str = "f32"):
        if stabilizer is not None and (clip_grad_norm or clip_grad_value or loss_scale):
            raise ConfigError("pass either a Stabilizer or the clip/loss_scale arguments")
        self.stabilizer = stabilizer if stabilizer is not None else _stabilizer_from_args(
            clip_grad_norm, clip_grad_value, loss_scale)
        if (self.stabilizer is not None
                and self.stabilizer.clip.kind is ClipKind.BY_GROUP_NORM):
            raise ConfigError("grouped clipping is provided by GroupedLOMO")
        if math not in _MATH_CODE:
            raise ConfigError(f"math must be 'f32' or 'f64', got {math!r}")
        self.lr = float(lr)
        self.weight_decay = float(weight_decay)
        self.math = math
        self._math = _MATH_CODE[math]

        params = list(model.parameters()) if hasattr(model, "parameters") else list(model)
        seen, uniq = set(), []
        for p in params:
            if p.requires_grad and id(p) not in seen:
                seen.add(id(p))
                uniq.append(p)
        if not uniq:
            raise ConfigError("model has no trainable parameters")
        dev = uniq[0].device
        if dev.type != "cuda":
            raise ConfigError(f"LOMO runs on CUDA devices only (got {dev}); there is no CPU path")
        for p in uniq:
            if p.device != dev:
                raise ConfigError("all parameters must live on one CUDA device")
            if not p.is_contiguous():
                raise ConfigError("parameters must be contiguous")
            dtype_code(p.dtype)
        self.params = uniq
        self.device = dev
        self._lib = _lib.load()

        # Slot i <-> the i-th parameter in reference delivery order: non-increasing
        # layer, reverse build order within a layer == reverse registration
        # order (tape.py:350-360).  K3a sums the slots in this order (stabilize.py:199).
        self._slot = {id(p): i for i, p in enumerate(reversed(uniq))}
        self.nslots = len(uniq)
        self._state = torch.zeros(_lib.state_bytes(self.nslots), dtype=torch.uint8, device=dev)
        self._state_ptr = self._state.data_ptr()
        off = _lib.SCALE_F32_OFFSET
        self._scale_view = self._state[off:off + 4].view(torch.float32).view(())
        self._status = _lib.LomoStatus()

        st = self.stabilizer
        scaler = st.scaler if st is not None else None
        self._has_scaler = scaler is not None
        self._norm_clip = st is not None and st.clip.kind is ClipKind.BY_GLOBAL_NORM
        self._clip_value = (st.clip.threshold if st is not None
                            and st.clip.kind is ClipKind.BY_VALUE else 0.0)
        self.passes = st.backward_passes_per_step if st is not None else 1
        with torch.cuda.device(dev):
            s = torch.cuda.current_stream(dev).cuda_stream
            _lib.check(self._lib.lomo_state_init(
                self._state_ptr, self.nslots,
                float(scaler.scale) if scaler else 0.0,
                int(scaler.growth_interval) if scaler else 1,
                float(scaler.min_scale) if scaler else 1.0,
                float(scaler.max_scale) if scaler else 1.0,
                float(st.clip.max_norm) if self._norm_clip else 0.0, s), "lomo_state_init")

        self._dispatch = HookDispatcher(self._lib, self._state_ptr, self._math)
        self._mode = 0
        self._pending = None          # None | "apply" | "skip" after grad_norm
        self.last_outcome: StepOutcome | None = None
        self.clip_coef: float | None = None
        self.last_norm: float | None = None
        self.hook_calls = 0
        self._handles = [p.register_post_accumulate_grad_hook(self._hook) for p in uniq]

    # ------------------------------------------------------------------ hooks
    def _hook(self, p: torch.Tensor) -> None:
        """The hook body (tape.py:387-405 boundary; optim.py:126-128)."""
        mode = self._mode
        g = p.grad
        if mode == 0 or g is None:
            return  # a plain backward outside the LOMO protocol: leave .grad alone
        if g.shape != p.shape:
            raise ShapeError("backward", f"gradient {tuple(g.shape)} vs parameter {tuple(p.shape)}")
        if g.dtype != p.dtype:
            raise ShapeError("backward", f"gradient dtype {g.dtype} vs parameter {p.dtype}")
        if not g.is_contiguous():
            g = g.contiguous()
        stream = torch.cuda.current_stream(p.device).cuda_stream
        dt = _DTYPE_CODE[p.dtype]
        if mode == _PROBE:
            self._dispatch.probe(g, dt, self._slot[id(p)], stream)
        else:
            self._dispatch.update(p, g, dt, stream)
        self.hook_calls += 1
        p.grad = None  # CONSUME: the caching allocator reuses the block stream-ordered

    # ------------------------------------------------------------- internals
    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _begin(self, loss: torch.Tensor | None) -> None:
        if loss is not None:
            lt = loss.detach()
            if lt.numel() != 1:
                raise ShapeError("backward", f"loss must be a scalar, got {tuple(lt.shape)}")
            if not lt.is_contiguous():
                lt = lt.contiguous()
            self._loss_keep = lt  # keep alive until the kernel has read it
            _lib.check(self._lib.lomo_begin_step(self._state_ptr, lt.data_ptr(),
                                                 dtype_code(lt.dtype), self._stream()),
                       "lomo_begin_step")
        else:
            _lib.check(self._lib.lomo_begin_step(self._state_ptr, None, 0, self._stream()),
                       "lomo_begin_step")

    def _backward(self, loss: torch.Tensor, mode: int, flags: int, retain_graph: bool,
                  lr: float = 0.0) -> None:
        for p in self.params:
            if p.grad is not None:
                raise TapeStateError("a parameter already holds a gradient; LOMO consumes "
                                     "gradients inside backward (call zero_grad(set_to_none=True))")
        target = loss.float() * self._scale_view if self._has_scaler else loss
        self._dispatch.configure(lr, self._clip_value, self.weight_decay, flags)
        self._mode = mode
        try:
            target.backward(retain_graph=retain_graph)
        finally:
            self._mode = 0
            # launch the parked tiny tensors (same stream as the hooks)
            self._dispatch.flush(self._stream())

    def read_status(self) -> _lib.LomoStatus:
        """Copy the device step status to the host (synchronises the stream)."""
        _lib.check(self._lib.lomo_read_status(self._state_ptr, self._status, self._stream()),
                   "lomo_read_status")
        torch.cuda.current_stream(self.device).synchronize()
        return self._status

    # -------------------------------------------------------------- public API
    def grad_norm(self, loss: torch.Tensor, retain_graph: bool = True) -> float | None:
        """Pass 1 of the two-pass protocol (stabilize.py:180-213).

        Backward of ``loss*scale`` with the probe hook (K2): overflow flag and
        the unscaled sum of squares per parameter; then K3a decides N, the clip
        coefficient and whether the step is skipped (halving the scale on
        device).  Returns the global gradient norm, or ``None`` when the step
        was skipped for overflow.  Raises :class:`ScaleUnderflowError` when the
        scale would fall below its minimum.
        """
        if self.passes != 2:
            raise TapeStateError("grad_norm is only needed with clip_grad_norm or loss_scale")
        self._begin(loss)
        flags = (_lib.USE_SCALE if self._has_scaler else 0) | \
            (_lib.ACCUM_F64 if self._math == _lib.MATH_F64 else 0)
        self._backward(loss, _PROBE, flags, retain_graph)
        _lib.check(self._lib.lomo_finalize_norm(self._state_ptr, self._stream()),
                   "lomo_finalize_norm")
        st = self.read_status()  # the one host sync of the step
        if st.underflow:
            raise ScaleUnderflowError(
                f"loss scale would fall below {st.min_scale}; training diverged")
        self.last_norm = float(st.total_norm)
        self.clip_coef = float(st.clip_coef)
        if st.skip:
            self._pending = "skip"
            self.last_outcome = StepOutcome.SKIPPED_OVERFLOW
            return None
        self._pending = "apply"
        return self.last_norm

    def fused_backward(self, loss: torch.Tensor, lr: float | None = None) -> None:
        """The fused pass: backward whose per-parameter hook runs K1 in place.

        Two-pass mode (norm clip and/or loss scale) requires ``grad_norm``
        first; after a skipped pass 1 this is a no-op (the step is dropped,
        stabilize.py:204-205).  Single-pass mode raises
        :class:`NonFiniteLossError` for a non-finite loss with every parameter
        untouched (optim.py:63-65; the check is a device flag K1 honours).
        """
        lr = self.lr if lr is None else float(lr)
        if self.passes == 2:
            if self._pending is None:
                raise TapeStateError("clip_grad_norm/loss_scale need grad_norm(loss) "
                                     "before fused_backward(loss, lr)")
            pending, self._pending = self._pending, None
            if pending == "skip":
                return
            flags = _lib.USE_SKIP | (_lib.USE_SCALE if self._has_scaler else 0) \
                | (_lib.USE_COEF if self._norm_clip else 0)
            self._backward(loss, _UPDATE, flags, retain_graph=False, lr=lr)
            _lib.check(self._lib.lomo_scaler_on_clean(self._state_ptr, self._stream()),
                       "lomo_scaler_on_clean")
            self.last_outcome = StepOutcome.APPLIED
            return
        self._begin(loss)
        self._backward(loss, _UPDATE, _lib.USE_SKIP, retain_graph=False, lr=lr)
        _lib.check(self._lib.lomo_scaler_on_clean(self._state_ptr, self._stream()),
                   "lomo_scaler_on_clean")
        st = self.read_status()
        if st.skip:
            self.last_outcome = None
            raise NonFiniteLossError(f"loss is non-finite ({float(loss.detach())}); step aborted")
        self.last_outcome = None if self.stabilizer is None else StepOutcome.APPLIED

    def step(self, closure: Callable[[], torch.Tensor], lr: float | None = None,
             recompute_forward: bool = False) -> float:
        """The reference step protocol (optim.py:118-132, stabilize.py:148-230).

        ``closure()`` runs the forward and returns the scalar loss.  Two-pass
        mode reuses the pass-1 graph for pass 2 (identical values: pass 1
        does not touch parameters); ``recompute_forward=True`` re-runs the
        forward instead, as stabilize.py:226 does.  Returns the loss as a float.
        """
        loss = closure()
        if self.passes == 2:
            self.grad_norm(loss, retain_graph=not recompute_forward)
            if self._pending == "skip":
                self._pending = None
                return float(loss.detach())
            if recompute_forward:
                loss = closure()
            self.fused_backward(loss, lr)
            return float(loss.detach())
        self.fused_backward(loss, lr)
        return float(loss.detach())

    # ------------------------------------------------------------ accessors
    @property
    def loss_scale(self) -> float:
        """Current loss scale (reads the device state: synchronises)."""
        return float(self.read_status().scale) if self._has_scaler else 1.0

    def state_nbytes(self) -> int:
        """Optimizer state per parameter: zero (optim.py:115-116)."""
        return 0

    def remove_hooks(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []


def lomo_step(model, closure, lr: float, stabilizer: Stabilizer | None = None,
              math: str = "f32") -> float:
    """One fused step as a free function (optim.py:189-192)."""
    opt = LOMO(model, lr, stabilizer=stabilizer, math=math)
    try:
        return opt.step(closure, lr)
    finally:
        opt.remove_hooks()
