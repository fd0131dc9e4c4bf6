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

import ctypes
import os
from typing import Callable

import torch

from . import _lib
from . import replay as _replay
from .engine import CudaEngine, dtype_code
from .errors import (ConfigError, NonFiniteLossError, ScaleUnderflowError, ShapeError,
                     TapeStateError)
from .replay import ReplayStash
from .stabilize import (ClipKind, ClipMode, LossScaler, Stabilizer, StepOutcome,
                        is_power_of_two)

_PROBE = 1
_UPDATE = 2
_E_ARG = -1  # LOMO_E_ARG (include/lomo_b200.h)


def stabilizer_from_args(clip_grad_norm, clip_grad_value, loss_scale) -> Stabilizer | None:
    """Map the north-star keyword arguments onto the reference's Stabilizer."""
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


def trainable_params(model) -> list[torch.Tensor]:
    params = list(model.parameters()) if hasattr(model, "parameters") else list(model)
    seen, uniq = set(), []
    for p in params:
        if p.requires_grad and id(p) not in seen:
            seen.add(id(p))
            uniq.append(p)
    if not uniq:
        raise ConfigError("model has no trainable parameters")
    return uniq


def _as_closure(opt, closure):
    """step(closure) or the reference's step(batch) with batch = (inputs, targets)."""
    if callable(closure):
        return closure
    model = getattr(opt, "_model", None)
    if model is None or not callable(getattr(model, "loss", None)):
        raise TypeError("step(batch, lr) needs a model with .loss(inputs, targets) (the "
                        "reference's _forward_loss, optim.py:57-60); otherwise pass a closure "
                        "returning the loss")
    inputs, targets = closure
    return lambda: model.loss(inputs, targets)


class _Protocol:
    """The two-pass / single-pass step protocol shared by LOMO and ShardedLOMO
    (stabilize.py:148-230), over a CudaEngine and a backward driver.

    Subclasses provide ``self.engine``, ``_run_backward(target, mode,
    retain_graph)`` and ``_decide()`` (K3a, with a cross-rank exchange in the
    sharded case)."""

    _always_scale = False  # sharded mode: inv_scale also carries 1/world

    def _init_protocol(self, stabilizer, lr, weight_decay):
        st = stabilizer
        if st is not None and st.clip.kind is ClipKind.BY_GROUP_NORM:
            raise ConfigError("grouped clipping is the single-pass GroupedLOMO")
        self.stabilizer = st
        self.lr = float(lr)
        self.weight_decay = float(weight_decay)
        self.scaler = st.scaler if st is not None else None
        self.has_scaler = self.scaler is not None
        self.norm_clip = st is not None and st.clip.kind is ClipKind.BY_GLOBAL_NORM
        self.max_norm = st.clip.max_norm if self.norm_clip else None
        self.clip_value = (st.clip.threshold if st is not None
                           and st.clip.kind is ClipKind.BY_VALUE else 0.0)
        self.passes = st.backward_passes_per_step if st is not None else 1
        self._pending = None          # None | "apply" | "skip" after grad_norm
        # two-pass mode: read the loss's finiteness on the host before pass 1,
        # so a non-finite loss runs no backward (the reference's order,
        # stabilize.py:185-189); graphs.py turns it off inside its captures
        self.check_loss_first = True
        self.last_outcome: StepOutcome | None = None
        self.clip_coef: float | None = None
        self.last_norm: float | None = None

    def _check_loss(self, loss):
        """The loss whose finiteness decides the step (per rank by default)."""
        return loss

    def _scaled(self, loss):
        return loss.float() * self.engine.scale_view if self.has_scaler else loss

    def _flags(self, mode) -> int:
        scale = _lib.USE_SCALE if (self.has_scaler or self._always_scale) else 0
        if mode == _PROBE:
            return scale | (_lib.ACCUM_F64 if self.engine.math == _lib.MATH_F64 else 0)
        return _lib.USE_SKIP | scale | (_lib.USE_COEF if self.norm_clip else 0)

    def grad_norm(self, loss: torch.Tensor, retain_graph: bool = True) -> float | None:
        """Pass 1 of the two-pass protocol (stabilize.py:180-213).

        Backward of ``loss*scale`` with the probe hook (K2): overflow flag and
        the unscaled sum of squares; then K3a decides N, the clip coefficient
        and whether the step is skipped (halving the scale on device).
        Returns the global gradient norm, or ``None`` when the step was
        skipped for overflow.  Raises :class:`ScaleUnderflowError` when the
        scale would fall below its minimum.
        """
        if self.passes != 2:
            raise TapeStateError("grad_norm is only needed with clip_grad_norm or loss_scale")
        checked = self._check_loss(loss)
        self.engine.begin(checked)
        self.engine.configure(flags=self._flags(_PROBE))
        # stabilize.py:185-189: a non-finite loss skips the step BEFORE any
        # backward.  The device flag alone (begin_step) gives the same
        # decision, but the backward would still run; the host check costs
        # one sync after the forward (the graphed step keeps the device flag)
        if not (self.check_loss_first and not bool(torch.isfinite(checked.detach()).all())):
            self._run_backward(self._scaled(loss), _PROBE, retain_graph)
        self._decide()  # K3a: skip (overflow set by begin_step) + LossScaler.on_overflow
        st = self.engine.read_status()  # the one host sync of the step
        self._mirror_scaler(st)
        if st.underflow:
            raise ScaleUnderflowError(
                f"loss scale would fall below {st.min_scale}; training diverged")
        self.last_norm = float(st.total_norm)
        self.clip_coef = float(st.clip_coef)
        self._pass1 = (float(st.clip_coef) if self.norm_clip else 1.0,
                       float(st.inv_scale) if (self.has_scaler or self._always_scale) else 1.0)
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
        flags = self._flags(_UPDATE)
        if self.passes == 2:
            if self._pending is None:
                raise TapeStateError("clip_grad_norm/loss_scale need grad_norm(loss) "
                                     "before fused_backward(loss, lr)")
            pending, self._pending = self._pending, None
            if pending == "skip":
                self._drop_stash()
                return
            self.engine.configure(lr, self.clip_value, self.weight_decay, flags)
            if getattr(self, "_stash", None) is not None:
                self._replay_pass(lr)
            else:
                self._run_backward(self._scaled(loss), _UPDATE, False)
            self.engine.on_clean()
            self._scaler_clean()
            self._after_update()
            self.last_outcome = StepOutcome.APPLIED
            return
        if getattr(self, "_fused_update", False) and not bool(torch.isfinite(loss.detach()).all()):
            # K5 applies p <- alpha*acc + beta*p: a skip (alpha = 0) would still
            # turn a non-finite accumulator into NaN, so the non-finite-loss
            # check runs on the host here, as the reference's does (optim.py:63-65)
            self.last_outcome = None
            raise NonFiniteLossError(f"loss is non-finite ({float(loss.detach())}); step aborted")
        self.engine.begin(self._check_loss(loss))
        self.engine.configure(lr, self.clip_value, self.weight_decay, flags)
        self._run_backward(loss, _UPDATE, False)
        self.engine.on_clean()
        st = self.engine.read_status()
        if st.skip:
            self.last_outcome = None
            raise NonFiniteLossError(f"loss is non-finite ({float(loss.detach())}); step aborted")
        self._after_update()
        self.last_outcome = None if self.stabilizer is None else StepOutcome.APPLIED

    def _after_update(self) -> None:
        pass

    def state_dict(self) -> dict:
        """The optimizer's whole state (LOMO keeps no per-parameter state,
        optim.py:115-116): the loss scaler's live fields and the step
        counters, read from the device (one sync)."""
        st = self.engine.read_status()
        self._mirror_scaler(st)
        return {"scale": float(st.scale) if self.has_scaler else None,
                "clean_steps": int(st.clean_steps), "steps_applied": int(st.steps_applied),
                "steps_skipped": int(st.steps_skipped)}

    def load_state_dict(self, sd: dict) -> None:
        """Restore :meth:`state_dict` (resume from a checkpoint): the device
        state machine and the user's LossScaler object continue from it."""
        scale = sd.get("scale")
        if self.has_scaler:
            if scale is None:
                raise ConfigError("state_dict has no loss scale for a scaled optimizer")
            if not is_power_of_two(float(scale)):
                raise ConfigError(f"scale must be a positive power of two, got {scale}")
        _lib.check(self.engine.lib.lomo_set_scaler_state(
            self.engine.ptr, float(scale) if scale else 1.0, int(sd.get("clean_steps", 0)),
            int(sd.get("steps_applied", 0)), int(sd.get("steps_skipped", 0)),
            self.engine.stream()), "lomo_set_scaler_state")
        if self.has_scaler:
            self.scaler.scale = float(scale)
            self.scaler.clean_steps = int(sd.get("clean_steps", 0))

    def _mirror_scaler(self, st) -> None:
        """The user's LossScaler object reads as the reference's: the device
        state machine's scale / clean_steps at this step's status read."""
        if self.scaler is not None:
            self.scaler._mirror(st)

    def _scaler_clean(self) -> None:
        """After an applied step K3b ran LossScaler.on_clean on the device;
        the host mirror applies the same arithmetic (no extra sync)."""
        if self.scaler is not None:
            self.scaler.on_clean()

    def _drop_stash(self) -> None:
        st = getattr(self, "_stash", None)
        if st is not None:
            st.clear()

    def step(self, closure: Callable[[], torch.Tensor], lr: float | None = None,
             recompute_forward: bool = False) -> float:
        """The reference step protocol (optim.py:118-132, stabilize.py:148-230).

        ``closure()`` runs the forward and returns the scalar loss; the
        reference's own form ``step(batch, lr)`` with ``batch = (inputs,
        targets)`` is accepted too (``model.loss(inputs, targets)``, its
        ``_forward_loss``, optim.py:57-60).  Two-pass mode reuses the pass-1
        graph for pass 2 (identical values: pass 1 does not touch
        parameters); ``recompute_forward=True`` re-runs the forward instead,
        as stabilize.py:226 does.  Returns the loss as a float.
        """
        closure = _as_closure(self, closure)
        loss = closure()
        if self.passes == 2:
            replay = getattr(self, "_stash", None) is not None
            self.grad_norm(loss, retain_graph=not (recompute_forward or replay))
            if self._pending == "skip":
                self._pending = None
                return float(loss.detach())
            if recompute_forward and not replay:
                loss = closure()
            self.fused_backward(loss, lr)
            return float(loss.detach())
        self.fused_backward(loss, lr)
        return float(loss.detach())

    @property
    def loss_scale(self) -> float:
        """Current loss scale (reads the device state: synchronises)."""
        return float(self.engine.read_status().scale) if self.has_scaler else 1.0

    def read_status(self) -> _lib.LomoStatus:
        return self.engine.read_status()

    def state_nbytes(self) -> int:
        """Optimizer state per parameter: zero (optim.py:115-116)."""
        return 0


class LOMO(_Protocol):
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
        stabilizer: alternatively, the reference's :class:`Stabilizer`; the
            reference's positional form ``LOMO(model, stabilizer)`` works too
            (optim.py:108-112: the learning rate is then ``step``'s).
        ledger: accepted for the reference's signature and ignored (the
            memory ledger is outside this path; ``torch.cuda`` memory stats
            report the same quantities).
        math: ``"f32"`` (fp32 arithmetic, the hot path) or ``"f64"`` (the
            reference's float64 arithmetic, rounded directly to storage).
        overlap: launch the hook kernels on a side stream so each update
            overlaps the rest of the backward (a few gradients may be alive at
            once instead of one; off by default to keep the reference's
            one-gradient invariant).
        replay: two-pass mode only -- pass 2 recomputes each weight gradient
            from the (input, output-gradient) pair stashed in pass 1 instead of
            running a second backward (see replay.py); the model's linears
            must go through ``paper_2306_09782_b200.replay.linear``.
        fuse_gemm: run each linear's update as the epilogue of its
            weight-gradient GEMM on the tensor cores (K5,
            csrc/lomo_gemm_update.cu): ``p <- p - lr*coef/scale * (dy^T x)`` from
            the fp32 accumulator, the gradient never materialised -- over the
            pass-1 stash with ``replay``, else inside each linear's backward
            (the single fused pass, or the strict protocol's second backward).
            16-bit parameters, fp32 math, no value clip; other parameters keep
            K1, and an embedding routed through ``replay.embedding`` keeps its
            gradient as the batch's rows (exact; not with weight decay).
        fuse_probe: two-pass mode (default: on when ``fuse_gemm`` is): run
            each linear's pass-1 probe as the epilogue of its weight-gradient
            GEMM (K6, csrc/lomo_gemm_probe.cu): the overflow flag and the sum of
            squares come out of the tensor-core accumulator, so no K2 launch
            re-reads the gradient and autograd never holds it.
        gemm_streams / probe_stream: run pass 2's K5 GEMMs over that many
            streams / pass 1's K6 GEMMs on a side stream (off by default).
    """

    def __init__(self, model, lr: float = 1e-3, clip_grad_norm: float | None = None,
                 loss_scale=None, *, clip_grad_value: float | None = None,
                 weight_decay: float = 0.0, stabilizer: Stabilizer | None = None,
                 math: str = "f32", overlap: bool = False, replay: bool = False,
                 fuse_gemm: bool = False, fuse_probe: bool | None = None,
                 gemm_streams: int = 1, probe_stream: bool = False, ledger=None):
        if isinstance(lr, Stabilizer):  # the reference's LOMO(model, stabilizer)
            if stabilizer is not None:
                raise ConfigError("stabilizer given twice")
            stabilizer, lr = lr, 1e-3
        if stabilizer is not None and (clip_grad_norm or clip_grad_value or loss_scale):
            raise ConfigError("pass either a Stabilizer or the clip/loss_scale arguments")
        st = stabilizer if stabilizer is not None else stabilizer_from_args(
            clip_grad_norm, clip_grad_value, loss_scale)
        self._init_protocol(st, lr, weight_decay)
        self._model = model
        uniq = trainable_params(model)
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
        self.math = math
        self.engine = CudaEngine(dev, len(uniq), self.scaler, self.max_norm, math,
                                 overlap=overlap)
        # Slot i <-> the i-th parameter in reference delivery order: non-increasing
        # layer, reverse build order within a layer == reverse registration
        # order (tape.py:350-360).  K3a sums the slots in this order (stabilize.py:199).
        self._slot = {id(p): i for i, p in enumerate(reversed(uniq))}
        self._mode = 0
        self.hook_calls = 0
        if replay and self.passes != 2:
            raise ConfigError("replay applies to the two-pass protocol (clip_grad_norm / loss_scale)")
        self._stash = ReplayStash() if replay else None
        self._replay_checked = False
        self._replay_mismatch: list = []
        # the fused GEMMs apply/probe the fp32 accumulator: not the f64
        # exactness mode, and value clipping is not linear in dW
        self.fuse_gemm = bool(fuse_gemm) and self.clip_value == 0.0 and math == "f32"
        if fuse_probe and self.passes != 2:
            raise ConfigError("fuse_probe fuses pass 1's probe into the weight-gradient GEMM: "
                              "it needs the two-pass protocol (clip_grad_norm / loss_scale)")
        self.fuse_probe = bool(fuse_gemm if fuse_probe is None else fuse_probe) \
            and self.passes == 2 and math == "f32"
        # the linears' backward context: the replay stash, or (no replay) just
        # the fused-GEMM callbacks -- K6 in pass 1, and K5 inside the update
        # backward (the single fused pass, or the strict second backward)
        self._fused_update = self.fuse_gemm and not replay
        # with the fused paths, an embedding routed through replay.embedding
        # keeps its gradient as the batch's rows (exact: untouched rows do not
        # move), never as a dense [V, h] tensor; not with weight decay
        self.sparse_embedding = self.fuse_gemm and self.weight_decay == 0.0
        self._lin = self._stash if replay else (
            ReplayStash(keep=False) if (self.fuse_probe or self._fused_update) else None)
        self._by_id = {id(p): p for p in uniq}
        if self._fused_update and hasattr(model, "named_parameters"):
            # tied weights (one Parameter under several names): K5 would apply
            # the linear's share in place before autograd delivered the rest,
            # and a single pass cannot be rolled back -- refuse up front.
            # (A weight reused by two linears without being registered twice
            # is only seen during backward: ConfigError after that step.)
            seen: set[int] = set()
            for name, p in model.named_parameters(remove_duplicate=False):
                if p.requires_grad and id(p) in seen:
                    raise ConfigError(f"fuse_gemm without replay: {name} is a tied weight; "
                                      "use replay=True or fuse_gemm=False")
                seen.add(id(p))
        self._coefs = None
        self._lr_from_state = False  # graph capture: the state's lr, set per replay
        self._pws = {}         # K6 workspace per weight (its partial sums stay until
                               # the end of pass 1: one deferred reduction launch)
        self._pending_probe = []  # (workspace ptr, out, in, slot) awaiting that launch
        self._gscratch = None  # K6's clipped by-product store, shared by every linear
        self._ws = {}          # K5 workspace per stream
        # Optional stream concurrency of the tensor-core GEMMs: pass 2's K5
        # launches are independent of each other and may rotate over
        # `gemm_streams` streams; pass 1's K6 may run on a side stream beside
        # the rest of the backward (it only reads the stashed x/dy).  Joined
        # before K3a / at the end of pass 2.  Off by default: on LLaMA-7B the
        # overlap cost more than the filled wave tails (profiles/r01_gemm_shapes.md).
        # LOMO_GEMM_STREAMS / LOMO_PROBE_STREAM override.
        self.gemm_streams = max(1, int(os.environ.get("LOMO_GEMM_STREAMS", gemm_streams)))
        self.probe_stream = os.environ.get("LOMO_PROBE_STREAM", "1" if probe_stream else "0") == "1"
        self._streams = None
        self._pstream = None
        self._largest = max(p.numel() * p.element_size() for p in uniq)
        self._handles = [p.register_post_accumulate_grad_hook(self._hook) for p in uniq]

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
        if mode == _PROBE:
            self.engine.probe(g, self._slot[id(p)])
            lin, st = self._lin, self._stash
            if lin is not None and (id(p) in lin.probed or id(p) in lin.embedded):
                # K6 already probed this weight's linear: a hook means another
                # op contributed gradient too (tied weight), which the fused
                # paths cannot fold into the norm or the update
                self._replay_mismatch.append(tuple(p.shape))
            elif st is not None:
                if id(p) not in st.linear:
                    st.grads[id(p)] = g  # not a replayable linear: keep its gradient
                elif not self._replay_checked:
                    # first step: the replayed dW must BE the whole gradient
                    # (a weight tied to another op would also collect that op's
                    # contribution, which replay would silently drop)
                    x, dy = st.linear[id(p)]
                    r = _replay.weight_grad(x, dy)
                    # NaN-aware: an overflowing first step must not read as a mismatch
                    if not torch.equal(r, g) and not bool(((r == g) | (r.isnan() & g.isnan()))
                                                          .all()):
                        self._replay_mismatch.append(tuple(p.shape))
        else:
            lin = self._lin
            if lin is not None and (id(p) in lin.updated or id(p) in lin.embedded):
                # K5 already applied this weight's linear gradient in place; a
                # hook means another op fed it too (tied weight)
                self._replay_mismatch.append(tuple(p.shape))
            self.engine.update(p, g)
        self.hook_calls += 1
        p.grad = None  # CONSUME: the caching allocator reuses the block stream-ordered

    def _run_backward(self, target: torch.Tensor, mode: int, retain_graph: bool) -> None:
        for p in self.params:
            if p.grad is not None:
                raise TapeStateError("a parameter already holds a gradient; LOMO consumes "
                                     "gradients inside backward (call zero_grad(set_to_none=True))")
        self._mode = mode
        lin = self._lin
        if lin is not None and not (
                (mode == _PROBE and (lin.keep or self.fuse_probe)) or
                (mode == _UPDATE and self._fused_update)):
            lin = None
        stash = lin if (lin is not None and lin.keep) else None
        if lin is not None:
            lin.clear()
            lin.probe = self._gemm_probe if (mode == _PROBE and self.fuse_probe) else None
            lin.update = self._gemm_update_bw if mode == _UPDATE else None
            lin.embed = (self._embed_rows if self.sparse_embedding and
                         (mode == _UPDATE or self.fuse_probe) else None)
            if mode == _UPDATE:
                self._load_coefs()
            _replay._ACTIVE = lin
            if stash is not None:
                retain_graph = False  # pass 2 replays from the stash, not from the graph
        try:
            target.backward(retain_graph=retain_graph)
        finally:
            self._mode = 0
            if lin is not None:
                _replay._ACTIVE = None
            self._finish_probes()  # deferred K6 partial sums -> their slots
            self.engine.flush()  # the parked tiny tensors, same stream as the hooks
        if lin is not None and stash is None:
            bad = None
            if lin.shared:
                bad = f"fuse_gemm: {len(lin.shared)} weight(s) feed more than one linear"
            elif self._replay_mismatch:
                bad = (f"fuse_gemm: weights {self._replay_mismatch[:3]} receive gradient from "
                       "ops other than their linear (tied weights?)")
            if bad is not None:
                self._replay_mismatch = []
                raise ConfigError(bad)
        if stash is not None:
            kept = sum(g.numel() * g.element_size() for g in stash.grads.values())
            bad = None
            if kept > 2 * self._largest:
                bad = (f"replay would keep {kept / 2**20:.0f} MiB of gradients: route the model's "
                       "linear layers through paper_2306_09782_b200.replay.linear")
            elif stash.shared:
                bad = f"replay: {len(stash.shared)} weight(s) feed more than one linear"
            elif self._replay_mismatch:
                bad = (f"replay: weights {self._replay_mismatch[:3]} receive gradient from ops "
                       "other than their linear (tied weights?)")
            if bad is not None:
                stash.clear()
                raise ConfigError(bad)
            self._replay_checked = True

    def _gemm_update(self, p, x, dy, lr: float, coefs: torch.Tensor | None = None) -> bool:
        """K5: p <- alpha * dy^T x + beta * p on the tensor cores; False when the
        shape/dtype is not supported (the caller falls back to GEMM + K1).
        ``coefs``: a device [alpha, beta] pair (graph capture) instead of host
        scalars from the pass-1 status."""
        if p.dtype not in (torch.bfloat16, torch.float16) or p.dim() != 2:
            return False
        out_f, in_f = p.shape
        if out_f % 8 or in_f % 8:
            return False
        dy2 = dy.reshape(-1, out_f)
        x2 = x.reshape(-1, in_f)
        if not (dy2.is_contiguous() and x2.is_contiguous()) or dy2.dtype != p.dtype:
            return False
        lib, dt = self.engine.lib, dtype_code(p.dtype)
        need = lib.lomo_gemm_update_workspace(out_f, in_f, dy2.shape[0], dt)
        ws = None
        if need:
            key = self.engine.stream()
            buf = self._ws.get(key)
            if buf is None or buf.numel() < need:
                buf = self._ws[key] = torch.empty(need, dtype=torch.uint8, device=p.device)
            ws = buf.data_ptr()
        if coefs is not None:
            rc = lib.lomo_gemm_update_dev(p.data_ptr(), dy2.data_ptr(), x2.data_ptr(), out_f,
                                          in_f, dy2.shape[0], dt, coefs.data_ptr(), ws, need,
                                          self.engine.stream())
        else:
            coef, inv_scale = self._pass1
            alpha = -lr * coef * inv_scale
            beta = 1.0 - lr * self.weight_decay
            rc = lib.lomo_gemm_update(p.data_ptr(), dy2.data_ptr(), x2.data_ptr(), out_f, in_f,
                                      dy2.shape[0], dt, alpha, beta, ws, need,
                                      self.engine.stream())
        if rc == _E_ARG:
            return False
        _lib.check(rc, "lomo_gemm_update")
        return True

    def _gemm_probe(self, wid: int, w, x, dy) -> bool:
        """K6 (from the linear's backward in pass 1): probe dW = dy^T x on the
        tensor cores into w's norm slot.  False when the shape/dtype is not
        supported -- the caller then returns dW to autograd and K2 probes it."""
        if w.dtype not in (torch.bfloat16, torch.float16) or w.dim() != 2:
            return False
        out_f, in_f = w.shape
        if out_f % 8 or in_f % 8:
            return False
        dy2 = dy.reshape(-1, out_f)
        x2 = x.reshape(-1, in_f)
        if not (dy2.is_contiguous() and x2.is_contiguous()) or dy2.dtype != w.dtype \
                or x2.dtype != w.dtype:
            return False
        lib, dt = self.engine.lib, dtype_code(w.dtype)
        need = lib.lomo_gemm_probe_workspace(out_f, in_f, dy2.shape[0], dt)
        if need == 0:
            return False
        ws = self._pws.get(wid)
        if ws is None or ws.numel() < need:
            ws = self._pws[wid] = torch.empty(need, dtype=torch.uint8, device=w.device)
        if self._gscratch is None:  # K6's clipped by-product store: 16 bytes
            self._gscratch = torch.empty(256, dtype=torch.uint8, device=w.device)
        slot = self._slot.get(wid)
        if slot is None:  # not a managed leaf (e.g. w.to(dtype)): autograd's dW + hook
            return False
        stream = self.engine.stream()
        if self.probe_stream:
            # beside the rest of the backward; the partial sums go to this
            # weight's own workspace; joined in _finish_probes, before K3a.
            # dy / x may be freed by autograd as soon as the linear's backward
            # returns (strict protocol, checkpoint recompute): record_stream
            # keeps the allocator from handing their blocks to the main stream
            # before K6 has read them
            if self._pstream is None:
                self._pstream = torch.cuda.Stream(w.device)
            self._pstream.wait_stream(torch.cuda.current_stream(w.device))
            dy2.record_stream(self._pstream)
            x2.record_stream(self._pstream)
            stream = self._pstream.cuda_stream
        rc = lib.lomo_gemm_probe(dy2.data_ptr(), x2.data_ptr(), self._gscratch.data_ptr(), out_f,
                                 in_f, dy2.shape[0], dt, slot,
                                 self.engine.dispatch.flags | _lib.DEFER_ROWS, self.engine.ptr,
                                 ws.data_ptr(), need, stream)
        if rc == _E_ARG:
            return False
        _lib.check(rc, "lomo_gemm_probe")
        self._pending_probe.append((ws.data_ptr(), out_f, in_f, slot, dt))
        self.hook_calls += 1
        return True

    def _load_coefs(self) -> None:
        """K5-in-backward constants on device: alpha = -lr*coef/scale (0 on a
        skipped step), beta = 1 - lr*wd, from the step state (lomo_update_coefs)."""
        eng = self.engine
        if self._coefs is None:
            self._coefs = torch.zeros(2, dtype=torch.float32, device=self.device)
        d = eng.dispatch
        if not self._lr_from_state:
            _lib.check(eng.lib.lomo_set_lr(eng.ptr, d.lr, eng.stream()), "lomo_set_lr")
        _lib.check(eng.lib.lomo_update_coefs(eng.ptr, self.weight_decay, d.flags,
                                             self._coefs.data_ptr(), eng.stream()),
                   "lomo_update_coefs")

    def _gemm_update_bw(self, wid: int, w, x, dy) -> bool:
        """K5 from inside the update backward: the weight's update applied as
        the epilogue of its weight-gradient GEMM (alpha/beta from device)."""
        p = self._by_id.get(wid)
        if p is None:  # not a managed leaf (e.g. w.to(dtype)): autograd's dW + hook
            return False
        if not self._gemm_update(p, x, dy, 0.0, coefs=self._coefs):
            return False
        self.hook_calls += 1
        return True

    def _embed_rows(self, wid: int, ids, dy) -> bool:
        """An embedding's gradient as the batch's aggregated rows: probed by
        K2 in pass 1 (kept for the replayed pass 2), or updated in place by
        the rows form of K1 in an update pass."""
        p = self._by_id.get(wid)
        if p is None or p.dim() != 2 or p.dtype == torch.float64:
            return False
        h = p.shape[1]
        ids1 = ids.reshape(-1)
        dy2 = dy.reshape(-1, h)
        if not dy2.is_contiguous() or dy2.dtype != p.dtype or ids1.dtype != torch.int64:
            return False
        ntok = ids1.numel()
        sorted_ids, perm = torch.sort(ids1, stable=True)
        rows = torch.empty(ntok, h, dtype=p.dtype, device=p.device)
        row_ids = torch.empty(ntok, dtype=torch.int64, device=p.device)
        eng, dt = self.engine, dtype_code(p.dtype)
        _lib.check(eng.lib.lomo_rows_aggregate(sorted_ids.data_ptr(), perm.data_ptr(),
                                               dy2.data_ptr(), ntok, h, dt, rows.data_ptr(),
                                               row_ids.data_ptr(), eng.stream()),
                   "lomo_rows_aggregate")
        if self._mode == _PROBE:
            eng.probe(rows, self._slot[wid])
            if self._lin is not None and self._lin.keep:
                self._lin.rows[wid] = (rows, row_ids)
        else:
            self._update_rows(p, rows, row_ids)
        self.hook_calls += 1
        return True

    def _update_rows(self, p, rows, row_ids) -> None:
        eng, d = self.engine, self.engine.dispatch
        _lib.check(eng.lib.lomo_fused_update_rows(
            p.data_ptr(), rows.data_ptr(), row_ids.data_ptr(), rows.shape[0], rows.shape[1],
            dtype_code(p.dtype), eng.math, d.lr, d.clip, d.wd, d.flags, eng.ptr, eng.stream()),
            "lomo_fused_update_rows")

    def _finish_probes(self) -> None:
        """One launch (per 64 linears) folds every deferred K6 partial-sum matrix
        of this pass into its norm slot, in stream order before K3a."""
        pend, self._pending_probe = self._pending_probe, []
        if not pend:
            return
        if self._pstream is not None:
            torch.cuda.current_stream(self.device).wait_stream(self._pstream)
        for dt in {e[4] for e in pend}:
            sel = [e for e in pend if e[4] == dt]
            k = len(sel)
            _lib.check(self.engine.lib.lomo_gemm_probe_finish(
                (ctypes.c_void_p * k)(*[e[0] for e in sel]),
                (ctypes.c_int64 * k)(*[e[1] for e in sel]),
                (ctypes.c_int64 * k)(*[e[2] for e in sel]),
                (ctypes.c_int * k)(*[e[3] for e in sel]), k, dt, self.engine.ptr,
                self.engine.stream()), "lomo_gemm_probe_finish")

    def _gemm_stream_list(self) -> list:
        """[current stream] + the side streams K5 rotates over."""
        main = torch.cuda.current_stream(self.device)
        if self.gemm_streams <= 1:
            return [main]
        if self._streams is None or len(self._streams) != self.gemm_streams - 1:
            self._streams = [torch.cuda.Stream(self.device) for _ in range(self.gemm_streams - 1)]
        return [main] + self._streams

    def _replay_pass(self, lr: float, coefs: torch.Tensor | None = None) -> None:
        """Pass 2 from the stash, in delivery order: for a replayable linear
        either K5 (GEMM with the update as epilogue) or dW = dy^T x (the
        pass-1 GEMM) -> K1; other parameters K1 on their kept gradient.  Every
        gradient is dropped right after its launch.  ``coefs``: device
        [alpha, beta] for K5 (graph capture, graphs.py)."""
        st = self._stash
        streams = self._gemm_stream_list() if self.fuse_gemm else []
        main = torch.cuda.current_stream(self.device)
        for s in streams[1:]:
            s.wait_stream(main)
        j = 0
        for p in reversed(self.params):
            pid = id(p)
            if pid in st.linear:
                x, dy = st.linear.pop(pid)
                if self.fuse_gemm:
                    s = streams[j % len(streams)]
                    with torch.cuda.stream(s):
                        ok = self._gemm_update(p, x, dy, lr, coefs=coefs)
                    if ok:
                        j += 1
                        if s is not main:   # freed on main: keep them until s used them
                            x.record_stream(s)
                            dy.record_stream(s)
                        self.hook_calls += 1
                        continue
                g = _replay.weight_grad(x, dy)
                del x, dy
            elif pid in st.rows:
                rows, row_ids = st.rows.pop(pid)
                self._update_rows(p, rows, row_ids)
                self.hook_calls += 1
                continue
            elif pid in st.grads:
                g = st.grads.pop(pid)
            else:
                continue  # no gradient this step (unused parameter)
            self.engine.update(p, g)
            self.hook_calls += 1
            del g
        for s in streams[1:]:
            main.wait_stream(s)
        self.engine.flush()
        st.clear()

    def _decide(self) -> None:
        self.engine.finalize()

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
