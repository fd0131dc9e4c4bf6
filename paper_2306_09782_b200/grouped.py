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

With ``fuse_gemm=True`` every linear routed through ``replay.linear`` /
``replay.matmul_in_out`` is probed inside its weight-gradient GEMM (K6): the
GEMM's epilogue writes the retained gradient *and* its group slot's sum of
squares / overflow, so the group flush runs K2 only over the other
parameters (norm scales, embedding) before K3a and K1.
"""
from __future__ import annotations

import ctypes
import re
from typing import Callable

import torch

from . import _lib
from . import replay as _replay
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
                 layer_of: dict | None = None, math: str = "f32", weight_decay: float = 0.0,
                 fuse_gemm: bool = False):
        self.clip = ClipMode.by_group_norm(max_norm, window)  # validation (stabilize.py:65-74)
        params = trainable_params(model)
        dev = params[0].device
        for p in params:
            if p.device != dev:
                raise ConfigError("all parameters must live on one CUDA device")
            dtype_code(p.dtype)
        self.params = params
        self._model = model
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
        self.fuse_gemm = bool(fuse_gemm) and math == "f32"
        self._lin = _replay.ReplayStash(keep=False) if self.fuse_gemm else None
        self._by_id = {id(p): p for p in params}
        self._probed: set[int] = set()       # this group's K6-probed weights
        self._pending = []                   # deferred K6 partial sums of this group
        self._lr_from_state = False          # graph capture: K1 reads lr from the state
        self._pws = {}                       # K6 workspace per weight
        self._mismatch: list = []
        self._handles = [p.register_post_accumulate_grad_hook(self._hook) for p in params]

    def _enter_group(self, pid: int) -> None:
        group = self.layer[pid] // self.clip.window
        if self._group is not None and group != self._group:
            self._flush()
        if self._group != group:
            self.engine.begin(None)           # fresh slots / overflow for this group
        self._group = group

    def _retain(self, p, g) -> None:
        self._buf.append((p, g))
        self.peak_group_grads = max(self.peak_group_grads,
                                    sum(x.numel() * x.element_size() for _, x in self._buf))

    def _hook(self, p: torch.Tensor) -> None:
        if not self._active or p.grad is None:
            return
        if id(p) in self._probed:             # K6 took this weight: another op fed it too
            self._mismatch.append(tuple(p.shape))
        g = p.grad if p.grad.is_contiguous() else p.grad.contiguous()
        p.grad = None  # RETAIN in our buffer (stabilize.py:260-266), not in .grad
        self._enter_group(id(p))
        self._retain(p, g)

    def _gemm_probe(self, wid: int, w, x, dy) -> bool:
        """K6 from the linear's backward: the retained gradient and the group
        slot's sum of squares / overflow from one tensor-core GEMM."""
        p = self._by_id.get(wid)
        if p is None or wid not in self._slot:  # not a managed leaf: autograd's dW + hook
            return False
        if p.dtype not in (torch.bfloat16, torch.float16) or p.dim() != 2:
            return False
        out_f, in_f = p.shape
        if out_f % 8 or in_f % 8:
            return False
        dy2, x2 = dy.reshape(-1, out_f), x.reshape(-1, in_f)
        if not (dy2.is_contiguous() and x2.is_contiguous()) or dy2.dtype != p.dtype \
                or x2.dtype != p.dtype:
            return False
        eng, dt = self.engine, dtype_code(p.dtype)
        need = eng.lib.lomo_gemm_probe_workspace(out_f, in_f, dy2.shape[0], dt)
        if need == 0:
            return False
        self._enter_group(wid)
        ws = self._pws.get(wid)
        if ws is None or ws.numel() < need:
            ws = self._pws[wid] = torch.empty(need, dtype=torch.uint8, device=p.device)
        g = torch.empty_like(p)               # the retained gradient: K6's store
        slot = self._slot[wid]
        rc = eng.lib.lomo_gemm_probe(dy2.data_ptr(), x2.data_ptr(), g.data_ptr(), out_f, in_f,
                                     dy2.shape[0], dt, slot,
                                     _lib.DEFER_ROWS | _lib.PROBE_KEEP_GRAD, eng.ptr,
                                     ws.data_ptr(), need, eng.stream())
        if rc == -1:
            return False
        _lib.check(rc, "lomo_gemm_probe")
        self._pending.append((ws.data_ptr(), out_f, in_f, slot, dt))
        self._probed.add(wid)
        self._retain(p, g)
        return True

    def _finish_probes(self) -> None:
        pend, self._pending = self._pending, []
        for dt in {e[4] for e in pend}:
            sel = [e for e in pend if e[4] == dt]
            k = len(sel)
            _lib.check(self.engine.lib.lomo_gemm_probe_finish(
                (ctypes.c_void_p * k)(*[e[0] for e in sel]),
                (ctypes.c_int64 * k)(*[e[1] for e in sel]),
                (ctypes.c_int64 * k)(*[e[2] for e in sel]),
                (ctypes.c_int * k)(*[e[3] for e in sel]), k, dt, self.engine.ptr,
                self.engine.stream()), "lomo_gemm_probe_finish")

    def _flush(self) -> None:
        """stabilize.py:239-258 on the device: K2 (or K6's partials) -> K3a ->
        K1 for one group."""
        if not self._buf:
            return
        eng = self.engine
        eng.configure(flags=self._probe_flags, chain=True)  # the group's K2s back to back
        for p, g in self._buf:
            if id(p) not in self._probed:
                eng.probe(g, self._slot[id(p)])
        eng.flush()
        self._finish_probes()
        eng.finalize()                        # N, coef = min(1, max_norm/N), skip if !finite
        # the group's updates run back to back after K3a: chained K1 launches
        eng.configure(0.0 if self._lr_from_state else self._lr, 0.0, self.weight_decay,
                      _lib.USE_SKIP | _lib.USE_COEF |
                      (_lib.LR_FROM_STATE if self._lr_from_state else 0), chain=True)
        for p, g in self._buf:
            eng.update(p, g)
        eng.flush()
        self._buf = []                        # gradients released (stream-ordered)
        self._probed = set()

    def fused_backward(self, loss: torch.Tensor, lr: float | None = None) -> None:
        """One grouped fused pass (stabilize.py:234-274)."""
        if not torch.isfinite(loss.detach()).all():   # _require_finite (optim.py:63-65)
            raise NonFiniteLossError(f"loss is non-finite ({float(loss.detach())}); step aborted")
        for p in self.params:
            if p.grad is not None:
                raise TapeStateError("a parameter already holds a gradient")
        self._lr = self.lr if lr is None else float(lr)
        self._backward_core(loss, False)
        st = self.engine.read_status()
        skipped = st.steps_skipped > self._skipped_before
        self._skipped_before = st.steps_skipped
        self.last_outcome = StepOutcome.SKIPPED_OVERFLOW if skipped else StepOutcome.APPLIED

    def _backward_core(self, loss: torch.Tensor, retain_graph: bool) -> None:
        """The backward with the group hooks and flushes (no host sync)."""
        self._active, self._group = True, None
        self._mismatch = []
        if self._lin is not None:
            self._lin.clear()
            self._lin.probe = self._gemm_probe
            _replay._ACTIVE = self._lin
        try:
            loss.backward(retain_graph=retain_graph)
            self._flush()
        finally:
            if self._lin is not None:
                _replay._ACTIVE = None
            self._active, self._buf, self._group = False, [], None
            self._pending, self._probed = [], set()
        if self._lin is not None and (self._lin.shared or self._mismatch):
            raise ConfigError("fuse_gemm: a weight feeds more than one op (shared or tied); "
                              "use GroupedLOMO(fuse_gemm=False)")

    def step(self, closure: Callable[[], torch.Tensor], lr: float | None = None) -> float:
        """closure() -> loss, or the reference's step(batch, lr) (see LOMO.step)."""
        from .lomo import _as_closure
        loss = _as_closure(self, closure)()
        self.fused_backward(loss, lr)
        return float(loss.detach())

    def state_nbytes(self) -> int:
        return 0

    def remove_hooks(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []
