"""CUDA-graph capture of a whole LOMO step: the two-pass replay step (below),
the strict two-pass step (pass 2 a second backward over the retained autograd
graph, with or without the fused GEMMs), the single fused pass, and
GroupedLOMO's single pass (``GraphedGroupedStep``), and ShardedLOMO's
two-pass step with its NCCL collectives (``GraphedShardedStep``).

A LLaMA-7B step issues ~3,000 kernels -- autograd's, the hook kernels, K5 --
and at seq 1024 the host cannot launch them as fast as the B200 runs them.
``GraphedLOMOStep`` captures the step into two CUDA graphs around the one
host decision of the protocol (stabilize.py:204-205):

* graph 1: forward, ``begin_step`` (loss check), pass-1 backward whose hooks
  launch K2 and stash (x, dy) for replay, the end-of-backward flush, K3a;
* host: read the 128-byte status (the one sync) -- skip, underflow, or go;
* graph 2: ``lomo_update_coefs`` (alpha/beta from the device state), the
  replayed updates -- K5 with device-side alpha/beta for every linear, K1
  with ``LOMO_LR_FROM_STATE`` for the rest -- and K3b.

Everything the step reads that changes between steps lives in device memory
(the batch in static input tensors, loss scale, clip coefficient, skip flag,
and the learning rate, set with ``lomo_set_lr`` before each replay), so the
graphs are captured once.  The numerics are those of the eager replay step.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch

from . import _lib
from .errors import ConfigError, NonFiniteLossError, ScaleUnderflowError
from .lomo import LOMO, _PROBE, _UPDATE
from .stabilize import StepOutcome


class GraphedLOMOStep:
    """Capture ``loss_fn(*static_inputs)`` + the LOMO two-pass replay step.

    Args:
        opt: a :class:`LOMO` with a two-pass stabiliser (clip_grad_norm and/or
            loss_scale), built with ``replay=True`` (``fuse_gemm`` optional), or
            with ``fuse_gemm=True`` alone: the reference's protocol as is -- pass
            2 a second backward over the retained graph, K6 in pass 1 and K5
            inside pass 2 -- captured the same way (no replay stash; also
            without ``fuse_gemm``: the hook kernels K2 / K1 in the two
            backwards); or a
            single-pass LOMO with ``fuse_gemm=True`` (K5 inside the one
            backward): graph 1 is the forward, the host checks the loss
            (optim.py:63-65), graph 2 the backward.
        loss_fn: the forward, returning the scalar loss.
        static_inputs: tensors ``loss_fn`` reads; copy each batch into them.
        warmup: eager steps run before capture (they also perform replay's
            first-step gradient check).
        lr: learning rate for the warm-up steps.
    """

    def __init__(self, opt: LOMO, loss_fn: Callable[..., torch.Tensor],
                 static_inputs: Sequence[torch.Tensor], warmup: int = 2, lr: float = 1e-3):
        if not isinstance(opt, LOMO) or (opt.passes == 1 and not opt._fused_update):
            raise ConfigError("GraphedLOMOStep needs a two-pass LOMO (clip_grad_norm and/or "
                              "loss_scale) or a single-pass LOMO with fuse_gemm=True")
        self.single = opt.passes == 1
        self.strict = opt._stash is None
        if opt.clip_value:
            raise ConfigError("value clipping is a single-pass mode; graph it with LOMO directly")
        self.opt, self.loss_fn, self.inputs = opt, loss_fn, tuple(static_inputs)
        eng = opt.engine
        self.coefs = torch.zeros(2, dtype=torch.float32, device=opt.device)
        side = torch.cuda.Stream(opt.device)
        side.wait_stream(torch.cuda.current_stream(opt.device))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                opt.step(lambda: loss_fn(*self.inputs), lr)
        torch.cuda.current_stream(opt.device).wait_stream(side)
        torch.cuda.synchronize(opt.device)
        if not self.strict and not opt._replay_checked:
            raise ConfigError("replay's first-step check did not run during warm-up")

        pool = torch.cuda.graph_pool_handle()
        if self.single:
            self._capture_single(pool)
            self.steps = 0
            return
        self.g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g1, pool=pool):
            self.loss = loss_fn(*self.inputs)
            eng.begin(self.loss)
            eng.configure(flags=opt._flags(_PROBE))
            # strict: the autograd graph is kept for pass 2's backward (and
            # across replays -- its saved tensors live in the graph pool)
            opt._run_backward(opt._scaled(self.loss), _PROBE, self.strict)
            opt._decide()
        self.g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g2, pool=pool):
            self._capture_pass2()
        self.steps = 0

    def _capture_single(self, pool) -> None:
        """Single pass: g1 = forward (+ the device loss flag), g2 = the
        backward with K5 in every linear and K1 for the rest (lr, alpha and
        beta from the device state).  The autograd graph is kept across
        replays (its saved tensors live in the graph pool)."""
        opt, eng = self.opt, self.opt.engine
        self.g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g1, pool=pool):
            self.loss = self.loss_fn(*self.inputs)
            eng.begin(opt._check_loss(self.loss))
        self.g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g2, pool=pool):
            eng.configure(0.0, opt.clip_value, opt.weight_decay,
                          opt._flags(_UPDATE) | _lib.LR_FROM_STATE)
            opt._lr_from_state = True
            try:
                opt._run_backward(self.loss, _UPDATE, True)
            finally:
                opt._lr_from_state = False
            eng.on_clean()

    def _capture_pass2(self) -> None:
        opt, eng = self.opt, self.opt.engine
        flags = opt._flags(2) | _lib.LR_FROM_STATE
        if self.strict:
            # the second backward with K5 in every linear (alpha/beta computed on
            # device from the state, whose lr step() sets before each replay)
            eng.configure(0.0, opt.clip_value, opt.weight_decay, flags)
            opt._lr_from_state = True
            try:
                opt._run_backward(opt._scaled(self.loss), _UPDATE, True)
            finally:
                opt._lr_from_state = False
            eng.on_clean()
            return
        _lib.check(eng.lib.lomo_update_coefs(eng.ptr, opt.weight_decay, flags,
                                             self.coefs.data_ptr(), eng.stream()),
                   "lomo_update_coefs")
        eng.configure(0.0, opt.clip_value, opt.weight_decay, flags)
        opt._replay_pass(0.0, coefs=self.coefs if opt.fuse_gemm else None)
        eng.on_clean()

    def step(self, lr: float) -> torch.Tensor:
        """One captured step; returns the (device) loss tensor of this step."""
        opt, eng = self.opt, self.opt.engine
        _lib.check(eng.lib.lomo_set_lr(eng.ptr, float(lr), eng.stream()), "lomo_set_lr")
        self.g1.replay()
        if self.single:
            loss = float(self.loss.detach())  # the one host sync: the loss check
            if loss != loss or loss in (float("inf"), float("-inf")):
                opt.last_outcome = None
                raise NonFiniteLossError(f"loss is non-finite ({loss}); step aborted")
            self.g2.replay()
            opt.last_outcome = None if opt.stabilizer is None else StepOutcome.APPLIED
            self.steps += 1
            return self.loss
        st = eng.read_status()          # the one host sync of the step
        opt._mirror_scaler(st)
        if st.underflow:
            raise ScaleUnderflowError(
                f"loss scale would fall below {st.min_scale}; training diverged")
        opt.last_norm, opt.clip_coef = float(st.total_norm), float(st.clip_coef)
        if st.skip:
            opt.last_outcome = StepOutcome.SKIPPED_OVERFLOW
        else:
            self.g2.replay()
            opt._scaler_clean()
            opt.last_outcome = StepOutcome.APPLIED
        self.steps += 1
        return self.loss


class GraphedGroupedStep:
    """``GroupedLOMO``'s single pass (per-group clipping, stabilize.py:234-274)
    captured as two CUDA graphs: graph 1 the forward; the host checks the
    loss (optim.py:63-65); graph 2 the backward, whose group flushes run K2
    (or read K6's partials), K3a and K1 with the learning rate from the
    device state.  The outcome is read after graph 2, as the eager step does.

    Args as :class:`GraphedLOMOStep`.
    """

    def __init__(self, opt, loss_fn: Callable[..., torch.Tensor],
                 static_inputs: Sequence[torch.Tensor], warmup: int = 2, lr: float = 1e-3):
        from .grouped import GroupedLOMO
        if not isinstance(opt, GroupedLOMO):
            raise ConfigError("GraphedGroupedStep needs a GroupedLOMO")
        self.opt, self.loss_fn, self.inputs = opt, loss_fn, tuple(static_inputs)
        dev = opt.params[0].device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                opt.step(lambda: loss_fn(*self.inputs), lr)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        pool = torch.cuda.graph_pool_handle()
        self.g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g1, pool=pool):
            self.loss = loss_fn(*self.inputs)
        self.g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g2, pool=pool):
            opt._lr_from_state = True
            try:
                opt._backward_core(self.loss, True)
            finally:
                opt._lr_from_state = False
        self.steps = 0

    def step(self, lr: float) -> torch.Tensor:
        opt, eng = self.opt, self.opt.engine
        _lib.check(eng.lib.lomo_set_lr(eng.ptr, float(lr), eng.stream()), "lomo_set_lr")
        self.g1.replay()
        loss = float(self.loss.detach())
        if loss != loss or loss in (float("inf"), float("-inf")):
            raise NonFiniteLossError(f"loss is non-finite ({loss}); step aborted")
        self.g2.replay()
        st = eng.read_status()
        skipped = st.steps_skipped > opt._skipped_before
        opt._skipped_before = st.steps_skipped
        opt.last_outcome = StepOutcome.SKIPPED_OVERFLOW if skipped else StepOutcome.APPLIED
        self.steps += 1
        return self.loss


class GraphedShardedStep:
    """:class:`~paper_2306_09782_b200.sharded.ShardedLOMO`'s two-pass step
    captured as two CUDA graphs, NCCL collectives included (one process per
    GPU; every rank captures and replays the same sequence):

    * graph 1: the refresh all-gathers of the updated parameter shards (each
      layer's forward waits for its own bucket), the forward, the cross-rank
      loss sum and ``begin_step``, the pass-1 backward -- per bucket the
      asynchronous ``reduce_scatter_tensor`` and K2 on this rank's shard --,
      then the local K3 partial, the ``all_gather`` of ``{sumsq, overflow}``
      and K3a on the rank-ordered sum;
    * host: the one status read (stabilize.py:204-205);
    * graph 2: pass 2 -- K1 over pass 1's kept gradient shards
      (``keep_grads``), or the replayed buckets' reduce-scatter + K1
      (``replay``) -- with the learning rate from the device state, and K3b.

    The host-side step (``ShardedLOMO.step``) launches ~2,000 kernels and
    ~80 collectives per step; replaying the graphs removes that host cost.
    Needs the layers kept gathered (``reshard_after_forward=False``: ZeRO-3's
    per-layer free and re-gather resize storage, which a graph cannot).  With
    ``fused_rs`` the K4 kernels and their device barriers are captured too
    (the barriers' epochs are device counters the replays advance; the peer
    ring's buffer rotation is the captured one, identical on every rank).
    Numerics are those of the eager step.

    Args as :class:`GraphedLOMOStep`.
    """

    def __init__(self, opt, loss_fn: Callable[..., torch.Tensor],
                 static_inputs: Sequence[torch.Tensor], warmup: int = 2, lr: float = 1e-3):
        from .sharded import ShardedLOMO, _KeptShards
        if not isinstance(opt, ShardedLOMO) or opt.passes != 2:
            raise ConfigError("GraphedShardedStep needs a two-pass ShardedLOMO "
                              "(clip_grad_norm and/or loss_scale)")
        if any(not b.persistent for b in opt.buckets):
            raise ConfigError("GraphedShardedStep needs reshard_after_forward=False (ZeRO-3's "
                              "per-layer free/re-gather resizes storage inside the step)")
        if opt._stash is None:
            raise ConfigError("GraphedShardedStep needs keep_grads=True or replay=True (pass 2 "
                              "without a second forward/backward)")
        if opt.clip_value:
            raise ConfigError("value clipping is a single-pass mode")
        self.opt, self.loss_fn, self.inputs = opt, loss_fn, tuple(static_inputs)
        self.keep = isinstance(opt._stash, _KeptShards)
        dev = opt.device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                opt.step(lambda: loss_fn(*self.inputs), lr)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        for b in opt.buckets:
            b.wait()
        for ring in opt._rings.values():
            # every buffer's first use in the captured sequence waits for the
            # peers to finish reading it (its previous use is the previous replay)
            ring.read_pending = [True] * ring.NBUF
        eng = opt.engine
        pool = torch.cuda.graph_pool_handle()
        self.g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g1, pool=pool):
            # the refresh gathers of every bucket (captured unconditionally:
            # after a skipped step they re-gather unchanged shards)
            for b in opt.buckets:
                b.dirty = True
            opt._refresh()
            self.loss = loss_fn(*self.inputs)
            eng.begin(opt._check_loss(self.loss))
            eng.configure(flags=opt._flags(_PROBE))
            opt._run_backward(opt._scaled(self.loss), _PROBE, False)
            opt._decide()
        self.g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g2, pool=pool):
            eng.configure(0.0, 0.0, opt.weight_decay, opt._flags(_UPDATE) | _lib.LR_FROM_STATE)
            opt._replay_pass(0.0)
            eng.on_clean()
        for b in opt.buckets:
            b.dirty = False  # the refresh lives in graph 1
        self.steps = 0

    def step(self, lr: float) -> torch.Tensor:
        """One captured sharded step; returns the (device) loss tensor."""
        opt, eng = self.opt, self.opt.engine
        _lib.check(eng.lib.lomo_set_lr(eng.ptr, float(lr), eng.stream()), "lomo_set_lr")
        self.g1.replay()
        st = eng.read_status()          # the one host sync of the step
        opt._mirror_scaler(st)
        if st.underflow:
            raise ScaleUnderflowError(
                f"loss scale would fall below {st.min_scale}; training diverged")
        opt.last_norm, opt.clip_coef = float(st.total_norm), float(st.clip_coef)
        if st.skip:
            opt.last_outcome = StepOutcome.SKIPPED_OVERFLOW
        else:
            self.g2.replay()
            opt._scaler_clean()
            opt.last_outcome = StepOutcome.APPLIED
            for b in opt.buckets:
                # the next graph-1 replay re-gathers them; an eager refresh
                # before that (gather_all, an eager step) must too
                b.dirty = True
        self.steps += 1
        return self.loss
