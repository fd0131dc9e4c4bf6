"""ShardedLOMO: the fused update with ZeRO-3 parameter sharding across the
GPUs of one box (north star (3)).

* Parameters are grouped into buckets (default: one per decoder layer, i.e.
  per entry of ``model.layers``, plus one "rest" bucket for the embedding,
  final norm and head).  A bucket is one flat buffer padded to a multiple of
  ``8 * world`` elements; rank r permanently owns the contiguous slice
  ``[r*S, (r+1)*S)`` (``bucket.shard``).  That slice is the authoritative copy
  of those parameters -- the only one that is ever updated.
* ZeRO-3 life cycle of a layer bucket: ``all_gather_into_tensor`` into the full
  buffer before the module's forward, released (storage freed) after it;
  gathered again before the module's backward, released once its gradients
  have been reduced; each gather prefetches the next layer's.  With
  ``reshard_after_forward=False`` (or for the rest bucket) the full buffer
  stays and is refreshed from the updated shards after every applied step:
  all refresh gathers are issued at once, each layer waits for its own.
* Gradients: a linear's backward GEMMs its weight gradient straight into the
  bucket's flat buffer (``direct_grads``); other parameters' hooks copy theirs
  and drop ``p.grad``.  When the last gradient of a bucket arrives, ONE
  asynchronous ``reduce_scatter_tensor`` (SUM, NCCL over NVLink) produces this
  rank's shard of the summed gradient and the fused kernel runs on it --
  enqueued once the next bucket's collective is issued, so the collective
  overlaps the backward: K2 (pass 1: overflow + sum of squares) or K1 (pass 2 /
  single pass: ``p_shard -= lr * ...``).  The 1/world of the data-parallel
  mean is folded into the state's ``inv_scale`` (``grad_div``), so clipping
  sees the mean gradient exactly like the single-GPU reference.
* ``replay=True``: pass 2 re-derives the local gradients from the stashed
  (x, dy) of pass 1 instead of a second forward/backward.
* Global norm (two-pass mode): each rank reduces its slots (K3, local mode),
  one ``all_gather`` exchanges ``{sumsq, overflow}`` per rank, and K3a decides
  on the rank-ordered sum -- the same bits on every rank, no float atomics.
* Gradient peak: one bucket (flat) instead of one tensor.
* ``fused_rs`` (K4): the flat gradient buffers are peer-mapped (``peer.py``:
  CUDA IPC, or an NVSwitch multicast object); when a bucket is complete every
  rank runs ONE kernel that reduces its slice over all ranks' buffers -- P2P
  loads summed in rank order (IPC), or ``multimem.ld_reduce`` (NVLS) -- and
  applies the update (or the probe) directly: no reduce-scatter output is
  ever written.  Three buffers rotate between buckets (autograd can
  interleave adjacent buckets); a device barrier before the kernel (all ranks
  wrote the bucket) and one before a buffer is refilled (all ranks finished
  reading it) order the ranks.
"""
from __future__ import annotations

import math
import os

import torch
import torch.distributed as dist

from . import peer as _peer
from . import replay as _replay
from .engine import CudaEngine, dtype_code
from .errors import ConfigError
from .lomo import _PROBE, _UPDATE, _Protocol, stabilizer_from_args, trainable_params
from .stabilize import Stabilizer


def _backend(group) -> str:
    return dist.get_backend(group)


def all_gather_into(out: torch.Tensor, inp: torch.Tensor, group, async_op: bool = False):
    """out[r*S:(r+1)*S] = inp of rank r (NCCL all_gather_into_tensor);
    ``async_op``: returns the NCCL work handle (gloo completes, None)."""
    if _backend(group) == "nccl":
        return dist.all_gather_into_tensor(out, inp, group=group, async_op=async_op)
    # gloo (CPU tests): list form; the input may be this rank's chunk of
    # `out` (persistent buckets gather in place), so it is copied first
    dist.all_gather(list(out.chunk(dist.get_world_size(group))), inp.clone(), group=group)
    return None


def reduce_scatter(out: torch.Tensor, inp: torch.Tensor, group, async_op: bool = False):
    """out = (sum over ranks of inp)[rank*S:(rank+1)*S] (NCCL reduce_scatter_tensor).
    ``async_op``: returns the NCCL work handle (``wait()`` makes the current
    stream wait for it); gloo always completes before returning (None)."""
    if _backend(group) == "nccl":
        return dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group,
                                          async_op=async_op)
    # gloo has no reduce_scatter_tensor: all_reduce + slice (CPU tests only)
    tmp = inp.clone()
    dist.all_reduce(tmp, group=group)
    r, w = dist.get_rank(group), dist.get_world_size(group)
    out.copy_(tmp.chunk(w)[r])
    return None


class _Bucket:
    def __init__(self, idx: int, params: list, module, persistent: bool, world: int,
                 rank: int, group):
        self.idx = idx
        self.params = params
        self.module = module
        self.persistent = persistent
        self.group = group
        dev, dt = params[0].device, params[0].dtype
        for p in params:
            if p.dtype != dt or p.device != dev:
                raise ConfigError("a bucket's parameters must share dtype and device")
        self.dtype, self.device = dt, dev
        self.numels = [p.numel() for p in params]
        self.offsets = [0]
        for n in self.numels[:-1]:
            self.offsets.append(self.offsets[-1] + n)
        total = sum(self.numels)
        align = 8 * world
        self.padded = int(math.ceil(total / align) * align)
        self.S = self.padded // world
        full = torch.zeros(self.padded, dtype=dt, device=dev)
        with torch.no_grad():
            for p, off, n in zip(params, self.offsets, self.numels):
                full[off:off + n].copy_(p.detach().reshape(-1))
                p.data = full[off:off + n].view(p.shape)  # frees the original storage
        dist.broadcast(full, src=dist.get_global_rank(group, 0) if group is not None else 0,
                       group=group)  # every rank starts from rank 0's weights
        # a persistent bucket's shard IS its slice of the full buffer: the
        # update writes the gathered parameters in place and the refresh
        # all-gather runs in place (no copy of this rank's own slice; at
        # world 1 no copy at all).  A ZeRO-3 bucket frees `full` after use, so
        # its shard is its own allocation.
        sl = full[rank * self.S:(rank + 1) * self.S]
        self.shard = sl if persistent else sl.clone()
        self.full = full
        self.nbytes = self.padded * full.element_size()
        self.gathered = True
        self.dirty = False
        self.gflat = None
        self.remaining = len(params)
        self.filled = [False] * len(params)  # which ranges of gflat hold a gradient
        self.reduced = False  # this pass's reduce-scatter + kernel already ran
        self.pending = None   # in-flight refresh all-gather (persistent buckets)
        if not persistent:
            self.release()

    def wait(self) -> None:
        """Make the current stream wait for this bucket's refresh gather."""
        if self.pending is not None:
            self.pending.wait()
            self.pending = None

    def gather(self, async_op: bool = False) -> None:
        """All-gather the full parameters; ``async_op`` only issues it (a
        prefetch: the next ``gather()`` or ``wait()`` orders the stream)."""
        if not self.gathered:
            self.full.untyped_storage().resize_(self.nbytes)
            self.pending = all_gather_into(self.full, self.shard, self.group, async_op=True)
            self.gathered = True
            self.dirty = False
        if not async_op:
            self.wait()

    def release(self) -> None:
        if self.persistent or not self.gathered:
            return
        self.wait()  # never free a buffer a gather is still writing
        self.full.untyped_storage().resize_(0)
        self.gathered = False


class _KeptShards:
    """ShardedLOMO(keep_grads=True): pass 1's reduced gradient shard per
    bucket, consumed by pass 2 (the protocol treats it like a replay stash)."""

    def __init__(self):
        self.shards: dict[int, torch.Tensor] = {}

    def clear(self) -> None:
        self.shards.clear()


def _pick_transport(fused_rs, device, group) -> str:
    """fused_rs=True / "auto": NVLS when every rank has its own multicast-capable
    GPU, else CUDA IPC; "ipc" / "nvls" force one."""
    if fused_rs in ("ipc", "nvls"):
        return fused_rs
    if fused_rs not in (True, "auto"):
        raise ConfigError(f"fused_rs must be False, True, 'auto', 'ipc' or 'nvls', got {fused_rs!r}")
    world = dist.get_world_size(group)
    props = torch.cuda.get_device_properties(device)
    mine = (os.uname().nodename, str(getattr(props, "uuid", device)),
            _peer.nvls_available(device))
    everyone: list = [None] * world
    dist.all_gather_object(everyone, mine, group=group)
    distinct = len({(h, u) for h, u, _ in everyone}) == world
    return "nvls" if distinct and all(ok for _, _, ok in everyone) else "ipc"


class ShardedLOMO(_Protocol):
    """LOMO over ZeRO-3 parameter shards, one process per GPU.

    Same public API as :class:`~paper_2306_09782_b200.LOMO`
    (``grad_norm``, ``fused_backward``, ``step``); the model must be built
    identically on every rank (rank 0's weights are broadcast at construction).

    Args:
        buckets: modules whose parameters form one bucket each (default:
            ``model.layers``); remaining parameters form a persistent bucket.
        reshard_after_forward: free each layer bucket's full parameters after
            its forward (ZeRO-3); False keeps them resident (ZeRO-2-like).
        process_group: the data-parallel group (default: WORLD).
        fused_rs: K4 -- reduce over peer memory fused with the update instead
            of NCCL reduce_scatter + K1/K2.  ``True``/``"auto"``: NVLS
            multicast when every rank has its own multicast-capable GPU, else
            CUDA IPC; ``"ipc"`` / ``"nvls"`` force a transport.
        direct_grads: weight gradients of the model's linears
            (``replay.linear`` / ``replay.matmul_in_out``) are computed by the
            linear's backward straight into the bucket's flat buffer
            (``mm(..., out=)``): no per-parameter copy, autograd never holds
            them.  A weight that feeds several linears gets the later
            contributions added through its hook; one whose bucket was already
            reduced raises ``ConfigError`` (pass ``direct_grads=False``).
        replay: two-pass mode without the second forward/backward, as
            :class:`~paper_2306_09782_b200.LOMO` ``replay=True``: pass 1 keeps
            each linear's (x, dy) and the other parameters' gradients; pass 2
            re-derives every local gradient from them (the same GEMM) into the
            buckets and runs the same reduce-scatter + K1 per bucket.  Pass 2
            needs no parameter gather.  Needs ``direct_grads``.
        keep_grads: two-pass mode keeping this rank's reduced gradient shard
            of every bucket from pass 1 (1/world of the gradients: 180 GB of
            HBM holds them) -- pass 2 is K1 over the kept shards, with no
            gradient recompute and no second reduce-scatter.  The update is
            the same as the strict protocol's (pass 1's reduced gradient IS
            pass 2's).  With ``fused_rs`` the K4 probe writes the reduced
            slice as it sums it (``lomo_fused_rs_probe_keep``).
    """

    _always_scale = True  # inv_scale carries the 1/world of the data-parallel mean

    def __init__(self, model, lr: float = 1e-3, clip_grad_norm: float | None = None,
                 loss_scale=None, *, clip_grad_value: float | None = None,
                 weight_decay: float = 0.0, stabilizer: Stabilizer | None = None,
                 math: str = "f32", buckets=None, reshard_after_forward: bool = True,
                 process_group=None, fused_rs: bool | str = False, direct_grads: bool = True,
                 replay: bool = False, keep_grads: bool = False, _engine=None):
        if not dist.is_initialized():
            raise ConfigError("ShardedLOMO needs torch.distributed to be initialised")
        if stabilizer is not None and (clip_grad_norm or clip_grad_value or loss_scale):
            raise ConfigError("pass either a Stabilizer or the clip/loss_scale arguments")
        st = stabilizer if stabilizer is not None else stabilizer_from_args(
            clip_grad_norm, clip_grad_value, loss_scale)
        self._init_protocol(st, lr, weight_decay)
        # option checks before the parameters are moved into buckets
        if keep_grads and replay:
            raise ConfigError("keep_grads replaces replay (pass 2 updates from the kept shards)")
        if keep_grads and self.passes != 2:
            raise ConfigError("keep_grads replaces the second pass: it needs clip_grad_norm "
                              "or loss_scale")
        if replay and not direct_grads:
            raise ConfigError("ShardedLOMO(replay=True) needs direct_grads=True")
        if replay and self.passes != 2:
            raise ConfigError("replay replaces the second pass: it needs clip_grad_norm or "
                              "loss_scale")
        self.group = process_group
        self.world = dist.get_world_size(process_group)
        self.rank = dist.get_rank(process_group)
        params = trainable_params(model)
        for p in params:
            dtype_code(p.dtype)
        mods = list(buckets) if buckets is not None else list(getattr(model, "layers", []))
        assigned: set[int] = set()
        self.buckets: list[_Bucket] = []
        for m in mods:
            ps = [p for p in m.parameters() if p.requires_grad and id(p) not in assigned]
            if not ps:
                continue
            assigned.update(id(p) for p in ps)
            self.buckets.append(_Bucket(len(self.buckets), ps, m, not reshard_after_forward,
                                        self.world, self.rank, process_group))
        rest = [p for p in params if id(p) not in assigned]
        by_dtype: dict = {}
        for p in rest:
            by_dtype.setdefault(p.dtype, []).append(p)
        for ps in by_dtype.values():
            self.buckets.append(_Bucket(len(self.buckets), ps, None, True, self.world,
                                        self.rank, process_group))
        self._loc = {}
        for b in self.buckets:
            for j, (p, off, n) in enumerate(zip(b.params, b.offsets, b.numels)):
                self._loc[id(p)] = (b, off, n, j)
        self.params = params
        self._model = model
        self.device = params[0].device
        self.engine = _engine if _engine is not None else CudaEngine(
            self.device, len(self.buckets), self.scaler, self.max_norm, math,
            grad_div=float(self.world))
        self._mode = 0
        self.fused_rs = fused_rs is not False and fused_rs is not None
        self._rings: dict = {}
        self.transport = None
        if self.fused_rs:
            if self.device.type != "cuda" or self.world > 16:
                raise ConfigError("fused_rs needs CUDA peers (<= 16 ranks over NVLink)")
            self.transport = _pick_transport(fused_rs, self.device, process_group)
            if self.transport == "nvls" and any(b.dtype == torch.float64 for b in self.buckets):
                raise ConfigError("fused_rs='nvls' reduces f32/f16/bf16 buckets (multimem has no "
                                  "f64 vector form); use fused_rs='ipc'")
            for dt in sorted({b.dtype for b in self.buckets}, key=str):  # same order on every rank
                n = max(b.padded for b in self.buckets if b.dtype == dt)
                self._rings[dt] = _peer.PeerRing(n, dt, self.device, process_group,
                                                 self.transport, err_ptr=self.engine.error_ptr)
        self._lin = None
        if direct_grads:
            self._lin = _replay.ReplayStash(keep=replay)
            self._lin.probe = self._lin.update = self._dw_into_bucket
        self._stash = self._lin if replay else (_KeptShards() if keep_grads else None)
        self._replay_mismatch = False
        self._inflight: list = []
        self._handles = [p.register_post_accumulate_grad_hook(self._hook) for p in params]
        layers = [b for b in self.buckets if b.module is not None and not b.persistent]
        for k, b in enumerate(layers):
            # ZeRO-3: gather this layer, prefetch the next one in execution
            # order (forward: k+1; backward: k-1) so its all-gather overlaps
            # this layer's compute
            nxt = layers[k + 1] if k + 1 < len(layers) else None
            prv = layers[k - 1] if k > 0 else None
            self._handles.append(b.module.register_forward_pre_hook(
                lambda mod, args, b=b, n=nxt: self._gather_fwd(b, n)))
            self._handles.append(b.module.register_forward_hook(
                lambda mod, args, out, b=b: self._after_forward(b)))
            self._handles.append(b.module.register_full_backward_pre_hook(
                lambda mod, gout, b=b, n=prv: self._gather_bwd(b, n)))
        for b in self.buckets:
            if b.module is not None and b.persistent:
                # the refresh gather was issued at the model's forward start;
                # this layer waits for its own bucket only
                self._handles.append(b.module.register_forward_pre_hook(
                    lambda mod, args, b=b: b.wait()))
        self._handles.append(model.register_forward_pre_hook(lambda mod, args: self._refresh()))

    # ---------------------------------------------------------------- ZeRO-3
    @staticmethod
    def _gather_fwd(b: _Bucket, nxt) -> None:
        b.gather()
        if nxt is not None and torch._C._current_graph_task_id() == -1:
            nxt.gather(async_op=True)  # not during a checkpoint recompute

    @staticmethod
    def _gather_bwd(b: _Bucket, prv) -> None:
        b.gather()
        if prv is not None:
            prv.gather(async_op=True)

    def _after_forward(self, b: _Bucket) -> None:
        # keep the parameters while autograd recomputes a checkpointed layer
        if torch._C._current_graph_task_id() == -1:
            b.release()

    def _refresh(self) -> None:
        """Re-gather persistent buckets whose shards were updated: every
        gather is issued at once (NCCL runs them in order: the module-less
        buckets -- embedding, final norm, head -- first, then the layers in
        forward order) and each layer's forward pre-hook waits for its own,
        so the later gathers overlap the earlier layers' forward."""
        order = [b for b in self.buckets if b.module is None] + \
                [b for b in self.buckets if b.module is not None]
        for b in order:
            if b.persistent and b.dirty:
                b.pending = all_gather_into(b.full, b.shard, self.group, async_op=True)
                b.dirty = False
        for b in order:
            if b.module is None:
                b.wait()

    # ----------------------------------------------------------------- hooks
    def _hook(self, p: torch.Tensor) -> None:
        if self._mode == 0 or p.grad is None:
            return
        b, off, n, j = self._loc[id(p)]
        if b.reduced:
            raise ConfigError("direct_grads: a weight shared by several linears completed "
                              "its bucket before its last gradient; use direct_grads=False")
        if b.filled[j]:
            # a weight shared by several linears: direct_grads wrote the first
            # contributions, autograd delivers the rest here
            b.gflat[off:off + n].add_(p.grad.reshape(-1))
            p.grad = None
            self._replay_mismatch = True  # replay would drop this contribution
            return
        if self._stash is self._lin and self._stash is not None and self._mode == _PROBE:
            self._stash.grads[id(p)] = p.grad  # replay: not a linear, kept for pass 2
        if b.gflat is None:
            self._new_gflat(b)
        b.gflat[off:off + n].copy_(p.grad.reshape(-1))
        b.filled[j] = True
        p.grad = None
        b.remaining -= 1
        if b.remaining == 0:
            self._reduce(b)

    def _dw_into_bucket(self, wid: int, w, a: torch.Tensor, d: torch.Tensor) -> bool:
        """The linear's weight gradient dW = d^T a, written by the GEMM into
        the bucket's flat buffer (replay.weight_grad's GEMM with out=)."""
        loc = self._loc.get(wid)
        if loc is None or self._mode == 0:
            return False
        b, off, n, j = loc
        if b.reduced:
            return False  # -> autograd -> _hook raises ConfigError
        if a.dtype != b.dtype or d.dtype != b.dtype:
            return False  # e.g. autocast activations: autograd's dW, then the hook
        if b.gflat is None:
            self._new_gflat(b)
        view = b.gflat[off:off + n].view(d.shape[-1], a.shape[-1])
        d2, a2 = d.reshape(-1, d.shape[-1]), a.reshape(-1, a.shape[-1])
        if b.filled[j]:
            view.addmm_(d2.t(), a2)
            return True
        torch.mm(d2.t(), a2, out=view)
        b.filled[j] = True
        b.remaining -= 1
        if b.remaining == 0:
            self._reduce(b)
        return True

    def _new_gflat(self, b: _Bucket) -> None:
        """The bucket's flat gradient buffer, uninitialised: every range is
        either written by its parameter's hook or zeroed in _zero_unfilled."""
        if self.fused_rs:
            ring = self._rings[b.dtype]
            b.ring_k = ring.acquire(b.idx)
            b.gflat = ring.bufs[b.ring_k][:b.padded]
        else:
            b.gflat = torch.empty(b.padded, dtype=b.dtype, device=b.device)

    @staticmethod
    def _zero_unfilled(b: _Bucket) -> None:
        """Zero the padding and the ranges of parameters that received no
        gradient this pass (the summed gradient there is exactly 0)."""
        end = b.offsets[-1] + b.numels[-1]
        if end < b.padded:
            b.gflat[end:].zero_()
        for j, done in enumerate(b.filled):
            if not done:
                b.gflat[b.offsets[j]:b.offsets[j] + b.numels[j]].zero_()

    def _reduce(self, b: _Bucket) -> None:
        """One reduce-scatter feeding the fused kernel on this rank's shard."""
        if b.gflat is None:
            self._new_gflat(b)
        self._zero_unfilled(b)
        if self.fused_rs:
            # K4: every rank has written the bucket -> reduce over peer memory
            # fused with the update / probe; nothing is written back
            ring = self._rings[b.dtype]
            ring.filled(b.ring_k)  # every rank has written this bucket
            if self._mode == _PROBE:
                if isinstance(self._stash, _KeptShards):
                    # keep_grads over K4: the probe also writes the reduced
                    # slice (rounded to storage), pass 2's K1 input
                    gshard = torch.empty(b.S, dtype=b.dtype, device=b.device)
                    ring.probe(self.engine, b.ring_k, self.rank * b.S, b.S, b.idx, out=gshard)
                    self._stash.shards[b.idx] = gshard
                else:
                    ring.probe(self.engine, b.ring_k, self.rank * b.S, b.S, b.idx)
            else:
                ring.update(self.engine, b.shard, b.ring_k, self.rank * b.S)
                b.dirty = True
            ring.release(b.ring_k)
            b.gflat = None
            b.remaining = len(b.params)
            b.reduced = True
            b.release()
            return
        # the reduce-scatter runs on NCCL's stream while the backward goes on;
        # this bucket's K2/K1 is enqueued once the NEXT bucket has been handed
        # to NCCL (or at the end of the pass), so the compute stream never
        # waits on the collective it could overlap
        self._drain(keep=0)
        if isinstance(self._stash, _KeptShards) and self._mode == _PROBE and self.world > 1:
            # a kept shard outlives the step: its own compact allocation
            gshard = torch.empty(b.S, dtype=b.dtype, device=b.device)
        else:
            # in place: this rank's slice of the flat buffer receives the sum
            # (NCCL's in-place reduce-scatter; no copy at all at world 1)
            gshard = b.gflat[self.rank * b.S:(self.rank + 1) * b.S]
        work = reduce_scatter(gshard, b.gflat, self.group, async_op=True)
        self._inflight.append((work, gshard, b, self._mode))
        b.gflat = None
        b.remaining = len(b.params)
        b.reduced = True
        b.release()

    def _drain(self, keep: int = 0) -> None:
        """Run the fused kernel of every in-flight bucket but the newest
        ``keep`` (after its reduce-scatter, stream-ordered)."""
        while len(self._inflight) > keep:
            work, gshard, b, mode = self._inflight.pop(0)
            if work is not None:
                work.wait()
            if mode == _PROBE:
                self.engine.probe(gshard, b.idx)
                if isinstance(self._stash, _KeptShards):
                    self._stash.shards[b.idx] = gshard  # pass 2 updates from it
            else:
                self.engine.update(b.shard, gshard)
                b.dirty = True

    def _run_backward(self, target: torch.Tensor, mode: int, retain_graph: bool) -> None:
        self._mode = mode
        for b in self.buckets:
            b.reduced = False
            b.filled = [False] * len(b.params)
        if self._lin is not None:
            self._lin.clear()
            _replay._ACTIVE = self._lin
        try:
            target.backward(retain_graph=retain_graph)
            # parameters that received no gradient: reduce their (zero) buckets
            # in bucket order -- the same collective order on every rank
            for b in self.buckets:
                if b.remaining != len(b.params) or b.gflat is not None:
                    self._reduce(b)
            self._drain()
        finally:
            self._mode = 0
            if self._lin is not None:
                _replay._ACTIVE = None
            self.engine.flush()
        st = self._stash
        if st is not None and st is self._lin and mode == _PROBE and \
                (st.shared or self._replay_mismatch):
            st.clear()
            self._replay_mismatch = False
            raise ConfigError("replay: a weight receives gradient from more than one op "
                              "(shared or tied); use replay=False")

    def _replay_pass(self, lr: float, coefs=None) -> None:
        """Pass 2 from the stash: per bucket (a fixed order, identical on
        every rank), every local gradient re-derived into the flat buffer --
        dW = dy^T x for the linears, the kept tensor for the rest -- then the
        bucket's reduce-scatter + K1 on this rank's shard."""
        st = self._stash
        if isinstance(st, _KeptShards):
            # pass 1 already produced this rank's reduced gradient shards; the
            # K1s over them run back to back (chained launches)
            self.engine.chain_updates()
            try:
                for b in self.buckets:
                    g = st.shards.pop(b.idx, None)
                    if g is not None:
                        self.engine.update(b.shard, g)
                        b.dirty = True
                        del g
            finally:
                st.clear()
                self.engine.flush()
            return
        self._mode = _UPDATE
        try:
            with torch.no_grad():
                self._replay_buckets(st)
        finally:
            self._mode = 0
            st.clear()
            self.engine.flush()

    def _replay_buckets(self, st) -> None:
        for b in reversed(self.buckets):
            b.reduced = False
            b.filled = [False] * len(b.params)
            got = False
            for j, p in enumerate(b.params):
                pid, off, n = id(p), b.offsets[j], b.numels[j]
                if pid in st.grads:  # not a linear (or a linear autograd handled)
                    st.linear.pop(pid, None)
                    if b.gflat is None:
                        self._new_gflat(b)
                    b.gflat[off:off + n].copy_(st.grads.pop(pid).reshape(-1))
                elif pid in st.linear:
                    a, d = st.linear.pop(pid)
                    if b.gflat is None:
                        self._new_gflat(b)
                    view = b.gflat[off:off + n].view(d.shape[-1], a.shape[-1])
                    torch.mm(d.reshape(-1, d.shape[-1]).t(), a.reshape(-1, a.shape[-1]),
                             out=view)
                    del a, d
                else:
                    continue
                b.filled[j] = True
                got = True
            if got:
                self._reduce(b)
        self._drain()

    def _decide(self) -> None:
        """K3 local partial -> all_gather of {sumsq, overflow} -> K3a on the
        rank-ordered sum (identical on every rank)."""
        part = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.engine.local_partial(part)
        parts = torch.empty(self.world * 2, dtype=torch.float64, device=self.device)
        all_gather_into(parts, part, self.group)
        self.engine.finalize_ranks(parts.view(self.world, 2))

    def _check_loss(self, loss: torch.Tensor) -> torch.Tensor:
        """Sum of the per-rank losses: non-finite on every rank if it is on
        any, so every rank takes the same skip / abort decision."""
        t = loss.detach().float().reshape(1).clone()
        dist.all_reduce(t, group=self.group)
        return t

    def _after_update(self) -> None:
        self._refresh()

    def remove_hooks(self) -> None:
        for b in self.buckets:
            b.wait()  # no refresh gather may outlive the hooks that wait for it
        for h in self._handles:
            h.remove()
        self._handles = []
        for ring in self._rings.values():
            ring.close()  # collective: every rank calls remove_hooks
        self._rings = {}

    def gather_all(self) -> None:
        """Materialise every bucket's full parameters (e.g. for evaluation)."""
        self._refresh()
        for b in self.buckets:
            b.wait()
            b.gather()
