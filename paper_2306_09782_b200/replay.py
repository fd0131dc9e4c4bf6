"""Pass-2 replay for the two-pass protocol (an optional caller-side speedup).

The reference's two-pass step (stabilize.py:180-230) runs a second forward
and a second full backward only to regenerate the gradients that pass 1
already produced (pass 1 leaves parameters untouched, so they are identical).
On B200 the memory is there to avoid most of that work: during pass 1 every
linear layer routed through :func:`linear` keeps its input ``x`` (already
saved by autograd) and its output gradient ``dy`` (~2.8 GB for LLaMA-7B at
seq 1024), and every other parameter (norm scales, embedding) keeps its
gradient.  Pass 2 then recomputes each weight gradient with exactly the
GEMM autograd used in pass 1 (``dy^T x``) and hands it straight to K1 --
no second forward, no input-gradient GEMMs, no elementwise backward.

The update arithmetic is untouched: K1 sees bit-identical gradients to the
ones K2 probed (same kernels, same inputs).  Enabled with
``LOMO(..., replay=True)``; models opt in by calling :func:`linear` instead of
``F.linear`` (``workloads.Llama`` does), or :func:`matmul_in_out` for weights
stored ``[in, out]`` (the reference zoo's layout).

The same backward context also carries the fused-GEMM callbacks, with or
without replay: ``probe`` (K6: the pass-1 probe inside the weight-gradient
GEMM), ``update`` (K5 inside the backward) and ``embed`` (an embedding's
gradient kept as the batch's aggregated rows, :func:`embedding`).  A weight
taken by a callback returns ``None`` to autograd: its gradient never exists.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

_ACTIVE: "ReplayStash | None" = None


class ReplayStash:
    """What the linears' backward consults while a LOMO pass is active.

    ``keep``: stash each linear's (x, dy) for pass-2 replay (``replay=True``);
    without it the object only carries the fused-GEMM callbacks."""

    def __init__(self, keep: bool = True):
        self.keep = keep
        self.linear: dict[int, tuple[torch.Tensor, torch.Tensor]] = {}
        self.grads: dict[int, torch.Tensor] = {}
        self.seen: set[int] = set()     # weights whose linear backward ran this pass
        self.shared: set[int] = set()   # weights that fed more than one linear
        # pass-1 probe fused into the weight-gradient GEMM (K6): called as
        # probe(weight id, w, x, dy) -> bool from the linear's backward (under
        # activation checkpointing the saved `w` is not the Parameter object
        # itself, so the id recorded at forward time names it); True means the
        # gradient was probed on the tensor cores and is not returned to autograd
        self.probe = None
        self.probed: set[int] = set()
        # the update fused into the weight-gradient GEMM inside the backward
        # (K5, single pass or the strict second backward): update(weight id,
        # w, x, dy) -> bool, True when the weight was updated in place
        self.update = None
        self.updated: set[int] = set()
        # row-sparse embedding gradient: embed(weight id, w, ids, dy) -> bool;
        # `rows` keeps (rows, row_ids) per embedding for pass-2 replay
        self.embed = None
        self.embedded: set[int] = set()
        self.rows: dict[int, tuple[torch.Tensor, torch.Tensor]] = {}

    def clear(self):
        self.linear.clear()
        self.grads.clear()
        self.seen.clear()
        self.shared.clear()
        self.probed.clear()
        self.updated.clear()
        self.embedded.clear()
        self.rows.clear()

    def nbytes(self) -> int:
        n = sum(x.numel() * x.element_size() + d.numel() * d.element_size()
                for x, d in self.linear.values())
        return n + sum(g.numel() * g.element_size() for g in self.grads.values())


def weight_grad(x: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
    """dW = dy^T x for y = x W^T (W: [out, in]) -- the one GEMM both passes use."""
    return dy.reshape(-1, dy.shape[-1]).t().mm(x.reshape(-1, x.shape[-1]))


class _StashLinear(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w):
        ctx.save_for_backward(x, w)
        ctx.wid = id(w)
        return F.linear(x, w)

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        dx = dy.matmul(w) if ctx.needs_input_grad[0] else None
        st = _ACTIVE
        dw = None
        if st is not None:
            if ctx.wid in st.seen:
                st.shared.add(ctx.wid)
            st.seen.add(ctx.wid)
            if st.keep:
                st.linear[ctx.wid] = (x, dy)
        if ctx.needs_input_grad[1]:
            # dx above was enqueued first: it reads w before an in-place update
            if st is not None and ctx.wid not in st.shared and st.probe is not None \
                    and st.probe(ctx.wid, w, x, dy):
                st.probed.add(ctx.wid)   # K6 probed dW: nothing for autograd to deliver
            elif st is not None and ctx.wid not in st.shared and st.update is not None \
                    and st.update(ctx.wid, w, x, dy):
                st.updated.add(ctx.wid)  # K5 applied the update: dW never existed
            else:
                dw = weight_grad(x, dy)
        return dx, dw


class _StashLinearIO(torch.autograd.Function):
    """y = x @ W for a weight stored [in, out] (the reference zoo's layout,
    ops.py:58-75).  dW = x^T dy is the same GEMM as the [out, in] case with
    the operands' roles swapped, so stash and callbacks receive (dy, x) in
    place of (x, dy): ``weight_grad(dy, x)`` = x^T dy, and the fused kernels'
    out x in problem is W's own [in, out] shape."""

    @staticmethod
    def forward(ctx, x, w):
        ctx.save_for_backward(x, w)
        ctx.wid = id(w)
        return x.matmul(w)

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        dx = dy.matmul(w.t()) if ctx.needs_input_grad[0] else None
        st = _ACTIVE
        dw = None
        if st is not None:
            if ctx.wid in st.seen:
                st.shared.add(ctx.wid)
            st.seen.add(ctx.wid)
            if st.keep:
                st.linear[ctx.wid] = (dy, x)
        if ctx.needs_input_grad[1]:
            if st is not None and ctx.wid not in st.shared and st.probe is not None \
                    and st.probe(ctx.wid, w, dy, x):
                st.probed.add(ctx.wid)
            elif st is not None and ctx.wid not in st.shared and st.update is not None \
                    and st.update(ctx.wid, w, dy, x):
                st.updated.add(ctx.wid)
            else:
                dw = weight_grad(dy, x)
        return dx, dw


def matmul_in_out(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """``x @ w`` for a weight stored [in, out], with the same stash/fused-GEMM
    backward as :func:`linear`."""
    if torch.is_grad_enabled() and w.requires_grad:
        return _StashLinearIO.apply(x, w)
    return x.matmul(w)


class _Embedding(torch.autograd.Function):
    """F.embedding whose backward can hand LOMO the batch's rows instead of
    a dense [V, h] gradient (lomo_rows_aggregate / lomo_fused_update_rows)."""

    @staticmethod
    def forward(ctx, ids, w):
        ctx.save_for_backward(ids)
        ctx.wid = id(w)
        ctx.num = w.shape[0]
        return F.embedding(ids, w)

    @staticmethod
    def backward(ctx, dy):
        (ids,) = ctx.saved_tensors
        st = _ACTIVE
        if st is not None:
            if ctx.wid in st.seen:
                st.shared.add(ctx.wid)
            st.seen.add(ctx.wid)
            if ctx.wid not in st.shared and st.embed is not None \
                    and st.embed(ctx.wid, ids, dy):
                st.embedded.add(ctx.wid)
                return None, None
        return None, torch.ops.aten.embedding_backward(dy, ids, ctx.num, -1, False, False)


def embedding(ids: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """``F.embedding(ids, w)`` whose backward can stay row-sparse under LOMO."""
    if torch.is_grad_enabled() and w.requires_grad:
        return _Embedding.apply(ids, w)
    return F.embedding(ids, w)


def linear(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """``F.linear(x, w)`` whose backward can stash (x, dy) for pass-2 replay."""
    if torch.is_grad_enabled() and w.requires_grad:
        return _StashLinear.apply(x, w)
    return F.linear(x, w)
