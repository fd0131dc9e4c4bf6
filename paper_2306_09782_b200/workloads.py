"""Models and synthetic inputs that drive the fused-update path.

The models are the *callers* of the hot path (autograd produces the
gradients the hook consumes); they are plain PyTorch and not part of the
product kernels.

* ``MiniTransformer`` restates the reference's bundled pre-norm decoder
  (fusedtrain/zoo.py:150-201) op for op -- weights stored ``[in, out]`` and
  applied as ``x @ W`` (ops.py:58-75), additive sinusoidal positions
  (ops.py:209-223), RMSNorm ``x / sqrt(mean(x^2) + 1e-5) * s`` (ops.py:228-236),
  no causal mask (zoo.py:173-178), tanh-GELU gate times up (zoo.py:189-193),
  untied head, mean cross entropy (ops.py:332-352) -- so config 1 (C1) can be
  checked against the reference's own run.  ``mini_transformer_init`` draws
  the initial weights with the reference's RNG sequence (zoo.py:150-224,
  ``INIT_RANGE`` zoo.py:26) and ``sequence_copy_batch`` its tokens
  (zoo.py:227-241).
* ``Llama`` is a LLaMA-1 decoder (RMSNorm, rotary, causal SDPA, SwiGLU, untied
  head) with random init, for configs 3-5 (7B/13B/65B).
* ``llama_param_shapes`` lists the 291 (7B) parameter shapes for the
  fused-update microbench (config 2), in registration order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .replay import embedding as rembedding
from .replay import linear as rlinear
from .replay import matmul_in_out as _mm_in_out

INIT_RANGE = 0.08   # zoo.py:26
RMSNORM_EPS = 1e-5  # zoo.py:27


# ---------------------------------------------------------------------------
# C1: the reference's mini transformer
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class MiniConfig:
    layers: int = 2
    hidden: int = 256
    heads: int = 4
    vocab: int = 1024
    seed: int = 0

    @property
    def ffn(self) -> int:
        return 4 * self.hidden  # zoo.py:86-88


def round_half_np(x: np.ndarray) -> np.ndarray:
    """float64 -> binary16 -> float64, RNE, overflow to inf (tensor.py:30-38)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def mini_transformer_init(cfg: MiniConfig) -> list[tuple[str, np.ndarray]]:
    """Initial parameters in build (registration) order, float64 (zoo.py:150-201)."""
    rng = np.random.default_rng(cfg.seed)
    h, f = cfg.hidden, cfg.ffn
    uni = lambda *shape: rng.uniform(-INIT_RANGE, INIT_RANGE, shape)
    out = [("embedding.weight", uni(cfg.vocab, h))]
    for l in range(cfg.layers):
        pre = f"block{l}"
        out.append((f"{pre}.attn_norm.scale", np.ones(h)))
        for name in ("q", "k", "v"):
            out.append((f"{pre}.attn.{name}_proj", uni(h, h)))
        out.append((f"{pre}.attn.out_proj", uni(h, h)))
        out.append((f"{pre}.ffn_norm.scale", np.ones(h)))
        out.append((f"{pre}.ffn.gate_proj", uni(h, f)))
        out.append((f"{pre}.ffn.up_proj", uni(h, f)))
        out.append((f"{pre}.ffn.down_proj", uni(f, h)))
    out.append(("final_norm.scale", np.ones(h)))
    out.append(("head.weight", uni(h, cfg.vocab)))
    return out


def sequence_copy_batch(dataset_seed: int, step: int, batch: int, seq_len: int,
                        vocab: int) -> np.ndarray:
    """Token ids for (dataset_seed, step); targets are the ids (zoo.py:227-241)."""
    rng = np.random.default_rng([dataset_seed, step])
    return rng.integers(0, vocab, (batch, seq_len))


def sinusoidal_table(seq_len: int, width: int) -> np.ndarray:
    """ops.py:209-215."""
    pos = np.arange(seq_len, dtype=np.float64)[:, None]
    idx = np.arange(width, dtype=np.float64)[None, :]
    angle = pos / np.power(10000.0, 2.0 * np.floor(idx / 2.0) / width)
    return np.where(idx % 2 == 0, np.sin(angle), np.cos(angle))


def _op(x: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    """Round an op output to the storage dtype (tape.py:286-289 / :377)."""
    return x if x.dtype == dtype else x.to(dtype)


class MiniTransformer(nn.Module):
    """zoo._build_mini_transformer in torch; every op's output is rounded to
    the parameter dtype, nonlinear ops compute in fp32 (or fp64 for fp64)."""

    def __init__(self, cfg: MiniConfig, dtype: torch.dtype = torch.float32,
                 device: str | torch.device = "cuda",
                 init: list[tuple[str, np.ndarray]] | None = None,
                 fused_linear: bool = False):
        super().__init__()
        self.cfg = cfg
        self.dtype = dtype
        # route every x @ W through replay.matmul_in_out, so LOMO's replay /
        # fused-GEMM paths (K6, K5) apply to the reference's own model
        self._mm = _mm_in_out if fused_linear else torch.matmul
        init = init if init is not None else mini_transformer_init(cfg)
        self._names = []
        for name, arr in init:
            if dtype in (torch.float16,):
                arr = round_half_np(arr)  # Tensor(data, HALF) rounds at build (tensor.py:44-46)
            t = torch.tensor(arr, dtype=torch.float64).to(dtype=dtype, device=device)
            self.register_parameter(name.replace(".", "__"), nn.Parameter(t))
            self._names.append(name)
        self.inner = torch.float64 if dtype == torch.float64 else torch.float32

    def param(self, name: str) -> nn.Parameter:
        return getattr(self, name.replace(".", "__"))

    def named_reference_parameters(self):
        for name in self._names:
            yield name, self.param(name)

    def _rmsnorm(self, x, s):
        xi, si = x.to(self.inner), s.to(self.inner)
        r = torch.sqrt(torch.mean(xi * xi, dim=-1, keepdim=True) + RMSNORM_EPS)
        return _op(xi / r * si, self.dtype)

    def _gelu(self, x):
        xi = x.to(self.inner)
        c = math.sqrt(2.0 / math.pi)
        return _op(0.5 * xi * (1.0 + torch.tanh(c * (xi + 0.044715 * xi ** 3))), self.dtype)

    def forward(self, ids: torch.Tensor) -> torch.Tensor:
        cfg, dt = self.cfg, self.dtype
        b, s = ids.shape
        h, nh = cfg.hidden, cfg.heads
        dh = h // nh
        pos = torch.tensor(sinusoidal_table(s, h), dtype=self.inner, device=ids.device)
        x = F.embedding(ids, self.param("embedding.weight"))
        x = _op(x.to(self.inner) + pos, dt)
        for l in range(cfg.layers):
            pre = f"block{l}"
            a = self._rmsnorm(x, self.param(f"{pre}.attn_norm.scale"))
            heads = []
            for nm in ("q", "k", "v"):
                y = self._mm(a, self.param(f"{pre}.attn.{nm}_proj"))
                heads.append(y.view(b, s, nh, dh).transpose(1, 2))
            q, k, v = heads
            scores = _op((q @ k.transpose(-1, -2)).to(self.inner) * (1.0 / math.sqrt(dh)), dt)
            probs = _op(torch.softmax(scores.to(self.inner), dim=-1), dt)
            ctx = (probs @ v).transpose(1, 2).reshape(b, s, h)
            x = x + self._mm(ctx, self.param(f"{pre}.attn.out_proj"))
            y = self._rmsnorm(x, self.param(f"{pre}.ffn_norm.scale"))
            gated = self._gelu(self._mm(y, self.param(f"{pre}.ffn.gate_proj"))) * \
                self._mm(y, self.param(f"{pre}.ffn.up_proj"))
            x = x + self._mm(gated, self.param(f"{pre}.ffn.down_proj"))
        xf = self._rmsnorm(x, self.param("final_norm.scale"))
        return self._mm(xf, self.param("head.weight"))


def mean_cross_entropy(logits: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
    """Mean per-position CE (ops.py:332-352), computed in >= fp32."""
    inner = torch.float64 if logits.dtype == torch.float64 else torch.float32
    return F.cross_entropy(logits.reshape(-1, logits.shape[-1]).to(inner), targets.reshape(-1))


# ---------------------------------------------------------------------------
# LLaMA-1 shapes (configs 2-5)
# ---------------------------------------------------------------------------
LLAMA = {
    "7b": dict(hidden=4096, layers=32, heads=32, ffn=11008, vocab=32000),
    "13b": dict(hidden=5120, layers=40, heads=40, ffn=13824, vocab=32000),
    "30b": dict(hidden=6656, layers=60, heads=52, ffn=17920, vocab=32000),
    "65b": dict(hidden=8192, layers=80, heads=64, ffn=22016, vocab=32000),
}


def llama_param_shapes(size: str = "7b") -> list[tuple[str, tuple[int, ...]]]:
    """All parameter shapes of LLaMA-``size`` in registration order."""
    c = LLAMA[size]
    h, f, v = c["hidden"], c["ffn"], c["vocab"]
    out = [("embed_tokens.weight", (v, h))]
    for l in range(c["layers"]):
        p = f"layers.{l}"
        out += [(f"{p}.input_layernorm.weight", (h,)),
                (f"{p}.self_attn.q_proj.weight", (h, h)),
                (f"{p}.self_attn.k_proj.weight", (h, h)),
                (f"{p}.self_attn.v_proj.weight", (h, h)),
                (f"{p}.self_attn.o_proj.weight", (h, h)),
                (f"{p}.post_attention_layernorm.weight", (h,)),
                (f"{p}.mlp.gate_proj.weight", (f, h)),
                (f"{p}.mlp.up_proj.weight", (f, h)),
                (f"{p}.mlp.down_proj.weight", (h, f))]
    out += [("norm.weight", (h,)), ("lm_head.weight", (v, h))]
    return out


def llama_param_count(size: str = "7b") -> int:
    return sum(math.prod(s) for _, s in llama_param_shapes(size))


# ---------------------------------------------------------------------------
# Fused layers (csrc/workload_kernels.cu, include/lomo_workload.h): one kernel
# per layer per direction for fp16/bf16 CUDA tensors; other dtypes/devices use
# the eager formulas below (same math, several kernels).  Not the LOMO path.
# ---------------------------------------------------------------------------
_WL_DTYPES = {torch.float16: 1, torch.bfloat16: 2}


def _wl():
    from . import _lib
    return _lib.load()


def _wl_ok(*ts) -> bool:
    return all(t.is_cuda and t.dtype in _WL_DTYPES and t.is_contiguous() for t in ts)


def _wl_call(rc, what):
    if rc != 0:
        from .errors import NativeError
        raise NativeError(f"{what} failed with status {rc}")


def _stream():
    return torch.cuda.current_stream().cuda_stream


class _RMSNormFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, eps):
        h = x.shape[-1]
        rows = x.numel() // h
        y = torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        _wl_call(_wl().lomo_wl_rmsnorm_fwd(x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                           rstd.data_ptr(), rows, h, _WL_DTYPES[x.dtype], eps,
                                           _stream()), "lomo_wl_rmsnorm_fwd")
        ctx.save_for_backward(x, w, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, w, rstd = ctx.saved_tensors
        dy = dy.contiguous()
        h = x.shape[-1]
        rows = x.numel() // h
        lib = _wl()
        dx, dw = torch.empty_like(x), torch.empty_like(w)
        part = torch.empty(lib.lomo_wl_rmsnorm_partial_rows(rows) * h, dtype=torch.float32,
                           device=x.device)
        _wl_call(lib.lomo_wl_rmsnorm_bwd(dy.data_ptr(), x.data_ptr(), w.data_ptr(),
                                         rstd.data_ptr(), dx.data_ptr(), dw.data_ptr(),
                                         part.data_ptr(), rows, h, _WL_DTYPES[x.dtype],
                                         _stream()), "lomo_wl_rmsnorm_bwd")
        return dx, dw, None


class _RopeFn(torch.autograd.Function):
    """q, k: [b, s, heads, dh] contiguous -> rotated copies (same layout)."""

    @staticmethod
    def _run(q, k, cos, sin, direction):
        b, s, nh, dh = q.shape
        qo, ko = torch.empty_like(q), torch.empty_like(k)
        _wl_call(_wl().lomo_wl_rope(q.data_ptr(), k.data_ptr(), qo.data_ptr(), ko.data_ptr(),
                                    cos.data_ptr(), sin.data_ptr(), b * s, s, nh, dh,
                                    _WL_DTYPES[q.dtype], direction, _stream()), "lomo_wl_rope")
        return qo, ko

    @staticmethod
    def forward(ctx, q, k, cos, sin):
        ctx.save_for_backward(cos, sin)
        return _RopeFn._run(q, k, cos, sin, 0)

    @staticmethod
    def backward(ctx, dq, dk):
        cos, sin = ctx.saved_tensors
        dq, dk = _RopeFn._run(dq.contiguous(), dk.contiguous(), cos, sin, 1)
        return dq, dk, None, None


class _SwiGLUFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, u):
        out = torch.empty_like(g)
        _wl_call(_wl().lomo_wl_swiglu_fwd(g.data_ptr(), u.data_ptr(), out.data_ptr(), g.numel(),
                                          _WL_DTYPES[g.dtype], _stream()), "lomo_wl_swiglu_fwd")
        ctx.save_for_backward(g, u)
        return out

    @staticmethod
    def backward(ctx, dout):
        g, u = ctx.saved_tensors
        dout = dout.contiguous()
        dg, du = torch.empty_like(g), torch.empty_like(u)
        _wl_call(_wl().lomo_wl_swiglu_bwd(dout.data_ptr(), g.data_ptr(), u.data_ptr(),
                                          dg.data_ptr(), du.data_ptr(), g.numel(),
                                          _WL_DTYPES[g.dtype], _stream()), "lomo_wl_swiglu_bwd")
        return dg, du


class _QKVRopeFn(torch.autograd.Function):
    """Fused QKV projection [b, s, 3h] -> rotated q, k ([b, s, heads, dh],
    contiguous) and v (a [b, heads, s, dh] view of qkv, as SDPA takes it).  The
    backward assembles d(qkv) in place -- the rotary transpose writes dq/dk
    into their column blocks, dv is copied into its block -- instead of
    autograd's zero-filled slice gradients."""

    @staticmethod
    def forward(ctx, qkv, cos, sin, nh):
        b, s, h3 = qkv.shape
        h = h3 // 3
        dh = h // nh
        qo = torch.empty(b, s, nh, dh, dtype=qkv.dtype, device=qkv.device)
        ko = torch.empty_like(qo)
        _wl_call(_wl().lomo_wl_rope_ld(qkv.data_ptr(), qkv[..., h:].data_ptr(), h3,
                                       qo.data_ptr(), ko.data_ptr(), h, cos.data_ptr(),
                                       sin.data_ptr(), b * s, s, nh, dh, _WL_DTYPES[qkv.dtype],
                                       0, _stream()), "lomo_wl_rope_ld")
        v = qkv[..., 2 * h:].view(b, s, nh, dh).transpose(1, 2)  # strided view: SDPA takes it
        ctx.save_for_backward(cos, sin)
        ctx.dims = (b, s, h, nh, dh)
        return qo, ko, v

    @staticmethod
    def backward(ctx, dq, dk, dv):
        cos, sin = ctx.saved_tensors
        b, s, h, nh, dh = ctx.dims
        dqkv = torch.empty(b, s, 3 * h, dtype=dq.dtype, device=dq.device)
        dq, dk = dq.contiguous(), dk.contiguous()
        if dv.stride(3) != 1:
            dv = dv.contiguous()
        # rotary transpose of dq/dk and the dv copy, all into d(qkv), one launch
        _wl_call(_wl().lomo_wl_qkv_rope_bwd(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                            dv.stride(0), dv.stride(1), dv.stride(2),
                                            dqkv.data_ptr(), cos.data_ptr(), sin.data_ptr(), b,
                                            s, nh, dh, _WL_DTYPES[dq.dtype], _stream()),
                 "lomo_wl_qkv_rope_bwd")
        return dqkv, None, None, None


class _SwiGLUGuFn(torch.autograd.Function):
    """silu(gu[..., :f]) * gu[..., f:] for a fused gate/up projection."""

    @staticmethod
    def forward(ctx, gu):
        f = gu.shape[-1] // 2
        rows = gu.numel() // (2 * f)
        out = torch.empty(*gu.shape[:-1], f, dtype=gu.dtype, device=gu.device)
        _wl_call(_wl().lomo_wl_swiglu_gu_fwd(gu.data_ptr(), out.data_ptr(), rows, f,
                                             _WL_DTYPES[gu.dtype], _stream()),
                 "lomo_wl_swiglu_gu_fwd")
        ctx.save_for_backward(gu)
        return out

    @staticmethod
    def backward(ctx, dout):
        (gu,) = ctx.saved_tensors
        dout = dout.contiguous()
        f = gu.shape[-1] // 2
        dgu = torch.empty_like(gu)
        _wl_call(_wl().lomo_wl_swiglu_gu_bwd(dout.data_ptr(), gu.data_ptr(), dgu.data_ptr(),
                                             gu.numel() // (2 * f), f, _WL_DTYPES[gu.dtype],
                                             _stream()), "lomo_wl_swiglu_gu_bwd")
        return dgu


class _AddRMSNormFn(torch.autograd.Function):
    """(x, r) -> (h = x + r, y = rmsnorm(h) * w): the decoder's residual add and
    the norm after it in one kernel each way.  The backward receives the
    residual stream's gradient dh and the norm output's dy and returns
    round(round(rms_bwd(dy)) + dh) for both x and r -- what autograd would
    sum -- from the same kernel (csrc/workload_kernels.cu)."""

    @staticmethod
    def forward(ctx, x, r, w, eps):
        hdim = x.shape[-1]
        rows = x.numel() // hdim
        h, y = torch.empty_like(x), torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        _wl_call(_wl().lomo_wl_add_rmsnorm_fwd(x.data_ptr(), r.data_ptr(), w.data_ptr(),
                                               h.data_ptr(), y.data_ptr(), rstd.data_ptr(), rows,
                                               hdim, _WL_DTYPES[x.dtype], eps, _stream()),
                 "lomo_wl_add_rmsnorm_fwd")
        ctx.save_for_backward(h, w, rstd)
        return h, y

    @staticmethod
    def backward(ctx, dh, dy):
        h, w, rstd = ctx.saved_tensors
        hdim = h.shape[-1]
        rows = h.numel() // hdim
        if dy is None:
            return dh, dh, None, None
        dy = dy.contiguous()
        lib = _wl()
        dx, dw = torch.empty_like(h), torch.empty_like(w)
        part = torch.empty(lib.lomo_wl_rmsnorm_partial_rows(rows) * hdim, dtype=torch.float32,
                           device=h.device)
        if dh is None:
            _wl_call(lib.lomo_wl_rmsnorm_bwd(dy.data_ptr(), h.data_ptr(), w.data_ptr(),
                                             rstd.data_ptr(), dx.data_ptr(), dw.data_ptr(),
                                             part.data_ptr(), rows, hdim, _WL_DTYPES[h.dtype],
                                             _stream()), "lomo_wl_rmsnorm_bwd")
        else:
            dh = dh.contiguous()
            _wl_call(lib.lomo_wl_rmsnorm_bwd_add(dy.data_ptr(), h.data_ptr(), w.data_ptr(),
                                                 rstd.data_ptr(), dh.data_ptr(), dx.data_ptr(),
                                                 dw.data_ptr(), part.data_ptr(), rows, hdim,
                                                 _WL_DTYPES[h.dtype], _stream()),
                     "lomo_wl_rmsnorm_bwd_add")
        return dx, dx, dw, None


def add_rms_norm(x, r, w, eps=RMSNORM_EPS):
    """(x + r, rmsnorm(x + r) * w); r may be None (no residual pending)."""
    if r is None:
        return x, rms_norm(x, w, eps)
    if _wl_ok(x, r, w) and x.shape[-1] % 8 == 0 and x.shape[-1] <= 8192:
        return _AddRMSNormFn.apply(x, r, w, eps)
    h = x + r
    return h, rms_norm(h, w, eps, fused=False)


class _CrossEntropyFn(torch.autograd.Function):
    """Mean token cross entropy of fp16/bf16 logits in one kernel per
    direction (csrc/workload_kernels.cu): the forward keeps only the per-row
    log-sum-exp; the backward writes dlogits in the logits' dtype, scaled by
    the upstream gradient read on device (it carries the loss scale)."""

    @staticmethod
    def forward(ctx, logits, targets):
        rows, V = logits.shape
        lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
        loss_rows = torch.empty(rows, dtype=torch.float32, device=logits.device)
        _wl_call(_wl().lomo_wl_ce_fwd(logits.data_ptr(), targets.data_ptr(), lse.data_ptr(),
                                      loss_rows.data_ptr(), rows, V, _WL_DTYPES[logits.dtype],
                                      _stream()), "lomo_wl_ce_fwd")
        ctx.save_for_backward(logits, targets, lse)
        return loss_rows.mean()

    @staticmethod
    def backward(ctx, g):
        logits, targets, lse = ctx.saved_tensors
        rows, V = logits.shape
        g = g.detach().to(torch.float32).contiguous()
        dlogits = torch.empty_like(logits)
        _wl_call(_wl().lomo_wl_ce_bwd(logits.data_ptr(), targets.data_ptr(), lse.data_ptr(),
                                      g.data_ptr(), 1.0 / rows, dlogits.data_ptr(), rows, V,
                                      _WL_DTYPES[logits.dtype], _stream()), "lomo_wl_ce_bwd")
        return dlogits, None


def token_cross_entropy(logits, targets):
    """Mean cross entropy over [rows, V] logits (fp32 math)."""
    if _wl_ok(logits, targets.new_empty(0, dtype=logits.dtype)) and logits.dim() == 2 \
            and logits.shape[1] % 8 == 0 and targets.dtype == torch.int64 \
            and targets.is_contiguous():
        return _CrossEntropyFn.apply(logits, targets)
    inner = torch.float64 if logits.dtype == torch.float64 else torch.float32
    return F.cross_entropy(logits.to(inner), targets)


def rms_norm(x, w, eps=RMSNORM_EPS, fused=True):
    if fused and _wl_ok(x, w) and x.shape[-1] % 8 == 0 and x.shape[-1] <= 8192:
        return _RMSNormFn.apply(x, w, eps)
    xf = x.float()
    y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return y.to(x.dtype) * w


def rope_qk(q, k, cos, sin, fused=True):
    """Rotary embedding of q, k in [b, s, heads, dh] layout."""
    if fused and _wl_ok(q, k, cos, sin) and q.shape[-1] % 16 == 0:
        return _RopeFn.apply(q, k, cos, sin)
    c, s_ = cos[:, None, :], sin[:, None, :]       # [s, 1, dh] against [b, s, heads, dh]
    return _rope(q, c, s_), _rope(k, c, s_)


def swiglu(g, u, fused=True):
    if fused and _wl_ok(g, u) and g.numel() % 8 == 0:
        return _SwiGLUFn.apply(g, u)
    return F.silu(g) * u


class RMSNorm(nn.Module):
    def __init__(self, h: int, dtype, device):
        super().__init__()
        self.weight = nn.Parameter(torch.ones(h, dtype=dtype, device=device))
        self.fused = True

    def forward(self, x):
        return rms_norm(x, self.weight, RMSNORM_EPS, self.fused)


def _linear(h_in: int, h_out: int, dtype, device, std: float) -> nn.Parameter:
    w = torch.empty(h_out, h_in, dtype=dtype, device=device)
    w.normal_(0.0, std)
    return nn.Parameter(w)


class LlamaLayer(nn.Module):
    def __init__(self, h, nh, f, dtype, device, std, fused_proj: bool = False):
        super().__init__()
        self.nh = nh
        self.fused_proj = fused_proj
        self.input_layernorm = RMSNorm(h, dtype, device)
        if fused_proj:
            # q, k, v stacked in one [3h, h] weight and gate, up in one [2f, h]:
            # the same parameters and arithmetic, 2 GEMMs instead of 5 per
            # direction (bigger tiles grids, fewer launches; tools/proj_fusion.py)
            self.qkv = _linear(h, 3 * h, dtype, device, std)
        else:
            self.q = _linear(h, h, dtype, device, std)
            self.k = _linear(h, h, dtype, device, std)
            self.v = _linear(h, h, dtype, device, std)
        self.o = _linear(h, h, dtype, device, std)
        self.post_attention_layernorm = RMSNorm(h, dtype, device)
        if fused_proj:
            self.gate_up = _linear(h, 2 * f, dtype, device, std)
        else:
            self.gate = _linear(h, f, dtype, device, std)
            self.up = _linear(h, f, dtype, device, std)
        self.down = _linear(f, h, dtype, device, std)

    def forward_res(self, x, pending, cos, sin):
        """Stacked-projection layer on the residual stream: ``x`` plus the
        previous layer's not-yet-added MLP output ``pending`` (None for the
        first layer) -> (residual stream, this layer's MLP output).  Each
        residual add is fused into the RMSNorm after it."""
        b, s, h = x.shape
        nh, dh = self.nh, h // self.nh
        x, a = add_rms_norm(x, pending, self.input_layernorm.weight)
        qkv = rlinear(a, self.qkv)                                  # [b, s, 3h]
        if _wl_ok(qkv, cos, sin) and dh % 16 == 0:
            q, k, v = _QKVRopeFn.apply(qkv, cos, sin, nh)
        else:
            q, k, v = qkv.split(h, dim=-1)
            q, k = rope_qk(q.reshape(b, s, nh, dh), k.reshape(b, s, nh, dh), cos, sin, False)
            v = v.reshape(b, s, nh, dh).transpose(1, 2)
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v,
                                           is_causal=True)
        x, y = add_rms_norm(x, rlinear(o.transpose(1, 2).reshape(b, s, h), self.o),
                            self.post_attention_layernorm.weight)
        gu = rlinear(y, self.gate_up)                                # [b, s, 2f]
        if _wl_ok(gu) and gu.shape[-1] % 16 == 0:
            m = _SwiGLUGuFn.apply(gu)
        else:
            f = gu.shape[-1] // 2
            m = F.silu(gu[..., :f]) * gu[..., f:]
        return x, rlinear(m, self.down)

    def forward(self, x, cos, sin, pending=None, stream: bool = False):
        """``stream=True`` (stacked projections): the residual-stream form
        ``forward_res`` -> (stream, MLP output).  Llama calls every layer
        through ``Module.__call__`` so per-layer module hooks (ShardedLOMO's
        ZeRO-3 gather / release / refresh wait) fire on both forms."""
        if self.fused_proj:
            x, mlp = self.forward_res(x, pending, cos, sin)
            return (x, mlp) if stream else x + mlp
        b, s, h = x.shape
        nh, dh = self.nh, h // self.nh
        fused = self.input_layernorm.fused
        a = self.input_layernorm(x)
        q = rlinear(a, self.q).view(b, s, nh, dh)
        k = rlinear(a, self.k).view(b, s, nh, dh)
        v = rlinear(a, self.v).view(b, s, nh, dh).transpose(1, 2)
        q, k = rope_qk(q, k, cos, sin, fused)          # rotated in [b, s, heads, dh]
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v,
                                           is_causal=True)
        x = x + rlinear(o.transpose(1, 2).reshape(b, s, h), self.o)
        y = self.post_attention_layernorm(x)
        return x + rlinear(swiglu(rlinear(y, self.gate), rlinear(y, self.up), fused), self.down)


def _rope(x, cos, sin):
    x1, x2 = x.chunk(2, dim=-1)
    return x * cos + torch.cat((-x2, x1), dim=-1) * sin


class Llama(nn.Module):
    """LLaMA-1 decoder, random init N(0, 0.02), parameters in ``dtype``."""

    def __init__(self, size="7b", dtype=torch.float16, device="cuda",
                 checkpointing: bool = False, layers: int | None = None, seed: int = 0,
                 fused_layers: bool = True, fused_proj: bool = False):
        super().__init__()
        c = dict(LLAMA[size]) if isinstance(size, str) else dict(size)
        if layers is not None:
            c["layers"] = layers
        self.cfg = c
        self.checkpointing = checkpointing
        self.fused_proj = fused_proj
        h, f, v, nh = c["hidden"], c["ffn"], c["vocab"], c["heads"]
        if str(device).startswith("cuda"):
            torch.cuda.manual_seed(seed)
        else:
            torch.manual_seed(seed)
        std = 0.02
        self.embed_tokens = nn.Parameter(torch.empty(v, h, dtype=dtype, device=device).normal_(0, std))
        self.layers = nn.ModuleList(LlamaLayer(h, nh, f, dtype, device, std, fused_proj)
                                    for _ in range(c["layers"]))
        self.norm = RMSNorm(h, dtype, device)
        self.lm_head = nn.Parameter(torch.empty(v, h, dtype=dtype, device=device).normal_(0, std))
        self._rope_cache = {}
        for m in self.modules():
            if isinstance(m, RMSNorm):
                m.fused = fused_layers

    def _cos_sin(self, s, device, dtype):
        key = (s, device, dtype)
        if key not in self._rope_cache:
            dh = self.cfg["hidden"] // self.cfg["heads"]
            inv = 1.0 / (10000 ** (torch.arange(0, dh, 2, device=device, dtype=torch.float32) / dh))
            t = torch.arange(s, device=device, dtype=torch.float32)
            fr = torch.outer(t, inv)
            emb = torch.cat((fr, fr), dim=-1)
            self._rope_cache[key] = (emb.cos().to(dtype), emb.sin().to(dtype))
        return self._rope_cache[key]

    def forward(self, ids):
        x = rembedding(ids, self.embed_tokens)
        cos, sin = self._cos_sin(ids.shape[1], ids.device, x.dtype)
        if self.fused_proj:  # residual adds fused into the norms (forward_res)
            pending = None
            for layer in self.layers:
                if self.checkpointing and self.training:
                    x, pending = torch.utils.checkpoint.checkpoint(
                        layer, x, cos, sin, pending, True, use_reentrant=False)
                else:
                    x, pending = layer(x, cos, sin, pending, True)
            _, y = add_rms_norm(x, pending, self.norm.weight)
            return rlinear(y, self.lm_head)
        for layer in self.layers:
            if self.checkpointing and self.training:
                x = torch.utils.checkpoint.checkpoint(layer, x, cos, sin, use_reentrant=False)
            else:
                x = layer(x, cos, sin)
        return rlinear(self.norm(x), self.lm_head)

    def loss(self, ids, targets):
        logits = self(ids)
        return token_cross_entropy(logits.reshape(-1, logits.shape[-1]),
                                   targets.reshape(-1).contiguous())
