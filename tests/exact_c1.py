"""Exactness harness for config 1 -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's tape semantics for the bundled mini
transformer (fusedtrain/tape.py:286-405, ops.py, zoo.py:150-201) in torch
float64 on the GPU, with the reference's HALF_EMULATED rounding rules:

* every op output is rounded f64 -> binary16 -> f64 directly, RNE, overflow
  to inf (tape.py:286-289, tensor.py:30-38) -- torch's own f64->f16 cast rounds
  twice (through f32), so ``rnd`` restates the direct rounding;
* every VJP output is rounded (tape.py:377); adjoints of values with several
  consumers are summed UNrounded in reverse record order (tape.py:382-385);
* the loss seed ``dout * scale`` is rounded at backward start (tape.py:346);
* parameter gradients are delivered to a hook in the tape's delivery order
  (non-increasing layer, reverse build order; tape.py:350-360).

The hook is the product's: it calls the C-ABI (K2 probe, K3 decide, K1 update
in f64 math) on the fp16 parameter storage, exactly where the reference calls
its hook bodies.  With the ops' arithmetic in float64 on both sides, the end-
to-end fp16 run matches the reference's recorded run element for element
(differences only where a float64 last bit of a contraction's summation
order decides a binary16 rounding).
"""
from __future__ import annotations

import math

import torch

from paper_2306_09782_b200.workloads import (MiniConfig, mini_transformer_init, round_half_np,
                                             sinusoidal_table)

GELU_C = math.sqrt(2.0 / math.pi)
GELU_K = 0.044715
EPS = 1e-5


def rnd(x: torch.Tensor) -> torch.Tensor:
    """f64 -> binary16 -> f64 with ONE rounding (RNE), overflow to +-inf."""
    a = x.abs()
    _, e = torch.frexp(a)
    ex = torch.clamp(e.to(torch.int64) - 1, min=-14)
    q = ((ex - 10 + 1023) << 52).view(torch.float64)   # exactly 2**(ex-10), built from bits
    r = torch.round(a / q) * q                      # a/q exact; round = half-to-even
    r = torch.where(r >= 65536.0, torch.full_like(r, math.inf), r)
    out = torch.copysign(r, x)
    return torch.where(torch.isfinite(x), out, x)


class ExactMini:
    """Parameters live in fp16 storage (the product's tensors); compute in f64."""

    def __init__(self, cfg: MiniConfig, device="cuda"):
        self.cfg = cfg
        self.names = []
        self.p16 = {}
        for name, arr in mini_transformer_init(cfg):
            self.names.append(name)
            self.p16[name] = torch.tensor(round_half_np(arr), dtype=torch.float64,
                                          device=device).to(torch.float16)  # exact
        self.device = device

    def P(self, name):
        return self.p16[name].double()

    # ------------------------------------------------------------- forward
    def forward(self, ids: torch.Tensor):
        c = self.cfg
        b, s = ids.shape
        h, nh = c.hidden, c.heads
        dh = h // nh
        S = {"ids": ids}
        table = torch.tensor(sinusoidal_table(s, h), dtype=torch.float64, device=self.device)
        x = rnd(self.P("embedding.weight")[ids] + table)       # embedding, add_pos
        blocks = []
        for l in range(c.layers):
            pre = f"block{l}"
            B = {"x_in": x}
            s1 = self.P(f"{pre}.attn_norm.scale")
            r1 = torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + EPS)
            a = rnd(x / r1 * s1)
            B["a"] = a
            heads = []
            for nm in ("q", "k", "v"):
                y = rnd(torch.einsum("bsi,io->bso", a, self.P(f"{pre}.attn.{nm}_proj")))
                heads.append(y.reshape(b, s, nh, dh).permute(0, 2, 1, 3).contiguous())
            qh, kh, vh = heads
            B["qh"], B["kh"], B["vh"] = qh, kh, vh
            kt = kh.transpose(-1, -2)
            sc0 = rnd(torch.einsum("bhij,bhjk->bhik", qh, kt))
            factor = 1.0 / math.sqrt(dh)
            sc = rnd(sc0 * factor)
            ex = torch.exp(sc - sc.max(dim=-1, keepdim=True).values)
            probs = rnd(ex / ex.sum(dim=-1, keepdim=True))
            B["probs"] = probs
            ctx = rnd(torch.einsum("bhij,bhjk->bhik", probs, vh))
            merged = ctx.permute(0, 2, 1, 3).reshape(b, s, h)
            B["merged"] = merged
            attn = rnd(torch.einsum("bsi,io->bso", merged, self.P(f"{pre}.attn.out_proj")))
            x = rnd(x + attn)
            B["x_mid"] = x
            s2 = self.P(f"{pre}.ffn_norm.scale")
            r2 = torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + EPS)
            yv = rnd(x / r2 * s2)
            B["y"] = yv
            g0 = rnd(torch.einsum("bsi,io->bso", yv, self.P(f"{pre}.ffn.gate_proj")))
            B["g0"] = g0
            t = torch.tanh(GELU_C * (g0 + GELU_K * g0 ** 3))
            g1 = rnd(0.5 * g0 * (1.0 + t))
            B["g1"] = g1
            u = rnd(torch.einsum("bsi,io->bso", yv, self.P(f"{pre}.ffn.up_proj")))
            B["u"] = u
            gated = rnd(g1 * u)
            B["gated"] = gated
            dn = rnd(torch.einsum("bsi,io->bso", gated, self.P(f"{pre}.ffn.down_proj")))
            x = rnd(x + dn)
            blocks.append(B)
        S["blocks"] = blocks
        S["x_f"] = x
        sf = self.P("final_norm.scale")
        rf = torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + EPS)
        xf = rnd(x / rf * sf)
        S["xf"] = xf
        logits = rnd(torch.einsum("bsi,io->bso", xf, self.P("head.weight")))
        S["logits"] = logits
        return logits, S

    @staticmethod
    def loss_and_grad(logits, targets):
        """ops.py:332-352 in float64."""
        m = logits.max(dim=-1, keepdim=True).values
        e = torch.exp(logits - m)
        z = e.sum(dim=-1, keepdim=True)
        logp = logits - m - torch.log(z)
        n = targets.numel()
        idx = targets.unsqueeze(-1)
        loss = -float(torch.gather(logp, -1, idx).sum()) / n
        d = e / z / n
        d.scatter_(-1, idx, torch.gather(d, -1, idx) - 1.0 / n)
        return loss, d

    # ------------------------------------------------------------ backward
    def _rms_vjp(self, x, s, g):
        r = torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + EPS)
        xhat = x / r
        ds = torch.sum(g * xhat, dim=tuple(range(x.dim() - 1)))
        dx = (g * s - xhat * torch.mean(g * s * xhat, dim=-1, keepdim=True)) / r
        return rnd(dx), rnd(ds)

    def backward(self, S, seed, hook):
        """Reverse traversal; ``hook(name, grad_f64_rounded)`` per parameter."""
        c = self.cfg
        b, s = S["ids"].shape
        h, nh = c.hidden, c.heads
        dh = h // nh
        g = rnd(seed)
        # head: matmul(xf, head)
        xf = S["xf"]
        dw = rnd(torch.einsum("bsi,bso->io", xf, g))
        g_xf = rnd(torch.einsum("bso,io->bsi", g, self.P("head.weight")))
        hook("head.weight", dw)   # after the VJP used the old value (tape.py:371-380)
        dx, ds = self._rms_vjp(S["x_f"], self.P("final_norm.scale"), g_xf)
        hook("final_norm.scale", ds)
        adj_x = dx                                    # single consumer
        for l in reversed(range(c.layers)):
            pre = f"block{l}"
            B = S["blocks"][l]
            # x_out = add(x_mid, dn): [g, g]
            g_add = adj_x
            g_dn = rnd(g_add)
            adj_xmid = rnd(g_add)                     # first contribution (record D)
            # dn = matmul(gated, Wd)
            dw = rnd(torch.einsum("bsi,bso->io", B["gated"], g_dn))
            g_gated = rnd(torch.einsum("bso,io->bsi", g_dn, self.P(f"{pre}.ffn.down_proj")))
            hook(f"{pre}.ffn.down_proj", dw)
            # gated = mul(g1, u): [g*u, g*g1]
            g_g1 = rnd(g_gated * B["u"])
            g_u = rnd(g_gated * B["g1"])
            # u = matmul(y, Wu)   (processed before gelu/gate: later record)
            dw = rnd(torch.einsum("bsi,bso->io", B["y"], g_u))
            adj_y = rnd(torch.einsum("bso,io->bsi", g_u, self.P(f"{pre}.ffn.up_proj")))
            hook(f"{pre}.ffn.up_proj", dw)
            # g1 = gelu(g0)
            x0 = B["g0"]
            t = torch.tanh(GELU_C * (x0 + GELU_K * x0 ** 3))
            du = GELU_C * (1.0 + 3.0 * GELU_K * x0 * x0)
            g_g0 = rnd(g_g1 * (0.5 * (1.0 + t) + 0.5 * x0 * (1.0 - t * t) * du))
            # g0 = matmul(y, Wg)
            dw = rnd(torch.einsum("bsi,bso->io", B["y"], g_g0))
            adj_y = adj_y + rnd(torch.einsum("bso,io->bsi", g_g0, self.P(f"{pre}.ffn.gate_proj")))
            hook(f"{pre}.ffn.gate_proj", dw)
            # y = rmsnorm(x_mid, s2)
            dx, ds = self._rms_vjp(B["x_mid"], self.P(f"{pre}.ffn_norm.scale"), adj_y)
            hook(f"{pre}.ffn_norm.scale", ds)
            adj_xmid = adj_xmid + dx
            # x_mid = add(x_in, attn): [g, g]
            g_attn = rnd(adj_xmid)
            adj_xin = rnd(adj_xmid)
            # attn = matmul(merged, Wo)
            dw = rnd(torch.einsum("bsi,bso->io", B["merged"], g_attn))
            g_merged = rnd(torch.einsum("bso,io->bsi", g_attn, self.P(f"{pre}.attn.out_proj")))
            hook(f"{pre}.attn.out_proj", dw)
            g_ctx = g_merged.reshape(b, s, nh, dh).permute(0, 2, 1, 3).contiguous()
            # ctx = bmm(probs, vh)
            g_probs = rnd(torch.einsum("bhik,bhjk->bhij", g_ctx, B["vh"]))
            g_vh = rnd(torch.einsum("bhij,bhik->bhjk", B["probs"], g_ctx))
            # probs = softmax(sc)
            out = B["probs"]
            inner = torch.sum(g_probs * out, dim=-1, keepdim=True)
            g_sc = rnd(out * (g_probs - inner))
            # sc = scale(sc0)
            g_sc0 = rnd(g_sc * (1.0 / math.sqrt(dh)))
            # sc0 = bmm(qh, kt)
            kt = B["kh"].transpose(-1, -2)
            g_qh = rnd(torch.einsum("bhik,bhjk->bhij", g_sc0, kt))
            g_kt = rnd(torch.einsum("bhij,bhik->bhjk", B["qh"], g_sc0))
            g_kh = rnd(g_kt.transpose(-1, -2))
            # v, k, q matmuls (reverse record order: v, k, q)
            adj_a = None
            for nm, gh in (("v", g_vh), ("k", g_kh), ("q", g_qh)):
                gy = rnd(gh.permute(0, 2, 1, 3).reshape(b, s, h))   # split_heads VJP
                dw = rnd(torch.einsum("bsi,bso->io", B["a"], gy))
                ga = rnd(torch.einsum("bso,io->bsi", gy, self.P(f"{pre}.attn.{nm}_proj")))
                hook(f"{pre}.attn.{nm}_proj", dw)
                adj_a = ga if adj_a is None else adj_a + ga
            # a = rmsnorm(x_in, s1)
            dx, ds = self._rms_vjp(B["x_in"], self.P(f"{pre}.attn_norm.scale"), adj_a)
            hook(f"{pre}.attn_norm.scale", ds)
            adj_x = adj_xin + dx
        # x0 = add_pos(emb): [g]; emb = embedding(ids, E): scatter-add
        g_emb = rnd(adj_x)
        table = self.P("embedding.weight")
        dtable = torch.zeros_like(table)
        dtable.index_add_(0, S["ids"].reshape(-1), g_emb.reshape(-1, table.shape[1]))
        hook("embedding.weight", rnd(dtable))
