"""A CPU stand-in for CudaEngine -- TEST INFRASTRUCTURE ONLY.

It restates K1/K2/K3's semantics with the oracle's float64 arithmetic so the
multi-process (gloo, CPU) tests can exercise ShardedLOMO's host logic --
bucketing, ZeRO-3 gather/release, reduce-scatter, the rank-ordered norm
exchange and the skip agreement -- without a GPU.  The product path never
uses it (ShardedLOMO builds a CudaEngine unless a test injects this).
"""
from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np
import torch

from paper_2306_09782_b200 import _lib


class CpuEngine:
    def __init__(self, nslots, scaler=None, max_norm=None, grad_div=1.0):
        self.math = _lib.MATH_F64
        self.nslots = nslots
        self.has_scaler = scaler is not None
        self.scale = float(scaler.scale) if scaler else 1.0
        self.growth = scaler.growth_interval if scaler else 1
        self.min_scale = scaler.min_scale if scaler else 1.0
        self.max_scale = scaler.max_scale if scaler else 1.0
        self.max_norm = max_norm
        self.grad_div = float(grad_div)
        self.clean = 0
        self.scale_view = torch.tensor(self.scale, dtype=torch.float32)
        self.sumsq = np.zeros(nslots)
        self.overflow = self.skip = self.underflow = False
        self.coef, self.total_norm = 1.0, 0.0
        self.launches = 0
        self.configure()

    @property
    def inv_scale(self):
        return 1.0 / (self.scale * self.grad_div)

    def begin(self, loss):
        self.sumsq[:] = 0.0
        self.overflow = self.skip = not math.isfinite(float(loss.detach().reshape(-1)[0]))
        self.underflow = False
        self.coef = 1.0

    def configure(self, lr=0.0, clip=0.0, wd=0.0, flags=0, chain=False):
        self.lr, self.clip, self.wd, self.flags = lr, clip, wd, flags

    def chain_updates(self):
        pass  # launch chaining has no CPU counterpart

    def probe(self, g, slot):
        x = g.detach().double().numpy()
        if not np.all(np.isfinite(x)):
            self.overflow = True
        if self.flags & _lib.USE_SCALE:
            x = x * self.inv_scale
        self.sumsq[slot] = float(np.dot(x, x)) if np.all(np.isfinite(x)) else float("inf")

    def update(self, p, g):
        if (self.flags & _lib.USE_SKIP) and self.skip:
            return
        x = g.detach().double().numpy()
        if self.flags & _lib.USE_SCALE:
            x = x * self.inv_scale
        if self.clip > 0:
            x = np.clip(x, -self.clip, self.clip)
        if self.flags & _lib.USE_COEF:
            x = x * self.coef
        pv = p.detach().double().numpy()
        if self.wd:
            pv = pv * (1.0 - self.lr * self.wd)
        with torch.no_grad():
            p.copy_(torch.from_numpy(pv - self.lr * x).to(p.dtype))

    def flush(self):
        pass

    def _decide(self, total):
        n = math.sqrt(total) if total >= 0 else float("nan")
        self.total_norm = n
        skip = self.overflow
        coef = 1.0
        if not skip and self.max_norm:
            if not math.isfinite(n):
                skip = True
            elif n > 0:
                coef = min(1.0, self.max_norm / n)
        self.coef, self.skip = coef, skip
        if skip and self.has_scaler:
            if self.scale / 2.0 < self.min_scale:
                self.underflow = True
            else:
                self.scale /= 2.0
                self.clean = 0
        self.scale_view.fill_(self.scale)

    def finalize(self):
        self._decide(float(sum(self.sumsq)))

    def local_partial(self, out2):
        out2[0] = float(sum(self.sumsq))
        out2[1] = 1.0 if self.overflow else 0.0

    def finalize_ranks(self, parts):
        total = 0.0
        for r in range(parts.shape[0]):
            total += float(parts[r, 0])
            self.overflow |= float(parts[r, 1]) != 0.0
        self._decide(total)

    def on_clean(self):
        if self.skip or not self.has_scaler:
            return
        self.clean += 1
        if self.clean >= self.growth:
            self.scale = min(self.scale * 2.0, self.max_scale)
            self.clean = 0
        self.scale_view.fill_(self.scale)

    def read_status(self):
        return SimpleNamespace(scale=self.scale, clean_steps=self.clean,
                               inv_scale=self.inv_scale, skip=int(self.skip),
                               underflow=int(self.underflow),
                               overflow=int(self.overflow), total_norm=self.total_norm,
                               clip_coef=self.coef, min_scale=self.min_scale)
