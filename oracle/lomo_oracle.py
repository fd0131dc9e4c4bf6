"""CPU oracle for the LOMO fused-update path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference's hot path
(/root/reference/pkg/src/fusedtrain, a CPU/numpy package).  It is the
*checker*: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs may import it.  The product path
(``paper_2306_09782_b200``) never calls it and has no CPU fallback.

Parity is pinned: ``tests/golden/make_golden.py`` imports the reference
itself (in the build container, where /root/reference exists) and records
its outputs as fixtures; ``tests/test_oracle.py`` checks every function
below against those fixtures (and against the live reference when present).

Restated functions (reference file:line):

* ``round_through_half``      tensor.py:30-38   (f64 -> binary16 RNE, overflow to inf)
* ``round_direct``            bit-level RNE to any IEEE binary format; for
                              binary16 it equals tests/oracles.py:115-133
* ``round_through_bf16``      this framework's bf16 rule (the reference has no
                              bf16): direct RNE f64 -> bfloat16, overflow to inf
* ``apply_update``            optim.py:52-54 + Tensor.assign tensor.py:74-81
* ``clip_by_value``           stabilize.py:82-86 (np.clip: NaN propagates)
* ``value_clip_update``       stabilize.py:165-171 (single-pass hook)
* ``probe``                   stabilize.py:190-200 (pass-1 hook: overflow + sumsq)
* ``norm_decision``           stabilize.py:201-213
* ``update_hook``             stabilize.py:215-224 (pass-2 hook)
* ``LossScaler``              stabilize.py:94-127
* ``two_pass_step``           stabilize.py:180-230 over pre-computed gradients
* ``grouped_step``            stabilize.py:234-274 (single-pass grouped clipping)
* ``update_pass_threads``     the CPU baseline: apply_update over many tensors
                              on all host cores (numpy releases the GIL)
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

FULL = "full"   # float64 storage (tensor.py:19-21 Precision.FULL)
HALF = "half"   # binary16 emulation (Precision.HALF_EMULATED)
BF16 = "bf16"   # bfloat16 (new in this framework)
F32 = "f32"     # float32 storage (the B200 fp32 path)

HALF_MAX = 65504.0  # tensor.py:27


def round_through_half(values) -> np.ndarray:
    """tensor.py:30-38: numpy's float64->float16 cast (RNE, overflow to inf)."""
    with np.errstate(over="ignore"):
        return np.asarray(values, dtype=np.float64).astype(np.float16).astype(np.float64)


def round_direct(values, mant_bits: int, emin: int, emax: int) -> np.ndarray:
    """Round float64 directly (single rounding, ties-to-even) to a binary
    format with ``mant_bits`` fraction bits and normal exponents [emin, emax];
    subnormals keep the fixed quantum 2**(emin-mant_bits); results at or above
    2**(emax+1) become inf.  NaN/inf pass through."""
    x = np.asarray(values, dtype=np.float64)
    a = np.abs(x)
    with np.errstate(invalid="ignore", over="ignore"):
        _, e = np.frexp(a)
        exp = np.maximum(e.astype(np.int64) - 1, emin)
        q = np.ldexp(1.0, (exp - mant_bits).astype(np.int64))
        r = np.rint(a / q) * q          # a/q is exact (power-of-two scaling)
        r = np.where(r >= 2.0 ** (emax + 1), np.inf, r)
        out = np.copysign(r, x)
    return np.where(np.isfinite(x), out, x)


def round_through_bf16(values) -> np.ndarray:
    """f64 -> bfloat16 -> f64, one RNE rounding (8-bit exponent, 7-bit fraction)."""
    return round_direct(values, 7, -126, 127)


def round_to(values, precision: str) -> np.ndarray:
    """The write-back rounding of Tensor.assign for each storage precision."""
    if precision == FULL:
        return np.asarray(values, dtype=np.float64)
    if precision == HALF:
        return round_through_half(values)
    if precision == BF16:
        return round_through_bf16(values)
    if precision == F32:
        return np.asarray(values, dtype=np.float64).astype(np.float32).astype(np.float64)
    raise ValueError(precision)


# --- hook bodies -------------------------------------------------------------

def apply_update(p: np.ndarray, g: np.ndarray, lr: float, precision: str) -> np.ndarray:
    """optim.py:52-54: p <- round(p - lr * g), arithmetic in float64."""
    p = np.asarray(p, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    if p.shape != g.shape:
        raise ValueError(f"assign shape {g.shape} != tensor shape {p.shape}")  # tensor.py:77-78
    with np.errstate(over="ignore", invalid="ignore"):
        return round_to(p - lr * g, precision)


def clip_by_value(g: np.ndarray, threshold: float) -> np.ndarray:
    """stabilize.py:82-86."""
    if threshold <= 0:
        raise ValueError(f"clip threshold must be positive, got {threshold}")
    return np.clip(g, -threshold, threshold)


def value_clip_update(p, g, lr, threshold, precision):
    """Single-pass hook of Stabilizer._single_pass_step (stabilize.py:165-171)."""
    g = np.asarray(g, dtype=np.float64)
    if threshold is not None:
        g = np.clip(g, -threshold, threshold)
    return apply_update(p, g, lr, precision)


def probe(grads, scale: float, norm_clip: bool) -> tuple[bool, float]:
    """probe_hook over grads in delivery order (stabilize.py:190-200)."""
    overflow, sq = False, 0.0
    for g in grads:
        g = np.asarray(g, dtype=np.float64)
        if not np.all(np.isfinite(g)):
            overflow = True
        elif norm_clip:
            u = (g / scale).ravel()
            sq += float(np.dot(u, u))
    return overflow, sq


def norm_decision(sq_norm: float, max_norm: float | None) -> tuple[bool, float, float]:
    """stabilize.py:204-213 after a clean probe: (skip, norm_scale, total_norm)."""
    if max_norm is None:
        return False, 1.0, math.sqrt(sq_norm)
    total = math.sqrt(sq_norm)
    if not math.isfinite(total):
        return True, 1.0, total
    coef = min(1.0, max_norm / total) if total > 0.0 else 1.0
    return False, coef, total


def update_hook(p, g_scaled, lr, scale, threshold, norm_scale, precision):
    """Pass-2 hook (stabilize.py:217-224): unscale, clip, *norm_scale, update."""
    g = np.asarray(g_scaled, dtype=np.float64) / scale
    if threshold is not None:
        g = np.clip(g, -threshold, threshold)
    if norm_scale is not None:
        g = g * norm_scale
    return apply_update(p, g, lr, precision)


class LossScaler:
    """stabilize.py:94-127 (validation omitted: configs come from the tests)."""

    def __init__(self, scale=2.0 ** 10, growth_interval=16, min_scale=1.0, max_scale=2.0 ** 24):
        self.scale = float(scale)
        self.growth_interval = int(growth_interval)
        self.min_scale = float(min_scale)
        self.max_scale = float(max_scale)
        self.clean_steps = 0

    def on_overflow(self) -> bool:
        """Returns False (and leaves the scale) on underflow (ScaleUnderflowError)."""
        if self.scale / 2.0 < self.min_scale:
            return False
        self.scale /= 2.0
        self.clean_steps = 0
        return True

    def on_clean(self) -> None:
        self.clean_steps += 1
        if self.clean_steps >= self.growth_interval:
            self.scale = min(self.scale * 2.0, self.max_scale)
            self.clean_steps = 0


def two_pass_step(params, grads_unscaled, lr, precision, scaler: LossScaler | None,
                  max_norm: float | None, threshold: float | None = None):
    """Stabilizer._two_pass_step over fixed per-parameter gradients
    (stabilize.py:180-230).  ``params``/``grads_unscaled`` are in build
    (registration) order; ``grads_unscaled`` are dL/dp; the delivered
    gradient is round(g * scale) (tape.py:346,377 round through the storage
    precision).  Returns (new_params, outcome, total_norm, norm_scale);
    outcome is "applied", "skipped" or "underflow"."""
    scale = scaler.scale if scaler is not None else 1.0
    delivered = [round_to(np.asarray(g, dtype=np.float64) * scale, precision)
                 for g in grads_unscaled]
    # the reference tape delivers in non-increasing layer order, i.e. reverse
    # build order (tape.py:350-360); the sum of squares follows it (:199)
    overflow, sq = probe(delivered[::-1], scale, max_norm is not None)
    if overflow:
        if scaler is not None and not scaler.on_overflow():
            return list(params), "underflow", float("nan"), 1.0
        return list(params), "skipped", float("nan"), 1.0
    skip, coef, total = norm_decision(sq, max_norm)
    if skip:
        if scaler is not None and not scaler.on_overflow():
            return list(params), "underflow", total, 1.0
        return list(params), "skipped", total, 1.0
    out = [update_hook(p, g, lr, scale, threshold, coef if max_norm is not None else None,
                       precision) for p, g in zip(params, delivered)]
    if scaler is not None:
        scaler.on_clean()
    return out, "applied", total, coef


def grouped_step(params, grads, layers, lr, precision, max_norm, window):
    """Stabilizer._grouped_step (stabilize.py:234-274): one pass; gradients are
    retained per window of ``window`` adjacent layers (group = layer // window,
    tape delivery order = reverse build order); each group is clipped by its own
    norm, a group with a non-finite norm is dropped alone.  ``params``,
    ``grads`` and ``layers`` are in build order; grads are delivered rounded to
    the storage precision.  Returns (new_params, outcome)."""
    out = [np.asarray(p, dtype=np.float64) for p in params]
    delivered = [round_to(g, precision) for g in grads]
    skipped = False
    buffered: list[int] = []
    cur = None

    def flush():
        nonlocal skipped
        if not buffered:
            return
        sq = 0.0
        for i in buffered:
            flat = delivered[i].ravel()
            sq += float(np.dot(flat, flat))
        norm = math.sqrt(sq)
        if not math.isfinite(norm):
            skipped = True
        else:
            factor = min(1.0, max_norm / norm) if norm > 0.0 else 1.0
            for i in buffered:
                out[i] = apply_update(out[i], delivered[i] * factor, lr, precision)
        buffered.clear()

    for i in reversed(range(len(params))):
        group = layers[i] // window
        if cur is not None and group != cur:
            flush()
        cur = group
        buffered.append(i)
    flush()
    return out, ("skipped" if skipped else "applied")


# --- CPU baseline --------------------------------------------------------------

def update_pass_threads(params, grads, lr, precision, threads: int | None = None,
                        chunk: int = 1 << 20) -> None:
    """apply_update over many tensors in place, on all host cores.

    Arrays are float64 like the reference's Tensor buffers (tensor.py:46-55);
    work is split in ``chunk``-element slices of every tensor and run on a
    thread pool (numpy ufuncs and casts release the GIL).
    """
    threads = threads or os.cpu_count() or 1
    jobs = []
    for p, g in zip(params, grads):
        fp, fg = p.reshape(-1), g.reshape(-1)
        for s in range(0, fp.size, chunk):
            jobs.append((fp[s:s + chunk], fg[s:s + chunk]))

    def run(job):
        pp, gg = job
        pp[...] = apply_update(pp, gg, lr, precision)

    if threads == 1:
        for j in jobs:
            run(j)
        return
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(run, jobs))
