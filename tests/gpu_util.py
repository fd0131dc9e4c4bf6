"""Helpers shared by the GPU parity tests (device buffers, ulp distance)."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from paper_2306_09782_b200 import _lib

TORCH_DT = {"half": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32,
            "full": torch.float64}
CODE = {torch.float16: _lib.F16, torch.bfloat16: _lib.BF16, torch.float32: _lib.F32,
        torch.float64: _lib.F64}
MATH = {"f32": _lib.MATH_F32, "f64": _lib.MATH_F64}
INT_VIEW = {torch.float16: (torch.int16, -(1 << 15)), torch.bfloat16: (torch.int16, -(1 << 15)),
            torch.float32: (torch.int32, -(1 << 31)), torch.float64: (torch.int64, -(1 << 63))}


def lib():
    return _lib.load()


def stream():
    return torch.cuda.current_stream().cuda_stream


def to_dev(x: np.ndarray, dtype: torch.dtype, offset: int = 0) -> torch.Tensor:
    """Device tensor holding x, starting `offset` elements into its buffer."""
    flat = np.asarray(x, dtype=np.float64).reshape(-1)
    buf = torch.zeros(flat.size + offset + 8, dtype=torch.float64)
    buf[offset:offset + flat.size] = torch.from_numpy(flat)
    # f64 -> dtype: values are already representable (exact cast)
    dev = buf.to(dtype).cuda()
    return dev[offset:offset + flat.size]


def ordered(t: torch.Tensor) -> torch.Tensor:
    it, imin = INT_VIEW[t.dtype]
    i = t.contiguous().view(it).to(torch.int64)
    return torch.where(i < 0, imin - i, i)


def ulp_diff(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Elementwise distance in units of the last place (same dtype)."""
    assert a.dtype == b.dtype
    return (ordered(a) - ordered(b)).abs()


class State:
    """A device lomo_state block driven through the C-ABI."""

    def __init__(self, nslots, scale=0.0, growth=16, min_scale=1.0, max_scale=2.0 ** 24,
                 max_norm=0.0):
        self.buf = torch.zeros(_lib.state_bytes(nslots), dtype=torch.uint8, device="cuda")
        self.ptr = self.buf.data_ptr()
        _lib.check(lib().lomo_state_init(self.ptr, nslots, scale, growth, min_scale, max_scale,
                                         max_norm, 1.0, stream()), "init")

    def status(self) -> _lib.LomoStatus:
        st = _lib.LomoStatus()
        _lib.check(lib().lomo_read_status(self.ptr, st, stream()), "status")
        torch.cuda.synchronize()
        return st

    def write_header(self, **fields):
        """Overwrite header fields from the host (unit tests of K1 flags)."""
        st = self.status()
        for k, v in fields.items():
            setattr(st, k, v)
        raw = bytes(ctypes.string_at(ctypes.addressof(st), ctypes.sizeof(st)))
        self.buf[:128].copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
        # the fp32 kernels read the pass-2 record the state kernels republish
        # from the header; lomo_set_lr (same lr) is one of them
        _lib.check(lib().lomo_set_lr(self.ptr, st.lr, stream()), "lomo_set_lr")
        torch.cuda.synchronize()

    def begin(self, loss: torch.Tensor | None = None):
        if loss is None:
            _lib.check(lib().lomo_begin_step(self.ptr, None, 0, stream()), "begin")
        else:
            _lib.check(lib().lomo_begin_step(self.ptr, loss.data_ptr(), CODE[loss.dtype],
                                             stream()), "begin")

    def probe(self, g: torch.Tensor, slot: int, flags: int):
        _lib.check(lib().lomo_probe(g.data_ptr(), g.numel(), CODE[g.dtype], slot, flags,
                                    self.ptr, stream()), "probe")

    def finalize(self):
        _lib.check(lib().lomo_finalize_norm(self.ptr, stream()), "finalize")

    def on_clean(self):
        _lib.check(lib().lomo_scaler_on_clean(self.ptr, stream()), "on_clean")

    def slots(self, n) -> np.ndarray:
        # K2 leaves per-CTA partials; K3's reduction (local-partial mode, which
        # does not run the decision) folds them into the per-slot sums
        tmp = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.check(lib().lomo_local_norm_partial(self.ptr, tmp.data_ptr(), stream()), "partial")
        torch.cuda.synchronize()
        o = _lib.SLOTS_OFFSET
        return self.buf[o:o + 8 * n].view(torch.float64).cpu().numpy()


def fused_update(p, g, math="f32", lr=0.05, clip=0.0, wd=0.0, flags=0, state=None):
    _lib.check(lib().lomo_fused_update(p.data_ptr(), g.data_ptr(), p.numel(), CODE[p.dtype],
                                       MATH[math], lr, clip, wd, flags,
                                       state.ptr if state is not None else None, stream()),
               "lomo_fused_update")
