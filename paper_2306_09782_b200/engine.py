"""The device side of one optimizer: the lomo_state block plus the hook
dispatcher, behind a small interface shared by LOMO (one GPU) and
ShardedLOMO (ZeRO-3 shards).

Every method only enqueues work on the current CUDA stream except
``read_status`` (the one host sync of a step).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .dispatch import HookDispatcher
from .errors import ConfigError, NativeError, ShapeError

DTYPE_CODE = {
    torch.float32: _lib.F32,
    torch.float16: _lib.F16,
    torch.bfloat16: _lib.BF16,
    torch.float64: _lib.F64,
}
MATH_CODE = {"f32": _lib.MATH_F32, "f64": _lib.MATH_F64}


try:
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover - older torch
    def _raw_stream(idx):
        return torch.cuda.current_stream(idx).cuda_stream


def dtype_code(dtype: torch.dtype) -> int:
    try:
        return DTYPE_CODE[dtype]
    except KeyError:
        raise ConfigError(f"unsupported parameter dtype {dtype}") from None


def apply_update(param: torch.Tensor, grad: torch.Tensor, lr: float, math: str = "f64") -> None:
    """optim.py:52-54 on the device: ``param <- round(param - lr * grad)`` in
    place with one K1 launch on the current stream (``math="f64"``: the
    reference's float64 arithmetic and direct rounding, bit-exact; "f32": the
    fp32 hot path).  Both tensors on one CUDA device, same dtype and shape."""
    if param.device.type != "cuda" or grad.device != param.device:
        raise ConfigError("apply_update needs both tensors on one CUDA device (no CPU path)")
    if grad.shape != param.shape:  # tensor.py:77-78
        raise ShapeError("assign", f"shape {tuple(grad.shape)} != tensor shape {tuple(param.shape)}")
    if grad.dtype != param.dtype or not (param.is_contiguous() and grad.is_contiguous()):
        raise ConfigError("apply_update needs contiguous tensors of one dtype")
    if math not in MATH_CODE:
        raise ConfigError(f"math must be 'f32' or 'f64', got {math!r}")
    idx = param.device.index if param.device.index is not None else torch.cuda.current_device()
    _lib.check(_lib.load().lomo_fused_update(param.data_ptr(), grad.data_ptr(), param.numel(),
                                             dtype_code(param.dtype), MATH_CODE[math],
                                             float(lr), 0.0, 0.0, 0, None, _raw_stream(idx)),
               "lomo_fused_update")


class CudaEngine:
    """State block + K1/K2/K3 launches for one optimizer on one device.

    Args:
        device: the CUDA device holding parameters and gradients.
        nslots: number of norm slots (one per parameter, or per bucket).
        scaler: LossScaler config or None.
        max_norm: global-norm clip threshold or None.
        math: "f32" | "f64".
        grad_div: data-parallel divisor folded into inv_scale (world size).
        overlap: run K1/K2 on a side stream, overlapping the backward GEMMs
            (see HookDispatcher).
    """

    def __init__(self, device: torch.device, nslots: int, scaler=None,
                 max_norm: float | None = None, math: str = "f32", grad_div: float = 1.0,
                 overlap: bool = False):
        if device.type != "cuda":
            raise ConfigError(f"the fused-update path runs on CUDA devices only (got {device}); "
                              "there is no CPU path")
        if math not in MATH_CODE:
            raise ConfigError(f"math must be 'f32' or 'f64', got {math!r}")
        self.device = device
        self._dev_idx = device.index if device.index is not None else torch.cuda.current_device()
        self.lib = _lib.load()
        self.math = MATH_CODE[math]
        self.nslots = int(nslots)
        self.has_scaler = scaler is not None
        self.state = torch.zeros(_lib.state_bytes(self.nslots), dtype=torch.uint8, device=device)
        self.ptr = self.state.data_ptr()
        off = _lib.SCALE_F32_OFFSET
        self.scale_view = self.state[off:off + 4].view(torch.float32).view(())
        # the status block lands in pinned host memory: the read is one DMA,
        # not a staged pageable copy, on the step's one host round trip
        self._status_buf = torch.empty(ctypes.sizeof(_lib.LomoStatus), dtype=torch.uint8,
                                       pin_memory=True)
        self.status = _lib.LomoStatus.from_address(self._status_buf.data_ptr())
        with torch.cuda.device(device):
            _lib.check(self.lib.lomo_state_init(
                self.ptr, self.nslots,
                float(scaler.scale) if scaler else 0.0,
                int(scaler.growth_interval) if scaler else 1,
                float(scaler.min_scale) if scaler else 1.0,
                float(scaler.max_scale) if scaler else 1.0,
                float(max_norm) if max_norm else 0.0, float(grad_div), self.stream()),
                "lomo_state_init")
            clean = int(getattr(scaler, "clean_steps", 0) or 0) if scaler else 0
            if clean:
                # a scaler handed over mid-count continues it, as the
                # reference's live object does (stabilize.py:123-127); K3b
                # republishes nothing for clean_steps, so a plain header write
                off = _lib.LomoStatus.clean_steps.offset
                self.state[off:off + 4].copy_(
                    torch.tensor([clean], dtype=torch.int32).view(torch.uint8))
        side = torch.cuda.Stream(device) if overlap else None
        self.dispatch = HookDispatcher(self.lib, self.ptr, self.math, side_stream=side)

    def stream(self) -> int:
        # raw cudaStream_t of the current stream, without building a Stream object
        return _raw_stream(self._dev_idx)

    # -- step protocol --------------------------------------------------------
    def begin(self, loss: torch.Tensor | None) -> None:
        if loss is None:
            _lib.check(self.lib.lomo_begin_step(self.ptr, None, 0, self.stream()), "begin")
            return
        lt = loss.detach()
        if lt.numel() != 1:
            raise ShapeError("backward", f"loss must be a scalar, got {tuple(lt.shape)}")
        lt = lt.contiguous()
        self._loss_keep = lt  # alive until the kernel has read it (stream order)
        _lib.check(self.lib.lomo_begin_step(self.ptr, lt.data_ptr(), dtype_code(lt.dtype),
                                            self.stream()), "lomo_begin_step")

    def configure(self, lr: float = 0.0, clip: float = 0.0, wd: float = 0.0, flags: int = 0,
                  chain: bool = False):
        self.dispatch.configure(lr, clip, wd, flags, chain)

    def chain_updates(self) -> None:
        """The next updates are issued back to back (a pass over kept or
        replayed gradients): chain their K1 launches (LOMO_CHAINED)."""
        d = self.dispatch
        d.configure(d.lr, d.clip, d.wd, d.flags, True)

    def probe(self, g: torch.Tensor, slot: int) -> None:
        self.dispatch.probe(g, DTYPE_CODE[g.dtype], slot, self.stream())

    def update(self, p: torch.Tensor, g: torch.Tensor) -> None:
        self.dispatch.update(p, g, DTYPE_CODE[p.dtype], self.stream())

    def flush(self) -> None:
        self.dispatch.flush(self.stream())

    # K4: reduce-scatter fused with the update / probe (sharded mode)
    def rs_update(self, p_shard: torch.Tensor, peers_dev: int, world: int, offset: int) -> None:
        d = self.dispatch
        _lib.check(self.lib.lomo_fused_rs_update(
            p_shard.data_ptr(), peers_dev, world, offset, p_shard.numel(), DTYPE_CODE[p_shard.dtype],
            self.math, d.lr, d.clip, d.wd, d.flags, self.ptr, self.stream()), "lomo_fused_rs_update")

    def rs_probe(self, peers_dev: int, world: int, offset: int, n: int, dtype: torch.dtype,
                 slot: int, out: torch.Tensor | None = None) -> None:
        """K4 probe; ``out``: also keep the reduced slice (lomo_fused_rs_probe_keep)."""
        d = self.dispatch
        if out is not None:
            _lib.check(self.lib.lomo_fused_rs_probe_keep(
                peers_dev, world, offset, n, DTYPE_CODE[dtype], slot, d.flags, self.ptr,
                out.data_ptr(), self.stream()), "lomo_fused_rs_probe_keep")
            return
        _lib.check(self.lib.lomo_fused_rs_probe(peers_dev, world, offset, n, DTYPE_CODE[dtype],
                                                slot, d.flags, self.ptr, self.stream()),
                   "lomo_fused_rs_probe")

    # K4, NVLS form: `mc` = this rank's slice of the bucket at the multicast address
    def mc_update(self, p_shard: torch.Tensor, mc: int) -> None:
        d = self.dispatch
        _lib.check(self.lib.lomo_fused_mc_update(
            p_shard.data_ptr(), mc, p_shard.numel(), DTYPE_CODE[p_shard.dtype], self.math, d.lr,
            d.clip, d.wd, d.flags, self.ptr, self.stream()), "lomo_fused_mc_update")

    def mc_probe(self, mc: int, n: int, dtype: torch.dtype, slot: int,
                 out: torch.Tensor | None = None) -> None:
        d = self.dispatch
        if out is not None:
            _lib.check(self.lib.lomo_fused_mc_probe_keep(mc, n, DTYPE_CODE[dtype], slot, d.flags,
                                                         self.ptr, out.data_ptr(), self.stream()),
                       "lomo_fused_mc_probe_keep")
            return
        _lib.check(self.lib.lomo_fused_mc_probe(mc, n, DTYPE_CODE[dtype], slot, d.flags, self.ptr,
                                                self.stream()), "lomo_fused_mc_probe")

    def finalize(self) -> None:
        _lib.check(self.lib.lomo_finalize_norm(self.ptr, self.stream()), "lomo_finalize_norm")

    def local_partial(self, out2: torch.Tensor) -> None:
        _lib.check(self.lib.lomo_local_norm_partial(self.ptr, out2.data_ptr(), self.stream()),
                   "lomo_local_norm_partial")

    def finalize_ranks(self, parts: torch.Tensor) -> None:
        _lib.check(self.lib.lomo_finalize_norm_ranks(self.ptr, parts.data_ptr(), parts.shape[0],
                                                     self.stream()), "lomo_finalize_norm_ranks")

    def on_clean(self) -> None:
        _lib.check(self.lib.lomo_scaler_on_clean(self.ptr, self.stream()), "lomo_scaler_on_clean")

    def read_status(self) -> _lib.LomoStatus:
        _lib.check(self.lib.lomo_read_status(self.ptr, self.status, self.stream()),
                   "lomo_read_status")
        torch.cuda.current_stream(self.device).synchronize()
        if self.status.error:
            raise NativeError(_lib.STATE_ERRORS.get(self.status.error,
                                                    f"device error {self.status.error}"))
        return self.status

    @property
    def error_ptr(self) -> int:
        """Device address of the state's sticky ``error`` word (peer barriers
        report a timeout there, so the step's status read surfaces it)."""
        return self.ptr + _lib.LomoStatus.error.offset

    @property
    def launches(self) -> int:
        return self.dispatch.launches
