"""ctypes binding of the C-ABI in include/lomo_b200.h (liblomo_b200.so).

There is no fallback: if the shared library is missing or a CUDA device is
absent, every compute entry point raises.  The library is built in-tree by
``__graft_entry__.build()`` (nvcc, -gencode arch=compute_100a,code=sm_100a).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NativeError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_native" / "liblomo_b200.so"

# lomo_dtype (include/lomo_b200.h)
F32, F16, BF16, F64 = 0, 1, 2, 3
MATH_F32, MATH_F64 = 0, 1
USE_SCALE, USE_COEF, USE_SKIP, ACCUM_F64, LR_FROM_STATE = 0x1, 0x2, 0x4, 0x8, 0x10
CHAINED = 0x80  # K1: previous launch on the stream is a K1 on other tensors
DEFER_ROWS = 0x20
PROBE_KEEP_GRAD = 0x40
PROBE_BLOCKS_PER_SLOT = 8192
E_ARG, E_SLOT, E_UNSUPPORTED = -1, -2, -3
PEER_MAX, PEER_CHANNELS = 16, 16
PEER_SIGNAL_BYTES = 8 * PEER_CHANNELS * PEER_MAX
# lomo_state.error codes (sticky, surfaced by the step's status read)
STATE_ERRORS = {1: "a probe kernel was given a norm slot outside [0, nslots) (LOMO_E_SLOT)",
                2: "a peer barrier timed out: a rank did not reach the same collective point "
                   "(sharded fused_rs mode)"}
ABI_VERSION = 2

# every symbol the header declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "lomo_abi_version",
    "lomo_state_bytes",
    "lomo_state_init",
    "lomo_begin_step",
    "lomo_read_status",
    "lomo_fused_update",
    "lomo_fused_update_multi",
    "lomo_probe",
    "lomo_probe_multi",
    "lomo_finalize_norm",
    "lomo_scaler_on_clean",
    "lomo_local_norm_partial",
    "lomo_finalize_norm_ranks",
    "lomo_num_sms",
    "lomo_gemm_update",
    "lomo_gemm_update_workspace",
    "lomo_fused_rs_update",
    "lomo_fused_rs_probe",
    "lomo_set_lr",
    "lomo_set_scaler_state",
    "lomo_update_coefs",
    "lomo_gemm_update_dev",
    "lomo_gemm_probe",
    "lomo_gemm_probe_workspace",
    "lomo_probe_rows",
    "lomo_probe_rows_multi",
    "lomo_gemm_probe_finish",
    "lomo_rows_aggregate",
    "lomo_fused_update_rows",
    "lomo_fused_mc_update",
    "lomo_fused_mc_probe",
    "lomo_fused_rs_probe_keep",
    "lomo_fused_mc_probe_keep",
    "lomo_ipc_handle_bytes",
    "lomo_ipc_alloc",
    "lomo_ipc_open",
    "lomo_ipc_close",
    "lomo_ipc_free",
    "lomo_peer_barrier",
    "lomo_peer_barrier_dev",
    "lomo_mc_supported",
    "lomo_mc_create",
    "lomo_mc_import",
    "lomo_mc_add_device",
    "lomo_mc_bind",
    "lomo_mc_free",
    "lomo_mc_barrier",
    "lomo_mc_barrier_dev",
)

# include/lomo_workload.h: the benchmark decoder's fused layers (not the LOMO path)
WL_EXPORTS = (
    "lomo_wl_rmsnorm_fwd",
    "lomo_wl_rmsnorm_bwd",
    "lomo_wl_rmsnorm_partial_rows",
    "lomo_wl_rope",
    "lomo_wl_swiglu_fwd",
    "lomo_wl_swiglu_bwd",
    "lomo_wl_rope_ld",
    "lomo_wl_swiglu_gu_fwd",
    "lomo_wl_swiglu_gu_bwd",
    "lomo_wl_qkv_rope_bwd",
    "lomo_wl_add_rmsnorm_fwd",
    "lomo_wl_rmsnorm_bwd_add",
    "lomo_wl_ce_fwd",
    "lomo_wl_ce_bwd",
)


class LomoStatus(ctypes.Structure):
    """Host mirror of ``lomo_state`` (128 bytes, include/lomo_b200.h)."""

    _fields_ = [
        ("scale", ctypes.c_double),
        ("inv_scale", ctypes.c_double),
        ("min_scale", ctypes.c_double),
        ("max_scale", ctypes.c_double),
        ("clip_coef", ctypes.c_double),
        ("total_norm", ctypes.c_double),
        ("sumsq_total", ctypes.c_double),
        ("max_norm", ctypes.c_double),
        ("growth_interval", ctypes.c_int32),
        ("clean_steps", ctypes.c_int32),
        ("overflow", ctypes.c_int32),
        ("skip", ctypes.c_int32),
        ("underflow", ctypes.c_int32),
        ("nslots", ctypes.c_int32),
        ("steps_applied", ctypes.c_int32),
        ("steps_skipped", ctypes.c_int32),
        ("ticket", ctypes.c_uint32),
        ("has_scaler", ctypes.c_int32),
        ("scale_f32", ctypes.c_float),
        ("error", ctypes.c_int32),
        ("grad_div", ctypes.c_double),
        ("lr", ctypes.c_double),
    ]


assert ctypes.sizeof(LomoStatus) == 128
STATE_HEADER_BYTES = 128
K1_RECORD_BYTES = 32  # the pass-2 record between the header and sumsq[]
SLOTS_OFFSET = STATE_HEADER_BYTES + K1_RECORD_BYTES  # LOMO_STATE_SLOTS_OFFSET
SCALE_F32_OFFSET = LomoStatus.scale_f32.offset

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_dbl = ctypes.c_double
_u32 = ctypes.c_uint

_SIGS = {
    "lomo_abi_version": (_i32, []),
    "lomo_state_bytes": (ctypes.c_size_t, [_i32]),
    "lomo_state_init": (_i32, [_vp, _i32, _dbl, _i32, _dbl, _dbl, _dbl, _dbl, _vp]),
    "lomo_begin_step": (_i32, [_vp, _vp, _i32, _vp]),
    "lomo_read_status": (_i32, [_vp, ctypes.POINTER(LomoStatus), _vp]),
    "lomo_fused_update": (_i32, [_vp, _vp, _i64, _i32, _i32, _dbl, _dbl, _dbl, _u32, _vp, _vp]),
    "lomo_fused_update_multi": (
        _i32, [_vp, _vp, _vp, _i32, _i32, _i32, _dbl, _dbl, _dbl, _u32, _vp, _vp]),
    "lomo_probe": (_i32, [_vp, _i64, _i32, _i32, _u32, _vp, _vp]),
    "lomo_probe_multi": (_i32, [_vp, _vp, _vp, _i32, _i32, _u32, _vp, _vp]),
    "lomo_finalize_norm": (_i32, [_vp, _vp]),
    "lomo_scaler_on_clean": (_i32, [_vp, _vp]),
    "lomo_local_norm_partial": (_i32, [_vp, _vp, _vp]),
    "lomo_finalize_norm_ranks": (_i32, [_vp, _vp, _i32, _vp]),
    "lomo_num_sms": (_i32, []),
    "lomo_gemm_update": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _dbl, _dbl, _vp,
                                ctypes.c_size_t, _vp]),
    "lomo_gemm_update_workspace": (ctypes.c_size_t, [_i64, _i64, _i64, _i32]),
    "lomo_fused_rs_update": (_i32, [_vp, _vp, _i32, _i64, _i64, _i32, _i32, _dbl, _dbl, _dbl,
                                    _u32, _vp, _vp]),
    "lomo_fused_rs_probe": (_i32, [_vp, _i32, _i64, _i64, _i32, _i32, _u32, _vp, _vp]),
    "lomo_set_lr": (_i32, [_vp, _dbl, _vp]),
    "lomo_set_scaler_state": (_i32, [_vp, _dbl, _i32, _i32, _i32, _vp]),
    "lomo_update_coefs": (_i32, [_vp, _dbl, _u32, _vp, _vp]),
    "lomo_gemm_update_dev": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp,
                                    ctypes.c_size_t, _vp]),
    "lomo_gemm_probe": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _u32, _vp, _vp,
                               ctypes.c_size_t, _vp]),
    "lomo_gemm_probe_workspace": (ctypes.c_size_t, [_i64, _i64, _i64, _i32]),
    "lomo_probe_rows": (_i32, [_vp, _i64, _i64, _i64, _i32, _vp, _vp]),
    "lomo_probe_rows_multi": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "lomo_rows_aggregate": (_i32, [_vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp]),
    "lomo_fused_update_rows": (_i32, [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _dbl, _dbl, _dbl,
                                      _u32, _vp, _vp]),
    "lomo_gemm_probe_finish": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "lomo_fused_mc_update": (_i32, [_vp, _vp, _i64, _i32, _i32, _dbl, _dbl, _dbl, _u32, _vp, _vp]),
    "lomo_fused_mc_probe": (_i32, [_vp, _i64, _i32, _i32, _u32, _vp, _vp]),
    "lomo_fused_rs_probe_keep": (_i32, [_vp, _i32, _i64, _i64, _i32, _i32, _u32, _vp, _vp, _vp]),
    "lomo_fused_mc_probe_keep": (_i32, [_vp, _i64, _i32, _i32, _u32, _vp, _vp, _vp]),
    "lomo_ipc_handle_bytes": (ctypes.c_size_t, []),
    "lomo_ipc_alloc": (_i32, [ctypes.c_size_t, ctypes.POINTER(_vp), _vp]),
    "lomo_ipc_open": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "lomo_ipc_close": (_i32, [_vp]),
    "lomo_ipc_free": (_i32, [_vp]),
    "lomo_peer_barrier": (_i32, [_vp, _i32, _i32, _i32, ctypes.c_uint64, _i64, _vp, _vp]),
    "lomo_peer_barrier_dev": (_i32, [_vp, _vp, _i32, _i32, _i32, _i64, _vp, _vp]),
    "lomo_mc_supported": (_i32, [_i32]),
    "lomo_mc_create": (_i32, [_i32, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint64),
                              ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(_i32)]),
    "lomo_mc_import": (_i32, [_i32, _i32, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint64)]),
    "lomo_mc_add_device": (_i32, [ctypes.c_uint64, _i32]),
    "lomo_mc_bind": (_i32, [ctypes.c_uint64, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "lomo_mc_free": (_i32, [ctypes.c_uint64]),
    "lomo_mc_barrier": (_i32, [_vp, _vp, _i32, _i32, ctypes.c_uint64, _i64, _vp, _vp]),
    "lomo_mc_barrier_dev": (_i32, [_vp, _vp, _vp, _i32, _i32, _i64, _vp, _vp]),
    "lomo_wl_rmsnorm_fwd": (_i32, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, ctypes.c_float, _vp]),
    "lomo_wl_rmsnorm_bwd": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp]),
    "lomo_wl_rmsnorm_partial_rows": (_i32, [_i64]),
    "lomo_wl_rope": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32,
                            _vp]),
    "lomo_wl_swiglu_fwd": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "lomo_wl_swiglu_bwd": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "lomo_wl_rope_ld": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _i32,
                               _i32, _i32, _vp]),
    "lomo_wl_swiglu_gu_fwd": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp]),
    "lomo_wl_ce_fwd": (_i32, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp]),
    "lomo_wl_ce_bwd": (_i32, [_vp, _vp, _vp, _vp, ctypes.c_float, _vp, _i64, _i32, _i32, _vp]),
    "lomo_wl_add_rmsnorm_fwd": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32,
                                       ctypes.c_float, _vp]),
    "lomo_wl_rmsnorm_bwd_add": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32,
                                       _vp]),
    "lomo_wl_qkv_rope_bwd": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _i32,
                                    _i32, _i32, _i32, _vp]),
    "lomo_wl_swiglu_gu_bwd": (_i32, [_vp, _vp, _vp, _i64, _i64, _i32, _vp]),
}

_LIB = None


def load() -> ctypes.CDLL:
    """Load liblomo_b200.so once; raise loudly if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("LOMO_B200_LIB", LIB_PATH))
    if not path.exists():
        raise NativeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the fused-update path)"
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.lomo_abi_version() != ABI_VERSION:
        raise NativeError(f"ABI version mismatch: {lib.lomo_abi_version()} != {ABI_VERSION}")
    _LIB = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed with status {rc}")


def state_bytes(nslots: int) -> int:
    # pure arithmetic restated so it works without loading (must equal the C side)
    n = int(nslots)
    return SLOTS_OFFSET + 8 * (n + (n + 1) // 2 + n * PROBE_BLOCKS_PER_SLOT)
