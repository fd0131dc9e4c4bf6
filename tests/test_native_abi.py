"""The C-ABI library loads on a CPU-only host and exports exactly what
include/lomo_b200.h declares (no compute calls without a GPU)."""
import ctypes
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2306_09782_b200 import _lib

HEADER = ROOT / "include" / "lomo_b200.h"
WL_HEADER = ROOT / "include" / "lomo_workload.h"


def _declared(header=None):
    text = "".join(h.read_text() for h in ([header] if header else sorted((ROOT / "include").glob("*.h"))))
    return sorted(set(re.findall(r"^\s*(?:int|size_t)\s+(lomo_\w+)\s*\(", text, re.M)))


def test_header_declarations_match_binding():
    assert _declared(HEADER) == sorted(_lib.EXPORTS)
    assert _declared(WL_HEADER) == sorted(_lib.WL_EXPORTS)
    assert _declared() == sorted(_lib.EXPORTS + _lib.WL_EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lomo_\w+)", out))
    assert set(_declared()) <= exported


def test_abi_version_and_state_size():
    lib = _lib.load()
    assert lib.lomo_abi_version() == _lib.ABI_VERSION
    for n in (0, 1, 291, 5000):
        assert lib.lomo_state_bytes(n) == _lib.state_bytes(n)


def test_argument_errors_need_no_gpu():
    lib = _lib.load()
    assert lib.lomo_fused_update(None, None, -1, 1, 0, 0.1, 0.0, 0.0, 0, None, None) == -1
    assert lib.lomo_fused_update(None, None, 0, 1, 0, 0.1, 0.0, 0.0, 0, None, None) == 0
    assert lib.lomo_fused_update(None, None, 5, 1, 0, 0.1, 0.0, 0.0, 0, None, None) == -1
    # state-dependent flags without a state
    assert lib.lomo_fused_update(1, 1, 5, 1, 0, 0.1, 0.0, 0.0, _lib.USE_SKIP, None, None) == -1
    assert lib.lomo_probe(None, 10, 1, 0, 0, None, None) == -1
    assert lib.lomo_probe(None, 10, 1, -1, 0, 1, None) == -2
    assert lib.lomo_finalize_norm(None, None) == -1
    assert lib.lomo_state_init(None, 1, 1.0, 1, 1.0, 1.0, 0.0, 1.0, None) == -1
    assert lib.lomo_finalize_norm_ranks(1, None, 2, None) == -1
    # workload layers: shape / dtype / alignment checks happen before any launch
    assert lib.lomo_wl_rmsnorm_fwd(16, 16, 16, 16, 4, 12, 1, 1e-6, None) == -1      # h % 8
    assert lib.lomo_wl_rmsnorm_fwd(16, 16, 16, 16, 4, 16384, 1, 1e-6, None) == -1   # h > 8192
    assert lib.lomo_wl_rmsnorm_fwd(None, None, None, None, 0, 4096, 1, 1e-6, None) == 0
    assert lib.lomo_wl_rope(16, 16, 16, 16, 16, 16, 2, 2, 1, 24, 1, 0, None) == -1  # dh % 16
    assert lib.lomo_wl_rope(16, 16, 16, 32, 16, 16, 2, 2, 1, 32, 1, 0, None) == -1  # q aliases qo
    assert lib.lomo_wl_swiglu_fwd(16, 16, 16, 12, 1, None) == -1
    assert lib.lomo_wl_swiglu_fwd(16, 16, 16, 16, 0, None) == -1                    # f32 storage
    assert lib.lomo_wl_swiglu_bwd(8, 16, 16, 16, 16, 16, 1, None) == -1             # misaligned
    assert lib.lomo_wl_rmsnorm_partial_rows(1024) == 256
    assert lib.lomo_wl_rmsnorm_partial_rows(0) == 0
    # K6 and its reductions, the row-sparse embedding forms
    assert lib.lomo_gemm_probe(None, None, None, 64, 64, 64, _lib.BF16, 0, 0, None, None, 0,
                               None) == -1
    assert lib.lomo_gemm_probe(16, 16, 16, 64, 64, 64, _lib.BF16, -1, 0, 16, 16, 1 << 20,
                               None) == -2                                          # slot
    assert lib.lomo_gemm_probe(16, 16, 16, 64, 64, 64, _lib.BF16, 0, _lib.ACCUM_F64, 16, 16,
                               1 << 20, None) == -1                                 # f64 mode
    assert lib.lomo_gemm_probe_workspace(0, 64, 64, _lib.BF16) == 0
    assert lib.lomo_gemm_probe_finish(None, None, None, None, 0, _lib.BF16, 16, None) == 0
    assert lib.lomo_gemm_probe_finish(None, None, None, None, 1, _lib.BF16, 16, None) == -1
    assert lib.lomo_probe_rows(16, 0, 8, 8, 0, 16, None) == -1                      # rows < 1
    assert lib.lomo_probe_rows(16, 2, 4, 8, 0, 16, None) == -1                      # ld < cols
    assert lib.lomo_probe_rows(16, 2, 8, 8, -1, 16, None) == -2
    assert lib.lomo_probe_rows_multi(None, None, None, None, None, 0, 16, None) == 0
    assert lib.lomo_rows_aggregate(None, None, None, 0, 8, _lib.BF16, None, None, None) == 0
    assert lib.lomo_rows_aggregate(None, None, None, 4, 8, _lib.BF16, None, None, None) == -1
    assert lib.lomo_fused_update_rows(16, 16, 16, 4, 8, _lib.BF16, 0, 0.1, 0.0, 0.01, 0,
                                      None, None) == -1                             # wd != 0
    assert lib.lomo_fused_update_rows(16, 16, 16, 4, 8, _lib.BF16, 0, 0.1, 0.0, 0.0,
                                      _lib.USE_SKIP, None, None) == -1              # no state


def test_status_struct_layout_matches_c(tmp_path):
    """offsetof() of every lomo_state field, compiled from the header by gcc."""
    fields = [f for f, _ in _lib.LomoStatus._fields_]
    src = tmp_path / "off.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "lomo_b200.h"\n'
                   "int main(void){\n" +
                   "".join(f'printf("{f} %zu\\n", offsetof(lomo_state, {f}));\n' for f in fields) +
                   'printf("sizeof %zu\\n", sizeof(lomo_state));\nreturn 0;}\n')
    exe = tmp_path / "off"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                       text=True).stdout.splitlines())
    for f in fields:
        assert int(got[f]) == getattr(_lib.LomoStatus, f).offset, f
    assert int(got["sizeof"]) == ctypes.sizeof(_lib.LomoStatus) == 128


def test_product_path_has_no_cpu_fallback():
    import torch
    from paper_2306_09782_b200 import LOMO, ConfigError
    m = torch.nn.Linear(4, 4)
    with pytest.raises(ConfigError):
        LOMO(m, lr=0.1)  # CPU parameters: refused, never silently updated on the host


def test_package_does_not_import_the_oracle():
    for p in (ROOT / "paper_2306_09782_b200").rglob("*.py"):
        assert "lomo_oracle" not in p.read_text(), p


def test_cpp_dispatcher_extension_loads():
    """The C++ hook dispatcher (csrc/lomo_dispatch.cpp) is built in-tree next
    to liblomo_b200.so and exposes the HookDispatcher surface (no launches
    without a GPU)."""
    from paper_2306_09782_b200.dispatch import cpp_dispatch
    mod = cpp_dispatch()
    assert mod is not None, "the _lomo_dispatch extension was not built"
    assert mod.abi_version() == _lib.ABI_VERSION
    d = mod.Dispatcher(0, _lib.MATH_F32, 1 << 16)
    d.configure(0.05, 0.0, 0.0, 0)
    assert (d.lr, d.flags, d.launches, d.pending()) == (0.05, 0, 0, 0)
