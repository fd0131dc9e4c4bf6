"""Launch K6 (dW GEMM + probe epilogue) a few times per LLaMA-7B linear shape
-- the command the K6 ncu capture under profiles/ was taken from.

    ncu --set full --clock-control none -k regex:device_kernel -s 2 -c 1 \\
        python tools/prof_k6.py 4096 11008
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import _lib  # noqa: E402

out_f, in_f = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 11008)
T, reps = 1024, 3
torch.cuda.set_device(0)
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
dy = (torch.randn(T, out_f, device="cuda") * 0.01).half()
x = torch.randn(T, in_f, device="cuda").half()
g = torch.empty(out_f, in_f, device="cuda", dtype=torch.half)
st = torch.zeros(_lib.state_bytes(1), dtype=torch.uint8, device="cuda")
_lib.check(lib.lomo_state_init(st.data_ptr(), 1, 1024.0, 16, 1.0, 2.0 ** 24, 1.0, 1.0, s), "i")
need = lib.lomo_gemm_probe_workspace(out_f, in_f, T, _lib.F16)
ws = torch.empty(need, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    _lib.check(lib.lomo_gemm_probe(dy.data_ptr(), x.data_ptr(), g.data_ptr(), out_f, in_f, T,
                                   _lib.F16, 0, _lib.USE_SCALE | _lib.DEFER_ROWS, st.data_ptr(),
                                   ws.data_ptr(), need, s), "k6")
torch.cuda.synchronize()
print(f"K6 {out_f}x{in_f}x{T} x{reps}")
