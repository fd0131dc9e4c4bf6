"""Launch K5 (dW GEMM with the LOMO update as epilogue, p updated in place) a
few times for one LLaMA-7B linear shape -- the command the K5 ncu capture under
profiles/ was taken from.

    ncu --set full --clock-control none -k regex:device_kernel -s 2 -c 1 \\
        python tools/prof_k5.py 4096 11008
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
p = (torch.randn(out_f, in_f, device="cuda") * 0.02).half()
need = lib.lomo_gemm_update_workspace(out_f, in_f, T, _lib.F16)
ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    _lib.check(lib.lomo_gemm_update(p.data_ptr(), dy.data_ptr(), x.data_ptr(), out_f, in_f, T,
                                    _lib.F16, -1e-3, 1.0, ws.data_ptr(), need, s), "k5")
torch.cuda.synchronize()
print(f"K5 {out_f}x{in_f}x{T} x{reps}")
