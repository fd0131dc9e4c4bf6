"""Per-shape timing of the weight-gradient GEMM family on the LLaMA-7B linears
(tokens = 1024): cuBLAS dW (what autograd runs), cuBLAS dW + K2, K6 (dW GEMM
with the probe epilogue) and K5 (dW GEMM with the update epilogue).

    python tools/gemm_shapes.py [--tokens 1024] [--reps 20]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=1024)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--fused", action="store_true", help="the stacked-projection shapes (qkv, gate_up)")
a = ap.parse_args()
torch.cuda.set_device(0)
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
dt = torch.float16
code = _lib.F16
T = a.tokens
# (out, in, count per 7B model)
shapes = [(4096, 4096, 128), (11008, 4096, 64), (4096, 11008, 32), (32000, 4096, 1)]
if a.fused:
    shapes = [(12288, 4096, 32), (4096, 4096, 32), (22016, 4096, 32), (4096, 11008, 32),
              (32000, 4096, 1)]
state = torch.zeros(_lib.state_bytes(4), dtype=torch.uint8, device="cuda")
_lib.check(lib.lomo_state_init(state.data_ptr(), 4, 1024.0, 16, 1.0, 2.0 ** 24, 1.0, 1.0, s),
           "init")


def timeit(fn):
    for _ in range(3):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / a.reps * 1e3


tot = {"cublas": 0.0, "cublas+K2": 0.0, "K6": 0.0, "K6 gemm": 0.0, "K5": 0.0}
print(f"{'out x in':>14} {'cuBLAS dW':>10} {'+K2':>8} {'K6':>8} {'K6 gemm':>8} {'K5':>8}"
      "  (us; PF/s of K6 gemm, K5)")
for out_f, in_f, cnt in shapes:
    dy = torch.randn(T, out_f, device="cuda").to(dt) * 0.01
    x = torch.randn(T, in_f, device="cuda").to(dt)
    p = torch.randn(out_f, in_f, device="cuda").to(dt) * 0.02
    g = torch.empty(out_f, in_f, device="cuda", dtype=dt)
    need6 = lib.lomo_gemm_probe_workspace(out_f, in_f, T, code)
    ws6 = torch.empty(need6, dtype=torch.uint8, device="cuda")
    need5 = lib.lomo_gemm_update_workspace(out_f, in_f, T, code)
    ws5 = torch.empty(max(need5, 1), dtype=torch.uint8, device="cuda")

    def cublas():
        torch.mm(dy.t(), x, out=g)

    def cublas_k2():
        torch.mm(dy.t(), x, out=g)
        lib.lomo_probe(g.data_ptr(), g.numel(), code, 0, _lib.USE_SCALE, state.data_ptr(), s)

    def k6():
        lib.lomo_gemm_probe(dy.data_ptr(), x.data_ptr(), g.data_ptr(), out_f, in_f, T, code, 1,
                            _lib.USE_SCALE, state.data_ptr(), ws6.data_ptr(), need6, s)

    def k6_gemm():  # deferred row reduction: the GEMM launch alone
        lib.lomo_gemm_probe(dy.data_ptr(), x.data_ptr(), g.data_ptr(), out_f, in_f, T, code, 1,
                            _lib.USE_SCALE | _lib.DEFER_ROWS, state.data_ptr(), ws6.data_ptr(),
                            need6, s)

    def k5():
        lib.lomo_gemm_update(p.data_ptr(), dy.data_ptr(), x.data_ptr(), out_f, in_f, T, code,
                             -1e-9, 1.0, ws5.data_ptr() if need5 else None, need5, s)

    r = {"cublas": timeit(cublas), "cublas+K2": timeit(cublas_k2), "K6": timeit(k6),
         "K6 gemm": timeit(k6_gemm), "K5": timeit(k5)}
    for k in r:
        tot[k] += r[k] * cnt
    fl = 2.0 * out_f * in_f * T / 1e15
    print(f"{out_f:>6} x {in_f:<6} {r['cublas']:10.1f} {r['cublas+K2']:8.1f} {r['K6']:8.1f} "
          f"{r['K6 gemm']:8.1f} {r['K5']:8.1f}  x{cnt:<3} {fl / (r['K6 gemm'] * 1e-6):.2f} "
          f"{fl / (r['K5'] * 1e-6):.2f}")
print("per 7B pass (ms): " + ", ".join(f"{k} {v / 1e3:.2f}" for k, v in tot.items()))
