"""Would fused projections (QKV as one [3h, h] weight, gate+up as one [2f, h])
pay on B200?  Times the three GEMMs of each linear (forward y = x W^T, input
gradient dx = dy W, and the K6 / K5 weight-gradient GEMMs) for the separate
and the fused layouts of one LLaMA-7B layer (tokens = 1024, fp16).

    python tools/proj_fusion.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
T, h, f = 1024, 4096, 11008
dt, code = torch.float16, _lib.F16
state = torch.zeros(_lib.state_bytes(4), dtype=torch.uint8, device="cuda")
_lib.check(lib.lomo_state_init(state.data_ptr(), 4, 1024.0, 16, 1.0, 2.0 ** 24, 1.0, 1.0, s), "i")


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps * 1e3


def linear_costs(out_f, in_f):
    x = torch.randn(T, in_f, device="cuda").to(dt)
    w = (torch.randn(out_f, in_f, device="cuda") * 0.02).to(dt)
    dy = (torch.randn(T, out_f, device="cuda") * 0.01).to(dt)
    y = torch.empty(T, out_f, device="cuda", dtype=dt)
    dx = torch.empty(T, in_f, device="cuda", dtype=dt)
    g = torch.empty(out_f, in_f, device="cuda", dtype=dt)
    n6 = lib.lomo_gemm_probe_workspace(out_f, in_f, T, code)
    ws6 = torch.empty(n6, dtype=torch.uint8, device="cuda")
    n5 = lib.lomo_gemm_update_workspace(out_f, in_f, T, code)
    ws5 = torch.empty(max(n5, 1), dtype=torch.uint8, device="cuda")
    fwd = timeit(lambda: torch.mm(x, w.t(), out=y))
    bwd = timeit(lambda: torch.mm(dy, w, out=dx))
    k6 = timeit(lambda: lib.lomo_gemm_probe(dy.data_ptr(), x.data_ptr(), g.data_ptr(), out_f,
                                            in_f, T, code, 0, _lib.USE_SCALE | _lib.DEFER_ROWS,
                                            state.data_ptr(), ws6.data_ptr(), n6, s))
    k5 = timeit(lambda: lib.lomo_gemm_update(w.data_ptr(), dy.data_ptr(), x.data_ptr(), out_f,
                                             in_f, T, code, -1e-9, 1.0,
                                             ws5.data_ptr() if n5 else None, n5, s))
    return {"fwd": fwd, "dx": bwd, "K6": k6, "K5": k5}


rows = {"q/k/v separate (x3)": (linear_costs(h, h), 3), "qkv fused": (linear_costs(3 * h, h), 1),
        "gate/up separate (x2)": (linear_costs(f, h), 2), "gate_up fused": (linear_costs(2 * f, h), 1)}
print(f"{'':24} {'fwd':>8} {'dx':>8} {'K6':>8} {'K5':>8} {'sum':>8}  (us per layer)")
for name, (r, k) in rows.items():
    v = {a: b * k for a, b in r.items()}
    print(f"{name:24} {v['fwd']:8.1f} {v['dx']:8.1f} {v['K6']:8.1f} {v['K5']:8.1f} "
          f"{sum(v.values()):8.1f}")
