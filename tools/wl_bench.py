"""Per-kernel times of the decoder's fused layers at the LLaMA-7B step shapes
(seq 1024, batch 1) against their HBM roofline.  Each op is captured 20x in a
CUDA graph so host launch cost is excluded."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
lib = _lib.load()
T, H, F, NH = 1024, 4096, 11008, 32
dt, code = torch.float16, _lib.F16


def timed(fn, reps=20, iters=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn(s.cuda_stream)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(iters):
        g.replay()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / (reps * iters) * 1e3


def P(t):
    return t.data_ptr()


x = torch.randn(T, H, device="cuda", dtype=dt)
w = torch.ones(H, device="cuda", dtype=dt)
y, dy, dx = torch.empty_like(x), torch.randn_like(x), torch.empty_like(x)
dw = torch.empty_like(w)
rstd = torch.empty(T, device="cuda")
part = torch.empty(lib.lomo_wl_rmsnorm_partial_rows(T) * H, device="cuda")
lib.lomo_wl_rmsnorm_fwd(P(x), P(w), P(y), P(rstd), T, H, code, 1e-5, None)
q = torch.randn(T, NH, H // NH, device="cuda", dtype=dt)
k, qo, ko = torch.randn_like(q), torch.empty_like(q), torch.empty_like(q)
cos, sin = (torch.randn(T, H // NH, device="cuda", dtype=dt) for _ in range(2))
g = torch.randn(T, F, device="cuda", dtype=dt)
u, o, d, dg, du = (torch.randn_like(g) for _ in range(5))
rows = [
    ("rmsnorm fwd", lambda s: lib.lomo_wl_rmsnorm_fwd(P(x), P(w), P(y), P(rstd), T, H, code, 1e-5, s),
     2 * T * H * 2),
    ("rmsnorm bwd (+dw reduce)", lambda s: lib.lomo_wl_rmsnorm_bwd(
        P(dy), P(x), P(w), P(rstd), P(dx), P(dw), P(part), T, H, code, s), 3 * T * H * 2),
    ("rope fwd (q and k)", lambda s: lib.lomo_wl_rope(P(q), P(k), P(qo), P(ko), P(cos), P(sin), T, T,
                                                      NH, H // NH, code, 0, s), 4 * T * H * 2),
    ("swiglu fwd", lambda s: lib.lomo_wl_swiglu_fwd(P(g), P(u), P(o), T * F, code, s), 3 * T * F * 2),
    ("swiglu bwd", lambda s: lib.lomo_wl_swiglu_bwd(P(d), P(g), P(u), P(dg), P(du), T * F, code, s),
     5 * T * F * 2),
]
for name, fn, b in rows:
    us = timed(fn)
    print(f"{name:28s} {us:7.2f} us  {b / us / 1e3:7.0f} GB/s")
