"""Why is K1 slower inside the training step than in the isolated pass?
Times the LLaMA-7B update pass (events around the whole pass) under
progressively training-like conditions.

    python tools/k1_context.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_09782_b200 import _lib  # noqa: E402
from paper_2306_09782_b200.engine import CudaEngine  # noqa: E402

torch.cuda.set_device(0)
P, G = bench.make_update_workload(0, 1, "fp16")
elems = sum(p.numel() for p in P)
eng = CudaEngine(torch.device("cuda:0"), len(P), None, 1.0, "f32")
s = torch.cuda.current_stream()
A = torch.randn(1024, 11008, device="cuda", dtype=torch.float16)
B = torch.randn(1024, 4096, device="cuda", dtype=torch.float16)
flush_buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")


def run(flags, probe=False, gemm=False, group=9, flush_l2=False):
    eng.begin(None)
    order = list(range(len(P) - 1, -1, -1))
    for g0 in range(0, len(order), group):
        idx = order[g0:g0 + group]
        if gemm:
            torch.mm(A.t(), B)          # a dW-sized GEMM before each group
        if flush_l2:
            flush_buf.add_(1)
        if probe:
            eng.begin(None)
            eng.configure(flags=0)
            for i in idx:
                eng.probe(G[i], i)
            eng.flush()
            eng.finalize()
        eng.configure(0.05, 0.0, 0.0, flags)
        for i in idx:
            eng.update(P[i], G[i])
        eng.flush()


def timed(name, **kw):
    for _ in range(2):
        run(**kw)
    torch.cuda.synchronize()
    # GEMM / probe / flush time measured separately and subtracted
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(5):
        run(**kw)
    e[1].record()
    torch.cuda.synchronize()
    ms = e[0].elapsed_time(e[1]) / 5
    return name, ms


res = [timed("plain K1 pass (fp16, no flags)", flags=0, group=1000),
       timed("flags SKIP|COEF", flags=_lib.USE_SKIP | _lib.USE_COEF, group=1000),
       timed("flags, groups of 9 (flush per group)", flags=_lib.USE_SKIP | _lib.USE_COEF),
       timed("K2+K3 then K1 per group", flags=_lib.USE_SKIP | _lib.USE_COEF, probe=True),
       timed("K2 only per group (K1 flags)", flags=_lib.USE_SKIP | _lib.USE_COEF, probe=True),
       timed("GEMM + K1 per group", flags=_lib.USE_SKIP | _lib.USE_COEF, gemm=True),
       timed("L2 flush + K1 per group", flags=_lib.USE_SKIP | _lib.USE_COEF, flush_l2=True)]


# the GEMM and flush alone
def only(kind):
    def f():
        for _ in range(33):
            if kind == "gemm":
                torch.mm(A.t(), B)
            else:
                flush_buf.add_(1)
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(5):
        f()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / 5


tg, tf = only("gemm"), only("flush")
for name, ms in res:
    print(f"{name:45s} {ms:7.3f} ms  ({6 * elems / ms / 1e6:.0f} GB/s if all K1)")
print(f"33 GEMMs alone {tg:.3f} ms; 33 L2 flushes alone {tf:.3f} ms")
