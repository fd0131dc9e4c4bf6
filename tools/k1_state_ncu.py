"""K1 flag-free vs K1 reading the step state (the pass-2 form), same shape.

    python tools/k1_state_ncu.py [--ncu]

Without --ncu: times back-to-back launches of each form over 12 LLaMA-7B
MLP-shaped bf16 tensors (4096 x 11008, 1.6 GB of p + g: no L2 reuse) with
CUDA events, PDL on, as the update pass issues them.  Under ncu (--ncu: a
short loop) the launches are serialised, so a difference that survives
there is inside the kernel, one that vanishes is launch overlap.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import _lib  # noqa: E402
from paper_2306_09782_b200.engine import CudaEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--n", type=int, default=12)
ap.add_argument("--shape", type=int, default=4096 * 11008)
args = ap.parse_args()
torch.cuda.set_device(0)
lib = _lib.load()
shape = args.shape
gen = torch.Generator(device="cuda").manual_seed(0)
P = [torch.empty(shape, dtype=torch.bfloat16, device="cuda").uniform_(-0.08, 0.08, generator=gen)
     for _ in range(args.n)]
G = [torch.empty(shape, dtype=torch.bfloat16, device="cuda").normal_(0, 1e-3, generator=gen)
     for _ in range(args.n)]
eng = CudaEngine(torch.device("cuda:0"), 1, None, 1.0, "f32")
_lib.check(lib.lomo_set_lr(eng.ptr, 0.05, eng.stream()), "set_lr")
FLAGS = {"plain": 0,
         "state": _lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE,
         "skip_only": _lib.USE_SKIP}


def run(flags):
    s = eng.stream()
    st = eng.ptr if flags else None
    for p, g in zip(P, G):
        _lib.check(lib.lomo_fused_update(p.data_ptr(), g.data_ptr(), shape, _lib.BF16,
                                         _lib.MATH_F32, 0.05, 0.0, 0.0, flags, st, s), "K1")


if args.ncu:
    for name, f in FLAGS.items():
        run(f)
    torch.cuda.synchronize()
    sys.exit(0)
for name, f in FLAGS.items():
    for _ in range(3):
        run(f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run(f)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (10 * args.n)
    print(f"{name:10s} {us:8.2f} us/launch  {6 * shape / (us * 1e-6) / 1e9:8.1f} GB/s")
