"""Run N LOMO update passes over the LLaMA-7B tensors (the bench workload) --
the command the ncu captures under profiles/ were taken from.

    python tools/update_pass.py [--passes 3] [--dtype bf16] [--math f32] [--unchained]

K1s after the first of a pass are chained (LOMO_CHAINED) as in the bench;
--unchained times the hook pattern (every K1 waits for its predecessor).
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_09782_b200 import _lib  # noqa: E402
from paper_2306_09782_b200.dispatch import HookDispatcher  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--passes", type=int, default=3)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--math", default="f32")
ap.add_argument("--unchained", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
lib = _lib.load()
disp = HookDispatcher(lib, None, _lib.MATH_F64 if a.math == "f64" else _lib.MATH_F32)
disp.configure(lr=0.05, chain=not a.unchained)
P, G = bench.make_update_workload(0, 1, a.dtype)
code = _lib.BF16 if a.dtype == "bf16" else _lib.F16
s = torch.cuda.current_stream().cuda_stream
for _ in range(a.passes):
    n = bench.run_update_pass(disp, P, G, code, s)
torch.cuda.synchronize()
print(f"{a.passes} passes, {n} launches per pass")
