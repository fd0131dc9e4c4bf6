"""Run N LOMO probe passes (K2 over every LLaMA-7B gradient, USE_SCALE, then
K3a) exactly as pass 1's hooks issue them -- the command the K2 ncu captures
under profiles/ were taken from.

    python tools/probe_pass.py [--passes 3] [--dtype bf16] [--unchained]
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
ap.add_argument("--unchained", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
lib = _lib.load()
P, G = bench.make_update_workload(0, 1, a.dtype)
code = _lib.BF16 if a.dtype == "bf16" else _lib.F16
s = torch.cuda.current_stream().cuda_stream
st = torch.zeros(_lib.state_bytes(len(G)), dtype=torch.uint8, device="cuda")
_lib.check(lib.lomo_state_init(st.data_ptr(), len(G), 1024.0, 16, 1.0, 2.0 ** 24, 1.0, 1.0, s),
           "init")
disp = HookDispatcher(lib, st.data_ptr(), _lib.MATH_F32)
disp.configure(flags=_lib.USE_SCALE, chain=not a.unchained)  # as the bench's probe pass
for _ in range(a.passes):
    lib.lomo_begin_step(st.data_ptr(), None, 0, s)
    for i in range(len(G) - 1, -1, -1):
        disp.probe(G[i], code, len(G) - 1 - i, s)
    disp.flush(s)
    lib.lomo_finalize_norm(st.data_ptr(), s)
torch.cuda.synchronize()
print(f"{a.passes} probe passes over {len(G)} tensors")
