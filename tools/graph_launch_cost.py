"""Host cost of the graphed LLaMA-7B LOMO step's pieces (set_lr, g1 replay,
status read, g2 replay), to see whether the host keeps up with the device.

    python tools/graph_launch_cost.py [--fused-proj]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import LOMO, LossScaler  # noqa: E402
from paper_2306_09782_b200 import _lib  # noqa: E402
from paper_2306_09782_b200.graphs import GraphedLOMOStep  # noqa: E402
from paper_2306_09782_b200.workloads import Llama  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fused-proj", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
model = Llama("7b", dtype=torch.float16, device="cuda", fused_proj=a.fused_proj)
opt = LOMO(model, lr=1e-3, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10),
           replay=True, fuse_gemm=True)
d = torch.randint(0, 32000, (1, 1025), device="cuda")
gs = GraphedLOMOStep(opt, lambda t: model.loss(t[:, :-1], t[:, 1:]), (d,), warmup=2)
for _ in range(3):
    gs.step(1e-3)
torch.cuda.synchronize()
eng = opt.engine
T = {"set_lr": 0.0, "g1.replay": 0.0, "read_status": 0.0, "g2.replay": 0.0}
N = 10
t_all = time.perf_counter()
for _ in range(N):
    t0 = time.perf_counter()
    _lib.check(eng.lib.lomo_set_lr(eng.ptr, 1e-3, eng.stream()), "set_lr")
    t1 = time.perf_counter()
    gs.g1.replay()
    t2 = time.perf_counter()
    st = eng.read_status()
    t3 = time.perf_counter()
    gs.g2.replay()
    t4 = time.perf_counter()
    T["set_lr"] += t1 - t0
    T["g1.replay"] += t2 - t1
    T["read_status"] += t3 - t2
    T["g2.replay"] += t4 - t3
torch.cuda.synchronize()
wall = (time.perf_counter() - t_all) / N
print({k: round(1e3 * v / N, 3) for k, v in T.items()}, "ms per step (host)")
print(f"wall per step {1e3 * wall:.2f} ms")
