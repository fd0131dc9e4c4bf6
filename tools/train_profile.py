"""Profile one LLaMA-7B LOMO step (config 3) with torch.profiler: GPU time by
kernel family vs wall time, to see where the step goes.

    python tools/train_profile.py [--seq 1024] [--batch 1] [--layers 32]
"""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import LOMO, LossScaler  # noqa: E402
from paper_2306_09782_b200.workloads import Llama  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=1024)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--ckpt", action="store_true")
ap.add_argument("--replay", action="store_true")
ap.add_argument("--fuse", action="store_true")
ap.add_argument("--grouped", action="store_true")
ap.add_argument("--graph", action="store_true", help="GraphedLOMOStep (implies --replay --fuse)")
ap.add_argument("--fused-proj", action="store_true", help="stacked qkv / gate_up weights")
a = ap.parse_args()
torch.cuda.set_device(0)
model = Llama("7b", dtype=torch.float16, device="cuda", layers=a.layers, checkpointing=a.ckpt,
              fused_proj=a.fused_proj)
if a.graph:
    a.replay = a.fuse = True
if a.grouped:
    from paper_2306_09782_b200 import GroupedLOMO  # noqa: E402
    opt = GroupedLOMO(model, lr=1e-3, max_norm=1.0, window=1)
else:
    opt = LOMO(model, lr=1e-3, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10),
               replay=a.replay, fuse_gemm=a.fuse)
d = torch.randint(0, 32000, (a.batch, a.seq + 1), device="cuda")
step = lambda: opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)
if a.graph:
    from paper_2306_09782_b200.graphs import GraphedLOMOStep  # noqa: E402
    gs = GraphedLOMOStep(opt, lambda t: model.loss(t[:, :-1], t[:, 1:]), (d,), warmup=2)
    step = lambda: gs.step(1e-3)
for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(3):
    step()
ev[1].record()
torch.cuda.synchronize()
print(f"wall (events, unprofiled) per step: {ev[0].elapsed_time(ev[1]) / 3:.2f} ms")
fam = defaultdict(float)
total = 0.0
for e in prof.events():          # device kernels only (no CPU-op double counting)
    if e.device_type.name != "CUDA" or e.device_time_total <= 0:
        continue
    t = e.device_time_total
    total += t
    n = e.name
    k = ("K1 k1_update" if "k1_update" in n else "K2 k2_probe" if "k2_probe" in n else
         "K3/begin" if ("k3_" in n or "k_begin" in n) else
         "K5 fused gemm+update" if "cutlass" in n.lower() or "GemmUniversal" in n else
         "gemm (cuBLAS)" if any(s in n.lower() for s in ("gemm", "nvjet", "xmma")) else
         "attention" if any(s in n.lower() for s in ("flash", "fmha", "attention", "sdpa")) else
         "elementwise/other")
    fam[k] += t
print(f"GPU time per step: {total / 2 / 1e3:.2f} ms")
for k, v in sorted(fam.items(), key=lambda x: -x[1]):
    print(f"  {k:20s} {v / 2 / 1e3:8.2f} ms  {100 * v / total:5.1f}%")
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=25))

# idle time between consecutive kernels on the device (the profiled steps):
# where the wall-minus-kernel time goes
ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type.name == "CUDA" and e.device_time_total > 0)
gaps = [(ks[i + 1][0] - ks[i][1], ks[i][2], ks[i + 1][2]) for i in range(len(ks) - 1)]
pos = [g for g in gaps if g[0] > 0]
print(f"kernels: {len(ks)}; device span {(ks[-1][1] - ks[0][0]) / 2 / 1e3:.2f} ms per step; "
      f"idle between kernels {sum(g[0] for g in pos) / 2 / 1e3:.2f} ms per step")
hist = defaultdict(float)
for g, _, _ in pos:
    b = "<1us" if g < 1 else "1-2us" if g < 2 else "2-5us" if g < 5 else "5-20us" if g < 20 \
        else "20-100us" if g < 100 else ">100us"
    hist[b] += g
print("  idle by gap size (ms per step): " +
      ", ".join(f"{k} {v / 2 / 1e3:.2f}" for k, v in sorted(hist.items())))
for g, a_, b_ in sorted(pos, reverse=True)[:12]:
    print(f"  {g:9.1f} us  after {a_[:50]!r}  before {b_[:50]!r}")
