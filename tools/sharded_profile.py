"""Profile ShardedLOMO (config 4's path) in a world-1 NCCL group: GPU time by
kernel family, idle time between kernels, and the largest gaps.

    python tools/sharded_profile.py [--model 7b] [--mode keep|replay|strict] [--graph]
                                    [--separate-proj]

--graph profiles the GraphedShardedStep replay of the same step.
"""
import argparse
import os
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2306_09782_b200 import LossScaler  # noqa: E402
from paper_2306_09782_b200.sharded import ShardedLOMO  # noqa: E402
from paper_2306_09782_b200.workloads import Llama  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--mode", default="keep", choices=["keep", "replay", "strict"])
ap.add_argument("--graph", action="store_true")
ap.add_argument("--separate-proj", action="store_true")
a = ap.parse_args()
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29571")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
model = Llama(a.model, dtype=torch.float16, device="cuda", fused_proj=not a.separate_proj)
opt = ShardedLOMO(model, lr=1e-3, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10),
                  reshard_after_forward=False, replay=a.mode == "replay",
                  keep_grads=a.mode == "keep")
d = torch.randint(0, 32000, (1, 1025), device="cuda")
step = lambda: opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)  # noqa: E731
if a.graph:
    from paper_2306_09782_b200.graphs import GraphedShardedStep  # noqa: E402
    gs = GraphedShardedStep(opt, lambda x: model.loss(x[:, :-1], x[:, 1:]), [d], warmup=2,
                            lr=1e-3)
    step = lambda: gs.step(1e-3)  # noqa: E731
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
ks = []
for e in prof.events():
    if e.device_type.name != "CUDA" or e.device_time_total <= 0:
        continue
    n = e.name
    ks.append((e.time_range.start, e.time_range.end, n))
    k = ("K1" if "k1_update" in n else "K2" if "k2_probe" in n else
         "NCCL" if "nccl" in n.lower() else
         "memcpy/memset" if ("Memcpy" in n or "Memset" in n) else
         "gemm" if any(s in n.lower() for s in ("gemm", "nvjet", "xmma", "cutlass")) else
         "attention" if any(s in n.lower() for s in ("flash", "fmha", "sdpa")) else "other")
    fam[k] += e.device_time_total
total = sum(fam.values())
print(f"GPU time per step: {total / 2 / 1e3:.2f} ms (streams may overlap)")
for k, v in sorted(fam.items(), key=lambda x: -x[1]):
    print(f"  {k:14s} {v / 2 / 1e3:8.2f} ms")
ks.sort()
end, idle, gaps = ks[0][1], 0.0, []
for s, e, n in ks[1:]:
    if s > end:
        idle += s - end
        gaps.append((s - end, n))
    end = max(end, e)
print(f"device idle (no kernel on any stream) {idle / 2 / 1e3:.2f} ms per step")
for g, n in sorted(gaps, reverse=True)[:8]:
    print(f"  {g:9.1f} us  before {n[:60]!r}")
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=14))
dist.destroy_process_group()
