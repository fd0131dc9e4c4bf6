"""Is the graphed step's one host sync worth removing?  Times the LLaMA-7B
GraphedLOMOStep (replay + K6/K5) with its mid-step status read against g1 and
g2 replayed back to back without it (the upper bound of a device-side
decision, e.g. a CUDA-graph conditional node; unsafe in general: a skipped
step needs the decision).

    python tools/nosync_probe.py
"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2306_09782_b200 import LOMO, LossScaler
from paper_2306_09782_b200.graphs import GraphedLOMOStep
from paper_2306_09782_b200.workloads import Llama
torch.cuda.set_device(0)
torch.backends.cuda.matmul.allow_tf32 = False
m = Llama("7b", dtype=torch.float16, device="cuda", fused_proj=True)
opt = LOMO(m, lr=1e-3, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10, growth_interval=1000),
           replay=True, fuse_gemm=True)
d = torch.randint(0, 32000, (1, 1025), device="cuda")
g = GraphedLOMOStep(opt, lambda x: m.loss(x[:, :-1], x[:, 1:]), (d,), warmup=2, lr=1e-3)
def timed(fn, n=40):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n
def synced(): g.step(1e-3)
def nosync():
    g.g1.replay(); g.g2.replay()
for r in range(3):
    a = timed(synced); b = timed(nosync)
    print(f"round {r}: with the mid-step status read {a:.2f} ms, without {b:.2f} ms ({100*(a-b)/a:.2f} %)")
print(opt.read_status().steps_skipped, "skipped")
