import sys; sys.path.insert(0, '/root/repo')
import torch
from collections import Counter
from paper_2306_09782_b200 import LOMO
from paper_2306_09782_b200.workloads import Llama
torch.cuda.set_device(0)
m = Llama(dict(hidden=1024, layers=2, heads=8, ffn=2816, vocab=4096), dtype=torch.float16, device="cuda")
opt = LOMO(m, lr=1e-3, clip_grad_norm=1.0, loss_scale=1024.0)
d = torch.randint(0, 4096, (1, 257), device="cuda")
for _ in range(2): opt.step(lambda: m.loss(d[:, :-1], d[:, 1:]), 1e-3)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    opt.step(lambda: m.loss(d[:, :-1], d[:, 1:]), 1e-3); torch.cuda.synchronize()
c = Counter()
for e in prof.events():
    if e.name == "torch::autograd::AccumulateGrad":
        for ch in e.cpu_children:
            c[ch.name] += 1
print(c.most_common(10))
# which params?
shapes = Counter()
for e in prof.events():
    if e.name == "torch::autograd::AccumulateGrad" and e.cpu_children:
        shapes[str([ch.name for ch in e.cpu_children][:3])] += 1
print(shapes.most_common(5))
# direct test: is a linear weight grad stolen?
w = torch.nn.Parameter(torch.randn(256, 128, device="cuda", dtype=torch.float16))
x = torch.randn(2, 8, 128, device="cuda", dtype=torch.float16, requires_grad=True)
ptrs = {}
def h(p): ptrs['g'] = (p.grad.data_ptr(), p.grad.stride(), p.grad.is_contiguous())
w.register_post_accumulate_grad_hook(h)
torch.nn.functional.linear(x, w).sum().backward()
print("linear grad", ptrs)
