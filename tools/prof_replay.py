"""Run N LLaMA-7B LOMO steps with replay + fused GEMM (config 3, the bench's
headline train variant) -- the command the K5 ncu captures were taken from."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import LOMO, LossScaler  # noqa: E402
from paper_2306_09782_b200.workloads import Llama  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
torch.cuda.set_device(0)
m = Llama("7b", dtype=torch.float16, device="cuda")
opt = LOMO(m, lr=1e-3, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10), replay=True,
           fuse_gemm=True)
d = torch.randint(0, 32000, (1, 1025), device="cuda")
for _ in range(steps):
    opt.step(lambda: m.loss(d[:, :-1], d[:, 1:]), 1e-3)
torch.cuda.synchronize()
print("ok")
