"""Pinned host<->device copy bandwidth on this box (the e2e leg's ceiling):
H2D alone, D2H alone, and both directions at once, over 1/2/4 copy streams."""
import torch, time
torch.cuda.set_device(0)
n = 256 << 20  # 512 MB of bf16 per buffer
H = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
D = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
S = [torch.cuda.Stream() for _ in range(4)]
def run(kind, ns):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(4):
        s = S[i % ns]
        s.wait_event(e0)
        with torch.cuda.stream(s):
            if kind == "h2d": D[i].copy_(H[i], non_blocking=True)
            elif kind == "d2h": H[i].copy_(D[i], non_blocking=True)
            else:
                if i % 2 == 0: D[i].copy_(H[i], non_blocking=True)
                else: H[i].copy_(D[i], non_blocking=True)
    for s in S[:ns]: torch.cuda.current_stream().wait_stream(s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return 4 * n * 2 / ms / 1e6
for kind in ("h2d", "d2h", "both"):
    for ns in (1, 2, 4):
        r = [run(kind, ns) for _ in range(3)]
        print(kind, ns, "GB/s", round(max(r), 1))
