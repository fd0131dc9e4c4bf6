"""K1 inside the LLaMA-7B grouped training step vs K1 in the isolated update
pass: event-timed K1 sections, plus nvidia-smi clocks/power under load.

    python tools/k1_in_train.py [--unchained]

The instrumented flush mirrors GroupedLOMO._flush (chained K2s, K3a, chained
K1s); --unchained times every launch waiting for its predecessor.
"""
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_09782_b200 import GroupedLOMO  # noqa: E402
from paper_2306_09782_b200.workloads import Llama  # noqa: E402

CHAIN = "--unchained" not in sys.argv
torch.cuda.set_device(0)
model = Llama("7b", dtype=torch.float16, device="cuda")
opt = GroupedLOMO(model, lr=1e-3, max_norm=1.0, window=1)
d = torch.randint(0, 32000, (1, 1025), device="cuda")
step = lambda: opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)
for _ in range(3):
    step()
torch.cuda.synchronize()

# time the K1/K2 sections of each group flush with events (instrumented copy of _flush)
eng = opt.engine
from paper_2306_09782_b200 import _lib  # noqa: E402
secs = {"k2": [], "k1": []}


def flush_timed():
    if not opt._buf:
        return
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    eng.begin(None)
    eng.configure(flags=opt._probe_flags, chain=CHAIN)
    e[0].record()
    for p, g in opt._buf:
        eng.probe(g, opt._slot[id(p)])
    eng.flush()
    e[1].record()
    eng.finalize()
    eng.configure(opt._lr, 0.0, opt.weight_decay, _lib.USE_SKIP | _lib.USE_COEF, chain=CHAIN)
    e[2].record()
    n = 0
    for p, g in opt._buf:
        eng.update(p, g)
        n += p.numel()
    eng.flush()
    e[3].record()
    secs["k2"].append((e[0], e[1], n))
    secs["k1"].append((e[2], e[3], n))
    opt._buf = []


opt._flush = flush_timed
samples = []
stop = False


def smi():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
        samples.append(out.strip())
        time.sleep(0.2)


th = threading.Thread(target=smi)
th.start()
t0 = time.time()
k = 0
while time.time() - t0 < 8:
    secs = {"k2": [], "k1": []}
    step()
    k += 1
torch.cuda.synchronize()
stop = True
th.join()
for key, bpe in (("k2", 2), ("k1", 6)):
    ms = sum(a.elapsed_time(b) for a, b, _ in secs[key])
    el = sum(n for _, _, n in secs[key])
    print(f"{key}: {ms:.2f} ms per step, {bpe * el / ms / 1e6:.0f} GB/s")
print("smi samples (sm MHz, mem MHz, W, reasons):", samples[len(samples) // 2: len(samples) // 2 + 8])
