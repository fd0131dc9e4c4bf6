"""K4 (the reduce-scatter fused with the update / probe) on ONE GPU with
simulated peers: rank 0 of a world of W ranks, its slice of every LLaMA-7B
bucket read from W distinct local buffers (what the peer-mapped buffers are
at N > 1, with NVLink in place of local HBM).  This measures the kernel's
HBM efficiency: algorithmic bytes (2W + 4) per element for the update (W
gradient slices + p read + p write), 2W for the probe.

    python tools/k4_local.py [--world 8] [--passes 10]
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_09782_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--passes", type=int, default=10)
a = ap.parse_args()
torch.cuda.set_device(0)
lib = _lib.load()
W = a.world
sizes, _ = bench._buckets_7b(W)
gen = torch.Generator(device="cuda").manual_seed(0)
shards, peers, tabs = [], [], []
for n in sizes:
    S = n // W
    shards.append(torch.empty(S, dtype=torch.bfloat16, device="cuda").uniform_(-0.08, 0.08,
                                                                               generator=gen))
    bufs = [torch.empty(S, dtype=torch.bfloat16, device="cuda").normal_(0, 1e-3, generator=gen)
            for _ in range(W)]
    peers.append(bufs)
    tabs.append(torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda"))
elems = sum(s.numel() for s in shards)
st = torch.zeros(_lib.state_bytes(len(sizes)), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
_lib.check(lib.lomo_state_init(st.data_ptr(), len(sizes), 0.0, 16, 1.0, 2.0 ** 24, 0.0, 1.0, s),
           "init")


def upd():
    for k in range(len(shards) - 1, -1, -1):
        _lib.check(lib.lomo_fused_rs_update(shards[k].data_ptr(), ctypes.c_void_p(tabs[k].data_ptr()),
                                            W, 0, shards[k].numel(), _lib.BF16, _lib.MATH_F32,
                                            0.05, 0.0, 0.0, 0, None, s), "rs_update")


def prb():
    lib.lomo_begin_step(st.data_ptr(), None, 0, s)
    for k in range(len(shards) - 1, -1, -1):
        _lib.check(lib.lomo_fused_rs_probe(ctypes.c_void_p(tabs[k].data_ptr()), W, 0,
                                           shards[k].numel(), _lib.BF16, k, 0, st.data_ptr(), s),
                   "rs_probe")


def timed(fn):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.passes):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / a.passes


peak = bench._peaks()[0]
for name, fn, bpe in (("K4 update", upd, 2 * W + 4), ("K4 probe", prb, 2 * W)):
    ms = timed(fn)
    gbs = bpe * elems / (ms * 1e-3) / 1e9
    print(f"world {W}: {name:10s} {ms:7.3f} ms per 7B pass  {gbs:7.1f} GB/s "
          f"({bpe} B/elem, {gbs / peak:.3f} of the copy peak)")
