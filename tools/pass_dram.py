"""Whole-pass DRAM bytes of the LLaMA-7B update pass (K1) and probe pass (K2).

    ncu --replay-mode app-range --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python tools/pass_dram.py

One profiler range per pass (cudaProfilerStart/Stop), after warm-up passes, so
ncu counts the DRAM traffic of the WHOLE pass -- 228 back-to-back launches,
the write-back of each launch's dirty lines included (a per-launch capture
ends with the last ~45 MB of written parameters still dirty in L2 and
under-counts the writes).  Ideal: 6 B/elem (update), 2 B/elem (probe).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_09782_b200 import _lib  # noqa: E402
from paper_2306_09782_b200.dispatch import HookDispatcher  # noqa: E402

torch.cuda.set_device(0)
lib = _lib.load()
P, G = bench.make_update_workload(0, 1, "bf16")
elems = sum(p.numel() for p in P)
s = torch.cuda.current_stream().cuda_stream
disp = HookDispatcher(lib, None, _lib.MATH_F32)
disp.configure(lr=0.05, chain=True)  # as the bench pass
st = torch.zeros(_lib.state_bytes(len(P)), dtype=torch.uint8, device="cuda")
_lib.check(lib.lomo_state_init(st.data_ptr(), len(P), 1024.0, 16, 1.0, 2.0 ** 24, 1.0, 1.0, s),
           "init")
pd = HookDispatcher(lib, st.data_ptr(), _lib.MATH_F32)
pd.configure(flags=_lib.USE_SCALE)


def probe_pass():
    lib.lomo_begin_step(st.data_ptr(), None, 0, s)
    for i in range(len(G) - 1, -1, -1):
        pd.probe(G[i], _lib.BF16, len(G) - 1 - i, s)
    pd.flush(s)
    lib.lomo_finalize_norm(st.data_ptr(), s)


for _ in range(2):
    bench.run_update_pass(disp, P, G, _lib.BF16, s)
    probe_pass()
torch.cuda.synchronize()
for name, fn in (("update", lambda: bench.run_update_pass(disp, P, G, _lib.BF16, s)),
                 ("probe", probe_pass)):
    torch.cuda.profiler.start()
    fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print(f"elements per pass {elems}: ideal update {6 * elems} B, probe {2 * elems} B")
