"""Host-side dispatch of the hook bodies onto the C-ABI (one place, used by
the LOMO optimizer's autograd hooks and by bench.py, so the benchmark times
exactly the launches training issues).

Every gradient >= ``small_numel`` elements is handed to its own K1 (update)
or K2 (probe) launch the moment its hook fires -- the LOMO contract
(optim.py:1-7): consume each gradient as soon as it exists.  Tiny tensors
(the RMSNorm scale vectors: 65 of the 291 LLaMA-7B tensors, 0.004% of the
elements) would each cost a full launch; they are parked (their gradients
total a few hundred KB) and flushed as ONE multi-tensor launch per 64 at
the end of the backward pass.  Peak gradient memory therefore stays at the
largest single tensor plus the parked tiny ones.
"""
from __future__ import annotations

import ctypes
import importlib.util

from . import _lib

SMALL_NUMEL = 1 << 16

_CPP = None


def cpp_dispatch():
    """The C++ form of this dispatcher (csrc/lomo_dispatch.cpp, built in-tree
    by __graft_entry__.build() next to liblomo_b200.so), or None if absent."""
    global _CPP
    if _CPP is None:
        import sysconfig
        path = _lib.LIB_PATH.parent / ("_lomo_dispatch" + sysconfig.get_config_var("EXT_SUFFIX"))
        _CPP = False
        if path.exists():
            spec = importlib.util.spec_from_file_location("_lomo_dispatch", path)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            _CPP = mod
    return _CPP or None


class HookDispatcher:
    """Per-pass launcher of K1/K2 for the hooks.

    ``side_stream``: when given, every launch goes to that stream after an
    event recorded on the hook's (autograd) stream -- the update of parameter
    i then overlaps the backward of the layers below it on the main stream.
    The gradient's block is protected with ``record_stream`` so the caching
    allocator cannot hand it out before the kernel has read it; the caller
    joins the side stream after backward (``join``).  Gradient lifetime grows
    from "until the launch" to "until the kernel ran", so more than one
    gradient can be alive -- hence opt-in.
    """

    def __init__(self, lib, state_ptr: int | None, math_code: int,
                 small_numel: int = SMALL_NUMEL, side_stream=None, use_cpp: bool = True):
        self.lib = lib
        self.state_ptr = state_ptr
        self.math = math_code
        self.small = small_numel
        self._upd = {}    # dtype code -> [(p, g)]
        self._prb = {}    # dtype code -> [(g, slot)]
        self._launches = 0
        self.side = side_stream
        # the same launches from C++ (one pybind call + the CUDA launch per
        # gradient, no ctypes argument conversion); the side-stream mode
        # stays in Python
        mod = cpp_dispatch() if (use_cpp and side_stream is None) else None
        self._cpp = mod.Dispatcher(state_ptr or 0, math_code, small_numel) if mod else None
        if side_stream is not None:
            import torch
            self._events = [torch.cuda.Event() for _ in range(32)]
            self._ev = 0
        self.configure()

    def _route(self, stream: int, tensors) -> int:
        """The stream to launch on (the hook's, or the side stream)."""
        if self.side is None:
            return stream
        import torch
        ev = self._events[self._ev]
        self._ev = (self._ev + 1) % len(self._events)
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        for t in tensors:
            t.record_stream(self.side)
        return self.side.cuda_stream

    def join(self) -> None:
        """Make the current stream wait for everything launched on the side stream."""
        if self.side is not None:
            import torch
            torch.cuda.current_stream().wait_stream(self.side)

    def configure(self, lr: float = 0.0, clip: float = 0.0, wd: float = 0.0, flags: int = 0,
                  chain: bool = False):
        """Per-pass constants (the same for every tensor of one backward).

        ``chain``: the caller issues this pass's updates back to back with no
        other kernel in between (a pass over kept or replayed gradients, the
        config-2 microbench) -- every K1 that directly follows one of this
        dispatcher's K1 launches on the same stream (every K2 that directly
        follows one of its K2 launches) gets ``LOMO_CHAINED`` and overlaps
        the previous launch's drain.  Never for the autograd
        hook path, where the gradient's producer runs just before the K1."""
        self.lr, self.clip, self.wd, self.flags = float(lr), float(clip), float(wd), int(flags)
        self.chain = bool(chain) and self.side is None
        self._chain = None  # (family, stream) of the last launch: "u" K1, "p" K2
        if self._cpp is not None:
            self._cpp.configure(self.lr, self.clip, self.wd, self.flags, self.chain)
            self.update = self._cpp_update
            self.probe = self._cpp_probe

    @property
    def launches(self) -> int:
        return self._launches + (self._cpp.launches if self._cpp is not None else 0)

    def _cpp_update(self, p, g, dt: int, stream: int) -> None:
        self._cpp.update(p, g, stream)

    def _cpp_probe(self, g, dt: int, slot: int, stream: int) -> None:
        self._cpp.probe(g, slot, stream)

    # ------------------------------------------------------------ K1 / K2
    def update(self, p, g, dt: int, stream: int) -> None:
        n = p.numel()
        if n <= self.small:
            lst = self._upd.setdefault(dt, [])
            lst.append((p, g))
            if len(lst) == 64:
                self._flush_upd(dt, stream)
            return
        stream = self._route(stream, (g,))
        flags = self.flags | (_lib.CHAINED if self.chain and self._chain == ("u", stream) else 0)
        rc = self.lib.lomo_fused_update(p.data_ptr(), g.data_ptr(), n, dt, self.math, self.lr,
                                        self.clip, self.wd, flags, self.state_ptr, stream)
        if rc:
            _lib.check(rc, "lomo_fused_update")
        self._chain = ("u", stream)
        self._launches += 1

    def probe(self, g, dt: int, slot: int, stream: int) -> None:
        n = g.numel()
        if n <= self.small:
            lst = self._prb.setdefault(dt, [])
            lst.append((g, slot))
            if len(lst) == 64:
                self._flush_prb(dt, stream)
            return
        stream = self._route(stream, (g,))
        flags = self.flags | (_lib.CHAINED if self.chain and self._chain == ("p", stream) else 0)
        rc = self.lib.lomo_probe(g.data_ptr(), n, dt, slot, flags, self.state_ptr, stream)
        self._chain = ("p", stream)
        if rc:
            _lib.check(rc, "lomo_probe")
        self._launches += 1

    # ------------------------------------------------------------ flushing
    def _flush_upd(self, dt, stream):
        lst = self._upd.pop(dt, [])
        if not lst:
            return
        k = len(lst)
        stream = self._route(stream, [g for _, g in lst])
        ps = (ctypes.c_void_p * k)(*[p.data_ptr() for p, _ in lst])
        gs = (ctypes.c_void_p * k)(*[g.data_ptr() for _, g in lst])
        ns = (ctypes.c_int64 * k)(*[p.numel() for p, _ in lst])
        _lib.check(self.lib.lomo_fused_update_multi(ps, gs, ns, k, dt, self.math, self.lr,
                                                    self.clip, self.wd, self.flags,
                                                    self.state_ptr, stream),
                   "lomo_fused_update_multi")
        self._chain = ("u", stream)  # a K1 multi on other tensors may precede a chained K1
        self._launches += (k + 63) // 64

    def _flush_prb(self, dt, stream):
        lst = self._prb.pop(dt, [])
        if not lst:
            return
        k = len(lst)
        stream = self._route(stream, [g for g, _ in lst])
        gs = (ctypes.c_void_p * k)(*[g.data_ptr() for g, _ in lst])
        ns = (ctypes.c_int64 * k)(*[g.numel() for g, _ in lst])
        ss = (ctypes.c_int * k)(*[s for _, s in lst])
        _lib.check(self.lib.lomo_probe_multi(gs, ns, ss, k, dt, self.flags, self.state_ptr, stream),
                   "lomo_probe_multi")
        self._chain = ("p", stream)
        self._launches += (k + 63) // 64

    def flush(self, stream: int) -> None:
        """Launch everything parked; the parked gradients are released after
        their kernel is enqueued (stream-ordered reuse by the allocator)."""
        if self._cpp is not None:
            self._cpp.flush(stream)
        for dt in list(self._upd):
            self._flush_upd(dt, stream)
        for dt in list(self._prb):
            self._flush_prb(dt, stream)
        self.join()

    def pending(self) -> int:
        return (sum(map(len, self._upd.values())) + sum(map(len, self._prb.values())) +
                (self._cpp.pending() if self._cpp is not None else 0))
