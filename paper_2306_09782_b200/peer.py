"""Peer-mapped gradient buffers for K4 (ShardedLOMO(fused_rs=...)).

K4 replaces "NCCL reduce_scatter, then K1/K2 on the shard" by one kernel that
reduces this rank's slice of a bucket straight out of every rank's buffer
(what it fuses is probe_hook, stabilize.py:193-200, and
apply_update, optim.py:52-54).  This module owns the buffers and the ordering
between ranks; the kernels and the transport primitives are in the C-ABI
(include/lomo_b200.h, csrc/lomo_peer.cu).

Transports:
  ``ipc``   one cudaMalloc per rank (NBUF bucket buffers + a signal area),
            CUDA-IPC handles exchanged over the process group and opened by
            every peer; K4 = ``lomo_fused_rs_update/probe`` (P2P loads of the
            slice from every peer, rank-order sum).  Works over NVLink and
            between processes sharing one GPU.
  ``nvls``  an NVSwitch multicast object (driver API): K4 =
            ``lomo_fused_mc_update/probe`` (``multimem.ld_reduce``: the switch
            sums the copies), barriers by ``multimem.red``.  Needs
            ``lomo_mc_supported`` and one GPU per rank.

Ordering (both transports): a buffer is owned by one open bucket from its
first gradient write to its K4 launch.  Before K4, a device barrier on the
buffer's "filled" channel (every rank wrote its bucket); before a buffer is
written again, one on its "free" channel (every rank's K4 finished reading
it).  Every rank acquires buffers in hook order, which is identical on all
ranks, so channel epochs match.  A barrier that waits longer than
``timeout_s`` writes error 2 into the optimizer's state block instead of
hanging the GPU; the step's status read raises it.
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError, NativeError

_ALIGN = 1 << 12


class _CudaArray:
    """A zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    _TS = {torch.float16: "<f2", torch.bfloat16: "<f2", torch.float32: "<f4",
           torch.float64: "<f8", torch.int64: "<i8", torch.int32: "<i4"}

    def __init__(self, ptr: int, numel: int, dtype: torch.dtype):
        self.__cuda_array_interface__ = {
            "shape": (numel,), "typestr": self._TS[dtype], "data": (ptr, False), "version": 3,
            "strides": None}


def tensor_at(ptr: int, numel: int, dtype: torch.dtype, device) -> torch.Tensor:
    # bf16 has no typestr: build it as f16 and reinterpret the bits
    t = torch.as_tensor(_CudaArray(ptr, numel, dtype), device=device)
    return t.view(dtype) if t.dtype != dtype else t


def nvls_available(device: torch.device) -> bool:
    return _lib.load().lomo_mc_supported(device.index if device.index is not None else
                                         torch.cuda.current_device()) == 1


class PeerRing:
    """NBUF peer-mapped flat buffers of ``numel`` elements of ``dtype``."""

    NBUF = 3

    def __init__(self, numel: int, dtype: torch.dtype, device: torch.device, group,
                 transport: str = "ipc", err_ptr: int = 0, timeout_s: float = 120.0,
                 nbuf: int | None = None):
        if transport not in ("ipc", "nvls"):
            raise ConfigError(f"peer transport must be 'ipc' or 'nvls', got {transport!r}")
        if nbuf is not None:
            if nbuf < 1:
                raise ConfigError("nbuf must be >= 1")
            self.NBUF = int(nbuf)
        self.lib = _lib.load()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > _lib.PEER_MAX:
            raise ConfigError(f"fused_rs supports at most {_lib.PEER_MAX} ranks")
        self.device = device
        self.dev_idx = device.index if device.index is not None else torch.cuda.current_device()
        self.dtype = dtype
        self.numel = int(numel)
        self.esize = torch.empty((), dtype=dtype).element_size()
        self.buf_bytes = -(-self.numel * self.esize // _ALIGN) * _ALIGN
        self.sig_off = self.NBUF * self.buf_bytes
        self.total = self.sig_off + _lib.PEER_SIGNAL_BYTES
        self.transport = transport
        self.timeout_ns = int(timeout_s * 1e9)
        self._own_err = None
        if not err_ptr:
            self._own_err = torch.zeros(1, dtype=torch.int32, device=device)
            err_ptr = self._own_err.data_ptr()
        self.err_ptr = err_ptr
        # per-channel epoch counters in device memory (lomo_*_barrier_dev): a
        # CUDA graph replaying a barrier advances them, so K4 can be captured
        self.epochs_dev = torch.zeros(_lib.PEER_CHANNELS, dtype=torch.int64, device=device)
        self.owner = [None] * self.NBUF
        self.read_pending = [False] * self.NBUF
        self.k = 0
        self._closed = False
        self._opened: list[int] = []
        self._base = 0
        self._mc_obj = 0
        with torch.cuda.device(self.dev_idx):
            if transport == "ipc":
                self._setup_ipc()
            else:
                self._setup_nvls()
        self.bufs = [tensor_at(self._base + k * self.buf_bytes, self.numel, dtype, device)
                     for k in range(self.NBUF)]

    # ------------------------------------------------------------------ setup
    def _setup_ipc(self) -> None:
        lib = self.lib
        hb = lib.lomo_ipc_handle_bytes()
        handle = (ctypes.c_char * hb)()
        base = ctypes.c_void_p()
        _lib.check(lib.lomo_ipc_alloc(self.total, ctypes.byref(base), handle), "lomo_ipc_alloc")
        self._base = base.value
        mine = bytes(handle)
        allh: list = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        bases = []
        for r, h in enumerate(allh):
            if r == self.rank:
                bases.append(self._base)
                continue
            ptr = ctypes.c_void_p()
            buf = (ctypes.c_char * hb).from_buffer_copy(h)
            _lib.check(lib.lomo_ipc_open(buf, ctypes.byref(ptr)), f"lomo_ipc_open(rank {r})")
            self._opened.append(ptr.value)
            bases.append(ptr.value)
        self.peers_dev = [torch.tensor([b + k * self.buf_bytes for b in bases], dtype=torch.int64,
                                       device=self.device) for k in range(self.NBUF)]
        self.sig_dev = torch.tensor([b + self.sig_off for b in bases], dtype=torch.int64,
                                    device=self.device)
        dist.barrier(group=self.group)  # every rank mapped every peer before any use

    def _setup_nvls(self) -> None:
        lib = self.lib
        obj = ctypes.c_uint64()
        if self.rank == 0:
            size = ctypes.c_size_t()
            fd = ctypes.c_int(-1)
            rc = lib.lomo_mc_create(self.world, self.total, ctypes.byref(obj), ctypes.byref(size),
                                    ctypes.byref(fd))
            info = [rc, os.getpid(), fd.value, size.value]
        else:
            info = None
        box = [info]
        dist.broadcast_object_list(box, src=dist.get_global_rank(self.group, 0)
                                   if self.group is not None else 0, group=self.group)
        rc0, pid, fd, size = box[0]
        if rc0 != 0:
            raise NativeError(f"lomo_mc_create failed with status {rc0}"
                              + (" (no multicast support)" if rc0 == _lib.E_UNSUPPORTED else ""))
        rc = 0
        if self.rank != 0:
            rc = lib.lomo_mc_import(pid, fd, size, ctypes.byref(obj))
        self._mc_obj = obj.value
        if rc == 0:
            rc = lib.lomo_mc_add_device(self._mc_obj, self.dev_idx)
        rcs: list = [None] * self.world
        dist.all_gather_object(rcs, rc, group=self.group)  # every device added (or a failure)
        if any(rcs):
            self.close()
            raise NativeError(f"NVLS setup failed on some rank: {rcs}")
        uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        rc = lib.lomo_mc_bind(self._mc_obj, self.dev_idx, ctypes.byref(uc), ctypes.byref(mc))
        dist.all_gather_object(rcs, rc, group=self.group)  # every copy bound and zeroed
        if any(rcs):
            self.close()
            raise NativeError(f"lomo_mc_bind failed on some rank: {rcs}")
        self.total = size
        self._base = uc.value
        self.mc_base = mc.value

    # ----------------------------------------------------------- ring logic
    def acquire(self, bucket_idx: int) -> int:
        for _ in range(self.NBUF):
            k = self.k
            self.k = (self.k + 1) % self.NBUF
            if self.owner[k] is None:
                if self.read_pending[k]:
                    self.barrier(self._free_ch(k))  # every rank's K4 finished reading k
                    self.read_pending[k] = False
                self.owner[k] = bucket_idx
                return k
        raise RuntimeError(f"more than {self.NBUF} buckets receive gradients at once")

    def release(self, k: int) -> None:
        self.owner[k] = None
        self.read_pending[k] = True

    def barrier(self, channel: int) -> None:
        """Device barrier over the ranks, stream-ordered on the current stream;
        the channel's epoch is a device counter (graph-capturable)."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        if self.transport == "ipc":
            rc = self.lib.lomo_peer_barrier_dev(self.sig_dev.data_ptr(), self.epochs_dev.data_ptr(),
                                                self.world, self.rank, channel, self.timeout_ns,
                                                self.err_ptr, s)
        else:
            rc = self.lib.lomo_mc_barrier_dev(self.mc_base + self.sig_off,
                                              self._base + self.sig_off,
                                              self.epochs_dev.data_ptr(), self.world, channel,
                                              self.timeout_ns, self.err_ptr, s)
        _lib.check(rc, "peer barrier")

    # Channels name epoch counters: buffer k's "filled" barriers use channel
    # k mod 8, its "free" barriers 8 + k mod 8.  Buffers may share a channel --
    # every rank issues the same sequence of barriers, so the epochs agree.
    _HALF = _lib.PEER_CHANNELS // 2

    def _filled_ch(self, k: int) -> int:
        return k % self._HALF

    def _free_ch(self, k: int) -> int:
        return self._HALF + k % self._HALF

    def filled(self, k: int) -> None:
        """Every rank has written buffer k (before its K4)."""
        self.barrier(self._filled_ch(k))

    # ------------------------------------------------------------------ K4
    def update(self, engine, p_shard: torch.Tensor, k: int, offset: int) -> None:
        if self.transport == "ipc":
            engine.rs_update(p_shard, self.peers_dev[k].data_ptr(), self.world, offset)
        else:
            engine.mc_update(p_shard, self.mc_base + k * self.buf_bytes + offset * self.esize)

    def probe(self, engine, k: int, offset: int, n: int, slot: int, out=None) -> None:
        """K4 probe of this rank's slice; ``out``: also keep the reduced slice."""
        if self.transport == "ipc":
            engine.rs_probe(self.peers_dev[k].data_ptr(), self.world, offset, n, self.dtype, slot,
                            out=out)
        else:
            engine.mc_probe(self.mc_base + k * self.buf_bytes + offset * self.esize, n,
                            self.dtype, slot, out=out)

    # ----------------------------------------------------------------- close
    def close(self) -> None:
        """Unmap the peers and free this rank's memory.  Collective: no rank
        frees a buffer a peer may still read."""
        if self._closed:
            return
        self._closed = True
        torch.cuda.synchronize(self.dev_idx)
        if dist.is_initialized():
            dist.barrier(group=self.group)
        for ptr in self._opened:
            self.lib.lomo_ipc_close(ptr)
        self._opened = []
        if self.transport == "ipc" and self._base:
            self.lib.lomo_ipc_free(self._base)
        if self._mc_obj:
            self.lib.lomo_mc_free(self._mc_obj)
        self._base = self._mc_obj = 0
        self.bufs = []
