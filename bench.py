#!/usr/bin/env python
"""Benchmark of the LOMO fused-update path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (``value``): the fused-update HBM throughput of one full LOMO update
pass over all 291 LLaMA-7B parameter tensors (config 2: bf16 storage, fp32
math, one K1 launch per tensor exactly as the autograd hook delivers them),
whole job, inputs resident in HBM.  A "step" = one such pass (6,738,415,616
elements, 6 B/elem algorithmic = 40.43 GB).  Each byte is touched once per
step and the per-step working set (27 GB) is > 200x L2, so no L2 flush is
needed between steps.

Also on the line:
  roofline      K1 achieved GB/s from per-launch CUDA events (byte weighted) vs
                MEASURED_PEAKS.json hbm_gbs; traffic from the committed ncu capture
  e2e           the same pass through the C-ABI with HOST buffers: pinned H2D of
                p and g, K1, D2H of p, all inside the timed region
  cpu_baseline  the reference's own fusedtrain.optim.apply_update (optim.py:52-54,
                HALF_EMULATED write-back) imported from baseline/_ref, on all
                host cores, plus its as-shipped single-thread rate
  c1_parity     config 1: the reference's mini transformer, fixtures A/B/C
                recorded from the reference, through the product path: decisions,
                max/mean ulp, normwise error, GPU vs reference seconds
  train         config 3: LLaMA-7B fp16 LOMO, dynamic loss scale + two-pass
                global-norm clip (1.0), seq 1024 x batch 1, tokens/s; a fresh
                model per variant; the measured Table-1 row beside the
                reference estimator's
  train_sharded_world1
                config 4's sharded train leg (LLaMA-13B, ShardedLOMO) in a world-1
                NCCL group: the sharded machinery's cost next to plain LOMO
  clocks        NVML SM clock / throttle reasons sampled during the timed region

N > 1 (torchrun): the headline is the SHARDED update pass of LLaMA-7B (SURVEY
8e): per rank 33 flat gradient buckets (its own backward's), reduced across
the ranks -- NCCL reduce_scatter -> K1 on the rank's 1/W shard, and K4 over
peer-mapped buffers -- ``value`` = the 7B update's algorithmic bytes / max-
over-ranks time (strong scaling: the total work is one 7B update).  e2e is
the same pass from pinned host buffers; the train leg is ShardedLOMO on
LLaMA-13B (config 4) with NCCL_DEBUG=INFO init lines in the log.
"""
from __future__ import annotations

import argparse
import datetime
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LOMO fused-update HBM GB/s (% of peak); LLaMA-7B train tokens/s at 1/2/4/8 B200"
BYTES_PER_ELEM = 6  # 2 B param read + 2 B param write + 2 B grad read (bf16)


def _peaks():
    try:
        m = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(m["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy, measured)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def _pass_traffic():
    """DRAM bytes of one WHOLE update pass (ncu range replay, every launch's
    write-back included) against its algorithmic bytes: profiles/r02_pass_dram.json."""
    p = ROOT / "profiles" / "r02_pass_dram.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    u = d["update_pass_k1"]
    return {"dram_bytes": u["dram_bytes_read"] + u["dram_bytes_write"],
            "algorithmic_bytes": 6 * d["elements_per_pass"], "bytes_per_elem": u["bytes_per_elem"],
            "probe_pass_bytes_per_elem": d["probe_pass_k2"]["bytes_per_elem"],
            "source": "profiles/r02_pass_dram.json"}


def _traffic():
    """DRAM bytes of one K1 launch (the largest shape) from the committed ncu
    --set full capture, with that launch's algorithmic bytes."""
    p = ROOT / "profiles" / "k1_traffic.json"
    if not p.exists():
        return None
    return json.loads(p.read_text())


# --------------------------------------------------------------------------
# clocks (NVML) sampled during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.02):
        self.samples, self.reasons, self.period = [], set(), period
        self.power = []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
            except Exception:
                self.limit_w = None
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
                except Exception:
                    pass
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power:
            out["power_w"] = round(statistics.median(self.power), 1)
            out["power_limit_w"] = self.limit_w
        return out


# --------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------
def _dist_init(gpus: int):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # LOMO_BENCH_SHARE_GPU=1 (validation only): every rank on cuda:0 over
        # gloo, to exercise the N>1 code path on a single-GPU box
        shared = os.environ.get("LOMO_BENCH_SHARE_GPU") == "1"
        dev = 0 if shared else local
        torch.cuda.set_device(dev)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # a collective that never completes aborts the job after 5 minutes
        # (NCCL watchdog) instead of holding the box until the driver's limit
        tmo = datetime.timedelta(minutes=5)
        if shared:
            dist.init_process_group("gloo", timeout=tmo)
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev), timeout=tmo)
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def _barrier(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def _max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def make_update_workload(rank: int, world: int, dtype_name="bf16"):
    """The 291 LLaMA-7B tensor shapes, p and g, on this rank.

    Weak scaling: every rank updates its own full 7B-shaped set (at N ranks:
    the rank's ZeRO-3 shards of an N x 7B-parameter model, e.g. ~56-65B at
    N = 8), so per-GPU work is fixed and no collective enters the data path."""
    import torch
    from paper_2306_09782_b200.workloads import llama_param_shapes
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16}[dtype_name]
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    P, G = [], []
    for _, shape in llama_param_shapes("7b"):
        m = math.prod(shape)
        p = torch.empty(m, dtype=dt, device="cuda").uniform_(-0.08, 0.08, generator=gen)
        g = torch.empty(m, dtype=dt, device="cuda").normal_(0.0, 1e-3, generator=gen)
        P.append(p)
        G.append(g)
    return P, G


def run_update_pass(disp, P, G, dt_code, stream, events=None):
    """One update pass exactly as LOMO's hooks issue it: tensors in autograd
    delivery order (reverse registration), each through HookDispatcher.update
    (own K1 launch, tiny tensors parked), then the end-of-backward flush."""
    before = disp.launches
    for i in range(len(P) - 1, -1, -1):
        if events is not None:
            events[i][0].record()
        disp.update(P[i], G[i], dt_code, stream)
        if events is not None:
            events[i][1].record()
    if events is not None:
        events[-1][2].record()
    disp.flush(stream)
    if events is not None:
        events[-1][3].record()
    return disp.launches - before


def bench_update(args, rank, world):
    import torch
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.dispatch import HookDispatcher
    lib = _lib.load()
    disp = HookDispatcher(lib, None, _lib.MATH_F32)
    # the pass issues its K1s back to back (no kernel in between), as a pass
    # over kept or replayed gradients does: every K1 after the first is
    # chained (LOMO_CHAINED: loads/stores before the PDL wait); the unchained
    # form -- the autograd-hook pattern -- is timed beside it
    disp.configure(lr=0.05, chain=True)
    P, G = make_update_workload(rank, world, args.dtype)
    dt_code = _lib.BF16 if args.dtype == "bf16" else _lib.F16
    elems = sum(p.numel() for p in P)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(args.warmup):
        run_update_pass(disp, P, G, dt_code, stream)
    _barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        _barrier(world)
        t0 = time.perf_counter()
        start.record()
        for _ in range(args.steps):
            launches += run_update_pass(disp, P, G, dt_code, stream)
        end.record()
        host_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        _barrier(world)
    ms_local = start.elapsed_time(end)
    ms = _max_over_ranks(ms_local, world)
    total_elems = _sum_over_ranks(elems, world)
    gbs = BYTES_PER_ELEM * total_elems * args.steps / (ms * 1e-3) / 1e9
    # the unchained (hook-pattern) pass right after the headline, same state
    # of the part: every K1 waits for its predecessor before its loads
    dun = HookDispatcher(lib, None, _lib.MATH_F32)
    dun.configure(lr=0.05)
    run_update_pass(dun, P, G, dt_code, stream)
    torch.cuda.synchronize()
    start.record()
    for _ in range(args.steps):
        run_update_pass(dun, P, G, dt_code, stream)
    end.record()
    torch.cuda.synchronize()
    un_head_ms = start.elapsed_time(end) / args.steps

    # host cost of enqueueing one pass, measured from an empty launch queue (a
    # sync before each pass: the host never blocks on a full queue), for the
    # C++ dispatcher the hooks use and for its Python/ctypes form
    def enqueue_ms(d, reps=7):
        out = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            run_update_pass(d, P, G, dt_code, stream)
            out.append((time.perf_counter() - t) * 1e3)
        torch.cuda.synchronize()
        return statistics.median(out)
    pyd = HookDispatcher(lib, None, _lib.MATH_F32, use_cpp=False)
    pyd.configure(lr=0.05, chain=True)
    host_enqueue = {"dispatcher": "C++ (csrc/lomo_dispatch.cpp)" if disp._cpp is not None
                    else "python/ctypes", "ms_per_pass": round(enqueue_ms(disp), 3),
                    "python_ctypes_ms_per_pass": round(enqueue_ms(pyd), 3),
                    "launches_per_pass": len([p for p in P if p.numel() > disp.small]) + 2}

    # instrumented replay with per-launch events (same steps) -> kernel roofline
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in P]
    kt = [0.0] * len(P)
    flush_ms = 0.0
    for _ in range(args.steps):
        run_update_pass(disp, P, G, dt_code, stream, events=ev)
        torch.cuda.synchronize()
        for i, e in enumerate(ev):
            kt[i] += e[0].elapsed_time(e[1])
        flush_ms += ev[-1][2].elapsed_time(ev[-1][3])
    ksum_ms = sum(kt) + flush_ms
    achieved = BYTES_PER_ELEM * elems * args.steps / (ksum_ms * 1e-3) / 1e9
    by_shape = {}
    from paper_2306_09782_b200.workloads import llama_param_shapes
    for (name, shape), t, p in zip(llama_param_shapes("7b"), kt, P):
        if p.numel() <= disp.small:
            continue
        key = "x".join(map(str, shape))
        d = by_shape.setdefault(key, {"launches": 0, "ms": 0.0, "elems": p.numel()})
        d["launches"] += args.steps
        d["ms"] += t
    shapes = {k: {"us_per_launch": round(1e3 * d["ms"] / d["launches"], 2),
                  "gbs": round(BYTES_PER_ELEM * d["elems"] / (d["ms"] / d["launches"] * 1e-3) / 1e9, 1)}
              for k, d in by_shape.items()}
    small = [p for p in P if p.numel() <= disp.small]
    shapes["coalesced_small"] = {"tensors": len(small), "us_per_step": round(1e3 * flush_ms / args.steps, 2)}
    # pass 1 of the two-pass protocol over the same tensors: K2 (2 B/elem)
    st = torch.zeros(_lib.state_bytes(len(P)), dtype=torch.uint8, device="cuda")
    _lib.check(lib.lomo_state_init(st.data_ptr(), len(P), 1024.0, 16, 1.0, 2.0 ** 24, 1.0, 1.0,
                                   stream), "init")
    pdisp = HookDispatcher(lib, st.data_ptr(), _lib.MATH_F32)
    pdisp.configure(flags=_lib.USE_SCALE, chain=True)  # K2s after the first chained
    pdun = HookDispatcher(lib, st.data_ptr(), _lib.MATH_F32)
    pdun.configure(flags=_lib.USE_SCALE)               # the hook pattern

    def probe_pass(s=stream, d=pdisp):
        lib.lomo_begin_step(st.data_ptr(), None, 0, s)
        for i in range(len(G) - 1, -1, -1):
            d.probe(G[i], dt_code, len(G) - 1 - i, s)
        d.flush(s)
        lib.lomo_finalize_norm(st.data_ptr(), s)
    for _ in range(args.warmup):
        probe_pass()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    start.record()
    for _ in range(args.steps):
        probe_pass()
    end.record()
    host_probe_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    torch.cuda.synchronize()
    probe_ms = start.elapsed_time(end) / args.steps
    start.record()
    for _ in range(args.steps):
        probe_pass(d=pdun)
    end.record()
    torch.cuda.synchronize()
    probe_un_ms = start.elapsed_time(end) / args.steps
    # the same launches captured in a CUDA graph (as GraphedLOMOStep runs them):
    # removes the host launch cost, leaving the kernels' own time
    def graphed(fn):
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            fn(cap.cuda_stream)
        torch.cuda.current_stream().wait_stream(cap)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            g.replay()
        end.record()
        torch.cuda.synchronize()
        ms_ = start.elapsed_time(end) / args.steps
        del g
        return ms_
    probe_graph_ms = graphed(probe_pass)
    upd_graph_ms = graphed(lambda s: run_update_pass(disp, P, G, dt_code, s))
    probe = {"gbs": round(2 * elems / (probe_ms * 1e-3) / 1e9, 1), "ms_per_pass": round(probe_ms, 4),
             "graphed_gbs": round(2 * elems / (probe_graph_ms * 1e-3) / 1e9, 1),
             "unchained_gbs": round(2 * elems / (probe_un_ms * 1e-3) / 1e9, 1),
             "host_ms_per_pass": round(host_probe_ms, 3),
             "algorithmic_bytes_per_elem": 2,
             "what": "K2 sum-of-squares + overflow flag over every gradient (back to back, "
                     "K2s after the first chained; unchained_gbs: the hook pattern), + "
                     "begin/finalize (K3a)"}
    # the exact-arithmetic mode (f64 math, direct rounding) on the same pass
    d64 = HookDispatcher(lib, None, _lib.MATH_F64)
    d64.configure(lr=0.05, chain=True)
    for _ in range(2):
        run_update_pass(d64, P, G, dt_code, stream)
    torch.cuda.synchronize()
    start.record()
    for _ in range(args.steps):
        run_update_pass(d64, P, G, dt_code, stream)
    end.record()
    torch.cuda.synchronize()
    f64_ms = start.elapsed_time(end) / args.steps
    f64 = {"gbs": round(BYTES_PER_ELEM * elems / (f64_ms * 1e-3) / 1e9, 1),
           "ms_per_pass": round(f64_ms, 4)}
    # the pass-2 form of K1 in the two-pass protocol: every kernel reads
    # skip / 1/scale / clip coefficient / lr from the device state block
    # (stabilize.py:215-224), no host scalars
    _lib.check(lib.lomo_set_lr(st.data_ptr(), 0.05, stream), "lomo_set_lr")
    dfl = HookDispatcher(lib, st.data_ptr(), _lib.MATH_F32)
    dfl.configure(flags=_lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE,
                  chain=True)
    # (dun: the unchained dispatcher, timed after the headline above)
    for _ in range(2):
        run_update_pass(dfl, P, G, dt_code, stream)
    torch.cuda.synchronize()

    def pass_ms(d):
        start.record()
        for _ in range(args.steps):
            run_update_pass(d, P, G, dt_code, stream)
        end.record()
        torch.cuda.synchronize()
        return start.elapsed_time(end) / args.steps
    # A/B alternation with the flag-free form (same tensors, back to back), so
    # the comparison does not depend on the order of the bench's legs
    ab = {"state": [], "plain": [], "plain_unchained": []}
    for _ in range(2):
        ab["state"].append(pass_ms(dfl))
        ab["plain"].append(pass_ms(disp))
        ab["plain_unchained"].append(pass_ms(dun))
    fl_ms = min(ab["state"])
    un_ms = min(ab["plain_unchained"])
    flags_pass = {"gbs": round(BYTES_PER_ELEM * elems / (fl_ms * 1e-3) / 1e9, 1),
                  "ms_per_pass": round(fl_ms, 4),
                  "ab_ms": {k: [round(x, 4) for x in v] for k, v in ab.items()},
                  "vs_flag_free_ab": round(min(ab["plain"]) / fl_ms, 4),
                  "flags": "USE_SKIP|USE_SCALE|USE_COEF|LR_FROM_STATE (state block read per CTA)"}
    unchained = {"gbs": round(BYTES_PER_ELEM * elems / (un_head_ms * 1e-3) / 1e9, 1),
                 "ms_per_pass": round(un_head_ms, 4),
                 "timed": "right after the chained headline passes (same thermal state)",
                 "ab_later_ms": round(un_ms, 4),
                 "vs_chained_ab": round(min(ab["plain"]) / un_ms, 4),
                 "what": "the same pass with every K1 waiting for its predecessor before "
                         "its loads (griddepcontrol.wait first): the autograd-hook pattern, "
                         "where the gradient's producer runs just before each K1"}
    del P, G
    torch.cuda.empty_cache()
    # SURVEY 8(d) C2's fp16 + scaler variant: fp16 p and g (g scaled by 2^10),
    # pass 2's flags -- unscale, clip coefficient, skip, lr from the state
    fp16 = None
    if args.dtype == "bf16":
        P16, G16 = make_update_workload(rank, world, "fp16")
        for g in G16:
            g.mul_(1024.0)
        st16 = torch.zeros(_lib.state_bytes(len(P16)), dtype=torch.uint8, device="cuda")
        _lib.check(lib.lomo_state_init(st16.data_ptr(), len(P16), 1024.0, 16, 1.0, 2.0 ** 24,
                                       1.0, 1.0, stream), "init")
        _lib.check(lib.lomo_set_lr(st16.data_ptr(), 0.05, stream), "lomo_set_lr")
        d16 = HookDispatcher(lib, st16.data_ptr(), _lib.MATH_F32)
        d16.configure(flags=_lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE,
                      chain=True)
        for _ in range(2):
            run_update_pass(d16, P16, G16, _lib.F16, stream)
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            run_update_pass(d16, P16, G16, _lib.F16, stream)
        end.record()
        torch.cuda.synchronize()
        f16_ms = start.elapsed_time(end) / args.steps
        fp16 = {"gbs": round(BYTES_PER_ELEM * elems / (f16_ms * 1e-3) / 1e9, 1),
                "ms_per_pass": round(f16_ms, 4),
                "what": "fp16 parameters and gradients (scaled by 2^10), K1 with "
                        "USE_SKIP|USE_SCALE|USE_COEF|LR_FROM_STATE, chained"}
        del P16, G16, st16
        torch.cuda.empty_cache()
    return {"gbs": gbs, "ms": ms / args.steps, "probe": probe, "f64_math": f64,
            "flags_pass": flags_pass, "unchained": unchained, "fp16_scaled": fp16,
            "graphed_gbs": BYTES_PER_ELEM * elems / (upd_graph_ms * 1e-3) / 1e9,
            "host_ms": host_ms, "host_enqueue": host_enqueue,
            "elems_per_rank": elems, "total_elems": total_elems,
            "launches": launches, "clocks": clk.summary(), "kernel_gbs": achieved,
            "kernel_ms_per_step": ksum_ms / args.steps, "shapes": shapes}


def bench_k4_local(args, world_sim: int = 8):
    """K4 (reduce-scatter fused with the update / probe) on this one GPU with
    simulated peers: rank 0 of ``world_sim`` ranks, its slice of every
    LLaMA-7B bucket read from ``world_sim`` distinct local buffers (at N > 1
    they are the peers' buffers over NVLink).  The kernel's HBM roofline:
    (2W + 4) B/elem for the update, 2W for the probe (tools/k4_local.py)."""
    import ctypes

    import torch
    from paper_2306_09782_b200 import _lib
    lib = _lib.load()
    W = world_sim
    sizes, _ = _buckets_7b(W)
    gen = torch.Generator(device="cuda").manual_seed(3)
    shards, keep, tabs = [], [], []
    for n in sizes:
        S = n // W
        shards.append(torch.empty(S, dtype=torch.bfloat16, device="cuda").uniform_(
            -0.08, 0.08, generator=gen))
        bufs = [torch.empty(S, dtype=torch.bfloat16, device="cuda").normal_(0, 1e-3, generator=gen)
                for _ in range(W)]
        keep.append(bufs)
        tabs.append(torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda"))
    elems = sum(x.numel() for x in shards)
    st = torch.zeros(_lib.state_bytes(len(sizes)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.lomo_state_init(st.data_ptr(), len(sizes), 0.0, 16, 1.0, 2.0 ** 24, 0.0, 1.0,
                                   s), "init")

    def upd():
        for k in range(len(shards) - 1, -1, -1):
            _lib.check(lib.lomo_fused_rs_update(
                shards[k].data_ptr(), ctypes.c_void_p(tabs[k].data_ptr()), W, 0,
                shards[k].numel(), _lib.BF16, _lib.MATH_F32, 0.05, 0.0, 0.0, 0, None, s),
                "rs_update")

    def prb():
        lib.lomo_begin_step(st.data_ptr(), None, 0, s)
        for k in range(len(shards) - 1, -1, -1):
            _lib.check(lib.lomo_fused_rs_probe(ctypes.c_void_p(tabs[k].data_ptr()), W, 0,
                                               shards[k].numel(), _lib.BF16, k, 0,
                                               st.data_ptr(), s), "rs_probe")

    kept = torch.empty(max(x.numel() for x in shards), dtype=torch.bfloat16, device="cuda")

    def prb_keep():
        lib.lomo_begin_step(st.data_ptr(), None, 0, s)
        for k in range(len(shards) - 1, -1, -1):
            _lib.check(lib.lomo_fused_rs_probe_keep(ctypes.c_void_p(tabs[k].data_ptr()), W, 0,
                                                    shards[k].numel(), _lib.BF16, k, 0,
                                                    st.data_ptr(), kept.data_ptr(), s),
                       "rs_probe_keep")

    peak, _ = _peaks()
    out = {"world_simulated": W, "buckets": len(sizes), "shard_elements": elems,
           "what": "rank 0's K4 over its 1/W slice of every LLaMA-7B bucket, the W peer "
                   "buffers local (HBM in place of NVLink): the kernel's own roofline"}
    for name, fn, bpe in (("update", upd, 2 * W + 4), ("probe", prb, 2 * W),
                          ("probe_keep", prb_keep, 2 * W + 2)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        gbs = bpe * elems / (ms * 1e-3) / 1e9
        out[name] = {"ms_per_pass": round(ms, 4), "gbs": round(gbs, 1),
                     "algorithmic_bytes_per_elem": bpe, "frac": round(gbs / peak, 4)}
    del keep, tabs, shards, kept
    torch.cuda.empty_cache()
    return out


def _buckets_7b(world: int, layers: int = 32):
    """ShardedLOMO's buckets of LLaMA-7B: one per decoder layer (its 9
    tensors) plus the embedding / final norm / head, each padded to a multiple
    of 8 * world elements; delivery order = reverse registration.  ``layers``
    < 32 keeps only the first layers (validation dry runs only)."""
    from paper_2306_09782_b200.workloads import llama_param_shapes
    groups: dict = {}
    for name, shape in llama_param_shapes("7b"):
        key = name.split(".")[1] if name.startswith("layers.") else "rest"
        if key != "rest" and int(key) >= layers:
            continue
        groups[key] = groups.get(key, 0) + math.prod(shape)
    sizes = [groups[k] for k in groups]
    align = 8 * world
    return [int(math.ceil(n / align) * align) for n in sizes], sum(sizes)


def bench_sharded_update(args, rank, world):
    """N > 1 headline: one sharded LOMO update pass of LLaMA-7B over the
    ranks.  Every rank holds the full flat gradient buckets of
    its own backward (33 buckets, 13.5 GB bf16, different data per rank);
    per bucket, in delivery order:

      nccl  reduce_scatter_tensor (SUM, NCCL over NVLink) -> K1 on this
            rank's 1/W shard (inv_scale = 1/W: the data-parallel mean), the
            K1 of bucket b enqueued once bucket b-1's collective is issued
            (ShardedLOMO._reduce/_drain);
      k4    the buckets live in peer-mapped buffers (peer.PeerRing: NVLS
            multicast when available, else CUDA IPC); a device barrier, then
            ONE kernel reduces this rank's slice over all ranks' buffers and
            applies the update -- the reduced gradient never reaches HBM.

    value = algorithmic update bytes of the whole job (6 B/param: the 7B
    update, split 1/W per rank) / max-over-ranks time: strong scaling, the
    total work is one 7B update.  Reported beside it: per-rank GB/s, the
    NVLink bytes each rank moves (its gradient's (W-1)/W, out and in), and
    K1's own roofline on the shard."""
    import torch
    import torch.distributed as dist
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.engine import CudaEngine
    from paper_2306_09782_b200.peer import PeerRing
    from paper_2306_09782_b200.sharded import _pick_transport, reduce_scatter
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    sizes, P = _buckets_7b(world, args.update_layers)
    nb = len(sizes)
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    G = [torch.empty(n, dtype=dt, device=dev).normal_(0.0, 1e-3, generator=gen) for n in sizes]
    W = [torch.empty(n // world, dtype=dt, device=dev).uniform_(-0.08, 0.08, generator=gen)
         for n in sizes]
    GS = [torch.empty(n // world, dtype=dt, device=dev) for n in sizes]
    eng = CudaEngine(dev, nb, None, None, "f32", grad_div=float(world))
    eng.configure(lr=0.05, flags=_lib.USE_SCALE)
    order = list(range(nb - 1, -1, -1))
    # gloo (LOMO_BENCH_SHARE_GPU dry run) cannot overlap; NCCL runs async
    async_ok = dist.get_backend() == "nccl"

    def nccl_pass(events=None):
        inflight = []
        for b in order:
            work = reduce_scatter(GS[b], G[b], None, async_op=async_ok)
            inflight.append((work, b))
            if len(inflight) > 1:  # K1 of the previous bucket once this one's RS is issued
                w_, b_ = inflight.pop(0)
                _k1(w_, b_, events)
        while inflight:
            w_, b_ = inflight.pop(0)
            _k1(w_, b_, events)

    def _k1(work, b, events):
        if work is not None:
            work.wait()
        if events is not None:
            events[b][0].record()
        eng.update(W[b], GS[b])
        if events is not None:
            events[b][1].record()

    def timed(fn, steps):
        _barrier(world)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(steps):
            fn()
        s1.record()
        _barrier(world)
        return _max_over_ranks(s0.elapsed_time(s1) / steps, world)

    out = {}
    for _ in range(args.warmup):
        nccl_pass()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms_nccl = timed(nccl_pass, args.steps)
    launches = args.steps * nb
    # K1's own time on the shards (per-launch events, a separate pass)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(nb)]
    nccl_pass(ev)
    torch.cuda.synchronize()
    k1_ms = sum(a.elapsed_time(b) for a, b in ev)
    k1_gbs = BYTES_PER_ELEM * (P / world) / (k1_ms * 1e-3) / 1e9
    link_bytes = 2 * P * (world - 1) / world  # this rank's gradient bytes leaving (and entering)
    out["nccl"] = {"ms_per_pass": round(ms_nccl, 3),
                   "gbs": round(BYTES_PER_ELEM * P / (ms_nccl * 1e-3) / 1e9, 1),
                   "per_rank_gbs": round(BYTES_PER_ELEM * P / world / (ms_nccl * 1e-3) / 1e9, 1),
                   "nvlink_gbs_per_rank": round(link_bytes / (ms_nccl * 1e-3) / 1e9, 1),
                   "k1_ms_per_pass": round(k1_ms, 3), "k1_gbs": round(k1_gbs, 1),
                   "collective": "reduce_scatter_tensor " + dist.get_backend(),
                   "clocks": clk.summary()}
    del GS
    # ---- K4 over peer-mapped buffers (every bucket resident, as the backward left it)
    try:
        transport = args.k4_transport or _pick_transport(True, dev, None)
        ring = PeerRing(max(sizes), dt, dev, None, transport, err_ptr=eng.error_ptr,
                        timeout_s=60.0, nbuf=nb)
        for b in range(nb):
            ring.bufs[b][:sizes[b]].copy_(G[b])
        del G
        torch.cuda.empty_cache()

        def k4_pass():
            for b in order:
                ring.filled(b)  # every rank's bucket b is written
                ring.update(eng, W[b], b, rank * (sizes[b] // world))
        for _ in range(args.warmup):
            k4_pass()
        eng.read_status()  # a barrier timeout would raise here
        ms_k4 = timed(k4_pass, args.steps)
        eng.read_status()
        out["k4"] = {"ms_per_pass": round(ms_k4, 3),
                     "gbs": round(BYTES_PER_ELEM * P / (ms_k4 * 1e-3) / 1e9, 1),
                     "per_rank_gbs": round(BYTES_PER_ELEM * P / world / (ms_k4 * 1e-3) / 1e9, 1),
                     "nvlink_gbs_per_rank": round(link_bytes / (ms_k4 * 1e-3) / 1e9, 1),
                     "transport": transport,
                     "kernel": "lomo_fused_mc_update (multimem.ld_reduce)" if transport == "nvls"
                               else "lomo_fused_rs_update (P2P loads, rank-order sum)"}
        launches = max(launches, args.steps * nb * 2)
        ring.close()
    except Exception as exc:  # noqa: BLE001
        import traceback
        traceback.print_exc()
        out["k4"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    best = "k4" if out["k4"].get("gbs", 0) > out["nccl"]["gbs"] else "nccl"
    out.update({"best": best, "ms": out[best]["ms_per_pass"], "gbs": out[best]["gbs"],
                "elements": P, "buckets": nb, "nvlink_bytes_per_rank": int(link_bytes),
                "launches": launches, "clocks": out["nccl"]["clocks"],
                "k1_gbs": k1_gbs})
    return out


def _sum_over_ranks(x: int, world: int) -> int:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.int64, device="cuda")
    dist.all_reduce(t)
    return int(t.item())


def bench_e2e(args, rank, world):
    """The same pass through the C-ABI with host buffers: per tensor, pinned
    H2D of p and g, K1, D2H of p -- all in the timed region, pipelined over
    two copy streams and the compute stream."""
    import torch
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.workloads import llama_param_shapes
    lib = _lib.load()
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    # (e2e stages every tensor through device slots, one K1 launch each)
    dt_code = _lib.BF16 if args.dtype == "bf16" else _lib.F16
    shapes = [math.prod(shape) for _, shape in llama_param_shapes("7b")]
    # device staging: NS slots per operand (H2D of tensor i+1.. overlaps K1 / D2H of i)
    maxn = max(shapes)
    NS = args.e2e_slots
    DP = [torch.empty(maxn, dtype=dt, device="cuda") for _ in range(NS)]
    DG = [torch.empty(maxn, dtype=dt, device="cuda") for _ in range(NS)]
    # host buffers (pinned), filled once (generated on the device, copied down)
    gen = torch.Generator(device="cuda").manual_seed(7 + rank)
    HP, HG = [], []
    for n in shapes:
        hp = torch.empty(n, dtype=dt, pin_memory=True)
        hg = torch.empty(n, dtype=dt, pin_memory=True)
        hp.copy_(DP[0][:n].uniform_(-0.08, 0.08, generator=gen))
        hg.copy_(DG[0][:n].normal_(0.0, 1e-3, generator=gen))
        HP.append(hp)
        HG.append(hg)
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.current_stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(NS)]
    ev_done = [torch.cuda.Event() for _ in range(NS)]
    ev_out = [torch.cuda.Event() for _ in range(NS)]
    order = list(range(len(shapes) - 1, -1, -1))

    def one_pass(compute=True):
        for k, i in enumerate(order):
            s = k % NS
            n = shapes[i]
            with torch.cuda.stream(h2d):
                h2d.wait_event(ev_out[s])  # slot free (its D2H finished)
                DP[s][:n].copy_(HP[i], non_blocking=True)
                DG[s][:n].copy_(HG[i], non_blocking=True)
                ev_in[s].record(h2d)
            comp.wait_event(ev_in[s])
            rc = lib.lomo_fused_update(DP[s].data_ptr(), DG[s].data_ptr(), n, dt_code,
                                       _lib.MATH_F32, 0.05, 0.0, 0.0, 0, None,
                                       comp.cuda_stream) if compute else 0
            if rc:
                raise RuntimeError(f"rc={rc}")
            ev_done[s].record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_done[s])
                HP[i].copy_(DP[s][:n], non_blocking=True)
                ev_out[s].record(d2h)
        comp.wait_stream(d2h)

    for _ in range(max(1, min(args.warmup, 2))):
        one_pass()
    _barrier(world)
    steps = max(1, min(args.steps, 5))
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        one_pass()
    end.record()
    _barrier(world)
    ms = _max_over_ranks(start.elapsed_time(end), world) / steps
    # the link bounds: (a) the same step's H2D copies alone (p and g of every
    # tensor into the slots, one copy stream); (b) the same pipeline with every
    # copy in both directions but no K1 -- PCIe carries H2D and D2H at once at
    # less than twice the one-way rate, so (b) is the bound e2e can reach
    with torch.cuda.stream(h2d):
        h2d.wait_stream(comp)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(h2d)
        for k, i in enumerate(order):
            s = k % NS
            DP[s][:shapes[i]].copy_(HP[i], non_blocking=True)
            DG[s][:shapes[i]].copy_(HG[i], non_blocking=True)
        s1.record(h2d)
    s1.synchronize()
    h2d_ms = s0.elapsed_time(s1)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(2):
        one_pass(compute=False)
    c1.record()
    c1.synchronize()
    copy_ms = c0.elapsed_time(c1) / 2
    elems = _sum_over_ranks(sum(shapes), world)
    esz = 2
    return {"value": round(BYTES_PER_ELEM * elems / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": 2 * esz * sum(shapes), "d2h_bytes_per_step": esz * sum(shapes),
            "ms_per_step": round(ms, 2), "steps": steps,
            "h2d_only_ms_per_step": round(h2d_ms, 2),
            "h2d_link_gbs": round(2 * esz * sum(shapes) / (h2d_ms * 1e-3) / 1e9, 2),
            "copies_only_ms_per_step": round(copy_ms, 2),
            "link_bound_frac": round(copy_ms / ms, 3),
            "link_bound": "the same H2D/D2H pipeline without K1 (bidirectional PCIe)",
            "path": "C-ABI lomo_fused_update, pinned host p/g -> HBM -> K1 -> host p"}


def bench_e2e_sharded(args, rank, world):
    """N > 1 e2e: the sharded update pass with HOST buffers.  Per bucket (delivery
    order): H2D of this rank's gradient bucket and of its parameter shard
    (pinned), NCCL reduce_scatter, K1 on the shard through the C-ABI, D2H of
    the updated shard -- all inside the timed region, pipelined over NS
    device slots and two copy streams.  The gradient host buffers cycle
    through NS pinned buckets (the bytes copied per step are the full 2P)."""
    import torch
    import torch.distributed as dist
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.engine import CudaEngine
    from paper_2306_09782_b200.sharded import reduce_scatter
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    sizes, P = _buckets_7b(world, args.update_layers)
    nb, NS = len(sizes), max(2, args.e2e_slots)
    mx = max(sizes)
    gen = torch.Generator(device="cuda").manual_seed(77 + rank)
    DG = [torch.empty(mx, dtype=dt, device=dev) for _ in range(NS)]
    DW = [torch.empty(mx // world, dtype=dt, device=dev) for _ in range(NS)]
    DS = [torch.empty(mx // world, dtype=dt, device=dev) for _ in range(NS)]
    HG = [torch.empty(mx, dtype=dt, pin_memory=True) for _ in range(NS)]
    for h in HG:
        h.copy_(DG[0].normal_(0.0, 1e-3, generator=gen))
    HW = [torch.empty(n // world, dtype=dt, pin_memory=True) for n in sizes]
    for h in HW:
        h.copy_(DW[0][:h.numel()].uniform_(-0.08, 0.08, generator=gen))
    eng = CudaEngine(dev, nb, None, None, "f32", grad_div=float(world))
    eng.configure(lr=0.05, flags=_lib.USE_SCALE)
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.current_stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(NS)]
    ev_done = [torch.cuda.Event() for _ in range(NS)]
    ev_out = [torch.cuda.Event() for _ in range(NS)]
    order = list(range(nb - 1, -1, -1))
    async_ok = dist.get_backend() == "nccl"

    def one_pass():
        for k, b in enumerate(order):
            s, n, S = k % NS, sizes[b], sizes[b] // world
            with torch.cuda.stream(h2d):
                h2d.wait_event(ev_out[s])
                DG[s][:n].copy_(HG[k % NS][:n], non_blocking=True)
                DW[s][:S].copy_(HW[b], non_blocking=True)
                ev_in[s].record(h2d)
            comp.wait_event(ev_in[s])
            work = reduce_scatter(DS[s][:S], DG[s][:n], None, async_op=async_ok)
            if work is not None:
                work.wait()
            eng.update(DW[s][:S], DS[s][:S])
            ev_done[s].record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_done[s])
                HW[b].copy_(DW[s][:S], non_blocking=True)
                ev_out[s].record(d2h)
        comp.wait_stream(d2h)

    for _ in range(max(1, min(args.warmup, 2))):
        one_pass()
    _barrier(world)
    steps = max(1, min(args.steps, 5))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(steps):
        one_pass()
    s1.record()
    _barrier(world)
    ms = _max_over_ranks(s0.elapsed_time(s1), world) / steps
    esz = 2
    return {"value": round(BYTES_PER_ELEM * P / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": esz * (sum(sizes) + sum(sizes) // world),
            "d2h_bytes_per_step": esz * sum(sizes) // world,
            "ms_per_step": round(ms, 2), "steps": steps,
            "path": "pinned host gradient bucket + parameter shard -> HBM -> NCCL "
                    "reduce_scatter -> K1 (C-ABI lomo_fused_update) -> host shard"}


def _lib_state_mib(nslots: int) -> float:
    from paper_2306_09782_b200 import _lib
    return _lib.state_bytes(nslots) / 2 ** 20


def _bf16_peak_tflops() -> tuple[float, str]:
    """Dense bf16 peak for a kernel inside a long step: MEASURED_PEAKS.json's
    sustained (power-capped) figure when the driver wrote it, else the
    B200_PROFILING.md fallback (1.59 PFLOP/s, an isolated-kernel number)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            for k in ("bf16_tflops_sustained", "bf16_tflops"):
                if d.get(k):
                    return float(d[k]), f"MEASURED_PEAKS.json {k}"
        except Exception:
            pass
    return 1590.0, "fallback 1.59 PF/s (B200_PROFILING.md, isolated kernel at max clock)"


_GRAPHED = ("replay_fused_gemm_graph", "strict_fused_gemm_graph", "single_pass_fused_gemm_graph",
            "grouped_fused_gemm_graph", "strict_graph", "replay_graph")


_TWO_PASS = ("strict", "strict_graph", "strict_fused_gemm", "strict_fused_gemm_graph", "replay",
             "replay_graph", "replay_fused_gemm", "replay_fused_gemm_graph")
TRAIN_HEADLINE = "replay_fused_gemm_graph"
TRAIN_DEFAULT = ("strict", "strict_fused_gemm_graph", TRAIN_HEADLINE, "grouped_fused_gemm_graph",
                 "single_pass_fused_gemm_graph")


def bench_train(args, rank, world):
    """Config 3: LLaMA-7B fp16 LOMO, dynamic loss scale + two-pass clip.

    Every variant trains a FRESH model (same seed, same batches), so the
    losses and outcomes of the variants are comparable.  The headline is the
    fixed variant ``replay_fused_gemm_graph`` timed over ``--train-steps-
    headline`` steps (default 30); ``strict`` -- the reference protocol as is
    (pass 2 = a second backward over the retained graph, hook kernels K2/K1,
    one gradient alive) -- is reported beside it, as are the other variants
    (``--train-variants`` selects; each ``--train-steps`` steps):
    ``strict_fused_gemm[_graph]`` -- the same protocol with each linear's probe
    (K6, pass 1) and update (K5, pass 2) inside its weight-gradient GEMM;
    ``replay*`` -- pass 2 recomputes each weight gradient from the (input,
    output-gradient) pairs stashed in pass 1 (replay.py) instead of a second
    backward; ``*_graph`` -- the step captured as two CUDA graphs around the
    one host decision (graphs.py); ``grouped*`` -- the paper's single-pass
    per-layer clip (GroupedLOMO); ``single_pass*`` -- LOMO's single fused
    pass, no clip and no scaler.  Afterwards the paper's Table-1 LOMO row is
    MEASURED on a fresh model (``table1``)."""
    import torch
    from paper_2306_09782_b200 import LOMO, GroupedLOMO, LossScaler
    from paper_2306_09782_b200.workloads import Llama
    size = args.train_model
    ckpt = args.ckpt or size == "65b"
    seq, batch = args.seq, args.batch

    def build():
        torch.cuda.empty_cache()
        m = Llama(size, dtype=torch.float16, device="cuda", checkpointing=ckpt,
                  fused_proj=not args.separate_proj, seed=0)
        m.train()
        return m

    gen = torch.Generator(device="cuda").manual_seed(0)
    data = [torch.randint(0, 32000, (batch, seq + 1), device="cuda", generator=gen)
            for _ in range(4)]
    out = {"model": f"llama-{size} (random init N(0,0.02), a fresh model per variant), fp16 "
                    "params, no master copy",
           "projections": "separate q/k/v, gate/up" if args.separate_proj else
           "stacked qkv [3h,h] and gate_up [2f,h] weights (same parameters and math)",
           "seq_len": seq, "batch": batch, "passes_per_step": 2,
           "clip_grad_norm": 1.0, "loss_scale": "dynamic, 2^10, growth 16",
           "activation_checkpointing": bool(ckpt), "paper_tgs_rtx3090": 769.92,
           "headline_variant": TRAIN_HEADLINE}
    variants = tuple(args.train_variants.split(",")) if args.train_variants else TRAIN_DEFAULT
    for key in variants:
        model = build()
        gstep = None
        if key in _GRAPHED:
            from paper_2306_09782_b200.graphs import GraphedGroupedStep, GraphedLOMOStep
            if key.startswith("grouped"):
                opt = GroupedLOMO(model, lr=1e-3, max_norm=1.0, window=1, fuse_gemm=True)
            elif key.startswith("single"):
                opt = LOMO(model, lr=1e-3, fuse_gemm=True)
            else:
                opt = LOMO(model, lr=1e-3, clip_grad_norm=1.0,
                           loss_scale=LossScaler(2.0 ** 10, growth_interval=16),
                           replay=key.startswith("replay"), fuse_gemm="fused_gemm" in key)
            static = data[0].clone()
            G = GraphedGroupedStep if key.startswith("grouped") else GraphedLOMOStep
            gstep = G(opt, lambda d, m=model: m.loss(d[:, :-1], d[:, 1:]), (static,),
                      warmup=max(2, args.train_warmup), lr=1e-3)

            def step(k, gstep=gstep, static=static):
                static.copy_(data[k % len(data)])
                # the loss stays on the device until the timed loop ends: the
                # graphed step's one host sync is its status read
                return gstep.step(1e-3).detach().clone()
        else:
            if key == "single_pass_fused_gemm":
                opt = LOMO(model, lr=1e-3, fuse_gemm=True)
            elif key in ("grouped", "grouped_fused_gemm"):
                opt = GroupedLOMO(model, lr=1e-3, max_norm=1.0, window=1,
                                  fuse_gemm=key == "grouped_fused_gemm")
            else:
                opt = LOMO(model, lr=1e-3, clip_grad_norm=1.0,
                           loss_scale=LossScaler(2.0 ** 10, growth_interval=16),
                           replay=key.startswith("replay"),
                           fuse_gemm=key in ("replay_fused_gemm", "strict_fused_gemm"))

            def step(k, opt=opt, model=model):
                d = data[k % len(data)]
                return opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)
        nsteps = args.train_steps_headline if key == TRAIN_HEADLINE else args.train_steps
        for k in range(args.train_warmup):
            step(k)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        losses, outcomes = [], []
        with ClockSampler(torch.cuda.current_device()) as clk:
            start.record()
            for k in range(nsteps):
                losses.append(step(args.train_warmup + k))
                outcomes.append(opt.last_outcome.value if opt.last_outcome else "applied")
            end.record()
            torch.cuda.synchronize()
        ms = start.elapsed_time(end) / nsteps
        losses = [float(x) for x in losses]
        out[key] = {"tokens_per_s": round(batch * seq / (ms * 1e-3), 1), "ms_per_step": round(ms, 2),
                    "steps": nsteps, "warmup": args.train_warmup,
                    "peak_mem_gib": round(torch.cuda.max_memory_allocated() / 2 ** 30, 2),
                    "loss_scale_final": getattr(opt, "loss_scale", None), "outcomes": outcomes,
                    "losses": [round(x, 4) for x in losses], "clocks": clk.summary()}
        pw = out[key]["clocks"].get("power_w")
        if pw:
            out[key]["tokens_per_joule"] = round(out[key]["tokens_per_s"] / pw, 2)
        opt.remove_hooks()
        del opt, step, gstep, model
        torch.cuda.empty_cache()
    hv_key = TRAIN_HEADLINE if TRAIN_HEADLINE in out else next(
        (k for k in variants if k in _TWO_PASS), variants[0])
    out["headline_variant"] = hv_key
    out["tokens_per_s"] = out[hv_key]["tokens_per_s"]
    out["ms_per_step"] = out[hv_key]["ms_per_step"]
    if "strict" in out:
        out["strict_tokens_per_s"] = out["strict"]["tokens_per_s"]
    # tensor work of the headline step (two-pass replay protocol): forward,
    # input-gradient, pass-1 weight-gradient (K6) and pass-2 weight-gradient
    # (K5) GEMMs over every linear, plus causal attention (fwd + ~2.5x bwd);
    # against the bf16 peak scaled to the median SM clock the leg ran at
    from paper_2306_09782_b200.workloads import LLAMA, llama_param_shapes
    cfg = LLAMA[size]
    tokens = batch * seq
    lin = sum(math.prod(s) for n, s in llama_param_shapes(size) if len(s) == 2
              and "embed" not in n)
    attn = 3.5 * 2 * 2 * tokens * seq * 0.5 * cfg["hidden"] * cfg["layers"]
    tflop = (4 * 2 * tokens * lin + attn) / 1e12
    hv = out[hv_key]
    pflops = tflop / (hv["ms_per_step"] * 1e-3) / 1e3
    peak_tf, peak_src = _bf16_peak_tflops()
    peak_pf = peak_tf / 1e3
    clk = hv.get("clocks", {})
    scale = (clk.get("sm_mhz") or 0) / (clk.get("sm_max_mhz") or 1) if clk.get("sm_mhz") else None
    sustained = "sustained" in peak_src
    out["tensor_roofline"] = {
        "tflop_per_step": round(tflop, 2), "achieved_pflops": round(pflops, 3),
        "peak_pflops": round(peak_pf, 3), "peak_source": peak_src,
        "frac": round(pflops / peak_pf, 3),
        "frac_at_run_clock": (round(pflops / (peak_pf * scale), 3)
                              if scale and not sustained else None)}
    if size == "7b" and not args.no_table1:
        out["table1"] = measure_table1(args, build)
    torch.cuda.empty_cache()
    return out


def measure_table1(args, build):
    """the paper's Table 1 LOMO row (LLaMA-7B, fp16, seq 512 x
    batch 8), MEASURED on the plain LOMO hook path, beside
    the reference estimator's row (fusedtrain/estimate.py:200-218, imported
    from baseline/_ref) for the same setting, with and without per-layer
    activation checkpointing.

      params      torch.cuda.memory_allocated() delta of building the model
      gradients   the largest total of live .grad tensors over every hook
                  call of a step (an instrumentation hook runs before LOMO's
                  and sums the gradients alive at that moment), and the most
                  gradient tensors ever alive at once
      optimizer   LOMO's per-parameter state (none) and its one state block
      step peak   max_memory_allocated() of one step minus what was
                  allocated before the model existed"""
    import torch
    from paper_2306_09782_b200 import LOMO, LossScaler
    seq, batch = 512, 8
    ref, where = _import_reference()
    gib = 2 ** 30
    rows = {}
    for ac in (True, False):
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        before = torch.cuda.memory_allocated()
        model = build()
        params_b = torch.cuda.memory_allocated() - before
        model.checkpointing = ac
        plist = list(model.parameters())
        live = {"bytes": 0, "count": 0, "largest": 0}

        def watch(p, plist=plist, live=live):
            b = c = 0
            for q in plist:
                if q.grad is not None:
                    b += q.grad.numel() * q.grad.element_size()
                    c += 1
            live["bytes"] = max(live["bytes"], b)
            live["count"] = max(live["count"], c)
            live["largest"] = max(live["largest"], p.grad.numel() * p.grad.element_size())
        hs = [p.register_post_accumulate_grad_hook(watch) for p in plist]  # before LOMO's
        opt = LOMO(model, lr=1e-3, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10))
        d = torch.randint(0, 32000, (batch, seq + 1), device="cuda",
                          generator=torch.Generator(device="cuda").manual_seed(5))
        opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)  # warm (allocator, kernels)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        live.update(bytes=0, count=0, largest=0)
        opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - before
        row = {"params_gib": round(params_b / gib, 3),
               "gradients_live_max_gib": round(live["bytes"] / gib, 3),
               "gradient_tensors_live_max": live["count"],
               "largest_gradient_gib": round(live["largest"] / gib, 3),
               "optimizer_state_per_param_bytes": 0,
               "optimizer_state_block_gib": round(opt.engine.state.numel() / gib, 4),
               "step_peak_gib": round(peak / gib, 2),
               "outcome": opt.last_outcome.value if opt.last_outcome else None}
        opt.remove_hooks()
        for h in hs:
            h.remove()
        del opt, model, plist
        if ref is not None:
            E = ref["estimate"]
            est = E.estimate(E.PRESETS["llama-7b"], E.TrainSetup(
                ref["optim"].OptimizerKind.LOMO, E.EstimatePrecision.MIXED16, ac, seq, batch))
            row["reference_estimator_gib"] = {
                "params": round(est.params_gib, 2), "gradients": round(est.gradients_gib, 2),
                "optim_states": round(est.optim_states_gib, 2),
                "activations": round(est.activations_gib, 2), "total": round(est.total_gib, 2),
                "source": f"fusedtrain.estimate.estimate ({where}), estimate.py:200-218"}
        rows["ac" if ac else "no_ac"] = row
    rows["paper_table1_lomo"] = {"params": 12.55, "gradients": 0.24, "optimizer_states": 0.0,
                                 "total_ac": 14.58, "source": "PAPER.md:193-196"}
    rows["setting"] = f"LLaMA-7B fp16, seq {seq} x batch {batch}, LOMO two-pass (clip 1.0, scale 2^10)"
    rows["note"] = ("activations: SDPA flash attention keeps no score matrix; the estimator "
                    "charges 4 width-equivalents per score element")
    torch.cuda.empty_cache()
    return rows


def bench_train_sharded(args, rank, world):
    """Configs 4/5: LLaMA-13B (or 65B with per-layer activation checkpointing)
    with ZeRO-3 parameter shards over ``world`` GPUs; each bucket's gradients
    are reduce-scattered with NCCL and each rank runs the fused update on its
    shard (ShardedLOMO).  Every rank trains on its own seq x batch tokens, so
    tokens/s is the whole-job sum."""
    import torch
    from paper_2306_09782_b200 import LossScaler
    from paper_2306_09782_b200.sharded import ShardedLOMO
    from paper_2306_09782_b200.workloads import Llama
    size = args.sharded_model
    ckpt = args.ckpt or size == "65b"
    spec = dict(hidden=512, layers=4, heads=8, ffn=1408, vocab=32000) if size == "tiny" else size
    model = Llama(spec, dtype=torch.float16, device="cuda", checkpointing=ckpt,
                  fused_proj=not args.separate_proj)
    model.train()
    # 180 GB per GPU: when the gathered model takes under 40 % of HBM, the layer
    # buckets stay gathered between forward and backward (parameters are still
    # owned and updated per shard, and re-gathered once per applied step);
    # otherwise (65B) ZeRO-3 frees each layer after its forward and re-gathers it
    pbytes = sum(p.numel() * p.element_size() for p in model.parameters())
    hbm = torch.cuda.get_device_properties(0).total_memory
    # (at world 1 a ZeRO-3 shard is the whole model: freeing the gathered
    # layers saves nothing and costs a gather per use, so never reshard)
    reshard = world > 1 and pbytes > 0.4 * hbm
    # pass 2: K1 over pass 1's reduced gradient shards when 1/world of the
    # gradients fits in 15 % of HBM, else replay of the stashed (x, dy)
    keep = not args.sharded_strict and pbytes / world < 0.15 * hbm
    opt = ShardedLOMO(model, lr=1e-3, clip_grad_norm=1.0,
                      loss_scale=LossScaler(2.0 ** 10, growth_interval=16),
                      reshard_after_forward=reshard,
                      replay=not args.sharded_strict and not keep, keep_grads=keep,
                      fused_rs=args.sharded_fused_rs or False)
    torch.cuda.empty_cache()
    seq, batch = args.seq, args.batch
    gen = torch.Generator(device="cuda").manual_seed(rank)
    data = [torch.randint(0, 32000, (batch, seq + 1), device="cuda", generator=gen)
            for _ in range(4)]

    def step(k):
        d = data[k % len(data)]
        return opt.step(lambda: model.loss(d[:, :-1], d[:, 1:]), 1e-3)

    for k in range(args.train_warmup):
        step(k)
    _barrier(world)
    torch.cuda.reset_peak_memory_stats()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outcomes = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        start.record()
        for k in range(args.train_steps):
            step(k)
            outcomes.append(opt.last_outcome.value)
        end.record()
        _barrier(world)
    ms = _max_over_ranks(start.elapsed_time(end), world) / args.train_steps
    eager_peak = torch.cuda.max_memory_allocated()
    graphed = None
    import torch.distributed as dist
    # the graphed form: at world 1 by default; at N > 1 only with --sharded-graph
    # (multi-rank NCCL capture has not run on a multi-GPU box yet, and a hung
    # capture would cost the whole line)
    if not reshard and not args.sharded_strict and not args.no_sharded_graph and \
            (world == 1 or args.sharded_graph) and \
            dist.get_backend() == "nccl":  # (not the gloo LOMO_BENCH_SHARE_GPU dry run)
        graphed = _graphed_sharded(args, opt, model, data, world)
    out = {"model": f"llama-{size} (random init), fp16, parameters sharded over {world} GPUs "
                    f"({'ZeRO-3: layers freed after use' if reshard else 'layers kept gathered'})"
                    + ("" if args.separate_proj else "; stacked qkv / gate_up weights"),
           "tokens_per_s": round(world * batch * seq / (ms * 1e-3), 1),
           "tokens_per_gpu_per_s": round(batch * seq / (ms * 1e-3), 1),
           "ms_per_step": round(ms, 2), "seq_len": seq, "batch_per_rank": batch,
           "activation_checkpointing": ckpt, "passes_per_step": 2, "outcomes": outcomes,
           "reshard_after_forward": reshard, "clocks": clk.summary(),
           "reduction": f"K4 over {opt.transport}" if opt.fused_rs else "NCCL reduce_scatter",
           "tensor_roofline": _sharded_roofline(model, batch, seq, ms, keep,
                                                args.sharded_strict, ckpt, clk.summary()),
           "pass2": "second forward + backward" if args.sharded_strict else
                    (f"K1 over pass 1's reduced gradient shards ({pbytes / world / 2**30:.1f} GiB "
                     "kept per rank)" if keep else "replay of the stashed (x, dy) into the buckets"),
           "peak_mem_gib_rank0": round(eager_peak / 2 ** 30, 2),
           "paper_tgs_rtx3090": {"13b": 66.19, "30b": 11.61, "65b": 4.93}.get(size)}
    if graphed is not None:
        out["graphed"] = graphed
        if "tokens_per_s" in graphed:
            out["eager_tokens_per_s"] = out["tokens_per_s"]
            if graphed["tokens_per_s"] > out["tokens_per_s"]:
                out["tokens_per_s"] = graphed["tokens_per_s"]
                out["tokens_per_gpu_per_s"] = graphed["tokens_per_gpu_per_s"]
                out["ms_per_step"] = graphed["ms_per_step"]
                out["headline_variant"] = "graphed (GraphedShardedStep)"
                out["tensor_roofline"] = _sharded_roofline(model, batch, seq, graphed["ms_per_step"],
                                                           keep, False, ckpt, graphed["clocks"])
            else:
                out["headline_variant"] = "eager"
    opt.remove_hooks()
    del opt, model
    torch.cuda.empty_cache()
    return out


def _graphed_sharded(args, opt, model, data, world):
    """The same ShardedLOMO step captured as two CUDA graphs
    (``GraphedShardedStep``: refresh all-gathers, reduce-scatters, K2/K3/K1
    and the rank exchange inside the graphs; the status read between them).
    Continues training the eager leg's model (throughput, not a fresh run)."""
    import torch
    from paper_2306_09782_b200.graphs import GraphedShardedStep
    try:
        torch.cuda.empty_cache()
        static = data[0].clone()
        gs = GraphedShardedStep(opt, lambda d: model.loss(d[:, :-1], d[:, 1:]), [static],
                                warmup=max(2, args.train_warmup), lr=1e-3)
        for k in range(2):
            static.copy_(data[k % len(data)])
            gs.step(1e-3)
        torch.cuda.synchronize()
        _barrier(world)
        torch.cuda.reset_peak_memory_stats()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        outcomes = []
        with ClockSampler(torch.cuda.current_device()) as clk:
            start.record()
            for k in range(args.train_steps):
                static.copy_(data[k % len(data)])
                gs.step(1e-3)
                outcomes.append(opt.last_outcome.value)
            end.record()
            _barrier(world)
        ms = _max_over_ranks(start.elapsed_time(end), world) / args.train_steps
        seq, batch = args.seq, args.batch
        res = {"tokens_per_s": round(world * batch * seq / (ms * 1e-3), 1),
               "tokens_per_gpu_per_s": round(batch * seq / (ms * 1e-3), 1),
               "ms_per_step": round(ms, 2), "steps": args.train_steps, "outcomes": outcomes,
               "clocks": clk.summary(),
               "peak_mem_gib_rank0": round(torch.cuda.max_memory_allocated() / 2 ** 30, 2),
               "note": "same model as the eager leg, continued; the graph removes the eager "
                       "step's host gaps (tools/sharded_profile.py)"}
        del gs
        torch.cuda.empty_cache()
        return res
    except Exception as exc:  # noqa: BLE001 -- a secondary leg must not cost the line
        import traceback
        traceback.print_exc()
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def _sharded_roofline(model, batch, seq, ms, keep, strict, ckpt, clk):
    """Tensor work per rank of one sharded step (the linears' GEMMs: 2 flop
    per weight per token for the forward, the input gradient and the weight
    gradient; plus causal attention) against the bf16 peak."""
    tokens = batch * seq
    lin = sum(p.numel() for n, p in model.named_parameters() if p.dim() == 2
              and "embed" not in n)
    cfg = model.cfg
    attn_fwd = 2 * 2 * tokens * seq * 0.5 * cfg["hidden"] * cfg["layers"]
    # forward + backward (dx, dW); strict adds a second forward + backward,
    # replay a second dW GEMM, keep_grads nothing; checkpointing one more forward
    gemms = 3 + (3 if strict else 0 if keep else 1) + (1 if ckpt else 0)
    attn = attn_fwd * (3.5 + (3.5 if strict else 0) + (1 if ckpt else 0))
    tflop = (gemms * 2 * tokens * lin + attn) / 1e12
    pflops = tflop / (ms * 1e-3) / 1e3
    peak_tf, peak_src = _bf16_peak_tflops()
    peak_pf = peak_tf / 1e3
    scale = (clk.get("sm_mhz") or 0) / (clk.get("sm_max_mhz") or 1) if clk.get("sm_mhz") else None
    return {"tflop_per_step_per_rank": round(tflop, 2), "achieved_pflops_per_rank": round(pflops, 3),
            "peak_pflops": round(peak_pf, 3), "peak_source": peak_src,
            "frac": round(pflops / peak_pf, 3),
            "frac_at_run_clock": (round(pflops / (peak_pf * scale), 3)
                                  if scale and "sustained" not in peak_src else None)}


def _sharded_world1(args):
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0),
                            timeout=datetime.timedelta(minutes=5))
    try:
        return bench_train_sharded(args, 0, 1)
    finally:
        dist.destroy_process_group()


def _ulps16(got, ref):
    import numpy as np
    g = got.astype(np.float16).view(np.int16).astype(np.int64)
    r = ref.astype(np.float16).view(np.int16).astype(np.int64)
    g = np.where(g < 0, -(1 << 15) - g, g)
    r = np.where(r < 0, -(1 << 15) - r, r)
    return np.abs(g - r)


def bench_c1(args):
    """Config 1 parity leg: the reference's own mini
    transformer (zoo.py:150-224), 10 LOMO steps, against the fixtures
    recorded from the reference itself (tests/golden/c1.*, made by
    tests/golden/make_golden.py): A = FULL, plain LOMO; B = HALF, two-pass
    global-norm clip 1.0 + LossScaler(2^16, growth 2); C = as B from 2^24 with
    max 2^24 (forced fp16 overflows).  Each fixture runs through the product
    path -- LOMO's hooks -> K2/K3/K1 (``hooks``), and for B/C also the
    training path with K6/K5 inside the weight-gradient GEMMs
    (``fused_gemm``) -- plus, for B/C, the exactness mode: the restated tape
    (tests/exact_c1.py, f64 ops with the reference's binary16 rounding)
    driving the product kernels in f64 math (``exact_tape``).  Reported:
    decision (outcome, log2 scale) equality, max / mean ulp (fp16) or
    normwise relative error (fp32) of the sampled final parameters, loss
    error, and the GPU run's wall seconds beside the reference's recorded
    CPU seconds for the same 10 steps."""
    import numpy as np
    import torch
    from paper_2306_09782_b200 import LOMO, ClipMode, LossScaler, Stabilizer
    from paper_2306_09782_b200.workloads import (MiniConfig, MiniTransformer,
                                                 mean_cross_entropy, sequence_copy_batch)
    meta = json.loads((ROOT / "tests" / "golden" / "c1.json").read_text())
    arr = np.load(ROOT / "tests" / "golden" / "c1.npz")
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    prev_rr = torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    cfg = MiniConfig(layers=2, hidden=256, heads=4, vocab=1024, seed=0)
    toks = [torch.from_numpy(sequence_copy_batch(0, s, 4, 128, 1024)).cuda() for s in range(10)]

    def stab(key):
        if key == "A":
            return None
        s0 = 2.0 ** 16 if key == "B" else 2.0 ** 24
        return Stabilizer(ClipMode.by_global_norm(1.0), LossScaler(s0, 2, max_scale=2.0 ** 24))

    def compare(key, named, losses, outcomes, scales, secs):
        ref = meta[key]
        r = {"gpu_seconds": round(secs, 3), "reference_cpu_seconds": round(ref["seconds"], 2),
             "outcomes_equal": outcomes == ref["outcomes"]}
        if ref["log2_scale"]:
            r["log2_scale_equal"] = [math.log2(s) for s in scales] == ref["log2_scale"]
        r["max_loss_rel"] = float(max(abs(a - b) / abs(b) for a, b in zip(losses, ref["losses"])
                                      if math.isfinite(b)))
        got = {n: t.detach().reshape(-1) for n, t in named}
        if ref["precision"] == "full":
            r["max_normwise_rel"] = float(max(
                np.linalg.norm(got[n][torch.from_numpy(arr[f"{key}/{n}/idx"]).cuda()]
                               .double().cpu().numpy() - arr[f"{key}/{n}/val"])
                / np.linalg.norm(arr[f"{key}/{n}/val"]) for n in got))
        else:
            u = np.concatenate([_ulps16(got[n][torch.from_numpy(arr[f"{key}/{n}/idx"]).cuda()]
                                        .double().cpu().numpy(), arr[f"{key}/{n}/val"])
                                for n in got])
            r.update(max_ulp=int(u.max()), mean_ulp=round(float(u.mean()), 5),
                     frac_gt_2ulp=float((u > 2).mean()), sampled=int(u.size))
        return r

    def run(key, dtype, fused):
        model = MiniTransformer(cfg, dtype=dtype, device="cuda", fused_linear=fused)
        kw = {"stabilizer": stab(key)}
        if fused:
            kw.update(replay=True, fuse_gemm=True)
        opt = LOMO(model, lr=0.05, **kw)
        losses, outcomes, scales = [], [], []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(10):
            ids = toks[s]
            losses.append(opt.step(lambda: mean_cross_entropy(model(ids), ids), 0.05))
            outcomes.append(opt.last_outcome.value if opt.last_outcome else "applied")
            scales.append(opt.loss_scale)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        res = compare(key, model.named_reference_parameters(), losses, outcomes, scales, secs)
        opt.remove_hooks()
        return res

    out = {"A": {"hooks": run("A", torch.float32, False)}}
    for key in ("B", "C"):
        out[key] = {"hooks": run(key, torch.float16, False),
                    "fused_gemm": run(key, torch.float16, True)}
    # the exactness mode: restated tape (test infrastructure) + product kernels, f64 math
    sys.path.insert(0, str(ROOT / "tests"))
    import gpu_util as U
    from exact_c1 import ExactMini
    from paper_2306_09782_b200 import _lib
    for key in ("B", "C"):
        m = ExactMini(MiniConfig())
        slot = {n: i for i, n in enumerate(reversed(m.names))}
        st = U.State(len(m.names), scale=2.0 ** 16 if key == "B" else 2.0 ** 24, growth=2,
                     min_scale=1.0, max_scale=2.0 ** 24, max_norm=1.0)
        losses, outcomes, scales = [], [], []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(10):
            scale = st.status().scale
            logits, S = m.forward(toks[s])
            loss, dout = m.loss_and_grad(logits, toks[s])
            st.begin(torch.tensor(loss, dtype=torch.float64, device="cuda"))
            m.backward(S, dout * scale, lambda n, g: st.probe(
                g.to(torch.float16), slot[n], _lib.USE_SCALE | _lib.ACCUM_F64))
            st.finalize()
            if st.status().skip:
                outcomes.append("skipped_overflow")
            else:
                logits2, S2 = m.forward(toks[s])
                loss, dout2 = m.loss_and_grad(logits2, toks[s])
                m.backward(S2, dout2 * scale, lambda n, g: U.fused_update(
                    m.p16[n], g.to(torch.float16), math="f64", lr=0.05,
                    flags=_lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF, state=st))
                st.on_clean()
                outcomes.append("applied")
            losses.append(loss)
            scales.append(st.status().scale)
        torch.cuda.synchronize()
        out[key]["exact_tape"] = compare(key, [(n, m.p16[n]) for n in m.names], losses, outcomes,
                                         scales, time.perf_counter() - t0)
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = prev_rr
    ok = all(v.get("outcomes_equal") and v.get("log2_scale_equal", True)
             for fx in out.values() for v in fx.values())
    out["decisions_identical"] = bool(ok)
    out["tolerances"] = {"A": "normwise rel <= 1e-5 (north star fp32)",
                         "B/C": "decisions identical; max/mean ulp reported (2-ulp contract "
                                "is the hook-level one, SURVEY 8c; exact_tape = 0 expected)"}
    return out


def _import_reference():
    """The reference package itself: baseline/_ref (pip-installed from a copy
    of /root/reference/pkg; git-ignored, travels to the GPU box).  The bench
    never reads /root/reference at run time.  Returns (fusedtrain modules,
    where) or (None, why)."""
    import importlib
    for where in (ROOT / "baseline" / "_ref",):
        if (where / "fusedtrain" / "optim.py").exists():
            if str(where) not in sys.path:
                sys.path.insert(0, str(where))
            try:
                mods = {m: importlib.import_module(f"fusedtrain.{m}")
                        for m in ("optim", "tape", "tensor", "estimate")}
                return mods, str(where.relative_to(ROOT) if where.is_relative_to(ROOT) else where)
            except Exception as exc:  # noqa: BLE001
                return None, f"import from {where} failed: {exc}"
    return None, "reference package not found (baseline/_ref missing)"


def cpu_baseline(max_seconds=20.0, steps=None, threads=None):
    """The reference's own CPU update (fusedtrain.optim.apply_update,
    optim.py:52-54, with Tensor.assign's binary16 write-back, tensor.py:30-38,
    74-81) over LLaMA-7B layer 0's 9 parameter tensors (202,383,360 elements,
    HALF_EMULATED = the reference's 16-bit path), imported from baseline/_ref.
    (i) as shipped: one thread (numpy elementwise), one 4096x4096 tensor;
    (ii) all host cores: the same function on disjoint row blocks of every
    tensor, one thread per block (numpy releases the GIL in the ufuncs).
    Falls back to the oracle restatement (kind "port") only when the
    reference cannot be imported."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from paper_2306_09782_b200.workloads import llama_param_shapes
    ref, where = _import_reference()
    cores = threads or os.cpu_count() or 1
    shapes = [s for name, s in llama_param_shapes("7b") if name.startswith("layers.0.")]
    rng = np.random.default_rng(0)
    if ref is not None:
        T, Prm, apply = ref["tensor"], ref["tape"].Parameter, ref["optim"].apply_update
        half = T.Precision.HALF_EMULATED

        def make(values):
            return Prm("w", 0, T.Tensor(values, half))

        def upd(pg):
            apply(pg[0], pg[1], 0.05)
        kind = "reference"
    else:
        sys.path.insert(0, str(ROOT / "oracle"))
        import lomo_oracle as O

        class _P:  # the oracle's restatement of apply_update on a holder
            def __init__(self, v):
                self.v = O.round_through_half(v)

        def make(values):
            return _P(values)

        def upd(pg):
            pg[0].v = O.apply_update(pg[0].v, pg[1], 0.05, O.HALF)
        kind = "port"
    # (i) as shipped: one tensor, one thread
    n1 = 4096 * 4096
    one = (make(rng.uniform(-0.08, 0.08, n1)), np.round(rng.normal(0.0, 1e-3, n1), 8))
    upd(one)
    t0 = time.perf_counter()
    upd(one)
    single = 6 * n1 / (time.perf_counter() - t0) / 1e9
    del one
    # (ii) all cores: disjoint row blocks of every layer-0 tensor
    work = []
    for s in shapes:
        rows, cols = s[0], math.prod(s[1:]) if len(s) > 1 else 1
        per = max(1, rows // max(1, (2 * cores * rows * cols) // sum(math.prod(x) for x in shapes)))
        for r0 in range(0, rows, per):
            m = (min(rows, r0 + per) - r0) * cols
            work.append((make(rng.uniform(-0.08, 0.08, m)),
                         make(rng.normal(0.0, 1e-3, m)).value.data if kind == "reference"
                         else O.round_through_half(rng.normal(0.0, 1e-3, m))))
    elems = sum(math.prod(s) for s in shapes)
    times = []
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(upd, work[:cores]))  # warm the pool
        t_all = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            list(ex.map(upd, work))
            times.append(time.perf_counter() - t0)
            if steps is not None and len(times) >= steps:
                break
            if steps is None and (time.perf_counter() - t_all > max_seconds or len(times) >= 20):
                break
    t = sum(times) / len(times)
    return {"value": round(BYTES_PER_ELEM * elems / t / 1e9, 3), "unit": "GB/s", "cores": cores,
            "kind": kind, "source": where if kind == "reference" else "oracle/lomo_oracle.py",
            "sample": f"fusedtrain.optim.apply_update (optim.py:52-54, HALF_EMULATED write-back "
                      f"tensor.py:30-38) over LLaMA-7B layer-0's 9 tensors ({elems} elements, "
                      f"{len(work)} disjoint row blocks) x {len(times)} passes, float64 buffers "
                      f"as the reference keeps them, {cores} host threads",
            "as_shipped_1thread_gbs": round(single, 3),
            "as_shipped_sample": "one 4096x4096 tensor, one thread (numpy elementwise, as shipped)",
            "seconds_per_pass": round(t, 3),
            "full_7b_pass_seconds_extrapolated": round(t * 6738415616 / elems, 1)}


# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["bf16", "fp16"], default="bf16")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c1", action="store_true", help="skip the config-1 parity leg")
    ap.add_argument("--no-table1", action="store_true", help="skip the measured Table-1 row")
    ap.add_argument("--e2e-slots", type=int, default=4, help="device staging slots of the e2e pipeline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--train-steps", type=int, default=10)
    ap.add_argument("--train-steps-headline", type=int, default=30)
    ap.add_argument("--train-warmup", type=int, default=3)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ckpt", action="store_true", help="per-layer activation checkpointing")
    ap.add_argument("--separate-proj", action="store_true",
                    help="train leg: q/k/v and gate/up as separate weights (default: stacked)")
    ap.add_argument("--train-model", default="7b", choices=["7b", "13b", "30b", "65b"],
                    help="model of the single-GPU train leg (config 3: 7b)")
    ap.add_argument("--train-variants", default="",
                    help="comma list (default: " + ",".join(TRAIN_DEFAULT) + "); also strict_graph, "
                         "strict_fused_gemm, replay, replay_graph, replay_fused_gemm, grouped, "
                         "grouped_fused_gemm, single_pass_fused_gemm")
    ap.add_argument("--sharded-train", action="store_true",
                    help="run the ZeRO-3 sharded train leg even at N=1 (world-1 NCCL group)")
    ap.add_argument("--no-sharded-world1", dest="sharded_world1", action="store_false",
                    help="skip the N=1 run of the sharded train leg (world-1 NCCL group)")
    ap.add_argument("--sharded-fused-rs", default="", choices=["", "auto", "ipc", "nvls"],
                    help="sharded train leg: K4 over peer memory instead of the NCCL "
                         "reduce-scatter (with kept shards: the K4 probe keeps the reduced slice)")
    ap.add_argument("--sharded-graph", action="store_true",
                    help="N>1: also time the GraphedShardedStep form of the sharded train leg")
    ap.add_argument("--no-sharded-graph", action="store_true",
                    help="sharded train leg: skip the GraphedShardedStep timing")
    ap.add_argument("--sharded-strict", action="store_true",
                    help="sharded train leg: pass 2 as a second forward+backward (default: replay)")
    ap.add_argument("--sharded-model", default="13b", choices=["tiny", "7b", "13b", "30b", "65b"],
                    help="model of the N>1 sharded train leg (config 4: 13b, config 5: 65b)")
    ap.add_argument("--update-layers", type=int, default=32,
                    help="N>1 sharded update: decoder-layer buckets (32 = LLaMA-7B; fewer only "
                         "for LOMO_BENCH_SHARE_GPU dry runs)")
    ap.add_argument("--k4-transport", default="", choices=["", "ipc", "nvls"],
                    help="N>1: force the K4 peer transport (default: NVLS when available)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_baseline(steps=args.warmup + args.steps)
        line = {"metric": METRIC, "value": cb["value"], "unit": "GB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(1e3 * cb["seconds_per_pass"], 2),
                "higher_is_better": True, "scaling": "none (host cores)", "vs_baseline": None,
                "dtype": "f64 math, fp16 storage (reference HALF_EMULATED)",
                "data": "synthetic p~U(-0.08,0.08), g~N(0,1e-3)", "impl": "reference",
                "config": {"workload": "reference apply_update over LLaMA-7B layer-0 tensors "
                                       "(bounded sample of config 2)"},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                    "source", "as_shipped_1thread_gbs")},
                "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        # NCCL's init lines (ranks, NVLink/NVLS transport) in the job log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    rank, world, local = _dist_init(args.gpus)
    if args.sharded_train and world == 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    import __graft_entry__
    __graft_entry__.build()
    torch.backends.cuda.matmul.allow_tf32 = False
    peak, peak_src = _peaks()
    tr = _traffic()

    def optional(fn, *a):
        """Secondary legs must never cost the headline line: report their error."""
        try:
            return fn(*a)
        except Exception as exc:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            torch.cuda.empty_cache()
            return {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if world == 1:
        up = bench_update(args, rank, world)
        value, ms = up["gbs"], up["ms"]
        head = {
            "scaling": "weak",
            "config": {
                "workload": "config 2: one LOMO fused-update pass (K1 per tensor, reverse "
                            "registration = autograd delivery order) over all 291 LLaMA-7B "
                            "parameter tensors, issued back to back as a pass over kept "
                            "gradients issues them (K1s after the first chained, "
                            "LOMO_CHAINED; the unchained hook pattern: "
                            "update_pass_unchained)",
                "elements": up["total_elems"], "algorithmic_bytes_per_elem": BYTES_PER_ELEM,
                "math": "fp32", "lr": 0.05, "parallelism": "single",
                "l2": "no flush: per-step working set 27 GB >> 126 MB L2, each byte touched "
                      "once per step"},
            "roofline": {"bound": "hbm", "achieved": round(up["gbs"], 1), "peak": peak,
                         "unit": "GB/s", "frac": round(up["gbs"] / peak, 4),
                         "traffic": tr["dram_bytes"] if tr else None,
                         "traffic_algorithmic": tr["algorithmic_bytes"] if tr else None,
                         "traffic_launch": tr["launch"] if tr else None,
                         "traffic_source": tr["source"] if tr else None,
                         "traffic_whole_pass": _pass_traffic(), "peak_source": peak_src,
                         "kernel": "k1_update<bf16,f32,chained>: the timed region holds only K1 "
                                   "launches (226 per-tensor + 2 k1_update_multi for the 65 [4096] "
                                   "tensors) on one stream, bracketed by CUDA events; achieved = "
                                   "6 B/elem x elements / their time",
                         "avg_launch_us": round(1e3 * up["ms"] / (up["launches"] / args.steps), 2),
                         "host_ms_per_pass": up["host_enqueue"]["ms_per_pass"],
                         "host_enqueue": up["host_enqueue"],
                         "host_ms_timed_loop": round(up["host_ms"], 3),
                         "graphed_pass_gbs": round(up["graphed_gbs"], 1),
                         "per_shape_instrumented": up["shapes"],
                         "per_shape_note": "per-launch event pairs (separate replay) break the PDL "
                                           "overlap, so these per-shape rates understate the pass"},
            "probe_pass": dict(up["probe"], frac=round(up["probe"]["gbs"] / peak, 4)),
            "update_pass_device_state": dict(up["flags_pass"],
                                             frac=round(up["flags_pass"]["gbs"] / peak, 4)),
            "update_pass_unchained": dict(up["unchained"],
                                          frac=round(up["unchained"]["gbs"] / peak, 4)),
            "update_pass_fp16_scaled": (dict(up["fp16_scaled"],
                                             frac=round(up["fp16_scaled"]["gbs"] / peak, 4))
                                        if up["fp16_scaled"] else None),
            "f64_math_update_pass": dict(up["f64_math"],
                                         frac=round(up["f64_math"]["gbs"] / peak, 4)),
            "gpu_launches": up["launches"], "clocks": up["clocks"]}
    else:
        sh = bench_sharded_update(args, rank, world)
        value, ms = sh["gbs"], sh["ms"]
        head = {
            "scaling": "strong",
            "config": {
                "workload": f"sharded LOMO update pass of LLaMA-7B over {world} ranks: "
                            f"{sh['buckets']} flat "
                            "gradient buckets per rank (its own backward's), reduced across ranks "
                            "and applied to each rank's 1/W parameter shard (best of NCCL "
                            "reduce_scatter -> K1 and K4)",
                "elements": sh["elements"], "algorithmic_bytes_per_elem": BYTES_PER_ELEM,
                "math": "fp32", "lr": 0.05, "parallelism": f"zero3-dp{world}",
                "l2": "no flush: 13.5 GB of gradients per rank per step >> 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": round(sh["k1_gbs"], 1), "peak": peak,
                         "unit": "GB/s", "frac": round(sh["k1_gbs"] / peak, 4),
                         "traffic": None, "peak_source": peak_src,
                         "kernel": "K1 on the reduce-scattered shards (per-launch CUDA events); "
                                   "the pass itself is NVLink-bound, see sharded_update"},
            "sharded_update": sh, "gpu_launches": sh["launches"], "clocks": sh["clocks"]}

    e2e = None if args.no_e2e else optional(bench_e2e if world == 1 else bench_e2e_sharded,
                                            args, rank, world)
    c1 = optional(bench_c1, args) if (world == 1 and not args.no_c1) else None
    k4l = optional(bench_k4_local, args) if world == 1 else None
    train = None
    if not args.no_train:
        train = optional(bench_train, args, rank, world) if (world == 1 and not
                                                              args.sharded_train) else \
            optional(bench_train_sharded, args, rank, world)
    sharded1 = None
    if world == 1 and not args.no_train and not args.sharded_train and args.sharded_world1:
        # config 4's data path (ZeRO-3 buckets, NCCL reduce-scatter -> K2/K1 per
        # shard) on this one GPU: a world-1 NCCL group, where the collectives are
        # local copies -- the sharded machinery's own cost, next to plain LOMO
        sharded1 = optional(_sharded_world1, args)
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb = optional(cpu_baseline)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": head.pop("scaling"),
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic: p~U(-0.08,0.08), g~N(0,1e-3) (torch.Generator seed 1234+rank)",
        }
        line.update(head)
        line.update({"e2e": e2e, "cpu_baseline": cb, "c1_parity": c1, "train": train})
        if k4l is not None:
            line["k4_simulated_peers"] = k4l
        if sharded1 is not None:
            line["train_sharded_world1"] = sharded1
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
