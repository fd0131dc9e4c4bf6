"""ShardedLOMO host logic with world_size 2 over gloo on CPU (no GPU here):
ZeRO-3 buckets, gather/release, reduce-scatter feeding the per-shard update,
the rank-ordered global-norm exchange and the cross-rank skip agreement.

The per-shard arithmetic comes from tests/cpu_engine.py (the oracle's float64
semantics); the GPU kernels are covered by tests/test_gpu_*.py.  Expected
results: a single process applying materialise-then-clipped-SGD
(stabilize.py:180-230, test_stabilize.py:23-37) to the FULL batch -- the two
ranks each see half of it, and the mean-CE gradient average equals the
full-batch gradient.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CFG = dict(hidden=32, layers=2, heads=4, ffn=64, vocab=64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CLIP_V = 0.01  # value-clip threshold of the "value" mode (small enough to bind)


def _batches(step, world):
    g = torch.Generator().manual_seed(100 + step)
    d = torch.randint(0, CFG["vocab"], (2 * world, 9), generator=g)
    return d[:, :-1], d[:, 1:]


def _reference(steps, world, max_norm, lr, inf_step=None, fused_proj=False, clip_value=None):
    from paper_2306_09782_b200.workloads import Llama
    model = Llama(CFG, dtype=torch.float64, device="cpu", seed=0, fused_proj=fused_proj)
    outcomes = []
    for step in range(steps):
        ids, tgt = _batches(step, world)
        loss = model.loss(ids, tgt)
        if inf_step == step:
            loss = loss * float("inf")
        if not math.isfinite(loss.item()):
            outcomes.append("skip")
            continue
        loss.backward()
        with torch.no_grad():
            ps = list(model.parameters())
            sq = sum(float((p.grad.double() ** 2).sum()) for p in ps)
            n = math.sqrt(sq)
            coef = min(1.0, max_norm / n) if (max_norm and n > 0) else 1.0
            for p in ps:
                g = p.grad.clamp(-clip_value, clip_value) if clip_value else p.grad * coef
                p.copy_(p - lr * g)
                p.grad = None
        outcomes.append("apply")
    return {n: p.detach().clone() for n, p in model.named_parameters()}, outcomes


def _worker(rank, world, port, mode, q):
    try:
        _run(rank, world, port, mode, q)
    except BaseException:
        import traceback
        q.put((rank, "error", traceback.format_exc(), None))
        raise


def _run(rank, world, port, mode, q):
    direct = not mode.endswith("_copy")  # weight gradients GEMM'd into the buckets
    replay = mode.endswith("_replay")    # pass 2 from the stashed (x, dy)
    keep = mode.endswith("_keep")        # pass 2 from pass 1's reduced shards
    mode = mode.removesuffix("_copy").removesuffix("_replay").removesuffix("_keep")
    fused_proj = mode.endswith("_fp")    # stacked projections (layers called as forward_res)
    mode = mode.removesuffix("_fp")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_engine import CpuEngine
        from paper_2306_09782_b200 import LossScaler, Stabilizer, ClipMode
        from paper_2306_09782_b200.sharded import ShardedLOMO
        from paper_2306_09782_b200.workloads import Llama
        torch.manual_seed(1234 + rank)  # ranks start different: broadcast must fix it
        model = Llama(CFG, dtype=torch.float64, device="cpu", seed=rank, fused_proj=fused_proj)
        lr = 0.05
        max_norm = 0.5 if mode not in ("plain", "value") else None
        stab = None
        if mode == "value":  # single pass, the clip applied to the reduced (mean) gradient
            stab = Stabilizer(ClipMode.by_value(CLIP_V))
        elif mode == "norm":
            stab = Stabilizer(ClipMode.by_global_norm(max_norm))
        elif mode in ("norm_scaler", "skip"):
            stab = Stabilizer(ClipMode.by_global_norm(max_norm), LossScaler(2.0 ** 8, 2))
        nb = len(model.layers) + 1
        eng = CpuEngine(nb, stab.scaler if stab else None, max_norm, grad_div=world)
        opt = ShardedLOMO(model, lr=lr, stabilizer=stab, math="f64", _engine=eng,
                          direct_grads=direct, replay=replay, keep_grads=keep)
        # ZeRO-3: layer buckets are released between uses
        released = [not b.gathered for b in opt.buckets if b.module is not None]
        outcomes = []
        inf_step = 1 if mode == "skip" else None
        for step in range(3):
            ids, tgt = _batches(step, world)
            ids, tgt = ids[2 * rank:2 * rank + 2], tgt[2 * rank:2 * rank + 2]

            def closure():
                loss = model.loss(ids, tgt)
                if inf_step == step and rank == 1:   # only ONE rank sees inf
                    loss = loss * float("inf")
                return loss
            opt.step(closure, lr)
            outcomes.append("skip" if (opt.last_outcome is not None
                                       and opt.last_outcome.value == "skipped_overflow")
                            else "apply")
        opt.gather_all()
        got = {n: p.detach().numpy().copy() for n, p in model.named_parameters()}
        q.put((rank, released, outcomes, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["plain", "value", "norm", "norm_scaler", "skip", "norm_scaler_copy",
                                  "norm_replay", "norm_scaler_replay", "skip_replay",
                                  "norm_scaler_keep", "skip_keep", "norm_scaler_fp",
                                  "norm_scaler_fp_keep"])
def test_sharded_lomo_matches_full_batch_reference(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        item = q.get(timeout=240)
        if item[1] == "error":
            for p in procs:
                p.kill()
            pytest.fail(f"rank {item[0]} failed:\n{item[2]}")
        res.append(item)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    mode = mode.removesuffix("_copy").removesuffix("_replay").removesuffix("_keep")
    fused_proj = mode.endswith("_fp")
    mode = mode.removesuffix("_fp")
    max_norm = 0.5 if mode not in ("plain", "value") else None
    want, want_out = _reference(3, world, max_norm, 0.05, inf_step=1 if mode == "skip" else None,
                                fused_proj=fused_proj,
                                clip_value=CLIP_V if mode == "value" else None)
    for rank, released, outcomes, got in res:
        assert all(released), "layer buckets must be released after construction (ZeRO-3)"
        assert outcomes == want_out, (rank, outcomes, want_out)
        for name, w in want.items():
            g = torch.from_numpy(got[name])
            assert torch.allclose(g, w, rtol=0, atol=1e-12), (rank, name, (g - w).abs().max())
    # both ranks hold identical parameters
    for name in want:
        assert np.array_equal(res[0][3][name], res[1][3][name])
