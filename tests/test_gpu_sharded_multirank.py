"""ShardedLOMO with the REAL CUDA engine at world size 2: two processes share
this box's single B200 (gloo carries the collectives -- NCCL refuses two ranks
on one device), so the multi-rank protocol runs through the actual kernels:
per-shard K1/K2, the rank-ordered norm exchange and K3 on every rank, ZeRO-3
gather/release.  Expected: a single process updating the full batch with
materialise-then-clipped-SGD in float64 (the reference two-pass step,
stabilize.py:180-230), to 1e-12."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(step, world):
    g = torch.Generator().manual_seed(300 + step)
    d = torch.randint(0, CFG["vocab"], (2 * world, 17), generator=g)
    return d[:, :-1], d[:, 1:]


def _worker(rank, world, port, mode, q):
    fused_rs = mode == "fused_rs"
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2306_09782_b200.sharded import ShardedLOMO
        from paper_2306_09782_b200.workloads import Llama
        model = Llama(CFG, dtype=torch.float64, device="cuda", seed=rank)  # rank 0 broadcast
        opt = ShardedLOMO(model, lr=0.05, clip_grad_norm=0.5, loss_scale=2.0 ** 8, math="f64",
                          fused_rs=fused_rs, replay=mode == "replay",
                          keep_grads=mode == "keep_grads")
        outs = []
        for step in range(3):
            ids, tgt = _batch(step, world)
            ids, tgt = ids[2 * rank:2 * rank + 2].cuda(), tgt[2 * rank:2 * rank + 2].cuda()
            opt.step(lambda: model.loss(ids, tgt), 0.05)
            outs.append(opt.last_outcome.value)
        opt.gather_all()
        q.put((rank, outs, {n: p.detach().cpu().numpy().copy()
                            for n, p in model.named_parameters()}))
        dist.destroy_process_group()
    except BaseException:
        import traceback
        q.put((rank, "error", traceback.format_exc()))
        raise


def _reference(world):
    from paper_2306_09782_b200.workloads import Llama
    model = Llama(CFG, dtype=torch.float64, device="cuda", seed=0)
    for step in range(3):
        ids, tgt = _batch(step, world)
        model.loss(ids.cuda(), tgt.cuda()).backward()
        with torch.no_grad():
            ps = list(model.parameters())
            n = math.sqrt(sum(float((p.grad ** 2).sum()) for p in ps))
            coef = min(1.0, 0.5 / n)
            for p in ps:
                p.copy_(p - 0.05 * (p.grad * coef))
                p.grad = None
    return {n: p.detach().cpu().numpy() for n, p in model.named_parameters()}


@pytest.mark.parametrize("mode", ["nccl_path", "fused_rs", "replay", "keep_grads"])
def test_sharded_two_ranks_real_kernels(mode):
    fused_rs = mode == "fused_rs"
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        item = q.get(timeout=300)
        if item[1] == "error":
            for p in procs:
                p.kill()
            if fused_rs and "symmetric" in item[2].lower():
                pytest.skip("symmetric memory unavailable between processes here: " +
                            item[2].splitlines()[-1])
            pytest.fail(f"rank {item[0]} failed:\n{item[2]}")
        res.append(item)
    for p in procs:
        p.join(timeout=60)
    want = _reference(world)
    res.sort(key=lambda t: t[0])
    for rank, outs, got in res:
        assert outs == ["applied"] * 3
        for name, w in want.items():
            assert np.allclose(got[name], w, rtol=0, atol=1e-12), (rank, name)
    for name in want:
        assert np.array_equal(res[0][2][name], res[1][2][name])
