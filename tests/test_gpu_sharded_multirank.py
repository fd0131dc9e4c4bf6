"""ShardedLOMO with the REAL CUDA engine at world size 2: two processes share
this box's single B200 (gloo carries the collectives -- NCCL refuses two ranks
on one device), so the multi-rank protocol runs through the actual kernels:
per-shard K1/K2, the rank-ordered norm exchange and K3 on every rank, ZeRO-3
gather/release -- and, for ``fused_rs``, K4 over CUDA-IPC peer buffers with
the device barriers of peer.py between the two processes.  Expected: a single process updating the full batch with
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
    fused_rs = "ipc" if mode.startswith("fused_rs") else False
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
                          keep_grads=mode.endswith("keep_grads"))
        outs = []
        for step in range(3):
            ids, tgt = _batch(step, world)
            ids, tgt = ids[2 * rank:2 * rank + 2].cuda(), tgt[2 * rank:2 * rank + 2].cuda()
            opt.step(lambda: model.loss(ids, tgt), 0.05)
            outs.append(opt.last_outcome.value)
        opt.gather_all()
        q.put((rank, outs, {n: p.detach().cpu().numpy().copy()
                            for n, p in model.named_parameters()}))
        opt.remove_hooks()  # collective: closes the peer rings
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


@pytest.mark.parametrize("mode", ["nccl_path", "fused_rs", "replay", "keep_grads",
                                  "fused_rs_keep_grads"])
def test_sharded_two_ranks_real_kernels(mode):
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


def _ring_worker(rank, world, port, q):
    """Transport-level checks of peer.PeerRing(ipc) between two processes:
    K4 (update and probe) over the peers' buffers against the same sums done
    by hand, several rounds through the ring's reuse barrier, and a barrier
    that one rank skips -> the timeout lands in the state's error word."""
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2306_09782_b200 import _lib
        from paper_2306_09782_b200.engine import CudaEngine
        from paper_2306_09782_b200.errors import NativeError
        from paper_2306_09782_b200.peer import PeerRing
        dev = torch.device("cuda", 0)
        n = 4096 * world + 8 * world * 3  # ragged multiple of 8*world
        S = n // world
        eng = CudaEngine(dev, 4, None, None, "f32", grad_div=1.0)
        ring = PeerRing(n, torch.bfloat16, dev, None, "ipc", err_ptr=eng.error_ptr, timeout_s=20)
        p = torch.zeros(S, dtype=torch.bfloat16, device=dev)
        results = []
        for rnd in range(7):  # > NBUF rounds: every buffer reused through its free barrier
            k = ring.acquire(rnd)
            g = torch.Generator(device="cuda").manual_seed(1000 * rnd + rank)
            ring.bufs[k][:n].copy_(torch.randn(n, generator=g, device=dev).to(torch.bfloat16))
            ring.filled(k)
            p.fill_(0.5)
            eng.configure(lr=0.25)
            ring.update(eng, p, k, rank * S)
            eng.configure(flags=0)
            _lib.check(eng.lib.lomo_begin_step(eng.ptr, None, 0, eng.stream()), "begin")
            ring.probe(eng, k, rank * S, S, slot=1)
            eng.finalize()
            st = eng.read_status()
            ring.release(k)
            results.append((k, p.float().cpu().numpy().copy(), float(st.sumsq_total)))
        # a barrier only rank 0 enters: it must time out into the error word
        timed_out = None
        if rank == 0:
            ring.timeout_ns = int(0.5e9)
            ring.barrier(15)
            try:
                eng.read_status()
                timed_out = False
            except NativeError as e:
                timed_out = "peer barrier" in str(e)
        dist.barrier()
        q.put((rank, results, timed_out))
        # (the skipped epoch leaves channel 15 unbalanced; the ring is dropped)
        dist.destroy_process_group()
    except BaseException:
        import traceback
        q.put((rank, "error", traceback.format_exc()))
        raise


def test_peer_ring_ipc_two_processes():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=300)
        if item[1] == "error":
            for p in procs:
                p.kill()
            pytest.fail(f"rank {item[0]} failed:\n{item[2]}")
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    n = 4096 * world + 8 * world * 3
    S = n // world
    for rnd in range(7):
        full = sum(torch.randn(n, generator=torch.Generator(device="cuda").manual_seed(1000 * rnd + r),
                               device="cuda").to(torch.bfloat16).double() for r in range(world))
        for r in range(world):
            k, p, sumsq = res[r][1][rnd]
            assert k == rnd % 3
            g = full[r * S:(r + 1) * S]
            # K4: the rank-order fp32 sum of two bf16 values is exact in fp32 here
            want = (0.5 - 0.25 * g.float()).to(torch.bfloat16).float().cpu().numpy()
            assert np.array_equal(p, want), (rnd, r)
            ref = float((g.float() ** 2).double().sum())
            assert abs(sumsq - ref) <= 1e-5 * ref, (rnd, r, sumsq, ref)
    assert res[0][2] is True
