"""ShardedLOMO on the GPU: the CUDA engine + NCCL collectives in a world of
one rank (this run has a single B200; world_size 2 host logic is covered by
tests/test_sharded_gloo.py).  With one rank the reduce-scatter is the
identity, so ShardedLOMO must reproduce single-GPU LOMO -- one K1 launch per
bucket shard instead of per tensor, and the global norm summed per bucket."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

CFG = dict(hidden=128, layers=3, heads=4, ffn=256, vocab=256)


@pytest.fixture(scope="module")
def nccl_world():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("stab_kind", ["plain", "norm_scaler", "norm_scaler_replay",
                                       "norm_scaler_replay_ckpt", "norm_scaler_keep"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_sharded_world1_matches_lomo(nccl_world, stab_kind, dtype):
    from paper_2306_09782_b200 import LOMO, ClipMode, LossScaler, Stabilizer
    from paper_2306_09782_b200.sharded import ShardedLOMO
    from paper_2306_09782_b200.workloads import Llama
    torch.backends.cuda.matmul.allow_tf32 = False

    def stab():
        if stab_kind == "plain":
            return None
        return Stabilizer(ClipMode.by_global_norm(0.5), LossScaler(2.0 ** 8, 2))

    replay, ckpt = "replay" in stab_kind, stab_kind.endswith("ckpt")
    keep = stab_kind.endswith("_keep")
    stab_kind = stab_kind.split("_replay")[0].removesuffix("_keep")
    a = Llama(CFG, dtype=dtype, device="cuda", seed=0)
    b = Llama(CFG, dtype=dtype, device="cuda", seed=0, checkpointing=ckpt)
    oa = LOMO(a, lr=0.05, stabilizer=stab())
    ob = ShardedLOMO(b, lr=0.05, stabilizer=stab(), replay=replay, keep_grads=keep)
    assert all(not bk.gathered for bk in ob.buckets if bk.module is not None)
    g = torch.Generator(device="cuda").manual_seed(1)
    for step in range(3):
        d = torch.randint(0, CFG["vocab"], (2, 33), device="cuda", generator=g)
        la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
        lb = ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
        assert abs(la - lb) <= 1e-6 * abs(la), (step, la, lb)
        assert ob.last_outcome == oa.last_outcome
    ob.gather_all()
    tol = 1e-6 if dtype == torch.float32 else 1e-2
    for (n, x), (_, y) in zip(a.named_parameters(), b.named_parameters()):
        err = (x.float() - y.float()).abs().max().item()
        assert err <= tol * max(1.0, x.float().abs().max().item()), (n, err)
    ob.remove_hooks()


def test_sharded_with_checkpointing_world1(nccl_world):
    """ZeRO-3 gather/release interleaved with the per-layer recompute."""
    from paper_2306_09782_b200 import LOMO
    from paper_2306_09782_b200.sharded import ShardedLOMO
    from paper_2306_09782_b200.workloads import Llama
    a = Llama(CFG, dtype=torch.float32, device="cuda", seed=0, checkpointing=True)
    b = Llama(CFG, dtype=torch.float32, device="cuda", seed=0, checkpointing=True)
    oa = LOMO(a, lr=0.05, clip_grad_norm=0.5)
    ob = ShardedLOMO(b, lr=0.05, clip_grad_norm=0.5)
    g = torch.Generator(device="cuda").manual_seed(2)
    for step in range(2):
        d = torch.randint(0, CFG["vocab"], (2, 17), device="cuda", generator=g)
        la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
        lb = ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
        assert abs(la - lb) <= 1e-5 * abs(la)
    ob.gather_all()
    for (n, x), (_, y) in zip(a.named_parameters(), b.named_parameters()):
        assert (x - y).abs().max().item() <= 1e-5, n
    ob.remove_hooks()


def _need_nvls(transport):
    from paper_2306_09782_b200.peer import nvls_available
    if transport == "nvls" and not nvls_available(torch.device("cuda", 0)):
        pytest.skip("no NVLS multicast on this GPU (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0)")


@pytest.mark.parametrize("transport", ["ipc", "nvls"])
@pytest.mark.parametrize("two_pass", [False, True, "keep"])
def test_fused_rs_world1_equals_nccl_path(nccl_world, two_pass, transport):
    """K4 over peer buffers (world 1: the only peer is this GPU) gives the
    same parameters as NCCL reduce_scatter + K1/K2 -- over a CUDA-IPC
    allocation, and over an NVLS multicast object (multimem.ld_reduce of one
    copy is the copy); "keep": keep_grads on both, the K4 probe writing the
    reduced slice pass 2 updates from."""
    from paper_2306_09782_b200.sharded import ShardedLOMO
    from paper_2306_09782_b200.workloads import Llama
    _need_nvls(transport)
    a = Llama(CFG, dtype=torch.bfloat16, device="cuda", seed=0)
    b = Llama(CFG, dtype=torch.bfloat16, device="cuda", seed=0)
    kw = dict(clip_grad_norm=0.5, loss_scale=2.0 ** 8) if two_pass else {}
    keep = two_pass == "keep"
    oa = ShardedLOMO(a, lr=0.05, keep_grads=keep, **kw)
    ob = ShardedLOMO(b, lr=0.05, fused_rs=transport, keep_grads=keep, **kw)
    assert ob.transport == transport
    g = torch.Generator(device="cuda").manual_seed(5)
    for step in range(3):
        d = torch.randint(0, CFG["vocab"], (2, 33), device="cuda", generator=g)
        la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
        lb = ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
        assert la == lb
    oa.gather_all()
    ob.gather_all()
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)
    oa.remove_hooks()
    ob.remove_hooks()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16, torch.bfloat16])
def test_nvls_k4_kernels_world1(nccl_world, dtype):
    """The NVLS K4 kernels on a one-device multicast object: ld_reduce over
    the multicast address returns the one copy, so K4-mc equals K1/K2 on the
    buffer itself (bit for bit; probe to fp32 summation order), and the
    multimem.red barrier completes."""
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.engine import CudaEngine
    from paper_2306_09782_b200.peer import PeerRing
    _need_nvls("nvls")
    dev = torch.device("cuda", 0)
    n = 3 * 8192 + 64
    eng = CudaEngine(dev, 2, None, None, "f32")
    ring = PeerRing(n, dtype, dev, None, "nvls", err_ptr=eng.error_ptr, timeout_s=10)
    g = torch.Generator(device="cuda").manual_seed(3)
    for rnd in range(4):
        k = ring.acquire(rnd)
        ring.bufs[k].copy_(torch.randn(n, generator=g, device=dev).to(dtype))
        ring.filled(k)
        p = torch.rand(n, generator=g, device=dev).to(dtype)
        q = p.clone()
        eng.configure(lr=0.125)
        ring.update(eng, p, k, 0)
        eng.update(q, ring.bufs[k])
        eng.flush()
        eng.configure(flags=0)
        _lib.check(eng.lib.lomo_begin_step(eng.ptr, None, 0, eng.stream()), "begin")
        ring.probe(eng, k, 0, n, 0)
        eng.probe(ring.bufs[k], 1)
        eng.flush()
        _lib.check(eng.lib.lomo_local_norm_partial(eng.ptr, torch.zeros(2, dtype=torch.float64,
                                                                      device=dev).data_ptr(),
                                                   eng.stream()), "partial")
        st = eng.read_status()  # raises on a barrier timeout
        ring.release(k)
        assert torch.equal(p, q), rnd
        sl = torch.empty(2, dtype=torch.float64)
        off = _lib.SLOTS_OFFSET
        sl.copy_(eng.state[off:off + 16].view(torch.float64))
        assert abs(sl[0] - sl[1]) <= 1e-6 * float(sl[1]), (rnd, sl)
        assert not st.overflow
    ring.close()


@pytest.mark.parametrize("fused", [False, "ipc"])
@pytest.mark.parametrize("mode", ["keep", "replay"])
@pytest.mark.parametrize("dtype,scale", [(torch.float32, 2.0 ** 8), (torch.float16, 2.0 ** 20)])
def test_graphed_sharded_step_equals_eager(nccl_world, mode, dtype, scale, fused):
    """GraphedShardedStep (refresh all-gathers, reduce-scatters, K2/K3/K1 and
    the rank exchange captured in two CUDA graphs) == the eager ShardedLOMO
    step bit for bit, including overflow-skipped steps (fp16 at 2^20)."""
    from paper_2306_09782_b200 import LossScaler
    from paper_2306_09782_b200.graphs import GraphedShardedStep
    from paper_2306_09782_b200.sharded import ShardedLOMO
    from paper_2306_09782_b200.workloads import Llama
    torch.backends.cuda.matmul.allow_tf32 = False
    a = Llama(CFG, dtype=dtype, device="cuda", seed=0)
    b = Llama(CFG, dtype=dtype, device="cuda", seed=0)

    def make(m):
        return ShardedLOMO(m, lr=0.05, clip_grad_norm=0.5,
                           loss_scale=LossScaler(scale, growth_interval=2),
                           reshard_after_forward=False, keep_grads=mode == "keep",
                           replay=mode == "replay", fused_rs=fused)
    oa, ob = make(a), make(b)
    g = torch.Generator(device="cuda").manual_seed(3)
    batches = [torch.randint(0, CFG["vocab"], (2, 33), device="cuda", generator=g)
               for _ in range(8)]
    static = batches[0].clone()
    warm = 2
    for k in range(warm):  # the graphed object's warm-up steps, mirrored eagerly
        oa.step(lambda: a.loss(static[:, :-1], static[:, 1:]), 0.05)
    gs = GraphedShardedStep(ob, lambda d: b.loss(d[:, :-1], d[:, 1:]), [static], warmup=warm,
                            lr=0.05)
    outcomes = []
    for k in range(1, 7):
        static.copy_(batches[k])
        la = oa.step(lambda: a.loss(static[:, :-1], static[:, 1:]), 0.05)
        lb = float(gs.step(0.05).detach())
        assert ob.last_outcome == oa.last_outcome, k
        outcomes.append(oa.last_outcome.value)
        assert la == lb or (la != la and lb != lb), (k, la, lb)
    oa.gather_all()
    ob.gather_all()
    for (n, x), (_, y) in zip(a.named_parameters(), b.named_parameters()):
        assert torch.equal(x, y), n
    if dtype == torch.float16:
        assert "skipped_overflow" in outcomes or oa.engine.read_status().steps_skipped > 0
    oa.remove_hooks()
    ob.remove_hooks()
