"""K5: the weight-gradient GEMM with the LOMO update as its epilogue
(csrc/lomo_gemm_update.cu, tcgen05 tensor cores), through the C-ABI.

The epilogue first rounds the fp32 accumulator to the storage dtype -- the
gradient the reference tape delivers to the hook (tape.py:377) and K1 reads
-- then applies p <- fma(alpha, g, beta * p) (optim.py:52-54 with the
update_hook factors folded into alpha, stabilize.py:217-224).

* K5 == K6 (same tcgen05 mainloop, gradient kept) -> K1, BIT FOR BIT, when
  alpha = -lr (identical gradients, identical arithmetic).
* Against float64: p_ref = round(beta * p + alpha * round16(dy^T x)); within
  TWO ulps of the operands' scale |p| + |alpha g| (stated tolerance): one for
  the update's rounding, one because the fp32 accumulation can move the
  16-bit gradient by one of its ulps near a rounding tie (alpha * ulp(g) is
  at most one operand ulp).  Measured: max 2.0, mismatching elements
  <= 8.4e-4.
"""
import numpy as np
import pytest
import torch

import lomo_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import gpu_util as U
    from paper_2306_09782_b200 import _lib


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    torch.cuda.set_device(0)


def _run(p, dy, x, alpha, beta):
    lib = U.lib()
    dt = U.CODE[p.dtype]
    out_f, in_f = p.shape
    need = lib.lomo_gemm_update_workspace(out_f, in_f, dy.shape[0], dt)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
    return lib.lomo_gemm_update(p.data_ptr(), dy.data_ptr(), x.data_ptr(), out_f, in_f,
                                dy.shape[0], dt, alpha, beta, ws.data_ptr(), need, U.stream())


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("out_f,in_f,tokens", [(256, 128, 64), (4096, 4096, 1024),
                                               (1024, 2816, 1000), (11008, 4096, 512)])
def test_gemm_update_matches_f64_reference(dtype, out_f, in_f, tokens):
    prec = "bf16" if dtype == torch.bfloat16 else "half"
    g = torch.Generator(device="cuda").manual_seed(out_f + tokens)
    p = torch.empty(out_f, in_f, device="cuda").uniform_(-0.08, 0.08, generator=g).to(dtype)
    dy = (torch.randn(tokens, out_f, device="cuda", generator=g) * 1e-2).to(dtype)
    x = torch.randn(tokens, in_f, device="cuda", generator=g).to(dtype)
    alpha, beta = -0.05 * 0.7 / 1024.0 * 1024.0, 1.0
    p0 = p.double()
    upd = alpha * (dy.double().t() @ x.double()).to(dtype).double()  # the rounded gradient
    want = O.round_to((beta * p0 + upd).cpu().numpy(), prec)
    assert _run(p, dy, x, alpha, beta) == 0
    torch.cuda.synchronize()
    d = U.ulp_diff(p, torch.from_numpy(want).to(dtype).cuda())
    frac = (d > 0).float().mean().item()
    err = (p.double().cpu() - torch.from_numpy(want)).abs().numpy()
    scale = (p0.abs() + upd.abs()).cpu().numpy()
    mant, emin = (7, -126) if prec == "bf16" else (10, -14)
    _, e = np.frexp(scale)                      # scale in [2^(e-1), 2^e)
    ulp = np.ldexp(1.0, np.maximum(e - 1, emin) - mant)
    print(f"{dtype} {out_f}x{in_f}x{tokens}: max result-ulp {d.max().item()}, "
          f"mismatch {frac:.2e}, max err/operand-ulp {np.max(err / ulp):.3f}")
    assert np.all(err <= 2 * ulp)
    assert frac <= 2e-3


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("out_f,in_f,tokens", [(256, 128, 64), (4096, 4096, 1024),
                                               (1000, 2816, 1000), (11008, 4096, 512)])
def test_gemm_update_equals_k6_grad_then_k1(dtype, out_f, in_f, tokens):
    """Identical gradients: K6 with LOMO_PROBE_KEEP_GRAD stores the rounded
    accumulator of the same mainloop K5 runs; K1 (f32 math) on that gradient
    must equal K5 bit for bit."""
    from paper_2306_09782_b200.engine import CudaEngine
    lib = U.lib()
    dt = U.CODE[dtype]
    g = torch.Generator(device="cuda").manual_seed(7 * out_f + tokens)
    p = torch.empty(out_f, in_f, device="cuda").uniform_(-0.08, 0.08, generator=g).to(dtype)
    dy = (torch.randn(tokens, out_f, device="cuda", generator=g) * 1e-2).to(dtype)
    x = torch.randn(tokens, in_f, device="cuda", generator=g).to(dtype)
    lr = 0.05 * 0.7
    q = p.clone()
    assert _run(p, dy, x, -lr, 1.0) == 0
    st = CudaEngine(torch.device("cuda", 0), 1)
    need = lib.lomo_gemm_probe_workspace(out_f, in_f, tokens, dt)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
    grad = torch.empty(out_f, in_f, dtype=dtype, device="cuda")
    assert lib.lomo_gemm_probe(dy.data_ptr(), x.data_ptr(), grad.data_ptr(), out_f, in_f, tokens,
                               dt, 0, _lib.PROBE_KEEP_GRAD, st.ptr, ws.data_ptr(), need,
                               U.stream()) == 0
    _lib.check(lib.lomo_fused_update(q.data_ptr(), grad.data_ptr(), q.numel(), dt, _lib.MATH_F32,
                                     lr, 0.0, 0.0, 0, None, U.stream()), "K1")
    torch.cuda.synchronize()
    d = U.ulp_diff(p, q)
    print(f"{dtype} {out_f}x{in_f}x{tokens}: K5 vs K6-grad->K1 max ulp {d.max().item()}")
    assert torch.equal(p, q)


def test_gemm_update_weight_decay_and_zero_alpha():
    g = torch.Generator(device="cuda").manual_seed(0)
    p = torch.empty(512, 256, device="cuda").uniform_(-0.08, 0.08, generator=g).to(torch.bfloat16)
    dy = torch.randn(128, 512, device="cuda", generator=g).to(torch.bfloat16)
    x = torch.randn(128, 256, device="cuda", generator=g).to(torch.bfloat16)
    before = p.clone()
    assert _run(p, dy, x, 0.0, 1.0) == 0           # skip-equivalent: p unchanged
    assert torch.equal(p, before)
    assert _run(p, dy, x, 0.0, 0.5) == 0           # pure decay
    assert torch.equal(p, (before.float() * 0.5).to(torch.bfloat16))


def test_gemm_update_rejects_bad_shapes():
    lib = U.lib()
    assert lib.lomo_gemm_update(None, None, None, 8, 8, 8, _lib.BF16, 1.0, 1.0, None, 0,
                                None) == -1
    p = torch.zeros(8, 8, dtype=torch.float32, device="cuda")
    assert lib.lomo_gemm_update(p.data_ptr(), p.data_ptr(), p.data_ptr(), 8, 8, 8, _lib.F32,
                                1.0, 1.0, None, 0, U.stream()) == -1  # fp32: not on K5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_lomo_replay_fused_gemm_matches_replay_k1(dtype):
    from paper_2306_09782_b200 import LOMO
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=128, layers=2, heads=4, ffn=256, vocab=256)
    # full-precision accumulation in cuBLAS for the unfused reference path
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    a = Llama(cfg, dtype=dtype, device="cuda", seed=0)
    b = Llama(cfg, dtype=dtype, device="cuda", seed=0)
    # a loss scale that keeps the 16-bit gradients of the unfused path out of
    # the fp16 subnormal range (there K1's rounded dW loses relative precision)
    scale = 2.0 ** 16 if dtype == torch.float16 else 2.0 ** 8
    oa = LOMO(a, lr=0.05, clip_grad_norm=0.3, loss_scale=scale, replay=True)
    ob = LOMO(b, lr=0.05, clip_grad_norm=0.3, loss_scale=scale, replay=True, fuse_gemm=True)
    gen = torch.Generator(device="cuda").manual_seed(4)
    d = torch.randint(0, 256, (2, 65), device="cuda", generator=gen)
    p0 = [p.detach().float().clone() for p in a.parameters()]
    la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
    lb = ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
    assert oa.last_outcome == ob.last_outcome and la == lb
    # identical protocol; the gradients differ only by cuBLAS's vs the
    # tcgen05 kernel's fp32 summation order before their rounding to 16 bits,
    # and alpha folds lr * coef / scale into one fp32 constant: within one ulp
    d = U.ulp_diff(torch.cat([x.detach().reshape(-1) for x in a.parameters()]),
                   torch.cat([y.detach().reshape(-1) for y in b.parameters()]))
    moved = torch.cat([(x.detach().float() - q).reshape(-1) != 0
                       for x, q in zip(a.parameters(), p0)])
    print(f"{dtype}: fused vs unfused max ulp {d.max().item()}, mean ulp "
          f"{d.double().mean().item():.2e}, {int(moved.sum())} elements moved")
    assert d.max().item() <= 1
    assert d.double().mean().item() <= 1e-3


# --- CUDA-graph capture of the replay step (graphs.py) -----------------------------

@pytest.mark.parametrize("fuse", [False, True])
def test_graphed_step_equals_eager_step(fuse):
    """The captured two-pass replay step reproduces the eager step exactly
    (same kernels; alpha/beta and lr read from device memory)."""
    from paper_2306_09782_b200 import LOMO
    from paper_2306_09782_b200.graphs import GraphedLOMOStep
    from paper_2306_09782_b200.workloads import Llama
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    cfg = dict(hidden=128, layers=2, heads=4, ffn=256, vocab=256)
    a = Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0)
    b = Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0)
    kw = dict(lr=0.05, clip_grad_norm=0.3, loss_scale=2.0 ** 8, replay=True, fuse_gemm=fuse)
    oa, ob = LOMO(a, **kw), LOMO(b, **kw)
    gen = torch.Generator(device="cuda").manual_seed(7)
    data = [torch.randint(0, 256, (2, 65), device="cuda", generator=gen) for _ in range(6)]
    static = data[0].clone()
    # the graph object runs 2 eager warm-up steps on data[0]: mirror them on `a`
    for _ in range(2):
        oa.step(lambda: a.loss(data[0][:, :-1], data[0][:, 1:]), 0.05)
    gs = GraphedLOMOStep(ob, lambda d: b.loss(d[:, :-1], d[:, 1:]), (static,), warmup=2, lr=0.05)
    for k in range(1, 6):
        lr = 0.05 / k                          # a schedule: lr comes from the state
        la = oa.step(lambda: a.loss(data[k][:, :-1], data[k][:, 1:]), lr)
        static.copy_(data[k])
        lb = gs.step(lr).item()
        assert oa.last_outcome == ob.last_outcome
        assert la == lb, (k, la, lb)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)


@pytest.mark.parametrize("fuse", [True, False])
def test_graphed_strict_fused_step_equals_eager(fuse):
    """The reference's two-pass protocol (pass 2 a second backward, no stash)
    with K6/K5 inside the backward, captured in two CUDA graphs: decisions
    and loss-scale trajectory equal to the eager step, parameters equal up to
    the second backward's attention nondeterminism."""
    from paper_2306_09782_b200 import LOMO
    from paper_2306_09782_b200.graphs import GraphedLOMOStep
    from paper_2306_09782_b200.workloads import Llama
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    cfg = dict(hidden=128, layers=2, heads=4, ffn=256, vocab=256)
    a = Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0, fused_proj=True)
    b = Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0, fused_proj=True)
    kw = dict(lr=0.05, clip_grad_norm=0.3, loss_scale=2.0 ** 8, fuse_gemm=fuse)
    oa, ob = LOMO(a, **kw), LOMO(b, **kw)
    gen = torch.Generator(device="cuda").manual_seed(7)
    data = [torch.randint(0, 256, (2, 65), device="cuda", generator=gen) for _ in range(6)]
    static = data[0].clone()
    for _ in range(2):
        oa.step(lambda: a.loss(data[0][:, :-1], data[0][:, 1:]), 0.05)
    gs = GraphedLOMOStep(ob, lambda d: b.loss(d[:, :-1], d[:, 1:]), (static,), warmup=2, lr=0.05)
    assert gs.strict
    for k in range(1, 6):
        lr = 0.05 / k
        la = oa.step(lambda: a.loss(data[k][:, :-1], data[k][:, 1:]), lr)
        static.copy_(data[k])
        lb = gs.step(lr).item()
        assert oa.last_outcome == ob.last_outcome
        assert abs(la - lb) <= 1e-3 * abs(la)
    assert oa.loss_scale == ob.loss_scale
    for x, y in zip(a.parameters(), b.parameters()):
        torch.testing.assert_close(x.float(), y.float(), rtol=2 ** -6, atol=1e-4)


def test_graphed_single_pass_fused_step_equals_eager():
    """LOMO's single fused pass (K5 inside the backward) captured as forward
    graph + host loss check + backward graph: losses and parameters equal
    to the eager single pass up to the attention backward's nondeterminism;
    a non-finite loss raises with every parameter untouched."""
    from paper_2306_09782_b200 import LOMO
    from paper_2306_09782_b200.errors import NonFiniteLossError
    from paper_2306_09782_b200.graphs import GraphedLOMOStep
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=128, layers=2, heads=4, ffn=256, vocab=256)
    a = Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0, fused_proj=True)
    b = Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0, fused_proj=True)
    oa, ob = LOMO(a, lr=0.05, fuse_gemm=True), LOMO(b, lr=0.05, fuse_gemm=True)
    gen = torch.Generator(device="cuda").manual_seed(9)
    data = [torch.randint(0, 256, (2, 65), device="cuda", generator=gen) for _ in range(6)]
    static = data[0].clone()
    poison = torch.ones((), device="cuda")
    for _ in range(2):
        oa.step(lambda: a.loss(data[0][:, :-1], data[0][:, 1:]), 0.05)
    gs = GraphedLOMOStep(ob, lambda d: b.loss(d[:, :-1], d[:, 1:]) * poison, (static,),
                         warmup=2, lr=0.05)
    assert gs.single
    for k in range(1, 6):
        lr = 0.05 / k
        la = oa.step(lambda: a.loss(data[k][:, :-1], data[k][:, 1:]), lr)
        static.copy_(data[k])
        lb = gs.step(lr).item()
        assert abs(la - lb) <= 1e-3 * abs(la)
    for x, y in zip(a.parameters(), b.parameters()):
        torch.testing.assert_close(x.float(), y.float(), rtol=2 ** -6, atol=1e-4)
    before = [p.detach().clone() for p in b.parameters()]
    poison.fill_(float("inf"))
    with pytest.raises(NonFiniteLossError):
        gs.step(0.05)
    assert all(torch.equal(p, q) for p, q in zip(before, b.parameters()))
