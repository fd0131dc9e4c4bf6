"""The benchmark decoder's fused layers (csrc/workload_kernels.cu) against a
plain PyTorch fp32 reference of the same op, forward and backward.

These kernels are not on the LOMO path; they make the config-3 training step
(workloads.Llama) GEMM-bound.  Tolerance: the fused kernels compute in fp32
and round once per output, so they are compared with the fp32 reference
rounded to the storage dtype at 2 ulp of the storage type (relative), plus an
absolute floor for values that cancel."""
import pytest
import torch

from paper_2306_09782_b200 import workloads as W

pytestmark = pytest.mark.gpu

DT = [torch.float16, torch.bfloat16]
ULP = {torch.float16: 2.0 ** -10, torch.bfloat16: 2.0 ** -7}


def close(got, want, dtype, k=2.0, floor=None):
    want = want.float()
    tol = k * ULP[dtype] * want.abs() + (floor if floor is not None else k * ULP[dtype] * want.abs().mean())
    err = (got.float() - want).abs()
    bad = (err > tol).sum().item()
    assert bad == 0, f"{bad} elements out of tolerance; max err {err.max().item():.3e}"


@pytest.fixture(autouse=True)
def _dev():
    torch.cuda.set_device(0)
    torch.manual_seed(0)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("rows,h", [(1, 8), (7, 4096), (1024, 4096), (33, 5120), (5, 8192), (3, 2056)])
def test_rmsnorm_fwd_bwd(dtype, rows, h):
    x = torch.randn(rows, h, device="cuda").to(dtype)
    w = (1 + 0.1 * torch.randn(h, device="cuda")).to(dtype)
    dy = torch.randn(rows, h, device="cuda").to(dtype)
    xa, wa = x.clone().requires_grad_(), w.clone().requires_grad_()
    y = W.rms_norm(xa, wa)
    y.backward(dy)
    # fp32 reference (the eager formula, all in fp32)
    xr, wr = x.float().requires_grad_(), w.float().requires_grad_()
    yr = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + W.RMSNORM_EPS) * wr
    yr.backward(dy.float())
    close(y, yr.detach(), dtype)
    close(xa.grad, xr.grad, dtype, k=4.0)
    close(wa.grad, wr.grad, dtype, k=4.0, floor=4 * ULP[dtype] * wr.grad.abs().max().item())


def test_rmsnorm_deterministic():
    x = torch.randn(1024, 4096, device="cuda").half().requires_grad_()
    w = torch.ones(4096, device="cuda").half().requires_grad_()
    dy = torch.randn(1024, 4096, device="cuda").half()
    out = []
    for _ in range(2):
        x.grad = w.grad = None
        W.rms_norm(x, w).backward(dy)
        out.append((x.grad.clone(), w.grad.clone()))
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])


def _cos_sin(s, dh, dtype):
    inv = 1.0 / (10000 ** (torch.arange(0, dh, 2, device="cuda", dtype=torch.float32) / dh))
    fr = torch.outer(torch.arange(s, device="cuda", dtype=torch.float32), inv)
    emb = torch.cat((fr, fr), -1)
    return emb.cos().to(dtype), emb.sin().to(dtype)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("b,s,nh,dh", [(1, 1024, 32, 128), (2, 17, 3, 64), (1, 5, 1, 16)])
def test_rope_fwd_bwd(dtype, b, s, nh, dh):
    cos, sin = _cos_sin(s, dh, dtype)
    q = torch.randn(b, s, nh, dh, device="cuda").to(dtype)
    k = torch.randn(b, s, nh, dh, device="cuda").to(dtype)
    dq = torch.randn_like(q)
    dk = torch.randn_like(k)
    qa, ka = q.clone().requires_grad_(), k.clone().requires_grad_()
    qo, ko = W.rope_qk(qa, ka, cos, sin)
    torch.autograd.backward((qo, ko), (dq, dk))
    qr, kr = q.float().requires_grad_(), k.float().requires_grad_()
    qro, kro = W.rope_qk(qr, kr, cos.float(), sin.float())      # eager formula in fp32
    torch.autograd.backward((qro, kro), (dq.float(), dk.float()))
    close(qo, qro.detach(), dtype)
    close(ko, kro.detach(), dtype)
    close(qa.grad, qr.grad, dtype)
    close(ka.grad, kr.grad, dtype)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [8, 1024 * 11008, 40])
def test_swiglu_fwd_bwd(dtype, n):
    g = (2 * torch.randn(n, device="cuda")).to(dtype)
    u = torch.randn(n, device="cuda").to(dtype)
    d = torch.randn(n, device="cuda").to(dtype)
    ga, ua = g.clone().requires_grad_(), u.clone().requires_grad_()
    out = W.swiglu(ga, ua)
    out.backward(d)
    gr, ur = g.float().requires_grad_(), u.float().requires_grad_()
    ref = torch.nn.functional.silu(gr) * ur
    ref.backward(d.float())
    close(out, ref.detach(), dtype, k=3.0)
    close(ga.grad, gr.grad, dtype, k=4.0)
    close(ua.grad, ur.grad, dtype, k=3.0)


@pytest.mark.parametrize("dtype", DT)
def test_llama_fused_layers_match_eager(dtype):
    """A 2-layer decoder with fused layers vs the same weights through the
    eager formulas: same loss to storage precision, gradients close."""
    cfg = dict(hidden=256, ffn=688, heads=4, vocab=512, layers=2)
    a = W.Llama(cfg, dtype=dtype, device="cuda", seed=0, fused_layers=True)
    b = W.Llama(cfg, dtype=dtype, device="cuda", seed=0, fused_layers=False)
    d = torch.randint(0, 512, (2, 65), device="cuda")
    la = a.loss(d[:, :-1], d[:, 1:])
    lb = b.loss(d[:, :-1], d[:, 1:])
    la.backward()
    lb.backward()
    assert abs(la.item() - lb.item()) <= 1e-2 * abs(lb.item())
    for (n, pa), pb in zip(a.named_parameters(), b.parameters()):
        ga, gb = pa.grad.float(), pb.grad.float()
        rel = (ga - gb).norm() / gb.norm().clamp_min(1e-30)
        assert rel < (2e-2 if dtype == torch.float16 else 6e-2), (n, rel.item())


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("rows,f", [(1, 8), (1024, 11008), (33, 40)])
def test_swiglu_fused_gate_up(dtype, rows, f):
    """SwiGLU over one [rows, 2f] gate/up projection (no split/cat copies)."""
    gu = (2 * torch.randn(rows, 2 * f, device="cuda")).to(dtype)
    d = torch.randn(rows, f, device="cuda").to(dtype)
    ga = gu.clone().requires_grad_()
    out = W._SwiGLUGuFn.apply(ga)
    out.backward(d)
    gr = gu.float().requires_grad_()
    ref = torch.nn.functional.silu(gr[:, :f]) * gr[:, f:]
    ref.backward(d.float())
    close(out, ref.detach(), dtype, k=3.0)
    close(ga.grad[:, :f], gr.grad[:, :f], dtype, k=4.0)
    close(ga.grad[:, f:], gr.grad[:, f:], dtype, k=3.0)


@pytest.mark.parametrize("dtype", DT)
def test_rope_fused_qkv(dtype):
    """Rotary over q/k read from a fused QKV projection, forward and backward,
    equals the contiguous kernels on split copies bit for bit; d(qkv) holds
    dq/dk/dv in their column blocks."""
    b, s, nh, dh = 2, 33, 4, 64
    h = nh * dh
    cos, sin = _cos_sin(s, dh, dtype)
    qkv = torch.randn(b, s, 3 * h, device="cuda").to(dtype).requires_grad_()
    qo, ko, v = W._QKVRopeFn.apply(qkv, cos, sin, nh)
    q0, k0, v0 = (t.detach().clone().requires_grad_() for t in qkv.split(h, -1))
    qc, kc = W.rope_qk(q0.view(b, s, nh, dh), k0.view(b, s, nh, dh), cos, sin)
    vc = v0.view(b, s, nh, dh).transpose(1, 2)
    assert torch.equal(qo, qc) and torch.equal(ko, kc) and torch.equal(v, vc)
    gq, gk = torch.randn_like(qo), torch.randn_like(ko)
    gv = torch.randn(b, nh, s, dh, device="cuda").to(dtype)
    torch.autograd.backward((qo, ko, v), (gq, gk, gv))
    torch.autograd.backward((qc, kc, vc), (gq, gk, gv))
    assert torch.equal(qkv.grad, torch.cat([q0.grad, k0.grad, v0.grad], -1))


@pytest.mark.parametrize("dtype", DT)
def test_llama_fused_projections_match_separate(dtype):
    """QKV / gate+up stacked in one weight each: the same model (weights
    copied across), loss to storage precision and gradients close -- the
    fused layout only changes which GEMMs run."""
    cfg = dict(hidden=256, ffn=688, heads=4, vocab=512, layers=2)
    a = W.Llama(cfg, dtype=dtype, device="cuda", seed=0, fused_proj=True)
    b = W.Llama(cfg, dtype=dtype, device="cuda", seed=0)
    with torch.no_grad():
        a.embed_tokens.copy_(b.embed_tokens)
        a.lm_head.copy_(b.lm_head)
        a.norm.weight.copy_(b.norm.weight)
        for la_, lb_ in zip(a.layers, b.layers):
            la_.qkv.copy_(torch.cat([lb_.q, lb_.k, lb_.v], 0))
            la_.gate_up.copy_(torch.cat([lb_.gate, lb_.up], 0))
            la_.o.copy_(lb_.o)
            la_.down.copy_(lb_.down)
            la_.input_layernorm.weight.copy_(lb_.input_layernorm.weight)
            la_.post_attention_layernorm.weight.copy_(lb_.post_attention_layernorm.weight)
    d = torch.randint(0, 512, (2, 65), device="cuda")
    la = a.loss(d[:, :-1], d[:, 1:])
    lb = b.loss(d[:, :-1], d[:, 1:])
    la.backward()
    lb.backward()
    assert abs(la.item() - lb.item()) <= 1e-2 * abs(lb.item())
    tol = 2e-2 if dtype == torch.float16 else 6e-2
    for la_, lb_ in zip(a.layers, b.layers):
        pairs = [(la_.qkv.grad, torch.cat([lb_.q.grad, lb_.k.grad, lb_.v.grad], 0)),
                 (la_.gate_up.grad, torch.cat([lb_.gate.grad, lb_.up.grad], 0)),
                 (la_.o.grad, lb_.o.grad), (la_.down.grad, lb_.down.grad)]
        for ga, gb in pairs:
            rel = (ga.float() - gb.float()).norm() / gb.float().norm().clamp_min(1e-30)
            assert rel < tol, rel.item()


def test_lomo_step_on_fused_projections():
    """The replay + K6/K5 LOMO step runs on the stacked weights (shapes
    3h x h and 2f x h) and agrees with the unfused-GEMM replay step."""
    from paper_2306_09782_b200 import LOMO
    cfg = dict(hidden=256, ffn=688, heads=4, vocab=512, layers=2)
    a = W.Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0, fused_proj=True)
    b = W.Llama(cfg, dtype=torch.bfloat16, device="cuda", seed=0, fused_proj=True)
    kw = dict(lr=0.05, clip_grad_norm=0.3, loss_scale=2.0 ** 8, replay=True)
    oa, ob = LOMO(a, **kw), LOMO(b, fuse_gemm=True, **kw)
    d = torch.randint(0, 512, (2, 65), device="cuda")
    oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
    ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
    assert oa.last_outcome == ob.last_outcome
    assert abs(oa.last_norm - ob.last_norm) <= 1e-5 * oa.last_norm
    for x, y in zip(a.parameters(), b.parameters()):
        torch.testing.assert_close(x.float(), y.float(), rtol=2 ** -7, atol=1e-6)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("rows,h", [(3, 8), (1024, 4096), (33, 2056)])
def test_add_rmsnorm_equals_add_then_norm(dtype, rows, h):
    """The fused residual add + RMSNorm (both directions) is bit-identical to
    the separate add followed by the fused RMSNorm: same roundings."""
    x = torch.randn(rows, h, device="cuda").to(dtype)
    r = torch.randn(rows, h, device="cuda").to(dtype)
    w = (1 + 0.1 * torch.randn(h, device="cuda")).to(dtype)
    dh = torch.randn(rows, h, device="cuda").to(dtype)
    dy = torch.randn(rows, h, device="cuda").to(dtype)
    xa, ra, wa = (t.clone().requires_grad_() for t in (x, r, w))
    ha, ya = W._AddRMSNormFn.apply(xa, ra, wa, W.RMSNORM_EPS)
    torch.autograd.backward((ha, ya), (dh, dy))
    xb, rb, wb = (t.clone().requires_grad_() for t in (x, r, w))
    hb = xb + rb
    yb = W.rms_norm(hb, wb)
    torch.autograd.backward((hb, yb), (dh, dy))
    assert torch.equal(ha, hb) and torch.equal(ya, yb)
    assert torch.equal(xa.grad, xb.grad) and torch.equal(ra.grad, rb.grad)
    assert torch.equal(wa.grad, wb.grad)


@pytest.mark.parametrize("dtype", DT)
def test_fused_decoder_residual_stream_is_exact(dtype):
    """The stacked-projection decoder threads the residual stream through the
    fused add+norm kernels; with every layer fused it equals the same layers
    called one by one (x + layer(x)) bit for bit, and per-layer activation
    checkpointing of the (x, pending) stream is transparent."""
    cfg = dict(hidden=256, ffn=688, heads=4, vocab=512, layers=3)
    m = W.Llama(cfg, dtype=dtype, device="cuda", seed=0, fused_proj=True)
    mc = W.Llama(cfg, dtype=dtype, device="cuda", seed=0, fused_proj=True, checkpointing=True)
    d = torch.randint(0, 512, (2, 65), device="cuda")
    la = m.loss(d[:, :-1], d[:, 1:])
    la.backward()
    lc = mc.loss(d[:, :-1], d[:, 1:])
    lc.backward()
    assert la.item() == lc.item()
    for p, q in zip(m.parameters(), mc.parameters()):
        assert torch.equal(p.grad, q.grad)
    # the unfused residual decomposition of the same model
    with torch.no_grad():
        x = torch.nn.functional.embedding(d[:, :-1], m.embed_tokens)
        cos, sin = m._cos_sin(64, x.device, x.dtype)
        for layer in m.layers:
            x = layer(x, cos, sin)
        ref = W.rlinear(W.rms_norm(x, m.norm.weight), m.lm_head)
        assert torch.equal(m(d[:, :-1]), ref)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("rows,V", [(1, 8), (1024, 32000), (37, 520)])
def test_cross_entropy_fused(dtype, rows, V):
    """The fused token cross entropy against torch's fp32 cross entropy of the
    same logits: loss to fp32 rounding, dlogits to 2 ulp of the storage type
    (with a loss-scale-like upstream gradient)."""
    x = (3 * torch.randn(rows, V, device="cuda")).to(dtype)
    t = torch.randint(0, V, (rows,), device="cuda")
    xa = x.clone().requires_grad_()
    la = W._CrossEntropyFn.apply(xa, t)
    (la * 1024.0).backward()
    xr = x.float().requires_grad_()
    lr_ = torch.nn.functional.cross_entropy(xr, t)
    (lr_ * 1024.0).backward()
    assert abs(la.item() - lr_.item()) <= 1e-5 * abs(lr_.item()) + 1e-6
    close(xa.grad, xr.grad, dtype, k=2.0, floor=1e-3 * xr.grad.abs().max().item())
