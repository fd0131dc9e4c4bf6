"""Host logic of the linears' backward context (replay.py) on CPU: what the
backward hands to the fused-GEMM callbacks (K6 probe / K5 update), what it
returns to autograd, what it stashes for pass-2 replay, and the shared-weight
detection.  The callbacks here are Python stand-ins; the kernels themselves
are tested on the GPU (tests/test_gpu_gemm_probe.py)."""
import pytest
import torch

from paper_2306_09782_b200 import replay as R


@pytest.fixture
def ctx():
    st = R.ReplayStash(keep=False)
    R._ACTIVE = st
    yield st
    R._ACTIVE = None


def _data(out_f=6, in_f=4, tokens=5, seed=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(tokens, in_f, generator=g, dtype=torch.float64, requires_grad=True)
    w = torch.randn(out_f, in_f, generator=g, dtype=torch.float64, requires_grad=True)
    return x, w


def test_no_context_is_plain_linear():
    x, w = _data()
    R.linear(x, w).sum().backward()
    xr, wr = (t.detach().clone().requires_grad_() for t in (x, w))
    torch.nn.functional.linear(xr, wr).sum().backward()
    assert torch.equal(x.grad, xr.grad) and torch.equal(w.grad, wr.grad)


def test_probe_callback_consumes_the_weight_gradient(ctx):
    x, w = _data()
    seen = {}

    def probe(wid, w_, x_, dy_):
        seen["dw"] = R.weight_grad(x_, dy_)
        seen["wid"] = wid
        return True

    ctx.probe = probe
    dy = torch.randn(5, 6, dtype=torch.float64)
    R.linear(x, w).backward(dy)
    assert w.grad is None                      # nothing delivered to autograd
    assert seen["wid"] == id(w) and ctx.probed == {id(w)}
    assert torch.allclose(seen["dw"], dy.t() @ x.detach())
    assert torch.allclose(x.grad, dy @ w.detach())
    assert ctx.linear == {}                    # keep=False: nothing stashed


def test_refused_callback_returns_the_gradient(ctx):
    x, w = _data()
    ctx.probe = lambda *a: False
    ctx.update = lambda *a: False
    dy = torch.randn(5, 6, dtype=torch.float64)
    R.linear(x, w).backward(dy)
    assert torch.allclose(w.grad, dy.t() @ x.detach())
    assert ctx.probed == set() and ctx.updated == set()


def test_update_callback_runs_after_dx_uses_the_old_weight(ctx):
    x, w = _data()
    w0 = w.detach().clone()

    def update(wid, w_, x_, dy_):       # an in-place update, like K5
        with torch.no_grad():
            w_.sub_(0.1 * R.weight_grad(x_, dy_))
        return True

    ctx.update = update
    dy = torch.randn(5, 6, dtype=torch.float64)
    R.linear(x, w).backward(dy)
    assert torch.allclose(x.grad, dy @ w0)     # dx saw the pre-update weight
    assert torch.allclose(w.detach(), w0 - 0.1 * dy.t() @ x.detach())
    assert w.grad is None and ctx.updated == {id(w)}


def test_replay_stash_and_shared_weight_detection():
    st = R.ReplayStash(keep=True)
    R._ACTIVE = st
    try:
        x, w = _data()
        (R.linear(x, w).sum() + R.linear(x * 2, w).sum()).backward()
    finally:
        R._ACTIVE = None
    assert st.shared == {id(w)}               # one weight, two linears
    assert id(w) in st.linear                  # (x, dy) kept for replay


def test_in_out_layout_swaps_roles(ctx):
    """x @ W with W [in, out] (the reference zoo layout): the callbacks get
    (dy, x) in place of (x, dy), so weight_grad and the fused kernels'
    out x in problem are W's own [in, out] shape."""
    g = torch.Generator().manual_seed(1)
    x = torch.randn(5, 4, generator=g, dtype=torch.float64, requires_grad=True)
    w = torch.randn(4, 6, generator=g, dtype=torch.float64, requires_grad=True)
    got = {}

    def probe(wid, w_, a, b):
        got["dw"] = R.weight_grad(a, b)
        return True

    ctx.probe = probe
    dy = torch.randn(5, 6, dtype=torch.float64)
    R.matmul_in_out(x, w).backward(dy)
    assert got["dw"].shape == w.shape
    assert torch.allclose(got["dw"], x.detach().t() @ dy)
    assert torch.allclose(x.grad, dy @ w.detach().t())
    assert w.grad is None
