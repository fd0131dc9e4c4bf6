"""ShardedLOMO's gradient routing on CPU (gloo, one rank, the float64 CPU
engine of tests/cpu_engine.py): linear weight gradients GEMM'd straight into
the bucket buffer (``direct_grads``), a weight shared by two linears (the
later contribution added through its hook), and the replay mode refusing
such a weight.  The expected update is plain SGD on the autograd gradient."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

from paper_2306_09782_b200 import replay as R
from paper_2306_09782_b200.errors import ConfigError


@pytest.fixture(scope="module")
def gloo_world1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


class Layer(torch.nn.Module):
    def __init__(self, h, shared):
        super().__init__()
        self.w1 = torch.nn.Parameter(torch.randn(h, h, dtype=torch.float64) * 0.3)
        self.w2 = torch.nn.Parameter(torch.randn(h, h, dtype=torch.float64) * 0.3)
        self.scale = torch.nn.Parameter(torch.ones(h, dtype=torch.float64))
        self.shared = shared

    def forward(self, x):
        y = torch.tanh(R.linear(x, self.w1)) * self.scale
        return R.linear(y, self.w1 if self.shared else self.w2)


class Net(torch.nn.Module):
    def __init__(self, h=8, shared=False, seed=0):
        super().__init__()
        torch.manual_seed(seed)
        self.layers = torch.nn.ModuleList([Layer(h, shared), Layer(h, False)])

    def forward(self, x):
        for m in self.layers:
            x = m(x)
        return (x ** 2).mean()


def _sgd_reference(net, x, lr):
    loss = net(x)
    gs = torch.autograd.grad(loss, [p for p in net.parameters()], allow_unused=True)
    with torch.no_grad():
        for p, g in zip(net.parameters(), gs):
            if g is not None:
                p -= lr * g


@pytest.mark.parametrize("shared", [False, True])
@pytest.mark.parametrize("direct", [True, False])
def test_direct_gradients_match_sgd(gloo_world1, shared, direct):
    from cpu_engine import CpuEngine
    from paper_2306_09782_b200.sharded import ShardedLOMO
    a, b = Net(shared=shared), Net(shared=shared)
    x = torch.randn(5, 8, dtype=torch.float64, generator=torch.Generator().manual_seed(3))
    eng = CpuEngine(len(a.layers) + 1)
    opt = ShardedLOMO(a, lr=0.1, math="f64", _engine=eng, direct_grads=direct)
    for _ in range(2):
        opt.step(lambda: a(x), 0.1)
        _sgd_reference(b, x, 0.1)
    opt.gather_all()
    for (n, p), (_, q) in zip(a.named_parameters(), b.named_parameters()):
        assert torch.allclose(p, q, rtol=0, atol=1e-13), n
    opt.remove_hooks()


def test_replay_refuses_a_shared_weight(gloo_world1):
    from cpu_engine import CpuEngine
    from paper_2306_09782_b200 import ClipMode, Stabilizer
    from paper_2306_09782_b200.sharded import ShardedLOMO
    a = Net(shared=True)
    x = torch.randn(5, 8, dtype=torch.float64)
    eng = CpuEngine(len(a.layers) + 1, None, 1.0)
    opt = ShardedLOMO(a, lr=0.1, math="f64", _engine=eng, replay=True,
                      stabilizer=Stabilizer(ClipMode.by_global_norm(1.0)))
    with pytest.raises(ConfigError):
        opt.step(lambda: a(x), 0.1)
    opt.remove_hooks()
