"""The reference's own hot-path test cases, restated against the B200 path
(fusedtrain tests/test_optim.py and tests/test_stabilize.py, SURVEY.md section
4), with the same names so they read side by side."""
import math

import pytest
import torch

from paper_2306_09782_b200 import LOMO, LossScaler, Stabilizer, ClipMode
from paper_2306_09782_b200.stabilize import StepOutcome
from paper_2306_09782_b200.workloads import (MiniConfig, MiniTransformer, mean_cross_entropy,
                                             sequence_copy_batch)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    torch.cuda.set_device(0)


class ScalarModel(torch.nn.Module):
    """zoo/tests ScalarModel: y = w * x, loss = 0.5 * (y - t)^2 (test_optim.py:22-36)."""

    def __init__(self, w: float, dtype=torch.float64):
        super().__init__()
        self.w = torch.nn.Parameter(torch.tensor([w], dtype=dtype, device="cuda"))

    def loss(self, x, t):
        y = self.w * x
        return 0.5 * ((y - t) ** 2).sum()


def _scalar_batch(dtype=torch.float64):
    return (torch.tensor([3.0], dtype=dtype, device="cuda"),
            torch.tensor([0.0], dtype=dtype, device="cuda"))


def test_lomo_matches_sgd_on_scalar_case():
    """test_optim.py:33-36: w=2, x=3, t=0, lr=0.1 -> g=18, w'=0.2."""
    m = ScalarModel(2.0)
    opt = LOMO(m, lr=0.1, math="f64")
    x, t = _scalar_batch()
    loss = opt.step(lambda: m.loss(x, t), 0.1)
    assert loss == pytest.approx(18.0)
    assert m.w.item() == pytest.approx(0.2)
    assert m.w.item() == 2.0 - 0.1 * 18.0        # the reference's float64 sequence


@pytest.mark.parametrize("dtype,math_mode", [(torch.float64, "f64"), (torch.float32, "f32"),
                                             (torch.float16, "f32"), (torch.bfloat16, "f32")])
def test_zero_lr_leaves_parameters_unchanged(dtype, math_mode):
    """test_optim.py:39-44 (digest equality) on the zoo model, every storage dtype."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=0)
    m = MiniTransformer(cfg, dtype=dtype, device="cuda")
    before = [p.detach().clone() for p in m.parameters()]
    opt = LOMO(m, lr=0.0, math=math_mode)
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 4, 16, cfg.vocab)).cuda()
    opt.step(lambda: mean_cross_entropy(m(ids), ids), 0.0)
    for a, b in zip(before, m.parameters()):
        assert torch.equal(a, b)


def test_half_lomo_matches_half_sgd_within_tolerance():
    """test_optim.py:184-196: fp16 LOMO vs fp16 materialise-then-SGD within
    5e-3 relative after several steps."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=2)
    a = MiniTransformer(cfg, dtype=torch.float16, device="cuda")
    b = MiniTransformer(cfg, dtype=torch.float16, device="cuda")
    opt = LOMO(a, lr=0.05)
    for step in range(5):
        ids = torch.from_numpy(sequence_copy_batch(1, step, 4, 16, cfg.vocab)).cuda()
        opt.step(lambda: mean_cross_entropy(a(ids), ids), 0.05)
        mean_cross_entropy(b(ids), ids).backward()
        with torch.no_grad():
            for p in b.parameters():
                p.copy_((p.double() - 0.05 * p.grad.double()).to(p.dtype))
                p.grad = None
    for x, y in zip(a.parameters(), b.parameters()):
        rel = (x.double() - y.double()).norm() / y.double().norm()
        assert rel < 5e-3, rel.item()


def test_scaled_step_in_full_precision_equals_unscaled():
    """test_stabilize.py:218-230: fp64 storage, loss scale 2^14 vs plain LOMO:
    same losses, parameters within 1e-12, every step applied."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=3)
    scaled = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    plain = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    os_ = LOMO(scaled, lr=0.05, loss_scale=LossScaler(2.0 ** 14), math="f64")
    op = LOMO(plain, lr=0.05, math="f64")
    for step in range(5):
        ids = torch.from_numpy(sequence_copy_batch(4, step, 4, 16, cfg.vocab)).cuda()
        ls = os_.step(lambda: mean_cross_entropy(scaled(ids), ids), 0.05)
        lp = op.step(lambda: mean_cross_entropy(plain(ids), ids), 0.05)
        assert os_.last_outcome is StepOutcome.APPLIED
        assert ls == lp
    worst = max((x - y).abs().max().item() for x, y in zip(scaled.parameters(),
                                                          plain.parameters()))
    assert worst < 1e-12, worst


def test_two_pass_runs_two_backward_passes_of_hook_calls():
    """test_stabilize.py:103-110: norm clipping costs exactly two backward
    passes (every parameter's hook twice), no third."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=0)
    m = MiniTransformer(cfg, dtype=torch.float32, device="cuda")
    opt = LOMO(m, lr=0.05, stabilizer=Stabilizer(ClipMode.by_global_norm(1.0)))
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 4, 16, cfg.vocab)).cuda()
    opt.step(lambda: mean_cross_entropy(m(ids), ids), 0.05)
    assert opt.passes == 2
    assert opt.hook_calls == 2 * len(list(m.parameters()))
    assert math.isfinite(opt.last_norm) and opt.last_norm > 0
