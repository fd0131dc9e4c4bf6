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


# --- more of the reference's test_stabilize.py, through the same public API --

class MLP(torch.nn.Module):
    """A small regression MLP (the reference's MLP_CFG / REG_TASK shape):
    loss = mean squared error; ``loss(x, t)`` is the step(batch) entry."""

    def __init__(self, dtype=torch.float64, seed=0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.w1 = torch.nn.Parameter((torch.rand(4, 16, generator=g, dtype=torch.float64) - .5)
                                     .to(dtype).cuda())
        self.w2 = torch.nn.Parameter((torch.rand(16, 1, generator=g, dtype=torch.float64) - .5)
                                     .to(dtype).cuda())

    def forward(self, x):
        return torch.tanh(x @ self.w1) @ self.w2

    def loss(self, x, t):
        return ((self(x) - t) ** 2).mean()


def _reg_batch(step, dtype=torch.float64):
    g = torch.Generator().manual_seed(100 + step)
    x = torch.rand(4, 4, generator=g, dtype=torch.float64)
    return x.to(dtype).cuda(), x.sum(1, keepdim=True).sin().to(dtype).cuda()


def test_value_clip_is_single_pass():
    """test_stabilize.py:64-70."""
    from paper_2306_09782_b200 import lomo_step
    stab = Stabilizer(ClipMode.by_value(0.5))
    assert stab.backward_passes_per_step == 1
    m = MLP()
    x, t = _reg_batch(0)
    calls = []
    m.register_forward_hook(lambda *a: calls.append(1))
    lomo_step(m, lambda: m.loss(x, t), 0.05, stabilizer=stab)
    assert len(calls) == 1


def test_two_pass_matches_clipped_sgd_oracle():
    """test_stabilize.py:75-82 (the reference: digest equality in f64; here
    f64 math, <= 1e-13 -- our fixed-order norm sum vs torch's)."""
    from paper_2306_09782_b200 import two_pass_norm_clip_step
    fused, oracle = MLP(), MLP()
    for step in range(20):
        x, t = _reg_batch(step)
        two_pass_norm_clip_step(fused, (x, t), 0.05, max_norm=1.0, math="f64")
        oracle.loss(x, t).backward()
        with torch.no_grad():
            n = math.sqrt(sum(float((p.grad ** 2).sum()) for p in oracle.parameters()))
            for p in oracle.parameters():
                p -= 0.05 * (p.grad * min(1.0, 1.0 / n))
                p.grad = None
    for a, b in zip(fused.parameters(), oracle.parameters()):
        assert (a - b).abs().max().item() < 1e-13


def test_two_pass_with_big_max_norm_equals_plain_step_batch_form():
    """test_stabilize.py:85-91."""
    from paper_2306_09782_b200 import lomo_step, two_pass_norm_clip_step
    clipped, plain = MLP(), MLP()
    x, t = _reg_batch(0)
    two_pass_norm_clip_step(clipped, (x, t), 0.05, max_norm=1e9, math="f64")
    lomo_step(plain, lambda: plain.loss(x, t), 0.05, math="f64")
    for a, b in zip(clipped.parameters(), plain.parameters()):
        assert torch.equal(a, b)


def test_two_pass_skips_on_non_finite_gradients_without_scaler():
    """test_stabilize.py:94-101: inf targets -> SKIPPED_OVERFLOW, params untouched."""
    m = MLP()
    before = [p.detach().clone() for p in m.parameters()]
    x, t = _reg_batch(0)
    _, outcome = Stabilizer(ClipMode.by_global_norm(1.0)).run_step(
        m, (x, torch.full_like(t, float("inf"))), 0.05)
    assert outcome is StepOutcome.SKIPPED_OVERFLOW
    for a, b in zip(before, m.parameters()):
        assert torch.equal(a, b)


def test_all_zero_gradients_are_a_noop():
    """test_stabilize.py:144-150: target == prediction -> every gradient 0."""
    from paper_2306_09782_b200 import grouped_norm_clip_step
    m = MLP()
    x, _ = _reg_batch(0)
    with torch.no_grad():
        perfect = m(x).clone()
    before = [p.detach().clone() for p in m.parameters()]
    grouped_norm_clip_step(m, (x, perfect), 0.05, max_norm=1.0, window=1)
    for a, b in zip(before, m.parameters()):
        assert torch.equal(a, b)


def test_scaler_grows_after_growth_interval_end_to_end():
    """test_stabilize.py:243-249: two clean fp16 steps at interval 2 double
    the scale -- read from the user's LossScaler object."""
    from paper_2306_09782_b200 import scaled_step
    m = MLP(dtype=torch.float16)
    scaler = LossScaler(scale=1024.0, growth_interval=2)
    for step in range(2):
        _, outcome = scaled_step(m, _reg_batch(step, torch.float16), 0.05, scaler)
        assert outcome is StepOutcome.APPLIED
    assert scaler.scale == 2048.0


def test_half_precision_scaled_run_tracks_full_run():
    """test_stabilize.py:252-263: fp16 + scaler vs fp64 plain within 1e-2."""
    from paper_2306_09782_b200 import lomo_step, scaled_step
    full, half = MLP(), MLP(dtype=torch.float16)
    scaler = LossScaler()
    for step in range(20):
        xf, tf = _reg_batch(step)
        loss_full = lomo_step(full, lambda: full.loss(xf, tf), 0.05, math="f64")
        loss_half, outcome = scaled_step(half, _reg_batch(step, torch.float16), 0.05, scaler)
        assert outcome is StepOutcome.APPLIED
    assert abs(loss_half - loss_full) / abs(loss_full) < 1e-2


def test_scaled_norm_clip_matches_unscaled_norm_clip_in_full_precision():
    """test_stabilize.py:275-285."""
    from paper_2306_09782_b200 import scaled_step, two_pass_norm_clip_step
    scaled, plain = MLP(), MLP()
    scaler = LossScaler(scale=2.0 ** 10)
    for step in range(5):
        batch = _reg_batch(step)
        scaled_step(scaled, batch, 0.05, scaler, ClipMode.by_global_norm(0.5), math="f64")
        two_pass_norm_clip_step(plain, batch, 0.05, max_norm=0.5, math="f64")
    for a, b in zip(scaled.parameters(), plain.parameters()):
        assert (a - b).abs().max().item() < 1e-12
