"""End-to-end parity of the LOMO optimizer (autograd hooks -> C-ABI -> K1/K2/K3)
on config 1 (the reference's mini transformer), against fixtures recorded from
the reference itself (tests/golden/c1.*), plus the protocol invariants of
fusedtrain's tests (test_optim.py, test_stabilize.py, test_acceptance.py).

Tolerances (stated): fp32 storage -- per-step loss rel 1e-5 and final
parameters normwise-relative 1e-5 (north star "fp32 rel 1e-5"); fp64
storage + f64 math -- loss rel 1e-10, parameters abs 1e-12; fp16 -- every
overflow-skip / clip decision and the loss-scale trajectory identical, the
element error reported as max/mean ulp and bounded below.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2306_09782_b200 import (LOMO, ClipMode, LossScaler, NonFiniteLossError, Stabilizer,
                                   StepOutcome, TapeStateError)
from paper_2306_09782_b200.workloads import (MiniConfig, MiniTransformer, mean_cross_entropy,
                                             sequence_copy_batch)


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    torch.cuda.set_device(0)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False


C1 = MiniConfig(layers=2, hidden=256, heads=4, vocab=1024, seed=0)


def _tokens(step):
    return torch.from_numpy(sequence_copy_batch(0, step, 4, 128, 1024)).cuda()


def _run_c1(dtype, opt_kwargs, steps=10, math_mode="f32", fused_linear=False):
    model = MiniTransformer(C1, dtype=dtype, device="cuda", fused_linear=fused_linear)
    opt = LOMO(model, lr=0.05, math=math_mode, **opt_kwargs)
    losses, outcomes, scales = [], [], []
    for step in range(steps):
        ids = _tokens(step)
        loss = opt.step(lambda: mean_cross_entropy(model(ids), ids), 0.05)
        losses.append(loss)
        outcomes.append(opt.last_outcome.value if opt.last_outcome else "applied")
        scales.append(opt.loss_scale)
    return model, opt, losses, outcomes, scales


def _sampled(model, c1_arrays, key):
    out = {}
    for name, p in model.named_reference_parameters():
        idx = torch.from_numpy(c1_arrays[f"{key}/{name}/idx"]).cuda()
        out[name] = (p.detach().reshape(-1)[idx].double().cpu().numpy(),
                     c1_arrays[f"{key}/{name}/val"])
    return out


def test_c1_fixture_A_fp32(c1_meta, c1_arrays):
    model, opt, losses, _, _ = _run_c1(torch.float32, {})
    want = c1_meta["A"]["losses"]
    for got, ref in zip(losses, want):
        assert abs(got - ref) <= 1e-5 * abs(ref), (got, ref)
    worst = 0.0
    for name, (got, ref) in _sampled(model, c1_arrays, "A").items():
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        worst = max(worst, rel)
        assert rel <= 1e-5, (name, rel)
    print(f"fixture A fp32: worst normwise rel {worst:.2e}, "
          f"max |dloss|/loss {max(abs(a - b) / b for a, b in zip(losses, want)):.2e}")


def test_c1_fixture_A_fp64_f64_math(c1_meta, c1_arrays):
    model, _, losses, _, _ = _run_c1(torch.float64, {}, math_mode="f64")
    for got, ref in zip(losses, c1_meta["A"]["losses"]):
        assert abs(got - ref) <= 1e-10 * abs(ref), (got, ref)
    worst = 0.0
    for name, (got, ref) in _sampled(model, c1_arrays, "A").items():
        worst = max(worst, float(np.max(np.abs(got - ref))))
    assert worst <= 1e-12, worst
    print(f"fixture A fp64: max abs param error {worst:.2e}")


def _ulps16(got, ref):
    g = got.astype(np.float16).view(np.int16).astype(np.int64)
    r = ref.astype(np.float16).view(np.int16).astype(np.int64)
    g = np.where(g < 0, -(1 << 15) - g, g)
    r = np.where(r < 0, -(1 << 15) - r, r)
    return np.abs(g - r)


@pytest.mark.parametrize("key,scaler", [("B", LossScaler(2.0 ** 16, 2)),
                                        ("C", LossScaler(2.0 ** 24, 2, max_scale=2.0 ** 24))])
@pytest.mark.parametrize("math_mode", ["f32", "f64"])
def test_c1_fixture_fp16_two_pass(c1_meta, c1_arrays, key, scaler, math_mode):
    # a fresh scaler per run: LossScaler is the reference's live state
    # machine, and the optimizer mirrors the device's scale into it
    scaler = LossScaler(scaler.scale, scaler.growth_interval, max_scale=scaler.max_scale)
    stab = Stabilizer(ClipMode.by_global_norm(1.0), scaler)
    model, opt, losses, outcomes, scales = _run_c1(torch.float16, {"stabilizer": stab},
                                                   math_mode=math_mode)
    ref = c1_meta[key]
    assert outcomes == ref["outcomes"]                        # skip decisions: exact
    assert [math.log2(s) for s in scales] == ref["log2_scale"]  # scaler trajectory: exact
    u = np.concatenate([_ulps16(g, r) for g, r in _sampled(model, c1_arrays, key).values()])
    rel = max(abs(a - b) / abs(b) for a, b in zip(losses, ref["losses"]) if math.isfinite(b))
    print(f"fixture {key} fp16 ({math_mode} math): max ulp {u.max()}, mean ulp {u.mean():.4f}, "
          f">2ulp fraction {(u > 2).mean():.2e}, max loss rel {rel:.2e}")
    assert rel < 5e-3
    # measured (B200): max 15 / 9 ulp, mean 0.0154 / 0.0078 (f32 math);
    # the error is the torch fp16 forward/backward ops', not the update's
    assert u.mean() <= 0.02 and u.max() <= 16


@pytest.mark.parametrize("replay", [True, False])
@pytest.mark.parametrize("key,scaler", [("B", LossScaler(2.0 ** 16, growth_interval=2)),
                                        ("C", LossScaler(2.0 ** 24, growth_interval=2,
                                                         max_scale=2.0 ** 24))])
def test_c1_fixture_fp16_two_pass_fused_gemm(c1_meta, c1_arrays, key, scaler, replay):
    """The reference's own model (weights [in, out]) through the fused
    training path: K6 probes every weight gradient inside its GEMM in pass 1,
    K5 applies every update inside its GEMM in pass 2 (replayed, or in the
    strict second backward).  Fixtures B (norm clip + growing scale) and C
    (forced fp16 overflows): skip decisions and the scale trajectory equal the
    reference run's exactly; parameters carry the same error profile as the
    hook path (K5 rounds the accumulator to fp16 before the update)."""
    stab = Stabilizer(ClipMode.by_global_norm(1.0), LossScaler(
        scaler.scale, growth_interval=scaler.growth_interval, max_scale=scaler.max_scale))
    model, opt, losses, outcomes, scales = _run_c1(
        torch.float16, {"stabilizer": stab, "replay": replay, "fuse_gemm": True},
        fused_linear=True)
    assert opt.fuse_probe and opt.fuse_gemm
    ref = c1_meta[key]
    assert outcomes == ref["outcomes"]
    assert [math.log2(s) for s in scales] == ref["log2_scale"]
    u = np.concatenate([_ulps16(g, r) for g, r in _sampled(model, c1_arrays, key).values()])
    rel = max(abs(a - b) / abs(b) for a, b in zip(losses, ref["losses"]) if math.isfinite(b))
    print(f"fixture {key} fp16 fused GEMM path ({'replay' if replay else 'strict'}): "
          f"max ulp {u.max()}, mean ulp {u.mean():.4f}, >2ulp fraction {(u > 2).mean():.2e}, "
          f"max loss rel {rel:.2e}")
    assert rel < 5e-3
    # measured (B200): max 12 / 9 ulp, mean 0.0154 / 0.0079 -- the same
    # profile as the hook path (K5 rounds the accumulator to fp16 first,
    # tape.py:377, as K1 receives it)
    assert u.mean() <= 0.02 and u.max() <= 16


def test_lomo_equals_sgd_bit_exact_fp64():
    """test_optim.py:59-71 / criterion 1: fused update == materialise-then-SGD."""
    torch.use_deterministic_algorithms(True, warn_only=True)
    try:
        cfg = MiniConfig(layers=2, hidden=64, heads=4, vocab=128, seed=3)
        fused = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
        plain = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
        opt = LOMO(fused, lr=0.05, math="f64")
        for step in range(10):
            ids = torch.from_numpy(sequence_copy_batch(4, step, 4, 16, 128)).cuda()
            lf = opt.step(lambda: mean_cross_entropy(fused(ids), ids), 0.05)
            lp = mean_cross_entropy(plain(ids), ids)
            lp.backward()
            with torch.no_grad():
                for p in plain.parameters():
                    p.copy_(p - 0.05 * p.grad)  # two roundings, like optim.py:54
                    p.grad = None
            assert lf == lp.item()
        for a, b in zip(fused.parameters(), plain.parameters()):
            assert torch.equal(a, b)
    finally:
        torch.use_deterministic_algorithms(False)


def test_two_pass_with_huge_max_norm_equals_plain_step():
    """test_stabilize.py:85-91."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=1)
    a = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    b = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    oa = LOMO(a, lr=0.05, clip_grad_norm=1e9, math="f64")
    ob = LOMO(b, lr=0.05, math="f64")
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 16, 128)).cuda()
    oa.step(lambda: mean_cross_entropy(a(ids), ids), 0.05)
    ob.step(lambda: mean_cross_entropy(b(ids), ids), 0.05)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)


def test_gradient_peak_is_one_tensor():
    """test_optim.py:74-91: never two parameter gradients alive at once."""
    cfg = MiniConfig(layers=2, hidden=128, heads=4, vocab=512, seed=0)
    model = MiniTransformer(cfg, dtype=torch.float16, device="cuda")
    params = list(model.parameters())
    alive = []

    def checker(p):
        alive.append(sum(q.grad is not None for q in params))
    for p in params:
        p.register_post_accumulate_grad_hook(checker)   # runs before LOMO's hook
    opt = LOMO(model, lr=0.05)
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 32, 512)).cuda()
    opt.step(lambda: mean_cross_entropy(model(ids), ids), 0.05)
    assert alive and max(alive) == 1 and len(alive) == len(params)
    assert all(p.grad is None for p in params)
    assert opt.state_nbytes() == 0


def test_gradient_memory_peak_vs_retained_grads():
    cfg = MiniConfig(layers=4, hidden=512, heads=8, vocab=8192, seed=0)
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 1, 8, 8192)).cuda()
    sizes = []

    def peak_delta(use_lomo):
        model = MiniTransformer(cfg, dtype=torch.float16, device="cuda")
        sizes[:] = [p.numel() * 2 for p in model.parameters()]
        opt = LOMO(model, lr=0.05) if use_lomo else None
        loss = mean_cross_entropy(model(ids), ids)
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        if use_lomo:
            opt.fused_backward(loss, 0.05)
        else:
            loss.backward()
        torch.cuda.synchronize()
        return torch.cuda.max_memory_allocated() - base
    lomo, sgd = peak_delta(True), peak_delta(False)
    total, largest = sum(sizes), max(sizes)
    print(f"peak grad-phase delta: LOMO {lomo / 2**20:.1f} MiB, retained {sgd / 2**20:.1f} MiB, "
          f"largest tensor {largest / 2**20:.1f} MiB, all grads {total / 2**20:.1f} MiB")
    # LOMO holds at most the largest gradient above the post-forward level
    # (plus allocator rounding); retaining every gradient costs far more
    assert lomo <= largest + (1 << 20)
    assert sgd - lomo >= 0.5 * (total - largest)


def test_non_finite_loss_aborts_without_touching_params():
    """test_optim.py:162-170."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=0)
    model = MiniTransformer(cfg, dtype=torch.float32, device="cuda")
    before = [p.detach().clone() for p in model.parameters()]
    opt = LOMO(model, lr=0.05)
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 8, 128)).cuda()
    with pytest.raises(NonFiniteLossError):
        opt.step(lambda: mean_cross_entropy(model(ids), ids) * float("inf"), 0.05)
    for a, b in zip(before, model.parameters()):
        assert torch.equal(a, b)
    # the optimizer keeps working afterwards
    opt.step(lambda: mean_cross_entropy(model(ids), ids), 0.05)
    assert not all(torch.equal(a, b) for a, b in zip(before, model.parameters()))


@pytest.mark.parametrize("check_first", [True, False])
def test_two_pass_non_finite_loss_skips_before_backward(check_first):
    """stabilize.py:185-189: a non-finite loss skips the step (halving the
    scale) before any backward.  With the host check (the default) no hook
    runs; with the device flag alone the decision is the same."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=0)
    model = MiniTransformer(cfg, dtype=torch.float16, device="cuda")
    before = [p.detach().clone() for p in model.parameters()]
    opt = LOMO(model, lr=0.05, clip_grad_norm=1.0, loss_scale=LossScaler(2.0 ** 10))
    opt.check_loss_first = check_first
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 8, 128)).cuda()
    opt.step(lambda: mean_cross_entropy(model(ids), ids) * float("nan"), 0.05)
    assert opt.last_outcome == StepOutcome.SKIPPED_OVERFLOW
    assert opt.loss_scale == 2.0 ** 9
    assert (opt.hook_calls == 0) == check_first
    for a, b in zip(before, model.parameters()):
        assert torch.equal(a, b)
    assert all(p.grad is None for p in model.parameters())


def test_overflow_skip_leaves_params_byte_identical_and_halves_scale():
    """test_stabilize.py:233-240 / criterion 6."""
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=0)
    model = MiniTransformer(cfg, dtype=torch.float16, device="cuda")
    before = [p.detach().clone() for p in model.parameters()]
    opt = LOMO(model, lr=0.05, stabilizer=Stabilizer(
        ClipMode.none(), LossScaler(2.0 ** 24, max_scale=2.0 ** 24)))
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 8, 128)).cuda()
    opt.step(lambda: mean_cross_entropy(model(ids), ids) * 1e4, 0.05)
    assert opt.last_outcome is StepOutcome.SKIPPED_OVERFLOW
    assert opt.loss_scale == 2.0 ** 23
    for a, b in zip(before, model.parameters()):
        assert torch.equal(a, b)


def test_fused_backward_requires_grad_norm_in_two_pass_mode():
    cfg = MiniConfig(layers=1, hidden=32, heads=2, vocab=64, seed=0)
    model = MiniTransformer(cfg, dtype=torch.float32, device="cuda")
    opt = LOMO(model, lr=0.05, clip_grad_norm=1.0)
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 8, 64)).cuda()
    loss = mean_cross_entropy(model(ids), ids)
    with pytest.raises(TapeStateError):
        opt.fused_backward(loss, 0.05)
    norm = opt.grad_norm(loss)
    assert norm is not None and norm > 0
    opt.fused_backward(loss, 0.05)
    assert opt.last_outcome is StepOutcome.APPLIED


def test_recompute_forward_equals_retained_graph():
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=2)
    a = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    b = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    stab = lambda: Stabilizer(ClipMode.by_global_norm(0.05), LossScaler(2.0 ** 8, 2))
    oa = LOMO(a, lr=0.05, stabilizer=stab(), math="f64")
    ob = LOMO(b, lr=0.05, stabilizer=stab(), math="f64")
    for step in range(3):
        ids = torch.from_numpy(sequence_copy_batch(1, step, 2, 16, 128)).cuda()
        la = oa.step(lambda: mean_cross_entropy(a(ids), ids), 0.05)
        lb = ob.step(lambda: mean_cross_entropy(b(ids), ids), 0.05, recompute_forward=True)
        assert la == lb
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)


# --- grouped-norm clipping (stabilize.py:234-274) ------------------------------

def test_grouped_single_group_equals_two_pass_bit_exact():
    """test_stabilize.py:115-121: window covering every layer == global clip."""
    from paper_2306_09782_b200 import GroupedLOMO
    cfg = MiniConfig(layers=2, hidden=64, heads=2, vocab=128, seed=5)
    a = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    b = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    oa = GroupedLOMO(a, lr=0.05, max_norm=0.05, window=99, math="f64")
    ob = LOMO(b, lr=0.05, clip_grad_norm=0.05, math="f64")
    for step in range(3):
        ids = torch.from_numpy(sequence_copy_batch(2, step, 2, 16, 128)).cuda()
        oa.step(lambda: mean_cross_entropy(a(ids), ids), 0.05)
        ob.step(lambda: mean_cross_entropy(b(ids), ids), 0.05)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)


def test_grouped_window_one_matches_per_group_reference():
    """test_stabilize.py:124-141: every layer clipped by its own norm."""
    from paper_2306_09782_b200 import GroupedLOMO
    from paper_2306_09782_b200.grouped import infer_layers
    cfg = MiniConfig(layers=2, hidden=64, heads=2, vocab=128, seed=6)
    a = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    ref = MiniTransformer(cfg, dtype=torch.float64, device="cuda")
    layers = infer_layers(ref)
    opt = GroupedLOMO(a, lr=0.05, max_norm=0.02, window=1, math="f64")
    ids = torch.from_numpy(sequence_copy_batch(3, 0, 2, 16, 128)).cuda()
    opt.step(lambda: mean_cross_entropy(a(ids), ids), 0.05)
    mean_cross_entropy(ref(ids), ids).backward()
    groups = {}
    for p in ref.parameters():
        groups.setdefault(layers[id(p)], []).append(p)
    factors = set()
    with torch.no_grad():
        for ps in groups.values():
            n = torch.sqrt(sum((p.grad.double() ** 2).sum() for p in ps)).item()
            f = min(1.0, 0.02 / n) if n > 0 else 1.0
            factors.add(f)
            for p in ps:
                p.copy_(p - 0.05 * (p.grad * f))
    assert len(factors) > 1  # groups really got different factors
    for x, y in zip(a.parameters(), ref.parameters()):
        assert torch.allclose(x, y, rtol=0, atol=1e-15)
    assert opt.last_outcome is StepOutcome.APPLIED
    largest_group = max(sum(p.numel() * 8 for p in ps) for ps in groups.values())
    assert opt.peak_group_grads <= largest_group  # gradient peak = largest group


# --- per-layer activation checkpointing (tape.py:224-250, criterion 8) ----------

@pytest.mark.parametrize("two_pass", [False, True])
def test_checkpointing_is_transparent(two_pass):
    """test_acceptance.py:220-246: same bits with and without per-layer
    checkpointing; the recompute runs each layer's forward at most once more."""
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=3, heads=4, ffn=128, vocab=128)
    torch.use_deterministic_algorithms(True, warn_only=True)
    try:
        a = Llama(cfg, dtype=torch.float64, device="cuda", seed=0, checkpointing=False)
        b = Llama(cfg, dtype=torch.float64, device="cuda", seed=0, checkpointing=True)
        calls = {"n": 0}
        for layer in b.layers:
            layer.register_forward_pre_hook(lambda m, a_: calls.__setitem__("n", calls["n"] + 1))
        kw = dict(clip_grad_norm=0.5, loss_scale=2.0 ** 8) if two_pass else {}
        oa = LOMO(a, lr=0.05, math="f64", **kw)
        ob = LOMO(b, lr=0.05, math="f64", **kw)
        g = torch.Generator(device="cuda").manual_seed(3)
        for step in range(3):
            d = torch.randint(0, 128, (2, 17), device="cuda", generator=g)
            la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
            lb = ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
            assert la == lb
        for x, y in zip(a.parameters(), b.parameters()):
            assert torch.equal(x, y)
        passes = 2 if two_pass else 1
        # forward once + one recompute per backward pass, per layer
        assert calls["n"] == 3 * 3 * (1 + passes)
    finally:
        torch.use_deterministic_algorithms(False)


# --- pass-2 replay (replay.py) ---------------------------------------------------

@pytest.mark.parametrize("dtype,mode", [(torch.float64, "f64"), (torch.bfloat16, "f32")])
def test_replay_equals_second_backward(dtype, mode):
    """Replaying pass 2 from the stashed (x, dy) gives the very gradients a
    second backward produces: identical parameters (deterministic kernels)."""
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)
    torch.use_deterministic_algorithms(True, warn_only=True)
    try:
        a = Llama(cfg, dtype=dtype, device="cuda", seed=0)
        b = Llama(cfg, dtype=dtype, device="cuda", seed=0)
        oa = LOMO(a, lr=0.05, clip_grad_norm=0.3, loss_scale=2.0 ** 8, math=mode)
        ob = LOMO(b, lr=0.05, clip_grad_norm=0.3, loss_scale=2.0 ** 8, math=mode, replay=True)
        g = torch.Generator(device="cuda").manual_seed(4)
        for step in range(3):
            d = torch.randint(0, 128, (2, 17), device="cuda", generator=g)
            la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
            lb = ob.step(lambda: b.loss(d[:, :-1], d[:, 1:]), 0.05)
            assert la == lb and oa.last_outcome == ob.last_outcome
            assert ob.hook_calls == oa.hook_calls
        for x, y in zip(a.parameters(), b.parameters()):
            assert torch.equal(x, y)
        assert ob._stash.nbytes() == 0  # stash released after the replay
    finally:
        torch.use_deterministic_algorithms(False)


def test_replay_refuses_models_without_replayable_linears():
    from paper_2306_09782_b200 import ConfigError
    cfg = MiniConfig(layers=1, hidden=64, heads=2, vocab=128, seed=0)
    model = MiniTransformer(cfg, dtype=torch.float32, device="cuda")   # uses x @ W
    opt = LOMO(model, lr=0.05, clip_grad_norm=1.0, replay=True)
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 8, 128)).cuda()
    with pytest.raises(ConfigError):
        opt.step(lambda: mean_cross_entropy(model(ids), ids), 0.05)


def test_replay_refuses_tied_weights():
    """A weight used by the embedding AND a replayable linear would lose the
    embedding's contribution under replay: detected on the first step."""
    from paper_2306_09782_b200 import ConfigError
    from paper_2306_09782_b200.replay import linear as rlinear

    class Tied(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.emb = torch.nn.Parameter(torch.randn(64, 32, device="cuda") * 0.1)

        def forward(self, ids):
            return rlinear(torch.nn.functional.embedding(ids, self.emb), self.emb)

    m = Tied()
    opt = LOMO(m, lr=0.05, clip_grad_norm=1.0, replay=True)
    ids = torch.randint(0, 64, (2, 8), device="cuda")
    with pytest.raises(ConfigError):
        opt.step(lambda: mean_cross_entropy(m(ids), ids), 0.05)


@pytest.mark.parametrize("graphed", [False, True])
def test_loss_scaler_object_mirrors_the_device_state(graphed):
    """After every step the user's LossScaler reads as the reference's would:
    scale and clean_steps equal the device state machine's (halved on the
    forced overflows, doubled after growth_interval clean steps), without an
    extra host sync; eager and CUDA-graphed steps."""
    from paper_2306_09782_b200.graphs import GraphedLOMOStep
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)
    m = Llama(cfg, dtype=torch.float16, device="cuda", seed=0)
    sc = LossScaler(2.0 ** 22, growth_interval=2, max_scale=2.0 ** 24)
    opt = LOMO(m, lr=0.01, clip_grad_norm=1.0, loss_scale=sc, replay=graphed)
    assert opt.scaler is sc
    d = torch.randint(0, 128, (2, 33), device="cuda",
                      generator=torch.Generator(device="cuda").manual_seed(2))
    static = d.clone()
    if graphed:
        g = GraphedLOMOStep(opt, lambda x: m.loss(x[:, :-1], x[:, 1:]), (static,), warmup=1,
                            lr=0.01)
        step = lambda: g.step(0.01)  # noqa: E731
    else:
        step = lambda: opt.step(lambda: m.loss(static[:, :-1], static[:, 1:]), 0.01)  # noqa: E731
    seen = set()
    for _ in range(12):
        step()
        seen.add(opt.last_outcome)
        st = opt.read_status()
        assert (sc.scale, sc.clean_steps) == (st.scale, st.clean_steps)
    assert StepOutcome.SKIPPED_OVERFLOW in seen and StepOutcome.APPLIED in seen


def test_reference_style_step_batch_form():
    """step((inputs, targets), lr) -- the reference's LOMO.step(batch, lr)
    (optim.py:118-132, _forward_loss optim.py:57-60) -- equals
    step(closure, lr) bit for bit, single and two-pass."""
    from paper_2306_09782_b200 import GroupedLOMO
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)
    d = torch.randint(0, 128, (2, 33), device="cuda",
                      generator=torch.Generator(device="cuda").manual_seed(4))
    for kw in ({}, {"clip_grad_norm": 1.0, "loss_scale": LossScaler(2.0 ** 8)}, "grouped"):
        a = Llama(cfg, dtype=torch.float32, device="cuda", seed=0)
        b = Llama(cfg, dtype=torch.float32, device="cuda", seed=0)
        if kw == "grouped":
            oa, ob = (GroupedLOMO(m, lr=0.05, max_norm=1.0, window=1) for m in (a, b))
        else:
            oa = LOMO(a, lr=0.05, **kw)
            ob = LOMO(b, lr=0.05, **{k: (LossScaler(2.0 ** 8) if k == "loss_scale" else v)
                                     for k, v in kw.items()})
        for _ in range(2):
            la = oa.step(lambda: a.loss(d[:, :-1], d[:, 1:]), 0.05)
            lb = ob.step((d[:, :-1], d[:, 1:]), 0.05)
            assert la == lb
        for x, y in zip(a.parameters(), b.parameters()):
            assert torch.equal(x, y)
        oa.remove_hooks()
        ob.remove_hooks()
    with pytest.raises(TypeError):
        LOMO(torch.nn.Linear(4, 4).cuda(), lr=0.1).step((d, d), 0.1)


def test_stabilizer_run_step_carries_the_scaler_like_the_reference():
    """Stabilizer.run_step(model, batch, lr) (stabilize.py:148-153) and the
    reference's helpers (scaled_step, two_pass_norm_clip_step,
    grouped_norm_clip_step): a fresh optimizer per call, the scaler object
    carrying scale AND clean_steps between calls -- so a run of run_step
    calls equals one long-lived LOMO bit for bit, growth and skips included."""
    from paper_2306_09782_b200 import (grouped_norm_clip_step, scaled_step,
                                       two_pass_norm_clip_step)
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)
    a = Llama(cfg, dtype=torch.float16, device="cuda", seed=0)
    b = Llama(cfg, dtype=torch.float16, device="cuda", seed=0)
    sa = LossScaler(2.0 ** 21, growth_interval=2, max_scale=2.0 ** 24)
    sb = LossScaler(2.0 ** 21, growth_interval=2, max_scale=2.0 ** 24)
    oa = LOMO(a, lr=0.01, stabilizer=Stabilizer(ClipMode.by_global_norm(1.0), sa))
    stab_b = Stabilizer(ClipMode.by_global_norm(1.0), sb)
    g = torch.Generator(device="cuda").manual_seed(6)
    outs = []
    for _ in range(8):
        d = torch.randint(0, 128, (2, 33), device="cuda", generator=g)
        la = oa.step((d[:, :-1], d[:, 1:]), 0.01)
        lb, ob = stab_b.run_step(b, (d[:, :-1], d[:, 1:]), 0.01)
        assert la == lb and ob == oa.last_outcome
        assert (sa.scale, sa.clean_steps) == (sb.scale, sb.clean_steps)
        outs.append(ob)
    assert StepOutcome.APPLIED in outs
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)
    oa.remove_hooks()
    d = torch.randint(0, 128, (2, 33), device="cuda", generator=g)
    c = Llama(cfg, dtype=torch.float32, device="cuda", seed=0)
    assert math.isfinite(two_pass_norm_clip_step(c, (d[:, :-1], d[:, 1:]), 0.01, 1.0))
    assert math.isfinite(grouped_norm_clip_step(c, (d[:, :-1], d[:, 1:]), 0.01, 1.0, 1))
    loss, outcome = scaled_step(c, (d[:, :-1], d[:, 1:]), 0.01, LossScaler(2.0 ** 4))
    assert math.isfinite(loss) and outcome is StepOutcome.APPLIED


def test_reference_constructor_form():
    """LOMO(model, stabilizer) -- the reference's positional signature
    (optim.py:108-112), lr given to step -- equals the keyword form."""
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)
    a = Llama(cfg, dtype=torch.float32, device="cuda", seed=0)
    b = Llama(cfg, dtype=torch.float32, device="cuda", seed=0)
    oa = LOMO(a, Stabilizer(ClipMode.by_global_norm(1.0)), ledger=None)
    ob = LOMO(b, lr=0.05, clip_grad_norm=1.0)
    d = torch.randint(0, 128, (2, 33), device="cuda")
    assert oa.step((d[:, :-1], d[:, 1:]), 0.05) == ob.step((d[:, :-1], d[:, 1:]), 0.05)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)
    with pytest.raises(Exception):
        LOMO(a, Stabilizer(), stabilizer=Stabilizer())


def test_state_dict_resume_equals_uninterrupted_run():
    """LOMO.state_dict / load_state_dict (the optimizer's only state: the
    loss scaler's scale and clean-step count, and the step counters): a run
    checkpointed after 5 steps and resumed in a fresh optimizer on a copy
    of the weights equals the uninterrupted run bit for bit -- scales,
    outcomes (growth and overflow skips) and parameters."""
    from paper_2306_09782_b200.workloads import Llama
    cfg = dict(hidden=64, layers=2, heads=4, ffn=128, vocab=128)
    g = torch.Generator(device="cuda").manual_seed(8)
    batches = [torch.randint(0, 128, (2, 33), device="cuda", generator=g) for _ in range(10)]
    mk = lambda m: LOMO(m, lr=0.01, clip_grad_norm=1.0,  # noqa: E731
                        loss_scale=LossScaler(2.0 ** 21, growth_interval=2, max_scale=2.0 ** 24))
    a = Llama(cfg, dtype=torch.float16, device="cuda", seed=0)
    oa = mk(a)
    trace_a = []
    for d in batches:
        oa.step((d[:, :-1], d[:, 1:]), 0.01)
        trace_a.append((oa.last_outcome, oa.scaler.scale))
    b = Llama(cfg, dtype=torch.float16, device="cuda", seed=0)
    ob = mk(b)
    trace_b = []
    for d in batches[:5]:
        ob.step((d[:, :-1], d[:, 1:]), 0.01)
        trace_b.append((ob.last_outcome, ob.scaler.scale))
    sd = ob.state_dict()
    ob.remove_hooks()
    c = Llama(cfg, dtype=torch.float16, device="cuda", seed=0)
    with torch.no_grad():
        for x, y in zip(c.parameters(), b.parameters()):
            x.copy_(y)
    oc = mk(c)
    oc.load_state_dict(sd)
    assert (oc.scaler.scale, oc.scaler.clean_steps) == (sd["scale"], sd["clean_steps"])
    for d in batches[5:]:
        oc.step((d[:, :-1], d[:, 1:]), 0.01)
        trace_b.append((oc.last_outcome, oc.scaler.scale))
    assert trace_a == trace_b
    assert {o for o, _ in trace_a} == {StepOutcome.APPLIED, StepOutcome.SKIPPED_OVERFLOW}
    for x, y in zip(a.parameters(), c.parameters()):
        assert torch.equal(x, y)
    st = oc.read_status()
    assert st.steps_applied + st.steps_skipped == 10
