"""Host-side logic on CPU: configuration mirrors, the C1 restatement's init and
tokens against the reference's recorded digests, hook delivery order."""
import hashlib

import numpy as np
import pytest
import torch

from paper_2306_09782_b200 import ClipMode, ConfigError, LossScaler, Stabilizer
from paper_2306_09782_b200.workloads import (MiniConfig, MiniTransformer, llama_param_count,
                                             llama_param_shapes, mean_cross_entropy,
                                             mini_transformer_init, round_half_np,
                                             sequence_copy_batch)


# --- stabilize.py validation mirror (test_stabilize.py:57-61,153-155,190-194) ----

def test_clip_threshold_must_be_positive():
    with pytest.raises(ConfigError):
        ClipMode.by_value(0.0)
    with pytest.raises(ConfigError):
        ClipMode.by_value(-1.0)
    with pytest.raises(ConfigError):
        ClipMode.by_global_norm(0.0)


def test_scale_must_be_power_of_two():
    with pytest.raises(ConfigError):
        LossScaler(scale=1000.0)
    with pytest.raises(ConfigError):
        LossScaler(scale=2.0 ** 30, max_scale=2.0 ** 24)
    with pytest.raises(ConfigError):
        LossScaler(growth_interval=0)


def test_grouped_does_not_combine_with_scaler():
    with pytest.raises(ConfigError):
        Stabilizer(ClipMode.by_group_norm(1.0, 1), LossScaler())


def test_pass_counts():
    assert Stabilizer(ClipMode.by_value(0.5)).backward_passes_per_step == 1
    assert Stabilizer(ClipMode.by_global_norm(1.0)).backward_passes_per_step == 2
    assert Stabilizer(ClipMode.none(), LossScaler()).backward_passes_per_step == 2
    assert Stabilizer(ClipMode.by_global_norm(1.0), LossScaler()).backward_passes_per_step == 2


# --- C1 restatement pinned to the reference run ---------------------------------

def _digest(named):
    h = hashlib.sha256()  # zoo.py:124-129
    for name, arr in named:
        h.update(name.encode())
        h.update(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
    return h.hexdigest()


def test_c1_init_matches_reference_digest(c1_meta):
    init = mini_transformer_init(MiniConfig())
    assert _digest(init) == c1_meta["A"]["init_digest"]
    assert _digest([(n, round_half_np(a)) for n, a in init]) == c1_meta["B"]["init_digest"]
    assert [n for n, _ in init] == c1_meta["A"]["names"]


def test_c1_tokens_match_reference(c1_meta):
    ids = sequence_copy_batch(0, 0, 4, 128, 1024)
    assert hashlib.sha256(np.ascontiguousarray(ids).tobytes()).hexdigest() == \
        c1_meta["tokens_step0_sha256"]


def test_slot_order_is_reference_delivery_order(c1_meta):
    """LOMO slots = reverse registration order == the reference tape's delivery
    order (tape.py:350-360), so the norm sums in the reference's order."""
    names = [n for n, _ in mini_transformer_init(MiniConfig())]
    assert list(reversed(names)) == c1_meta["delivery_order"]


def test_c1_first_loss_on_cpu_fp64(c1_meta):
    model = MiniTransformer(MiniConfig(), dtype=torch.float64, device="cpu")
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 4, 128, 1024))
    loss = mean_cross_entropy(model(ids), ids).item()
    assert abs(loss - c1_meta["A"]["losses"][0]) < 1e-12


def test_torch_hooks_fire_once_per_parameter_on_cpu():
    model = MiniTransformer(MiniConfig(layers=1, hidden=32, heads=2, vocab=64), torch.float64,
                            "cpu")
    fired = []
    for name, p in model.named_reference_parameters():
        p.register_post_accumulate_grad_hook(lambda t, n=name: fired.append(n))
    ids = torch.from_numpy(sequence_copy_batch(0, 0, 2, 8, 64))
    mean_cross_entropy(model(ids), ids).backward()
    assert sorted(fired) == sorted(n for n, _ in model.named_reference_parameters())
    assert len(fired) == len(set(fired))


def test_llama_shapes():
    assert llama_param_count("7b") == 6_738_415_616   # test_estimate.py:18-21
    assert len(llama_param_shapes("7b")) == 291
    assert llama_param_count("13b") == 13_015_864_320
    assert llama_param_count("65b") == 65_285_660_672


def test_dispatcher_chains_only_consecutive_k1_launches():
    """HookDispatcher(chain=True): LOMO_CHAINED on a K1 (K2) only when the
    previous launch of this dispatcher on the same stream was a K1 or K1
    multi (a K2 or K2 multi); the first launch of a pass, any launch after
    one of the other family, after a reconfigure or on another stream waits
    for its predecessor (no flag)."""
    import torch

    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.dispatch import HookDispatcher

    class Lib:
        def __init__(self):
            self.calls = []

        def lomo_fused_update(self, p, g, n, dt, math, lr, clip, wd, flags, state, stream):
            self.calls.append(("k1", flags, stream))
            return 0

        def lomo_fused_update_multi(self, ps, gs, ns, k, dt, math, lr, clip, wd, flags, state,
                                    stream):
            self.calls.append(("multi", flags, stream))
            return 0

        def lomo_probe(self, g, n, dt, slot, flags, state, stream):
            self.calls.append(("k2", flags, stream))
            return 0

    lib = Lib()
    d = HookDispatcher(lib, None, _lib.MATH_F32, small_numel=4, use_cpp=False)
    big, small = torch.zeros(16), torch.zeros(2)
    d.configure(lr=0.1, chain=True)
    d.update(big, big, _lib.F32, 7)      # first of the pass: waits
    d.update(big, big, _lib.F32, 7)      # chained
    d.update(small, small, _lib.F32, 7)  # parked
    d.flush(7)                           # K1 multi (never chained itself)
    d.update(big, big, _lib.F32, 7)      # after a K1 multi: chained
    d.update(big, big, _lib.F32, 8)      # another stream: waits
    d.probe(big, _lib.F32, 0, 8)         # after a K1: waits
    d.probe(big, _lib.F32, 1, 8)         # after a K2: chained
    d.update(big, big, _lib.F32, 8)      # after a probe: waits
    d.configure(lr=0.1, chain=True)
    d.update(big, big, _lib.F32, 8)      # after a reconfigure: waits
    d.configure(lr=0.1)
    d.update(big, big, _lib.F32, 8)
    d.update(big, big, _lib.F32, 8)      # chain off: never
    chained = [bool(f & _lib.CHAINED) for kind, f, _ in lib.calls]
    kinds = [kind for kind, _, _ in lib.calls]
    assert kinds == ["k1", "k1", "multi", "k1", "k1", "k2", "k2", "k1", "k1", "k1", "k1"]
    assert chained == [False, True, False, True, False, False, True, False, False, False, False]


def test_loss_scaler_host_state_machine_matches_reference_replays():
    """LossScaler is the reference's live object (stabilize.py:94-127):
    on_overflow / on_clean over the 300 recorded reference replays give the
    recorded scale trace, underflow raises ScaleUnderflowError."""
    import json

    from conftest import GOLDEN

    from paper_2306_09782_b200 import LossScaler
    from paper_2306_09782_b200.errors import ScaleUnderflowError
    seqs = json.loads((GOLDEN / "scaler_replay.json").read_text())
    assert len(seqs) == 300
    for s in seqs:
        sc = LossScaler(scale=2.0 ** 6, growth_interval=s["growth"], min_scale=1.0,
                        max_scale=2.0 ** 10)
        trace = []
        for ok in s["outcomes"]:
            try:
                sc.on_clean() if ok else sc.on_overflow()
            except ScaleUnderflowError:
                trace.append(None)
                break
            trace.append(sc.scale)
        assert trace == s["trace"]
    sc = LossScaler(scale=1024.0, growth_interval=4)
    sc.on_clean()
    assert sc.clean_steps == 1
    sc.on_overflow()
    assert sc.scale == 512.0 and sc.clean_steps == 0


def test_clip_by_value_kat_and_validation():
    """stabilize.py:82-86: KAT [1.3, 0.8] @ 1.0 -> [1.0, 0.8]; NaN stays NaN;
    a non-positive threshold is a ConfigError."""
    import math

    import torch

    from paper_2306_09782_b200 import ConfigError, clip_by_value
    out = clip_by_value(torch.tensor([1.3, 0.8, -2.5, float("nan")], dtype=torch.float64), 1.0)
    assert out[:3].tolist() == [1.0, 0.8, -1.0] and math.isnan(out[3].item())
    for t in (0.0, -1.0):
        with pytest.raises(ConfigError):
            clip_by_value(torch.zeros(2), t)


def test_step_batch_form_needs_a_model_loss():
    """step(batch, lr) maps (inputs, targets) to model.loss (optim.py:57-60);
    an optimizer whose model has no .loss raises TypeError, a closure passes
    through unchanged."""
    from types import SimpleNamespace

    from paper_2306_09782_b200.lomo import _as_closure
    f = lambda: 1.0  # noqa: E731
    assert _as_closure(SimpleNamespace(), f) is f
    with pytest.raises(TypeError):
        _as_closure(SimpleNamespace(_model=object()), (1, 2))
    m = SimpleNamespace(loss=lambda x, t: x + t)
    assert _as_closure(SimpleNamespace(_model=m), (1, 2))() == 3
