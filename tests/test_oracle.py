"""Pin the CPU oracle (oracle/lomo_oracle.py) to the reference's own outputs.

The fixtures under tests/golden were produced by running the reference
(fusedtrain) itself -- see tests/golden/make_golden.py.  When the reference is
mounted (build container) the oracle is also compared with it live.
"""
import json
import math

import numpy as np
import pytest
import torch

import lomo_oracle as O
from conftest import GOLDEN, case_arrays


# --- rounding ---------------------------------------------------------------

def test_round_through_half_matches_reference_fixture():
    r = np.load(GOLDEN / "rounding.npz")
    got = O.round_through_half(r["x"])
    want = r["half"]
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.array_equal(got[ok], want[ok])


def test_round_direct_binary16_equals_numpy_cast():
    r = np.load(GOLDEN / "rounding.npz")
    direct = O.round_direct(r["x"], 10, -14, 15)
    assert np.array_equal(direct, r["half"])


@pytest.mark.parametrize("value,want", [
    (65504.0, 65504.0), (65519.9, 65504.0), (65520.0, math.inf), (2.0 ** -24, 2.0 ** -24),
    (2.0 ** -25, 0.0), (1.5 * 2.0 ** -25, 2.0 ** -24), (-3.0e30, -math.inf),
])
def test_half_kat(value, want):  # test_tensor.py:19-42
    assert O.round_through_half(np.array([value]))[0] == want


def test_bf16_restatement_matches_torch_on_f32_inputs():
    # For inputs exactly representable in fp32, a direct f64->bf16 RNE must
    # equal torch's fp32->bf16 RNE cast (the bf16 rule has no reference).
    rng = np.random.default_rng(3)
    x32 = (rng.normal(0, 1, 200000) * np.exp2(rng.integers(-140, 128, 200000))).astype(np.float32)
    x32 = x32[np.isfinite(x32)]
    want = torch.from_numpy(x32).to(torch.bfloat16).to(torch.float64).numpy()
    got = O.round_through_bf16(x32.astype(np.float64))
    assert np.array_equal(got, want)


def test_bf16_direct_rounding_avoids_double_rounding():
    # a value just above a bf16 midpoint that rounds DOWN when first rounded
    # to fp32: direct rounding must round it up.
    one = 1.0
    mid = one + 2.0 ** -8           # midpoint between 1 and 1+2^-7
    x = mid + 2.0 ** -40            # above the midpoint -> rounds up directly
    assert O.round_through_bf16(np.array([x]))[0] == one + 2.0 ** -7
    assert O.round_through_bf16(np.array([mid]))[0] == one  # tie -> even


def test_bf16_overflow_to_inf():
    big = (2 - 2 ** -8) * 2.0 ** 127
    assert O.round_through_bf16(np.array([big]))[0] == math.inf
    assert O.round_through_bf16(np.array([-big]))[0] == -math.inf
    assert np.isnan(O.round_through_bf16(np.array([np.nan]))[0])


# --- hook cases: the oracle reproduces the reference bit for bit ---------------

def _replay_case(meta_case, arrays, nshapes, precision_override=None):
    name = meta_case["name"]
    prec = precision_override or meta_case["precision"]
    p, g = case_arrays(arrays, name, nshapes)
    params = list(p[0])
    clip = meta_case["clip"]
    sc_cfg = meta_case["scaler"]
    scaler = None
    if sc_cfg is not None:
        scaler = O.LossScaler(meta_case["init_scale"], sc_cfg["growth_interval"],
                              sc_cfg["min_scale"], sc_cfg["max_scale"])
    outs, scales, results = [], [], []
    two_pass = scaler is not None or (clip and clip["kind"] == "by_global_norm")
    threshold = clip["threshold"] if clip and clip["kind"] == "by_value" else None
    max_norm = clip["max_norm"] if clip and clip["kind"] == "by_global_norm" else None
    grouped = clip is not None and clip["kind"] == "by_group_norm"
    for k in range(meta_case["steps"]):
        loss = meta_case["losses"][k]
        if grouped:
            params, out = O.grouped_step(params, g[k], list(range(nshapes)), meta_case["lr"],
                                         prec, clip["max_norm"], clip["window"])
            outs.append("applied" if out == "applied" else "skipped_overflow")
        elif two_pass:
            if not math.isfinite(loss):
                ok = scaler.on_overflow() if scaler else True
                outs.append("skipped_overflow" if ok else "underflow")
            else:
                new, out, _, _ = O.two_pass_step(params, g[k], meta_case["lr"], prec, scaler,
                                                 max_norm, threshold)
                params = new
                outs.append({"applied": "applied", "skipped": "skipped_overflow",
                             "underflow": "underflow"}[out])
        else:
            if not math.isfinite(loss):
                outs.append("nonfinite_loss")
            else:
                params = [O.value_clip_update(pp, O.round_to(gg, prec), meta_case["lr"],
                                              threshold, prec) for pp, gg in zip(params, g[k])]
                outs.append("applied")
        scales.append(scaler.scale if scaler else None)
        results.append([x.copy() for x in params])
    return outs, scales, results, p


def test_oracle_reproduces_every_reference_hook_case(hook_cases):
    meta, arrays = hook_cases
    nshapes = len(meta["shapes"])
    for case in meta["cases"]:
        outs, scales, results, p = _replay_case(case, arrays, nshapes)
        want_outs = [o if not o.startswith("underflow") else "underflow" for o in case["outcomes"]]
        assert outs == want_outs, case["name"]
        if case["scaler"] is not None:
            assert scales == case["scales"], case["name"]
        for k in range(case["steps"]):
            for i in range(nshapes):
                assert np.array_equal(results[k][i], p[k + 1][i], equal_nan=True), \
                    (case["name"], k, i)


def test_scaler_replay_fixture():
    seqs = json.loads((GOLDEN / "scaler_replay.json").read_text())
    for s in seqs:
        sc = O.LossScaler(2.0 ** 6, s["growth"], 1.0, 2.0 ** 10)
        trace = []
        for ok in s["outcomes"]:
            if ok:
                sc.on_clean()
            elif not sc.on_overflow():
                trace.append(None)
                break
            trace.append(sc.scale)
        assert trace == s["trace"]


# --- live reference (build container only) ------------------------------------

def test_oracle_apply_update_matches_live_reference(reference):
    from fusedtrain.optim import apply_update
    from fusedtrain.tape import Parameter
    from fusedtrain.tensor import Precision, Tensor
    rng = np.random.default_rng(11)
    for prec, P in (("full", Precision.FULL), ("half", Precision.HALF_EMULATED)):
        p0 = O.round_to(rng.uniform(-0.08, 0.08, 50000), prec)
        g = O.round_to(rng.normal(0, 1e-3, 50000), prec)
        param = Parameter("w", 0, Tensor(p0, P))
        apply_update(param, g, 0.05)
        assert np.array_equal(param.value.data, O.apply_update(p0, g, 0.05, prec))


def test_oracle_probe_matches_live_reference_dot(reference):
    rng = np.random.default_rng(5)
    grads = [rng.normal(0, 1e-3, n) for n in (4096, 17, 300000)]
    ovf, sq = O.probe(grads, 1024.0, True)
    want = 0.0
    for g in grads:  # stabilize.py:199 verbatim arithmetic
        u = (g / 1024.0).ravel()
        want += float(np.dot(u, u))
    assert not ovf and sq == want
