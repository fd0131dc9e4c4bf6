"""GPU parity of the sm_100a kernels (K1/K2/K3) against the CPU oracle and the
reference's own recorded behaviour (tests/golden/hook_cases.*), through the C-ABI.

Tolerances (stated here, north star): f64 arithmetic mode is bit-exact
against the float64 oracle (the reference's own arithmetic, optim.py:9-13)
except where a global-norm coefficient enters (our deterministic f64
reduction order differs from BLAS ddot: <= 1 ulp); f32 arithmetic mode is
within 1 ulp per element of the oracle (north star: 2 ulp) with the
mismatch fraction reported.  Overflow-skip and clip decisions: identical.
"""
import math

import numpy as np
import pytest
import torch

import lomo_oracle as O
from conftest import case_arrays

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import gpu_util as U
    from paper_2306_09782_b200 import _lib


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    torch.cuda.set_device(0)


PRECS = ["half", "bf16", "f32"]


def _expected(p, g, prec, lr=0.05, clip=None, inv_scale=None, coef=None, wd=0.0):
    """The reference hook arithmetic (stabilize.py:217-224, optim.py:52-54) in f64."""
    g = np.asarray(g, np.float64)
    p = np.asarray(p, np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        if inv_scale is not None:
            g = g * inv_scale
        if clip is not None:
            g = np.clip(g, -clip, clip)
        if coef is not None:
            g = g * coef
        if wd:
            p = p * (1.0 - lr * wd)
        return O.round_to(p - lr * g, prec)


def _draw(n, prec, rng, gscale=1e-3):
    p = O.round_to(rng.uniform(-0.08, 0.08, n), prec)
    g = O.round_to(rng.normal(0, gscale, n), prec)
    return p, g


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", [1, 7, 8, 9, 4095, 4096, 4097, (1 << 20) + 3])
@pytest.mark.parametrize("offset", [0, 3])
def test_k1_plain_update_f64_math_bit_exact(prec, n, offset):
    rng = np.random.default_rng(n + offset)
    p0, g0 = _draw(n, prec, rng)
    dt = U.TORCH_DT[prec]
    p, g = U.to_dev(p0, dt, offset), U.to_dev(g0, dt, offset)
    U.fused_update(p, g, math="f64")
    got = p.double().cpu().numpy()
    assert np.array_equal(got, _expected(p0, g0, prec))


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", [5, 4097, 3 * (1 << 20) + 1])
def test_k1_plain_update_f32_math_within_one_ulp(prec, n):
    rng = np.random.default_rng(n)
    p0, g0 = _draw(n, prec, rng)
    dt = U.TORCH_DT[prec]
    p, g = U.to_dev(p0, dt), U.to_dev(g0, dt)
    U.fused_update(p, g, math="f32")
    want = U.to_dev(_expected(p0, g0, prec), dt)
    d = U.ulp_diff(p, want)
    frac = (d > 0).float().mean().item()
    print(f"{prec} n={n}: max ulp {d.max().item()}, mismatch fraction {frac:.2e}")
    if prec == "f32":
        # fp32 storage: the fp32 constant lr and one FMA rounding; where p and
        # lr*g cancel the result-ulp error grows, so bound the error by the
        # operands' magnitude (2 ulp of max(|p|, |lr g|)), i.e. fp32 rel 1e-7
        err = (p.double() - want.double()).abs().cpu().numpy()
        bound = 2 * np.spacing(np.maximum(np.abs(p0), np.abs(0.05 * g0)).astype(np.float32))
        assert np.all(err <= bound)
    else:
        assert d.max().item() <= 1


def test_k1_misaligned_pair_takes_scalar_path_and_matches():
    rng = np.random.default_rng(1)
    n = 100001
    p0, g0 = _draw(n, "half", rng)
    p, g = U.to_dev(p0, torch.float16, 1), U.to_dev(g0, torch.float16, 4)
    U.fused_update(p, g, math="f64")
    assert np.array_equal(p.double().cpu().numpy(), _expected(p0, g0, "half"))


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("math_mode", ["f64", "f32"])
def test_k1_all_stages(prec, math_mode):
    """unscale -> value clip -> coef -> weight decay -> update, flags from state."""
    rng = np.random.default_rng(7)
    n = 1 << 18
    scale = 2.0 ** 12
    p0 = O.round_to(rng.uniform(-0.08, 0.08, n), prec)
    g0 = O.round_to(rng.normal(0, 1e-3, n) * scale, prec)
    dt = U.TORCH_DT[prec]
    st = U.State(1, scale=scale)
    coef = 0.731
    st.write_header(clip_coef=coef)
    for wd in (0.0, 0.1):
        p, g = U.to_dev(p0, dt), U.to_dev(g0, dt)
        U.fused_update(p, g, math=math_mode, clip=1.5e-3, wd=wd,
                       flags=_lib.USE_SCALE | _lib.USE_COEF | _lib.USE_SKIP, state=st)
        want = U.to_dev(_expected(p0, g0, prec, clip=1.5e-3, inv_scale=1 / scale, coef=coef,
                                  wd=wd), dt)
        d = U.ulp_diff(p, want)
        if math_mode == "f64":
            assert d.max().item() == 0, (wd, d.max().item())
        elif prec == "f32":
            err = (p.double() - want.double()).abs().cpu().numpy()
            assert np.all(err <= 4e-7 * (np.abs(p0) + 0.05 * 1.5e-3)), wd
        else:
            assert d.max().item() <= 1, (wd, d.max().item())


def _record(st):
    """The 16-byte pass-2 record after the header: (skip, inv_scale, coef, lr) as fp32."""
    torch.cuda.synchronize()
    raw = st.buf[_lib.STATE_HEADER_BYTES:_lib.STATE_HEADER_BYTES + 16].cpu()
    skip = int(raw[:4].view(torch.int32).item())
    f = raw[4:16].view(torch.float32).numpy()
    return skip, float(f[0]), float(f[1]), float(f[2])


def _want_record(h):
    return (h.skip, float(np.float32(h.inv_scale)), float(np.float32(h.clip_coef)),
            float(np.float32(h.lr)))


def test_pass2_record_is_republished_by_every_state_kernel():
    """The fp32 K1 reads skip / 1/scale / coef / lr from the record; every
    kernel that changes one of those header fields must republish it."""
    st = U.State(2, scale=2.0 ** 10, growth=1, max_norm=1.0)
    assert _record(st) == _want_record(st.status())                    # init
    _lib.check(U.lib().lomo_set_lr(st.ptr, 0.0123, U.stream()), "lr")
    assert _record(st) == _want_record(st.status()) and _record(st)[3] == np.float32(0.0123)
    g = torch.full((1000,), 3.0, dtype=torch.float16, device="cuda") * 2 ** 10
    st.begin()
    st.probe(g, 0, _lib.USE_SCALE)
    st.finalize()                                                      # coef < 1
    h = st.status()
    assert 0 < h.clip_coef < 1 and _record(st) == _want_record(h)
    st.on_clean()                                                      # growth: scale x2
    h = st.status()
    assert h.scale == 2.0 ** 11 and _record(st) == _want_record(h)
    st.begin(torch.tensor(float("inf"), device="cuda"))                # non-finite loss
    h = st.status()
    assert h.skip == 1 and _record(st) == _want_record(h)
    st.begin()
    g[3] = float("nan")
    st.probe(g, 1, _lib.USE_SCALE)
    st.finalize()                                                      # overflow: halve, skip
    h = st.status()
    assert h.skip == 1 and h.scale == 2.0 ** 10 and _record(st) == _want_record(h)


def test_k1_skip_flag_is_a_noop():
    rng = np.random.default_rng(3)
    p0, g0 = _draw(50000, "half", rng)
    p, g = U.to_dev(p0, torch.float16), U.to_dev(g0, torch.float16)
    st = U.State(1)
    st.write_header(skip=1)
    U.fused_update(p, g, flags=_lib.USE_SKIP, state=st)
    assert np.array_equal(p.double().cpu().numpy(), p0)
    U.fused_update(p, g, flags=0, state=st)  # without USE_SKIP it applies
    assert not np.array_equal(p.double().cpu().numpy(), p0)


def test_k1_value_clip_propagates_nan_and_kat():
    # stabilize.py:82-86 KAT [1.3, 0.8] @ 1.0 -> [1.0, 0.8]; np.clip keeps NaN
    p = torch.zeros(4, dtype=torch.float64, device="cuda")
    g = torch.tensor([1.3, 0.8, -2.5, float("nan")], dtype=torch.float64, device="cuda")
    U.fused_update(p, g, math="f64", lr=1.0, clip=1.0)
    got = p.cpu().numpy()
    assert np.array_equal(got[:3], [-1.0, -0.8, 1.0]) and np.isnan(got[3])


def test_k1_scalar_kat():
    # test_optim.py:25-36: w=2, x=3, t=0 -> g=18, lr=0.1 -> w'=0.2
    p = torch.tensor([2.0], dtype=torch.float64, device="cuda")
    g = torch.tensor([18.0], dtype=torch.float64, device="cuda")
    U.fused_update(p, g, math="f64", lr=0.1)
    assert p.item() == 2.0 - 0.1 * 18.0


def test_k1_zero_lr_and_empty():
    rng = np.random.default_rng(9)
    p0, g0 = _draw(1000, "bf16", rng)
    p, g = U.to_dev(p0, torch.bfloat16), U.to_dev(g0, torch.bfloat16)
    U.fused_update(p, g, lr=0.0)
    assert np.array_equal(p.double().cpu().numpy(), p0)
    e = torch.empty(0, dtype=torch.bfloat16, device="cuda")
    U.fused_update(e, e)


def test_k1_fp16_overflow_to_inf_on_store():
    p = torch.tensor([65504.0, -65504.0, 1.0], dtype=torch.float16, device="cuda")
    g = torch.tensor([-1000.0, 1000.0, 0.0], dtype=torch.float16, device="cuda")
    U.fused_update(p, g, math="f64", lr=1.0)
    assert p[0].item() == math.inf and p[1].item() == -math.inf and p[2].item() == 1.0


def test_k1_f64_math_rounds_directly_not_through_fp32():
    """f64 -> f16 must be ONE rounding (numpy's cast, tensor.py:38).  On 1M
    random updates a double rounding through fp32 differs somewhere; the
    device result must match the direct rounding everywhere."""
    rng = np.random.default_rng(99)
    n = 1 << 20
    rng.uniform(size=3 * n)  # (same draws as the probe that found such cases)
    p0 = O.round_to(rng.uniform(-2.0, 2.0, n), "half")
    g0 = O.round_to(rng.normal(0, 0.3, n), "half")
    exact = p0 - 0.0123 * g0
    direct = O.round_through_half(exact)
    double = O.round_through_half(exact.astype(np.float32).astype(np.float64))
    assert (direct != double).sum() > 0  # the test has power
    p, g = U.to_dev(p0, torch.float16), U.to_dev(g0, torch.float16)
    U.fused_update(p, g, math="f64", lr=0.0123)
    assert np.array_equal(p.double().cpu().numpy(), direct)


# --- K2 probe ----------------------------------------------------------------

@pytest.mark.parametrize("accum", [0, 0x8])
@pytest.mark.parametrize("prec", ["half", "bf16", "f32", "full"])
@pytest.mark.parametrize("n", [1, 9, 4096, 1000003, 4096 * 11008])
def test_k2_sumsq_and_determinism(prec, n, accum):
    rng = np.random.default_rng(n)
    scale = 1024.0 if prec in ("half", "bf16") else 1.0
    g0 = O.round_to(rng.normal(0, 1e-3, n) * scale, prec)
    g = U.to_dev(g0, U.TORCH_DT[prec], offset=n % 5)
    st = U.State(2, scale=scale if scale != 1.0 else 0.0)
    flags = (_lib.USE_SCALE if scale != 1.0 else 0) | accum
    st.begin()
    st.probe(g, 0, flags)
    st.probe(g, 1, flags)
    s = st.slots(2)
    ovf, want = O.probe([g0], scale, True)
    assert not ovf and st.status().overflow == 0
    assert s[0] == s[1]  # deterministic, run to run
    tol = 1e-12 if prec in ("f32", "full") or accum else 2e-6
    assert abs(s[0] - want) <= tol * want, (s[0], want)


@pytest.mark.parametrize("prec", ["half", "bf16", "f32"])
@pytest.mark.parametrize("pos", ["head", "middle", "tail"])
@pytest.mark.parametrize("bad", [math.inf, -math.inf, math.nan])
def test_k2_overflow_flag(prec, pos, bad):
    n = 100003
    g0 = np.full(n, 1e-3)
    idx = {"head": 0, "middle": n // 2, "tail": n - 1}[pos]
    g0[idx] = bad
    g = U.to_dev(O.round_to(g0, prec), U.TORCH_DT[prec], offset=1)
    st = U.State(1)
    st.begin()
    st.probe(g, 0, 0)
    assert st.status().overflow == 1


@pytest.mark.parametrize("accum", [0, 0x8])
def test_k2_large_finite_fp16_does_not_flag(accum):
    g = torch.full((4097,), 65504.0, dtype=torch.float16, device="cuda")
    st = U.State(1)
    st.begin()
    st.probe(g, 0, accum)
    status = st.status()
    assert status.overflow == 0
    want = 4097 * 65504.0 ** 2
    got = st.slots(1)[0]
    # f64 accumulation is exact here; the default fp32-per-vector partial
    # sums round at 2^-24 relative
    assert got == want if accum else abs(got - want) <= 8 * 2 ** -24 * want


# --- K3 ------------------------------------------------------------------------

def test_k3_scaler_replay_matches_reference_fixture():
    import json
    from conftest import GOLDEN
    seqs = json.loads((GOLDEN / "scaler_replay.json").read_text())
    inf = torch.tensor(float("inf"), device="cuda")
    zero = torch.tensor(0.5, device="cuda")
    assert len(seqs) == 300
    for s in seqs:  # every recorded replay
        st = U.State(1, scale=2.0 ** 6, growth=s["growth"], min_scale=1.0, max_scale=2.0 ** 10)
        trace = []
        for ok in s["outcomes"]:
            st.begin(zero if ok else inf)  # a non-finite loss forces the overflow path
            st.finalize()
            st.on_clean()
            h = st.status()
            if h.underflow:
                trace.append(None)
                break
            assert h.skip == (0 if ok else 1)
            trace.append(h.scale)
            assert h.scale_f32 == h.scale and h.inv_scale == 1.0 / h.scale
        assert trace == s["trace"]


def test_k3_norm_decision():
    g = torch.full((10000,), 0.01, dtype=torch.float64, device="cuda")  # N = 1.0
    for max_norm, coef in ((0.5, 0.5), (2.0, 1.0)):
        st = U.State(3, max_norm=max_norm)
        st.begin()
        st.probe(g, 0, 0)
        st.probe(g, 2, 0)  # slot 1 unused -> stays 0 (begin_step zeroes it)
        st.finalize()
        h = st.status()
        assert abs(h.total_norm - math.sqrt(2.0)) < 1e-12
        assert h.clip_coef == min(1.0, max_norm / h.total_norm)
        assert h.skip == 0
    # zero gradients: N = 0 -> coef 1 (stabilize.py:212)
    st = U.State(1, max_norm=1.0)
    st.begin()
    st.probe(torch.zeros(100, dtype=torch.float32, device="cuda"), 0, 0)
    st.finalize()
    assert st.status().clip_coef == 1.0


def test_k3_rank_combination_is_rank_ordered():
    st = U.State(1, max_norm=1.0)
    parts = torch.tensor([[0.25, 0.0], [0.5, 0.0], [0.25, 0.0]], dtype=torch.float64,
                         device="cuda")
    st.begin()
    _lib.check(U.lib().lomo_finalize_norm_ranks(st.ptr, parts.data_ptr(), 3, U.stream()), "r")
    h = st.status()
    assert h.sumsq_total == 1.0 and h.clip_coef == 1.0 and h.skip == 0
    parts[1, 1] = 1.0  # one rank saw a non-finite gradient
    st.begin()
    _lib.check(U.lib().lomo_finalize_norm_ranks(st.ptr, parts.data_ptr(), 3, U.stream()), "r")
    assert st.status().skip == 1


def test_multi_tensor_update_matches_single():
    rng = np.random.default_rng(12)
    sizes = [4096, 4096, 17, 4096 * 3 + 5]
    ps = [_draw(n, "bf16", rng) for n in sizes]
    P = [U.to_dev(p, torch.bfloat16) for p, _ in ps]
    G = [U.to_dev(g, torch.bfloat16) for _, g in ps]
    import ctypes
    k = len(sizes)
    pt = (ctypes.c_void_p * k)(*[t.data_ptr() for t in P])
    gt = (ctypes.c_void_p * k)(*[t.data_ptr() for t in G])
    nt = (ctypes.c_int64 * k)(*sizes)
    _lib.check(U.lib().lomo_fused_update_multi(pt, gt, nt, k, _lib.BF16, _lib.MATH_F64,
                                               0.05, 0.0, 0.0, 0, None, U.stream()), "multi")
    for t, (p0, g0) in zip(P, ps):
        assert np.array_equal(t.double().cpu().numpy(), _expected(p0, g0, "bf16"))


# --- reference hook cases, replayed through the C-ABI ------------------------------

def _device_case(case, arrays, nshapes, prec, math_mode):
    p, g = case_arrays(arrays, case["name"], nshapes)
    dt = U.TORCH_DT[prec]
    P = [U.to_dev(O.round_to(x, prec), dt) for x in p[0]]
    sc, clip = case["scaler"], case["clip"]
    two = sc is not None or (clip is not None and clip["kind"] == "by_global_norm")
    thresh = clip["threshold"] if clip and clip["kind"] == "by_value" else 0.0
    max_norm = clip["max_norm"] if clip and clip["kind"] == "by_global_norm" else 0.0
    st = U.State(nshapes, scale=case["init_scale"] or 0.0,
                 growth=sc["growth_interval"] if sc else 1,
                 min_scale=sc["min_scale"] if sc else 1.0,
                 max_scale=sc["max_scale"] if sc else 1.0, max_norm=max_norm)
    outs, scales, results = [], [], []
    grouped = clip is not None and clip["kind"] == "by_group_norm"
    if grouped:
        st = U.State(nshapes, max_norm=clip["max_norm"])
    for k in range(case["steps"]):
        scale = st.status().scale
        loss = torch.tensor(case["losses"][k], dtype=torch.float32, device="cuda")
        st.begin(loss)
        delivered = [U.to_dev(O.round_to(x * scale, prec), dt) for x in g[k]]
        order = list(reversed(range(nshapes)))  # delivery order (tape.py:350-360)
        if grouped:
            # stabilize.py:234-274: per group (layer // window): K2 -> K3a -> K1
            skipped0 = st.status().steps_skipped
            groups = []
            for i in order:
                if groups and groups[-1][0] == i // clip["window"]:
                    groups[-1][1].append(i)
                else:
                    groups.append((i // clip["window"], [i]))
            for _, members in groups:
                st.begin()
                for slot, i in enumerate(members):
                    st.probe(delivered[i], slot, _lib.ACCUM_F64 if math_mode == "f64" else 0)
                st.finalize()
                for i in members:
                    U.fused_update(P[i], delivered[i], math=math_mode, lr=case["lr"],
                                   flags=_lib.USE_SKIP | _lib.USE_COEF, state=st)
            outs.append("skipped_overflow" if st.status().steps_skipped > skipped0 else "applied")
        elif two:
            for slot, i in enumerate(order):
                st.probe(delivered[i], slot, (_lib.USE_SCALE if sc else 0) |
                         (_lib.ACCUM_F64 if math_mode == "f64" else 0))
            st.finalize()
            h = st.status()
            if h.underflow:
                outs.append("underflow")
            elif h.skip:
                outs.append("skipped_overflow")
            else:
                flags = _lib.USE_SKIP | (_lib.USE_SCALE if sc else 0) | \
                    (_lib.USE_COEF if max_norm > 0 else 0)
                for i in order:
                    U.fused_update(P[i], delivered[i], math=math_mode, lr=case["lr"],
                                   clip=thresh, flags=flags, state=st)
                st.on_clean()
                outs.append("applied")
        else:
            for i in order:
                U.fused_update(P[i], delivered[i], math=math_mode, lr=case["lr"], clip=thresh,
                               flags=_lib.USE_SKIP, state=st)
            st.on_clean()
            outs.append("nonfinite_loss" if st.status().skip else "applied")
        scales.append(st.status().scale if sc else None)
        results.append([t.clone() for t in P])
    return outs, scales, results, p, g


@pytest.mark.parametrize("math_mode", ["f64", "f32"])
def test_reference_hook_cases_replayed_on_device(hook_cases, math_mode):
    meta, arrays = hook_cases
    nshapes = len(meta["shapes"])
    worst = {}
    for case in meta["cases"]:
        prec = case["precision"]
        outs, scales, results, p, g = _device_case(case, arrays, nshapes, prec, math_mode)
        want = [o if not o.startswith("underflow") else "underflow" for o in case["outcomes"]]
        assert outs == want, case["name"]                     # decisions: bit-exact
        if case["scaler"] is not None:
            assert scales == case["scales"], case["name"]
        norm = case["clip"] is not None and case["clip"]["kind"] in ("by_global_norm",
                                                                      "by_group_norm")
        dt = U.TORCH_DT[prec]
        for k in range(case["steps"]):
            for i in range(nshapes):
                ref = U.to_dev(p[k + 1][i], dt)
                d = U.ulp_diff(results[k][i], ref).max().item()
                worst[case["name"]] = max(worst.get(case["name"], 0), d)
                if math_mode == "f64" and not norm:
                    assert d == 0, (case["name"], k, i, d)
                elif prec == "full":
                    # f64 storage: a coef that differs in its last bits (our
                    # reduction order vs BLAS ddot) moves p by ~eps*|lr g|,
                    # which is many result-ulps where p and lr*g cancel
                    err = (results[k][i] - ref).abs().cpu().numpy()
                    bound = 8 * 2.0 ** -52 * (np.abs(p[k][i]) + np.abs(case["lr"] * g[k][i]))
                    bound = bound.reshape(err.shape)
                    ok = (err == 0) | (err <= bound)  # NaN grads (skipped steps): err 0
                    assert np.all(ok), (case["name"], k, i)
                else:
                    assert d <= 1, (case["name"], k, i, d)
    print(math_mode, "max ulp per case:", worst)


@pytest.mark.parametrize("math_mode", ["f64", "f32"])
def test_bf16_cases_match_oracle(hook_cases, math_mode):
    """bf16 has no reference: the oracle's bf16 restatement is the target."""
    meta, arrays = hook_cases
    nshapes = len(meta["shapes"])
    for case in meta["cases"]:
        if case["precision"] != "half" or case["name"].startswith("nonfinite"):
            continue
        c = dict(case)
        outs, scales, results, _, _ = _device_case(c, arrays, nshapes, "bf16", math_mode)
        # oracle replay in bf16
        p, g = case_arrays(arrays, case["name"], nshapes)
        params = [O.round_to(x, "bf16") for x in p[0]]
        sc = case["scaler"]
        scaler = O.LossScaler(case["init_scale"], sc["growth_interval"], sc["min_scale"],
                              sc["max_scale"]) if sc else None
        clip = case["clip"]
        max_norm = clip["max_norm"] if clip and clip["kind"] == "by_global_norm" else None
        thresh = clip["threshold"] if clip and clip["kind"] == "by_value" else None
        grouped = clip is not None and clip["kind"] == "by_group_norm"
        for k in range(case["steps"]):
            if grouped:
                params, out = O.grouped_step(params, g[k], list(range(nshapes)), case["lr"],
                                             "bf16", clip["max_norm"], clip["window"])
                out = "applied" if out == "applied" else "skipped_overflow"
                max_norm = clip["max_norm"]
            elif scaler is not None or max_norm is not None:
                params, out, _, _ = O.two_pass_step(params, g[k], case["lr"], "bf16", scaler,
                                                    max_norm, thresh)
                out = {"applied": "applied", "skipped": "skipped_overflow",
                       "underflow": "underflow"}[out]
            else:
                params = [O.value_clip_update(pp, O.round_to(gg, "bf16"), case["lr"], thresh,
                                              "bf16") for pp, gg in zip(params, g[k])]
                out = "applied"
            assert outs[k] == out, (case["name"], k)
            for i in range(nshapes):
                d = U.ulp_diff(results[k][i], U.to_dev(params[i], torch.bfloat16)).max().item()
                assert d <= (0 if math_mode == "f64" and max_norm is None else 1), \
                    (case["name"], k, i, d)


# --- K4: reduce over peer memory fused with the update / probe -------------------

@pytest.mark.parametrize("prec", ["half", "bf16", "f32"])
@pytest.mark.parametrize("math_mode", ["f64", "f32"])
@pytest.mark.parametrize("world", [1, 3, 8])
def test_k4_fused_reduce_update_matches_oracle(prec, math_mode, world):
    """Peers simulated by `world` buffers on this GPU (the kernel only sees
    pointers; over NVLink they would be peer-mapped).  Rank 1 of `world` owns
    the middle slice of a padded bucket."""
    rng = np.random.default_rng(world)
    S = 8 * 1000
    total = S * world
    dt = U.TORCH_DT[prec]
    bufs0 = [O.round_to(rng.normal(0, 1e-3, total), prec) for _ in range(world)]
    bufs = [U.to_dev(b, dt) for b in bufs0]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    rank = 1 if world > 1 else 0
    off = rank * S
    p0 = O.round_to(rng.uniform(-0.08, 0.08, S), prec)
    p = U.to_dev(p0, dt)
    gsum = np.sum([b[off:off + S] for b in bufs0], axis=0)
    _lib.check(U.lib().lomo_fused_rs_update(p.data_ptr(), peers.data_ptr(), world, off, S,
                                            U.CODE[dt], U.MATH[math_mode], 0.05, 0.0, 0.0, 0,
                                            None, U.stream()), "rs_update")
    want = U.to_dev(O.apply_update(p0, gsum, 0.05, prec), dt)
    d = U.ulp_diff(p, want)
    if math_mode == "f64":
        assert d.max().item() == 0
    elif prec != "f32":
        assert d.max().item() <= 1
    # probe: sum of squares of the reduced slice
    st = U.State(2)
    st.begin()
    _lib.check(U.lib().lomo_fused_rs_probe(peers.data_ptr(), world, off, S, U.CODE[dt], 1,
                                           _lib.ACCUM_F64 if math_mode == "f64" else 0, st.ptr,
                                           U.stream()), "rs_probe")
    got = st.slots(2)[1]
    want_sq = float(np.dot(gsum, gsum))
    assert abs(got - want_sq) <= (1e-12 if math_mode == "f64" else 1e-6) * want_sq


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("world", [1, 3, 8])
def test_k4_probe_keep_writes_the_reduced_slice(prec, world):
    """lomo_fused_rs_probe_keep: `out` = the rank-ordered sum of the peers'
    slices (f64 with ACCUM_F64) rounded to the storage dtype (what a
    reduce-scatter writes), and the slot's sum of squares is taken of those rounded values
    (f64 accumulation: 1e-12); a NaN in one peer raises the overflow flag."""
    rng = np.random.default_rng(40 + world)
    S = 8 * 1500
    total = S * world
    dt = U.TORCH_DT[prec]
    bufs0 = [O.round_to(rng.normal(0, 1e-2, total), prec) for _ in range(world)]
    bufs = [U.to_dev(b, dt) for b in bufs0]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    off = (world // 2) * S
    out = torch.empty(S, dtype=dt, device="cuda")
    st = U.State(2)
    st.begin()
    _lib.check(U.lib().lomo_fused_rs_probe_keep(peers.data_ptr(), world, off, S, U.CODE[dt], 1,
                                                _lib.ACCUM_F64, st.ptr, out.data_ptr(),
                                                U.stream()), "rs_probe_keep")
    acc = np.zeros(S)
    for b in bufs0:  # ACCUM_F64: f64 accumulation in rank order
        acc = acc + b[off:off + S]
    want = O.round_to(acc, prec)
    assert np.array_equal(out.double().cpu().numpy(), want)
    sq = float(np.dot(want, want))
    assert abs(st.slots(2)[1] - sq) <= 1e-12 * sq
    assert st.status().overflow == 0
    bufs[-1][off + 17] = float("nan")
    st.begin()
    _lib.check(U.lib().lomo_fused_rs_probe_keep(peers.data_ptr(), world, off, S, U.CODE[dt], 0,
                                                0, st.ptr, out.data_ptr(), U.stream()), "keep")
    assert st.status().overflow == 1


def test_k4_rejects_misaligned_slices():
    b = torch.zeros(64, dtype=torch.bfloat16, device="cuda")
    peers = torch.tensor([b.data_ptr()], dtype=torch.int64, device="cuda")
    p = torch.zeros(8, dtype=torch.bfloat16, device="cuda")
    assert U.lib().lomo_fused_rs_update(p.data_ptr(), peers.data_ptr(), 1, 3, 8, _lib.BF16,
                                        _lib.MATH_F32, 0.1, 0.0, 0.0, 0, None, U.stream()) == -1
    assert U.lib().lomo_fused_rs_update(p.data_ptr(), peers.data_ptr(), 17, 0, 8, _lib.BF16,
                                        _lib.MATH_F32, 0.1, 0.0, 0.0, 0, None, U.stream()) == -1


def test_k1_k2_beyond_2_31_elements():
    """One tensor of 2^31 + 27 bf16 elements (8.6 GB for p and g): 64-bit
    indexing in K1 and K2, the grid for more than 2^31 elements, the scalar
    tail.  K1 (f32 math) against torch's fp32 update on the slices around
    2^31 and at the tail (<= 1 ulp); K2's sum of squares against a float64
    sum; the overflow flag for a NaN placed beyond 2^31."""
    n = (1 << 31) + 27
    free, _ = torch.cuda.mem_get_info()
    if free < 12 * 2 ** 30:
        pytest.skip("needs 12 GiB of free device memory")
    gen = torch.Generator(device="cuda").manual_seed(5)
    p = torch.empty(n, dtype=torch.bfloat16, device="cuda").uniform_(-0.08, 0.08, generator=gen)
    g = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_(0.0, 1e-2, generator=gen)
    lo, hi = (1 << 31) - 4096, (1 << 31) + 27
    windows = [slice(0, 4096), slice(lo, hi)]
    want = [(p[w].float() - 0.05 * g[w].float()) for w in windows]
    st = U.State(1)
    st.begin()
    st.probe(g, 0, 0)
    ref = sum(float((g[i:i + (1 << 28)].double() ** 2).sum()) for i in range(0, n, 1 << 28))
    got = float(st.slots(1)[0])
    assert abs(got - ref) <= 1e-5 * ref, (got, ref)
    U.fused_update(p, g, lr=0.05)
    for w, x in zip(windows, want):
        d = U.ulp_diff(p[w], x.to(torch.bfloat16))
        assert int(d.max()) <= 1, w
    g[(1 << 31) + 20] = float("nan")
    st.begin()
    st.probe(g, 0, 0)
    assert st.status().overflow == 1
    del p, g
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype,math_mode", [(torch.bfloat16, "f32"), (torch.float16, "f32"),
                                             (torch.float32, "f32"), (torch.float16, "f64")])
@pytest.mark.parametrize("use_cpp", [True, False])
@pytest.mark.parametrize("state_flags", [False, True])
def test_chained_k1_pass_equals_unchained(use_cpp, state_flags, dtype, math_mode):
    """LOMO_CHAINED (loads and stores before the PDL wait, the wait at the
    end) over a pass of 40 independent tensors -- ragged sizes, one
    misaligned pair (scalar fallback), small parked ones -- gives the same
    bits as the unchained pass, with host or device-state constants."""
    from paper_2306_09782_b200.dispatch import HookDispatcher
    gen = torch.Generator(device="cuda").manual_seed(9)
    sizes = [(1 << 20) + 13 * k for k in range(30)] + [3000 + k for k in range(8)] + [5, 7]
    P = [torch.empty(n, dtype=dtype, device="cuda").uniform_(-0.08, 0.08, generator=gen)
         for n in sizes]
    G = [torch.empty(n, dtype=dtype, device="cuda").normal_(0, 1e-2, generator=gen)
         for n in sizes]
    G[3] = torch.cat([torch.zeros(1, dtype=dtype, device="cuda"), G[3]])[1:]  # misaligned
    Q = [p.clone() for p in P]
    st = U.State(1, scale=4.0, max_norm=1.0)
    st.write_header(clip_coef=0.5, lr=0.05)
    flags = (_lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE
             if state_flags else 0)
    for chain, T in ((False, P), (True, Q)):
        d = HookDispatcher(U.lib(), st.ptr if state_flags else None, U.MATH[math_mode],
                           small_numel=4096, use_cpp=use_cpp)
        d.configure(lr=0.0 if state_flags else 0.05, flags=flags, chain=chain)
        for _ in range(3):  # three passes back to back
            for p, g in zip(T, G):
                d.update(p, g, U.CODE[dtype], U.stream())
            d.flush(U.stream())
    torch.cuda.synchronize()
    for k, (a, b) in enumerate(zip(P, Q)):
        assert torch.equal(a, b), k


@pytest.mark.parametrize("use_cpp", [True, False])
def test_chained_k2_pass_equals_unchained(use_cpp):
    """Chained K2 launches (LOMO_CHAINED) give the same per-slot partials,
    sums and overflow decision as waiting ones, over 40 ragged gradients."""
    from paper_2306_09782_b200.dispatch import HookDispatcher
    gen = torch.Generator(device="cuda").manual_seed(4)
    sizes = [(1 << 20) + 13 * k for k in range(30)] + [3000 + k for k in range(8)] + [5, 7]
    G = [torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_(0, 1e-2, generator=gen) * 64
         for n in sizes]
    res = []
    for chain in (False, True, True):
        st = U.State(len(G), scale=64.0, max_norm=1.0)
        d = HookDispatcher(U.lib(), st.ptr, _lib.MATH_F32, small_numel=4096, use_cpp=use_cpp)
        d.configure(flags=_lib.USE_SCALE, chain=chain)
        st.begin()
        for k, g in enumerate(G):
            d.probe(g, _lib.BF16, k, U.stream())
        d.flush(U.stream())
        st.finalize()
        h = st.status()
        res.append((st.slots(len(G)).tolist(), h.total_norm, h.overflow, h.skip))
    assert res[0] == res[1] == res[2]
    G[17][5] = float("nan")
    st = U.State(len(G), scale=64.0, max_norm=1.0)
    d = HookDispatcher(U.lib(), st.ptr, _lib.MATH_F32, small_numel=4096, use_cpp=use_cpp)
    d.configure(flags=_lib.USE_SCALE, chain=True)
    st.begin()
    for k, g in enumerate(G):
        d.probe(g, _lib.BF16, k, U.stream())
    d.flush(U.stream())
    st.finalize()
    assert st.status().overflow == 1 and st.status().skip == 1


@pytest.mark.parametrize("prec", PRECS)
def test_apply_update_python_entry_matches_reference_kats(prec):
    """paper_2306_09782_b200.apply_update (optim.py:52-54 as a device call):
    f64 math is bit-exact against the oracle (the reference's float64
    arithmetic + write-back rounding); shape mismatch -> ShapeError."""
    from paper_2306_09782_b200 import ShapeError, apply_update
    rng = np.random.default_rng(17)
    p0, g0 = _draw(100003, prec, rng)
    dt = U.TORCH_DT[prec]
    p, g = U.to_dev(p0, dt), U.to_dev(g0, dt)
    apply_update(p, g, 0.05)
    assert np.array_equal(p.double().cpu().numpy(), O.apply_update(p0, g0, 0.05, prec))
    with pytest.raises(ShapeError):
        apply_update(p, g[:-1], 0.05)


def test_empty_and_tiny_inputs_everywhere():
    """Empty tensors through every entry point the hooks use: K2 of an empty
    gradient adds nothing to its slot, multi-tensor lists with empty and
    1-element members update exactly the non-empty ones, K4 of an empty
    slice is a no-op, and a model with an empty parameter trains."""
    import ctypes
    from paper_2306_09782_b200 import LOMO
    e = torch.empty(0, dtype=torch.bfloat16, device="cuda")
    st = U.State(3, max_norm=1.0)
    st.begin()
    st.probe(e, 0, 0)
    st.probe(torch.ones(8, dtype=torch.bfloat16, device="cuda"), 1, 0)
    st.finalize()
    assert st.status().sumsq_total == 8.0 and st.status().skip == 0
    rng = np.random.default_rng(21)
    sizes = [0, 1, 0, 7, 4096]
    ps = [_draw(max(n, 1), "bf16", rng) for n in sizes]
    P = [U.to_dev(p[:n], torch.bfloat16) for (p, _), n in zip(ps, sizes)]
    G = [U.to_dev(g[:n], torch.bfloat16) for (_, g), n in zip(ps, sizes)]
    k = len(sizes)
    pt = (ctypes.c_void_p * k)(*[t.data_ptr() for t in P])
    gt = (ctypes.c_void_p * k)(*[t.data_ptr() for t in G])
    nt = (ctypes.c_int64 * k)(*sizes)
    _lib.check(U.lib().lomo_fused_update_multi(pt, gt, nt, k, _lib.BF16, _lib.MATH_F64,
                                               0.05, 0.0, 0.0, 0, None, U.stream()), "multi")
    for t, (p0, g0), n in zip(P, ps, sizes):
        assert np.array_equal(t.double().cpu().numpy(), _expected(p0[:n], g0[:n], "bf16"))
    ss = (ctypes.c_int * k)(*range(k))
    st2 = U.State(k)
    st2.begin()
    _lib.check(U.lib().lomo_probe_multi(gt, nt, ss, k, _lib.BF16, _lib.ACCUM_F64, st2.ptr,
                                        U.stream()), "probe multi")
    got = st2.slots(k)
    for j, (g, n) in enumerate(zip(G, sizes)):
        assert got[j] == float((g.double() ** 2).sum())
    peers = torch.tensor([P[-1].data_ptr()], dtype=torch.int64, device="cuda")
    assert U.lib().lomo_fused_rs_update(P[-1].data_ptr(), peers.data_ptr(), 1, 0, 0, _lib.BF16,
                                        _lib.MATH_F32, 0.05, 0.0, 0.0, 0, None,
                                        U.stream()) == 0

    class M(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.w = torch.nn.Parameter(torch.ones(4, device="cuda"))
            self.empty = torch.nn.Parameter(torch.zeros(0, device="cuda"))

        def loss(self, x):
            return (self.w * x).sum() + self.empty.sum()

    m = M()
    opt = LOMO(m, lr=0.5, clip_grad_norm=10.0)
    x = torch.full((4,), 2.0, device="cuda")
    opt.step(lambda: m.loss(x), 0.5)
    assert torch.equal(m.w, torch.zeros(4, device="cuda"))  # 1 - 0.5 * 2


def test_chained_k1_stress_many_short_launches():
    """500 chained K1 launches of 70k-300k elements (each a few microseconds,
    so many grids overlap their predecessors' drains), 5 passes, against the
    same passes unchained: identical bits."""
    from paper_2306_09782_b200.dispatch import HookDispatcher
    rng = np.random.default_rng(99)
    sizes = [int(x) for x in rng.integers(70_000, 300_000, 500)]
    gen = torch.Generator(device="cuda").manual_seed(13)
    P = [torch.empty(n, dtype=torch.float16, device="cuda").uniform_(-0.08, 0.08, generator=gen)
         for n in sizes]
    G = [torch.empty(n, dtype=torch.float16, device="cuda").normal_(0, 1e-2, generator=gen)
         for n in sizes]
    Q = [p.clone() for p in P]
    for chain, T in ((False, P), (True, Q)):
        d = HookDispatcher(U.lib(), None, _lib.MATH_F32)
        d.configure(lr=0.05, chain=chain)
        for _ in range(5):
            for p, g in zip(T, G):
                d.update(p, g, _lib.F16, U.stream())
            d.flush(U.stream())
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(P, Q))


@pytest.mark.parametrize("prec", ["half", "bf16"])
def test_f64_math_widening_special_values(prec):
    """f64 math widens 16-bit storage by integer ops for normals and zeros
    and by conversion for the rest: every class -- +-0, subnormals, the
    smallest/largest normals, inf, NaN -- in p and g gives the oracle's bits."""
    dt = U.TORCH_DT[prec]
    info = torch.finfo(dt)
    sub = info.tiny / 4
    vals = [0.0, -0.0, sub, -sub, info.tiny, -info.tiny, info.max, -info.max, 1.0, -1.5,
            float("inf"), float("-inf"), 3.0e-3, -7.25e-2]
    rng = np.random.default_rng(5)
    p0 = O.round_to(np.array([vals[i % len(vals)] for i in range(4099)]), prec)
    g0 = O.round_to(np.array([vals[(7 * i + 3) % len(vals)] for i in range(4099)]), prec)
    p0[::97] = np.nan
    p, g = U.to_dev(p0, dt), U.to_dev(g0, dt)
    U.fused_update(p, g, math="f64", lr=0.5)
    got = p.double().cpu().numpy()
    want = _expected(p0, g0, prec, lr=0.5)
    same = (got == want) | (np.isnan(got) & np.isnan(want))
    assert same.all(), np.flatnonzero(~same)[:10]
