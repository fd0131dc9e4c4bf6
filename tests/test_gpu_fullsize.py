"""Parity at BASELINE.json's full size (config 2): the two-pass protocol's
kernels over all 291 LLaMA-7B parameter tensors (6.74 G bf16 elements, the
bench workload), issued exactly as the hooks issue them (HookDispatcher, C++
dispatcher, delivery order, small tensors coalesced).

The oracle cannot run 6.7 G elements in seconds, so the checks are the
size-independent ones:

* pass 1 (K2 per gradient -> K3a): every slot's sum of squares against a
  float64 sum of the same gradient (ACCUM_F64: 1e-12 relative), the global
  norm and clip coefficient from those sums, the overflow flag clear;
* pass 2 (K1 with skip / 1/scale / coef / lr from the device state): 4096
  sampled elements of every tensor (first, last and random positions)
  against the oracle's update_hook (stabilize.py:217-224, optim.py:52-54)
  with the device's own coefficient -- bit-exact in f64 math, <= 1 ulp in
  f32 math -- and, on copies taken before the pass, K1 with lr passed from
  the host (not LR_FROM_STATE) giving the same bits;
* a NaN planted in the first-delivered gradient (lm_head): the overflow flag, the skip
  decision, the halved scale, and a pass 2 that leaves all 6.7 G parameters
  unchanged (checksummed).
"""
import math

import numpy as np
import pytest
import torch

import lomo_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import gpu_util as U
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.dispatch import HookDispatcher
    from paper_2306_09782_b200.workloads import llama_param_shapes

SCALE = 2.0 ** 10
LR = 0.05
MAX_NORM = 1.0
NSAMP = 4096


@pytest.fixture(scope="module")
def work():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * 2 ** 30:
        pytest.skip("needs 40 GiB of free device memory")
    gen = torch.Generator(device="cuda").manual_seed(11)
    shapes = [math.prod(s) for _, s in llama_param_shapes("7b")]
    P, G = [], []
    for n in shapes:
        P.append(torch.empty(n, dtype=torch.bfloat16, device="cuda").uniform_(-0.08, 0.08,
                                                                              generator=gen))
        # gradients as pass 1 sees them: scaled by the loss scale
        G.append((torch.empty(n, dtype=torch.float32, device="cuda").normal_(
            0.0, 1e-3, generator=gen) * SCALE).to(torch.bfloat16))
    rng = np.random.default_rng(0)
    idx = []
    for n in shapes:
        k = min(n, NSAMP)
        i = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, k)]))
        idx.append(torch.from_numpy(i).cuda())
    yield P, G, idx
    del P, G
    torch.cuda.empty_cache()


def _probe_pass(lib, st, G, flags):
    d = HookDispatcher(lib, st.ptr, _lib.MATH_F64 if flags & _lib.ACCUM_F64 else _lib.MATH_F32)
    d.configure(flags=flags)
    st.begin()
    s = U.stream()
    for i in range(len(G) - 1, -1, -1):  # delivery order: slot = position in it
        d.probe(G[i], _lib.BF16, len(G) - 1 - i, s)
    d.flush(s)
    st.finalize()
    return st.status()


def _update_pass(lib, st, P, G, math_code, flags, lr=0.0):
    d = HookDispatcher(lib, st.ptr if st is not None else None, math_code)
    d.configure(lr=lr, flags=flags)
    s = U.stream()
    for i in range(len(P) - 1, -1, -1):
        d.update(P[i], G[i], _lib.BF16, s)
    d.flush(s)
    torch.cuda.synchronize()


def _sq64(g):
    return sum(float((g[j:j + (1 << 27)].double() / SCALE).pow(2).sum())
               for j in range(0, g.numel(), 1 << 27))


def test_two_pass_full_llama7b(work):
    P, G, idx = work
    lib = U.lib()
    st = U.State(len(P), scale=SCALE, max_norm=MAX_NORM)
    h = _probe_pass(lib, st, G, _lib.USE_SCALE | _lib.ACCUM_F64)
    assert not h.overflow and not h.skip
    got = st.slots(len(P))
    want = [_sq64(G[i]) for i in range(len(G) - 1, -1, -1)]  # slot order
    for s, (a, b) in enumerate(zip(got, want)):
        assert abs(a - b) <= 1e-12 * b, (s, a, b)
    total = sum(want)
    assert abs(h.total_norm - math.sqrt(total)) <= 1e-12 * math.sqrt(total)
    coef = min(1.0, MAX_NORM / h.total_norm)
    assert h.clip_coef == coef and coef < 1.0  # the clip engages at this size

    p0 = [P[i][idx[i]].double().cpu().numpy() for i in range(len(P))]
    g0 = [G[i][idx[i]].double().cpu().numpy() for i in range(len(P))]
    keep = [p.clone() for p in P[:3]]  # host-lr control on a few tensors
    _lib.check(lib.lomo_set_lr(st.ptr, LR, U.stream()), "lr")
    flags = _lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE
    _update_pass(lib, st, P, G, _lib.MATH_F64, flags)
    for i in range(len(P)):
        want_p = O.update_hook(p0[i], g0[i], LR, SCALE, None, coef, "bf16")
        got_p = P[i][idx[i]]
        d = U.ulp_diff(got_p, U.to_dev(want_p, torch.bfloat16))
        assert int(d.max()) == 0, (i, int(d.max()))
    # the same update with lr passed from the host (scale and coefficient
    # still from the state): the LR_FROM_STATE + USE_SKIP form above must
    # give the same bits
    for j, q in enumerate(keep):
        d = HookDispatcher(lib, st.ptr, _lib.MATH_F64)
        d.configure(lr=LR, flags=_lib.USE_SCALE | _lib.USE_COEF)
        d.update(q, G[j], _lib.BF16, U.stream())
        d.flush(U.stream())
        torch.cuda.synchronize()
        assert torch.equal(q, P[j]), j
    st.on_clean()


def test_f32_math_full_llama7b(work):
    P, G, idx = work
    lib = U.lib()
    st = U.State(len(P), scale=SCALE, max_norm=MAX_NORM)
    h = _probe_pass(lib, st, G, _lib.USE_SCALE)
    # f32 squares per 16-byte vector, f64 across vectors: 2e-6 relative
    assert abs(h.total_norm ** 2 - sum(_sq64(g) for g in G)) <= 2e-6 * h.total_norm ** 2
    p0 = [P[i][idx[i]].double().cpu().numpy() for i in range(len(P))]
    g0 = [G[i][idx[i]].double().cpu().numpy() for i in range(len(P))]
    _lib.check(lib.lomo_set_lr(st.ptr, LR, U.stream()), "lr")
    _update_pass(lib, st, P, G, _lib.MATH_F32,
                 _lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE)
    worst = 0
    for i in range(len(P)):
        want_p = O.update_hook(p0[i], g0[i], LR, SCALE, None, h.clip_coef, "bf16")
        d = U.ulp_diff(P[i][idx[i]], U.to_dev(want_p, torch.bfloat16))
        worst = max(worst, int(d.max()))
    assert worst <= 1, worst


def test_fp16_two_pass_full_llama7b():
    """Config 3's storage dtype at config 2's size: fp16 parameters and
    gradients scaled by 2^10 (pass 1 sees the scaled gradient), f32 math:
    every slot within 2e-6 of its float64 sum, the clip coefficient from the
    device norm, and sampled elements <= 1 ulp from the oracle's
    update_hook."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * 2 ** 30:
        pytest.skip("needs 40 GiB of free device memory")
    gen = torch.Generator(device="cuda").manual_seed(12)
    shapes = [math.prod(s) for _, s in llama_param_shapes("7b")]
    P = [torch.empty(n, dtype=torch.float16, device="cuda").uniform_(-0.08, 0.08, generator=gen)
         for n in shapes]
    G = [(torch.empty(n, dtype=torch.float32, device="cuda").normal_(0.0, 1e-3, generator=gen)
          * SCALE).half() for n in shapes]
    rng = np.random.default_rng(1)
    idx = [torch.from_numpy(np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, NSAMP)]))
                            ).cuda() for n in shapes]
    lib = U.lib()
    st = U.State(len(P), scale=SCALE, max_norm=MAX_NORM)
    d = HookDispatcher(lib, st.ptr, _lib.MATH_F32)
    d.configure(flags=_lib.USE_SCALE)
    st.begin()
    for i in range(len(G) - 1, -1, -1):
        d.probe(G[i], _lib.F16, len(G) - 1 - i, U.stream())
    d.flush(U.stream())
    st.finalize()
    h = st.status()
    assert not h.skip
    got = st.slots(len(P))
    for s, i in enumerate(range(len(G) - 1, -1, -1)):
        want = _sq64(G[i])
        assert abs(got[s] - want) <= 2e-6 * want, (s, got[s], want)
    p0 = [P[i][idx[i]].double().cpu().numpy() for i in range(len(P))]
    g0 = [G[i][idx[i]].double().cpu().numpy() for i in range(len(P))]
    _lib.check(lib.lomo_set_lr(st.ptr, LR, U.stream()), "lr")
    _update_pass_dt(lib, st, P, G, _lib.F16)
    for i in range(len(P)):
        want_p = O.update_hook(p0[i], g0[i], LR, SCALE, None, h.clip_coef, "half")
        dd = U.ulp_diff(P[i][idx[i]], U.to_dev(want_p, torch.float16))
        assert int(dd.max()) <= 1, (i, int(dd.max()))
    del P, G
    torch.cuda.empty_cache()


def _update_pass_dt(lib, st, P, G, dt):
    d = HookDispatcher(lib, st.ptr, _lib.MATH_F32)
    d.configure(flags=_lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE,
                chain=True)
    for i in range(len(P) - 1, -1, -1):
        d.update(P[i], G[i], dt, U.stream())
    d.flush(U.stream())
    torch.cuda.synchronize()


def test_overflow_skip_full_llama7b(work):
    P, G, _ = work
    lib = U.lib()
    st = U.State(len(P), scale=SCALE, max_norm=MAX_NORM)
    g0 = G[-1][7].clone()
    G[-1][7] = float("nan")  # the first-delivered gradient (the lm_head)
    try:
        h = _probe_pass(lib, st, G, _lib.USE_SCALE)
        assert h.overflow and h.skip and h.scale == SCALE / 2
        before = [float(p.float().sum()) for p in P]
        _lib.check(lib.lomo_set_lr(st.ptr, LR, U.stream()), "lr")
        _update_pass(lib, st, P, G, _lib.MATH_F32,
                     _lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF | _lib.LR_FROM_STATE)
        after = [float(p.float().sum()) for p in P]
        assert before == after
    finally:
        G[-1][7] = g0
