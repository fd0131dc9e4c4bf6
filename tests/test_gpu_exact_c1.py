"""Config 1, fp16, end to end: the reference's tape semantics (restated in
tests/exact_c1.py, float64 ops with binary16 rounding at every op boundary)
driving the product's hook kernels through the C-ABI -- K2 probe, K3a/K3b
decisions and scaler, K1 update in f64 math -- against fixtures B and C
recorded from the reference itself (tests/golden/c1.*).

Tolerance (stated, north star): every skip/clip decision and the loss-scale
trajectory identical; every sampled parameter within 2 ulp (binary16) of the
reference after 10 steps, max and mean ulp reported; losses within 1e-9
relative.  (With the model's own torch fp16 kernels instead of the restated
tape the update path is the same but the forward/backward ops round
differently: tests/test_gpu_lomo.py reports that variant.)
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import gpu_util as U
    from exact_c1 import ExactMini
    from paper_2306_09782_b200 import _lib
    from paper_2306_09782_b200.workloads import MiniConfig, sequence_copy_batch


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    torch.cuda.set_device(0)


def _ulps16(got, ref):
    g = got.astype(np.float16).view(np.int16).astype(np.int64)
    r = ref.astype(np.float16).view(np.int16).astype(np.int64)
    g = np.where(g < 0, -(1 << 15) - g, g)
    r = np.where(r < 0, -(1 << 15) - r, r)
    return np.abs(g - r)


def run_fixture(scale0, max_scale):
    cfg = MiniConfig()
    m = ExactMini(cfg)
    names = m.names
    slot = {n: i for i, n in enumerate(reversed(names))}       # delivery order
    st = U.State(len(names), scale=scale0, growth=2, min_scale=1.0, max_scale=max_scale,
                 max_norm=1.0)
    losses, outcomes, scales = [], [], []
    for step in range(10):
        ids = torch.from_numpy(sequence_copy_batch(0, step, 4, 128, 1024)).cuda()
        scale = st.status().scale
        logits, S = m.forward(ids)
        loss, dout = m.loss_and_grad(logits, ids)
        st.begin(torch.tensor(loss, dtype=torch.float64, device="cuda"))

        def probe(name, g):
            st.probe(g.to(torch.float16), slot[name], _lib.USE_SCALE | _lib.ACCUM_F64)
        m.backward(S, dout * scale, probe)                     # pass 1
        st.finalize()
        h = st.status()
        if h.skip:
            outcomes.append("skipped_overflow")
        else:
            logits2, S2 = m.forward(ids)                       # stabilize.py:226
            loss, dout2 = m.loss_and_grad(logits2, ids)

            def update(name, g):
                U.fused_update(m.p16[name], g.to(torch.float16), math="f64", lr=0.05,
                               flags=_lib.USE_SKIP | _lib.USE_SCALE | _lib.USE_COEF, state=st)
            m.backward(S2, dout2 * scale, update)              # pass 2
            st.on_clean()
            outcomes.append("applied")
        losses.append(loss)
        scales.append(st.status().scale)
    return m, losses, outcomes, scales


@pytest.mark.parametrize("key,scale0,max_scale", [("B", 2.0 ** 16, 2.0 ** 24),
                                                  ("C", 2.0 ** 24, 2.0 ** 24)])
def test_c1_fp16_end_to_end_within_2_ulp(c1_meta, c1_arrays, key, scale0, max_scale):
    torch.backends.cuda.matmul.allow_tf32 = False
    m, losses, outcomes, scales = run_fixture(scale0, max_scale)
    ref = c1_meta[key]
    assert outcomes == ref["outcomes"]
    assert [math.log2(s) for s in scales] == ref["log2_scale"]
    for a, b in zip(losses, ref["losses"]):
        if math.isfinite(b):
            assert abs(a - b) <= 1e-9 * abs(b), (a, b)
    u = []
    for name in m.names:
        idx = torch.from_numpy(c1_arrays[f"{key}/{name}/idx"]).cuda()
        got = m.p16[name].reshape(-1)[idx].double().cpu().numpy()
        u.append(_ulps16(got, c1_arrays[f"{key}/{name}/val"]))
    u = np.concatenate(u)
    print(f"fixture {key}: {u.size} sampled params, max ulp {u.max()}, mean ulp {u.mean():.2e}, "
          f"mismatches {(u > 0).sum()}")
    assert u.max() <= 2
