"""Generate the golden fixtures from the REFERENCE itself (build container only).

Run:  python tests/golden/make_golden.py          (needs /root/reference)

The reference is pure Python (fusedtrain, numpy), so it is imported
read-only from /root/reference/pkg/src and driven through its own public
code paths; nothing is copied.  Outputs (committed):

* hook_cases.npz / hook_cases.json -- the reference's LOMO.step /
  Stabilizer.run_step (optim.py:118-132, stabilize.py:148-230) driven by a
  fake model whose tape delivers chosen gradients to the reference's own hook
  bodies (apply_update, value clip, probe_hook, update_hook, LossScaler).
  Each case records p0, the per-step unscaled gradients G, and the
  reference's parameters / outcome / scale after every step.
* rounding.npz -- round_through_half (tensor.py:30-38) on the 18 KAT values
  of tests/test_tensor.py:35-42 plus random and midpoint-adjacent values.
* scaler_replay.json -- LossScaler (stabilize.py:94-127) over random outcome
  sequences (the replay of test_acceptance.py:151-169).
* c1.npz / c1.json -- config 1 (zoo MINI_TRANSFORMER layers=2 hidden=256
  heads=4 vocab=1024 seed=0; seq 128 batch 4; lr 0.05; 10 steps), fixtures
  A (FULL, plain LOMO), B (HALF, two-pass by_global_norm(1.0) +
  LossScaler(2^16, growth 2)), C (HALF, forced overflow LossScaler(2^24,
  growth 2, max 2^24)): per-step losses / outcomes / scales, the initial and
  final digests, per-tensor sums and a fixed sample of final elements.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from fusedtrain.errors import NonFiniteLossError  # noqa: E402
from fusedtrain.optim import LOMO  # noqa: E402
from fusedtrain.stabilize import ClipMode, LossScaler, Stabilizer  # noqa: E402
from fusedtrain.tape import Disposition, Parameter  # noqa: E402
from fusedtrain.tensor import Precision, Tensor, round_through_half  # noqa: E402
from fusedtrain.zoo import (ModelConfig, ModelKind, SyntheticTask, TaskKind,  # noqa: E402
                            build_model, sample_batch)

SHAPES = [(64, 48), (300,), (7,), (200, 33), (5,)]
PREC = {"full": Precision.FULL, "half": Precision.HALF_EMULATED}


# --------------------------------------------------------------------------
# fake model: the reference's step code runs unchanged on top of it
# --------------------------------------------------------------------------
class FakeTape:
    def __init__(self, params, precision):
        self.parameters = params
        self.precision = precision
        self.grads = None  # list of unscaled grads, build order
        self.ledger = None

    def backward(self, loss_grad, hook):
        s = float(loss_grad.data.ravel()[0])
        for p, g in zip(reversed(self.parameters), reversed(self.grads)):
            with np.errstate(over="ignore", invalid="ignore"):
                t = Tensor(g * s, self.precision)  # rounded per precision (tape.py:377,394)
            d = hook(p, t)
            if d is Disposition.RETAIN:        # tape.py:402-403
                p.grad_slot = t
            else:
                assert d is Disposition.CONSUME


class FakeModel:
    def __init__(self, p0, precision):
        self.precision = precision
        params = [Parameter(f"p{i}", i, Tensor(a, precision)) for i, a in enumerate(p0)]
        self.tape = FakeTape(params, precision)
        self.parameters = params

    def forward(self, inputs):
        return Tensor(np.zeros(1))

    def loss_and_grad(self, output, targets):
        return float(targets), np.ones(1)


def draw_case(rng, precision, steps, big_steps=(), mags=None):
    p0 = [rng.uniform(-0.08, 0.08, s) for s in SHAPES]
    G = []
    for k in range(steps):
        m = 1e-3 * (mags[k] if mags else 1.0)
        gs = [rng.normal(0.0, m, s) for s in SHAPES]
        if k in big_steps:  # a few large entries: overflow fp16 at big scales
            gs[3].flat[rng.integers(0, gs[3].size, 4)] = rng.uniform(0.01, 0.02, 4)
        G.append(gs)
    if precision == "half":
        p0 = [round_through_half(a) for a in p0]
        G = [[round_through_half(g) for g in gs] for gs in G]
    return p0, G


def run_case(name, precision, stab_factory, steps, lr, rng, losses=None, big_steps=(),
             mags=None, nan_step=None):
    p0, G = draw_case(rng, precision, steps, big_steps, mags)
    if nan_step is not None:
        G[nan_step][1][3] = np.nan
    model = FakeModel(p0, PREC[precision])
    stab = stab_factory()
    opt = LOMO(model, stab)
    rec = {"name": name, "precision": precision, "lr": lr, "steps": steps,
           "outcomes": [], "scales": [], "clean": [], "losses": [],
           "init_scale": stab.scaler.scale if stab is not None and stab.scaler else None}
    arrays = {f"{name}/p0_{i}": a for i, a in enumerate(p0)}
    for k in range(steps):
        model.tape.grads = G[k]
        loss = 0.5 if losses is None else losses[k]
        try:
            opt.step((None, loss), lr)
            out = opt.last_outcome.value if opt.last_outcome is not None else "applied"
        except NonFiniteLossError:
            out = "nonfinite_loss"
        rec["outcomes"].append(out)
        rec["losses"].append(loss)
        sc = stab.scaler if stab is not None else None
        rec["scales"].append(sc.scale if sc else None)
        rec["clean"].append(sc.clean_steps if sc else None)
        for i, g in enumerate(G[k]):
            arrays[f"{name}/G{k}_{i}"] = g
        for i, p in enumerate(model.parameters):
            arrays[f"{name}/p{k + 1}_{i}"] = p.value.data.copy()
    if stab is not None:
        rec["clip"] = {"kind": stab.clip.kind.value, "threshold": stab.clip.threshold,
                       "max_norm": stab.clip.max_norm, "window": stab.clip.window}
        sc = stab.scaler
        rec["scaler"] = None if sc is None else {
            "growth_interval": sc.growth_interval, "min_scale": sc.min_scale,
            "max_scale": sc.max_scale}
    else:
        rec["clip"], rec["scaler"] = None, None
    return rec, arrays


def hook_cases():
    rng = np.random.default_rng(20240617)
    cases, arrays = [], {}
    specs = []
    for prec in ("full", "half"):
        specs += [
            (f"plain_{prec}", prec, lambda: None, 3, 0.05, {}),
            (f"plain_lr0_{prec}", prec, lambda: None, 1, 0.0, {}),
            (f"valueclip_{prec}", prec, lambda: Stabilizer(ClipMode.by_value(1.5e-3)), 3, 0.05, {}),
            (f"normclip_{prec}", prec, lambda: Stabilizer(ClipMode.by_global_norm(0.08)), 4, 0.05,
             {"mags": [1.0, 0.5, 2.0, 0.25]}),
            (f"scaler_{prec}", prec,
             lambda: Stabilizer(ClipMode.none(), LossScaler(2.0 ** 10, growth_interval=2)), 5, 0.05, {}),
            (f"norm_scaler_{prec}", prec,
             lambda: Stabilizer(ClipMode.by_global_norm(0.08),
                                LossScaler(2.0 ** 12, growth_interval=2)), 4, 0.05,
             {"mags": [1.0, 0.5, 2.0, 0.25]}),
            (f"nonfinite_loss_{prec}", prec, lambda: None, 2, 0.05,
             {"losses": [float("inf"), 0.5]}),
            (f"nonfinite_loss_2pass_{prec}", prec,
             lambda: Stabilizer(ClipMode.by_global_norm(0.08)), 2, 0.05,
             {"losses": [float("nan"), 0.5]}),
            (f"nan_grad_2pass_{prec}", prec,
             lambda: Stabilizer(ClipMode.by_global_norm(0.08)), 2, 0.05, {"nan_step": 0}),
            # single-pass grouped clipping (stabilize.py:234-274), layer = index
            (f"grouped_w1_{prec}", prec,
             lambda: Stabilizer(ClipMode.by_group_norm(0.03, 1)), 3, 0.05, {}),
            (f"grouped_w2_{prec}", prec,
             lambda: Stabilizer(ClipMode.by_group_norm(0.03, 2)), 3, 0.05, {}),
            (f"grouped_nan_{prec}", prec,
             lambda: Stabilizer(ClipMode.by_group_norm(0.03, 2)), 2, 0.05, {"nan_step": 0}),
        ]
    specs += [
        ("overflow_half", "half",
         lambda: Stabilizer(ClipMode.none(), LossScaler(2.0 ** 24, growth_interval=2,
                                                        max_scale=2.0 ** 24)), 8, 0.05,
         {"big_steps": (0, 1, 2, 3, 4, 5, 6, 7)}),
        ("overflow_norm_half", "half",
         lambda: Stabilizer(ClipMode.by_global_norm(0.08),
                            LossScaler(2.0 ** 24, growth_interval=1, max_scale=2.0 ** 24)), 8, 0.05,
         {"big_steps": (0, 1, 2, 3, 4, 5, 6, 7)}),
        ("underflow_half", "half",
         lambda: Stabilizer(ClipMode.none(), LossScaler(2.0, growth_interval=4, min_scale=1.0)),
         3, 0.05, {"nan_step": 0}),
    ]
    for name, prec, fac, steps, lr, kw in specs:
        if name == "underflow_half":
            # nan grads every step: 2 -> 1 -> underflow (ScaleUnderflowError)
            p0, G = draw_case(rng, prec, steps)
            for k in range(steps):
                G[k][1][0] = np.nan
            model = FakeModel(p0, PREC[prec])
            stab = fac()
            opt = LOMO(model, stab)
            rec = {"name": name, "precision": prec, "lr": lr, "steps": steps, "outcomes": [],
                   "init_scale": stab.scaler.scale,
                   "scales": [], "clean": [], "losses": [],
                   "clip": {"kind": "none", "threshold": None, "max_norm": None},
                   "scaler": {"growth_interval": 4, "min_scale": 1.0, "max_scale": 2.0 ** 24}}
            arr = {f"{name}/p0_{i}": a for i, a in enumerate(p0)}
            for k in range(steps):
                model.tape.grads = G[k]
                try:
                    opt.step((None, 0.5), lr)
                    rec["outcomes"].append(opt.last_outcome.value)
                except Exception as exc:  # ScaleUnderflowError
                    rec["outcomes"].append("underflow:" + type(exc).__name__)
                rec["scales"].append(stab.scaler.scale)
                rec["clean"].append(stab.scaler.clean_steps)
                rec["losses"].append(0.5)
                for i, g in enumerate(G[k]):
                    arr[f"{name}/G{k}_{i}"] = g
                for i, p in enumerate(model.parameters):
                    arr[f"{name}/p{k + 1}_{i}"] = p.value.data.copy()
            cases.append(rec)
            arrays.update(arr)
            continue
        rec, arr = run_case(name, prec, fac, steps, lr, rng, **kw)
        cases.append(rec)
        arrays.update(arr)
    # half-case arrays hold binary16 values exactly: store them as float16
    half = {c["name"] for c in cases if c["precision"] == "half"}
    arrays = {k: (v.astype(np.float16) if k.split("/")[0] in half else v)
              for k, v in arrays.items()}
    np.savez_compressed(OUT / "hook_cases.npz", **arrays)
    (OUT / "hook_cases.json").write_text(json.dumps({"shapes": SHAPES, "cases": cases}, indent=1))
    print("hook cases:", [(c["name"], c["outcomes"]) for c in cases])


def rounding():
    kat = np.array([0.0, 1.0, -1.0, 0.1, 1e-5, 6.1e-5, 5.96e-8, 2.98e-8, 1e-9, 65504.0,
                    65519.9, 65520.0, 65536.0, 1e30, -3.14159, 2.0 ** -24, 2.0 ** -25, 1.5e-7])
    rng = np.random.default_rng(7)
    rnd = rng.normal(0, 1, 20000) * np.exp2(rng.integers(-30, 17, 20000))
    # values adjacent to binary16 rounding midpoints (double rounding through
    # fp32 would break these): midpoint +- a few f64 ulps
    h = rng.uniform(-2, 2, 4000).astype(np.float16).astype(np.float64)
    ulp = np.abs(np.spacing(h.astype(np.float16)).astype(np.float64))
    mid = h + ulp / 2
    near = np.concatenate([mid, np.nextafter(mid, np.inf), np.nextafter(mid, -np.inf),
                           mid + 2 ** -40, mid - 2 ** -40])
    x = np.concatenate([kat, rnd, near])
    np.savez_compressed(OUT / "rounding.npz", x=x, half=round_through_half(x))


def scaler_replay():
    rng = np.random.default_rng(2024)
    seqs = []
    for _ in range(300):
        outcomes = [bool(v) for v in rng.random(int(rng.integers(1, 40))) < 0.7]
        growth = int(rng.integers(1, 6))
        sc = LossScaler(scale=2.0 ** 6, growth_interval=growth, min_scale=1.0,
                        max_scale=2.0 ** 10)
        trace = []
        for ok in outcomes:
            try:
                sc.on_clean() if ok else sc.on_overflow()
            except Exception:
                trace.append(None)
                break
            trace.append(sc.scale)
        seqs.append({"outcomes": outcomes, "growth": growth, "trace": trace})
    (OUT / "scaler_replay.json").write_text(json.dumps(seqs))


def _sample_idx(n: int, k: int) -> np.ndarray:
    return np.unique(np.random.default_rng(n).integers(0, n, k)) if n > k else np.arange(n)


def c1():
    cfg = ModelConfig(kind=ModelKind.MINI_TRANSFORMER, layers=2, hidden=256, heads=4,
                      vocab=1024, seed=0)
    task = SyntheticTask(kind=TaskKind.SEQUENCE_COPY, seq_len=128, vocab=1024, dataset_seed=0)
    fixtures = {
        "A": (Precision.FULL, lambda: None),
        "B": (Precision.HALF_EMULATED,
              lambda: Stabilizer(ClipMode.by_global_norm(1.0), LossScaler(2.0 ** 16, 2))),
        "C": (Precision.HALF_EMULATED,
              lambda: Stabilizer(ClipMode.by_global_norm(1.0),
                                 LossScaler(2.0 ** 24, 2, max_scale=2.0 ** 24))),
    }
    meta = {"config": {"layers": 2, "hidden": 256, "heads": 4, "vocab": 1024, "seed": 0,
                       "seq_len": 128, "batch": 4, "dataset_seed": 0, "lr": 0.05, "steps": 10}}
    arrays = {}
    toks = sample_batch(task, 4, 0)[1]
    meta["tokens_step0_sha256"] = hashlib.sha256(np.ascontiguousarray(toks).tobytes()).hexdigest()
    for key, (prec, fac) in fixtures.items():
        t0 = time.perf_counter()
        model = build_model(cfg, precision=prec)
        stab = fac()
        opt = LOMO(model, stab)
        rec = {"precision": prec.value, "init_digest": model.digest(), "losses": [],
               "outcomes": [], "log2_scale": [],
               "names": [p.name for p in model.parameters],
               "delivery_order": None}
        for step in range(10):
            loss = opt.step(sample_batch(task, 4, step), 0.05)
            rec["losses"].append(loss)
            rec["outcomes"].append(opt.last_outcome.value if opt.last_outcome else "applied")
            if stab is not None:
                rec["log2_scale"].append(float(np.log2(stab.scaler.scale)))
        rec["seconds"] = time.perf_counter() - t0
        rec["final_digest"] = model.digest()
        rec["sum"] = [float(np.sum(p.value.data)) for p in model.parameters]
        rec["sumsq"] = [float(np.sum(p.value.data ** 2)) for p in model.parameters]
        for p in model.parameters:
            flat = p.value.data.ravel()
            idx = _sample_idx(flat.size, 8192)
            arrays[f"{key}/{p.name}/idx"] = idx.astype(np.int64)
            arrays[f"{key}/{p.name}/val"] = flat[idx]  # float64, exact
        meta[key] = rec
        print(key, rec["outcomes"], rec["log2_scale"], f"{rec['seconds']:.1f}s")
    # delivery order of the reference tape (tape.py:350-360)
    order = []
    m = build_model(cfg)
    out = m.forward(sample_batch(task, 4, 0)[0])
    _, dout = m.loss_and_grad(out, sample_batch(task, 4, 0)[1])

    def hook(p, g):
        order.append(p.name)
        return Disposition.CONSUME
    m.tape.backward(Tensor(dout), hook)
    meta["delivery_order"] = order
    np.savez_compressed(OUT / "c1.npz", **arrays)
    (OUT / "c1.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["hook", "rounding", "scaler", "c1"]
    if "hook" in which:
        hook_cases()
    if "rounding" in which:
        rounding()
    if "scaler" in which:
        scaler_replay()
    if "c1" in which:
        c1()
