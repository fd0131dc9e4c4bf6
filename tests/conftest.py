import json
import os
import sys

os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    # the C-ABI library is an in-tree build artefact (git-ignored): build it
    # once if a fresh checkout lacks it (nvcc cross-compiles without a GPU)
    lib = ROOT / "paper_2306_09782_b200" / "_native" / "liblomo_b200.so"
    if not lib.exists():
        import __graft_entry__
        __graft_entry__.build()


@pytest.fixture(scope="session")
def hook_cases():
    meta = json.loads((GOLDEN / "hook_cases.json").read_text())
    arrs = np.load(GOLDEN / "hook_cases.npz")
    return meta, {k: arrs[k].astype(np.float64) for k in arrs.files}


@pytest.fixture(scope="session")
def c1_meta():
    return json.loads((GOLDEN / "c1.json").read_text())


@pytest.fixture(scope="session")
def c1_arrays():
    arrs = np.load(GOLDEN / "c1.npz")
    return {k: arrs[k] for k in arrs.files}


@pytest.fixture(scope="session")
def reference():
    """The live reference package (build container only); skip elsewhere."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import fusedtrain
    return fusedtrain


def case_arrays(arrays, name, nshapes):
    """Unpack p0, per-step G and per-step p of one hook case."""
    p = {}
    g = {}
    k = 0
    while f"{name}/p{k}_0" in arrays:
        p[k] = [arrays[f"{name}/p{k}_{i}"] for i in range(nshapes)]
        if f"{name}/G{k}_0" in arrays:
            g[k] = [arrays[f"{name}/G{k}_{i}"] for i in range(nshapes)]
        k += 1
    return p, g
