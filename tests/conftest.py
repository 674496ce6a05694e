"""Shared fixtures.  Tests marked `gpu` need a B200 (run with -m gpu on the GPU box);
everything else runs on the CPU-only build container (-m "not gpu")."""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "golden_vectors.npz")

FAMILIES = {
    2: ["scale", "normalize", "norm", "naive", "quotient"],
    3: ["scale", "normalize", "norm", "naive", "quotient", "quotient3_fast"],
    4: ["scale", "normalize", "norm", "naive", "quotient"],
}
SCALING = {"scale", "normalize", "norm"}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    _ensure_built()


def _ensure_built():
    """Build the in-tree libraries if a fresh checkout lacks them (nvcc cross-compiles
    without a GPU; ~20 s).  Never falls back to anything: a failed build fails loudly."""
    import subprocess

    lib = os.path.join(REPO, "paper_1606_06508_b200", "libfastnorm_b200.so")
    orc = os.path.join(REPO, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j4", "-C", os.path.join(REPO, "paper_1606_06508_b200", "csrc")],
                       check=True)
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle"), "liboracle.so"], check=True)


def kernel_name(fam: str, dim: int, prec: str) -> str:
    return f"quotient3_fast_{prec}" if fam == "quotient3_fast" else f"{fam}{dim}_{prec}"


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def cuda_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def same_scalar(a: float, b: float) -> bool:
    """The reference's parity rule (test_backends.py:33-38)."""
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    return a == b and math.copysign(1.0, a) == math.copysign(1.0, b)
