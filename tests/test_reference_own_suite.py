"""The reference's OWN test suite (pkg/tests, every module, unmodified) run against this
repo's B200 backend, in a subprocess per mode (tests/refsuite/run.py):

* ``registry`` (GPU) -- ``_MODULES["cuda"]`` beside the reference's compiled and python
  backends, the maintainer's patch of INTEGRATION.md §2.  Every test that takes the
  reference conftest's ``backend`` fixture (tests/conftest.py:10-14) runs once with
  ``cuda``: the KATs and contracts of test_scale / test_normalize / test_baselines /
  test_rotation, the loop-checksum identities of test_backends.py:88-142, ...
* ``dropin`` (GPU) -- the B200 module in the compiled extension's slot.  The reference's
  compiled-vs-twin bit-parity sweeps (test_backends.py:52-85: 800 random full-range rows
  x 16 kernels x 2 precisions, and every special-value product) then compare the GPU
  with the pure-Python twin, and every default-backend call of the suite -- acceptance
  criteria 1-8 included, the accuracy bounds measured by the reference's own oracle --
  computes on the GPU.
* ``none`` (CPU) -- the reference as shipped, the control showing the staged suite and
  the gmpy2 stand-in are sound.

The staged copy (oracle/_ref/refpkg) is made by ``__graft_entry__.build()`` where
/root/reference exists and travels to the GPU box with the snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
STAGE = os.path.join(REPO, "oracle", "_ref", "refpkg")
RUN = os.path.join(HERE, "refsuite", "run.py")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(STAGE, "tests")),
                                reason="reference suite not staged (run __graft_entry__.build() where /root/reference exists)")


def _run(mode: str, tmp_path, timeout: int = 1800):
    # the reference's acceptance sweeps at 20k samples per suite (its knob,
    # tests/test_acceptance.py:1-8; the shipped 10^6 would take hours on the exact
    # rational oracle)
    os.environ.setdefault("FASTNORM_ACCEPT_SAMPLES", "20000")
    junit = str(tmp_path / f"refsuite_{mode}.xml")
    log = str(tmp_path / f"refsuite_{mode}.log")
    with open(log, "w") as f:
        rc = subprocess.call([sys.executable, RUN, "--mode", mode, "--junit", junit], stdout=f,
                             stderr=subprocess.STDOUT, timeout=timeout)
    out = os.environ.get("FNB_REFSUITE_LOG_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        import shutil

        shutil.copy(log, os.path.join(out, f"refsuite_{mode}.log"))
        shutil.copy(junit, os.path.join(out, f"refsuite_{mode}.xml"))
    cases = {}
    for tc in ET.parse(junit).getroot().iter("testcase"):
        name = f"{tc.get('classname')}::{tc.get('name')}"
        kinds = {c.tag for c in tc}
        cases[name] = ("failed" if kinds & {"failure", "error"} else "skipped" if "skipped" in kinds else "passed")
    with open(log) as f:
        tail = f.read()[-4000:]
    return rc, cases, tail


def _summary(cases):
    s = {"passed": 0, "failed": 0, "skipped": 0}
    for v in cases.values():
        s[v] += 1
    return s


def test_reference_suite_control_cpu(tmp_path):
    """The reference's suite on its own backends: everything passes (control)."""
    rc, cases, tail = _run("none", tmp_path)
    s = _summary(cases)
    assert rc == 0 and s["failed"] == 0, tail
    assert s["passed"] >= 340, s


@pytest.mark.gpu
def test_reference_suite_registry_mode(tmp_path):
    rc, cases, tail = _run("registry", tmp_path)
    s = _summary(cases)
    assert rc == 0 and s["failed"] == 0, tail
    cuda = {k: v for k, v in cases.items() if "[cuda" in k or "-cuda" in k}
    # every backend-parametrised test ran with the cuda backend, and passed
    assert len(cuda) >= 90, (len(cuda), s)
    assert all(v != "failed" for v in cuda.values())
    for mod in ("test_scale", "test_normalize", "test_baselines", "test_backends"):
        assert any(k.startswith(f"tests.{mod}") or f"{mod}." in k for k in cuda), mod


@pytest.mark.gpu
def test_reference_suite_dropin_mode(tmp_path):
    rc, cases, tail = _run("dropin", tmp_path)
    s = _summary(cases)
    assert rc == 0 and s["failed"] == 0, tail
    must_pass = [k for k in cases if "test_bit_parity_random_sweep" in k or "test_bit_parity_special_values" in k
                 or "test_criterion_5" in k or "test_criterion_2" in k or "test_backend_metadata" in k]
    assert len(must_pass) >= 8, must_pass
    assert all(cases[k] == "passed" for k in must_pass), {k: cases[k] for k in must_pass}
