"""pytest plugin (``-p plugin_cuda``) that plugs this repo's B200 backend into the
reference package before the reference's own conftest and tests are imported.

TEST INFRASTRUCTURE.  ``FNB_REFSUITE_MODE`` selects how, both as INTEGRATION.md
describes for a maintainer:

* ``registry`` -- the maintainer's patch of INTEGRATION.md §2: ``_MODULES["cuda"]`` is
  added beside the reference's compiled and python backends
  (pkg/src/fastnorm/_backend.py:25-28).  The reference conftest's ``backend`` fixture
  (tests/conftest.py:10-14) then runs every backend-parametrised test once per backend,
  cuda included.
* ``dropin`` -- the B200 module takes the compiled extension's slot (``_MODULES
  ["compiled"]``, what ``from fastnorm import _kernels`` resolves at
  _backend.py:21-24), under the extension's own ``BACKEND_NAME``.  The reference's
  compiled-vs-twin parity tests (tests/test_backends.py:52-85) then compare the GPU
  against the pure-Python twin bit for bit, and every default-backend call in the
  suite (wrappers, rotation, bench, CLI) computes on the GPU.
* ``none`` -- the reference as it ships (the control run).
"""

from __future__ import annotations

import os
import types

MODE = os.environ.get("FNB_REFSUITE_MODE", "registry")

from fastnorm import _backend  # noqa: E402  (the staged reference package)

if MODE != "none":
    from paper_1606_06508_b200 import _cuda_kernels  # noqa: E402

    if MODE == "registry":
        _backend._MODULES["cuda"] = _cuda_kernels
    elif MODE == "dropin":
        dropin = types.ModuleType("fastnorm._kernels")
        dropin.__dict__.update({k: v for k, v in vars(_cuda_kernels).items() if not k.startswith("__")})
        dropin.BACKEND_NAME = "compiled"
        dropin.BUILD_FLAGS = _cuda_kernels.BUILD_FLAGS  # a lazy module attribute there
        _backend._MODULES["compiled"] = dropin
        if _backend._DEFAULT != "compiled":
            raise RuntimeError("the reference's default backend is not the compiled slot")
    else:
        raise ValueError(f"FNB_REFSUITE_MODE={MODE!r}")


def pytest_report_header(config):
    mods = {k: getattr(v, "BACKEND_NAME", "?") + " @ " + getattr(v, "__name__", "?")
            for k, v in _backend._MODULES.items()}
    return [f"refsuite mode: {MODE}; registry: {mods}; default: {_backend.backend_name()}"]


def pytest_terminal_summary(terminalreporter):
    with open("/proc/self/maps") as f:
        libs = sorted({line.split()[-1] for line in f if line.rstrip().endswith(".so")
                       and ("fastnorm" in line or "_kernels" in line)})
    terminalreporter.write_line(f"refsuite mode {MODE}: libraries mapped: {libs}")
