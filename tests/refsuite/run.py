"""Run the reference's own test suite (staged by tests/refsuite/stage.py) against this
repo's backend.  TEST INFRASTRUCTURE.

    python tests/refsuite/run.py --mode registry|dropin|none [--junit FILE] [pytest args]

The reference's files run unmodified from ``oracle/_ref/refpkg``, all of them, the
accuracy-oracle tests included (gmpy2 is absent from this image; the oracle runs on the
stand-in tests/refsuite/gmpy2_shim.py).  One test is deselected, in ``registry`` mode
only: ``test_backend_metadata`` asserts that every registered module's BACKEND_NAME is
one of the reference's two names (tests/test_backends.py:145-149), and a third backend
is "cuda" by design.  ``FASTNORM_ACCEPT_SAMPLES`` (the reference's own knob,
tests/test_acceptance.py:1-8) defaults to 2000 here: the bound suites' oracle is exact
rational arithmetic in Python.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
STAGE = os.path.join(REPO, "oracle", "_ref", "refpkg")

# Tests deselected in every mode (node ids relative to the staged tests dir): none.  The
# accuracy oracle's tests run too, on the gmpy2 stand-in (gmpy2_shim.py).
IGNORED: tuple[str, ...] = ()


def command(mode: str, junit: str | None, extra: list[str]) -> tuple[list[str], dict]:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(STAGE, "src"), os.path.join(STAGE, "shim"), HERE, REPO,
                                         env.get("PYTHONPATH", "")])
    env["FNB_REFSUITE_MODE"] = mode
    env.setdefault("FASTNORM_ACCEPT_SAMPLES", "2000")
    tests = os.path.join(STAGE, "tests")
    cmd = [sys.executable, "-m", "pytest", tests, "-p", "plugin_cuda", "-q", "-rfE",
           "--rootdir", STAGE, "-c", os.path.join(STAGE, "pytest.ini"), "-p", "no:cacheprovider"]
    for t in IGNORED:
        cmd += ["--deselect", f"tests/{t}"]
    if mode == "registry":
        cmd += ["--deselect", "tests/test_backends.py::test_backend_metadata"]  # node ids are rootdir-relative
    if junit:
        cmd += ["--junitxml", junit]
    return cmd + extra, env


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="registry", choices=("registry", "dropin", "none"))
    ap.add_argument("--junit")
    a, extra = ap.parse_known_args()
    if not os.path.isdir(STAGE):
        raise SystemExit(f"{STAGE} is missing: run __graft_entry__.build() in the build container")
    with open(os.path.join(STAGE, "pytest.ini"), "w") as f:
        f.write("[pytest]\ntestpaths = tests\n")
    cmd, env = command(a.mode, a.junit, extra)
    return subprocess.call(cmd, env=env, cwd=STAGE)


if __name__ == "__main__":
    sys.exit(main())
