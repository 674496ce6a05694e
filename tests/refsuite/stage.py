"""Stage the reference package and its own test suite for runs against the "cuda" backend.

TEST INFRASTRUCTURE.  Called by ``__graft_entry__.build()`` in the build container, where
/root/reference exists.  It copies (never into git: ``oracle/_ref/`` is git-ignored, but
it travels to the GPU box with the snapshot, like the compiled reference kernels):

  /root/reference/pkg/src/fastnorm/*.py   -> oracle/_ref/refpkg/src/fastnorm/
  oracle/_ref/_kernels*.so                -> oracle/_ref/refpkg/src/fastnorm/  (the
                                             reference's compiled backend, built by
                                             ``make -C oracle ref`` from its own sources)
  /root/reference/pkg/tests/*.py          -> oracle/_ref/refpkg/tests/
  gmpy2 stand-in                          -> oracle/_ref/refpkg/shim/gmpy2.py

Nothing is edited: the reference's modules and tests run exactly as written.  gmpy2 (the
accuracy oracle's multiple-precision library, pyproject.toml:12) is not installed in this
image; the stand-in is tests/refsuite/gmpy2_shim.py.
"""

from __future__ import annotations

import glob
import os
import shutil

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_PKG = "/root/reference/pkg"
STAGE = os.path.join(REPO, "oracle", "_ref", "refpkg")


def stage() -> str:
    src = os.path.join(REF_PKG, "src", "fastnorm")
    if not os.path.isdir(src):
        raise FileNotFoundError(src)
    shutil.rmtree(STAGE, ignore_errors=True)
    pkg = os.path.join(STAGE, "src", "fastnorm")
    tests = os.path.join(STAGE, "tests")
    shim = os.path.join(STAGE, "shim")
    for d in (pkg, tests, shim):
        os.makedirs(d)
    for f in glob.glob(os.path.join(src, "*.py")):
        shutil.copy2(f, pkg)
    for f in glob.glob(os.path.join(REPO, "oracle", "_ref", "_kernels*.so")):
        shutil.copy2(f, pkg)
    for f in glob.glob(os.path.join(REF_PKG, "tests", "*.py")):
        shutil.copy2(f, tests)
    shutil.copy2(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gmpy2_shim.py"),
                 os.path.join(shim, "gmpy2.py"))
    return STAGE


if __name__ == "__main__":
    print(stage())
