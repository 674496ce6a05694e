"""Golden batches of the reference's ``generate_inputs`` (pkg/src/fastnorm/bench.py:146-207).

Run in the build container (needs /root/reference):

    python tests/golden/make_generate_inputs.py

Loads the reference's bench.py by path under a stand-in ``fastnorm`` package (its
``__init__`` needs gmpy2, absent here; bench.py itself needs only _backend, params and
scale) and stores one small batch per (regime, dimension, precision, seed) in
generate_inputs.npz.  tests/test_generate_inputs.py compares ours against these bit for
bit wherever the reference is absent, and against the live function where it is present.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src/fastnorm"

REGIMES = ("normal", "subnormal", "huge", "mixed", "unit-ish")
SEEDS = (0, 3, 2024, (1, 2), (7, 0, 3, 1))
COUNT = 97


def load_reference_bench():
    """The reference's bench module, loaded with its real dependencies by path."""
    saved = {k: v for k, v in sys.modules.items() if k == "fastnorm" or k.startswith("fastnorm.")}
    pkg = types.ModuleType("fastnorm")
    pkg.__path__ = [REF]
    sys.modules["fastnorm"] = pkg
    try:
        for name in ("_pykernels", "params", "_backend", "scale", "bench"):
            spec = importlib.util.spec_from_file_location(f"fastnorm.{name}", os.path.join(REF, f"{name}.py"))
            mod = importlib.util.module_from_spec(spec)
            sys.modules[f"fastnorm.{name}"] = mod
            spec.loader.exec_module(mod)
            setattr(pkg, name, mod)
        return sys.modules["fastnorm.bench"]
    finally:
        for k in list(sys.modules):
            if k == "fastnorm" or k.startswith("fastnorm."):
                del sys.modules[k]
        sys.modules.update(saved)


def key(regime, dim, prec, seed) -> str:
    s = "-".join(map(str, seed)) if isinstance(seed, tuple) else str(seed)
    return f"{regime}|{dim}|{prec}|{s}"


def cases():
    for regime in REGIMES:
        for dim in (2, 3, 4):
            for prec in ("double", "single"):
                for seed in SEEDS:
                    yield regime, dim, prec, seed


def main() -> None:
    ref = load_reference_bench()
    out = {key(*c): ref.generate_inputs(c[0], c[1], c[2], COUNT, c[3]) for c in cases()}
    np.savez_compressed(os.path.join(HERE, "generate_inputs.npz"), **out)
    print(f"wrote {len(out)} batches of {COUNT} rows")


if __name__ == "__main__":
    main()
