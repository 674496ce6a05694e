"""Generate the golden parity fixtures from the REFERENCE itself.

Run in the build container (needs /root/reference and the reference's compiled kernels
in oracle/_ref, built by `make -C oracle ref`):

    python tests/golden/make_golden.py

For every kernel family of the reference registry (tests/test_backends.py:20-27) and
both precisions it evaluates the reference's compiled Cython exports
(_kernels.pyx:419-634) AND its pure-Python twin (_pykernels.py:298-458), asserts they
agree bit for bit (the reference's own `_same` rule, test_backends.py:33-38), and
stores inputs and outputs in golden_vectors.npz.  Inputs follow the reference tests:

* random full-range rows (exponents over the whole format incl. subnormals, random
  signs; the construction of test_backends.py:41-49, seed 2024);
* Cartesian products of special values (test_backends.py:29-30 plus band-edge and
  out-of-band values) in every position;
* the known-answer rows of test_scale.py / test_normalize.py / test_baselines.py and
  the probes of SURVEY.md Appendix A.

Loop checksums (_kernels.pyx:646-789) over a small buffer are stored as well
(iters=37, mask=7 as in test_backends.py:103-104).

The f32 entry points take doubles and cast with <float> (_kernels.pyx:526-527), so the
stored f32 inputs are those casts (what the kernel actually computes on).
"""

from __future__ import annotations

import importlib.util
import itertools
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src/fastnorm"
sys.path.insert(0, REPO)

import oracle  # noqa: E402


def _load_pykernels():
    spec = importlib.util.spec_from_file_location("_ref_pykernels", os.path.join(REF, "_pykernels.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


L = math.ldexp
DBL_MAX = sys.float_info.max
FLT_MAX = float(np.finfo(np.float32).max)

KA = {
    "f64": (L(1, -482), L(1, 510), L(1, 592), L(1, -514), L(1, -592), L(1, 514)),
    "f32": (L(1, -49), L(1, 62), L(1, 100), L(1, -66), L(1, -100), L(1, 66)),
}

FAMILIES = {
    2: ["scale", "normalize", "norm", "naive", "quotient"],
    3: ["scale", "normalize", "norm", "naive", "quotient", "quotient3_fast"],
    4: ["scale", "normalize", "norm", "naive", "quotient"],
}
SCALING = {"scale", "normalize", "norm"}

SPECIALS = {
    "f64": [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 5e-324, L(1, -1022),
            L(1, -482), L(1, 510), DBL_MAX, L(1, -600), -L(3, 600)],
    "f32": [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, L(1, -149), L(1, -126),
            L(1, -49), L(1, 62), FLT_MAX, L(1, -80), -L(3, 80)],
}
SPECIALS4 = {
    "f64": [0.0, -0.0, 1.0, math.inf, math.nan, 5e-324, L(1, 600)],
    "f32": [0.0, -0.0, 1.0, math.inf, math.nan, L(1, -149), L(1, 80)],
}

KATS = {
    2: [(3.0, 4.0), (L(1, -1074), 0.0), (L(1, -500), 0.0), (L(1, 520), L(1, 519)),
        (L(1, -600), 0.0), (L(1, 600), 0.0), (L(1, -1022), math.nextafter(L(1, 510), math.inf)),
        (L(1, 70), 0.0), (L(1, -60), 0.0), (1.0, -0.5)],
    3: [(3.0, 4.0, 12.0), (2.0, 10.0, 11.0), (L(1, 600), L(1, 600), L(1, 600)),
        (DBL_MAX, DBL_MAX, 0.0), (DBL_MAX, DBL_MAX, DBL_MAX), (5e-324, -5e-324, 5e-324),
        (-3.0, 0.0, -0.0), (math.inf, 1.0, -2.0), (math.inf, -math.inf, 1.0),
        (math.inf, math.nan, 1.0), (3e38, 3e38, 1.0), (L(1, 511), L(1, -600), -L(1, 1000)),
        (math.nan, 1.0, 0.0), (math.nan, L(1, 600), 0.0), (L(1, 600), math.nan, 0.0),
        (0.0, math.nan, 0.0), (12.0, 4.0, 3.0), (4.0, 12.0, 3.0), (4.0, 3.0, 12.0),
        (-12.0, 4.0, -3.0), (1.0, 1.0, 1.0), (L(1, -1060), -L(3, -1070), L(1, -1074)),
        (0.0, L(1, -1074), 0.0), (L(1, 70), 0.0, 0.0)],
    4: [(1.0, 1.0, 1.0, 1.0), (3 * L(1, -520), 0.0, 4 * L(1, -520), 0.0),
        (L(1, 600), 0.0, 0.0, L(1, 599)), (1.0, 0.0, 0.0, L(1, -500)),
        (0.0, math.nan, 0.0, 0.0), (0.0, 0.0, math.nan, 0.0), (0.0, 0.0, 0.0, -0.0),
        (L(1, -1074), 0.0, 0.0, 0.0), (DBL_MAX, DBL_MAX, DBL_MAX, DBL_MAX)],
}


def _load_reference_rotation(compiled):
    """The reference's rotation.py (and params.py / scale.py it needs), loaded by path
    under a shim package whose _backend resolves to the reference's compiled kernels --
    the reference package __init__ (gmpy2) is never executed."""
    import types

    pkg = types.ModuleType("fastnorm")
    pkg.__path__ = []
    backend = types.ModuleType("fastnorm._backend")
    suffix = {"single": "f32", "double": "f64"}
    backend.scalar_kernel = lambda base, precision, backend=None: getattr(compiled, f"{base}_{suffix[precision]}")
    sys.modules["fastnorm"] = pkg
    sys.modules["fastnorm._backend"] = backend
    pkg._backend = backend
    mods = {}
    for name in ("params", "scale", "rotation"):
        spec = importlib.util.spec_from_file_location(f"fastnorm.{name}", os.path.join(REF, f"{name}.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[f"fastnorm.{name}"] = mod
        spec.loader.exec_module(mod)
        setattr(pkg, name, mod)
        mods[name] = mod
    return mods["rotation"]


ROT_KATS = [(0.0, 0.0, 0.0, 2.0), (1.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0),
            (0.0, 0.0, 0.0, 1.0), (L(1, 600), -L(1, 600), 3.0 * L(1, 599), 1.0),
            (L(1, -1000), 0.0, L(3, -1001), -L(1, -1070)), (DBL_MAX, DBL_MAX, 0.0, 1.0),
            (5e-324, 0.0, 0.0, 5e-324), (-0.0, 0.0, 1.0, -0.0),
            (0.0, 0.0, 0.0, 0.0), (-0.0, 0.0, -0.0, 0.0), (math.inf, 0.0, 0.0, 1.0),
            (0.0, math.nan, 0.0, 1.0), (0.0, 0.0, 0.0, -math.inf)]  # last 5: rejected (ValueError)


def random_rows(rng, m, dim, single):
    lo, hi = (-149, 127) if single else (-1074, 1023)
    e = rng.integers(lo, hi, (m, dim))
    mant = 1.0 + rng.random((m, dim))
    s = rng.integers(0, 2, (m, dim)) * 2 - 1
    v = np.ldexp(mant, e) * s
    if single:
        v = v.astype(np.float32).astype(np.float64)
    return v


def same(a, b):
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    return a == b and math.copysign(1.0, a) == math.copysign(1.0, b)


def main():
    comp = oracle.ref_module()
    if comp is None:
        oracle.build_ref()
        comp = oracle.ref_module()
    pure = _load_pykernels()
    assert comp.BUILD_FLAGS == "-O3 -ffp-contract=off"
    rng = np.random.default_rng(2024)
    out = {}
    for prec in ("f64", "f32"):
        single = prec == "f32"
        ka = KA[prec]
        for dim in (2, 3, 4):
            rows = []
            rows += [list(r) for r in random_rows(rng, 1024, dim, single)]
            sp = SPECIALS4[prec] if dim == 4 else SPECIALS[prec]
            rows += [list(t) for t in itertools.product(sp, repeat=dim)]
            rows += [list(t) for t in KATS[dim]]
            x64 = np.array(rows, dtype=np.float64)
            with np.errstate(over="ignore"):
                x = x64.astype(np.float32).astype(np.float64) if single else x64
            out[f"{prec}_{dim}_x"] = x
            for fam in FAMILIES[dim]:
                name = f"{fam}{dim}_{prec}" if fam != "quotient3_fast" else f"quotient3_fast_{prec}"
                fc = getattr(comp, name)
                fp = getattr(pure, name)
                res = []
                for row in x.tolist():
                    args = (*ka, *row) if fam in SCALING else tuple(row)
                    a = fc(*args)
                    b = fp(*args)
                    a = (a,) if not isinstance(a, tuple) else a
                    b = (b,) if not isinstance(b, tuple) else b
                    assert all(same(p, q) for p, q in zip(a, b)), (name, row, a, b)
                    res.append(a)
                out[f"{prec}_{name}"] = np.array(res, dtype=np.float64)
            # loop checksums (reference timing loops) over the first 8 random rows
            buf = x[:8]
            flat = np.ascontiguousarray(buf.reshape(-1).astype(np.float32 if single else np.float64))
            loops = {"scaling": f"loop_scaling{dim}", "quotient": f"loop_quotient{dim}",
                     "naive": f"loop_naive{dim}", "empty": f"loop_empty{dim}"}
            if dim == 3:
                loops["quotient_fast"] = "loop_quotient_fast3"
            for algo, base in loops.items():
                fn = getattr(comp, f"{base}_{prec}")
                if algo == "empty":
                    val = fn(flat, 37, 7)
                else:
                    val = fn(flat, 37, 7, *ka)
                out[f"{prec}_{dim}_loop_{algo}"] = np.array([val], dtype=np.float64)
    for prec in ("f64", "f32"):
        out[f"{prec}_ka"] = np.array(KA[prec], dtype=np.float64)

    # rotations (rotation.py:53-111) on quaternions of every magnitude class; rotation_unit
    # is fed both raw quaternions and the reference's own normalize4 unit outputs.
    rot = _load_reference_rotation(comp)
    q = np.concatenate([random_rows(rng, 600, 4, False),
                        rng.standard_normal((600, 4)),
                        np.ldexp(rng.standard_normal((300, 4)), rng.integers(-1000, 1000, (300, 1))),
                        np.array(ROT_KATS)])
    ka = KA["f64"]
    units = np.array([comp.normalize4_f64(*ka, *row)[1:] for row in q.tolist()])
    gen, uni, uni_n = [], [], []
    for row, urow in zip(q.tolist(), units.tolist()):
        try:
            gen.append(rot.rotation_general(row).flat())
        except ValueError:
            gen.append((math.nan,) * 9)
        for dst, src in ((uni, row), (uni_n, urow)):
            try:
                dst.append(rot.rotation_unit(src).flat())
            except ValueError:
                dst.append((math.nan,) * 9)
    out["rot_q"] = q
    out["rot_general"] = np.array(gen)
    out["rot_unit"] = np.array(uni)
    out["rot_unit_of_normalized"] = np.array(uni_n)
    # RotationMatrix.apply (rotation.py:39-41): matrices from rotation_unit of the
    # reference's normalized quaternions and from rotation_general of raw ones, each
    # applied to vectors of every magnitude class and to special-value products.
    mats = [rot.rotation_unit(tuple(u)) for u in units[:6].tolist()]
    mats += [rot.rotation_general(tuple(row)) for row in q[600:604].tolist()]
    mats.append(rot.rotation_unit((0.0, 0.0, 0.0, 1.0)))
    vecs = np.concatenate([random_rows(rng, 400, 3, False), rng.standard_normal((200, 3)),
                           np.array(list(itertools.product(SPECIALS["f64"][:8], repeat=3)))])
    out["rot_apply_R"] = np.array([m.flat() for m in mats])
    out["rot_apply_v"] = vecs
    out["rot_apply_out"] = np.array([[m.apply(tuple(v)) for v in vecs.tolist()] for m in mats])
    # per-row rotation of vectors (two inputs): the reference composition
    # rotation_unit(normalize4(q).unit).apply(v) per quaternion (ValueError -> NaN row), and
    # RotationMatrix.apply of every rotation_general golden matrix to its own vector.
    nq = len(q)
    v_rows = np.concatenate([random_rows(rng, nq // 2, 3, False), rng.standard_normal((nq - nq // 2, 3))])
    sp = SPECIALS["f64"]
    for i in range(0, nq, 37):  # special values sprinkled over the vectors
        v_rows[i, i % 3] = sp[(i // 37) % len(sp)]
    qrot = []
    for urow, vrow in zip(units.tolist(), v_rows.tolist()):
        try:
            qrot.append(rot.rotation_unit(urow).apply(tuple(vrow)))
        except ValueError:
            qrot.append((math.nan,) * 3)
    out["rot_rows_v"] = v_rows
    out["rot_rows_quat_out"] = np.array(qrot)
    mats = [tuple(tuple(m[3 * k:3 * k + 3]) for k in range(3)) for m in out["rot_general"].tolist()]
    out["rot_rows_mat_out"] = np.array([rot.RotationMatrix(m).apply(tuple(vrow))
                                        for m, vrow in zip(mats, v_rows.tolist())])
    path = os.path.join(HERE, "golden_vectors.npz")
    np.savez_compressed(path, **out)
    n = sum(v.size for v in out.values())
    print(f"wrote {path}: {len(out)} arrays, {n} values")


if __name__ == "__main__":
    main()
