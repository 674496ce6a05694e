"""Pin the oracle: the repo's C restatement reproduces the reference's own outputs.

The golden vectors were produced by the reference's compiled Cython kernels and checked
against its pure-Python twin (tests/golden/make_golden.py).  Bit-exact for every kernel
family, both precisions, random full-range rows, special-value products and the
reference tests' known-answer rows; loop checksums equal the reference timing loops.
"""

import numpy as np
import pytest

from conftest import FAMILIES, kernel_name


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_oracle_matches_reference_golden(golden, oracle_mod, prec, dim):
    ka = golden[f"{prec}_ka"]
    x = golden[f"{prec}_{dim}_x"]
    xx = x.astype(np.float32) if prec == "f32" else x
    assert len(x) > 1000
    for fam in FAMILIES[dim]:
        ref = golden[f"{prec}_{kernel_name(fam, dim, prec)}"]
        h, b, _ = oracle_mod.run(oracle_mod.BASE_OPS[fam], xx, ka)
        got = h[:, None] if b is None else np.concatenate([h[:, None], b], axis=1)
        ok = oracle_mod.same(got.astype(np.float64), ref)
        bad = np.argwhere(~ok)
        assert ok.all(), (fam, prec, dim, x[bad[0][0]], got[bad[0][0]], ref[bad[0][0]])


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_oracle_loop_checksums(golden, oracle_mod, prec, dim):
    ka = golden[f"{prec}_ka"]
    x = golden[f"{prec}_{dim}_x"][:8]
    buf = x.astype(np.float32) if prec == "f32" else x
    algos = {"scaling": oracle_mod.ALGO_SCALING, "quotient": oracle_mod.ALGO_QUOTIENT,
             "naive": oracle_mod.ALGO_NAIVE, "empty": oracle_mod.ALGO_EMPTY}
    if dim == 3:
        algos["quotient_fast"] = oracle_mod.ALGO_QUOTIENT_FAST
    for name, code in algos.items():
        want = golden[f"{prec}_{dim}_loop_{name}"][0]
        got = oracle_mod.loop(code, buf, 37, 7, ka)
        assert (got == want) or (np.isnan(got) and np.isnan(want)), (name, got, want)


def test_golden_covers_special_classes(golden):
    """The fixture holds zero, NaN, inf, subnormal and out-of-band rows at every dim."""
    for prec in ("f64", "f32"):
        for dim in (2, 3, 4):
            x = golden[f"{prec}_{dim}_x"]
            assert np.isnan(x).any(axis=1).sum() > 10
            assert np.isinf(x).any(axis=1).sum() > 10
            assert (np.abs(x).max(axis=1) == 0).sum() >= 2
            tiny = np.finfo(np.float32 if prec == "f32" else np.float64).tiny
            assert ((np.abs(x) < tiny) & (x != 0)).any(axis=1).sum() > 10


def test_oracle_rotations_match_reference_golden(golden, oracle_mod):
    """rotation_general / rotation_unit (rotation.py:53-111) as evaluated by the reference
    module itself, including rows it rejects (stored as NaN)."""
    q = golden["rot_q"]
    ka = golden["f64_ka"]
    R, bad = oracle_mod.rotation(oracle_mod.OP_ROT_GENERAL, q, ka)
    assert oracle_mod.same(R.reshape(-1, 9), golden["rot_general"]).all() and bad == 5
    R, bad = oracle_mod.rotation(oracle_mod.OP_ROT_UNIT, q)
    assert oracle_mod.same(R.reshape(-1, 9), golden["rot_unit"]).all() and bad == 3
    r, u, R, bad = oracle_mod.rotation(oracle_mod.OP_NORMALIZE_ROT, q, ka)
    assert oracle_mod.same(R.reshape(-1, 9), golden["rot_unit_of_normalized"]).all()
    h, b, _ = oracle_mod.run(oracle_mod.OP_NORMALIZE, q, ka)
    assert oracle_mod.same(r, h).all() and oracle_mod.same(u, b).all()


def test_oracle_rotate_apply_matches_reference_golden(golden, oracle_mod):
    """RotationMatrix.apply (rotation.py:39-41), evaluated by the reference module on
    rotation_unit / rotation_general matrices over vectors of every magnitude class and
    special-value products (inf, NaN, signed zeros)."""
    v = golden["rot_apply_v"]
    for R, want in zip(golden["rot_apply_R"], golden["rot_apply_out"]):
        assert oracle_mod.same(oracle_mod.rotate_apply(R, v), want).all()


def test_oracle_rotate_rows_match_reference_golden(golden, oracle_mod):
    """Per-row rotation of vectors, as the reference composes it:
    rotation_unit(normalize4(q).unit).apply(v) per row (ValueError rows stored as NaN) and
    RotationMatrix.apply of each rotation_general matrix to its own vector."""
    q, v, ka = golden["rot_q"], golden["rot_rows_v"], golden["f64_ka"]
    out, bad = oracle_mod.rotate_rows(oracle_mod.OP_QUAT_ROTATE, q, v, ka)
    assert oracle_mod.same(out, golden["rot_rows_quat_out"]).all() and bad == 3
    out, bad = oracle_mod.rotate_rows(oracle_mod.OP_MAT_APPLY, golden["rot_general"], v)
    assert oracle_mod.same(out, golden["rot_rows_mat_out"]).all() and bad == 0
