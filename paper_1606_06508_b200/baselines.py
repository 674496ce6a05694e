"""Comparison algorithms (reference: pkg/src/fastnorm/baselines.py).

Naive normalization and the quotient family (Algorithms 1-2 of the paper), kept as
comparison variants.  Scalar signatures and the ``precision=`` keyword follow
baselines.py:30-76; one ``[N, n]`` array selects the batched B200 kernel, whose
precision is the array's dtype (a conflicting ``precision=`` raises).
"""

from __future__ import annotations

from paper_1606_06508_b200 import _backend, _lib, batch
from paper_1606_06508_b200.normalize import NormalizeOutcome

__all__ = [
    "naive_normalize2",
    "naive_normalize3",
    "naive_normalize4",
    "quotient2",
    "quotient3_robust",
    "quotient3_fast",
    "quotient4",
]


def _call(base: str, dim: int, xs, precision, out) -> NormalizeOutcome:
    if len(xs) == dim + 1 and isinstance(xs[-1], str) and precision is None:
        xs, precision = xs[:-1], xs[-1]  # reference order: (x1, ..., xn, precision)
    if batch.is_soa(xs, dim):  # one array per component (structure of arrays)
        prec = batch.precision_of(xs[0])
        if precision is not None and precision != prec:
            raise TypeError(f"rows are {xs[0].dtype} but precision={precision!r}")
        op = {"naive": _lib.OP_NAIVE, "quotient": _lib.OP_QUOTIENT}.get(base.rstrip("234"), _lib.OP_QUOTIENT3_FAST)
        h, b, _ = batch.run_soa(op, dim, xs, None)
        return NormalizeOutcome(h, b)
    if len(xs) == 1 and batch.is_array(xs[0]):
        x = xs[0]
        prec = batch.precision_of(x)
        if precision is not None and precision != prec:
            raise TypeError(f"rows are {x.dtype} but precision={precision!r}")
        res = _backend.batch_kernel(base, prec)(x, None, out=out)
        return NormalizeOutcome(res.head, res.body)
    if len(xs) != dim:
        raise TypeError(f"{base} takes {dim} components or one [N, {dim}] array")
    r, *u = _backend.scalar_kernel(base, precision or "double")(*(float(v) for v in xs))
    return NormalizeOutcome(r, tuple(u))


def naive_normalize2(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    return _call("naive2", 2, xs, precision, out)


def naive_normalize3(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    return _call("naive3", 3, xs, precision, out)


def naive_normalize4(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    return _call("naive4", 4, xs, precision, out)


def quotient2(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    """Max-division quotient normalization of a 2-vector; zero input gives zeros."""
    return _call("quotient2", 2, xs, precision, out)


def quotient3_robust(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    """Divide by the max magnitude, take the norm, divide again (Algorithm 1)."""
    return _call("quotient3", 3, xs, precision, out)


def quotient3_fast(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    """Pivoting variant (Algorithm 2); NaN inputs give NaN outputs."""
    return _call("quotient3_fast", 3, xs, precision, out)


def quotient4(*xs, precision: str | None = None, out=None) -> NormalizeOutcome:
    """Max-division quotient normalization of a quaternion."""
    return _call("quotient4", 4, xs, precision, out)
