"""Comparison algorithms (reference: pkg/src/fastnorm/baselines.py).

Naive normalization and the quotient family (Algorithms 1-2 of the paper), kept as
comparison variants.  Scalar signatures -- named ``x1..xn`` and
``precision="double"`` -- follow baselines.py:30-76.  One ``[N, n]`` array as ``x1``
(``x2..xn`` left out) selects the batched B200 kernel, whose precision is the array's
dtype (an explicitly conflicting ``precision=`` raises).
"""

from __future__ import annotations

from paper_1606_06508_b200 import _backend, _lib, batch
from paper_1606_06508_b200.batch import ROWS, components
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


class _Double(str):
    """The reference's default ``precision="double"`` (baselines.py:30-76), as a distinct
    object so an array call can tell "not given" (the array's dtype decides) from an
    explicit ``precision="double"`` (must match the dtype)."""

    __slots__ = ()


DOUBLE = _Double("double")


def _call(base: str, dim: int, xs, precision, out) -> NormalizeOutcome:
    if len(xs) == 2 and isinstance(xs[1], str) and batch.is_array(xs[0]):
        xs, precision = xs[:1], xs[1]  # rows with a positional precision: quotient2(X, "single")
    explicit = precision is not DOUBLE
    if batch.is_soa(xs, dim):  # one array per component (structure of arrays)
        prec = batch.precision_of(xs[0])
        if explicit and precision != prec:
            raise TypeError(f"rows are {xs[0].dtype} but precision={precision!r}")
        op = {"naive": _lib.OP_NAIVE, "quotient": _lib.OP_QUOTIENT}.get(base.rstrip("234"), _lib.OP_QUOTIENT3_FAST)
        h, b, _ = batch.run_soa(op, dim, xs, None)
        return NormalizeOutcome(h, b)
    if len(xs) == 1 and batch.is_array(xs[0]):
        x = xs[0]
        prec = batch.precision_of(x)
        if explicit and precision != prec:
            raise TypeError(f"rows are {x.dtype} but precision={precision!r}")
        res = _backend.batch_kernel(base, prec)(x, None, out=out)
        return NormalizeOutcome(res.head, res.body)
    if len(xs) != dim:
        raise TypeError(f"{base} takes {dim} components or one [N, {dim}] array")
    r, *u = _backend.scalar_kernel(base, str(precision))(*(float(v) for v in xs))
    return NormalizeOutcome(r, tuple(u))


def naive_normalize2(x1: float, x2: float = ROWS, precision: str = DOUBLE, *, out=None) -> NormalizeOutcome:
    return _call("naive2", 2, components(x1, x2), precision, out)


def naive_normalize3(x1: float, x2: float = ROWS, x3: float = ROWS, precision: str = DOUBLE, *,
                     out=None) -> NormalizeOutcome:
    return _call("naive3", 3, components(x1, x2, x3), precision, out)


def naive_normalize4(
    x1: float, x2: float = ROWS, x3: float = ROWS, x4: float = ROWS, precision: str = DOUBLE, *, out=None
) -> NormalizeOutcome:
    return _call("naive4", 4, components(x1, x2, x3, x4), precision, out)


def quotient2(x1: float, x2: float = ROWS, precision: str = DOUBLE, *, out=None) -> NormalizeOutcome:
    """Max-division quotient normalization of a 2-vector; zero input gives zeros."""
    return _call("quotient2", 2, components(x1, x2), precision, out)


def quotient3_robust(x1: float, x2: float = ROWS, x3: float = ROWS, precision: str = DOUBLE, *,
                     out=None) -> NormalizeOutcome:
    """Divide by the max magnitude, take the norm, divide again (Algorithm 1)."""
    return _call("quotient3", 3, components(x1, x2, x3), precision, out)


def quotient3_fast(x1: float, x2: float = ROWS, x3: float = ROWS, precision: str = DOUBLE, *,
                   out=None) -> NormalizeOutcome:
    """Pivoting variant (Algorithm 2); NaN inputs give NaN outputs."""
    return _call("quotient3_fast", 3, components(x1, x2, x3), precision, out)


def quotient4(
    x1: float, x2: float = ROWS, x3: float = ROWS, x4: float = ROWS, precision: str = DOUBLE, *, out=None
) -> NormalizeOutcome:
    """Max-division quotient normalization of a quaternion."""
    return _call("quotient4", 4, components(x1, x2, x3, x4), precision, out)
