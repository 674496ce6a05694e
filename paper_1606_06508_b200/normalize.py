"""Scaling normalization (reference: pkg/src/fastnorm/normalize.py).

Scalar calls keep the reference signatures (``normalize3(p, x1, x2, x3)`` ->
``NormalizeOutcome(length, unit)``, normalize.py:51-89): same parameter names, order and
annotations, so keyword calls work.  Passing one ``[N, n]`` array as ``x1`` and leaving
``x2..xn`` out (their default is the ``ROWS`` marker) selects the batched overload (CUDA
tensor: device path; numpy / CPU tensor: host path),
which returns ``NormalizeOutcome(length=[N], unit=[N, n])`` computed by the B200 kernel
bit-identically to the reference (Appendix A of SURVEY.md).  ``out=(length, unit)``
writes into preallocated arrays.

``normalize{n}_sq`` adds the squared length (BASELINE config 3): no reference function
exists, so it is defined here as ldexp(ss, 2*log2(inv)) with ss the same scaled
left-to-right sum of squares that feeds r -- one correct rounding of inv^2 * ss.
"""

from __future__ import annotations

from typing import Any, NamedTuple

from paper_1606_06508_b200 import _backend, _lib, batch
from paper_1606_06508_b200.batch import ROWS, components
from paper_1606_06508_b200.params import FpParams
from paper_1606_06508_b200.scale import check_precision, kernel_args, kernel_args_array

__all__ = [
    "NormalizeOutcome",
    "NormalizeSqOutcome",
    "normalize2",
    "normalize3",
    "normalize4",
    "normalize2_sq",
    "normalize3_sq",
    "normalize4_sq",
    "norm2",
    "norm3",
    "norm4",
    "normalize_many",
    "norm_many",
]


class NormalizeOutcome(NamedTuple):
    length: Any
    unit: Any


class NormalizeSqOutcome(NamedTuple):
    squared_length: Any
    length: Any
    unit: Any


def _batched(xs) -> bool:
    return len(xs) == 1 and batch.is_array(xs[0])


def _scalars(name: str, dim: int, xs):
    if len(xs) != dim:
        raise TypeError(f"{name} takes {dim} components or one [N, {dim}] array")
    return tuple(float(v) for v in xs)


def _soa(p: FpParams, op: int, dim: int, xs):
    """The scalar signature with one array per component (structure of arrays)."""
    check_precision(p, xs[0])
    return batch.run_soa(op, dim, xs, kernel_args_array(p))


def _normalize(p: FpParams, dim: int, xs, out):
    if batch.is_soa(xs, dim):
        h, b, _ = _soa(p, _lib.OP_NORMALIZE, dim, xs)
        return NormalizeOutcome(h, b)
    if _batched(xs):
        prec = check_precision(p, xs[0])
        res = _backend.batch_kernel(f"normalize{dim}", prec)(xs[0], kernel_args_array(p), out=out)
        return NormalizeOutcome(res.head, res.body)
    k = _backend.scalar_kernel(f"normalize{dim}", p.precision)
    r, *u = k(*kernel_args(p), *_scalars(f"normalize{dim}", dim, xs))
    return NormalizeOutcome(r, tuple(u))


def _normalize_sq(p: FpParams, dim: int, xs, out):
    if batch.is_soa(xs, dim):
        h, b, q = _soa(p, _lib.OP_NORMALIZE_SQ, dim, xs)
        return NormalizeSqOutcome(q, h, b)
    if _batched(xs):
        prec = check_precision(p, xs[0])
        o = None if out is None else (out[1], out[2], out[0])
        res = _backend.batch_kernel(f"normalize{dim}_sq", prec)(xs[0], kernel_args_array(p), out=o)
        return NormalizeSqOutcome(res.sq, res.head, res.body)
    k = _backend.scalar_kernel(f"normalize{dim}_sq", p.precision)
    sq, r, *u = k(*kernel_args(p), *_scalars(f"normalize{dim}_sq", dim, xs))
    return NormalizeSqOutcome(sq, r, tuple(u))


def _norm(p: FpParams, dim: int, xs, out):
    if batch.is_soa(xs, dim):
        return _soa(p, _lib.OP_NORM, dim, xs)[0]
    if _batched(xs):
        prec = check_precision(p, xs[0])
        o = None if out is None else (out,)
        return _backend.batch_kernel(f"norm{dim}", prec)(xs[0], kernel_args_array(p), out=o).head
    k = _backend.scalar_kernel(f"norm{dim}", p.precision)
    return k(*kernel_args(p), *_scalars(f"norm{dim}", dim, xs))


def normalize2(p: FpParams, x1: float, x2: float = ROWS, *, out=None) -> NormalizeOutcome:
    """Length and unit direction of a 2-vector; zero input gives (0, (0, 0))."""
    return _normalize(p, 2, components(x1, x2), out)


def normalize3(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, *, out=None) -> NormalizeOutcome:
    """Length and unit direction of a 3-vector; zero input gives (0, (0, 0, 0))."""
    return _normalize(p, 3, components(x1, x2, x3), out)


def normalize4(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, x4: float = ROWS, *,
               out=None) -> NormalizeOutcome:
    """Length and unit quaternion; the zero quaternion maps to (0, (0, 0, 0, 1))."""
    return _normalize(p, 4, components(x1, x2, x3, x4), out)


def normalize2_sq(p: FpParams, x1: float, x2: float = ROWS, *, out=None) -> NormalizeSqOutcome:
    """normalize2 plus the squared length; ``out=(squared_length, length, unit)``."""
    return _normalize_sq(p, 2, components(x1, x2), out)


def normalize3_sq(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, *,
                  out=None) -> NormalizeSqOutcome:
    """normalize3 plus the squared length; ``out=(squared_length, length, unit)``."""
    return _normalize_sq(p, 3, components(x1, x2, x3), out)


def normalize4_sq(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, x4: float = ROWS, *,
                  out=None) -> NormalizeSqOutcome:
    """normalize4 plus the squared length (BASELINE config 3)."""
    return _normalize_sq(p, 4, components(x1, x2, x3, x4), out)


def norm2(p: FpParams, x1: float, x2: float = ROWS, *, out=None) -> float:
    """Length only; identical to ``normalize2(...).length`` bit for bit."""
    return _norm(p, 2, components(x1, x2), out)


def norm3(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, *, out=None) -> float:
    """Length only; identical to ``normalize3(...).length`` bit for bit."""
    return _norm(p, 3, components(x1, x2, x3), out)


def norm4(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, x4: float = ROWS, *,
          out=None) -> float:
    """Length only; identical to ``normalize4(...).length`` bit for bit."""
    return _norm(p, 4, components(x1, x2, x3, x4), out)


def normalize_many(p: FpParams, xs, out=None) -> list:
    """``normalize{n}`` over several independent ``[N_j, n]`` arrays at once (n from the
    first array): a list of NormalizeOutcome, bit-identical to calling ``normalize{n}`` on
    each.  CUDA tensors go to the device in one launch (fn_run_many), so a stream of small
    batches pays one launch ramp and tail instead of one per batch.  ``out``: optional
    list of ``(length, unit)`` pairs."""
    xs = list(xs)
    if not xs:
        return []
    for x in xs:  # every batch, not just the first: the kernel constants are per precision
        check_precision(p, x)
    dim = int(xs[0].shape[1])
    outs = None if out is None else [tuple(o) for o in out]
    return [NormalizeOutcome(r.head, r.body)
            for r in batch.run_many(_lib.OP_NORMALIZE, dim, xs, kernel_args_array(p), outs)]


def norm_many(p: FpParams, xs, out=None) -> list:
    """``norm{n}`` over several independent arrays at once (see ``normalize_many``)."""
    xs = list(xs)
    if not xs:
        return []
    for x in xs:  # every batch, not just the first: the kernel constants are per precision
        check_precision(p, x)
    dim = int(xs[0].shape[1])
    outs = None if out is None else [(o,) for o in out]
    return [r.head for r in batch.run_many(_lib.OP_NORM, dim, xs, kernel_args_array(p), outs)]
