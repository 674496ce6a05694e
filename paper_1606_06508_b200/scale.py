"""Scaling preprocessors (reference: pkg/src/fastnorm/scale.py).

``scale{2,3,4}(p, x1, ..., xn)`` keeps the reference's scalar signature and result
(``ScaleOutcome(inv_sigma, scaled)``, scale.py:21-51).  Passing one ``[N, n]`` array
instead of n scalars selects the batched overload: ``inv_sigma`` is then an ``[N]`` array
and ``scaled`` an ``[N, n]`` array, computed by the B200 kernel with the reference's
exact comparison cascade (_kernels.pyx:51-160).
"""

from __future__ import annotations

from functools import lru_cache
from typing import Any, NamedTuple

import numpy as np

from paper_1606_06508_b200 import _backend, _lib, batch
from paper_1606_06508_b200.batch import ROWS, components
from paper_1606_06508_b200.params import FpParams, require_valid

__all__ = ["ScaleOutcome", "kernel_args", "scale2", "scale3", "scale4"]


class ScaleOutcome(NamedTuple):
    inv_sigma: Any
    scaled: Any


@lru_cache(maxsize=None)
def kernel_args(p: FpParams) -> tuple[float, float, float, float, float, float]:
    """(tau_min, tau_max, sigma_min, sigma_max, 1/sigma_min, 1/sigma_max), validated."""
    require_valid(p)
    return (p.tau_min, p.tau_max, p.sigma_min, p.sigma_max, 1.0 / p.sigma_min, 1.0 / p.sigma_max)


@lru_cache(maxsize=None)
def kernel_args_array(p: FpParams) -> np.ndarray:
    arr = np.array(kernel_args(p), dtype=np.float64)
    arr.setflags(write=False)
    return arr


def check_precision(p: FpParams, x) -> str:
    prec = batch.precision_of(x)
    if prec != p.precision:
        raise TypeError(f"rows are {x.dtype} but the parameters are for {p.precision} precision")
    return prec


def _scale(p: FpParams, dim: int, xs, out):
    if batch.is_soa(xs, dim):  # one array per component (structure of arrays)
        check_precision(p, xs[0])
        inv, s, _ = batch.run_soa(_lib.OP_SCALE, dim, xs, kernel_args_array(p))
        return ScaleOutcome(inv, s)
    if len(xs) == 1 and batch.is_array(xs[0]):
        x = xs[0]
        prec = check_precision(p, x)
        res = _backend.batch_kernel(f"scale{dim}", prec)(x, kernel_args_array(p), out=out)
        return ScaleOutcome(res.head, res.body)
    if len(xs) != dim:
        raise TypeError(f"scale{dim} takes {dim} components or one [N, {dim}] array")
    k = _backend.scalar_kernel(f"scale{dim}", p.precision)
    inv, *s = k(*kernel_args(p), *(float(v) for v in xs))
    return ScaleOutcome(inv, tuple(s))


def scale2(p: FpParams, x1: float, x2: float = ROWS, *, out=None) -> ScaleOutcome:
    """Scale a 2-vector (or [N, 2] rows) so max |x_k| lands in [tau_min, tau_max]."""
    return _scale(p, 2, components(x1, x2), out)


def scale3(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, *, out=None) -> ScaleOutcome:
    """Scale a 3-vector (or [N, 3] rows) so its largest magnitude lands in the band."""
    return _scale(p, 3, components(x1, x2, x3), out)


def scale4(p: FpParams, x1: float, x2: float = ROWS, x3: float = ROWS, x4: float = ROWS, *,
           out=None) -> ScaleOutcome:
    """Scale a quaternion (or [N, 4] rows) so its largest magnitude lands in the band."""
    return _scale(p, 4, components(x1, x2, x3, x4), out)
