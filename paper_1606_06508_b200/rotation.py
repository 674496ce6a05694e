"""Quaternion -> 3x3 rotation matrix (reference: pkg/src/fastnorm/rotation.py).

Convention as the reference: q = (q1, q2, q3, q4), q4 the scalar part, (0, 0, 0, 1) the
identity; matrices row-major.  ``rotation_general`` scales the quaternion with the exact
``scale4`` cascade so any finite nonzero magnitude works (rotation.py:53-84);
``rotation_unit`` assumes norm 1 (rotation.py:87-111).

Scalar calls keep the reference signatures and return :class:`RotationMatrix` (one GPU
launch each).  One ``[N, 4]`` float64 array selects the batched kernels and returns an
``[N, 3, 3]`` array; rows the reference would reject with ValueError (non-finite
components; the zero quaternion for the general form) come back as NaN matrices and, with
``strict=True`` (default), make the call raise ValueError after the kernel ran.

:func:`normalize4_rotation` fuses ``normalize4`` with ``rotation_unit`` of its unit
output in one pass over HBM (reads 32 B, writes r, unit and R: 8 + 32 + 72 B per row),
saving the round trip through the unit quaternions; bit-identical to the two calls.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Any, NamedTuple

import numpy as np

from paper_1606_06508_b200 import _lib, batch
from paper_1606_06508_b200.params import FpParams, preset
from paper_1606_06508_b200.scale import check_precision, kernel_args_array

__all__ = ["RotationMatrix", "NormalizeRotationOutcome", "rotation_general", "rotation_unit",
           "normalize4_rotation", "rotate_vectors", "normalize4_rotate", "apply_rotations"]

Row = tuple[float, float, float]


@dataclass(frozen=True)
class RotationMatrix:
    """3x3 rotation matrix, row-major (rotation.py:27-41)."""

    rows: tuple[Row, Row, Row]

    def __getitem__(self, i: int) -> Row:
        return self.rows[i]

    def flat(self) -> tuple[float, ...]:
        return self.rows[0] + self.rows[1] + self.rows[2]

    def apply(self, v, out=None):
        """Matrix-vector product R @ v (rotation.py:39-41).

        A 3-tuple is evaluated like the reference (its Python glue, not a kernel).  One
        [N, 3] float64 array (CUDA tensor or host array) selects the batched kernel
        (FN_OP_ROT_APPLY: 24 B in, 24 B out per vector, R in the kernel arguments),
        bit-identical to applying the reference row by row."""
        if batch.is_array(v) and v.ndim == 2:
            if str(v.dtype).replace("torch.", "") != "float64":
                raise TypeError("apply takes float64 vectors (the reference computes in double)")
            R = np.array(self.flat(), dtype=np.float64)
            return batch.run(_lib.OP_ROT_APPLY, 3, v, R, out=None if out is None else (out,)).head
        return tuple(r[0] * v[0] + r[1] * v[1] + r[2] * v[2] for r in self.rows)


class NormalizeRotationOutcome(NamedTuple):
    length: Any
    unit: Any
    rotation: Any


def _scalar_quaternion(q) -> np.ndarray:
    vals = tuple(float(c) for c in q)
    if len(vals) != 4:
        raise ValueError(f"quaternion needs 4 components, got {len(vals)}")
    if not all(math.isfinite(c) for c in vals):
        raise ValueError(f"quaternion components must be finite, got {vals}")
    return np.array([vals], dtype=np.float64)


def _as_matrix(m: np.ndarray) -> RotationMatrix:
    return RotationMatrix(tuple(tuple(float(v) for v in row) for row in m))


def _batched(op: int, q, strict: bool, what: str, out=None):
    if str(q.dtype).replace("torch.", "") != "float64":
        raise TypeError(f"{what} takes float64 quaternions (the reference computes in double)")
    ka = kernel_args_array(preset("double")) if op != _lib.OP_ROT_UNIT else None
    if batch.is_torch(q) and q.is_cuda:
        import torch

        invalid = torch.zeros(1, dtype=torch.int64, device=q.device)
        res = batch.run(op, 4, q, ka, out=None if out is None else (out,), invalid=invalid)
        if strict:
            bad = int(invalid.item())
            if bad:
                raise ValueError(f"{what}: {bad} quaternion(s) are non-finite"
                                 + (" or zero" if op == _lib.OP_ROT_GENERAL else ""))
        return res.head
    res = batch.run(op, 4, q, ka, out=None if out is None else (out,))
    if strict:
        head = res.head.numpy() if batch.is_torch(res.head) else res.head
        bad = int(np.isnan(head[:, 0, 0]).sum())
        if bad:
            raise ValueError(f"{what}: {bad} quaternion(s) are non-finite"
                             + (" or zero" if op == _lib.OP_ROT_GENERAL else ""))
    return res.head


def _scalar_rotation(op: int, q) -> np.ndarray:
    """One quaternion through fn_scalar (row in the kernel parameters): R[3, 3]."""
    from paper_1606_06508_b200 import _cuda_kernels

    row = _scalar_quaternion(q)
    fast = _cuda_kernels._scalar_entry()
    if fast is None:  # extension not built: the host-array path (also the GPU)
        ka = kernel_args_array(preset("double")) if op == _lib.OP_ROT_GENERAL else None
        return batch.run(op, 4, row, ka).head[0]
    args = tuple(row[0].tolist())
    if op == _lib.OP_ROT_GENERAL:
        args = tuple(kernel_args_array(preset("double")).tolist()) + args
    res = fast(op, 4, _lib.F64, 9, False, args)
    if type(res) is int:
        _lib.check(res, "rotation")
    return np.array(res, dtype=np.float64).reshape(3, 3)


def rotation_general(q, strict: bool = True, out=None):
    """Rotation matrix of an arbitrary nonzero quaternion (or [N, 4] quaternions)."""
    if batch.is_array(q) and q.ndim == 2:
        return _batched(_lib.OP_ROT_GENERAL, q, strict, "rotation_general", out)
    m = _scalar_rotation(_lib.OP_ROT_GENERAL, q)
    if np.isnan(m[0, 0]):
        raise ValueError("zero quaternion has no rotation matrix")
    return _as_matrix(m)


def rotation_unit(q, strict: bool = True, out=None):
    """Rotation matrix of a unit quaternion (or [N, 4] unit quaternions); no norm taken."""
    if batch.is_array(q) and q.ndim == 2:
        return _batched(_lib.OP_ROT_UNIT, q, strict, "rotation_unit", out)
    return _as_matrix(_scalar_rotation(_lib.OP_ROT_UNIT, q))


def rotate_vectors(q, v, method: str = "unit", out=None):
    """Rotate the vectors v[N, 3] (float64; CUDA tensor or host array) by one quaternion:
    ``rotation_{method}(q).apply(v)`` -- one scalar launch for the matrix, then one
    streaming pass over the vectors."""
    if method not in ("unit", "general"):
        raise ValueError(f"method must be 'unit' or 'general', got {method!r}")
    m = rotation_unit(q) if method == "unit" else rotation_general(q)
    return m.apply(v, out=out)


def normalize4_rotation(p: FpParams, q, out=None) -> NormalizeRotationOutcome:
    """normalize4 and rotation_unit of its unit quaternion in one pass.

    ``q``: [N, 4] float64 (CUDA tensor or host array).  Returns (length [N], unit [N, 4],
    rotation [N, 3, 3]); rows with NaN / inf components give NaN rotations (the
    reference's rotation_unit would raise on their non-finite unit output)."""
    check_precision(p, q)
    if p.precision != "double":
        raise TypeError("normalize4_rotation computes in double precision")
    res = batch.run(_lib.OP_NORMALIZE_ROT, 4, q, kernel_args_array(p), out=out)
    return NormalizeRotationOutcome(res.head, res.body, res.sq)


def normalize4_rotate(p: FpParams, q, v, out=None, strict: bool = True):
    """Rotate every vector v[i] by its own quaternion q[i] in one pass:
    ``rotation_unit(normalize4(p, *q[i]).unit).apply(v[i])`` bit for bit
    (normalize.py:65, rotation.py:87-111, :39-41), without materialising the unit
    quaternions or the matrices (56 B in, 24 B out per row).

    ``q``: [N, 4], ``v``: [N, 3], float64, both CUDA tensors on one device or both host
    arrays.  Rows with a non-finite quaternion -- where the reference's rotation_unit
    raises ValueError -- come back as NaN and, with ``strict`` (default), make the call
    raise ValueError after the kernel ran."""
    check_precision(p, q)
    if p.precision != "double":
        raise TypeError("normalize4_rotate computes in double precision")
    ka = kernel_args_array(p)
    if batch.is_torch(q) and q.is_cuda:
        import torch

        invalid = torch.zeros(1, dtype=torch.int64, device=q.device)
        res = batch.run_rows2(_lib.OP_QUAT_ROTATE, q, v, ka, out=out, invalid=invalid)
        bad = int(invalid.item()) if strict else 0
    else:
        res = batch.run_rows2(_lib.OP_QUAT_ROTATE, q, v, ka, out=out)
        qa = q.numpy() if batch.is_torch(q) else np.asarray(q)
        bad = int((~np.isfinite(qa).all(axis=1)).sum()) if strict else 0
    if bad:
        raise ValueError(f"normalize4_rotate: {bad} quaternion(s) are non-finite")
    return res


def apply_rotations(R, v, out=None):
    """Per-row ``RotationMatrix.apply`` (rotation.py:39-41): out[i] = R[i] @ v[i] with the
    reference's evaluation order.  ``R``: [N, 3, 3] or [N, 9] row-major, ``v``: [N, 3],
    float64, same home (CUDA tensors on one device, or host arrays)."""
    n = int(v.shape[0])
    Rf = R.reshape(n, 9)
    return batch.run_rows2(_lib.OP_MAT_APPLY, Rf, v, None, out=out)
