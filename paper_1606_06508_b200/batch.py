"""Array plumbing between the public API and the C ABI.

Accepts ``[N, n]`` row arrays in either of two homes:

* a CUDA ``torch.Tensor`` -- outputs are allocated on the same device, the kernel is
  enqueued on torch's current stream of that device (``fn_run``), nothing synchronises;
* a host array (``numpy.ndarray`` or CPU ``torch.Tensor``) -- outputs are host arrays of
  the same kind; the library copies in, computes on the current CUDA device and copies
  out (``fn_host_run``: chunked H2D / kernel / D2H pipeline).  Page-locked (pinned)
  host memory gives full PCIe bandwidth.

No path computes on the CPU: without the CUDA library every call raises.
"""

from __future__ import annotations

from typing import Any, NamedTuple

import numpy as np

from paper_1606_06508_b200 import _lib

_HAS_BODY = {
    _lib.OP_SCALE: True,
    _lib.OP_NORMALIZE: True,
    _lib.OP_NORMALIZE_SQ: True,
    _lib.OP_NORM: False,
    _lib.OP_NAIVE: True,
    _lib.OP_QUOTIENT: True,
    _lib.OP_QUOTIENT3_FAST: True,
}


class BatchOut(NamedTuple):
    head: Any
    body: Any
    sq: Any


def _torch():
    import torch  # local: the numpy path must not pay for importing torch

    return torch


def is_torch(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and t.__name__ in ("Tensor", "Parameter")


def is_array(x) -> bool:
    """True for the batched overloads (an ``[N, n]`` array instead of n scalars)."""
    return isinstance(x, np.ndarray) or is_torch(x)


def _dtype_code(dtype_name: str) -> int:
    if dtype_name == "float64":
        return _lib.F64
    if dtype_name == "float32":
        return _lib.F32
    raise TypeError(f"rows must be float32 or float64, got {dtype_name}")


def precision_of(x) -> str:
    name = str(x.dtype).replace("torch.", "")
    return "double" if _dtype_code(name) == _lib.F64 else "single"


def _check_out(o, shape, like, what):
    if o is None:
        return None
    if tuple(o.shape) != tuple(shape):
        raise ValueError(f"out {what} has shape {tuple(o.shape)}, expected {tuple(shape)}")
    if str(o.dtype) != str(like.dtype):
        raise TypeError(f"out {what} has dtype {o.dtype}, expected {like.dtype}")
    if is_torch(like):
        if not is_torch(o) or o.device != like.device or not o.is_contiguous():
            raise ValueError(f"out {what} must be a contiguous tensor on {like.device}")
    elif not (isinstance(o, np.ndarray) and o.flags.c_contiguous):
        raise ValueError(f"out {what} must be a C-contiguous numpy array")
    return o


def run(op: int, dim: int, x, ka_arr: np.ndarray | None, out=None) -> BatchOut:
    """Run kernel family ``op`` over rows ``x[N, dim]``; return (head, body, sq)."""
    if x.ndim != 2 or x.shape[1] != dim:
        raise ValueError(f"expected rows of shape [N, {dim}], got {tuple(x.shape)}")
    has_body = _HAS_BODY[op]
    has_sq = op == _lib.OP_NORMALIZE_SQ
    n = int(x.shape[0])
    L = _lib.lib()
    kptr = None if ka_arr is None else ka_arr.ctypes.data
    outs = tuple(out) if out is not None else ()
    want = 1 + int(has_body) + int(has_sq)
    if out is not None and len(outs) != want:
        raise ValueError(f"out must hold {want} arrays")

    if is_torch(x):
        torch = _torch()
        dcode = _dtype_code(str(x.dtype).replace("torch.", ""))
        if x.is_cuda:
            x = x.contiguous()
            head = _check_out(outs[0] if outs else None, (n,), x, "head")
            body = _check_out(outs[1] if outs and has_body else None, (n, dim), x, "body")
            sq = _check_out(outs[-1] if outs and has_sq else None, (n,), x, "sq")
            head = head if head is not None else torch.empty((n,), dtype=x.dtype, device=x.device)
            if has_body and body is None:
                body = torch.empty((n, dim), dtype=x.dtype, device=x.device)
            if has_sq and sq is None:
                sq = torch.empty((n,), dtype=x.dtype, device=x.device)
            with torch.cuda.device(x.device):
                stream = torch.cuda.current_stream(x.device).cuda_stream
                rc = L.fn_run(op, dim, dcode, x.data_ptr(), n, head.data_ptr(),
                              body.data_ptr() if has_body else None,
                              sq.data_ptr() if has_sq else None, kptr, stream)
            _lib.check(rc, "fn_run")
            return BatchOut(head, body if has_body else None, sq if has_sq else None)
        # CPU tensor: host path, results as CPU tensors sharing the numpy buffers
        res = run(op, dim, x.contiguous().numpy(), ka_arr,
                  None if out is None else tuple(o.numpy() for o in outs))
        conv = (lambda a: None if a is None else torch.from_numpy(a))
        return BatchOut(conv(res.head), conv(res.body), conv(res.sq))

    if not isinstance(x, np.ndarray):
        raise TypeError(f"rows must be a numpy array or torch tensor, got {type(x).__name__}")
    dcode = _dtype_code(str(x.dtype))
    x = np.ascontiguousarray(x)
    head = _check_out(outs[0] if outs else None, (n,), x, "head")
    body = _check_out(outs[1] if outs and has_body else None, (n, dim), x, "body")
    sq = _check_out(outs[-1] if outs and has_sq else None, (n,), x, "sq")
    head = head if head is not None else np.empty((n,), dtype=x.dtype)
    if has_body and body is None:
        body = np.empty((n, dim), dtype=x.dtype)
    if has_sq and sq is None:
        sq = np.empty((n,), dtype=x.dtype)
    rc = L.fn_host_run(op, dim, dcode, x.ctypes.data, n, head.ctypes.data,
                       body.ctypes.data if has_body else None,
                       sq.ctypes.data if has_sq else None, kptr)
    _lib.check(rc, "fn_host_run")
    return BatchOut(head, body if has_body else None, sq if has_sq else None)
