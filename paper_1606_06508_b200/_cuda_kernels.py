"""The "cuda" backend module of the kernel registry.

It exports exactly the flat names the reference's registry resolves
(``getattr(module, f"{base}_{suffix}")``, _backend.py:86-93) with the reference's scalar
signatures (_kernels.pyx:419-634) and timing-loop signatures (:792-1008), plus
``BACKEND_NAME`` / ``BUILD_FLAGS`` (tests/test_backends.py:145-149).  Every one of them
computes on the GPU through the C ABI:

* scalar ``{base}_{f32,f64}(...)`` -- one row through ``fn_scalar`` (one kernel launch
  on a mapped page-locked row per call: correct and drop-in, but use the batched
  overloads for throughput);
* ``loop_*`` -- the rows the loop touches are normalised on the GPU in one launch and
  the checksum is accumulated on the host in the reference loop's exact order
  (``acc += <double>r + <double>u1 + ...``, _kernels.pyx:652-657), so it equals the
  reference's checksum bit for bit;
* ``batch_kernel(base, suffix)`` -- the batched entry used by the public API.
"""

from __future__ import annotations

import ctypes
import functools
import inspect
import threading

import numpy as np

from paper_1606_06508_b200 import _lib, batch

BACKEND_NAME = "cuda"

_OPS = {
    "scale": _lib.OP_SCALE,
    "normalize": _lib.OP_NORMALIZE,
    "normalize_sq": _lib.OP_NORMALIZE_SQ,
    "norm": _lib.OP_NORM,
    "naive": _lib.OP_NAIVE,
    "quotient": _lib.OP_QUOTIENT,
}
_SCALING = ("scale", "normalize", "normalize_sq", "norm")


def __getattr__(name: str):
    if name == "BUILD_FLAGS":
        return _lib.build_flags()
    raise AttributeError(name)


def parse_base(base: str) -> tuple[int, int]:
    """'normalize3' -> (OP_NORMALIZE, 3); 'quotient3_fast' -> (OP_QUOTIENT3_FAST, 3)."""
    if base == "quotient3_fast":
        return _lib.OP_QUOTIENT3_FAST, 3
    if base.endswith("_sq") and base[:-3].startswith("normalize"):
        fam, dim = "normalize_sq", base[len("normalize"):-3]
    else:
        fam, dim = base[:-1], base[-1:]
    if fam not in _OPS or dim not in ("2", "3", "4"):
        raise AttributeError(f"no kernel family {base!r}")
    return _OPS[fam], int(dim)


def _np_dtype(suffix: str):
    return np.float64 if suffix == "f64" else np.float32


def _ka_array(ka) -> np.ndarray:
    if type(ka) is np.ndarray and ka.dtype == np.float64 and ka.shape == (6,) and ka.flags.c_contiguous:
        return ka  # already the ABI's six doubles (kernel_args_array's cached arrays)
    arr = np.ascontiguousarray(np.asarray(ka, dtype=np.float64))
    if arr.shape != (6,):
        raise ValueError("kernel_args must be six numbers")
    return arr


@functools.lru_cache(maxsize=None)
def batch_kernel(base: str, suffix: str):
    """Batched callable ``f(x[N, n], ka_or_None, out=None) -> BatchOut``."""
    op, dim = parse_base(base)
    takes_ka = op in (_lib.OP_SCALE, _lib.OP_NORMALIZE, _lib.OP_NORMALIZE_SQ, _lib.OP_NORM)
    want = "float64" if suffix == "f64" else "float32"
    prec = "double" if suffix == "f64" else "single"

    def run(x, ka=None, out=None):
        if batch.precision_of(x) != prec:
            raise TypeError(f"{base}_{suffix} computes in {want}; rows are {str(x.dtype).replace('torch.', '')}")
        return batch.run(op, dim, x, _ka_array(ka) if takes_ka else None, out)

    run.__name__ = f"{base}_{suffix}_batch"
    return run


_tls = threading.local()


def _scalar_state():
    """Per-thread argument buffers for fn_scalar and their addresses."""
    st = getattr(_tls, "state", None)
    if st is None:
        xb, ob, kb = (ctypes.c_double * 8)(), (ctypes.c_double * 16)(), (ctypes.c_double * 6)()
        st = _tls.state = (xb, ob, kb, ctypes.addressof(xb), ctypes.addressof(ob), ctypes.addressof(kb))
    return st


_ext_state: list = []


def _scalar_entry():
    """The CPython fast path (csrc/scalar_ext.c) bound to the loaded library's
    fn_scalar, or None when that module was not built (the ctypes call is used then;
    both launch the same kernel)."""
    if not _ext_state:
        try:
            from paper_1606_06508_b200 import _scalar
        except ImportError:
            _ext_state.append(None)
        else:
            _scalar.bind(ctypes.cast(_lib.lib().fn_scalar, ctypes.c_void_p).value)
            _ext_state.append(_scalar.scalar)
    return _ext_state[0]


def _make_scalar(base: str, suffix: str):
    """Reference scalar signature -> fn_scalar (one launch; the row rides in the kernel
    parameters, the results come back through mapped page-locked memory)."""
    op, dim = parse_base(base)
    takes_ka = op in (_lib.OP_SCALE, _lib.OP_NORMALIZE, _lib.OP_NORMALIZE_SQ, _lib.OP_NORM)
    dcode = _lib.F64 if suffix == "f64" else _lib.F32
    nargs = dim + (6 if takes_ka else 0)
    nout = sum(batch.widths(op, dim))
    sq_first = op == _lib.OP_NORMALIZE_SQ
    name = f"{base}_{suffix}"

    def kernel(*args):
        if len(args) != nargs:
            raise TypeError(f"{name} takes {nargs} arguments ({len(args)} given)")
        fast = _scalar_entry()
        if fast is not None:
            res = fast(op, dim, dcode, nout, sq_first, args)
            if type(res) is int:
                _lib.check(res, name)
            return res
        xb, ob, kb, xa, oa, kaddr = _scalar_state()
        if takes_ka:
            kb[:] = args[:6]
            xb[:dim] = args[6:]
        else:
            xb[:dim] = args
        rc = _lib.lib().fn_scalar(op, dim, dcode, xa, oa, kaddr if takes_ka else None)
        if rc:
            _lib.check(rc, name)
        if nout == 1:
            return ob[0]
        vals = ob[:nout]
        return tuple([vals[-1]] + vals[:-1]) if sq_first else tuple(vals)

    kernel.__name__ = f"{base}_{suffix}"
    names = (["tau_min", "tau_max", "sigma_min", "sigma_max", "inv_min", "inv_max"] if takes_ka else []) + \
        [f"x{k + 1}" for k in range(dim)]
    kernel.__signature__ = inspect.Signature(
        [inspect.Parameter(nm, inspect.Parameter.POSITIONAL_OR_KEYWORD) for nm in names])
    return kernel


def _loop_terms(op: int, dim: int, dt, buf, rows: int, ka) -> np.ndarray:
    flat = np.asarray(buf, dtype=dt).reshape(-1)
    x = np.ascontiguousarray(flat[: rows * dim].reshape(rows, dim))
    res = batch.run(op, dim, x, ka)
    term = res.head.astype(np.float64)
    with np.errstate(invalid="ignore", over="ignore"):  # inf + -inf -> NaN, as in the C loop
        for k in range(dim):  # ((r + u1) + u2) + ... in double, left to right
            term = term + res.body[:, k].astype(np.float64)
    return term


def _ordered_sum(terms: np.ndarray, iters: int, mask: int) -> float:
    """acc = 0.0; for i < iters: acc += terms[i & mask]  -- strictly sequential."""
    acc = 0.0
    step = 1 << 22
    for lo in range(0, iters, step):
        idx = np.arange(lo, min(iters, lo + step), dtype=np.int64) & mask
        seq = np.concatenate(([acc], terms[idx]))
        acc = float(np.add.accumulate(seq)[-1])
    return acc


def _make_loop(algo: str, dim: int, suffix: str):
    dt = _np_dtype(suffix)
    if algo == "scaling":
        op = _lib.OP_NORMALIZE
    elif algo == "quotient_fast":
        op = _lib.OP_QUOTIENT3_FAST
    else:
        op = _OPS[algo]

    def loop(buf, iters, mask, p0=0.0, p1=0.0, p2=0.0, p3=0.0, p4=0.0, p5=0.0):
        rows = min(int(iters), int(mask) + 1)
        if rows <= 0:
            return 0.0
        ka = _ka_array((p0, p1, p2, p3, p4, p5)) if algo == "scaling" else None
        terms = _loop_terms(op, dim, dt, buf, rows, ka)
        return _ordered_sum(terms, int(iters), int(mask))

    return loop


def _make_empty_loop(dim: int, suffix: str):
    dt = _np_dtype(suffix)

    def loop(buf, iters, mask):
        rows = min(int(iters), int(mask) + 1)
        if rows <= 0:
            return 0.0
        x = np.asarray(buf, dtype=dt).reshape(-1)[: rows * dim].reshape(rows, dim).astype(np.float64)
        term = x[:, 0].copy()
        for k in range(1, dim):
            term = term + x[:, k]
        return _ordered_sum(term, int(iters), int(mask))

    return loop


def _export():
    g = globals()
    for suffix in ("f32", "f64"):
        for dim in (2, 3, 4):
            for fam in ("scale", "normalize", "norm", "naive", "quotient"):
                g[f"{fam}{dim}_{suffix}"] = _make_scalar(f"{fam}{dim}", suffix)
            g[f"normalize{dim}_sq_{suffix}"] = _make_scalar(f"normalize{dim}_sq", suffix)
            for algo in ("scaling", "quotient", "naive"):
                g[f"loop_{algo}{dim}_{suffix}"] = _make_loop(algo, dim, suffix)
            g[f"loop_empty{dim}_{suffix}"] = _make_empty_loop(dim, suffix)
        g[f"quotient3_fast_{suffix}"] = _make_scalar("quotient3_fast", suffix)
        g[f"loop_quotient_fast3_{suffix}"] = _make_loop("quotient_fast", 3, suffix)


_export()
