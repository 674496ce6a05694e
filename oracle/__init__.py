"""Parity oracle for the B200 library -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference``) may import this package.  The product package
``paper_1606_06508_b200`` never imports it and has no CPU fallback.

Two checkers live here:

* ``liboracle.so`` -- the repo's plain-C restatement of the reference kernels
  (``fastnorm_oracle.c``; each routine cites ``pkg/src/fastnorm/_kernels.pyx``), batched
  over AoS rows.  It is pinned against golden vectors made by the reference itself
  (``tests/golden/``) and, where ``_ref`` is built, against the live reference.
* ``_ref/_kernels*.so`` -- the reference's own Cython module compiled from the
  read-only sources by ``oracle/Makefile`` (target ``ref``).  Loaded by file path so the
  reference package's ``__init__`` (which needs gmpy2, absent here) is never run.
"""

from __future__ import annotations

import ctypes
import importlib.machinery
import importlib.util
import os
import subprocess
import sysconfig
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "liboracle.so")
_REF_DIR = os.path.join(HERE, "_ref")

# op codes (mirror include/fastnorm_b200.h)
OP_SCALE, OP_NORMALIZE, OP_NORM, OP_NAIVE, OP_QUOTIENT, OP_QUOTIENT3_FAST, OP_NORMALIZE_SQ = range(7)
# loop algorithms
ALGO_SCALING, ALGO_QUOTIENT, ALGO_QUOTIENT_FAST, ALGO_NAIVE, ALGO_EMPTY = range(5)

BASE_OPS = {
    "scale": OP_SCALE,
    "normalize": OP_NORMALIZE,
    "normalize_sq": OP_NORMALIZE_SQ,
    "norm": OP_NORM,
    "naive": OP_NAIVE,
    "quotient": OP_QUOTIENT,
    "quotient3_fast": OP_QUOTIENT3_FAST,
}

_lock = threading.Lock()
_lib = None


def build() -> str:
    """Compile liboracle.so (and, when /root/reference is present, the reference)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def build_ref() -> str | None:
    """Compile the reference's own kernels into oracle/_ref (needs /root/reference)."""
    if not os.path.exists("/root/reference/pkg/src/fastnorm/_kernels.pyx"):
        return None
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return _REF_DIR


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            L = ctypes.CDLL(_LIB_PATH)
            L.orc_run.restype = ctypes.c_int
            L.orc_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p]
            L.orc_rotation.restype = ctypes.c_int64
            L.orc_rotation.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]
            L.orc_rotate_apply.restype = None
            L.orc_rotate_apply.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_void_p]
            L.orc_rotate_rows.restype = ctypes.c_int64
            L.orc_rotate_rows.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p]
            L.orc_loop.restype = ctypes.c_double
            L.orc_loop.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
            _lib = L
    return _lib


def _ka_ptr(ka):
    if ka is None:
        return None, None
    arr = np.ascontiguousarray(np.asarray(ka, dtype=np.float64))
    assert arr.shape == (6,)
    return arr, arr.ctypes.data


def run(op: int, x: np.ndarray, ka=None, threads: int = 1):
    """Oracle outputs (head, body, sq) for AoS rows x[N, dim] (float32 or float64)."""
    x = np.ascontiguousarray(x)
    if x.dtype not in (np.float32, np.float64) or x.ndim != 2:
        raise TypeError("x must be a 2-D float32/float64 array")
    n, dim = x.shape
    head = np.empty(n, dtype=x.dtype)
    body = None if op == OP_NORM else np.empty((n, dim), dtype=x.dtype)
    sq = np.empty(n, dtype=x.dtype) if op == OP_NORMALIZE_SQ else None
    karr, kptr = _ka_ptr(ka)
    dt = 1 if x.dtype == np.float64 else 0
    L = lib()

    def part(lo, hi):
        if hi <= lo:
            return
        w = x.itemsize
        rc = L.orc_run(op, dim, dt, x.ctypes.data + lo * dim * w, hi - lo,
                       head.ctypes.data + lo * w,
                       None if body is None else body.ctypes.data + lo * dim * w,
                       None if sq is None else sq.ctypes.data + lo * w, kptr)
        if rc != 0:
            raise ValueError(f"oracle rejected op={op} dim={dim}")

    if threads <= 1 or n < 65536:
        part(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        ts = [threading.Thread(target=part, args=(int(bounds[i]), int(bounds[i + 1])))
              for i in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    return head, body, sq


OP_ROT_UNIT, OP_ROT_GENERAL, OP_NORMALIZE_ROT = 7, 8, 9


def rotation(op: int, q: np.ndarray, ka=None):
    """Oracle rotations of float64 quaternions q[N, 4] (rotation.py:53-111).

    Returns (R[N,3,3], invalid_count) for OP_ROT_UNIT / OP_ROT_GENERAL and
    (r[N], unit[N,4], R[N,3,3], invalid_count) for OP_NORMALIZE_ROT."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    n = q.shape[0]
    karr, kptr = _ka_ptr(ka)
    if op == OP_NORMALIZE_ROT:
        r = np.empty(n)
        u = np.empty((n, 4))
        R = np.empty((n, 3, 3))
        bad = lib().orc_rotation(op, q.ctypes.data, n, r.ctypes.data, u.ctypes.data, R.ctypes.data, kptr)
        return r, u, R, int(bad)
    R = np.empty((n, 3, 3))
    bad = lib().orc_rotation(op, q.ctypes.data, n, R.ctypes.data, None, None, kptr)
    return R, int(bad)


OP_ROT_APPLY = 10


def rotate_apply(R, v: np.ndarray) -> np.ndarray:
    """Oracle RotationMatrix.apply (rotation.py:39-41) of one matrix R (9 entries,
    row-major) over float64 vectors v[N, 3]."""
    Rm = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty_like(v)
    lib().orc_rotate_apply(Rm.ctypes.data, v.ctypes.data, v.shape[0], out.ctypes.data)
    return out


OP_QUAT_ROTATE, OP_MAT_APPLY = 11, 12


def rotate_rows(op: int, a: np.ndarray, v: np.ndarray, ka=None):
    """Oracle per-row rotation: op 11 (q[N,4] normalised, rotation_unit, applied to
    v[N,3]) or op 12 (R[N,3,3] applied to v[N,3]).  Returns (out[N,3], invalid rows)."""
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(len(v), -1)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty_like(v)
    karr, kptr = _ka_ptr(ka)
    bad = lib().orc_rotate_rows(op, a.ctypes.data, v.ctypes.data, v.shape[0], out.ctypes.data, kptr)
    return out, int(bad)


def loop(algo: int, buf: np.ndarray, iters: int, mask: int, ka=None) -> float:
    """The reference timing-loop checksum over AoS rows buf[M, dim]."""
    buf = np.ascontiguousarray(buf)
    dim = buf.shape[1]
    karr, kptr = _ka_ptr(ka)
    dt = 1 if buf.dtype == np.float64 else 0
    return lib().orc_loop(algo, dim, dt, buf.ctypes.data, iters, mask, kptr)


_ref_mod = None


def ref_module():
    """The reference's compiled Cython kernels (oracle/_ref), or None if not built."""
    global _ref_mod
    if _ref_mod is not None:
        return _ref_mod
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    path = os.path.join(_REF_DIR, "_kernels" + suffix)
    if not os.path.exists(path):
        return None
    loader = importlib.machinery.ExtensionFileLoader("_kernels", path)
    spec = importlib.util.spec_from_file_location("_kernels", path, loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    _ref_mod = mod
    return mod


def same(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Element-wise parity predicate of the reference tests (test_backends.py:33-38):
    NaN matches NaN; otherwise bit-equal (which also compares the sign of zero)."""
    a = np.asarray(a)
    b = np.asarray(b)
    ia = a.view(np.uint64 if a.dtype == np.float64 else np.uint32)
    ib = b.view(np.uint64 if b.dtype == np.float64 else np.uint32)
    return (ia == ib) | (np.isnan(a) & np.isnan(b))
