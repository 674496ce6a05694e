"""ctypes binding of the in-tree CUDA library ``libfastnorm_b200.so`` (include/fastnorm_b200.h).

There is no CPU fallback: if the shared library is missing or cannot be loaded, every
kernel entry point raises :class:`CudaLibraryError`.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_1606_06508_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# FASTNORM_B200_LIB points at another build of the library (A/B timing of variants).
LIB_PATH = os.environ.get("FASTNORM_B200_LIB") or os.path.join(HERE, "libfastnorm_b200.so")

# op codes / dtypes (include/fastnorm_b200.h)
OP_SCALE = 0
OP_NORMALIZE = 1
OP_NORM = 2
OP_NAIVE = 3
OP_QUOTIENT = 4
OP_QUOTIENT3_FAST = 5
OP_NORMALIZE_SQ = 6
OP_ROT_UNIT = 7
OP_ROT_GENERAL = 8
OP_NORMALIZE_ROT = 9
OP_ROT_APPLY = 10
OP_QUAT_ROTATE = 11
OP_MAT_APPLY = 12
F32 = 0
F64 = 1

STATUS = {0: "FN_OK", -1: "FN_EINVAL", -2: "FN_ECUDA", -3: "FN_ENODEV", -4: "FN_ENOMEM"}


class CudaLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or a call returned an error."""


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int


def _declare(L: ctypes.CDLL) -> None:
    L.fn_version.restype = ctypes.c_char_p
    L.fn_build_flags.restype = ctypes.c_char_p
    L.fn_backend_name.restype = ctypes.c_char_p
    L.fn_last_error.restype = ctypes.c_char_p
    L.fn_device_count.restype = _int
    L.fn_run.restype = _int
    L.fn_run.argtypes = [_int, _int, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.fn_run_many.restype = _int
    L.fn_run_many.argtypes = [_int, _int, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.fn_run_sharded.restype = _int
    L.fn_run_sharded.argtypes = [_int, _int, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.fn_run_ld.restype = _int
    L.fn_run_ld.argtypes = [_int, _int, _int, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]
    L.fn_host_run_ld.restype = _int
    L.fn_host_run_ld.argtypes = [_int, _int, _int, _vp, _i64, _i64, _vp, _vp, _vp, _vp]
    L.fn_host_run_multi_ld.restype = _int
    L.fn_host_run_multi_ld.argtypes = [_int, _int, _int, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _int]
    L.fn_scalar.restype = _int
    L.fn_scalar.argtypes = [_int, _int, _int, _vp, _vp, _vp]
    L.fn_host_run_multi.restype = _int
    L.fn_host_run_multi.argtypes = [_int, _int, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _int]
    L.fn_run_rot.restype = _int
    L.fn_run_rot.argtypes = [_int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]
    L.fn_host_run.restype = _int
    L.fn_host_run.argtypes = [_int, _int, _int, _vp, _i64, _vp, _vp, _vp, _vp]
    L.fn_generate.restype = _int
    L.fn_generate.argtypes = [_int, ctypes.c_uint64, _i64, _i64, _vp, _vp]
    L.fn_generate_regime.restype = _int
    L.fn_generate_regime.argtypes = [_int, _int, _int, ctypes.c_uint64, _i64, _i64, _vp, _vp]
    L.fn_measure_bounds.restype = _int
    L.fn_measure_bounds.argtypes = [_int, _int, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.fn_selftest_div.restype = _int
    L.fn_selftest_div.argtypes = [_int, ctypes.c_uint64, _i64, _vp, _vp]
    L.fn_host_alloc.restype = _int
    L.fn_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp)]
    L.fn_host_free.restype = _int
    L.fn_host_is_page_locked.restype = _int
    L.fn_host_is_page_locked.argtypes = [_vp]
    L.fn_host_free.argtypes = [_vp]
    L.fn_host_run_soa.restype = _int
    L.fn_host_run_soa.argtypes = [_int, _int, _int, _vp, _i64, _vp, _vp, _vp, _vp]
    L.fn_host_run_soa_multi.restype = _int
    L.fn_host_run_soa_multi.argtypes = [_int, _int, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _int]
    L.fn_launch_count.restype = _i64
    L.fn_launch_count.argtypes = []
    L.fn_small_contexts.restype = _i64
    L.fn_small_contexts.argtypes = []
    L.fn_run_soa.restype = _int
    L.fn_run_soa.argtypes = [_int, _int, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.fn_rotate_rows_f64.restype = _int
    L.fn_rotate_rows_f64.argtypes = [_int, _vp, _vp, _i64, _vp, _vp, _vp, _vp]
    L.fn_host_rotate_rows_f64.restype = _int
    L.fn_host_rotate_rows_f64.argtypes = [_int, _vp, _vp, _i64, _vp, _vp]
    L.fn_rotate_apply_f64.restype = _int
    L.fn_rotate_apply_f64.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.fn_row_stats.restype = _int
    L.fn_row_stats.argtypes = [_int, _int, _vp, _i64, _vp, _vp, _vp]


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raise if it is not there."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaLibraryError(
                    f"{LIB_PATH} is missing: build it with `make -C {os.path.join(HERE, 'csrc')}` "
                    "(there is no CPU fallback)")
            try:
                L = ctypes.CDLL(LIB_PATH)
            except OSError as e:  # pragma: no cover - depends on the box
                raise CudaLibraryError(f"cannot load {LIB_PATH}: {e}") from e
            _declare(L)
            _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().fn_last_error().decode(errors="replace")
        exc = ValueError if rc == -1 else CudaLibraryError
        raise exc(f"{what}: {STATUS.get(rc, rc)}: {msg}")


def version() -> str:
    return lib().fn_version().decode()


def build_flags() -> str:
    return lib().fn_build_flags().decode()


def device_count() -> int:
    return int(lib().fn_device_count())
