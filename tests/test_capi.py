"""The C-ABI library loads and exports every entry point include/fastnorm_b200.h declares;
argument errors are reported without touching a GPU (no compute calls here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1606_06508_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "fastnorm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fn_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_full_registry():
    names = set(declared_symbols())
    for prec in ("f32", "f64"):
        for dim in (2, 3, 4):
            for fam in ("scale", "normalize", "norm", "naive", "quotient"):
                assert f"fn_{fam}{dim}_{prec}" in names
            assert f"fn_normalize{dim}_sq_{prec}" in names
        assert f"fn_quotient3_fast_{prec}" in names
    for extra in ("fn_run", "fn_host_run", "fn_generate", "fn_row_stats", "fn_last_error",
                  "fn_version", "fn_build_flags", "fn_backend_name", "fn_device_count"):
        assert extra in names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_metadata():
    L = _lib.lib()
    assert L.fn_backend_name() == b"cuda"
    assert b"sm_100a" in L.fn_version()
    flags = _lib.build_flags()
    assert "compute_100a" in flags and "-fmad=false" in flags and "-ftz=false" in flags


def test_argument_errors_without_gpu():
    L = _lib.lib()
    x = np.zeros((4, 3))
    h = np.zeros(4)
    b = np.zeros((4, 3))
    ka = np.array([2.0 ** -482, 2.0 ** 510, 2.0 ** 592, 2.0 ** -514, 2.0 ** -592, 2.0 ** 514])
    vp = ctypes.c_void_p
    # unknown op / dim / dtype / negative n / NULL outputs -> FN_EINVAL
    assert L.fn_run(99, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    assert L.fn_run(1, 5, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    assert L.fn_run(1, 3, 7, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    assert L.fn_run(1, 3, 1, x.ctypes.data, -1, h.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    assert L.fn_run(1, 3, 1, x.ctypes.data, 4, h.ctypes.data, None, None, ka.ctypes.data, None) == -1
    assert b"body" in L.fn_last_error()
    # norm has no body output; quotient3_fast is 3-D only; normalize_sq needs sq
    assert L.fn_run(2, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    assert L.fn_run(5, 2, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, None, None) == -1
    assert L.fn_run(6, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    # scaling kernels need ka; negative / NaN tau is rejected (bit-pattern band test)
    assert L.fn_run(1, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, None, None) == -1
    bad = ka.copy()
    bad[0] = -1.0
    assert L.fn_run(1, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, bad.ctypes.data, None) == -1
    bad[0] = np.nan
    assert L.fn_run(1, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None, bad.ctypes.data, None) == -1
    assert b"tau" in L.fn_last_error()
    # FN_OP_ROT_APPLY: float64 3-vectors only, and ka carries the matrix
    assert L.fn_run(10, 4, 1, x.ctypes.data, 4, h.ctypes.data, None, None, ka.ctypes.data, None) == -1
    assert L.fn_run(10, 3, 0, x.ctypes.data, 4, h.ctypes.data, None, None, ka.ctypes.data, None) == -1
    assert L.fn_run(10, 3, 1, x.ctypes.data, 4, b.ctypes.data, b.ctypes.data, None, ka.ctypes.data, None) == -1
    assert L.fn_rotate_apply_f64(None, x.ctypes.data, 4, b.ctypes.data, None) == -1
    assert b"matrix" in L.fn_last_error()
    # two-input rotations: op, n and pointers are checked before any device work
    assert L.fn_rotate_rows_f64(1, x.ctypes.data, x.ctypes.data, 4, b.ctypes.data, ka.ctypes.data, None, None) == -1
    assert L.fn_rotate_rows_f64(11, x.ctypes.data, x.ctypes.data, -1, b.ctypes.data, ka.ctypes.data, None, None) == -1
    assert L.fn_rotate_rows_f64(12, None, x.ctypes.data, 4, b.ctypes.data, None, None, None) == -1
    assert L.fn_rotate_rows_f64(11, vp(0), vp(0), 0, vp(0), None, None, None) == 0
    assert L.fn_host_rotate_rows_f64(13, x.ctypes.data, x.ctypes.data, 4, b.ctypes.data, None) == -1
    assert L.fn_host_rotate_rows_f64(12, x.ctypes.data, x.ctypes.data, 4, None, None) == -1
    # structure-of-arrays entry: op range, dim, NULL component / output arrays
    xs = (ctypes.c_void_p * 3)(x.ctypes.data, x.ctypes.data, x.ctypes.data)
    bs = (ctypes.c_void_p * 3)(b.ctypes.data, b.ctypes.data, b.ctypes.data)
    assert L.fn_run_soa(7, 3, 1, ctypes.addressof(xs), 4, h.ctypes.data, ctypes.addressof(bs), None, ka.ctypes.data, None) == -1
    assert L.fn_run_soa(1, 5, 1, ctypes.addressof(xs), 4, h.ctypes.data, ctypes.addressof(bs), None, ka.ctypes.data, None) == -1
    assert L.fn_run_soa(1, 3, 1, ctypes.addressof(xs), 4, h.ctypes.data, None, None, ka.ctypes.data, None) == -1
    assert L.fn_run_soa(2, 3, 1, ctypes.addressof(xs), 4, h.ctypes.data, ctypes.addressof(bs), None, ka.ctypes.data, None) == -1
    assert L.fn_run_soa(1, 3, 1, None, 0, None, None, None, ka.ctypes.data, None) == 0
    # n == 0 is a no-op success
    assert L.fn_run(1, 3, 1, vp(0), 0, vp(0), vp(0), None, ka.ctypes.data, None) == 0
    assert L.fn_host_run(1, 3, 1, vp(0), 0, vp(0), vp(0), None, ka.ctypes.data) == 0
    assert L.fn_generate(9, 0, 0, 4, x.ctypes.data, None) == -1
    assert L.fn_row_stats(3, 1, x.ctypes.data, 4, None, ka.ctypes.data, None) == -1


def test_named_entry_points_validate_like_fn_run():
    L = _lib.lib()
    f = L.fn_normalize3_f64
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_void_p]
    x = np.zeros((4, 3))
    assert f(x.ctypes.data, 4, None, None, None, None) == -1  # NULL outputs
    g = L.fn_norm4_f32
    g.restype = ctypes.c_int
    g.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    assert g(x.ctypes.data, 0, None, None, None) == 0  # empty batch


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product raises instead of computing on the CPU."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1606_06508_b200 as fn

    with pytest.raises(_lib.CudaLibraryError):
        fn.normalize3(fn.preset("double"), np.ones((8, 3)))
    with pytest.raises(_lib.CudaLibraryError):
        fn.normalize3(fn.preset("double"), 3.0, 4.0, 12.0)


def test_host_run_multi_argument_errors():
    L = _lib.lib()
    x = np.zeros((4, 3))
    h = np.zeros(4)
    b = np.zeros((4, 3))
    ka = np.array([2.0 ** -482, 2.0 ** 510, 2.0 ** 592, 2.0 ** -514, 2.0 ** -592, 2.0 ** 514])
    devs = np.array([0], dtype=np.int32)
    assert L.fn_host_run_multi(1, 3, 1, x.ctypes.data, 4, h.ctypes.data, b.ctypes.data, None,
                               ka.ctypes.data, None, 0) == -1
    assert L.fn_host_run_multi(1, 3, 1, x.ctypes.data, 0, h.ctypes.data, b.ctypes.data, None,
                               ka.ctypes.data, devs.ctypes.data, 1) == 0


def test_c_example_builds():
    """A plain C program compiles and links against the C ABI (examples/normalize_host.c)."""
    import subprocess

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-s", "-B", "-C", os.path.join(repo, "examples")], check=True)
    assert os.path.exists(os.path.join(repo, "examples", "normalize_host"))


@pytest.mark.gpu
def test_c_example_runs():
    import subprocess

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-s", "-C", os.path.join(repo, "examples")], check=True)
    out = subprocess.run([os.path.join(repo, "examples", "normalize_host"), "1000000"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "r = " in out.stdout and "identical to the dense call" in out.stdout


def test_scalar_extension_binds_fn_scalar():
    """The CPython fast path for the scalar signatures is built in-tree and binds the
    loaded library's fn_scalar; without a GPU its calls fail loudly like the ABI."""
    from paper_1606_06508_b200 import _cuda_kernels, _scalar

    assert _cuda_kernels._scalar_entry() is _scalar.scalar
    if _lib.device_count() == 0:
        with pytest.raises(_lib.CudaLibraryError):
            _cuda_kernels.normalize3_f64(*[1.0] * 6, 3.0, 4.0, 12.0)
    with pytest.raises(TypeError):
        _scalar.scalar(1, 3, 1, 4, False, [3.0, 4.0, 12.0])


def test_host_alloc_without_gpu_fails_loudly():
    import paper_1606_06508_b200 as fn

    ptr = ctypes.c_void_p(1)
    L = _lib.lib()
    assert L.fn_host_alloc(0, ctypes.byref(ptr)) == 0 and not ptr.value
    assert L.fn_host_free(None) == 0
    assert fn.host_empty((0, 3)).shape == (0, 3)
    if _lib.device_count() == 0:
        with pytest.raises(_lib.CudaLibraryError):
            fn.host_empty((16, 3))
