"""Kernel registry (reference: _backend.py, tests/test_backends.py:145-166)."""

import pytest

from paper_1606_06508_b200 import _backend, _cuda_kernels


def test_registry_has_cuda_backend():
    assert _backend.available_backends() == ("cuda",)
    assert _backend.backend_name() == "cuda"
    assert _backend.get_module() is _cuda_kernels
    assert _cuda_kernels.BACKEND_NAME == "cuda"
    assert "sm_100a" in _cuda_kernels.BUILD_FLAGS


def test_every_reference_name_resolves():
    for prec in ("single", "double"):
        for dim in (2, 3, 4):
            for fam in ("scale", "normalize", "norm", "naive", "quotient"):
                assert callable(_backend.scalar_kernel(f"{fam}{dim}", prec))
                assert callable(_backend.batch_kernel(f"{fam}{dim}", prec))
            assert callable(_backend.batch_kernel(f"normalize{dim}_sq", prec))
            assert callable(_backend.loop_kernel(f"loop_empty{dim}", prec))
        assert callable(_backend.scalar_kernel("quotient3_fast", prec))
        for algo in _backend.ALGORITHMS:
            for dim in _backend.algorithm_dims(algo):
                assert callable(_backend.loop_kernel(_backend.loop_base(algo, dim), prec))
                assert callable(_backend.scalar_kernel(_backend.scalar_base(algo, dim), prec))


def test_override_context():
    original = _backend.backend_name()
    with _backend.override("cuda"):
        assert _backend.backend_name() == "cuda"
    assert _backend.backend_name() == original
    with pytest.raises(ValueError):
        with _backend.override("fortran"):
            pass


def test_register_extra_backend():
    class Fake:
        def normalize3_f64(self, *a):
            return "fake"

    _backend.register("fake", Fake())
    try:
        with _backend.override("fake"):
            assert _backend.scalar_kernel("normalize3", "double")() == "fake"
            with pytest.raises(ValueError):
                _backend.batch_kernel("normalize3", "double")
    finally:
        del _backend._MODULES["fake"]


def test_unknown_names_rejected():
    with pytest.raises(ValueError):
        _backend.scalar_base("quotient_fast", 2)
    with pytest.raises(ValueError):
        _backend.loop_base("simd", 3)
    with pytest.raises(ValueError):
        _backend.scalar_base("simd", 3)
    with pytest.raises(AttributeError):
        _backend.batch_kernel("normalize5", "double")
    assert _backend.takes_params("scaling") and not _backend.takes_params("quotient")
    assert _backend.scalar_base("scaling", 4) == "normalize4"
    assert _backend.loop_base("quotient_fast", 3) == "loop_quotient_fast3"


def test_parse_base():
    from paper_1606_06508_b200 import _lib

    assert _cuda_kernels.parse_base("normalize3") == (_lib.OP_NORMALIZE, 3)
    assert _cuda_kernels.parse_base("normalize4_sq") == (_lib.OP_NORMALIZE_SQ, 4)
    assert _cuda_kernels.parse_base("quotient3_fast") == (_lib.OP_QUOTIENT3_FAST, 3)
    assert _cuda_kernels.parse_base("norm2") == (_lib.OP_NORM, 2)


def test_batch_dtype_mismatch_raises_before_launch():
    import numpy as np

    import paper_1606_06508_b200 as fn

    with pytest.raises(TypeError):
        fn.normalize3(fn.preset("single"), np.zeros((4, 3)))
    with pytest.raises(ValueError):
        fn.normalize3(fn.preset("double"), np.zeros((4, 2)))
    with pytest.raises(TypeError):
        fn.quotient2(np.zeros((4, 2), dtype=np.float32), precision="double")
    with pytest.raises(TypeError):
        fn.normalize3(fn.preset("double"), 1.0, 2.0)
