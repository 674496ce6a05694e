"""Drop-in check against the reference's OWN registry and wrappers (container only).

Loads the reference's _backend.py, params.py, scale.py, normalize.py and baselines.py by
path under a shim package (its __init__ needs gmpy2, absent here), registers this
repo's "cuda" module into the reference's _MODULES exactly as INTEGRATION.md describes,
and checks that every name the reference's wrappers, bench harness and tests resolve is
provided with the reference's signature.  No GPU needed: names and arities only.
Skipped where /root/reference is absent (e.g. on the GPU box).
"""

import importlib.util
import inspect
import os
import sys
import types

import pytest

REF = "/root/reference/pkg/src/fastnorm"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")


@pytest.fixture(scope="module")
def ref_pkg():
    saved = {k: v for k, v in sys.modules.items() if k == "fastnorm" or k.startswith("fastnorm.")}
    pkg = types.ModuleType("fastnorm")
    pkg.__path__ = [REF]
    sys.modules["fastnorm"] = pkg
    # the reference's own pure-Python twin stands in for its compiled module
    mods = {}
    try:
        for name in ("_pykernels", "params", "_backend", "scale", "normalize", "baselines"):
            spec = importlib.util.spec_from_file_location(f"fastnorm.{name}", os.path.join(REF, f"{name}.py"))
            mod = importlib.util.module_from_spec(spec)
            sys.modules[f"fastnorm.{name}"] = mod
            spec.loader.exec_module(mod)
            setattr(pkg, name, mod)
            mods[name] = mod
        yield mods
    finally:
        for k in list(sys.modules):
            if k == "fastnorm" or k.startswith("fastnorm."):
                del sys.modules[k]
        sys.modules.update(saved)


def test_cuda_module_registers_into_reference_registry(ref_pkg):
    from paper_1606_06508_b200 import _cuda_kernels

    backend = ref_pkg["_backend"]
    backend._MODULES["cuda"] = _cuda_kernels  # the maintainer's patch
    assert "cuda" in backend.available_backends()
    py = backend.get_module("python")
    for prec in ("single", "double"):
        for algo in backend.ALGORITHMS:
            for dim in backend.algorithm_dims(algo):
                for base, resolve in ((backend.scalar_base(algo, dim), backend.scalar_kernel),
                                      (backend.loop_base(algo, dim), backend.loop_kernel)):
                    ours = resolve(base, prec, backend="cuda")
                    theirs = resolve(base, prec, backend="python")
                    assert callable(ours)
                    # same parameter names and order as the reference twin
                    p_ref = list(inspect.signature(theirs).parameters)
                    p_our = list(inspect.signature(ours).parameters)
                    assert p_our == p_ref, (base, prec, p_our, p_ref)
        for dim in (2, 3, 4):
            for fam in ("scale", "norm"):
                assert callable(backend.scalar_kernel(f"{fam}{dim}", prec, backend="cuda"))
            assert callable(backend.loop_kernel(f"loop_empty{dim}", prec, backend="cuda"))
    assert isinstance(_cuda_kernels.BACKEND_NAME, str) and _cuda_kernels.BUILD_FLAGS
    with backend.override("cuda"):
        assert backend.backend_name() == "cuda"


def test_reference_kernel_args_feed_our_abi(ref_pkg):
    """kernel_args of the reference (scale.py:26-30) == ours, for both presets."""
    import paper_1606_06508_b200 as fn

    for fmt in ("single", "double"):
        assert ref_pkg["scale"].kernel_args(ref_pkg["params"].preset(fmt)) == fn.kernel_args(fn.preset(fmt))


_WRAPPERS = {
    "normalize": ("normalize2", "normalize3", "normalize4", "norm2", "norm3", "norm4"),
    "scale": ("scale2", "scale3", "scale4"),
    "baselines": ("naive_normalize2", "naive_normalize3", "naive_normalize4", "quotient2",
                  "quotient3_robust", "quotient3_fast", "quotient4"),
}


def test_public_wrapper_signatures_match_reference(ref_pkg):
    """Every public scalar wrapper keeps the reference's parameters exactly: names, kinds,
    order, annotations and defaults (normalize.py:51-89, scale.py:33-51,
    baselines.py:30-76), and the same return annotation.  The only additions are the
    ROWS default on x2..xn (leaving them out is the [N, n] overload) and keyword-only
    ``out``."""
    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200.batch import ROWS

    for mod, names in _WRAPPERS.items():
        for name in names:
            ref = inspect.signature(getattr(ref_pkg[mod], name))
            ours = inspect.signature(getattr(fn, name))
            assert ours.return_annotation == ref.return_annotation, name
            rp, op = list(ref.parameters.values()), list(ours.parameters.values())
            assert [q.name for q in op[: len(rp)]] == [q.name for q in rp], name
            for r, o in zip(rp, op):
                assert o.kind == r.kind and o.annotation == r.annotation, (name, r, o)
                if r.default is inspect.Parameter.empty:
                    # x1 (and p) stay required; x2..xn gain only the ROWS marker
                    assert o.default is inspect.Parameter.empty or (o.default is ROWS and r.name not in ("p", "x1")), (name, o)
                else:
                    assert o.default == r.default and type(o.default).__mro__[-2] is type(r.default), (name, o)
            extra = op[len(rp):]
            assert [(q.name, q.kind, q.default) for q in extra] == [("out", inspect.Parameter.KEYWORD_ONLY, None)], name


def test_public_wrappers_accept_reference_keyword_calls():
    """Keyword calls written against the reference work unchanged (the GPU computes them;
    here only the argument binding is checked)."""
    import paper_1606_06508_b200 as fn

    p = fn.preset("double")
    inspect.signature(fn.normalize3).bind(p, x1=3.0, x2=4.0, x3=12.0)
    inspect.signature(fn.quotient3_robust).bind(x1=1.0, x2=2.0, x3=3.0, precision="single")
    inspect.signature(fn.scale4).bind(p, 1.0, 2.0, x3=3.0, x4=4.0)
    inspect.signature(fn.naive_normalize2).bind(1.0, 2.0, "single")
