"""The north star's integer exponent insertion (FNB_EXPONENT_INSERTION=1,
fastnorm_math.cuh: sigma * x_k as an integer add on the exponent field wherever x_k and
the product are normal, the IEEE multiply elsewhere) is a second build of the library,
libfastnorm_b200_insert.so.  The default build multiplies by the exact power of two
(measured faster on B200).  This runs the golden-vector and random
full-range parity of tests/test_gpu_parity.py and the full-size BASELINE configs 2, 4
and 5 of tests/test_gpu_configs.py against the insertion build, in a subprocess that
loads it through FASTNORM_B200_LIB."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB = os.path.join(REPO, "paper_1606_06508_b200", "libfastnorm_b200_insert.so")


def _env():
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} is missing (make -C paper_1606_06508_b200/csrc builds it)")
    return dict(os.environ, FASTNORM_B200_LIB=LIB)


def test_insertion_build_is_the_one_loaded():
    code = ("import paper_1606_06508_b200 as fn\nfrom paper_1606_06508_b200 import _lib\n"
            "print(_lib.LIB_PATH); print(_lib.build_flags())\n"
            "p = fn.preset('double'); print(fn.normalize3(p, 3.0, 4.0, 12.0).length)\n")
    out = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.split("\n")
    assert lines[0].endswith("libfastnorm_b200_insert.so")
    assert "FNB_EXPONENT_INSERTION=1" in lines[1]
    assert lines[2] == "13.0"


@pytest.mark.parametrize("select", [
    ("tests/test_gpu_parity.py", "golden or random_full_range or tail_sizes or reference_regimes or custom_parameter"),
    ("tests/test_gpu_configs.py", "cfg2 or cfg4 or cfg5"),
])
def test_parity_suite_on_insertion_build(select):
    path, expr = select
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", path, "-k", expr],
                         env=_env(), cwd=REPO, capture_output=True, text=True, timeout=2400)
    tail = out.stdout[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail
