"""The public wrappers called the reference's way -- named x1..xn, ``precision=`` by
keyword or position (normalize.py:51-89, scale.py:33-51, baselines.py:30-76) -- and
the batched overloads that share those names, on the GPU."""

import math

import numpy as np
import pytest

import paper_1606_06508_b200 as fn

pytestmark = pytest.mark.gpu


def test_keyword_calls_like_the_reference():
    p = fn.preset("double")
    out = fn.normalize3(p, x1=3.0, x2=4.0, x3=12.0)
    assert out.length == 13.0 and out.unit == (3 / 13, 4 / 13, 12 / 13)
    assert fn.norm2(p, x1=3.0, x2=4.0) == 5.0
    assert fn.scale3(p, 1.0, x2=2.0, x3=3.0) == fn.scale3(p, 1.0, 2.0, 3.0)
    q = fn.normalize4(p, x1=0.0, x2=0.0, x3=0.0, x4=0.0)
    assert q.length == 0.0 and q.unit == (0.0, 0.0, 0.0, 1.0)
    r = fn.quotient3_robust(x1=3.0, x2=4.0, x3=12.0)
    assert r.length == 13.0
    s = fn.quotient3_robust(3.0, 4.0, 12.0, precision="single")
    assert s.length == 13.0
    assert fn.quotient2(3.0, 4.0, "single") == fn.quotient2(x1=3.0, x2=4.0, precision="single")
    n = fn.naive_normalize2(x1=1e200, x2=1e200)
    assert math.isinf(n.length) and n.unit == (0.0, 0.0)


def test_batched_overloads_keep_working():
    p64, p32 = fn.preset("double"), fn.preset("single")
    x = np.array([[3.0, 4.0, 12.0], [0.0, 0.0, 0.0]])
    out = fn.normalize3(p64, x)
    assert out.length.tolist() == [13.0, 0.0]
    soa = fn.normalize3(p64, x[:, 0].copy(), x[:, 1].copy(), x[:, 2].copy())
    assert soa.length.tolist() == [13.0, 0.0]
    # baselines: the array's dtype is the precision unless precision= is given explicitly
    x32 = x.astype(np.float32)
    assert fn.quotient3_robust(x32).length.dtype == np.float32
    assert fn.quotient3_robust(x32, precision="single").length.tolist() == [13.0, 0.0]
    with pytest.raises(TypeError):
        fn.quotient3_robust(x32, precision="double")
    with pytest.raises(TypeError):
        fn.normalize3(p32, x)  # f64 rows under single-precision constants
    with pytest.raises(TypeError):
        fn.normalize3(p64, 1.0, 2.0)  # two of three components
