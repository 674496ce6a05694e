"""``generate_inputs`` reproduces the reference's seeded batches bit for bit
(pkg/src/fastnorm/bench.py:146-207): against the committed golden batches made by the
reference itself (tests/golden/make_generate_inputs.py) and, where /root/reference is
present, against the live reference function on more sizes and seeds."""

import os
import sys

import numpy as np
import pytest

from paper_1606_06508_b200 import bench

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import make_generate_inputs as gi  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "generate_inputs.npz")


def _bits(a):
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def test_generate_inputs_equals_reference_golden():
    gold = np.load(GOLDEN)
    n = 0
    for c in gi.cases():
        want = gold[gi.key(*c)]
        got = bench.generate_inputs(c[0], c[1], c[2], gi.COUNT, c[3])
        assert got.dtype == want.dtype and got.shape == want.shape and got.flags.c_contiguous
        assert np.array_equal(_bits(got), _bits(want)), c
        n += 1
    assert n == len(gold.files) == 5 * 3 * 2 * len(gi.SEEDS)


@pytest.mark.skipif(not os.path.isdir(gi.REF), reason="reference sources not present")
@pytest.mark.parametrize("count", [1, 2, 1000, 4097])
def test_generate_inputs_equals_live_reference(count):
    ref = gi.load_reference_bench()
    for regime in gi.REGIMES:
        for dim in (2, 3, 4):
            for prec in ("double", "single"):
                for seed in (11, (5, 1, dim)):
                    want = ref.generate_inputs(regime, dim, prec, count, seed)
                    got = bench.generate_inputs(regime, dim, prec, count, seed)
                    assert np.array_equal(_bits(got), _bits(want)), (regime, dim, prec, seed)
    for bad in (("weird", 3, "double", 4, 0), ("normal", 5, "double", 4, 0),
                ("normal", 3, "half", 4, 0), ("normal", 3, "double", 0, 0)):
        with pytest.raises(ValueError):
            ref.generate_inputs(*bad)
        with pytest.raises(ValueError):
            bench.generate_inputs(*bad)


def test_counter_generator_keeps_its_own_name():
    from paper_1606_06508_b200 import workloads

    y = bench.generate_regime_rows("mixed", 4, "single", 64, seed=7)
    assert np.array_equal(y, workloads.regime_rows("mixed", 4, "float32", 0, 64, seed=7))
