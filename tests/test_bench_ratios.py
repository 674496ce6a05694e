"""The GPU ratio harness (paper_1606_06508_b200.bench, mirror of the reference's
fastnorm.bench): configuration checks and input generation on CPU, one small protocol
run on the GPU."""

import json

import numpy as np
import pytest

from paper_1606_06508_b200 import bench, workloads


def test_generate_inputs_regimes_and_validation():
    for regime in bench.REGIMES:
        x = bench.generate_inputs(regime, 3, "double", 257, (1, 2))
        assert x.shape == (257, 3) and x.dtype == np.float64 and np.isfinite(x).all()
        assert (np.abs(x).max(axis=1) > 0).all()
    y = bench.generate_inputs("mixed", 4, "single", 64, 7)
    assert y.dtype == np.float32
    n = bench.generate_inputs("normal", 2, "double", 1000, 3)
    assert (np.abs(n) >= 2.0 ** -482).all() and (np.abs(n) < 2.0 ** 511).all()
    with pytest.raises(ValueError):
        bench.generate_inputs("weird", 3, "double", 4, 0)
    with pytest.raises(ValueError):
        bench.generate_inputs("normal", 5, "double", 4, 0)
    with pytest.raises(ValueError):
        bench.generate_inputs("normal", 3, "half", 4, 0)
    with pytest.raises(ValueError):
        bench.generate_inputs("normal", 3, "double", 0, 0)


@pytest.mark.parametrize("bad", [dict(experiments=0), dict(rows=-1), dict(dimensions=(5,)),
                                 dict(precisions=("half",)), dict(algorithms=("magic",)),
                                 dict(regime="weird"), dict(algorithms=())])
def test_config_validation(bad):
    with pytest.raises(bench.BenchConfigError):
        bench.run_bench(bench.BenchConfig(**bad))


@pytest.mark.gpu
def test_run_bench_small():
    cfg = bench.BenchConfig(experiments=2, rows=1 << 16, reps=2, dimensions=(2, 3),
                            precisions=("double", "single"), regime="mixed")
    rep = bench.run_bench(cfg)
    # 4 algorithms at n=3, 3 at n=2 (quotient_fast is 3-D only), 2 precisions
    assert len(rep.rows) == 2 * (4 + 3)
    assert all(r.mean_ns_per_vector > 0 and r.vectors_per_s > 0 for r in rep.rows)
    labels = sorted((r.label, r.task, r.precision, r.numerator) for r in rep.ratios)
    assert ("T3", "normalize3d", "double", "quotient_fast") in labels
    assert ("T3", "normalize2d", "double", "quotient_fast") not in labels
    assert len(rep.ratios) == 2 * (3 + 2)
    body = json.loads(rep.to_json())
    assert body["config"]["rows"] == 1 << 16 and len(body["rows"]) == len(rep.rows)
    assert rep.to_csv().count("\nratio,") == len(rep.ratios)
