"""Constants and validation (reference: tests/test_params.py, params.py:97-210)."""

import math
from fractions import Fraction

import pytest

from paper_1606_06508_b200.params import (
    CHECK_IDS,
    FpParams,
    FpParamsError,
    derive_tau,
    preset,
    require_valid,
    validate_conditions,
)
from paper_1606_06508_b200.scale import kernel_args

L = math.ldexp


def test_table2_constants():
    d = preset("double")
    assert (d.u, d.alpha, d.nu) == (L(1, -53), L(1, -1074), L(1, -1022))
    assert d.omega == 1.7976931348623157e308
    assert (d.tau_min, d.tau_max, d.sigma_min, d.sigma_max) == (L(1, -482), L(1, 510), L(1, 592), L(1, -514))
    s = preset("single")
    assert (s.u, s.alpha, s.nu) == (L(1, -24), L(1, -149), L(1, -126))
    assert s.omega == float.fromhex("0x1.fffffep+127")
    assert (s.tau_min, s.tau_max, s.sigma_min, s.sigma_max) == (L(1, -49), L(1, 62), L(1, 100), L(1, -66))
    assert preset("DOUBLE") == preset("double")
    with pytest.raises(ValueError):
        preset("half")


def test_precision_property():
    assert preset("double").precision == "double"
    assert preset("single").precision == "single"
    with pytest.raises(ValueError):
        preset("double").with_field("u", L(1, -40)).precision


def test_presets_are_valid():
    assert validate_conditions(preset("double")) == ()
    assert validate_conditions(preset("single")) == ()
    assert require_valid(preset("single")) is preset("single")


def test_kernel_args():
    ka = kernel_args(preset("double"))
    assert ka == (L(1, -482), L(1, 510), L(1, 592), L(1, -514), L(1, -592), L(1, 514))
    ka = kernel_args(preset("single"))
    assert ka == (L(1, -49), L(1, 62), L(1, 100), L(1, -66), L(1, -100), L(1, 66))


@pytest.mark.parametrize("field,value,check", [
    ("sigma_min", 3.0 * L(1, 590), "sigma-min-power-of-two"),
    ("sigma_max", 3.0 * L(1, -516), "sigma-max-power-of-two"),
    ("tau_max", L(1, 512), "tau-max-squares-below-omega"),
    ("tau_min", L(1, -500), "tau-min-squares-above-alpha"),
    ("sigma_min", L(1, 500), "upscale-lands-in-band"),
    ("sigma_max", L(1, -400), "downscale-lands-in-band"),
    ("u", L(1, -10), "u-small-enough"),
])
def test_single_violations(field, value, check):
    p = preset("double").with_field(field, value)
    ids = [v.check for v in validate_conditions(p)]
    assert check in ids
    assert set(ids) <= set(CHECK_IDS)
    with pytest.raises(FpParamsError) as e:
        kernel_args(p)
    assert check in str(e.value)
    assert any(v.check == check for v in e.value.violations)


def test_non_power_of_two_tau_is_allowed():
    # validate_conditions does not require tau to be a power of two (params.py:166-169)
    p = preset("double").with_field("tau_min", 3 * L(1, -484))
    assert validate_conditions(p) == ()


def test_fields_must_be_positive_finite():
    with pytest.raises(ValueError):
        FpParams(1.0, 1.0, 1.0, math.inf, 1.0, 1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        FpParams(1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.0)


def test_derive_tau():
    lo, hi = derive_tau("double")
    assert (lo, hi) == (L(1, -484), L(1, 510))
    lo, hi = derive_tau("single")
    assert (lo, hi) == (L(1, -50), L(1, 62))


def test_upscale_exact_sweep():
    # sigma_min * x for x in (0, tau_min] lands in the band exactly (powers of two)
    p = preset("double")
    for e in range(-1074, -482):
        v = Fraction(p.sigma_min) * Fraction(L(1, e))
        assert Fraction(p.tau_min) <= v <= Fraction(p.tau_max)
