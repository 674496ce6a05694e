"""CLI (reference cli.py): parsing and the GPU-free subcommands on CPU; the GPU ones
are exercised under -m gpu."""

import json
import math

import numpy as np
import pytest

from paper_1606_06508_b200 import cli


def test_parse_number():
    assert cli.parse_number("2^-1074") == 5e-324
    assert cli.parse_number("-2^10") == -1024.0
    assert cli.parse_number("0x1.8p+1") == 3.0
    assert math.isinf(cli.parse_number("inf")) and math.isnan(cli.parse_number("nan"))
    assert cli.parse_number("1e-3") == 1e-3


def test_validate_params(capsys, tmp_path):
    assert cli.main(["validate-params", "--format", "single", "--show-derived"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["valid"] and out["derived_tau"]["tau_min"] == 2.0 ** -50
    bad = {"u": "2^-53", "alpha": "2^-1074", "nu": "2^-1022", "omega": "1.7976931348623157e308",
           "tau_min": "2^-482", "tau_max": "2^512", "sigma_min": "2^592", "sigma_max": "2^-514"}
    f = tmp_path / "p.json"
    f.write_text(json.dumps(bad))
    assert cli.main(["validate-params", "--file", str(f)]) == 1
    out = json.loads(capsys.readouterr().out)
    assert not out["valid"] and "tau-max-squares-below-omega" in [v["check"] for v in out["violations"]]


def test_parser_rejects_bad_args():
    with pytest.raises(SystemExit):
        cli.main(["normalize", "--dim", "5", "1", "2"])
    with pytest.raises(SystemExit):
        cli.main(["rotate", "1", "2", "3"])


def test_compare(capsys, tmp_path):
    """compare: the reference's _same rule (NaN == NaN, zero signs count), per-array row
    counts and hex-float reports of the first mismatches."""
    u = np.array([[0.6, 0.8, 0.0], [np.nan, np.nan, np.nan], [1.0, -0.0, 0.0]])
    r = np.array([5.0, np.nan, 3.0])
    np.savez(tmp_path / "a.npz", length=r, unit=u)
    np.savez(tmp_path / "b.npz", length=r.copy(), unit=u.copy())
    assert cli.main(["compare", str(tmp_path / "a.npz"), str(tmp_path / "b.npz")]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["unit"]["mismatching_rows"] == 0 and out["length"]["rows"] == 3
    u2 = u.copy()
    u2[2, 1] = 0.0  # -0.0 -> +0.0 is a mismatch
    u2[0, 0] = np.nextafter(0.6, 1.0)
    np.savez(tmp_path / "c.npz", length=r, unit=u2)
    assert cli.main(["compare", str(tmp_path / "a.npz"), str(tmp_path / "c.npz"), "--array", "unit"]) == 1
    out = json.loads(capsys.readouterr().out)
    assert out["unit"]["mismatching_rows"] == 2 and list(out) == ["unit"]
    first = out["unit"]["first"][0]
    assert first["row"] == 0 and first["a"][0] == (0.6).hex() and first["b"][0] == np.nextafter(0.6, 1.0).hex()


@pytest.mark.gpu
def test_gpu_subcommands(capsys, tmp_path, cuda_dev):
    assert cli.main(["normalize", "--dim", "3", "3", "4", "12"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["length"] == 13.0
    assert cli.main(["normalize", "--dim", "2", "--algo", "quotient", "--hex", "3", "4"]) == 0
    assert json.loads(capsys.readouterr().out)["length"] == (5.0).hex()
    assert cli.main(["rotate", "1", "1", "1", "1", "--apply", "1", "0", "0"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["rows"] == [[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]] and out["applied"] == [0.0, 1.0, 0.0]
    assert cli.main(["rotate", "0", "0", "0", "0"]) == 2
    capsys.readouterr()
    assert cli.main(["verify-bounds", "--dim", "4", "--samples", "65536", "--regime", "all"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert all(r["violations"] == 0 for r in out["results"]) and len(out["results"]) == 5
    x = np.random.default_rng(0).standard_normal((1000, 3))
    np.save(tmp_path / "x.npy", x)
    assert cli.main(["batch", "--dim", "3", "--in", str(tmp_path / "x.npy"), "--out", str(tmp_path / "o.npz")]) == 0
    capsys.readouterr()
    o = np.load(tmp_path / "o.npz")
    assert o["unit"].shape == (1000, 3) and np.allclose(np.linalg.norm(o["unit"], axis=1), 1.0)
    assert cli.main(["bench", "--config", "1", "--steps", "3"]) == 0
    assert json.loads(capsys.readouterr().out)["vectors_per_s"] > 1e9
    assert cli.main(["bench", "--config", "4", "--rows", "3000001", "--steps", "3", "--devices", "0,0,0"]) == 0
    sharded = json.loads(capsys.readouterr().out)
    assert sharded["devices"] == [0, 0, 0] and sum(sharded["rows_per_shard"]) == 3000001
    assert sharded["vectors_per_s"] > 1e9
    assert cli.main(["selftest", "--pairs", "1000000"]) == 0
