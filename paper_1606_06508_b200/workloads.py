"""Seeded synthetic workloads for BASELINE.json configs 1-5.

The CUDA generator (csrc/workloads.cu, ``fn_generate``) writes rows straight into HBM;
:func:`host_rows` restates it in numpy for host-side use (the CPU baseline sample and
the tests).  Both derive every 64-bit word from splitmix64 of
``key + (row*16 + j) * GOLDEN`` with ``key = splitmix64(seed ^ cfg * K)``, so a row
depends only on (cfg, seed, global row index): shards generated on different GPUs, or
on the host, agree.  Configs 1, 2, 4 and 5 use only integer operations and exact
ldexp / rounding conversions and are bit-identical between host and device; config 3
(standard normals via Box-Muller) matches in distribution only (libm vs CUDA
log/sin/cos), so its parity tests always feed the oracle the device's own inputs.

Config recipes:
  1  3-D f64, N=1e6:   x_k = (w_k >> 11) * 2^-52 - 1                  (uniform [-1, 1))
  2  2-D f64, N=2^26:  1 % rows +-0; else x_k = +-(1 + m*2^-52) * 2^e, e ~ U{-1000..1000}
  3  4-D f64, N=2^27:  Box-Muller standard normals
  4  3-D f32, N=2^28:  0.1 % rows +-0; 0.01 % rows with one NaN/+inf/-inf component;
                       else x_k = f32(+-(1 + m*2^-23) * 2^e), e ~ U{-149..127}
  5  3-D f64, N=2^30:  0.5 % rows with one component +-[2^1023, DBL_MAX]; 0.5 % rows of
                       subnormals (random mantissa, random leading-bit position); else
                       x_k = +-(1 + m*2^-52) * 2^e, e ~ U{-1020..1020}
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_1606_06508_b200 import _lib

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_CFG_MUL = 0xD6E8FEB86659FD93

P1PCT = 90071992547409        # floor(0.01   * 2^53)
P01PCT = 9007199254740        # floor(0.001  * 2^53)
P001PCT = 900719925474        # floor(0.0001 * 2^53)
P05PCT = 45035996273704       # floor(0.005  * 2^53)


@dataclass(frozen=True)
class Config:
    cfg: int
    dim: int
    dtype: str          # "float64" | "float32"
    rows: int
    seed: int
    description: str

    @property
    def bytes_in_per_row(self) -> int:
        return self.dim * np.dtype(self.dtype).itemsize


CONFIGS = {
    1: Config(1, 3, "float64", 1_000_000, 0, "3D f64 uniform[-1,1], scaling"),
    2: Config(2, 2, "float64", 1 << 26, 2, "2D f64 sign*2^e*m e~U[-1000,1000], 1% zero rows; scaling + quotient"),
    3: Config(3, 4, "float64", 1 << 27, 3, "quaternion f64 N(0,1); squared norm, r, unit"),
    4: Config(4, 3, "float32", 1 << 28, 4, "3D f32 log-uniform full range incl. subnormals, 0.1% zero, 0.01% NaN/Inf rows"),
    5: Config(5, 3, "float64", 1 << 30, 5, "3D f64 e~U[-1020,1020], 0.5% near-DBL_MAX, 0.5% all-subnormal rows"),
}


def _mix(z: np.ndarray) -> np.ndarray:
    z = z + GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _key(cfg: int, seed: int) -> np.uint64:
    z = np.array([(seed ^ (cfg * _CFG_MUL)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return _mix(z)[0]


def _words(key: np.uint64, rows: np.ndarray, j: int) -> np.ndarray:
    c = rows.astype(np.uint64) * np.uint64(16) + np.uint64(j)
    return _mix(key + c * GOLDEN)


def _sign(w: np.ndarray) -> np.ndarray:
    return np.where((w >> np.uint64(63)) != 0, -1.0, 1.0)


def _mant52(w: np.ndarray) -> np.ndarray:
    return 1.0 + (w >> np.uint64(12)).astype(np.float64) * 2.0 ** -52


def _uexp(w: np.ndarray, lo: int, span: int) -> np.ndarray:
    return lo + ((w & np.uint64(0xFFFFFFFF)) % np.uint64(span)).astype(np.int64)


def host_rows(cfg: int, row0: int, n: int, seed: int | None = None) -> np.ndarray:
    """Rows [row0, row0+n) of config ``cfg`` as a host array (numpy restatement)."""
    c = CONFIGS[cfg]
    seed = c.seed if seed is None else seed
    key = _key(cfg, seed)
    rows = np.arange(row0, row0 + n, dtype=np.int64)
    W = lambda j: _words(key, rows, j)  # noqa: E731
    with np.errstate(over="ignore", invalid="ignore"):
        if cfg == 1:
            return np.stack([(W(k) >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0
                             for k in range(3)], axis=1)
        if cfg == 2:
            zero = (W(15) >> np.uint64(11)) < np.uint64(P1PCT)
            cols = []
            for k in range(2):
                w = W(k)
                v = np.ldexp(_mant52(W(4 + k)), _uexp(w, -1000, 2001))
                cols.append(_sign(w) * np.where(zero, 0.0, v))
            return np.stack(cols, axis=1)
        if cfg == 3:
            cols = []
            for p in range(2):
                u1 = ((W(2 * p) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
                u2 = (W(2 * p + 1) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
                rad = np.sqrt(-2.0 * np.log(u1))
                cols += [rad * np.cos(2.0 * np.pi * u2), rad * np.sin(2.0 * np.pi * u2)]
            return np.stack(cols, axis=1)
        if cfg == 4:
            v = W(15) >> np.uint64(11)
            zero = v < np.uint64(P01PCT)
            special = (~zero) & (v < np.uint64(P01PCT + P001PCT))
            which = (W(14) % np.uint64(3)).astype(np.int64)
            kind = (W(13) % np.uint64(3)).astype(np.int64)
            spec_val = np.choose(kind, [np.float32(np.nan), np.float32(np.inf), np.float32(-np.inf)])
            cols = []
            for k in range(3):
                w = W(k)
                m = 1.0 + (W(4 + k) >> np.uint64(41)).astype(np.float64) * 2.0 ** -23
                v32 = (_sign(w) * np.ldexp(m, _uexp(w, -149, 277))).astype(np.float32)
                v32 = np.where(zero, (_sign(w) * 0.0).astype(np.float32), v32)
                v32 = np.where(special & (which == k), spec_val.astype(np.float32), v32)
                cols.append(v32.astype(np.float32))
            return np.stack(cols, axis=1)
        if cfg == 5:
            v = W(15) >> np.uint64(11)
            nearmax = v < np.uint64(P05PCT)
            subn = (~nearmax) & (v < np.uint64(2 * P05PCT))
            which = (W(14) % np.uint64(3)).astype(np.int64)
            cols = []
            for k in range(3):
                w, wm = W(k), W(4 + k)
                normal = _sign(w) * np.ldexp(_mant52(wm), _uexp(w, -1020, 2041))
                big = _sign(w) * np.ldexp(_mant52(wm), 1023)
                shift = (W(8 + k) & np.uint64(0xFFFFFFFF)) % np.uint64(52)
                mant = ((wm >> np.uint64(12)) | np.uint64(1 << 51)) >> shift
                sub = ((w & np.uint64(0x8000000000000000)) | mant).view(np.float64)
                col = np.where(subn, sub, np.where(nearmax & (which == k), big, normal))
                cols.append(col)
            return np.stack(cols, axis=1)
    raise ValueError(f"unknown config {cfg}")


REGIMES = ("normal", "subnormal", "huge", "mixed", "unit-ish")
_REGIME_FMT = {  # (tau_min exp, tau_max exp, min subnormal, min normal, max) binade exponents
    "float64": (-482, 510, -1074, -1022, 1023),
    "float32": (-49, 62, -149, -126, 127),
}


def _regime_key(regime: int, dim: int, dtype: str, seed: int) -> np.uint64:
    cfg_id = 100 + regime * 16 + dim * 2 + (1 if dtype == "float64" else 0)
    z = np.array([(seed ^ (cfg_id * _CFG_MUL)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return _mix(z)[0]


def regime_rows(regime: str, dim: int, dtype: str, row0: int, n: int, seed: int = 0) -> np.ndarray:
    """Host restatement of fn_generate_regime: the reference harness's regimes
    (bench.py:146-207) on the counter-based generator.  Bit-identical to the device for
    every regime but unit-ish (Box-Muller through libm)."""
    r = REGIMES.index(regime)
    tmin, tmax, sub_min, norm_min, emax = _REGIME_FMT[dtype]
    key = _regime_key(r, dim, dtype, seed)
    rows = np.arange(row0, row0 + n, dtype=np.int64)
    W = lambda j: _words(key, rows, j)  # noqa: E731
    single = dtype == "float32"
    cap = (2.0 ** -126 - 2.0 ** -149) if single else (2.0 ** -1022 - 2.0 ** -1074)
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        if r == 4:
            g = []
            for p in range(2):
                u1 = ((W(2 * p) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
                u2 = (W(2 * p + 1) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
                rad = np.sqrt(-2.0 * np.log(u1))
                g += [rad * np.cos(2.0 * np.pi * u2), rad * np.sin(2.0 * np.pi * u2)]
            g = np.stack(g[:dim], axis=1)
            ss = np.zeros(n)
            for k in range(dim):
                ss = ss + g[:, k] * g[:, k]
            nrm = np.sqrt(ss)
            g[:, 0] = np.where(nrm == 0.0, 1.0, g[:, 0])
            nrm = np.maximum(nrm, np.finfo(np.float64).tiny)
            u = (W(12) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            vals = (g / nrm[:, None]) * (1.0 + (u * 2.0 - 1.0) * 2.0 ** -10)[:, None]
        else:
            lo, span = {0: (tmin, tmax - tmin), 1: (sub_min, norm_min - sub_min),
                        2: (tmax + 1, emax - 1 - (tmax + 1)), 3: (sub_min, emax - sub_min)}[r]
            cols = []
            for k in range(dim):
                w = W(k)
                mag = np.ldexp(_mant52(W(4 + k)), _uexp(w, lo, span))
                if r == 1:
                    mag = np.minimum(mag, cap)
                cols.append(_sign(w) * mag)
            vals = np.stack(cols, axis=1)
        out = vals.astype(np.float32 if single else np.float64)
        if single and r == 1:
            c = np.float32(cap)
            out = np.clip(out, -c, c)
    return np.ascontiguousarray(out)


def generate_regime_device(regime: str, x, row0: int = 0, seed: int = 0, stream=None) -> None:
    """Fill a contiguous CUDA tensor x[n, dim] (float32/float64) with regime rows."""
    import torch

    r = REGIMES.index(regime)
    dt = _lib.F64 if x.dtype == torch.float64 else _lib.F32
    s = torch.cuda.current_stream(x.device).cuda_stream if stream is None else stream
    with torch.cuda.device(x.device):
        rc = _lib.lib().fn_generate_regime(r, x.shape[1], dt, seed, row0, x.shape[0], x.data_ptr(), s)
    _lib.check(rc, "fn_generate_regime")


def generate_device(cfg: int, x, row0: int = 0, seed: int | None = None, stream=None) -> None:
    """Fill a contiguous CUDA tensor x[n, dim] with rows [row0, row0+n) of ``cfg``."""
    c = CONFIGS[cfg]
    if tuple(x.shape[1:]) != (c.dim,) or str(x.dtype).replace("torch.", "") != c.dtype:
        raise ValueError(f"config {cfg} needs [N, {c.dim}] {c.dtype}")
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("x must be a contiguous CUDA tensor")
    import torch

    s = torch.cuda.current_stream(x.device).cuda_stream if stream is None else stream
    with torch.cuda.device(x.device):
        rc = _lib.lib().fn_generate(cfg, c.seed if seed is None else seed, row0, x.shape[0],
                                    x.data_ptr(), s)
    _lib.check(rc, "fn_generate")


def row_stats_device(x, ka, counts, stream=None) -> None:
    """Accumulate the six per-row class counters of x into the uint64 CUDA tensor counts."""
    import torch

    dim = x.shape[1]
    dt = _lib.F64 if x.dtype == torch.float64 else _lib.F32
    ka_arr = np.ascontiguousarray(np.asarray(ka, dtype=np.float64))
    s = torch.cuda.current_stream(x.device).cuda_stream if stream is None else stream
    with torch.cuda.device(x.device):
        rc = _lib.lib().fn_row_stats(dim, dt, x.data_ptr(), x.shape[0], counts.data_ptr(),
                                     ka_arr.ctypes.data, s)
    _lib.check(rc, "fn_row_stats")


def row_stats_host(x: np.ndarray, ka) -> np.ndarray:
    """Host restatement of the six counters (for checks against fn_row_stats)."""
    ab = np.abs(x)
    nan = np.isnan(x).any(axis=1)
    inf = np.isinf(x).any(axis=1) & ~nan
    m = np.where(np.isnan(ab), 0, ab).max(axis=1)
    tmin, tmax = (np.asarray(ka[0], dtype=x.dtype), np.asarray(ka[1], dtype=x.dtype))
    rest = ~nan & ~inf
    zero = rest & (m == 0)
    small = rest & ~zero & (m < tmin)
    big = rest & ~zero & (m > tmax)
    band = rest & ~zero & ~small & ~big
    return np.array([nan.sum(), inf.sum(), zero.sum(), small.sum(), big.sum(), band.sum()],
                    dtype=np.uint64)
