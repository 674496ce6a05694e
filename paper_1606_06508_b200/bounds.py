"""Error-bound sweep of batched normalize outputs on the GPU.

GPU counterpart of the reference's ``oracle.sweep_bounds`` / ``measure``
(pkg/src/fastnorm/oracle.py:151-290): every finite nonzero row is checked against the
paper's guarantees for the scaling algorithm (|sin phi| <= 1.001u, direction error
<= (3.001 + n/2)u, length error <= (1 + n/2)u r (3u r for quaternions, + alpha/2 near
underflow) under the finiteness premise, the ten quaternion product bounds) in
double-double arithmetic by ``fn_measure_bounds`` -- millions of rows per millisecond
instead of the reference's per-row 256-bit mpfr loop.  Metrics are returned in units of
u, like the reference's acceptance report.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_1606_06508_b200 import _lib, batch
from paper_1606_06508_b200.params import FpParams

__all__ = ["SweepSummary", "sweep_bounds", "VIOLATION_IDS"]

VIOLATION_IDS = ("nan-output", "nonzero-length", "finite-unit", "sin-phi", "direction",
                 "finite-length", "length-in-range", "length-near-underflow", "quaternion-product")
_METRICS = ("rel_length_err", "abs_length_err", "dir_err", "sin_phi")


@dataclass
class SweepSummary:
    """Aggregate of the bound checks over a batch (reference oracle.SweepSummary)."""

    samples: int
    skipped: int
    violation_count: int
    violation_ids: dict[str, int]
    max_metrics: dict[str, float]          # rel/dir/sin in units of u; abs_length_err absolute
    worst_rows: dict[str, int]
    first_violation_row: int | None
    bounds_u: dict[str, float] = field(default_factory=dict)


def sweep_bounds(p: FpParams, x, outcome=None) -> SweepSummary:
    """Check the scaling algorithm's bounds on rows ``x[N, n]`` (a CUDA tensor).

    ``outcome``: a NormalizeOutcome (length [N], unit [N, n]) already computed for x;
    when omitted, ``normalize{n}(p, x)`` is run first."""
    import torch

    from paper_1606_06508_b200 import normalize

    if not (batch.is_torch(x) and x.is_cuda):
        raise TypeError("sweep_bounds takes a CUDA tensor (move host arrays with torch.as_tensor(..., device='cuda'))")
    x = x.contiguous()
    n, dim = x.shape
    if outcome is None:
        outcome = getattr(normalize, f"normalize{dim}")(p, x)
    r, u = outcome.length.contiguous(), outcome.unit.contiguous()
    dt = _lib.F64 if x.dtype == torch.float64 else _lib.F32
    if (p.precision == "double") != (dt == _lib.F64):
        raise TypeError("parameter precision and row dtype differ")
    limits = np.array([p.u, p.alpha, p.nu, p.omega], dtype=np.float64)
    counts = torch.zeros(12, dtype=torch.int64, device=x.device)
    maxbits = torch.zeros(4, dtype=torch.int64, device=x.device)
    argmax = torch.zeros(5, dtype=torch.int64, device=x.device)
    argmax[4] = -1  # UINT64_MAX for the atomicMin
    with torch.cuda.device(x.device):
        rc = _lib.lib().fn_measure_bounds(dim, dt, x.data_ptr(), r.data_ptr(), u.data_ptr(), n,
                                          limits.ctypes.data, counts.data_ptr(), maxbits.data_ptr(),
                                          argmax.data_ptr(), torch.cuda.current_stream(x.device).cuda_stream)
    _lib.check(rc, "fn_measure_bounds")
    c = counts.cpu().tolist()
    mx = maxbits.cpu().numpy().view(np.float64)
    am = argmax.cpu().numpy().view(np.uint64).tolist()
    cn = 3.0 if dim == 4 else 1.0 + dim / 2.0
    maxes = {"rel_length_err": float(mx[0]) / p.u, "abs_length_err": float(mx[1]),
             "dir_err": float(mx[2]) / p.u, "sin_phi": float(mx[3]) / p.u}
    worst = {m: int(am[k]) for k, m in enumerate(_METRICS) if mx[k] > 0}
    return SweepSummary(
        samples=int(c[9]), skipped=int(c[10]), violation_count=int(c[11]),
        violation_ids={vid: int(c[k]) for k, vid in enumerate(VIOLATION_IDS) if c[k]},
        max_metrics=maxes, worst_rows=worst,
        first_violation_row=None if am[4] == 2 ** 64 - 1 else int(am[4]),
        bounds_u={"sin_phi": 1.001, "dir_err": 3.001 + dim / 2.0, "rel_length_err": cn},
    )
