"""Helpers for the GPU parity tests: chunked full-size comparison against the oracle."""

from __future__ import annotations

import os

import numpy as np

import oracle

THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


def to_np(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def compare_chunked(op: int, x_dev, head_dev, body_dev=None, sq_dev=None, ka=None,
                    chunk: int = 1 << 25) -> tuple[int, str]:
    """Bit-compare device outputs with the oracle over every row, chunk by chunk.

    Returns (number of mismatching rows, description of the first mismatch)."""
    n = x_dev.shape[0]
    bad = 0
    first = ""
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        x = to_np(x_dev[lo:hi])
        h, b, q = oracle.run(op, x, ka, threads=THREADS)
        ok = oracle.same(to_np(head_dev[lo:hi]), h)
        if body_dev is not None:
            ok &= oracle.same(to_np(body_dev[lo:hi]), b).all(axis=1)
        if sq_dev is not None:
            ok &= oracle.same(to_np(sq_dev[lo:hi]), q)
        nbad = int((~ok).sum())
        if nbad and not first:
            i = int(np.argmax(~ok))
            got = [to_np(head_dev[lo + i: lo + i + 1])]
            first = f"row {lo + i}: x={x[i].tolist()} oracle head={h[i]!r}"
            if b is not None:
                first += f" body={b[i].tolist()} gpu body={to_np(body_dev[lo + i]).tolist()}"
            first += f" gpu head={got[0].tolist()}"
        bad += nbad
    return bad, first
