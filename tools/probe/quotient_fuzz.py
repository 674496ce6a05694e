"""Developer probe (GPU): the f64 comparison families on large batches of arbitrary bit
patterns (and of narrow-exponent rows), against the oracle; prints the first mismatching
rows as hex.  Usage: python tools/probe/quotient_fuzz.py [rows] [rounds]"""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_1606_06508_b200 import _cuda_kernels, _lib  # noqa: E402

OPS = {"quotient": _lib.OP_QUOTIENT, "quotient3_fast": _lib.OP_QUOTIENT3_FAST, "naive": _lib.OP_NAIVE}


def rows(rng, n, dim, kind):
    w = rng.integers(0, 2 ** 64, size=(n, dim), dtype=np.uint64)
    if kind == 1:  # exponents at the bottom of the range (subnormal / tiny rows)
        w = (w & np.uint64(0x800FFFFFFFFFFFFF)) | (rng.integers(0, 70, size=(n, dim), dtype=np.uint64) << np.uint64(52))
    if kind == 2:  # one row exponent, components spread up to 1100 binades below it
        top = rng.integers(0, 2047, size=(n, 1), dtype=np.int64)
        e = np.clip(top - rng.integers(0, 1100, size=(n, dim)), 0, 2046).astype(np.uint64)
        w = (w & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52))
    return w.view(np.float64)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    rng = np.random.default_rng(7)
    total = 0
    for r in range(rounds):
        for dim in (2, 3, 4):
            for fam in ("quotient", "quotient3_fast", "naive"):
                if fam == "quotient3_fast" and dim != 3:
                    continue
                base = "quotient3_fast" if fam == "quotient3_fast" else f"{fam}{dim}"
                for kind in (0, 1, 2):
                    x = rows(rng, n, dim, kind)
                    xd = torch.from_numpy(x).cuda()
                    res = _cuda_kernels.batch_kernel(base, "f64")(xd, None)
                    h, b, _ = oracle.run(OPS[fam], x, None)
                    gh, gb = res.head.cpu().numpy(), res.body.cpu().numpy()
                    ok = oracle.same(gh, h) & oracle.same(gb, b).all(axis=1)
                    bad = np.flatnonzero(~ok)
                    total += len(bad)
                    print(f"round {r} {base} kind {kind}: {len(bad)} mismatching rows of {n}", flush=True)
                    for i in bad[:4]:
                        print("   x", [hex(v) for v in x[i].view(np.uint64)],
                              "\n   gpu", gh[i].hex(), [v.hex() for v in gb[i]],
                              "\n   ref", h[i].hex(), [v.hex() for v in b[i]], flush=True)
    print("total mismatches", total)


if __name__ == "__main__":
    main()
