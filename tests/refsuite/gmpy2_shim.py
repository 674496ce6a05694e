"""A small stand-in for gmpy2 (absent from this image), enough for the reference's
accuracy oracle (pkg/src/fastnorm/oracle.py) and its tests.

TEST INFRASTRUCTURE -- never imported by the product.  The reference uses four names:

* ``mpq(x)``   -- an exact rational (here a ``fractions.Fraction``); floats convert
                  exactly, ``mpq()`` is 0;
* ``mpfr(x)``  -- a binary floating-point number of the current context's precision
                  (here an exact dyadic ``Fraction`` rounded to that many significant
                  bits, round-to-nearest-even), or +-inf / nan;
* ``sqrt(x)``  -- the square root rounded to the context's precision;
* ``context(precision=P)`` -- a context manager selecting P bits (oracle.py:54).

Arithmetic mixing mpfr with mpq / int / float gives an mpfr rounded to the context
precision, as in gmpy2; mpq with mpq stays exact.  Comparisons are exact.  The
reference's oracle works at 256+ bits and compares against rational tolerances with a
margin of 2^-250 of the bound (oracle.py:1-12), so how the last of those bits rounds
here cannot change any verdict.
"""

from __future__ import annotations

import math
from fractions import Fraction

__all__ = ["mpq", "mpfr", "sqrt", "context", "get_context"]

_precision = [53]


class context:
    def __init__(self, precision: int = 53):
        self.precision = int(precision)

    def __enter__(self):
        _precision.append(self.precision)
        return self

    def __exit__(self, *exc):
        _precision.pop()
        return False


def get_context() -> context:
    return context(_precision[-1])


class mpq(Fraction):
    def __new__(cls, *args):
        if not args:
            return super().__new__(cls, 0)
        if len(args) == 1:
            v = args[0]
            if isinstance(v, mpfr):
                if v._q is None:
                    raise ValueError("mpq() of a non-finite mpfr")
                return super().__new__(cls, v._q)
            if isinstance(v, float):
                if not math.isfinite(v):
                    raise ValueError("mpq() of a non-finite float")
                return super().__new__(cls, *v.as_integer_ratio())
        return super().__new__(cls, *args)


def _round(q: Fraction, prec: int) -> Fraction:
    """q rounded to ``prec`` significant bits, ties to even."""
    if q == 0:
        return Fraction(0)
    sign = -1 if q < 0 else 1
    num, den = abs(q.numerator), q.denominator
    # exponent e with 2^(e-1) <= |q| < 2^e
    e = num.bit_length() - den.bit_length()
    if (num << max(0, -e)) >= (den << max(0, e)):
        e += 1
    shift = prec - e  # scale so the integer part has exactly prec bits
    if shift >= 0:
        n, d = num << shift, den
    else:
        n, d = num, den << -shift
    m, r = divmod(n, d)
    if 2 * r > d or (2 * r == d and (m & 1)):
        m += 1
    return sign * (Fraction(m, 1 << shift) if shift >= 0 else Fraction(m << -shift))


def _exact(v):
    """(kind, value): kind 'q' with a Fraction, or 'f' with a non-finite float."""
    if isinstance(v, mpfr):
        return ("q", v._q) if v._q is not None else ("f", v._f)
    if isinstance(v, (Fraction, int)):
        return "q", Fraction(v)
    if isinstance(v, float):
        return ("q", Fraction(*v.as_integer_ratio())) if math.isfinite(v) else ("f", v)
    return None, None


class mpfr:
    __slots__ = ("_q", "_f")

    def __init__(self, v=0, precision: int | None = None):
        prec = precision or _precision[-1]
        if isinstance(v, str):
            s = v.strip().lower()
            if s in ("inf", "+inf", "-inf", "nan"):
                self._q, self._f = None, float(s)
                return
            v = Fraction(s)
        kind, val = _exact(v)
        if kind is None:
            raise TypeError(f"mpfr() of {type(v).__name__}")
        if kind == "f":
            self._q, self._f = None, val
        else:
            self._q, self._f = _round(val, prec), None

    @classmethod
    def _make(cls, kind, val):
        out = cls.__new__(cls)
        if kind == "f":
            out._q, out._f = None, val
        else:
            out._q, out._f = _round(val, _precision[-1]), None
        return out

    def _binop(self, other, op, reflected=False):
        ka, a = _exact(self)
        kb, b = _exact(other)
        if kb is None:
            return NotImplemented
        if reflected:
            ka, a, kb, b = kb, b, ka, a
        if ka == "q" and kb == "q":
            if op == "/" and b == 0:
                if a == 0:
                    return mpfr._make("f", math.nan)
                return mpfr._make("f", math.copysign(math.inf, a))
            r = {"+": lambda: a + b, "-": lambda: a - b, "*": lambda: a * b, "/": lambda: a / b}[op]()
            return mpfr._make("q", r)
        # one side is +-inf or nan: a finite side matters only through its sign / zero-ness
        fa = a if ka == "f" else (math.copysign(1.0, a) if a != 0 else 0.0)
        fb = b if kb == "f" else (math.copysign(1.0, b) if b != 0 else 0.0)
        try:
            r = {"+": lambda: fa + fb, "-": lambda: fa - fb, "*": lambda: fa * fb, "/": lambda: fa / fb}[op]()
        except ZeroDivisionError:
            r = math.copysign(math.inf, fa) if fa != 0 else math.nan
        if math.isfinite(r):  # finite / inf
            return mpfr._make("q", Fraction(0))
        return mpfr._make("f", r)

    def __add__(self, o):
        return self._binop(o, "+")

    def __radd__(self, o):
        return self._binop(o, "+", True)

    def __sub__(self, o):
        return self._binop(o, "-")

    def __rsub__(self, o):
        return self._binop(o, "-", True)

    def __mul__(self, o):
        return self._binop(o, "*")

    def __rmul__(self, o):
        return self._binop(o, "*", True)

    def __truediv__(self, o):
        return self._binop(o, "/")

    def __rtruediv__(self, o):
        return self._binop(o, "/", True)

    def __neg__(self):
        return mpfr._make("f", -self._f) if self._q is None else mpfr._make("q", -self._q)

    def __pos__(self):
        return self

    def __abs__(self):
        return mpfr._make("f", abs(self._f)) if self._q is None else mpfr._make("q", abs(self._q))

    def _cmp(self, other):
        ka, a = _exact(self)
        kb, b = _exact(other)
        if kb is None:
            return None
        if ka == "q" and kb == "q":
            return a, b
        return (a if ka == "f" else math.copysign(1.0, a) if a != 0 else 0.0), \
               (b if kb == "f" else math.copysign(1.0, b) if b != 0 else 0.0)

    def __eq__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c[0] == c[1]

    def __ne__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c[0] != c[1]

    def __lt__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c[0] < c[1]

    def __le__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c[0] <= c[1]

    def __gt__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c[0] > c[1]

    def __ge__(self, o):
        c = self._cmp(o)
        return NotImplemented if c is None else c[0] >= c[1]

    def __hash__(self):
        return hash(self._f if self._q is None else self._q)

    def __float__(self):
        if self._q is None:
            return self._f
        try:
            return float(self._q)
        except OverflowError:  # beyond the binary64 range, as gmpy2 converts it
            return math.copysign(math.inf, self._q)

    def __bool__(self):
        return bool(self._f) if self._q is None else self._q != 0

    def is_nan(self) -> bool:
        return self._q is None and math.isnan(self._f)

    def is_infinite(self) -> bool:
        return self._q is None and math.isinf(self._f)

    def __repr__(self):
        return f"mpfr('{float(self)!r}')"

    __str__ = __repr__


def sqrt(x):
    """Square root at the context precision (round to nearest)."""
    kind, q = _exact(x)
    if kind is None:
        raise TypeError(f"sqrt() of {type(x).__name__}")
    if kind == "f":
        return mpfr._make("f", math.sqrt(q) if q >= 0 else math.nan)
    if q < 0:
        return mpfr._make("f", math.nan)
    if q == 0:
        return mpfr._make("q", Fraction(0))
    prec = _precision[-1]
    # floor(sqrt(q) * 2^k) with k giving prec + 64 bits, then one rounding to prec bits; an
    # inexact root is represented as floor + 1/2 (a sticky bit), which rounds as it should.
    k = prec + 64 - (q.numerator.bit_length() - q.denominator.bit_length()) // 2
    if k >= 0:
        num, den = q.numerator << (2 * k), q.denominator
    else:
        num, den = q.numerator, q.denominator << (-2 * k)
    scaled, rem = divmod(num, den)
    s = math.isqrt(scaled)
    exact = rem == 0 and s * s == scaled
    root = Fraction(2 * s + (0 if exact else 1), 2) * Fraction(2) ** (-k)
    return mpfr._make("q", root)
