"""Extended-precision scalars and precision levels (mirror of polynewt.xprec).

Scalars here are immutable component containers with the reference's
equality, hashing, float conversion and decimal rendering
(xprec.py:52-345, 406-446).  Field arithmetic on them (+, -, *, /, abs,
sqrt) runs on the GPU through the element-wise kernels of the C ABI
(``pn_vec_op``), exactly like the vectorised arrays of :mod:`.varith`; there
is no CPU implementation of the extended-precision arithmetic in the
product.  Objects from the reference package itself (``polynewt.xprec``) are
accepted wherever a scalar is expected (duck typing on ``.comps`` /
``.re``/``.im``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from decimal import Decimal, localcontext
from fractions import Fraction

import numpy as np


class DomainError(ArithmeticError):
    """Raised for division by zero and square roots of negative values."""


# -- construction-time normalisation of scalar components -------------------
# The reference normalises in its constructors (DoubleDouble.__init__ runs
# quick_two_sum, xprec.py:57-58; QuadDouble.__init__ runs renorm5, 175-176).
# These few binary64 operations on Python floats only canonicalise a literal
# being built; no hot-path arithmetic happens here.

def _qts(a: float, b: float):
    s = a + b
    return s, b - (s - a)


def _renorm4(c0: float, c1: float, c2: float, c3: float):
    s, t4 = _qts(c3, 0.0)
    s, t3 = _qts(c2, s)
    s, t2 = _qts(c1, s)
    cur, t1 = _qts(c0, s)
    out = [0.0, 0.0, 0.0, 0.0]
    k = 0
    for v in (t1, t2, t3, t4):
        s, e = _qts(cur, v)
        if e != 0.0 and k < 3:
            out[k] = s
            cur = e
            k += 1
        else:
            cur = s
    out[k] = cur
    return tuple(out)


def _vec():
    from . import varith  # late import: varith imports this module
    return varith


class DoubleDouble:
    """Unevaluated sum of two binary64 values, non-overlapping."""

    __slots__ = ("comps",)

    def __init__(self, hi: float = 0.0, lo: float = 0.0):
        self.comps = _qts(float(hi), float(lo))

    @classmethod
    def _raw(cls, comps) -> "DoubleDouble":
        self = object.__new__(cls)
        self.comps = tuple(float(c) for c in comps)
        return self

    @property
    def hi(self) -> float:
        return self.comps[0]

    @property
    def lo(self) -> float:
        return self.comps[1]

    def __eq__(self, other):
        o = _coerce(other, 2)
        if o is None:
            return NotImplemented
        return self.comps == o

    def __hash__(self):
        return hash(self.comps)

    def __neg__(self):
        return DoubleDouble._raw((-self.comps[0], -self.comps[1]))

    def __abs__(self):
        return -self if self.comps[0] < 0.0 else self

    def __float__(self):
        return self.comps[0] + self.comps[1]

    def __repr__(self):
        return f"DoubleDouble({self.comps[0]!r}, {self.comps[1]!r})"

    def __str__(self):
        return render_decimal(self)

    # field arithmetic: GPU element-wise kernels
    def __add__(self, o): return _vec().scalar_op("add", self, o)
    def __radd__(self, o): return _vec().scalar_op("add", o, self)
    def __sub__(self, o): return _vec().scalar_op("sub", self, o)
    def __rsub__(self, o): return _vec().scalar_op("sub", o, self)
    def __mul__(self, o): return _vec().scalar_op("mul", self, o)
    def __rmul__(self, o): return _vec().scalar_op("mul", o, self)
    def __truediv__(self, o): return _vec().scalar_op("div", self, o)
    def __rtruediv__(self, o): return _vec().scalar_op("div", o, self)

    def __lt__(self, other):
        return (self - other).comps[0] < 0.0

    def __le__(self, other):
        return (self - other).comps[0] <= 0.0

    def __gt__(self, other):
        return not (self <= other)

    def __ge__(self, other):
        return not (self < other)

    def sqrt(self) -> "DoubleDouble":
        return _vec().scalar_sqrt(self)


class QuadDouble:
    """Unevaluated sum of four binary64 values, decreasing magnitude."""

    __slots__ = ("comps",)

    def __init__(self, c0: float = 0.0, c1: float = 0.0, c2: float = 0.0, c3: float = 0.0):
        self.comps = _renorm4(float(c0), float(c1), float(c2), float(c3))

    @classmethod
    def _raw(cls, comps) -> "QuadDouble":
        self = object.__new__(cls)
        self.comps = tuple(float(c) for c in comps)
        return self

    def __eq__(self, other):
        o = _coerce(other, 4)
        if o is None:
            return NotImplemented
        return self.comps == o

    def __hash__(self):
        return hash(self.comps)

    def __neg__(self):
        return QuadDouble._raw(tuple(-c for c in self.comps))

    def __abs__(self):
        return -self if self.comps[0] < 0.0 else self

    def __float__(self):
        return math.fsum(self.comps)

    def __repr__(self):
        return f"QuadDouble{self.comps!r}"

    def __str__(self):
        return render_decimal(self)

    def __add__(self, o): return _vec().scalar_op("add", self, o)
    def __radd__(self, o): return _vec().scalar_op("add", o, self)
    def __sub__(self, o): return _vec().scalar_op("sub", self, o)
    def __rsub__(self, o): return _vec().scalar_op("sub", o, self)
    def __mul__(self, o): return _vec().scalar_op("mul", self, o)
    def __rmul__(self, o): return _vec().scalar_op("mul", o, self)
    def __truediv__(self, o): return _vec().scalar_op("div", self, o)
    def __rtruediv__(self, o): return _vec().scalar_op("div", o, self)

    def __lt__(self, other):
        return (self - other).comps[0] < 0.0

    def __le__(self, other):
        return (self - other).comps[0] <= 0.0

    def __gt__(self, other):
        return not (self <= other)

    def __ge__(self, other):
        return not (self < other)

    def sqrt(self) -> "QuadDouble":
        return _vec().scalar_sqrt(self)


def _coerce(x, nc):
    """Components of a real scalar (own or reference type, or a number)."""
    if isinstance(x, (int, float)):
        return (float(x),) + (0.0,) * (nc - 1)
    comps = getattr(x, "comps", None)
    if comps is not None and len(comps) == nc:
        return tuple(comps)
    return None


class Complex:
    """Complex number over binary64, DoubleDouble, or QuadDouble parts."""

    __slots__ = ("re", "im")

    def __init__(self, re, im):
        self.re = re
        self.im = im

    def __eq__(self, other):
        if not isinstance(other, Complex) and not (hasattr(other, "re") and hasattr(other, "im")):
            return self.im == zero_like(self.im) and self.re == other
        return self.re == other.re and self.im == other.im

    def __hash__(self):
        return hash((self.re, self.im))

    def __neg__(self):
        return Complex(-self.re, -self.im)

    def conj(self) -> "Complex":
        return Complex(self.re, -self.im)

    def __repr__(self):
        return f"Complex({self.re!r}, {self.im!r})"

    def __str__(self):
        return f"({render_decimal(self.re)},{render_decimal(self.im)})"

    def __add__(self, o): return _vec().scalar_op("add", self, o)
    def __radd__(self, o): return _vec().scalar_op("add", o, self)
    def __sub__(self, o): return _vec().scalar_op("sub", self, o)
    def __rsub__(self, o): return _vec().scalar_op("sub", o, self)
    def __mul__(self, o): return _vec().scalar_op("mul", self, o)
    def __rmul__(self, o): return _vec().scalar_op("mul", o, self)
    def __truediv__(self, o): return _vec().scalar_op("div", self, o)
    def __rtruediv__(self, o): return _vec().scalar_op("div", o, self)

    def __abs__(self):
        return _vec().scalar_modulus(self)


def sqrt(x):
    """Square root dispatching on the scalar field (xprec.py:348-354)."""
    if isinstance(x, (DoubleDouble, QuadDouble)):
        return x.sqrt()
    if x < 0.0:
        raise DomainError("square root of negative value")
    return math.sqrt(x)


def conjugate(x):
    return x.conj() if isinstance(x, Complex) else x


def modulus(x):
    """Non-negative magnitude: |x| for real fields, complex modulus else."""
    return abs(x)


def zero_like(x):
    if isinstance(x, DoubleDouble) or (hasattr(x, "comps") and len(x.comps) == 2):
        return DoubleDouble._raw((0.0, 0.0))
    if isinstance(x, QuadDouble) or (hasattr(x, "comps") and len(x.comps) == 4):
        return QuadDouble._raw((0.0, 0.0, 0.0, 0.0))
    if isinstance(x, Complex) or (hasattr(x, "re") and hasattr(x, "im")):
        return Complex(zero_like(x.re), zero_like(x.im))
    return 0.0


def one_like(x):
    if isinstance(x, DoubleDouble):
        return DoubleDouble._raw((1.0, 0.0))
    if isinstance(x, QuadDouble):
        return QuadDouble._raw((1.0, 0.0, 0.0, 0.0))
    if isinstance(x, Complex):
        return Complex(one_like(x.re), zero_like(x.im))
    return 1.0


def is_zero(x) -> bool:
    comps = getattr(x, "comps", None)
    if comps is not None:
        return all(c == 0.0 for c in comps)
    if hasattr(x, "re") and hasattr(x, "im"):
        return is_zero(x.re) and is_zero(x.im)
    return x == 0.0


def to_float(x) -> float:
    return float(x)


# -- decimal rendering and parsing (host-side formatting, exact rationals) ----

def _digits(x) -> int:
    comps = getattr(x, "comps", None)
    return 17 if comps is None else (32 if len(comps) == 2 else 64)


def render_decimal(x) -> str:
    """Full-precision decimal text for a real scalar (xprec.py:406-420)."""
    if isinstance(x, (int, float)):
        return repr(float(x))
    fr = Fraction(0)
    for c in x.comps:
        fr += Fraction(c)
    if fr == 0:
        return "0.0"
    with localcontext() as ctx:
        ctx.prec = _digits(x)
        d = Decimal(fr.numerator) / Decimal(fr.denominator)
        return format(d, "E").replace("E", "e")


def _fraction_to_components(fr: Fraction, n: int) -> tuple:
    comps = []
    for _ in range(n):
        c = float(fr)
        comps.append(c)
        fr = fr - Fraction(c)
    return tuple(comps)


def parse_decimal(text: str, field: type):
    """Correctly rounded field value of a decimal literal (xprec.py:432-446)."""
    fr = Fraction(Decimal(text))
    if field is float:
        return float(fr)
    if field is DoubleDouble:
        return DoubleDouble._raw(_fraction_to_components(fr, 2))
    if field is QuadDouble:
        return QuadDouble._raw(_renorm4(*_fraction_to_components(fr, 4)))
    raise TypeError(f"unsupported field {field!r}")


@dataclass(frozen=True)
class PrecisionLevel:
    """Working precision tag: base in {'d','dd','qd'}, real or complex."""

    base: str
    cplx: bool = False

    _EPS = {"d": 2.0 ** -53, "dd": 2.0 ** -104, "qd": 2.0 ** -209}
    _NC = {"d": 1, "dd": 2, "qd": 4}

    def __post_init__(self):
        if self.base not in self._EPS:
            raise ValueError(f"unknown precision base {self.base!r}")

    @property
    def eps(self) -> float:
        return self._EPS[self.base]

    @property
    def ncomp(self) -> int:
        return self._NC[self.base]

    @property
    def field(self) -> type:
        return {"d": float, "dd": DoubleDouble, "qd": QuadDouble}[self.base]

    @property
    def name(self) -> str:
        return ("complex " if self.cplx else "real ") + self.base

    @property
    def cshape(self) -> tuple:
        return (2, self.ncomp) if self.cplx else (self.ncomp,)

    @property
    def es(self) -> int:
        return self.ncomp * (2 if self.cplx else 1)

    def from_float(self, v: float, im: float = 0.0):
        f = self.field
        x = float(v) if f is float else f(float(v))
        if not self.cplx:
            if im != 0.0:
                raise ValueError("imaginary part in a real-precision context")
            return x
        y = float(im) if f is float else f(float(im))
        return Complex(x, y)

    def from_int(self, v: int):
        return self.from_float(float(v))

    def from_fraction(self, fr: Fraction):
        f = self.field
        if f is float:
            x = float(fr)
        elif f is DoubleDouble:
            x = DoubleDouble._raw(_fraction_to_components(fr, 2))
        else:
            x = QuadDouble._raw(_renorm4(*_fraction_to_components(fr, 4)))
        return Complex(x, self.real_zero()) if self.cplx else x

    def real_zero(self):
        f = self.field
        return 0.0 if f is float else f()

    def zero(self):
        return self.from_float(0.0)

    def one(self):
        return self.from_float(1.0)

    def parse(self, text: str):
        """Parse "1.25" or, for complex levels, "(re,im)"."""
        text = text.strip()
        if text.startswith("("):
            if not self.cplx:
                raise ValueError("complex literal in a real-precision context")
            body = text[1:text.index(")")]
            re_s, im_s = body.split(",")
            return Complex(parse_decimal(re_s, self.field), parse_decimal(im_s, self.field))
        x = parse_decimal(text, self.field)
        return Complex(x, self.real_zero()) if self.cplx else x

    def render(self, x) -> str:
        if hasattr(x, "re") and hasattr(x, "im"):
            return f"({render_decimal(x.re)},{render_decimal(x.im)})"
        return render_decimal(x)

    def to_components(self, x) -> list:
        """Flat binary64 components: re components, then im for complex.

        Accepts this package's scalars, the reference's scalars, and plain
        numbers (padded with zero components)."""
        nc = self.ncomp

        def comps(v):
            c = _coerce(v, nc)
            if c is None:
                raise TypeError(f"cannot convert {v!r} to a {self.name} value")
            return list(c)
        if self.cplx:
            if hasattr(x, "re") and hasattr(x, "im"):
                return comps(x.re) + comps(x.im)
            return comps(x) + [0.0] * nc
        if hasattr(x, "re") and hasattr(x, "im"):
            raise TypeError("complex value in a real-precision context")
        return comps(x)

    def from_components(self, comps):
        f = self.field
        nc = self.ncomp

        def build(c):
            if f is float:
                return float(c[0])
            if f is DoubleDouble:
                return DoubleDouble._raw((c[0], c[1]))
            return QuadDouble._raw(tuple(c))
        if self.cplx:
            return Complex(build(comps[:nc]), build(comps[nc:]))
        return build(comps)

    # -- arrays ----------------------------------------------------------------

    def to_planes(self, values) -> np.ndarray:
        """Sequence of scalars -> component planes (cshape + (len,))."""
        flat = np.array([self.to_components(v) for v in values], dtype=np.float64).reshape(-1, self.es)
        return np.ascontiguousarray(flat.T.reshape(self.cshape + (flat.shape[0],)))

    def from_planes(self, arr) -> list:
        """Component planes with one trailing data axis -> list of scalars."""
        arr = np.asarray(arr)
        flat = arr.reshape(self.es, -1)
        cols = flat.T.tolist()
        return [self.from_components(c) for c in cols]


def precision_level(base: str, cplx: bool) -> PrecisionLevel:
    return PrecisionLevel(base.lower(), cplx)


def level_of(x) -> PrecisionLevel:
    """Infer the precision level of a scalar (own or reference types)."""
    if hasattr(x, "re") and hasattr(x, "im"):
        return PrecisionLevel(level_of(x.re).base, True)
    comps = getattr(x, "comps", None)
    if comps is None:
        return PrecisionLevel("d", False)
    return PrecisionLevel("dd" if len(comps) == 2 else "qd", False)
