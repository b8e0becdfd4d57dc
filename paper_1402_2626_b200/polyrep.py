"""Sparse distributed polynomial systems (mirror of polynewt.polyrep).

``Monomial`` / ``PolySystem`` keep the reference's validation and canonical
order (polyrep.py:23-107).  ``PackedSystem`` is the flat CSR form handed to
the C ABI (``pn_system_create``): supports in generation order, exponents,
and the coefficients as component planes.  Large synthetic systems are
generated directly in packed form (``generators.random_sparse_system``), so
no per-monomial Python objects are needed at benchmark scale.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

from .xprec import PrecisionLevel, is_zero, level_of


@dataclass(frozen=True)
class Monomial:
    """coeff * prod x_i^d_i with sorted variable indices and d_i >= 1."""

    coeff: object
    exponents: tuple  # ((var_index, d), ...) with strictly increasing indices

    def __post_init__(self):
        if is_zero(self.coeff):
            raise ValueError("monomials must carry a nonzero coefficient")
        prev = -1
        for var, d in self.exponents:
            if var <= prev:
                raise ValueError("variable indices must be strictly increasing")
            if d < 1:
                raise ValueError("listed exponents must be >= 1")
            prev = var

    def degree(self) -> int:
        return sum(d for _, d in self.exponents)

    def exponent_key(self, n_vars: int) -> tuple:
        dense = [0] * n_vars
        for var, d in self.exponents:
            dense[var] = d
        return tuple(dense)

    def sparse_key(self) -> tuple:
        """Sort key equal in order to exponent_key: compares like
        the dense vector but costs O(k) instead of O(n_vars)."""
        return tuple((-v, d) for v, d in self.exponents)


@dataclass(frozen=True)
class MonomialDecomposition:
    """Split of an exponent vector into distinct variables x common factor."""

    distinct_vars: tuple
    common_factor: tuple


def decompose(mon) -> MonomialDecomposition:
    distinct = tuple(var for var, _ in mon.exponents)
    common = tuple((var, d - 1) for var, d in mon.exponents if d >= 2)
    return MonomialDecomposition(distinct, common)


def recompose(dec: MonomialDecomposition) -> tuple:
    extra = dict(dec.common_factor)
    return tuple((var, 1 + extra.get(var, 0)) for var in dec.distinct_vars)


@dataclass
class PolySystem:
    """m polynomials in n_vars variables, each a list of monomials."""

    n_vars: int
    polys: list

    def __post_init__(self):
        for poly in self.polys:
            for mon in poly:
                for var, _ in mon.exponents:
                    if not 0 <= var < self.n_vars:
                        raise ValueError(f"variable index {var} out of range for n_vars={self.n_vars}")

    @property
    def n_eqs(self) -> int:
        return len(self.polys)

    def monomial_count(self) -> int:
        return sum(len(p) for p in self.polys)

    def max_exponent(self) -> dict:
        out = {}
        for poly in self.polys:
            for mon in poly:
                for var, d in mon.exponents:
                    if d > out.get(var, 0):
                        out[var] = d
        return out

    def canonicalized(self) -> "PolySystem":
        """Monomials of each polynomial in lexicographic exponent order
        (stable, so duplicates keep their order; polyrep.py:103-107)."""
        polys = [sorted(p, key=lambda m: tuple((-v, d) for v, d in m.exponents)) for p in self.polys]
        return PolySystem(self.n_vars, polys)


def system_level(system) -> PrecisionLevel:
    """Precision level of a system, inferred from its first coefficient."""
    for poly in system.polys:
        for mon in poly:
            return level_of(mon.coeff)
    raise ValueError("cannot infer the precision of an empty system")


@dataclass
class PackedSystem:
    """CSR form of a system for the C ABI (generation order)."""

    level: PrecisionLevel
    n_vars: int
    poly_ptr: np.ndarray   # int32 (m+1)
    mon_ptr: np.ndarray    # int32 (M+1)
    var_idx: np.ndarray    # int32 (nnz)
    exps: np.ndarray       # int32 (nnz)
    coeffs: np.ndarray     # float64 planes cshape + (M,)
    canonical: bool = False
    source: object = field(default=None, repr=False)  # the PolySystem, if any

    @property
    def n_eqs(self) -> int:
        return len(self.poly_ptr) - 1

    @property
    def monomials(self) -> int:
        return len(self.mon_ptr) - 1

    @property
    def support(self) -> int:
        return len(self.var_idx)

    @classmethod
    def from_system(cls, system, level: PrecisionLevel | None = None) -> "PackedSystem":
        level = level or system_level(system)
        poly_ptr = [0]
        mon_ptr = [0]
        var_idx, exps, comps = [], [], []
        for poly in system.polys:
            for mon in poly:
                for v, d in mon.exponents:
                    var_idx.append(v)
                    exps.append(d)
                mon_ptr.append(len(var_idx))
                comps.append(level.to_components(mon.coeff))
            poly_ptr.append(len(mon_ptr) - 1)
        M = len(comps)
        coeffs = np.asarray(comps, dtype=np.float64).reshape(M, level.es).T.reshape(level.cshape + (M,))
        return cls(level, system.n_vars, np.asarray(poly_ptr, np.int32), np.asarray(mon_ptr, np.int32),
                   np.asarray(var_idx, np.int32), np.asarray(exps, np.int32), np.ascontiguousarray(coeffs),
                   source=system)

    def to_system(self) -> PolySystem:
        """Rebuild Monomial objects (small systems only)."""
        polys = []
        coef = self.coeffs.reshape(self.level.es, -1)
        for i in range(self.n_eqs):
            terms = []
            for c in range(self.poly_ptr[i], self.poly_ptr[i + 1]):
                a, b = self.mon_ptr[c], self.mon_ptr[c + 1]
                exps = tuple((int(v), int(d)) for v, d in zip(self.var_idx[a:b], self.exps[a:b]))
                terms.append(Monomial(self.level.from_components(coef[:, c].tolist()), exps))
            polys.append(terms)
        return PolySystem(self.n_vars, polys)


@dataclass
class PowerTable:
    """Per evaluation point: powers[var][d] = x_var^d (polyrep.py:110-117)."""

    powers: dict = field(default_factory=dict)

    def get(self, var: int, d: int):
        return self.powers[var][d]


# ---------------------------------------------------------------------------
# System text format (polyrep.py:140-304).  Line 1 is "m n"; then m
# polynomials, each a '+'/'-'-separated list of terms closed by ';'.  A term
# is a '*'-product of at most one coefficient ("2.5", ".5", "(re,im)") and
# variable factors "x<i>" / "x<i>^<d>" (repeated variables add exponents;
# the coefficient defaults to one).  Errors carry the 1-based line and column
# of the offending character, exactly as the reference reports them.

class SystemParseError(ValueError):
    """Malformed system text (polyrep.py:16-20)."""

    def __init__(self, line: int, col: int, message: str):
        super().__init__(f"line {line}, column {col}: {message}")
        self.line = line
        self.col = col


# factor grammar: a variable, a parenthesised complex literal, or a number
# (digits, '.', '_', exponent letters and signs run greedily, so "3-x0" is
# one malformed number -- the reference's tokenizer behaves the same way)
_VAR_RE = re.compile(r"x(\d+)(?:\^(\d+))?")
_CPLX_RE = re.compile(r"\([^()]*\)")
_NUM_RE = re.compile(r"\.?[0-9][0-9_.eE+-]*")
_SIGNS = "+-−"


def _render_term(level: PrecisionLevel, coeff, exponents) -> str:
    return level.render(coeff) + "".join(f"*x{v}" + (f"^{d}" if d > 1 else "") for v, d in exponents)


def serialize_system(system: PolySystem, level: PrecisionLevel) -> str:
    """Text of the canonicalised system (polyrep.py:150-166).  Real levels
    write negative non-leading coefficients as " - |c|"."""
    out = [f"{system.n_eqs} {system.n_vars}"]
    for poly in system.canonicalized().polys:
        text = ""
        for i, mon in enumerate(poly):
            coeff = mon.coeff
            if i == 0:
                sep = ""
            elif not level.cplx and level.to_components(coeff)[0] < 0.0:
                sep, coeff = " - ", -coeff  # the sign of a normalised value is its leading component's
            else:
                sep = " + "
            text += sep + _render_term(level, coeff, mon.exponents)
        out.append(text + ";")
    return "\n".join(out) + "\n"


class _Text:
    """Cursor over the system text with reference-compatible error positions."""

    def __init__(self, text: str):
        self.s = text
        self.i = 0

    def fail(self, message: str, at: int | None = None):
        p = self.i if at is None else at
        line = self.s.count("\n", 0, p) + 1
        col = p - self.s.rfind("\n", 0, p)
        raise SystemParseError(line, col, message)

    def next_char(self) -> str:
        """First non-blank character from the cursor ('' at the end); the
        cursor moves past the blanks."""
        s, i = self.s, self.i
        while i < len(s) and s[i].isspace():
            i += 1
        self.i = i
        return s[i] if i < len(s) else ""


def parse_system(text: str, level: PrecisionLevel) -> PolySystem:
    """Inverse of serialize_system for any spacing (polyrep.py:190-207)."""
    cur = _Text(text)
    head = text.split("\n", 1)[0].split()
    if len(head) != 2:
        cur.fail("expected header line 'm n'")
    try:
        m, n_vars = int(head[0]), int(head[1])
    except ValueError:
        cur.fail("expected integer equation and variable counts")
    nl = text.find("\n")
    cur.i = len(text) if nl < 0 else nl + 1
    polys = [_read_poly(cur, level, n_vars) for _ in range(m)]
    if cur.next_char():
        cur.fail("trailing input after the last polynomial")
    return PolySystem(n_vars, polys)


def _read_poly(cur: _Text, level: PrecisionLevel, n_vars: int) -> list:
    """Terms up to ';' (polyrep.py:210-238)."""
    terms = []
    sign = None      # pending sign character, not yet followed by a term
    started = False  # any sign or term seen
    while True:
        ch = cur.next_char()
        if not ch:
            cur.fail("unexpected end of input, expected ';'")
        if ch == ";":
            if sign is not None:
                cur.fail("expected a term after the sign")
            cur.i += 1
            if not started:
                cur.fail("empty polynomial")
            return terms
        if ch in _SIGNS:
            if sign is not None:
                cur.fail("expected a term after the sign")
            cur.i += 1
            sign, started = ch, True
            continue
        if terms and sign is None:
            cur.fail("expected '+', '-' or ';' between terms")
        terms.append(_read_term(cur, level, n_vars, negate=sign is not None and sign != "+"))
        sign, started = None, True


def _read_term(cur: _Text, level: PrecisionLevel, n_vars: int, negate: bool):
    """One '*'-product of factors (polyrep.py:241-294)."""
    coeff = None
    powers: dict = {}
    while True:
        cur.next_char()
        at, s = cur.i, cur.s
        mv = _VAR_RE.match(s, at)
        if mv:
            idx = int(mv.group(1))
            if not 0 <= idx < n_vars:
                cur.fail(f"variable index {idx} out of range (n={n_vars})", at)
            d = int(mv.group(2)) if mv.group(2) else 1
            if d < 1:
                cur.fail("exponents must be >= 1", at)
            powers[idx] = powers.get(idx, 0) + d
            end = mv.end()
        else:
            mc = _CPLX_RE.match(s, at)
            mn = None if mc else _NUM_RE.match(s, at)
            tok = mc or mn
            if tok is None:
                cur.fail("expected a coefficient or variable factor")
            if coeff is not None:
                cur.fail("duplicate coefficient", at)
            try:
                coeff = level.parse(tok.group(0))
            except Exception:
                cur.fail("malformed complex coefficient" if mc else "malformed numeric coefficient", at)
            end = tok.end()
        cur.i = end
        if cur.next_char() != "*":
            break
        cur.i += 1
    if cur.next_char() == "^":  # "x0^": the exponent digits are missing
        cur.fail("malformed exponent")
    if coeff is None:
        coeff = level.one()
    if negate:
        coeff = -coeff
    try:
        return Monomial(coeff, tuple(sorted(powers.items())))
    except ValueError as exc:
        cur.fail(str(exc))


def parse_system_packed(text: str, level: PrecisionLevel) -> PackedSystem:
    """The text format straight into a PackedSystem (generation order) by
    the native scanner (pn_parse_system: CSR and exact coefficient
    components without Monomial objects -- for 10^6-monomial files).  Input
    the native scanner refuses (malformed text, or forms only Python's
    Decimal / str methods accept) goes through parse_system, so errors are
    the reference's SystemParseError with its line and column."""
    import ctypes

    from . import _lib
    raw = text.encode("utf-8")
    h = ctypes.c_void_p()
    lib = _lib.load()
    rc = lib.pn_parse_system(raw, len(raw), level.ncomp, int(level.cplx), ctypes.byref(h))
    if rc != 0:
        return PackedSystem.from_system(parse_system(text, level), level)
    try:
        m, n = ctypes.c_int32(), ctypes.c_int32()
        M, nnz = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.pn_text_system_sizes(h, ctypes.byref(m), ctypes.byref(n), ctypes.byref(M), ctypes.byref(nnz)))
        poly_ptr = np.empty(m.value + 1, np.int32)
        mon_ptr = np.empty(M.value + 1, np.int32)
        var_idx = np.empty(nnz.value, np.int32)
        exps = np.empty(nnz.value, np.int32)
        coeffs = np.empty(level.cshape + (M.value,))
        _lib.check(lib.pn_text_system_export(h, _lib.ptr(poly_ptr), _lib.ptr(mon_ptr), _lib.ptr(var_idx),
                                             _lib.ptr(exps), _lib.ptr(coeffs)))
    finally:
        lib.pn_text_system_free(h)
    return PackedSystem(level, n.value, poly_ptr, mon_ptr, var_idx, exps, coeffs)

