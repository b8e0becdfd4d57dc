"""Sparse distributed polynomial systems (mirror of polynewt.polyrep).

``Monomial`` / ``PolySystem`` keep the reference's validation and canonical
order (polyrep.py:23-107).  ``PackedSystem`` is the flat CSR form handed to
the C ABI (``pn_system_create``): supports in generation order, exponents,
and the coefficients as component planes.  Large synthetic systems are
generated directly in packed form (``generators.random_sparse_system``), so
no per-monomial Python objects are needed at benchmark scale.
"""

from __future__ import annotations

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
