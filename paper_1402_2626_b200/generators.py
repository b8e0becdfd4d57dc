"""Benchmark systems and seeded inputs (mirror of polynewt.bench, plus the
SURVEY 8(d) random sparse family F(n, T, k) generated natively).

Inputs are produced on the host once and shipped as component planes; the
points use Python's ``random.Random`` exactly like the reference
(bench.py:72-95), so both paths see identical values.
"""

from __future__ import annotations

import math
import random
from fractions import Fraction

import numpy as np

from . import _lib
from .polyrep import Monomial, PackedSystem, PolySystem
from .xprec import PrecisionLevel


def random_sparse_system(n: int, T: int, k: int, level: PrecisionLevel, seed: int, maxexp: int = 1,
                         m: int | None = None, kmin: int | None = None) -> PackedSystem:
    """F(n, T, k, level, seed, maxexp, m): m polynomials of T monomials, each
    a product of k distinct variables with exponents in [1, maxexp] and
    coefficient parts in +-[0.5, 2).  ``kmin`` < k gives the C2
    "mixed" variant (variable count per monomial uniform in [kmin, k]).
    Built by the C ABI's splitmix64 generator in generation order (not
    canonical)."""
    m = n if m is None else m
    kmin = k if kmin is None else kmin
    M = m * T
    nnz = M * k
    poly_ptr = np.empty(m + 1, np.int32)
    mon_ptr = np.empty(M + 1, np.int32)
    var_idx = np.empty(nnz, np.int32)
    exps = np.empty(nnz, np.int32)
    re = np.empty(M)
    im = np.empty(M) if level.cplx else None
    rc = _lib.load().pn_generate_random_system(m, n, T, kmin, k, maxexp, seed, _lib.ptr(poly_ptr),
                                               _lib.ptr(mon_ptr), _lib.ptr(var_idx), _lib.ptr(exps), _lib.ptr(re),
                                               _lib.ptr(im))
    _lib.check(rc)
    if kmin < k:
        var_idx = var_idx[:mon_ptr[M]].copy()
        exps = exps[:mon_ptr[M]].copy()
    coeffs = np.zeros(level.cshape + (M,))
    # level.from_float(v): DoubleDouble(v) = (v + 0.0, 0.0); QuadDouble alike
    if level.cplx:
        coeffs[0, 0] = re + 0.0
        coeffs[1, 0] = im + 0.0
    else:
        coeffs[0] = re + 0.0
    return PackedSystem(level, n, poly_ptr, mon_ptr, var_idx, exps, coeffs)


def random_point(n: int, seed: int, level: PrecisionLevel) -> list:
    """n random values with magnitudes in [0.5, 2) (bench.py:84-95)."""
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        re = rng.uniform(0.5, 2.0) * rng.choice((-1.0, 1.0))
        if level.cplx:
            out.append(level.from_float(re, rng.uniform(0.5, 2.0) * rng.choice((-1.0, 1.0))))
        else:
            out.append(level.from_float(re))
    return out


def random_unit_point(n: int, seed: int, level: PrecisionLevel) -> list:
    """n random unit-modulus complex values (bench.py:72-81)."""
    if not level.cplx:
        raise ValueError("unit-circle points need a complex level")
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        theta = rng.uniform(0.0, 2.0 * math.pi)
        out.append(level.from_float(math.cos(theta), math.sin(theta)))
    return out


def cyclic_n_roots(n: int, level: PrecisionLevel) -> PolySystem:
    """Cyclic n-roots system (bench.py:51-69)."""
    if n < 2:
        raise ValueError("need n >= 2")
    one = level.one()
    polys = []
    for i in range(1, n):
        terms = []
        for j in range(n):
            vars_ = sorted((j + k) % n for k in range(i))
            terms.append(Monomial(one, tuple((v, 1) for v in vars_)))
        polys.append(terms)
    polys.append([Monomial(one, tuple((v, 1) for v in range(n))), Monomial(-one, ())])
    return PolySystem(n, polys)


def chandrasekhar_system(n: int, level: PrecisionLevel, c: Fraction = Fraction(33, 64)) -> PolySystem:
    """Discretized H-equation (bench.py:19-43); the weights i/(i+j) and
    -(c*w) are formed in working precision on the GPU."""
    from .varith import VecContext
    if n < 1:
        raise ValueError("need n >= 1")
    ctx = VecContext(level)
    c_val = level.from_fraction(c)
    two_n = level.from_int(2 * n)
    num = level.to_planes([level.from_int(i) for i in range(1, n + 1) for _ in range(n)])
    den = level.to_planes([level.from_int(i + j) for i in range(1, n + 1) for j in range(n)])
    w = ctx.div(num, den)
    cw = ctx.mul(np.repeat(level.to_planes([c_val]), n * n, axis=-1), w)
    coeffs = level.from_planes(-cw)
    polys = []
    for i in range(1, n + 1):
        terms = [Monomial(two_n, ((i - 1, 1),)), Monomial(-two_n, ())]
        for j in range(n):
            coeff = coeffs[(i - 1) * n + j]
            exps = ((i - 1, 2),) if j == i - 1 else tuple(sorted(((i - 1, 1), (j, 1))))
            terms.append(Monomial(coeff, exps))
        polys.append(terms)
    return PolySystem(n, polys)


def chandrasekhar_start(n: int, level: PrecisionLevel) -> list:
    return [level.one() for _ in range(n)]


# ---------------------------------------------------------------------------
# The same families packed straight into CSR with numpy (paper scale: cyclic
# 512-roots has 67 M support entries, Chandrasekhar n = 4096 has 16.8 M
# monomials -- far beyond Monomial objects).  Generation order and values are
# identical to PackedSystem.from_system of the builders above.

def _int_planes(level: PrecisionLevel, values) -> np.ndarray:
    """level.from_int(v) for exact integers v: (float(v), 0, ...) planes."""
    values = np.asarray(values, dtype=np.float64)
    out = np.zeros(level.cshape + values.shape)
    out.reshape((level.es,) + values.shape)[0] = values
    return out


def cyclic_packed(n: int, level: PrecisionLevel) -> PackedSystem:
    """cyclic_n_roots(n, level) as a PackedSystem (bench.py:51-69): equation
    i < n holds the n cyclic products of i consecutive variables (sorted),
    the last one the full product and the constant -1."""
    if n < 2:
        raise ValueError("need n >= 2")
    ks = [i for i in range(1, n) for _ in range(n)] + [n, 0]
    var_parts = []
    for i in range(1, n):
        win = (np.arange(n)[:, None] + np.arange(i)[None, :]) % n
        var_parts.append(np.sort(win, axis=1).reshape(-1))
    var_parts.append(np.arange(n))
    var_idx = np.concatenate(var_parts).astype(np.int32)
    mon_ptr = np.concatenate(([0], np.cumsum(ks))).astype(np.int32)
    poly_ptr = np.concatenate((np.arange(0, n * (n - 1) + 1, n), [n * (n - 1) + 2])).astype(np.int32)
    M = len(ks)
    coeffs = _int_planes(level, np.ones(M))
    coeffs[..., M - 1] = -coeffs[..., M - 1]  # -one: every component negated
    return PackedSystem(level, n, poly_ptr, mon_ptr, var_idx, np.ones(len(var_idx), np.int32),
                        np.ascontiguousarray(coeffs))


def chandrasekhar_packed(n: int, level: PrecisionLevel, c: Fraction = Fraction(33, 64)) -> PackedSystem:
    """chandrasekhar_system(n, level, c) as a PackedSystem (bench.py:19-43).
    Equation i (1-based): 2n x_{i-1}, -2n, then for j = 0..n-1 the term
    -(c * i/(i+j)) x_{i-1} x_j (x_{i-1}^2 when j = i-1); the weights and
    coefficients are formed in working precision on the GPU (VecContext,
    the reference's operand order)."""
    from .varith import VecContext
    if n < 1:
        raise ValueError("need n >= 1")
    ctx = VecContext(level)
    i1 = np.repeat(np.arange(1, n + 1), n)
    j0 = np.tile(np.arange(n), n)
    w = ctx.div(_int_planes(level, i1), _int_planes(level, i1 + j0))
    cw = ctx.mul(np.repeat(level.to_planes([level.from_fraction(c)]), n * n, axis=-1), w)
    T = n + 2
    M = n * T
    coeffs = np.empty(level.cshape + (n, T))
    two_n = _int_planes(level, [2 * n])[..., 0]
    coeffs[..., 0] = two_n[..., None]
    coeffs[..., 1] = -two_n[..., None]
    coeffs[..., 2:] = (-cw).reshape(level.cshape + (n, n))
    rows = np.arange(n)
    ks = np.full((n, T), 2, np.int64)
    ks[:, 1] = 0
    ks[:, 0] = 1
    ks[rows, 2 + rows] = 1  # the square term x_{i-1}^2
    mon_ptr = np.concatenate(([0], np.cumsum(ks.reshape(-1)))).astype(np.int32)
    var_idx = np.empty(int(mon_ptr[-1]), np.int32)
    exps = np.ones(int(mon_ptr[-1]), np.int32)
    starts = mon_ptr[:-1].reshape(n, T)
    var_idx[starts[:, 0]] = rows
    jj = np.broadcast_to(np.arange(n), (n, n))
    ii = np.broadcast_to(rows[:, None], (n, n))
    s = starts[:, 2:]
    off = jj != ii
    var_idx[s[off]] = np.minimum(ii, jj)[off]
    var_idx[s[off] + 1] = np.maximum(ii, jj)[off]
    var_idx[s[~off]] = ii[~off]
    exps[s[~off]] = 2
    poly_ptr = (np.arange(n + 1) * T).astype(np.int32)
    return PackedSystem(level, n, poly_ptr, mon_ptr, var_idx, exps,
                        np.ascontiguousarray(coeffs.reshape(level.cshape + (M,))))


def random_stress_products(m: int, n: int, seed: int, level: PrecisionLevel) -> list:
    """m random coefficients on the full degree-n product (bench.py:98-110)."""
    rng = random.Random(seed)
    exps = tuple((v, 1) for v in range(n))
    out = []
    for _ in range(m):
        if level.cplx:
            coeff = level.from_float(rng.uniform(0.5, 2.0), rng.uniform(0.5, 2.0))
        else:
            coeff = level.from_float(rng.uniform(0.5, 2.0))
        out.append(Monomial(coeff, exps))
    return out
