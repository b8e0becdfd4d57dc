"""TEST INFRASTRUCTURE ONLY -- Python driver of the C oracle (pn_oracle.c).

This module is the parity checker and the CPU baseline.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it; the product package never does.

It restates the reference's host-side steps that are not arithmetic:
canonical monomial order (polyrep.py:103-107, literally with the dense
exponent key) and the packing of a system into CSR; the arithmetic itself is
in pn_oracle.c.  Arrays cross this interface in the reference's component
plane layout (varith.py:3-8): complex (2, nc, ...), real (nc, ...).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libpn_oracle.so")

_lib = None


def build():
    subprocess.run(["make", "-C", HERE], check=True, capture_output=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i, l = ctypes.c_void_p, ctypes.c_int, ctypes.c_long
        L.or_vec_op.argtypes = [i, i, i, l, vp, vp, vp]
        L.or_tree_sum.argtypes = [i, i, l, vp, vp]
        L.or_evaluate.argtypes = [i, i, i, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, i]
        L.or_mgs_qr.argtypes = [i, i, i, i, vp, vp, vp, vp, i]
        L.or_back_substitute.argtypes = [i, i, i, vp, vp, vp]
        L.or_least_squares.argtypes = [i, i, i, i, vp, vp, vp, vp, vp, vp, i]
        L.or_newton_step.argtypes = [i, i, i, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i]
        L.or_generate_random_system.argtypes = [i, i, i, i, i, i, ctypes.c_uint64, vp, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


@dataclass(frozen=True)
class Level:
    base: str
    cplx: bool

    @property
    def nc(self) -> int:
        return {"d": 1, "dd": 2, "qd": 4}[self.base]

    @property
    def es(self) -> int:
        return self.nc * (2 if self.cplx else 1)

    @property
    def cshape(self) -> tuple:
        return (2, self.nc) if self.cplx else (self.nc,)

    @property
    def eps(self) -> float:
        return {"d": 2.0 ** -53, "dd": 2.0 ** -104, "qd": 2.0 ** -209}[self.base]


def as_level(level) -> Level:
    return Level(level.base, bool(level.cplx))


def to_aos(planes: np.ndarray, level: Level) -> np.ndarray:
    """planes cshape + S  ->  S + (es,) contiguous"""
    k = len(level.cshape)
    a = np.asarray(planes, dtype=np.float64)
    S = a.shape[k:]
    return np.ascontiguousarray(np.moveaxis(a.reshape((level.es,) + S), 0, -1))


def to_planes(aos: np.ndarray, level: Level) -> np.ndarray:
    a = np.asarray(aos)
    S = a.shape[:-1]
    return np.ascontiguousarray(np.moveaxis(a, -1, 0).reshape(level.cshape + S))


# -- systems -------------------------------------------------------------------

@dataclass
class CSR:
    """A system in CSR (generation order), the oracle's input format."""

    n_vars: int
    poly_ptr: np.ndarray
    mon_ptr: np.ndarray
    var_idx: np.ndarray
    exps: np.ndarray
    coeffs: np.ndarray  # planes cshape + (M,)

    @classmethod
    def from_packed(cls, p) -> "CSR":
        return cls(p.n_vars, np.asarray(p.poly_ptr, np.int32), np.asarray(p.mon_ptr, np.int32),
                   np.asarray(p.var_idx, np.int32), np.asarray(p.exps, np.int32), np.asarray(p.coeffs))

    @classmethod
    def from_polys(cls, n_vars, polys, level) -> "CSR":
        """polys: list of lists of (coeff_components(es), ((var, d), ...))"""
        pp, mp, vi, ex, co = [0], [0], [], [], []
        for poly in polys:
            for comps, exps in poly:
                for v, d in exps:
                    vi.append(v)
                    ex.append(d)
                mp.append(len(vi))
                co.append(list(comps))
            pp.append(len(mp) - 1)
        M = len(co)
        coeffs = np.asarray(co, np.float64).reshape(M, level.es)
        return cls(n_vars, np.asarray(pp, np.int32), np.asarray(mp, np.int32), np.asarray(vi, np.int32),
                   np.asarray(ex, np.int32), to_planes(coeffs, level))

    def canonical_perm(self) -> np.ndarray:
        """Canonical order (polyrep.py:103-107): per polynomial, a stable
        sort by the dense exponent vector.  Small systems use the dense key
        literally; large ones the equivalent sparse key."""
        M = len(self.mon_ptr) - 1
        perm = np.arange(M, dtype=np.int64)
        dense = self.n_vars * M <= 4_000_000
        for i in range(len(self.poly_ptr) - 1):
            lo, hi = int(self.poly_ptr[i]), int(self.poly_ptr[i + 1])

            def key(c):
                a, b = self.mon_ptr[c], self.mon_ptr[c + 1]
                vs, ds = self.var_idx[a:b].tolist(), self.exps[a:b].tolist()
                if dense:
                    d = [0] * self.n_vars
                    for v, e in zip(vs, ds):
                        d[v] = e
                    return tuple(d)
                return tuple((-v, e) for v, e in zip(vs, ds))
            perm[lo:hi] = sorted(range(lo, hi), key=key)
        return perm

    def canonical(self) -> "CSR":
        perm = self.canonical_perm()
        mp = [0]
        vi, ex = [], []
        for c in perm:
            a, b = self.mon_ptr[c], self.mon_ptr[c + 1]
            vi.append(self.var_idx[a:b])
            ex.append(self.exps[a:b])
            mp.append(mp[-1] + (b - a))
        cat = (lambda xs: np.concatenate(xs).astype(np.int32)) if vi else (lambda xs: np.zeros(0, np.int32))
        return CSR(self.n_vars, self.poly_ptr.copy(), np.asarray(mp, np.int32), cat(vi), cat(ex),
                   np.ascontiguousarray(self.coeffs[..., perm]))

    def rows(self, rows) -> "CSR":
        """Sub-system of the given polynomial rows (a row depends only on its
        own polynomial and x, evaldiff.py:252-265, so row sampling is exact)."""
        pp, mp, vi, ex, cols = [0], [0], [], [], []
        for i in rows:
            for c in range(self.poly_ptr[i], self.poly_ptr[i + 1]):
                a, b = self.mon_ptr[c], self.mon_ptr[c + 1]
                vi.append(self.var_idx[a:b])
                ex.append(self.exps[a:b])
                mp.append(mp[-1] + (b - a))
                cols.append(c)
            pp.append(len(mp) - 1)
        cat = (lambda xs: np.concatenate(xs).astype(np.int32)) if vi else (lambda xs: np.zeros(0, np.int32))
        return CSR(self.n_vars, np.asarray(pp, np.int32), np.asarray(mp, np.int32), cat(vi), cat(ex),
                   np.ascontiguousarray(self.coeffs[..., cols]))


def random_sparse_csr(n: int, T: int, k: int, level: Level, seed: int, maxexp: int = 1, m=None,
                      kmin=None) -> CSR:
    """F(n, T, k, level, seed, maxexp, m[, kmin]) from the
    oracle's own generator (or_generate_random_system), in generation order;
    coefficients as level.from_float(re, im) planes.  Same arrays as the
    product's random_sparse_system, without loading the product library."""
    m = n if m is None else m
    kmin = k if kmin is None else kmin
    M = m * T
    poly_ptr = np.empty(m + 1, np.int32)
    mon_ptr = np.empty(M + 1, np.int32)
    var_idx = np.empty(M * k, np.int32)
    exps = np.empty(M * k, np.int32)
    re = np.empty(M)
    im = np.empty(M) if level.cplx else None
    rc = lib().or_generate_random_system(m, n, T, kmin, k, maxexp, seed, _p(poly_ptr), _p(mon_ptr), _p(var_idx),
                                         _p(exps), _p(re), _p(im))
    if rc:
        raise ValueError("or_generate_random_system: bad arguments")
    nnz = int(mon_ptr[M])
    coeffs = np.zeros(level.cshape + (M,))
    if level.cplx:
        coeffs[0, 0] = re + 0.0
        coeffs[1, 0] = im + 0.0
    else:
        coeffs[0] = re + 0.0
    return CSR(n, poly_ptr, mon_ptr, var_idx[:nnz].copy(), exps[:nnz].copy(), coeffs)


# -- entry points ----------------------------------------------------------------

OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "abs2": 4, "sqrt": 5, "conj": 6}


def vec_op(level: Level, op: str, a, b=None):
    code = OPS[op]
    a_real = op == "sqrt"
    out_real = op in ("abs2", "sqrt")
    la = Level(level.base, False) if a_real else level
    A = to_aos(a, la)
    n = A.size // la.es
    B = to_aos(b, level) if b is not None else None
    lo = Level(level.base, False) if out_real else level
    out = np.empty(A.shape[:-1] + (lo.es,))
    rc = lib().or_vec_op(level.nc, int(level.cplx and not a_real), code, n, _p(A), _p(B), _p(out))
    assert rc == 0
    return to_planes(out, lo)


def tree_sum(level: Level, a) -> np.ndarray:
    A = to_aos(a, level)
    n = A.shape[0]
    out = np.empty((level.es,))
    lib().or_tree_sum(level.nc, int(level.cplx), n, _p(A), _p(out))
    return to_planes(out.reshape(1, -1), level)[..., 0]


def evaluate(level: Level, csr: CSR, x, nthreads: int = 1, canonical: bool = False):
    """Values f (planes (m,)) and Jacobian J (planes (m, n)) + (eval, grad) counts."""
    c = csr if canonical else csr.canonical()
    m, n = len(c.poly_ptr) - 1, c.n_vars
    X = to_aos(x, level)
    f = np.empty((m, level.es))
    J = np.empty((m, n, level.es))
    counts = np.zeros(2, np.int64)
    coeffs = to_aos(c.coeffs, level)
    rc = lib().or_evaluate(level.nc, int(level.cplx), m, n, _p(c.poly_ptr), _p(c.mon_ptr), _p(c.var_idx),
                           _p(c.exps), _p(coeffs), _p(X), _p(f), _p(J), _p(counts), nthreads)
    assert rc == 0
    return to_planes(f, level), to_planes(J, level), (int(counts[0]), int(counts[1]))


class Breakdown(ArithmeticError):
    def __init__(self, k, rkk, thr):
        super().__init__(f"MGS breakdown at column {k}")
        self.k, self.rkk, self.threshold = k, rkk, thr


class Singular(ArithmeticError):
    def __init__(self, j):
        super().__init__(f"zero diagonal entry at index {j}")
        self.index = j


def _raise(rc, info):
    if rc == 1:
        raise Breakdown(int(info[0]), float(info[1]), float(info[2]))
    if rc == 2:
        raise Singular(int(info[0]))
    assert rc == 0, rc


def mgs_qr(level: Level, aug, nthreads: int = 1):
    """Q (planes (m, n)), R (planes (n+1, n+1)) of [A b] (mgs.py:145-221)."""
    A = to_aos(aug, level)
    m, n1 = A.shape[:2]
    n = n1 - 1
    Q = np.empty((m, n, level.es))
    R = np.empty((n1, n1, level.es))
    info = np.zeros(4)
    rc = lib().or_mgs_qr(level.nc, int(level.cplx), m, n, _p(A), _p(Q), _p(R), _p(info), nthreads)
    _raise(rc, info)
    return to_planes(Q, level), to_planes(R, level)


def back_substitute(level: Level, R_aug):
    """x of R x = y with y = R[:n, n] (mgs.py:229-247)."""
    Ra = to_aos(R_aug, level)
    n = Ra.shape[0] - 1
    x = np.empty((n, level.es))
    info = np.zeros(4)
    rc = lib().or_back_substitute(level.nc, int(level.cplx), n, _p(Ra), _p(x), _p(info))
    _raise(rc, info)
    return to_planes(x, level)


def least_squares(level: Level, aug, nthreads: int = 1):
    A = to_aos(aug, level)
    m, n1 = A.shape[:2]
    n = n1 - 1
    Q = np.empty((m, n, level.es))
    R = np.empty((n1, n1, level.es))
    x = np.empty((n, level.es))
    z = np.zeros(1)
    info = np.zeros(4)
    rc = lib().or_least_squares(level.nc, int(level.cplx), m, n, _p(A), _p(Q), _p(R), _p(x), _p(z), _p(info),
                                nthreads)
    _raise(rc, info)
    return to_planes(x, level), float(z[0]), to_planes(Q, level), to_planes(R, level)


def newton_step(level: Level, csr: CSR, x, nthreads: int = 1, canonical: bool = False):
    """(x_next, f, dx) planes of one Gauss-Newton step (newton.py:82-103)."""
    c = csr if canonical else csr.canonical()
    m, n = len(c.poly_ptr) - 1, c.n_vars
    X = to_aos(x, level)
    f = np.empty((m, level.es))
    dx = np.empty((n, level.es))
    xn = np.empty((n, level.es))
    info = np.zeros(4)
    counts = np.zeros(2, np.int64)
    coeffs = to_aos(c.coeffs, level)
    rc = lib().or_newton_step(level.nc, int(level.cplx), m, n, _p(c.poly_ptr), _p(c.mon_ptr), _p(c.var_idx),
                              _p(c.exps), _p(coeffs), _p(X), _p(f), _p(dx), _p(xn), _p(info), _p(counts),
                              nthreads)
    _raise(rc, info)
    return to_planes(xn, level), to_planes(f, level), to_planes(dx, level)


# -- Newton driver with the reference's trace (newton.py:33-132) -----------------

def _render(comps) -> str:
    """render_decimal (xprec.py:406-420) of a real value given by components."""
    from decimal import Decimal, localcontext
    from fractions import Fraction
    if len(comps) == 1:
        return repr(float(comps[0]))
    fr = sum((Fraction(c) for c in comps), Fraction(0))
    if fr == 0:
        return "0.0"
    with localcontext() as ctx:
        ctx.prec = 32 if len(comps) == 2 else 64
        return format(Decimal(fr.numerator) / Decimal(fr.denominator), "E").replace("E", "e")


def _scalar_json(level: Level, comps):
    nc = level.nc
    if level.cplx:
        return [_render(comps[:nc]), _render(comps[nc:])]
    return _render(comps)


def _to_float(comps) -> float:
    import math
    if len(comps) == 1:
        return float(comps[0])
    if len(comps) == 2:
        return comps[0] + comps[1]
    return math.fsum(comps)


def inf_norm(level: Level, arr) -> float:
    """max over float(modulus(v)) (newton.py:33-34; xprec.py:327-328, 361-363)."""
    if level.cplx:
        mod = vec_op(Level(level.base, False), "sqrt", vec_op(level, "abs2", arr))
    else:
        mod = np.array(arr, copy=True)
        neg = mod[0] < 0.0
        mod[:, neg] = -mod[:, neg]
    cols = mod.reshape(level.nc, -1).T.tolist()
    return max((_to_float(c) for c in cols), default=0.0)


def run_newton_trace(level: Level, csr: CSR, x0, max_iters: int, tol=None, nthreads: int = 1):
    """(json_lines, x_final planes, converged) exactly as run_newton + to_json_lines."""
    import json
    c = csr.canonical()
    x = np.asarray(x0)
    lines = []
    converged = False
    for it in range(1, max_iters + 1):
        xn, f, dx = newton_step(level, c, x, nthreads=nthreads, canonical=True)
        entry = {
            "iter": it,
            "f_norm": inf_norm(level, f),
            "dx_norm": inf_norm(level, dx),
            "b0": _scalar_json(level, (-f[..., 0]).reshape(-1).tolist()),
            "dx0": _scalar_json(level, dx[..., 0].reshape(-1).tolist()),
            "x0": _scalar_json(level, xn[..., 0].reshape(-1).tolist()),
        }
        lines.append(json.dumps(entry) + "\n")
        x = xn
        t = tol if tol is not None else 10.0 * level.eps * (1.0 + inf_norm(level, x))
        if entry["dx_norm"] <= t:
            converged = True
            break
    return "".join(lines), x, converged
