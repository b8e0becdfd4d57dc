"""Least squares by modified Gram-Schmidt on [A b], on the GPU
(mirror of polynewt.mgs, mgs.py:145-305).

The factorisation runs as the right-looking sweep kernels of ``pn_mgs_qr``;
back substitution as ``pn_back_substitute``.  Results are bit-identical to
the reference for every tiling capacity, with or without delayed
normalisation (the reference's variants are bit-identical to each other,
mgs.py:72-108 of its tests), so those options are accepted and have no
numerical effect.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .varith import VecContext
from .xprec import PrecisionLevel


class MgsBreakdownError(ArithmeticError):
    """Rank deficiency at working precision: r_kk at or below threshold."""

    def __init__(self, k: int, rkk: float, threshold: float):
        super().__init__(f"MGS breakdown at column {k}: r_kk={rkk:.3e} <= {threshold:.3e}")
        self.k = k
        self.rkk = rkk
        self.threshold = threshold


class SingularMatrixError(ArithmeticError):
    def __init__(self, index: int):
        super().__init__(f"zero diagonal entry at index {index}")
        self.index = index


@dataclass(frozen=True)
class TilingConfig:
    """Row-tile capacity K; L = ceil(m/K) rounds per inner product."""

    K: int | None = None

    def capacity(self, m: int) -> int:
        if self.K is None:
            return m
        if self.K < 1:
            raise ValueError("tile capacity K must be >= 1")
        return min(self.K, m)

    def rounds(self, m: int) -> int:
        k = self.capacity(m)
        return (m + k - 1) // k

    def tiles(self, m: int):
        k = self.capacity(m)
        return [(lo, min(lo + k, m)) for lo in range(0, m, k)]


@dataclass
class AugmentedMatrix:
    """[A b] as a component array, data axes (rows, n+1 columns)."""

    ctx: VecContext
    data: np.ndarray

    @property
    def m(self) -> int:
        return self.data.shape[-2]

    @property
    def n(self) -> int:
        return self.data.shape[-1] - 1

    @classmethod
    def from_scalars(cls, level: PrecisionLevel, a_rows, b) -> "AugmentedMatrix":
        ctx = VecContext(level)
        rows = [list(r) + [bv] for r, bv in zip(a_rows, b)]
        return cls(ctx, ctx.from_scalars(rows))

    @classmethod
    def from_arrays(cls, ctx: VecContext, a: np.ndarray, b: np.ndarray) -> "AugmentedMatrix":
        return cls(ctx, np.concatenate((a, b[..., None]), axis=-1))


@dataclass
class QRFactors:
    """Q (m x n) and the (n+1)x(n+1) triangular factor of [A b]."""

    ctx: VecContext
    Q: np.ndarray
    R: np.ndarray

    @property
    def n(self) -> int:
        return self.Q.shape[-1]

    @property
    def y(self) -> np.ndarray:
        return self.R[..., : self.n, self.n]

    @property
    def z(self) -> float:
        zc = self.ctx.real_part(self.R[..., self.n, self.n])
        return float(zc[0])

    @property
    def r_square(self) -> np.ndarray:
        return self.R[..., : self.n, : self.n]


BREAKDOWN_FACTOR = 1.0  # mgs.py:118-119; applied inside the sweep kernels


def _level(ctx: VecContext):
    return ctx.nc, int(ctx.cplx)


def mgs_qr(aug: AugmentedMatrix, cfg: TilingConfig = TilingConfig(), delayed: bool = False,
           parallel: bool = False) -> QRFactors:
    """Modified Gram-Schmidt on [A b] (mgs.py:145-221)."""
    ctx = aug.ctx
    m, n = aug.m, aug.n
    if not (m >= n >= 1):
        raise ValueError(f"need m >= n >= 1, got m={m}, n={n}")
    cfg.capacity(m)  # validates K like the reference
    data = np.ascontiguousarray(aug.data, dtype=np.float64)
    Q = np.empty(ctx.cshape + (m, n))
    R = np.empty(ctx.cshape + (n + 1, n + 1))
    info = _lib.NumInfo()
    nc, cplx = _level(ctx)
    rc = _lib.load().pn_mgs_qr(nc, cplx, m, n, _lib.ptr(data), _lib.ptr(Q), _lib.ptr(R), ctypes.byref(info), None)
    _lib.check(rc, info)
    return QRFactors(ctx, Q, R)


def mgs_qr_delayed(aug: AugmentedMatrix, cfg: TilingConfig = TilingConfig(), parallel: bool = False) -> QRFactors:
    return mgs_qr(aug, cfg, delayed=True, parallel=parallel)


def _augmented_r(R: np.ndarray, y: np.ndarray, ctx: VecContext) -> np.ndarray:
    """Embed (R, y) into the (n+1)x(n+1) layout pn_back_substitute expects."""
    n = y.shape[-1]
    Ra = np.zeros(ctx.cshape + (n + 1, n + 1))
    Ra[..., :n, :n] = R[..., :n, :n]
    Ra[..., :n, n] = y
    return Ra


def back_substitute(R: np.ndarray, y: np.ndarray, ctx: VecContext) -> np.ndarray:
    """Solve R x = y (mgs.py:229-247)."""
    n = y.shape[-1]
    Ra = _augmented_r(np.asarray(R), np.asarray(y), ctx)
    x = np.empty(ctx.cshape + (n,))
    info = _lib.NumInfo()
    nc, cplx = _level(ctx)
    rc = _lib.load().pn_back_substitute(nc, cplx, n, _lib.ptr(Ra), _lib.ptr(x), ctypes.byref(info), None)
    _lib.check(rc, info)
    return x


def back_substitute_staged(R: np.ndarray, y: np.ndarray, ctx: VecContext, cfg: TilingConfig = TilingConfig(),
                           parallel: bool = False) -> np.ndarray:
    """Staged tile solve (mgs.py:250-289); bit-identical to back_substitute."""
    cfg.tiles(y.shape[-1])
    return back_substitute(R, y, ctx)


@dataclass
class LeastSquaresResult:
    x: np.ndarray
    z: float
    factors: QRFactors = field(repr=False)


def least_squares_solve(aug: AugmentedMatrix, cfg: TilingConfig = TilingConfig(), delayed: bool = False,
                        parallel: bool = False) -> LeastSquaresResult:
    """Minimize ||b - Ax||_2 via MGS QR of [A b] and back substitution."""
    ctx = aug.ctx
    m, n = aug.m, aug.n
    if not (m >= n >= 1):
        raise ValueError(f"need m >= n >= 1, got m={m}, n={n}")
    cfg.capacity(m)
    data = np.ascontiguousarray(aug.data, dtype=np.float64)
    Q = np.empty(ctx.cshape + (m, n))
    R = np.empty(ctx.cshape + (n + 1, n + 1))
    x = np.empty(ctx.cshape + (n,))
    z = ctypes.c_double(0.0)
    info = _lib.NumInfo()
    nc, cplx = _level(ctx)
    rc = _lib.load().pn_least_squares(nc, cplx, m, n, _lib.ptr(data), _lib.ptr(x), ctypes.byref(z), _lib.ptr(Q),
                                      _lib.ptr(R), ctypes.byref(info), None)
    _lib.check(rc, info)
    return LeastSquaresResult(x=x, z=float(z.value), factors=QRFactors(ctx, Q, R))


def residual_check(A: np.ndarray, Q: np.ndarray, R: np.ndarray, level) -> float:
    """max componentwise |A - QR| in the next-higher precision (mgs.py:311-357).

    d and dd factorizations are re-checked on the GPU in dd and qd arithmetic
    with the reference's operation order, so the result is the reference's
    float bit for bit.  Quad-double factorizations (320-bit mpfr in the
    reference) are checked by exact fixed-point accumulation of every
    component product on the GPU; the float agrees with the reference's
    unless the value lies within ~1e-30 relative of a rounding boundary.
    R may be the (n+1)x(n+1) augmented factor; only its leading n x n block
    is used."""
    n = Q.shape[-1]
    m = Q.shape[-2]
    a = np.ascontiguousarray(A[..., :m, :n], dtype=np.float64)
    q = np.ascontiguousarray(Q, dtype=np.float64)
    r = np.ascontiguousarray(R[..., :n, :n], dtype=np.float64)
    out = ctypes.c_double(0.0)
    rc = _lib.load().pn_residual_check(level.ncomp, int(level.cplx), m, n, _lib.ptr(a), _lib.ptr(q), _lib.ptr(r),
                                       ctypes.byref(out), None)
    _lib.check(rc)
    return float(out.value)
