"""Vectorised component arithmetic on the GPU (mirror of polynewt.varith).

Arrays keep the reference's component-plane layout (varith.py:3-8, 73): a
real array at precision nc has a leading component axis of length nc; a
complex one has leading shape (2, nc).  Every operation runs as an sm_100a
element-wise kernel (``pn_vec_op`` / ``pn_tree_sum``) replaying the
reference's exact binary64 sequence, so results are bit-identical to
``polynewt.varith.VecContext``.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .xprec import Complex, PrecisionLevel, level_of

_OPS = {"add": _lib.OP_ADD, "sub": _lib.OP_SUB, "mul": _lib.OP_MUL, "div": _lib.OP_DIV}


class VecContext:
    """Element-wise operations for one precision level (real or complex)."""

    def __init__(self, level: PrecisionLevel):
        self.level = level
        self.nc = level.ncomp
        self.cplx = level.cplx
        self.eps = level.eps
        self.cshape = (2, self.nc) if self.cplx else (self.nc,)
        self.rshape = (self.nc,)

    # -- construction ------------------------------------------------------

    def zeros(self, shape) -> np.ndarray:
        if isinstance(shape, int):
            shape = (shape,)
        return np.zeros(self.cshape + tuple(shape))

    def from_scalars(self, values) -> np.ndarray:
        """Nested list of scalars -> component array, data axes trailing."""
        def rec(v):
            if isinstance(v, list):
                return [rec(x) for x in v]
            return self.level.to_components(v)
        arr = np.asarray(rec(values), dtype=np.float64)
        arr = np.moveaxis(arr, -1, 0)
        return np.ascontiguousarray(arr.reshape(self.cshape + arr.shape[1:]))

    def to_scalar(self, arr):
        return self.level.from_components(np.asarray(arr).reshape(-1).tolist())

    def to_scalars(self, arr) -> list:
        flat = np.asarray(arr).reshape((-1,) + np.asarray(arr).shape[len(self.cshape):])
        return [self.level.from_components(flat[:, i].tolist()) for i in range(flat.shape[1])]

    # -- device execution --------------------------------------------------

    def _run(self, op: int, a, b=None, a_real=False, b_real=False, out_real=False):
        a = np.asarray(a, dtype=np.float64)
        ashape = self.rshape if a_real else self.cshape
        dshape = a.shape[len(ashape):]
        if b is not None:
            b = np.asarray(b, dtype=np.float64)
            bshape = self.rshape if b_real else self.cshape
            dshape = np.broadcast_shapes(dshape, b.shape[len(bshape):])
            b = np.ascontiguousarray(np.broadcast_to(b, bshape + tuple(dshape)))
        a = np.ascontiguousarray(np.broadcast_to(a, ashape + tuple(dshape)))
        n = int(np.prod(dshape)) if dshape else 1
        out = np.empty((self.rshape if out_real else self.cshape) + tuple(dshape))
        if n:
            rc = _lib.load().pn_vec_op(self.nc, int(self.cplx), op, n, _lib.ptr(a), _lib.ptr(b), _lib.ptr(out), None)
            _lib.check(rc)
        return out

    # -- arithmetic --------------------------------------------------------

    def add(self, a, b):
        return self._run(_lib.OP_ADD, a, b)

    def sub(self, a, b):
        return self._run(_lib.OP_SUB, a, b)

    def mul(self, a, b):
        return self._run(_lib.OP_MUL, a, b)

    def div(self, a, b):
        return self._run(_lib.OP_DIV, a, b)

    def neg(self, a):
        return -np.asarray(a)

    def conj(self, a):
        if not self.cplx:
            return a
        a = np.asarray(a)
        return np.stack((a[0], -a[1]))

    def div_real(self, a, r):
        """Divide by a real value (component array without the re/im axis)."""
        return self._run(_lib.OP_DIV_REAL, a, r, b_real=True)

    def abs2(self, a):
        """Squared modulus as a real component array."""
        return self._run(_lib.OP_ABS2, a, out_real=True)

    def modulus(self, a):
        """Field modulus (xprec.modulus) as a real component array."""
        return self._run(_lib.OP_MODULUS, a, out_real=True)

    def sqrt_real(self, r):
        return self._run(_lib.OP_SQRT, r, a_real=True, out_real=True)

    def real_embed(self, r):
        if not self.cplx:
            return r
        r = np.asarray(r)
        return np.stack((r, np.zeros_like(r)))

    def real_part(self, a):
        return a[0] if self.cplx else a

    # -- reductions --------------------------------------------------------

    def tree_sum(self, a, axis: int):
        """Balanced pairwise sum over one data axis, fixed canonical order."""
        a = np.asarray(a, dtype=np.float64)
        k = len(self.cshape)
        moved = np.moveaxis(a, axis + k, -1)
        rest = moved.shape[k:-1]
        n = moved.shape[-1]
        flat = np.ascontiguousarray(moved.reshape(self.cshape + (-1, n)))
        out = np.empty(self.cshape + (flat.shape[k],))
        lib = _lib.load()
        for i in range(flat.shape[k]):
            src = np.ascontiguousarray(flat[..., i, :])
            dst = np.empty(self.cshape + (1,))
            _lib.check(lib.pn_tree_sum(self.nc, int(self.cplx), n, _lib.ptr(src), _lib.ptr(dst), None))
            out[..., i] = dst[..., 0]
        return out.reshape(self.cshape + rest)

    def float_approx(self, a) -> np.ndarray:
        if self.cplx:
            return a[0][0] + 1j * a[1][0]
        return a[0]


def promote(arr: np.ndarray, src: PrecisionLevel, dst: PrecisionLevel) -> np.ndarray:
    """Exact embedding of a component array into a wider precision."""
    if dst.ncomp < src.ncomp or dst.cplx != src.cplx:
        raise ValueError("promotion must widen the precision")
    if dst.ncomp == src.ncomp:
        return arr
    nc_axis = 1 if src.cplx else 0
    pad = [(0, 0)] * arr.ndim
    pad[nc_axis] = (0, dst.ncomp - src.ncomp)
    return np.pad(arr, pad)


# -- scalar arithmetic (used by the scalar classes in xprec) ------------------

def _scalar_level(a, b) -> PrecisionLevel:
    la = level_of(a) if not isinstance(a, (int, float)) else None
    lb = level_of(b) if not isinstance(b, (int, float)) else None
    if la is None and lb is None:
        return PrecisionLevel("d", False)
    base = (la or lb).base
    cplx = (la is not None and la.cplx) or (lb is not None and lb.cplx)
    return PrecisionLevel(base, cplx)


def _is_cplx(x) -> bool:
    return hasattr(x, "re") and hasattr(x, "im")


def scalar_op(name: str, a, b):
    """One field operation on two scalars, run on the GPU.

    Mixed complex/real operands follow xprec.Complex (xprec.py:287-322): the
    real operand acts on each part (add/sub touch only the real part), and
    real / complex promotes the real to a complex with zero imaginary part."""
    from .xprec import DomainError, is_zero, zero_like
    level = _scalar_level(a, b)
    if _is_cplx(a) != _is_cplx(b) and level.cplx:
        if _is_cplx(a):  # Complex (op) real
            if name in ("add", "sub"):
                return Complex(scalar_op(name, a.re, b), a.im)
            return Complex(scalar_op(name, a.re, b), scalar_op(name, a.im, b))
        # real (op) Complex: __radd__ / __rmul__ are the Complex methods,
        # __rsub__ is (-self) + other, __rtruediv__ promotes the real
        if name == "add":
            return Complex(scalar_op("add", b.re, a), b.im)
        if name == "mul":
            return Complex(scalar_op("mul", b.re, a), scalar_op("mul", b.im, a))
        if name == "sub":
            return Complex(scalar_op("add", -b.re, a), -b.im)
        a = Complex(a if not isinstance(a, (int, float)) or level.base == "d" else level.field(float(a)),
                    zero_like(b.re))
    if name == "div" and is_zero(b):
        raise DomainError(f"{level.name} division by zero")
    ctx = VecContext(level)
    out = ctx._run(_OPS[name], ctx.from_scalars([a]), ctx.from_scalars([b]))
    return ctx.to_scalars(out)[0]


def scalar_sqrt(x):
    from .xprec import DomainError
    level = level_of(x)
    if x.comps[0] < 0.0:
        raise DomainError("square root of negative value")
    ctx = VecContext(level)
    return ctx.to_scalars(ctx.sqrt_real(ctx.from_scalars([x])))[0]


def scalar_modulus(x):
    level = level_of(x)
    ctx = VecContext(level)
    rl = PrecisionLevel(level.base, False)
    return rl.from_components(ctx.modulus(ctx.from_scalars([x]))[:, 0].tolist())
