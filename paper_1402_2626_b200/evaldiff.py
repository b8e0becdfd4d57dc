"""Evaluation and differentiation of polynomial systems on the GPU
(mirror of polynewt.evaldiff, evaldiff.py:183-266).

``PreparedSystem`` uploads the packed, canonically ordered supports once
(``pn_system_create``); ``evaluate_system`` then runs the power-table,
product-tree/gradient and accumulation kernels (``pn_evaldiff``).  Values and
Jacobian come back as component planes (``.f``, ``.J``); the reference's
scalar lists ``.values`` / ``.jacobian`` are built from them on first use.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .polyrep import PackedSystem, PolySystem, decompose, system_level
from .xprec import PrecisionLevel


@dataclass
class OpCounter:
    """Multiplication tallies split by phase (evaldiff.py:21-30)."""

    eval_mults: int = 0
    grad_mults: int = 0

    def merge(self, other: "OpCounter"):
        self.eval_mults += other.eval_mults
        self.grad_mults += other.grad_mults


class PreparedSystem:
    """A system resident on the GPU in canonical order (evaldiff.py:183-194).

    Accepts a PolySystem (own or reference objects) or a PackedSystem."""

    def __init__(self, system, level: PrecisionLevel | None = None):
        _lib.require_gpu()
        if isinstance(system, PackedSystem):
            packed = system
        else:
            packed = PackedSystem.from_system(system, level or system_level(system))
        self.packed = packed
        self.level = packed.level
        self.n_vars = packed.n_vars
        self.n_eqs = packed.n_eqs
        self._source = packed.source
        self._handle = ctypes.c_void_p()
        lib = _lib.load()
        rc = lib.pn_system_create(self.level.ncomp, int(self.level.cplx), packed.n_eqs, packed.n_vars,
                                  packed.monomials, packed.support, _lib.ptr(packed.poly_ptr),
                                  _lib.ptr(packed.mon_ptr), _lib.ptr(packed.var_idx), _lib.ptr(packed.exps),
                                  _lib.ptr(packed.coeffs), int(packed.canonical), ctypes.byref(self._handle))
        _lib.check(rc)

    @property
    def handle(self):
        return self._handle

    @property
    def system(self) -> PolySystem:
        """The canonicalised system (evaldiff.py:191-192)."""
        src = self._source if self._source is not None else self.packed.to_system()
        return src.canonicalized()

    @property
    def terms(self) -> list:
        return [[(mon.coeff, decompose(mon)) for mon in poly] for poly in self.system.polys]

    def canonical_order(self) -> np.ndarray:
        perm = np.empty(self.packed.monomials, dtype=np.int64)
        _lib.check(_lib.load().pn_system_canonical_order(self._handle, _lib.ptr(perm)))
        return perm

    def counts(self) -> OpCounter:
        c = _lib.Counts()
        _lib.check(_lib.load().pn_system_counts(self._handle, ctypes.byref(c)))
        return OpCounter(int(c.eval_mults), int(c.grad_mults))

    def stats(self) -> _lib.SystemStats:
        s = _lib.SystemStats()
        _lib.check(_lib.load().pn_system_get_stats(self._handle, ctypes.byref(s)))
        return s

    def rows_plan(self) -> dict:
        """The row-evaluation plan of this system (pn_system_plan_info)."""
        pi = _lib.PlanInfo()
        _lib.check(_lib.load().pn_system_plan_info(self._handle, ctypes.byref(pi)))
        return {"ok": bool(pi.rows_ok), "K": pi.K, "chunk": pi.chunk, "depth": pi.depth, "nchunks": pi.nchunks}

    def close(self):
        if getattr(self, "_handle", None) and self._handle.value:
            _lib.load().pn_system_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class SystemEvaluation:
    f: np.ndarray                 # planes cshape + (m,)
    J: np.ndarray                 # planes cshape + (m, n)
    counter: OpCounter
    seconds: float
    level: PrecisionLevel = field(repr=False, default=None)
    _values: list = field(default=None, repr=False)
    _jacobian: list = field(default=None, repr=False)

    @property
    def values(self) -> list:
        if self._values is None:
            self._values = self.level.from_planes(self.f)
        return self._values

    @property
    def jacobian(self) -> list:
        if self._jacobian is None:
            m, n = self.J.shape[-2:]
            flat = self.level.from_planes(self.J.reshape(self.level.cshape + (m * n,)))
            self._jacobian = [flat[i * n:(i + 1) * n] for i in range(m)]
        return self._jacobian


def point_planes(point, level: PrecisionLevel, n: int | None = None, batch: int | None = None) -> np.ndarray:
    """A point (list of scalars or a planes array / torch tensor) as
    contiguous float64 planes of shape level.cshape + (n,) -- or
    level.cshape + (batch, n) for a batch of points.  The C ABI reads exactly
    that many doubles from the pointer, so a wrong shape or dtype is refused
    here (ValueError) instead of reading past the end of the buffer."""
    if isinstance(point, np.ndarray):
        x = np.ascontiguousarray(point, dtype=np.float64)
    elif hasattr(point, "data_ptr"):
        import torch
        if point.dtype != torch.float64 or not point.is_contiguous():
            raise ValueError("point tensor must be contiguous float64 planes")
        x = point
    else:
        x = level.to_planes(list(point))
    want = tuple(level.cshape) + (() if batch is None else (batch,)) + (() if n is None else (n,))
    got = tuple(x.shape)
    if n is not None and (len(got) != len(want) or got != want):
        raise ValueError(f"point planes have shape {got}, expected {want} for this system and precision")
    return x


def evaluate_system(system, point, counter: OpCounter | None = None,
                    parallel: bool = False) -> SystemEvaluation:
    """Values and Jacobian of a system at one point (evaldiff.py:215-266).

    ``parallel`` is accepted for API compatibility; the GPU result is the
    same bit pattern either way (the reduction order is fixed)."""
    t0 = time.perf_counter()
    prep = system if isinstance(system, PreparedSystem) else PreparedSystem(system)
    level = prep.level
    n = prep.n_vars
    if isinstance(point, (list, tuple)) and len(point) != n:
        raise ValueError(f"point dimension {len(point)} != n_vars {n}")
    x = point_planes(point, level, n)
    m = prep.n_eqs
    f = np.empty(level.cshape + (m,))
    J = np.empty(level.cshape + (m, n))
    c = _lib.Counts()
    rc = _lib.load().pn_evaldiff(prep.handle, _lib.ptr(x), _lib.ptr(f), _lib.ptr(J), ctypes.byref(c), None)
    _lib.check(rc)
    cnt = OpCounter(int(c.eval_mults), int(c.grad_mults))
    if counter is not None:
        counter.merge(cnt)
    return SystemEvaluation(f, J, cnt, time.perf_counter() - t0, level)
