"""Gauss-Newton iteration on polynomial systems, device resident
(mirror of polynewt.newton, newton.py:23-172).

Each step is one fused C-ABI call (``pn_newton_step``): evaluation and
Jacobian into [J | -f], MGS least squares, x + dx, and the field moduli of f,
dx and x_next.  The host only turns those moduli into the reference's float
norms (float(hi+lo) for dd, math.fsum for qd; xprec.py:153-154, 261-262) and
keeps the JSON trace.
"""

from __future__ import annotations

import ctypes
import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .evaldiff import OpCounter, PreparedSystem, evaluate_system, point_planes
from .mgs import TilingConfig
from .polyrep import Monomial, PackedSystem, PolySystem
from .varith import VecContext
from .xprec import Complex, PrecisionLevel, is_zero, render_decimal, to_float


@dataclass
class NewtonConfig:
    level: PrecisionLevel
    max_iters: int = 10
    tol: float | None = None      # None: 10 * eps * (1 + ||x||_inf) per step
    tiling: TilingConfig = field(default_factory=TilingConfig)
    delayed: bool = False
    parallel: bool = False


def inf_norm(values) -> float:
    """max |v| over scalars (newton.py:33-34); moduli computed on the GPU."""
    values = list(values)
    if not values:
        return 0.0
    if all(isinstance(v, (int, float)) for v in values):
        return max(abs(float(v)) for v in values)
    from .xprec import level_of
    level = level_of(values[0])
    return planes_inf_norm(VecContext(level).modulus(level.to_planes(values)), level)


def moduli_to_floats(mod: np.ndarray, level: PrecisionLevel) -> np.ndarray:
    """Real field moduli (nc, len) -> Python-float semantics of float(x)."""
    mod = np.asarray(mod).reshape(level.ncomp, -1)
    if level.ncomp == 1:
        return mod[0].copy()
    if level.ncomp == 2:
        return mod[0] + mod[1]
    return np.array([math.fsum(c) for c in mod.T.tolist()])


def planes_inf_norm(mod: np.ndarray, level: PrecisionLevel) -> float:
    f = moduli_to_floats(mod, level)
    return float(max(f.tolist(), default=0.0))


def _scalar_json(x):
    if hasattr(x, "re") and hasattr(x, "im"):
        return [render_decimal(x.re), render_decimal(x.im)]
    return render_decimal(x)


@dataclass
class TraceEntry:
    """One iteration: residual and correction norms plus probe entries."""

    iteration: int
    f_norm: float
    dx_norm: float
    b0: object
    dx0: object
    x0: object

    def to_json(self) -> str:
        return json.dumps({
            "iter": self.iteration,
            "f_norm": self.f_norm,
            "dx_norm": self.dx_norm,
            "b0": _scalar_json(self.b0),
            "dx0": _scalar_json(self.dx0),
            "x0": _scalar_json(self.x0),
        })


@dataclass
class IterationTrace:
    entries: list
    x: list
    converged: bool
    counter: OpCounter
    timings: dict

    def to_json_lines(self) -> str:
        return "".join(e.to_json() + "\n" for e in self.entries)


@dataclass
class StepResult:
    """Planes-level result of one device step."""

    x_next: np.ndarray
    f: np.ndarray
    dx: np.ndarray
    f_norm: float
    dx_norm: float
    x_norm: float
    z: float
    seconds: dict


def device_step(prep: PreparedSystem, x) -> StepResult:
    """One fused GPU Newton step on planes (host or device arrays)."""
    level = prep.level
    m, n = prep.n_eqs, prep.n_vars
    xp = point_planes(x, level, n)
    x_next = np.empty(level.cshape + (n,))
    f = np.empty(level.cshape + (m,))
    dx = np.empty(level.cshape + (n,))
    fm = np.empty((level.ncomp, m))
    dm = np.empty((level.ncomp, n))
    xm = np.empty((level.ncomp, n))
    info = _lib.NumInfo()
    rc = _lib.load().pn_newton_step(prep.handle, _lib.ptr(xp), _lib.ptr(x_next), _lib.ptr(f), _lib.ptr(dx),
                                    _lib.ptr(fm), _lib.ptr(dm), _lib.ptr(xm), ctypes.byref(info), None)
    _lib.check(rc, info)
    return StepResult(x_next, f, dx, planes_inf_norm(fm, level), planes_inf_norm(dm, level),
                      planes_inf_norm(xm, level), info.z,
                      {"evaluate": info.t_evaluate, "solve": info.t_solve, "update": info.t_update})


def _entry(level: PrecisionLevel, res: StepResult) -> TraceEntry:
    neg_f0 = -res.f[..., 0]
    return TraceEntry(iteration=0, f_norm=res.f_norm, dx_norm=res.dx_norm,
                      b0=level.from_components(neg_f0.reshape(-1).tolist()),
                      dx0=level.from_components(res.dx[..., 0].reshape(-1).tolist()),
                      x0=level.from_components(res.x_next[..., 0].reshape(-1).tolist()))


def _prepare(system, cfg: NewtonConfig | None = None) -> PreparedSystem:
    if isinstance(system, PreparedSystem):
        return system
    return PreparedSystem(system, cfg.level if cfg is not None else None)


def newton_step(prep, x, cfg: NewtonConfig):
    """One correction: returns (x_next, entry, counter, phase_seconds)."""
    prep = _prepare(prep, cfg)
    res = device_step(prep, x)
    x_next = prep.level.from_planes(res.x_next)
    return x_next, _entry(prep.level, res), prep.counts(), res.seconds


def run_newton(system, x0, cfg: NewtonConfig) -> IterationTrace:
    """Iterate until the correction norm drops under tolerance (newton.py:106-132)."""
    prep = _prepare(system, cfg)
    level = prep.level
    x = point_planes(x0, level)
    entries = []
    counter = OpCounter()
    timings = {"evaluate": 0.0, "solve": 0.0, "update": 0.0}
    converged = False
    step_counts = prep.counts()
    for it in range(1, cfg.max_iters + 1):
        res = device_step(prep, x)
        x = res.x_next
        entry = _entry(level, res)
        entry.iteration = it
        entries.append(entry)
        counter.merge(step_counts)
        for k, v in res.seconds.items():
            timings[k] += v
        tol = cfg.tol
        if tol is None:
            tol = 10.0 * cfg.level.eps * (1.0 + res.x_norm)
        if entry.dx_norm <= tol:
            converged = True
            break
    timings["total"] = sum(timings.values())
    return IterationTrace(entries, level.from_planes(x), converged, counter, timings)


def _shift_values(level: PrecisionLevel, f: np.ndarray, t) -> np.ndarray:
    """-(t * f_i) on the GPU, with the reference's operand semantics
    (newton.py:145: t * fz, Complex.__rmul__ for a real t)."""
    ctx = VecContext(level)
    m = f.shape[-1]
    if level.cplx and not (hasattr(t, "re") and hasattr(t, "im")):
        rlevel = PrecisionLevel(level.base, False)
        rctx = VecContext(rlevel)
        tp = np.repeat(rlevel.to_planes([t]), m, axis=-1)
        prod = np.stack((rctx.mul(f[0], tp), rctx.mul(f[1], tp)))
    else:
        tp = np.repeat(level.to_planes([t]), m, axis=-1)
        prod = ctx.mul(tp, f)
    return -prod


def homotopy_start_system(system, z, t):
    """Shift each equation by -t * f_i(z) (newton.py:135-159).

    Works on a PolySystem (returns a PolySystem) or a PackedSystem (returns a
    PackedSystem); f(z), t*f and const + shift all run on the GPU."""
    packed = system if isinstance(system, PackedSystem) else PackedSystem.from_system(system)
    level = packed.level
    prep = PreparedSystem(packed)
    ev = evaluate_system(prep, z)
    shift = _shift_values(level, ev.f, t)
    ctx = VecContext(level)
    m = packed.n_eqs
    # locate constant terms (at most one per polynomial)
    const_idx = np.full(m, -1, dtype=np.int64)
    ks = np.diff(packed.mon_ptr)
    for i in range(m):
        lo, hi = packed.poly_ptr[i], packed.poly_ptr[i + 1]
        consts = np.nonzero(ks[lo:hi] == 0)[0]
        if len(consts) > 1:
            raise ValueError("duplicate constant term")
        if len(consts):
            const_idx[i] = lo + consts[0]
    total = shift.copy()
    have = const_idx >= 0
    if have.any():
        cc = packed.coeffs[..., const_idx[have]]
        total[..., have] = ctx.add(cc, shift[..., have])
    flat_total = total.reshape(level.es, m)
    keep_const = ~np.all(flat_total == 0.0, axis=0)
    if not isinstance(system, PackedSystem):
        polys = []
        for i, poly in enumerate(system.polys):
            terms = [mon for mon in poly if mon.exponents != ()]
            if keep_const[i]:
                terms.append(Monomial(level.from_components(flat_total[:, i].tolist()), ()))
            polys.append(terms)
        return PolySystem(system.n_vars, polys)
    # packed: rebuild CSR with the constant appended last in each polynomial
    # (vectorised: drop the old constants, insert the new ones at the ends)
    pp = np.asarray(packed.poly_ptr, np.int64)
    coef = packed.coeffs.reshape(level.es, -1)
    keep = ks != 0
    poly_of = np.repeat(np.arange(m), np.diff(pp))
    kept_per_poly = np.bincount(poly_of[keep], minlength=m)
    ends = np.concatenate(([0], np.cumsum(kept_per_poly)))[1:]  # end of each poly among the kept monomials
    add = np.nonzero(keep_const)[0]
    new_ks = np.insert(ks[keep], ends[add], 0)
    new_coef = np.insert(coef[:, keep], ends[add], flat_total[:, add], axis=1)
    added = np.concatenate(([0], np.cumsum(keep_const.astype(np.int64))))
    poly_ptr = np.concatenate(([0], np.cumsum(kept_per_poly))) + added
    mon_ptr = np.concatenate(([0], np.cumsum(new_ks)))
    return PackedSystem(level, packed.n_vars, poly_ptr.astype(np.int32), mon_ptr.astype(np.int32),
                        np.asarray(packed.var_idx, np.int32).copy(), np.asarray(packed.exps, np.int32).copy(),
                        np.ascontiguousarray(new_coef.reshape(level.cshape + (new_coef.shape[1],))))


def convergence_ratio(trace: IterationTrace, floor: float = 0.0) -> list:
    """Quadratic-convergence quotients dx_{k+1} / dx_k^2 above a floor."""
    norms = [e.dx_norm for e in trace.entries if e.dx_norm > floor]
    out = []
    for a, b in zip(norms, norms[1:]):
        out.append(b / (a * a) if a > 0.0 else math.inf)
    return out
