"""Batched Newton runs over independent start points
and their sharding across GPUs.

A batch is B runs of ``run_newton`` (newton.py:106-132) on the homotopy start
systems ``homotopy_start_system(system, z_b, t)`` (newton.py:135-159): all
starts share the supports and coefficients and differ only in the constant
term of each polynomial.  The GPU keeps one resident system and swaps the m
constants per start (``pn_newton_batch``); results are bit-identical to the
one-at-a-time path.  Starts are independent units: ``shard_range`` splits
them across ranks with no collective on the data path, and ``gather_batch``
collects status, iteration counts and final iterates once at the end
(NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .evaldiff import PreparedSystem, point_planes
from .polyrep import PackedSystem
from .varith import VecContext
from .xprec import PrecisionLevel

STATUS = {0: "converged", 1: "max_iters", 2: "breakdown", 3: "singular"}


@dataclass
class BatchResult:
    x: np.ndarray        # planes cshape + (B, n)
    iters: np.ndarray    # int32 (B,)
    status: np.ndarray   # int32 (B,)


def shard_range(B: int, world: int, rank: int) -> tuple:
    """Contiguous block of start indices owned by `rank` (balanced)."""
    base, extra = divmod(B, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def evaluate_batch(prep: PreparedSystem, X: np.ndarray) -> np.ndarray:
    """f(x_b) for X planes cshape + (B, n) -> planes cshape + (B, m)."""
    level = prep.level
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim < 2:
        raise ValueError("X must be planes cshape + (B, n)")
    B = X.shape[-2]
    X = point_planes(X, level, prep.n_vars, B)
    F = np.empty(level.cshape + (B, prep.n_eqs))
    _lib.check(_lib.load().pn_evaldiff_batch(prep.handle, B, _lib.ptr(X), _lib.ptr(F), None))
    return F


def _with_constant_terms(packed: PackedSystem):
    """Copy of the system in which every polynomial has a constant term (a
    placeholder 1 where the base has none, appended at the polynomial's end:
    canonical order puts it first anyway); returns it and, per polynomial,
    the index of the base constant monomial or -1.  Vectorised over the CSR."""
    level = packed.level
    m = packed.n_eqs
    pp = np.asarray(packed.poly_ptr, np.int64)
    ks = np.diff(np.asarray(packed.mon_ptr, np.int64))
    is_const = ks == 0
    poly_of = np.repeat(np.arange(m), np.diff(pp))
    nconst = np.bincount(poly_of[is_const], minlength=m) if m else np.zeros(0, np.int64)
    if (nconst > 1).any():
        raise ValueError("duplicate constant term")
    base_const = np.full(m, -1, dtype=np.int64)
    base_const[poly_of[is_const]] = np.nonzero(is_const)[0]
    lacking = np.nonzero(nconst == 0)[0]
    # insert one empty monomial at the end of every polynomial lacking a constant
    new_ks = np.insert(ks, pp[lacking + 1], 0)
    mon_ptr = np.concatenate(([0], np.cumsum(new_ks))).astype(np.int32)
    added = np.zeros(m + 1, np.int64)
    added[1:] = np.cumsum(nconst == 0)
    poly_ptr = (pp + added).astype(np.int32)
    coef = packed.coeffs.reshape(level.es, -1)
    placeholder = np.zeros((level.es, 1))
    placeholder[0, 0] = 1.0  # replaced per start
    newc = np.insert(coef, pp[lacking + 1], placeholder, axis=1) if len(lacking) else coef.copy()
    out = PackedSystem(level, packed.n_vars, poly_ptr, mon_ptr, np.asarray(packed.var_idx, np.int32).copy(),
                       np.asarray(packed.exps, np.int32).copy(),
                       np.ascontiguousarray(newc.reshape(level.cshape + (newc.shape[1],))))
    return out, base_const


def homotopy_batch(packed: PackedSystem, Z: np.ndarray, t):
    """Per-start constants of homotopy_start_system(system, z_b, t) for all b.

    Returns (system_with_constants, consts planes cshape + (B, m)).  The
    arithmetic (f(z_b), -(t*f), const + shift) runs on the GPU with the
    reference's operand order."""
    level = packed.level
    B = Z.shape[-2]
    m = packed.n_eqs
    base_prep = PreparedSystem(packed)
    F = evaluate_batch(base_prep, Z)                      # cshape + (B, m)
    Ff = F.reshape(level.cshape + (B * m,))
    ctx = VecContext(level)
    if level.cplx and not (hasattr(t, "re") and hasattr(t, "im")):
        rl = PrecisionLevel(level.base, False)
        rctx = VecContext(rl)
        tp = np.repeat(rl.to_planes([t]), B * m, axis=-1)
        prod = np.stack((rctx.mul(Ff[0], tp), rctx.mul(Ff[1], tp)))
    else:
        tp = np.repeat(level.to_planes([t]), B * m, axis=-1)
        prod = ctx.mul(tp, Ff)
    shift = (-prod).reshape(level.cshape + (B, m))
    system, base_const = _with_constant_terms(packed)
    consts = shift.copy()
    have = base_const >= 0
    if have.any():
        cc = packed.coeffs[..., base_const[have]]                       # cshape + (h,)
        cc = np.broadcast_to(cc[..., None, :], level.cshape + (B, int(have.sum())))
        sub = np.ascontiguousarray(shift[..., have])
        consts[..., have] = ctx.add(np.ascontiguousarray(cc), sub)
    zero = np.all(consts.reshape(level.es, B, m) == 0.0, axis=0)
    if zero.any():
        raise ValueError("a homotopy constant is exactly zero; the reference would drop that term "
                         "(run those starts individually)")
    return system, np.ascontiguousarray(consts)


def run_newton_batch(prep: PreparedSystem, X0: np.ndarray, consts: np.ndarray | None = None,
                     max_iters: int = 10, tol: float | None = None) -> BatchResult:
    """B independent Newton runs on the GPU (pn_newton_batch)."""
    level = prep.level
    X0 = np.ascontiguousarray(X0, dtype=np.float64)
    if X0.ndim < 2:
        raise ValueError("X0 must be planes cshape + (B, n)")
    B = X0.shape[-2]
    X0 = point_planes(X0, level, prep.n_vars, B)
    if consts is not None:
        consts = point_planes(consts, level, prep.n_eqs, B)
    X = np.empty_like(X0)
    iters = np.zeros(B, np.int32)
    status = np.zeros(B, np.int32)
    c = None if consts is None else np.ascontiguousarray(consts, dtype=np.float64)
    rc = _lib.load().pn_newton_batch(prep.handle, B, _lib.ptr(X0), _lib.ptr(c), max_iters,
                                     -1.0 if tol is None else float(tol), _lib.ptr(X), _lib.ptr(iters),
                                     _lib.ptr(status), None)
    _lib.check(rc)
    del level
    return BatchResult(X, iters, status)


def gather_batch(shard: BatchResult, B: int, group=None) -> BatchResult:
    """All-gather the shards of a batch (one collective at the end of the run:
    NCCL over NVLink on GPUs, gloo on CPU).  Every rank gets the full result."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    lo, hi = shard_range(B, world, rank)
    assert shard.x.shape[-2] == hi - lo
    cshape = shard.x.shape[:-2]
    n = shard.x.shape[-1]
    width = -(-B // world)  # pad every shard to the same count
    es = int(np.prod(cshape))

    def pad(a, cols):
        out = np.zeros(a.shape[:-1] + (width,) if cols is None else (width,) + a.shape[1:], a.dtype)
        if cols is None:
            out[..., : a.shape[-1]] = a
        else:
            out[: a.shape[0]] = a
        return out
    xs = np.moveaxis(shard.x.reshape(es, hi - lo, n), 1, 0)               # (count, es, n)
    payload = {"x": pad(xs, 1), "iters": pad(shard.iters, None), "status": pad(shard.status, None)}
    out = {}
    for key, arr in payload.items():
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        bufs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(bufs, t, group=group)
        parts = []
        for r, buf in enumerate(bufs):
            rlo, rhi = shard_range(B, world, r)
            a = buf.cpu().numpy()
            parts.append(a[..., : rhi - rlo] if a.ndim == 1 else a[: rhi - rlo])
        out[key] = np.concatenate(parts, axis=0 if key == "x" else -1)
    x = np.moveaxis(out["x"], 0, 1).reshape(cshape + (B, n))
    return BatchResult(np.ascontiguousarray(x), out["iters"].astype(np.int32), out["status"].astype(np.int32))


class NcclComm:
    """The C ABI's communicator (pn_comm_*): NCCL straight from the library,
    no torch.distributed.  ``uid`` is the 128-byte id of
    NcclComm.unique_id() created on rank 0 and handed to every rank."""

    def __init__(self, world: int, rank: int, uid: bytes, device: int = 0):
        if len(uid) != 128:
            raise ValueError("a communicator id is 128 bytes")
        self.world, self.rank = world, rank
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
        _lib.check(_lib.load().pn_comm_init(world, rank, ctypes.cast(buf, ctypes.c_void_p), device,
                                            ctypes.byref(self._h)))

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_ubyte * 128)()
        _lib.check(_lib.load().pn_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        return bytes(buf)

    def gather_batch(self, shard: BatchResult, B: int, level: PrecisionLevel) -> BatchResult:
        """pn_batch_allgather: every rank's shard_range block -> the full batch."""
        n = shard.x.shape[-1]
        x = np.ascontiguousarray(shard.x, dtype=np.float64)
        it = np.ascontiguousarray(shard.iters, dtype=np.int32)
        stt = np.ascontiguousarray(shard.status, dtype=np.int32)
        lo, hi = shard_range(B, self.world, self.rank)
        if x.shape != level.cshape + (hi - lo, n) or it.shape != (hi - lo,) or stt.shape != (hi - lo,):
            raise ValueError("shard does not match shard_range(B, world, rank)")
        X = np.empty(level.cshape + (B, n))
        I = np.empty(B, np.int32)
        S = np.empty(B, np.int32)
        _lib.check(_lib.load().pn_batch_allgather(self._h, level.ncomp, int(level.cplx), n, B, _lib.ptr(x),
                                                   _lib.ptr(it), _lib.ptr(stt), _lib.ptr(X), _lib.ptr(I),
                                                   _lib.ptr(S), None))
        return BatchResult(X, I, S)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().pn_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _prepare_shard(packed: PackedSystem, Zs: np.ndarray, t):
    system, consts = homotopy_batch(packed, Zs, t)
    return PreparedSystem(system), consts


def run_batched(packed: PackedSystem, Z: np.ndarray, t, max_iters: int = 10, tol: float | None = None,
                group=None, prepare=None, solve=None, comm: NcclComm | None = None):
    """Config C5 on this rank: the B starts Z (planes cshape + (B, n)) are
    split by shard_range over the process group, the rank builds the
    homotopy constants of its shard (homotopy_start_system semantics,
    newton.py:135-159), runs its batch of run_newton (newton.py:106-132)
    and all ranks all_gather status, iterations and final x once (the only
    collective).  Returns (shard_result, full_result, (lo, hi)).

    ``prepare(packed, Zs, t) -> (prep, consts)`` and ``solve(prep, Zs,
    consts, max_iters=, tol=) -> BatchResult`` default to the GPU path; the
    CPU tests substitute stubs to check the orchestration with gloo.  With
    ``comm`` (an NcclComm) the gather is the C ABI's pn_batch_allgather
    instead of torch.distributed."""
    import torch.distributed as dist
    init = dist.is_available() and dist.is_initialized()
    world = comm.world if comm else dist.get_world_size(group) if init else 1
    rank = comm.rank if comm else dist.get_rank(group) if init else 0
    B = Z.shape[-2]
    lo, hi = shard_range(B, world, rank)
    Zs = np.ascontiguousarray(Z[..., lo:hi, :])
    prep, consts = (prepare or _prepare_shard)(packed, Zs, t)
    shard = (solve or run_newton_batch)(prep, Zs, consts, max_iters=max_iters, tol=tol)
    if comm is not None:
        full = comm.gather_batch(shard, B, packed.level if packed is not None else prep.level)
    else:
        full = gather_batch(shard, B, group) if init else shard
    return shard, full, (lo, hi)

