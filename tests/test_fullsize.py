"""Parity at the BASELINE.json configurations' full sizes.

The oracle cannot evaluate a dim-1024 system in seconds, but every row of
f and J depends only on its own polynomial and x (evaldiff.py:252-265), so
rows sampled from the full C2 system are compared exactly.  MGS runs at the
full C3 size in double-double (the C oracle takes seconds there); the batched
C5 path is compared start by start with single runs."""

import os

import numpy as np
import pytest

import oracle
from conftest import level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu


def _point(level, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, level.cshape + (n,)) * rng.choice([-1.0, 1.0], level.cshape + (n,))
    x.reshape(-1, n)[[i for i in range(level.es) if i % level.ncomp != 0]] *= 1e-17
    return np.ascontiguousarray(x)


@pytest.mark.parametrize("lv", ["cqd", "cdd", "cd"])
def test_c2_full_system_rows_vs_oracle(gpu, lv):
    """C2: F(1024, 1024, 32) evaluated in full on the GPU (TMA-staged trees);
    8 sampled rows of f and J against the oracle, bit for bit."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(1024, 1024, 32, level, seed=2024)
    x = _point(level, 1024, 11)
    ev = evaluate_system(PreparedSystem(p), x)
    rows = [0, 1, 255, 511, 512, 777, 1000, 1023]
    sub = oracle.CSR.from_packed(p).rows(rows)
    f, J, _ = oracle.evaluate(oracle_level(lv), sub, x, nthreads=os.cpu_count() or 1)
    assert same(ev.f[..., rows], f)
    assert same(ev.J[..., rows, :], J)


def test_c3_full_size_least_squares_cdd(gpu):
    """C3: MGS least squares on a 1024 x 1025 complex double-double [A b]."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level("cdd")
    rng = np.random.default_rng(1024)
    aug = rng.uniform(-1, 1, L.cshape + (1024, 1025))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    aug = np.ascontiguousarray(aug)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name("cdd")), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=os.cpu_count() or 1)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z


def test_c3_cqd_least_squares_512(gpu):
    """The cqd MGS at half the C3 size (the full cqd oracle run takes ~20 s x 8)."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level("cqd")
    rng = np.random.default_rng(512)
    aug = rng.uniform(-1, 1, L.cshape + (520, 513))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    aug = np.ascontiguousarray(aug)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name("cqd")), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=os.cpu_count() or 1)
    assert same(res.factors.R, R)
    assert same(res.x, x)
    assert res.z == z


def test_c5_batch_starts_match_single_runs(gpu):
    """C5 system F(256, 256, 32) cdd: 64 batched homotopy starts; four of
    them re-run one at a time through run_newton give identical x, iteration
    counts and status."""
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.newton import NewtonConfig, homotopy_start_system, run_newton
    level = level_from_name("cdd")
    p = random_sparse_system(256, 256, 32, level, seed=2024)
    B = 64
    rng = np.random.default_rng(7)
    theta = rng.uniform(0.0, 2.0 * np.pi, (B, 256))
    Z = np.zeros(level.cshape + (B, 256))
    Z[0, 0], Z[1, 0] = np.cos(theta), np.sin(theta)
    t = level.from_float(0.99)
    system, consts = homotopy_batch(p, Z, t)
    res = run_newton_batch(PreparedSystem(system), Z, consts, max_iters=8)
    assert (res.status == 0).sum() >= B // 2  # quadratic convergence from these starts
    for b in (0, 17, 40, 63):
        zb = np.ascontiguousarray(Z[..., b, :])
        tr = run_newton(homotopy_start_system(p, zb, t), zb, NewtonConfig(level=level, max_iters=8))
        assert same(res.x[..., b, :], level.to_planes(tr.x)), b
        assert res.iters[b] == len(tr.entries), b
        assert res.status[b] == (0 if tr.converged else 1), b


def test_headline_cqd_newton_step_full_size(gpu):
    """The bench workload itself: one complex quad-double Newton step on
    F(1024, 1024, 32) (eval + diff + 1024 x 1025 MGS + back substitution +
    update) against the oracle's full step (about 25 s of CPU on the box)."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.newton import device_step
    level = level_from_name("cqd")
    p = random_sparse_system(1024, 1024, 32, level, seed=2024)
    x = _point(level, 1024, 3)
    res = device_step(PreparedSystem(p), x)
    xn, f, dx = oracle.newton_step(oracle_level("cqd"), oracle.CSR.from_packed(p), x,
                                   nthreads=os.cpu_count() or 1)
    assert same(res.f, f)
    assert same(res.dx, dx)
    assert same(res.x_next, xn)


@pytest.mark.parametrize("m,n", [(1536, 64), (700, 300)])
def test_cqd_tail_split_vs_oracle(gpu, m, n):
    """Row-split tail of the quad-double MGS (k_mgs_tail): m = 1536 puts every
    column in the tail (six 256-row parts); m = 700 splits the work between the
    flow kernel and the tail with a ragged third part."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level("cqd")
    rng = np.random.default_rng(m + n)
    aug = rng.uniform(-1, 1, L.cshape + (m, n + 1))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    aug = np.ascontiguousarray(aug)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name("cqd")), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=os.cpu_count() or 1)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z
