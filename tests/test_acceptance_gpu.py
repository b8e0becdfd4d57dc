"""The reference's acceptance criteria 6-8 (pkg/tests/test_acceptance.py:183-257)
re-run on the GPU path at the reference's own scale.

The published log (pkg/test_output.txt:264-266) prints the final residuals
|f| = 8.4e-31 / 1.6e-30 / 3.5e-30 (Chandrasekhar H-equation, complex dd,
n = 64/128/256, 6 iterations), 7.4e-63 (real qd, n = 127, 7 iterations) and
9.3e-31 (cyclic-64 homotopy, complex dd, t = 0.99, 7 iterations).  The GPU
runs must print the same numbers, and their JSONL traces must be
byte-identical to the oracle's (which is pinned to the reference)."""

import os

import numpy as np
import pytest

import oracle
from conftest import level_from_name

pytestmark = pytest.mark.gpu


def _oracle_trace(system, level, x0, max_iters, tol):
    from paper_1402_2626_b200.polyrep import PackedSystem
    p = PackedSystem.from_system(system, level)
    L = oracle.Level(level.base, level.cplx)
    lines, _, _ = oracle.run_newton_trace(L, oracle.CSR.from_packed(p), level.to_planes(list(x0)), max_iters,
                                          tol=tol, nthreads=os.cpu_count() or 1)
    return lines


def _final_norm(system, level, x):
    from paper_1402_2626_b200.evaldiff import evaluate_system
    from paper_1402_2626_b200.newton import inf_norm
    return inf_norm(evaluate_system(system, level.to_planes(list(x))).values)


@pytest.mark.parametrize("n,published", [(64, "8.4e-31"), (128, "1.6e-30"), (256, "3.5e-30")])
def test_criterion6_chandrasekhar_cdd(gpu, n, published):
    from paper_1402_2626_b200.generators import chandrasekhar_start, chandrasekhar_system
    from paper_1402_2626_b200.newton import NewtonConfig, run_newton
    level = level_from_name("cdd")
    system = chandrasekhar_system(n, level)
    x0 = chandrasekhar_start(n, level)
    trace = run_newton(system, x0, NewtonConfig(level=level, max_iters=6, tol=0.0))
    assert f"{_final_norm(system, level, trace.x):.1e}" == published
    assert trace.to_json_lines() == _oracle_trace(system, level, x0, 6, 0.0)


def test_criterion7_chandrasekhar_real_qd(gpu):
    from paper_1402_2626_b200.generators import chandrasekhar_start, chandrasekhar_system
    from paper_1402_2626_b200.newton import NewtonConfig, run_newton
    level = level_from_name("rqd")
    system = chandrasekhar_system(127, level)
    x0 = chandrasekhar_start(127, level)
    trace = run_newton(system, x0, NewtonConfig(level=level, max_iters=7, tol=0.0))
    assert f"{_final_norm(system, level, trace.x):.1e}" == "7.4e-63"
    assert trace.to_json_lines() == _oracle_trace(system, level, x0, 7, 0.0)


def test_criterion8_cyclic64_homotopy_cdd(gpu):
    from paper_1402_2626_b200.generators import cyclic_n_roots, random_unit_point
    from paper_1402_2626_b200.newton import NewtonConfig, homotopy_start_system, run_newton
    level = level_from_name("cdd")
    system = cyclic_n_roots(64, level)
    z = random_unit_point(64, 2718, level)
    shifted = homotopy_start_system(system, level.to_planes(z), level.from_float(0.99))
    trace = run_newton(shifted, z, NewtonConfig(level=level, max_iters=7))
    assert len(trace.entries) <= 7
    assert f"{_final_norm(shifted, level, trace.x):.1e}" == "9.3e-31"
    assert trace.to_json_lines() == _oracle_trace(shifted, level, z, 7, None)


@pytest.mark.parametrize("base,resid,ortho", [("d", "9.5e-16", "2.2e-16"), ("dd", "7.9e-32", "3.5e-32"),
                                              ("qd", "7.2e-65", "2.4e-65")])
def test_criterion5_mgs_qr_accuracy(gpu, base, resid, ortho):
    """Criterion 5 (test_acceptance.py:129-180) at its printed shape 100 x 64:
    |A - QR| in the next precision (qd: exact fixed-point accumulation vs the
    reference's 320-bit mpfr; its float is pinned in residuals.json) and
    |Q^H Q - I| from tree_sum of conj(q_i) q_j, on the GPU."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, mgs_qr, residual_check
    from paper_1402_2626_b200.varith import VecContext
    from paper_1402_2626_b200.xprec import precision_level
    level = precision_level(base, True)
    ctx = VecContext(level)
    m, n = 100, 64
    rng = np.random.default_rng(1000 + m + n)  # random_aug (tests/test_mgs.py:14-24)
    data = np.zeros(ctx.cshape + (m, n + 1))
    data[0, 0] = rng.uniform(-1.0, 1.0, (m, n + 1))
    data[1, 0] = rng.uniform(-1.0, 1.0, (m, n + 1))
    f = mgs_qr(AugmentedMatrix(ctx, data))
    got = residual_check(data[..., :, :n], f.Q, f.r_square, level)
    assert f"{got:.1e}" == resid
    if base == "qd":
        import json
        from conftest import GOLDEN
        with open(os.path.join(GOLDEN, "residuals.json")) as fh:
            assert got == json.load(fh)["criterion5_cqd_100x64"]
    outer = ctx.mul(ctx.conj(np.ascontiguousarray(np.broadcast_to(f.Q[..., :, :, None], ctx.cshape + (m, n, n)))),
                    np.ascontiguousarray(np.broadcast_to(f.Q[..., :, None, :], ctx.cshape + (m, n, n))))
    gram = ctx.float_approx(ctx.tree_sum(outer, axis=0))
    assert f"{float(np.max(np.abs(gram - np.eye(n)))):.1e}" == ortho


def test_criterion9_structure_checks(gpu):
    """Criterion 9 (test_acceptance.py:259-287): cyclic monomial counts
    n^2 - n + 2 for n = 2..64, and Jacobians of Chandrasekhar n = 32 and
    cyclic-12 (real double) equal binary64 central differences at 1e-6, all
    evaluated by the GPU path."""
    from paper_1402_2626_b200.evaldiff import evaluate_system
    from paper_1402_2626_b200.generators import (chandrasekhar_system, cyclic_n_roots, cyclic_packed,
                                                 random_point)
    cdd = level_from_name("cdd")
    D = level_from_name("rd")
    for n in range(2, 65):
        assert cyclic_n_roots(n, cdd).monomial_count() == n * n - n + 2
        assert cyclic_packed(n, cdd).monomials == n * n - n + 2
    h = 2.0 ** -26
    for system, point in [(chandrasekhar_system(32, D), random_point(32, 5, D)),
                          (cyclic_n_roots(12, D), random_point(12, 6, D))]:
        n = system.n_vars
        ev = evaluate_system(system, point)
        J = np.asarray(ev.jacobian, dtype=np.float64)
        # every +-h perturbation of every variable in one batched evaluation
        X = np.repeat(np.asarray(point, np.float64)[None, :], 2 * n, axis=0)
        X[np.arange(n), np.arange(n)] += h
        X[n + np.arange(n), np.arange(n)] -= h
        from paper_1402_2626_b200.batch import evaluate_batch
        from paper_1402_2626_b200.evaldiff import PreparedSystem
        F = evaluate_batch(PreparedSystem(system), X[None])[0]          # (2n, m)
        want = ((F[:n] - F[n:]) / (2.0 * h)).T                            # (m, n)
        assert np.all(np.abs(J - want) <= 1e-6 * (np.abs(want) + 1.0))


@pytest.mark.parametrize("lv", ["cdd", "rqd", "cd"])
def test_chandrasekhar_packed_equals_object_builder(gpu, lv):
    """The numpy CSR builder of the H-equation (paper scale) equals
    PackedSystem.from_system of the Monomial builder, component for
    component (weights and -(c w) formed on the GPU in both)."""
    from paper_1402_2626_b200.generators import chandrasekhar_packed, chandrasekhar_system
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name(lv)
    for n in (1, 2, 7, 33):
        a = chandrasekhar_packed(n, level)
        b = PackedSystem.from_system(chandrasekhar_system(n, level), level)
        for x, y in ((a.poly_ptr, b.poly_ptr), (a.mon_ptr, b.mon_ptr), (a.var_idx, b.var_idx), (a.exps, b.exps)):
            assert np.array_equal(x, y)
        assert np.array_equal(a.coeffs, b.coeffs)
        assert np.array_equal(np.signbit(a.coeffs), np.signbit(b.coeffs))
