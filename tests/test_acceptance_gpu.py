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
