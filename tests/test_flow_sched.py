"""The quad-double flow kernel's schedule knobs change only who applies which
sweep when, never the operation sequence of a column (mgs.py:171-215): Q, R,
x and z must stay bit-identical to the oracle under every column ownership
(PN_FLOW_OWN=smsnake|rr|snake|<table file>) and hold rule (PN_FLOW_HOLD), and a table
that leaves a column unowned is refused instead of stalling the pivots."""

import os
from contextlib import contextmanager

import numpy as np
import pytest

import oracle
from conftest import level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu

M, N = 400, 330  # n + 1 > 296 CTAs: several columns per CTA


@contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.fixture(scope="module")
def case():
    L = oracle_level("cqd")
    rng = np.random.default_rng(M * N)
    aug = rng.uniform(-1, 1, L.cshape + (M, N + 1))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    aug = np.ascontiguousarray(aug)
    return aug, oracle.least_squares(L, aug, nthreads=os.cpu_count() or 1)


def _solve(aug):
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    return least_squares_solve(AugmentedMatrix(VecContext(level_from_name("cqd")), aug))


def _check(res, ref):
    x, z, Q, R = ref
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z


@pytest.mark.parametrize("own,hold,pick", [("rr", "0", "0"), ("rr", "3", "1"), ("snake", "1", "0"),
                                           ("snake", "0", "1"), ("rr", "1", "0"), ("smsnake", "1", "1"),
                                           ("smsnake", "0", "0")])
def test_flow_schedules_bit_identical(gpu, case, own, hold, pick):
    aug, ref = case
    with env(PN_MGS_MODE="flow", PN_FLOW_OWN=own, PN_FLOW_HOLD=hold, PN_FLOW_PICK=pick):
        _check(_solve(aug), ref)


