"""k_mono_tree_tma with padded support rows (opt-in PN_TREE_PAD=1, read at
launch): rows staged one bulk copy each at a bank-spreading stride.  Same
arithmetic as the contiguous layout, so f and J must match the oracle
(evaldiff.py:215-266) bit for bit, with unit and non-unit exponents."""

import os
from contextlib import contextmanager

import numpy as np
import pytest

import oracle
from conftest import level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu


@contextmanager
def env(name, value):
    old = os.environ.get(name)
    os.environ[name] = value
    try:
        yield
    finally:
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old


def _point(level, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, level.cshape + (n,)) * rng.choice([-1.0, 1.0], level.cshape + (n,))
    x.reshape(-1, n)[[i for i in range(level.es) if i % level.ncomp != 0]] *= 1e-17
    return np.ascontiguousarray(x)


@pytest.mark.parametrize("pad", ["1", "0"])
@pytest.mark.parametrize("lv,n,T,k,maxexp", [("cqd", 64, 40, 32, 1), ("cdd", 96, 37, 12, 2), ("rdd", 80, 50, 20, 3),
                                             ("cdd", 70, 33, 32, 2), ("cqd", 50, 21, 5, 1)])
def test_tree_pad_vs_oracle(gpu, pad, lv, n, T, k, maxexp):
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(n, T, k, level, seed=n * T + k, maxexp=maxexp)
    x = _point(level, n, 9)
    with env("PN_TREE_PAD", pad):
        ev = evaluate_system(PreparedSystem(p), x)
    f, J, _ = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x, nthreads=8)
    assert same(ev.f, f)
    assert same(ev.J, J)
